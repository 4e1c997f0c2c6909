#!/bin/bash
# r02 call F (fresh container): full GPU tests, smoke, default bench, fwd ablation.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -rf --durations=12 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 300 python scripts/fwd_ablate.py d1,d5,d20,t1,t5 >> gpurun_out/ablate.jsonl 2>>gpurun_out/ablate.err
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
tail -n 6 gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.log; cat gpurun_out/ablate.jsonl
