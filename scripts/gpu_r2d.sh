#!/bin/bash
# r02 call D: GPU tests (boundary API, reference cases through the C++ shim),
# fused residual epilogues with atomic split-K (vs SSD_B200_DETERMINISTIC=1),
# KTL timeline of the new forward, colocated round, bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rf --durations=8 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for env in "SSD_B200_DETERMINISTIC=1" "SSD_B200_DETERMINISTIC=0"; do
  env $env timeout 300 python scripts/fwd_ablate.py d1,d5,d20,t1,t5 >> gpurun_out/ablate.jsonl 2>>gpurun_out/ablate.err
  env $env timeout 300 python scripts/split_sms_sweep.py >> gpurun_out/rounds.jsonl 2>>gpurun_out/rounds.err
done
timeout 600 python scripts/ktl.py d1 d20 t1 > gpurun_out/ktl.log 2>&1; echo "ktl exit $?" >> gpurun_out/ktl.log
timeout 1200 python bench.py --steps 4 --warmup 2 > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
tail -n 4 gpurun_out/pytest_gpu.log gpurun_out/bench.log; cat gpurun_out/ablate.jsonl gpurun_out/rounds.jsonl
