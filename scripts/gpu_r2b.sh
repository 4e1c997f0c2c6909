#!/bin/bash
# r02 call B: GPU tests (pruned library, fp64 noise-floor logit checks), the
# real kernel timeline (KTL build) of the 1B / 8B forwards, forward ablation
# of the co-resident GEMM config, and the new multi-prompt bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rf --durations=10 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/ktl.py d1 d5 d20 t1 t5 > gpurun_out/ktl.log 2>&1; echo "ktl exit $?" >> gpurun_out/ktl.log
for sg in 0 2000; do
  SSD_B200_SMALL_GEMM_MB=$sg timeout 300 python scripts/fwd_ablate.py d1,d5,d20,t1,t5 >> gpurun_out/ablate.jsonl 2>>gpurun_out/ablate.err
done
timeout 1200 python bench.py --steps 4 --warmup 2 > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
tail -n 4 gpurun_out/pytest_gpu.log gpurun_out/bench.log; cat gpurun_out/ablate.jsonl
