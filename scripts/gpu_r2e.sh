#!/bin/bash
# r02 call E: GPU tests; branch-step GEMM route (cluster split-K vs fused
# stream-K with atomics), whole-tile SwiGLU; colocated round; bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -rf --durations=8 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for env in "SSD_B200_SWIGLU_WHOLE=0" "SSD_B200_SWIGLU_WHOLE=1" "SSD_B200_CL_GEMM_MB=0" "SSD_B200_CL_GEMM_MB=0 SSD_B200_SPEC_PRIO=1"; do
  env $env timeout 300 python scripts/fwd_ablate.py d1,d5,d20,t1,t5 >> gpurun_out/ablate.jsonl 2>>gpurun_out/ablate.err
  env $env timeout 300 python scripts/split_sms_sweep.py >> gpurun_out/rounds.jsonl 2>>gpurun_out/rounds.err
done
tail -n 4 gpurun_out/pytest_gpu.log; cat gpurun_out/ablate.jsonl gpurun_out/rounds.jsonl
