#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/gemv_ablate.jsonl; : > $out
for i in 1 2; do timeout 300 python scripts/fwd_ablate.py t1,d1 >> $out 2>>gpurun_out/gemv.err; SSD_B200_GEMV_M=0 timeout 300 python scripts/fwd_ablate.py t1,d1 >> $out 2>>gpurun_out/gemv.err; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -q -x --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_gemv.log 2>&1
cat $out; tail -3 gpurun_out/gemv.err; tail -4 gpurun_out/pytest_gemv.log
