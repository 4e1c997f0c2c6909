#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_paged.py tests/test_gpu_bench_shapes.py -m gpu -q -p no:cacheprovider -x > gpurun_out/a_tests.log 2>&1
timeout 300 python scripts/fwd_ablate.py d1,d5,d20,t1,t5 > gpurun_out/ablate_a.jsonl 2>&1
: > gpurun_out/rounds_a.jsonl; for i in 1 2; do timeout 300 python scripts/split_sms_sweep.py >> gpurun_out/rounds_a.jsonl 2>&1; done
timeout 300 python scripts/ktl.py d20 > gpurun_out/ktl_a.log 2>&1
tail -3 gpurun_out/a_tests.log; cat gpurun_out/ablate_a.jsonl gpurun_out/rounds_a.jsonl; sed -n 1,8p gpurun_out/ktl_a.log
