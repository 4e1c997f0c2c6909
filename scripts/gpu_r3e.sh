#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_loops.py tests/test_gpu_bench_shapes.py tests/test_split_gpu.py tests/test_gpu_paged.py -m gpu -q -p no:cacheprovider -rf > gpurun_out/e_tests.log 2>&1
timeout 300 python scripts/fwd_ablate.py d1,d5,d20 > gpurun_out/ablate_e.jsonl 2>&1
SSD_B200_ATTN_QB=0 timeout 300 python scripts/fwd_ablate.py d20 >> gpurun_out/ablate_e.jsonl 2>&1
: > gpurun_out/rounds_e.jsonl; for i in 1 2; do timeout 300 python scripts/split_sms_sweep.py >> gpurun_out/rounds_e.jsonl 2>&1; done
SSD_B200_ATTN_QB=0 timeout 300 python scripts/split_sms_sweep.py >> gpurun_out/rounds_e.jsonl 2>&1
tail -4 gpurun_out/e_tests.log; cat gpurun_out/ablate_e.jsonl gpurun_out/rounds_e.jsonl
