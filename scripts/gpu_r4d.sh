#!/bin/bash
# default green partition: GPU suite, round sweep, bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_partition.py -q -p no:cacheprovider -rf > gpurun_out/d_part.log 2>&1
tail -3 gpurun_out/d_part.log
O=gpurun_out/green_d.jsonl; : > $O
timeout 200 python scripts/split_sms_sweep.py >> $O 2>&1
for v in 0 44 48 64; do SSD_B200_GREEN=$v timeout 200 python scripts/split_sms_sweep.py >> $O 2>&1; done
cat $O
timeout 600 python bench.py > gpurun_out/d_bench.jsonl 2> gpurun_out/d_bench.err; tail -c 3000 gpurun_out/d_bench.jsonl
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/d_pytest_gpu.log 2>&1; tail -5 gpurun_out/d_pytest_gpu.log
