#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for part in v none; do for M in 5 20; do echo "== trace part $part M 5"; SSD_B200_LIB=$PWD/paper_2603_03251_b200/libssd_b200_trace.so SSD_B200_PROFILE_PART=$part timeout 300 python scripts/gemm_trace.py $M 2>&1 | tail -4; done; done > gpurun_out/j_trace.log
cat gpurun_out/j_trace.log
O=gpurun_out/j.jsonl; : > $O
timeout 300 python scripts/fwd_ablate.py t5,d5,d20 >> $O 2>&1
SSD_B200_PROFILE_PART=v timeout 300 python scripts/fwd_ablate.py t5 >> $O 2>&1
SSD_B200_PROFILE_PART=s timeout 300 python scripts/fwd_ablate.py d5,d20 >> $O 2>&1
timeout 300 python scripts/round_profile.py >> $O 2>&1
cat $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py -q -x -p no:cacheprovider 2>&1 | tail -3
