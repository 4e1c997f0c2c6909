#!/bin/bash
# green partition: segment profile and the co-resident GEMM budget
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/green_b.jsonl; : > $O
timeout 200 python scripts/round_profile.py >> $O 2>&1
for v in 48 52 56 60 64; do SSD_B200_GREEN=$v timeout 200 python scripts/round_profile.py >> $O 2>&1; done
for v in 48 56 64; do SSD_B200_GREEN=$v SSD_B200_CORUN_SMALL_GEMM_MB=0 timeout 200 python scripts/round_profile.py >> $O 2>&1; done
SSD_B200_GREEN=56 SSD_B200_CORUN_SMALL_GEMM_MB=40 timeout 200 python scripts/round_profile.py >> $O 2>&1
SSD_B200_GREEN=56 SSD_B200_CORUN_ATTN_KB=100 timeout 200 python scripts/round_profile.py >> $O 2>&1
cat $O
