#!/bin/bash
# green partition x tail sweep (SMALL=0: full-budget GEMM configs)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/green_c.jsonl; : > $O
timeout 200 python scripts/split_sms_sweep.py >> $O 2>&1
export SSD_B200_CORUN_SMALL_GEMM_MB=0
for v in 52 56 60; do SSD_B200_GREEN=$v timeout 200 python scripts/split_sms_sweep.py >> $O 2>&1; done
for v in 56 64 72 80; do for t in 0 1 2 3; do
  SSD_B200_GREEN=$v SSD_B200_GREEN_TAIL=$t timeout 200 python scripts/split_sms_sweep.py >> $O 2>&1
done; done
cat $O
