#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/k.jsonl; : > $O
for v in 32 36 40 44 48 52 56; do SSD_B200_GREEN=$v timeout 300 python scripts/round_profile.py >> $O 2>&1; done
SSD_B200_GREEN=0 timeout 300 python scripts/round_profile.py >> $O 2>&1
cat $O
