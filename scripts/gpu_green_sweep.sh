#!/bin/bash
# round time and in-graph segments under SM partitions (SSD_B200_GREEN),
# the extend-first ordering (SSD_B200_EXTEND_FULL) and the whole-device tail
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/green_sweep.jsonl; : > $O
timeout 120 python scripts/round_profile.py >> $O 2>&1
for v in 48 56 64 72 80; do SSD_B200_EXTEND_FULL=1 SSD_B200_GREEN=$v timeout 120 python scripts/round_profile.py >> $O 2>&1; done
SSD_B200_EXTEND_FULL=1 SSD_B200_GREEN=56 SSD_B200_GREEN_TAIL=3 timeout 120 python scripts/round_profile.py >> $O 2>&1
SSD_B200_EXTEND_FULL=1 SSD_B200_GREEN=64 SSD_B200_GREEN_TAIL=3 timeout 120 python scripts/round_profile.py >> $O 2>&1
timeout 120 python scripts/round_profile.py >> $O 2>&1
cat $O
