#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/n.jsonl; : > $O
SSD_B200_PROFILE_PART=s timeout 300 python scripts/fwd_ablate.py d5,d20 >> $O 2>&1
SSD_B200_SWIGLU_REDUCE_UNITS=0 SSD_B200_PROFILE_PART=s timeout 300 python scripts/fwd_ablate.py d5,d20 >> $O 2>&1
timeout 300 python scripts/fwd_ablate.py t5,d1,d5,d20 >> $O 2>&1
timeout 300 python scripts/round_profile.py >> $O 2>&1
cat $O
SSD_B200_PROFILE_PART=s timeout 600 python scripts/ktl.py d20 > gpurun_out/ktl_d20_s4.log 2>&1
head -8 gpurun_out/ktl_d20_s4.log; grep -n "embed        entry" -A16 gpurun_out/ktl_d20_s4.log | sed -n 9,17p
