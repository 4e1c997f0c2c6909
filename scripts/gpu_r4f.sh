#!/bin/bash
# forward timings on the partitions of the colocated round
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/part_fwd.jsonl; : > $O
timeout 300 python scripts/fwd_ablate.py t5,d5,d20 >> $O 2>&1
SSD_B200_PROFILE_PART=v timeout 300 python scripts/fwd_ablate.py t5 >> $O 2>&1
SSD_B200_PROFILE_PART=s timeout 300 python scripts/fwd_ablate.py d5,d20 >> $O 2>&1
SSD_B200_GREEN=74 SSD_B200_PROFILE_PART=v timeout 300 python scripts/fwd_ablate.py t5 >> $O 2>&1
SSD_B200_GREEN=74 SSD_B200_PROFILE_PART=s timeout 300 python scripts/fwd_ablate.py d5,d20 >> $O 2>&1
cat $O
SSD_B200_PROFILE_PART=v timeout 600 python scripts/ktl.py t5 > gpurun_out/ktl_t5_v.log 2>&1
SSD_B200_PROFILE_PART=s timeout 600 python scripts/ktl.py d20 > gpurun_out/ktl_d20_s.log 2>&1
head -12 gpurun_out/ktl_t5_v.log; head -12 gpurun_out/ktl_d20_s.log
