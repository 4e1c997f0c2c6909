#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SSD_B200_PROFILE_PART=s timeout 600 python scripts/ktl.py d20 > gpurun_out/ktl_d20_s3.log 2>&1
SSD_B200_PROFILE_PART=s timeout 600 python scripts/ktl.py d5 > gpurun_out/ktl_d5_s3.log 2>&1
head -9 gpurun_out/ktl_d20_s3.log; grep -n "embed        entry" -A16 gpurun_out/ktl_d20_s3.log | sed -n 9,17p
grep "launch  *[0-9]* " gpurun_out/ktl_d20_s3.log | head -8
head -9 gpurun_out/ktl_d5_s3.log
