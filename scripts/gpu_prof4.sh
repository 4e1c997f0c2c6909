#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention -s 66 -c 1 \
  -o gpurun_out/prof_attn2 python scripts/profile_run.py --rounds 1 --what ar > gpurun_out/prof4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rmsnorm -s 130 -c 1 \
  -o gpurun_out/prof_norm python scripts/profile_run.py --rounds 1 --what ar >> gpurun_out/prof4.log 2>&1
echo done >> gpurun_out/prof4.log
