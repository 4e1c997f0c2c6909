#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
# the AR step's first 4 GEMMs (QKV, O, gate/up, down at M=1) after 258 prefill GEMMs
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 258 -c 4 \
  -o gpurun_out/prof_gemm_m1 python scripts/profile_run.py --rounds 1 --what ar > gpurun_out/prof3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention -s 64 -c 1 \
  -o gpurun_out/prof_attn_m1 python scripts/profile_run.py --rounds 1 --what ar >> gpurun_out/prof3.log 2>&1
echo done >> gpurun_out/prof3.log
