#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/launches_ar.csv \
  python scripts/profile_run.py --rounds 2 --what ar > gpurun_out/prof_ar.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 400 -c 3 \
  -o gpurun_out/prof_gemm_m1 python scripts/profile_run.py --rounds 1 --what ar >> gpurun_out/prof_ar.log 2>&1
echo done >> gpurun_out/prof_ar.log
