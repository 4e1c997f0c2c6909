#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
# launch list of one 2-round SSD decode (+ prefill/initial draft)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ssd.csv \
  python scripts/profile_run.py --rounds 2 --what ssd > gpurun_out/prof_ssd.log 2>&1
echo "ncu list exit $?" >> gpurun_out/prof_ssd.log
# full capture of the top kernels: tcgen05 GEMM (branch step) and the M=1 GEMV
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 300 -c 2 \
  -o gpurun_out/prof_gemm_tc python scripts/profile_run.py --rounds 1 --what ssd > gpurun_out/prof_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:linear_cc_kernel -s 200 -c 2 \
  -o gpurun_out/prof_gemv python scripts/profile_run.py --rounds 1 --what ar >> gpurun_out/prof_full.log 2>&1
echo "ncu full exit $?" >> gpurun_out/prof_full.log
ls -la gpurun_out
