#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/alpha_sweep.py llama8b_1b 0.1,0.06,0.04,0.03,0.02 > gpurun_out/alpha.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_fwd.csv python scripts/prof_fwd.py t1,d20 > gpurun_out/prof_fwd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:gemm_tc_kernel<2, 16>' -s 8 -c 1 -o gpurun_out/prof_gu_t1 python scripts/prof_fwd.py t1 > gpurun_out/prof_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:gemm_tc_kernel<2, 32>' -s 8 -c 1 -o gpurun_out/prof_gu_d20 python scripts/prof_fwd.py d20 >> gpurun_out/prof_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention -s 8 -c 1 \
  -o gpurun_out/prof_attn_d20 python scripts/prof_fwd.py d20 >> gpurun_out/prof_full.log 2>&1
echo done >> gpurun_out/prof_full.log
tail -n 8 gpurun_out/alpha.log gpurun_out/prof_fwd.log gpurun_out/prof_full.log
