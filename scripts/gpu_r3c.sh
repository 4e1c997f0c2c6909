#!/bin/bash
# ncu evidence on the final kernels: launch lists of exactly one timed
# forward (d20 branch step: launches 520..634; t5 verify: 696..922), cold
# (default cache control) and warm (no flush between kernels: the DRAM
# traffic of the whole forward), and full captures of one layer's GEMMs of
# the d20 step (matches 130..133: QKV, O, gate/up, down).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 900 ncu --metrics $M --clock-control none -s 520 -c 115 --csv --log-file gpurun_out/launches_d20.csv python scripts/prof_fwd.py d20 > /dev/null 2>&1
timeout 900 ncu --metrics $M --cache-control none --clock-control none -s 520 -c 115 --csv --log-file gpurun_out/traffic_d20.csv python scripts/prof_fwd.py d20 > /dev/null 2>&1
timeout 900 ncu --metrics $M --clock-control none -s 696 -c 227 --csv --log-file gpurun_out/launches_t5.csv python scripts/prof_fwd.py t5 > /dev/null 2>&1
timeout 900 ncu --metrics $M --cache-control none --clock-control none -s 696 -c 227 --csv --log-file gpurun_out/traffic_t5.csv python scripts/prof_fwd.py t5 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 130 -c 4 -o gpurun_out/prof_gemm_d20 python scripts/prof_fwd.py d20 > /dev/null 2>&1
for f in launches_d20 traffic_d20 launches_t5 traffic_t5; do python scripts/launches.py gpurun_out/$f.csv | head -9; done
