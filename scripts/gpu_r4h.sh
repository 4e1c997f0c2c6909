#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in trace_mmaonly_c2; do
  echo "== $v part v M 5"; SSD_B200_LIB=$PWD/paper_2603_03251_b200/libssd_b200_$v.so SSD_B200_PROFILE_PART=v timeout 300 python scripts/gemm_trace.py 5 2>&1 | tail -5
done > gpurun_out/gemm_trace_c2.log
cat gpurun_out/gemm_trace_c2.log
