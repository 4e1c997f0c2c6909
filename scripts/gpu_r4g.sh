#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for part in none v; do for M in 1 5; do
  echo "== part $part M $M"; SSD_B200_PROFILE_PART=$part timeout 300 python scripts/gemm_trace.py $M 2>&1 | tail -30
done; done > gpurun_out/gemm_trace_part.log
cat gpurun_out/gemm_trace_part.log
