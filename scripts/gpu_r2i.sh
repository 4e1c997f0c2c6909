#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for env in "SSD_B200_PK_CTAS=40" "SSD_B200_PK_CTAS=148"; do
  echo "== $env" >> gpurun_out/pk_dbg.log
  env $env timeout 120 python scripts/pk_check.py tiny >> gpurun_out/pk_dbg.log 2>&1
done
cat gpurun_out/pk_dbg.log
timeout 600 python scripts/pk_check.py llama8b_1b > gpurun_out/pk_1b.log 2>&1; echo "exit $?" >> gpurun_out/pk_1b.log
cat gpurun_out/pk_1b.log
