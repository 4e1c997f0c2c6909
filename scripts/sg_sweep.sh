#!/bin/bash
cd "$(dirname "$0")/.."
for sg in 0 20 40; do
  echo "SMALL_GEMM_MB=$sg"; SSD_B200_SMALL_GEMM_MB=$sg timeout 300 python scripts/pf_sweep.py 16 2>&1 | tail -1
done
