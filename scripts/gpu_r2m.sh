#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
DIAG_SEEDS=200,1200,2200 SSD_B200_DETERMINISTIC=0 timeout 600 python scripts/diag_width.py 33 > gpurun_out/diag_width.log 2>&1
DIAG_SEEDS=200,1200,2200 SSD_B200_DETERMINISTIC=1 timeout 600 python scripts/diag_width.py 33 >> gpurun_out/diag_width.log 2>&1
cat gpurun_out/diag_width.log
