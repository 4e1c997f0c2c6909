#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/diag_fanout.py 4 8 12 16 > gpurun_out/diag_fanout.log 2>&1; echo "exit $?" >> gpurun_out/diag_fanout.log
SSD_B200_DETERMINISTIC=1 timeout 900 python scripts/diag_fanout.py 16 > gpurun_out/diag_fanout_det.log 2>&1; echo "exit $?" >> gpurun_out/diag_fanout_det.log
cat gpurun_out/diag_fanout.log gpurun_out/diag_fanout_det.log
