#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/q3.jsonl; : > $O
timeout 300 python scripts/diag_tiny_logits.py >> $O 2>&1
SSD_B200_SWIGLU_WHOLE=0 timeout 300 python scripts/diag_tiny_logits.py >> $O 2>&1
SSD_B200_SWIGLU_REDUCE_UNITS=0 timeout 300 python scripts/diag_tiny_logits.py >> $O 2>&1
cat $O
