#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python scripts/pk_check.py tiny > gpurun_out/pk_tiny.log 2>&1
timeout 600 python scripts/pk_check.py llama8b_1b > gpurun_out/pk_1b.log 2>&1
timeout 300 python scripts/pk_trace.py d1 d20 > gpurun_out/pk_trace.log 2>&1
cat gpurun_out/pk_tiny.log gpurun_out/pk_1b.log
