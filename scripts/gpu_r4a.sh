#!/bin/bash
# green-context SM partition sweep of the colocated SSD round (bench workload)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/green_a.jsonl
timeout 200 python scripts/split_sms_sweep.py >> gpurun_out/green_a.jsonl 2>&1
for v in 24 32 40 48 56 64 72 88; do
  SSD_B200_GREEN=$v timeout 200 python scripts/split_sms_sweep.py >> gpurun_out/green_a.jsonl 2>&1
done
for v in 40 56; do
  SSD_B200_GREEN=$v SSD_B200_VERIFY_AFTER_EXTEND=1 timeout 200 python scripts/split_sms_sweep.py >> gpurun_out/green_a.jsonl 2>&1
done
timeout 200 python scripts/split_sms_sweep.py >> gpurun_out/green_a.jsonl 2>&1
cat gpurun_out/green_a.jsonl
