#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/rounds_z.jsonl
for env in "SSD_B200_SPLIT_SMS=0,0" "SSD_B200_SPLIT_SMS=120,0" "SSD_B200_SPLIT_SMS=96,0" "SSD_B200_SPLIT_SMS=74,0" "SSD_B200_VERIFY_AFTER_EXTEND=1" "SSD_B200_VERIFY_AFTER_EXTEND=1 SSD_B200_SPLIT_SMS=96,0"; do
  env $env timeout 300 python scripts/split_sms_sweep.py >> gpurun_out/rounds_z.jsonl 2>>gpurun_out/rounds_z.err
done
cat gpurun_out/rounds_z.jsonl
