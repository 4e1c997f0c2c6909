#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/rounds_w.jsonl; : > gpurun_out/ablate_w.jsonl
for env in "SSD_B200_SWIGLU_WHOLE_FRAC8=7" "SSD_B200_SWIGLU_WHOLE_FRAC8=6"; do
  env $env timeout 300 python scripts/fwd_ablate.py d1,d5,d20,t5 >> gpurun_out/ablate_w.jsonl 2>>gpurun_out/ablate_w.err
  env $env timeout 300 python scripts/split_sms_sweep.py >> gpurun_out/rounds_w.jsonl 2>>gpurun_out/rounds_w.err
done
timeout 600 python scripts/ktl.py d20 > gpurun_out/ktl_w.log 2>&1
cat gpurun_out/ablate_w.jsonl gpurun_out/rounds_w.jsonl; head -9 gpurun_out/ktl_w.log
