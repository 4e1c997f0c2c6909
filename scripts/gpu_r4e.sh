#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/green_e.jsonl; : > $O
timeout 200 python scripts/round_profile.py >> $O 2>&1
SSD_B200_GREEN=0 timeout 200 python scripts/round_profile.py >> $O 2>&1
SSD_B200_GREEN=64 SSD_B200_GREEN_TAIL=3 timeout 200 python scripts/round_profile.py >> $O 2>&1
cat $O
timeout 600 python bench.py > gpurun_out/e_bench.jsonl 2> gpurun_out/e_bench.err; tail -c 2500 gpurun_out/e_bench.jsonl
