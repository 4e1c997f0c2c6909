#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attention_dec -s 20 -c 1 -o gpurun_out/t_attn_d20 python scripts/prof_fwd.py d20 > /dev/null 2>&1
ls -la gpurun_out/t_attn_d20.ncu-rep
