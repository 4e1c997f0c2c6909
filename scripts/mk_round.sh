#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for i in 1 2 3; do
MK_TIMEOUT=200 timeout 500 python scripts/mk_check.py tiny,llama8b_1b > gpurun_out/mk_check_$i.log 2>&1
echo "== check $i"; grep -E "FAILED|max\||MK=1 rc" gpurun_out/mk_check_$i.log
done
grep -A5 "llama8b_1b MK=" gpurun_out/mk_check_1.log
for pf in 0 8 16 24; do
  echo "== PF $pf"; SSD_B200_MK_PF=$pf timeout 200 python scripts/mk_trace.py llama8b_1b 0 1 2>&1 | head -1
  SSD_B200_MK_PF=$pf timeout 200 python scripts/mk_trace.py llama8b_1b 1 20 2>&1 | head -1
done
SSD_B200_MK_PF=8 timeout 200 python scripts/mk_trace.py llama8b_1b 0 1 > gpurun_out/mk_trace.log 2>&1; tail -60 gpurun_out/mk_trace.log
