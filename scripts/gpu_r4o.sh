#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/o.jsonl; : > $O
for mb in 0 9 13 40; do
  SSD_B200_SMALL_GEMM_MB=$mb timeout 300 python scripts/round_profile.py >> $O 2>&1
  SSD_B200_SMALL_GEMM_MB=$mb SSD_B200_PROFILE_PART=s timeout 300 python scripts/fwd_ablate.py d5,d20 >> $O 2>&1
  SSD_B200_SMALL_GEMM_MB=$mb timeout 300 python scripts/fwd_ablate.py t5,d1 >> $O 2>&1
done
cat $O
