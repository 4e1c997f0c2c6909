#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/v.jsonl; : > $O
for k in 0 2 3 4 0; do
  SSD_B200_ATOMIC_CTAS_PER_TILE=$k SSD_B200_PROFILE_PART=s timeout 120 python scripts/fwd_ablate.py d5,d20 >> $O 2>&1
  SSD_B200_ATOMIC_CTAS_PER_TILE=$k timeout 120 python scripts/fwd_ablate.py t5,d1 >> $O 2>&1
  SSD_B200_ATOMIC_CTAS_PER_TILE=$k timeout 120 python scripts/round_profile.py >> $O 2>&1
done
cat $O
