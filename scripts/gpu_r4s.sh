#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/s.jsonl; : > $O
timeout 120 python scripts/fwd_ablate.py t5,d1,d5,d20 >> $O 2>&1
SSD_B200_NORM_TAIL=0 timeout 120 python scripts/fwd_ablate.py t5,d1,d5,d20 >> $O 2>&1
SSD_B200_PROFILE_PART=s timeout 120 python scripts/fwd_ablate.py d5,d20 >> $O 2>&1
timeout 120 python scripts/round_profile.py >> $O 2>&1
SSD_B200_NORM_TAIL=0 timeout 120 python scripts/round_profile.py >> $O 2>&1
SSD_B200_GREEN=0 timeout 120 python scripts/round_profile.py >> $O 2>&1
timeout 120 python scripts/diag_tiny_logits.py >> $O 2>&1
cat $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_loops.py -q -x -p no:cacheprovider 2>&1 | tail -3
