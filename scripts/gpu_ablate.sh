#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/ablate.jsonl; : > $out
timeout 300 python scripts/fwd_ablate.py >> $out 2>gpurun_out/ablate.err
SSD_B200_SKIP=1 timeout 300 python scripts/fwd_ablate.py >> $out 2>>gpurun_out/ablate.err
SSD_B200_SKIP=2 timeout 300 python scripts/fwd_ablate.py >> $out 2>>gpurun_out/ablate.err
SSD_B200_SKIP=3 timeout 300 python scripts/fwd_ablate.py >> $out 2>>gpurun_out/ablate.err
SSD_B200_MK=1 timeout 300 python scripts/fwd_ablate.py d1,d5,d20 >> $out 2>>gpurun_out/ablate.err
SSD_B200_PF_MB=0 timeout 300 python scripts/fwd_ablate.py d1,d20 >> $out 2>>gpurun_out/ablate.err
cat $out; tail -3 gpurun_out/ablate.err
