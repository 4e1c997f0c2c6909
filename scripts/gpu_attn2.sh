#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/attn_ablate.jsonl; : > $out
for i in 1 2; do timeout 300 python scripts/fwd_ablate.py >> $out 2>>gpurun_out/attn_ablate.err; SSD_B200_ATTN_DEC=0 timeout 300 python scripts/fwd_ablate.py >> $out 2>>gpurun_out/attn_ablate.err; done
timeout 300 python scripts/ktl.py t1 d1 > gpurun_out/ktl_dec.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
cat $out; grep -v "launch \|per-CTA" gpurun_out/ktl_dec.log | grep "==\|attention\|sub-phases"; tail -8 gpurun_out/pytest_gpu.log
