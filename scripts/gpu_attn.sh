#!/bin/bash
# attention_dec check: GPU tests, forward timings (new vs chunked attention), kernel timeline
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/attn_ablate.jsonl; : > $out
timeout 300 python scripts/fwd_ablate.py >> $out 2>gpurun_out/attn_ablate.err
SSD_B200_ATTN_DEC=0 timeout 300 python scripts/fwd_ablate.py >> $out 2>>gpurun_out/attn_ablate.err
SSD_B200_SKIP=2 timeout 300 python scripts/fwd_ablate.py >> $out 2>>gpurun_out/attn_ablate.err
timeout 300 python scripts/ktl.py t1 d1 d20 > gpurun_out/ktl_dec.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
cat $out; tail -3 gpurun_out/attn_ablate.err; grep -v "launch \|per-CTA" gpurun_out/ktl_dec.log | grep "==\|attention\|sub-phases"; tail -15 gpurun_out/pytest_gpu.log
