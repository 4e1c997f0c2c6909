#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/bisect.log
for k in "widths" "logits_match or widths" "topk or widths" "verify_decision or widths" "run_ar or widths" "run_sd or widths" "statistically or widths" "run_ssd or widths" "build_cache or widths" "errors or widths"; do
  echo "== -k '$k'" >> gpurun_out/bisect.log
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "$k" 2>&1 | grep -E "passed|failed|AssertionError: \{" >> gpurun_out/bisect.log
done
cat gpurun_out/bisect.log
