#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r_pytest_gpu.log 2>&1; tail -3 gpurun_out/r_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r_bench.jsonl 2> gpurun_out/r_bench.err; python - <<'P'
import json
d=json.loads(open('gpurun_out/r_bench.jsonl').read().strip().splitlines()[-1])
print({k:d[k] for k in ['value','ssd_tokens_per_s','ar_tokens_per_s','sd_tokens_per_s','speedup_vs_ar','speedup_vs_sd','hit_rate','alpha','gpu_launches']}, d['e2e']['value'], d['roofline']['frac'], d['roofline']['ms_per_round'], d['clocks'])
P
timeout 300 python scripts/diag_tiny_logits.py > gpurun_out/r_diag_tiny.jsonl 2>&1
SSD_B200_SWIGLU_WHOLE=0 timeout 300 python scripts/diag_tiny_logits.py >> gpurun_out/r_diag_tiny.jsonl 2>&1
