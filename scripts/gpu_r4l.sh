#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/l_pytest_gpu.log 2>&1; tail -5 gpurun_out/l_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/l_bench.jsonl 2> gpurun_out/l_bench.err; python - <<'P'
import json
d=json.loads(open('gpurun_out/l_bench.jsonl').read().strip().splitlines()[-1])
print({k:d[k] for k in ['value','ssd_tokens_per_s','ar_tokens_per_s','sd_tokens_per_s','speedup_vs_ar','speedup_vs_sd','hit_rate','alpha']}, d['e2e']['value'], d['roofline']['frac'], d['roofline']['ms_per_round'])
P
