#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/rounds_y.jsonl
timeout 300 python scripts/fwd_ablate.py d1,d5,d20,t1,t5 > gpurun_out/ablate_y.jsonl 2>&1
for i in 1 2; do timeout 300 python scripts/split_sms_sweep.py >> gpurun_out/rounds_y.jsonl 2>&1; done
timeout 1200 python bench.py --steps 4 --warmup 2 --no-cpu-baseline > gpurun_out/bench_y.log 2>&1
cat gpurun_out/ablate_y.jsonl gpurun_out/rounds_y.jsonl; python -c "
import json; d=json.loads(open('gpurun_out/bench_y.log').readline())
print({k: d[k] for k in ['value','ar_tokens_per_s','sd_tokens_per_s','speedup_vs_sd','alpha','hit_rate']}, d['round_ms']['round'], d['e2e']['value'])"
