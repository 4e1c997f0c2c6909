#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_partition.py tests/test_gpu_loops.py tests/test_batch_gpu.py tests/test_gpu_parity.py tests/test_gpu_bench_shapes.py tests/test_gpu_paged.py -q -p no:cacheprovider -rf > gpurun_out/a5_pytest.log 2>&1; tail -3 gpurun_out/a5_pytest.log
timeout 600 python bench.py > gpurun_out/a5_bench.jsonl 2> gpurun_out/a5_bench.err; python - <<'P'
import json
d=json.loads(open('gpurun_out/a5_bench.jsonl').read().strip().splitlines()[-1])
print({k:d[k] for k in ['value','ssd_tokens_per_s','ar_tokens_per_s','sd_tokens_per_s','speedup_vs_ar','speedup_vs_sd','hit_rate','alpha']}, d['e2e']['value'], d['roofline']['frac'], d['roofline']['ms_per_round'], d['clocks'])
P
