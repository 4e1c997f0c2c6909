#!/bin/bash
# round-2g evidence: GPU suite, bench, ncu launch lists (cold + warm) of one
# d20 / t5 forward, full capture of one layer's d20 GEMMs
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/f_smoke.log 2>&1; tail -1 gpurun_out/f_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/f_pytest_gpu.log 2>&1; tail -3 gpurun_out/f_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/f_bench.jsonl 2> gpurun_out/f_bench.err; python - <<'P'
import json
d=json.loads(open('gpurun_out/f_bench.jsonl').read().strip().splitlines()[-1])
print({k:d[k] for k in ['value','ssd_tokens_per_s','ar_tokens_per_s','sd_tokens_per_s','speedup_vs_ar','speedup_vs_sd','hit_rate','alpha']}, d['e2e']['value'], d['roofline']['frac'], d['roofline']['ms_per_round'])
P
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 900 ncu --metrics $M --clock-control none -s 520 -c 115 --csv --log-file gpurun_out/f_launches_d20.csv python scripts/prof_fwd.py d20 > /dev/null 2>&1
timeout 900 ncu --metrics $M --cache-control none --clock-control none -s 520 -c 115 --csv --log-file gpurun_out/f_traffic_d20.csv python scripts/prof_fwd.py d20 > /dev/null 2>&1
timeout 900 ncu --metrics $M --clock-control none -s 696 -c 227 --csv --log-file gpurun_out/f_launches_t5.csv python scripts/prof_fwd.py t5 > /dev/null 2>&1
timeout 900 ncu --metrics $M --cache-control none --clock-control none -s 696 -c 227 --csv --log-file gpurun_out/f_traffic_t5.csv python scripts/prof_fwd.py t5 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 130 -c 4 -o gpurun_out/f_gemm_d20 python scripts/prof_fwd.py d20 > /dev/null 2>&1
for f in f_launches_d20 f_traffic_d20 f_launches_t5 f_traffic_t5; do python scripts/launches.py gpurun_out/$f.csv | head -9; done
