#!/bin/bash
# Re-entry evidence call: GPU tests, smoke, default bench (+reference arm),
# ncu launch list of the bench-shaped forwards (t1 = 8B M=1, t5 = 8B verify, d20 = 1B branch step).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
cp MEASURED_PEAKS.json gpurun_out/ 2>/dev/null
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 0 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?" >> gpurun_out/bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_fwd.csv python scripts/prof_fwd.py t1,t5,d20 > gpurun_out/prof_fwd.log 2>&1
echo "ncu exit $?" >> gpurun_out/prof_fwd.log
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.log gpurun_out/bench_ref.log gpurun_out/prof_fwd.log
