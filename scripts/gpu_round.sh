#!/bin/bash
# One gpurun call: GPU parity tests, smoke, default bench (+reference arm),
# ncu launch list of the bench-shaped workload, one full capture of the top kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1; nproc > gpurun_out/nproc.txt; lscpu >> gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
cp MEASURED_PEAKS.json gpurun_out/ 2>/dev/null
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?" >> gpurun_out/bench_ref.log
if [ "${PROF:-1}" = "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_ssd.csv \
  python scripts/profile_run.py --rounds 2 --what ssd > gpurun_out/prof_ssd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 300 -c 2 \
  -o gpurun_out/prof_gemm_tc python scripts/profile_run.py --rounds 1 --what ssd > gpurun_out/prof_full.log 2>&1
echo "ncu exit $?" >> gpurun_out/prof_full.log
fi
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.log gpurun_out/bench_ref.log
