#!/bin/bash
# One gpurun call: GPU parity tests, a short bench, AR/SSD launch lists.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 2 --rounds 16 --no-cpu-baseline > gpurun_out/bench_8b.log 2>&1
echo "bench 8b exit $?" >> gpurun_out/bench_8b.log
if [ "${PROF:-1}" = "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/launches_ar.csv \
  python scripts/profile_run.py --rounds 2 --what ar > gpurun_out/prof_ar.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/launches_ssd.csv \
  python scripts/profile_run.py --rounds 2 --what ssd > gpurun_out/prof_ssd.log 2>&1
fi
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/bench_8b.log
