#!/bin/bash
# One gpurun call: GPU parity tests, a short bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 2 --rounds 16 --no-cpu-baseline > gpurun_out/bench_8b.log 2>&1
echo "bench 8b exit $?" >> gpurun_out/bench_8b.log
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/bench_8b.log
