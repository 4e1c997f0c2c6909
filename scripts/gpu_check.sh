#!/bin/bash
# One gpurun call: GPU parity tests, a short bench, the kernel launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config tiny --steps 3 --warmup 2 --rounds 16 --no-cpu-baseline > gpurun_out/bench_tiny.log 2>&1
echo "bench tiny exit $?" >> gpurun_out/bench_tiny.log
timeout 900 python bench.py --steps 3 --warmup 2 --rounds 16 --no-cpu-baseline > gpurun_out/bench_8b.log 2>&1
echo "bench 8b exit $?" >> gpurun_out/bench_8b.log
tail -3 gpurun_out/pytest_gpu.log gpurun_out/bench_tiny.log gpurun_out/bench_8b.log
