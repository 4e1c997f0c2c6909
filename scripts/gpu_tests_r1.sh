#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_split_gpu.py tests/test_shim.py -m gpu -q -x --timeout 1200 -p no:cacheprovider -rf > gpurun_out/pytest_split.log 2>&1
echo "split exit $?" >> gpurun_out/pytest_split.log
timeout 900 python -m pytest tests -m gpu -q --timeout 800 -p no:cacheprovider -rf --deselect tests/test_split_gpu.py > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -n 15 gpurun_out/pytest_split.log; tail -n 3 gpurun_out/pytest_gpu.log
