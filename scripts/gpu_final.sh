#!/bin/bash
# Final round-1 evidence on the committed build: smoke, bench (+CPU baseline), reference arm.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 0 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?" >> gpurun_out/bench_ref.log
tail -n 2 gpurun_out/smoke.log gpurun_out/bench.log gpurun_out/bench_ref.log | cut -c1-400
