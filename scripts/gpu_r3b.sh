#!/bin/bash
# r02f final evidence on the committed kernels: full GPU tests, smoke, bench,
# ncu launch lists (d20 branch step, t5 verify, warm caches for traffic) and
# full captures of the branch-step GEMMs (stream-K + bulk reduce, whole-tile SwiGLU).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -rf --durations=10 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 900 ncu --metrics $M --clock-control none -s 700 -c 400 --csv --log-file gpurun_out/launches_d20.csv python scripts/prof_fwd.py d20 > /dev/null 2>&1
timeout 900 ncu --metrics $M --cache-control none --clock-control none -s 700 -c 400 --csv --log-file gpurun_out/traffic_d20.csv python scripts/prof_fwd.py d20 > /dev/null 2>&1
timeout 900 ncu --metrics $M --cache-control none --clock-control none -s 1000 -c 600 --csv --log-file gpurun_out/traffic_t5.csv python scripts/prof_fwd.py t5 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 40 -c 4 -o gpurun_out/prof_gemm_d20 python scripts/prof_fwd.py d20 > /dev/null 2>&1
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -c 300 gpurun_out/bench.log; ls gpurun_out/
