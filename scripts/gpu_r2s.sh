#!/bin/bash
# r02f evidence: full GPU tests, smoke, bench, ncu launch lists (d20 branch
# step, t5 verify) and full captures of the branch-step GEMM and the verify
# gate/up GEMM.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -rf --durations=10 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 900 ncu --metrics $M --clock-control none -c 600 --csv --log-file gpurun_out/launches_d20.csv python scripts/prof_fwd.py d20 > /dev/null 2>&1
timeout 900 ncu --metrics $M --clock-control none -c 600 --csv --log-file gpurun_out/launches_t5.csv python scripts/prof_fwd.py t5 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_cl -s 20 -c 2 -o gpurun_out/prof_gemm_cl_d20 python scripts/prof_fwd.py d20 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 60 -c 2 -o gpurun_out/prof_gemm_t5 python scripts/prof_fwd.py t5 > /dev/null 2>&1
tail -n 4 gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -c 600 gpurun_out/bench.log; ls -la gpurun_out/
