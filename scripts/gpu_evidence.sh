#!/bin/bash
# Round-1 evidence: bench (+reference arm), launch lists of the bench-shaped
# forwards with DRAM traffic, full ncu captures of the top kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?" >> gpurun_out/bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_fwd.csv python scripts/prof_fwd.py t1,t5,d20 > gpurun_out/prof_fwd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:gemm_tc_kernel<2' -s 40 -c 1 -o gpurun_out/prof_gu_t1 python scripts/prof_fwd.py t1 > gpurun_out/prof_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:gemm_tc_kernel<0' -s 300 -c 1 -o gpurun_out/prof_head_t1 python scripts/prof_fwd.py t1 >> gpurun_out/prof_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention_cl -s 20 -c 1 \
  -o gpurun_out/prof_attn_t1 python scripts/prof_fwd.py t1 >> gpurun_out/prof_full.log 2>&1
echo "ncu done" >> gpurun_out/prof_full.log
grep '^{' gpurun_out/bench.log | head -c 1500; echo; tail -2 gpurun_out/bench_ref.log; tail -3 gpurun_out/prof_full.log
