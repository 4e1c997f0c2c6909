#!/bin/bash
# r02f: colocated-round knobs — verify after the extend forward, stream-K
# (atomic) instead of the cluster GEMM for the M=20 branch steps.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/rounds_t.jsonl; : > gpurun_out/ablate_t.jsonl
for env in "SSD_B200_VERIFY_AFTER_EXTEND=0" "SSD_B200_VERIFY_AFTER_EXTEND=1" "SSD_B200_CL_GEMM_MB=0" "SSD_B200_VERIFY_AFTER_EXTEND=1 SSD_B200_CL_GEMM_MB=0"; do
  env $env timeout 300 python scripts/split_sms_sweep.py >> gpurun_out/rounds_t.jsonl 2>>gpurun_out/rounds_t.err
done
for env in "SSD_B200_CL_GEMM_MB=72" "SSD_B200_CL_GEMM_MB=0"; do
  env $env timeout 300 python scripts/fwd_ablate.py d5,d20 >> gpurun_out/ablate_t.jsonl 2>>gpurun_out/ablate_t.err
done
cat gpurun_out/rounds_t.jsonl gpurun_out/ablate_t.jsonl
# whole-forward DRAM traffic with warm caches between kernels (no per-kernel flush):
# the sum over a forward's launches vs its algorithmic bytes
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 900 ncu --metrics $M --cache-control none --clock-control none -c 600 --csv --log-file gpurun_out/traffic_t5.csv python scripts/prof_fwd.py t5 > /dev/null 2>&1
timeout 900 ncu --metrics $M --cache-control none --clock-control none -c 600 --csv --log-file gpurun_out/traffic_d20.csv python scripts/prof_fwd.py d20 > /dev/null 2>&1
python scripts/launches.py gpurun_out/traffic_t5.csv embed_kernel 2>&1 | head -8
python scripts/launches.py gpurun_out/traffic_d20.csv embed_kernel 2>&1 | head -8
