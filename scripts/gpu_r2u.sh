#!/bin/bash
# r02f: with stream-K at M=20 (no cluster GEMM in fused mode): GEMM budget
# and L2 look-ahead knobs, standalone forwards and the colocated round.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/rounds_u.jsonl; : > gpurun_out/ablate_u.jsonl
for env in "SSD_B200_SMALL_GEMM_MB=0" "SSD_B200_SMALL_GEMM_MB=80"; do
  env $env timeout 300 python scripts/fwd_ablate.py d1,d5,d20,t1,t5 >> gpurun_out/ablate_u.jsonl 2>>gpurun_out/ablate_u.err
done
for env in "SSD_B200_CORUN_SMALL_GEMM_MB=2000" "SSD_B200_CORUN_SMALL_GEMM_MB=80" "SSD_B200_CORUN_SMALL_GEMM_MB=0" "SSD_B200_PF_MB=8" "SSD_B200_PF_MB=32" "SSD_B200_VERIFY_AFTER_EXTEND=1" "SSD_B200_SPEC_PRIO=1"; do
  env $env timeout 300 python scripts/split_sms_sweep.py >> gpurun_out/rounds_u.jsonl 2>>gpurun_out/rounds_u.err
done
cat gpurun_out/ablate_u.jsonl gpurun_out/rounds_u.jsonl
