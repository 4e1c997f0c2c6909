#!/bin/bash
# r02 call A: GPU tests after the stream-ordering fix (incl. the new bench-shape
# GQA parity tests and the fresh-process stress test), forward ablation of the
# draft's persistent kernel (SSD_B200_MK=2), colocated round times, bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rf --durations=15 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for mk in 0 2; do
  SSD_B200_MK=$mk timeout 300 python scripts/fwd_ablate.py d1,d5,d20,t1,t5 >> gpurun_out/ablate.jsonl 2>>gpurun_out/ablate.err
done
for mk in 0 2; do
  SSD_B200_MK=$mk timeout 300 python scripts/split_sms_sweep.py >> gpurun_out/rounds.jsonl 2>>gpurun_out/rounds.err
done
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
tail -n 5 gpurun_out/pytest_gpu.log gpurun_out/bench.log; cat gpurun_out/ablate.jsonl gpurun_out/rounds.jsonl
