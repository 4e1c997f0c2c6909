#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python scripts/pk_check.py tiny > gpurun_out/x_check.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_shapes.py -m gpu -q -p no:cacheprovider -x -k "widths or logits or harness_matches or bench_shape" >> gpurun_out/x_check.log 2>&1
timeout 300 python scripts/fwd_ablate.py d1,d5,d20,t1,t5 > gpurun_out/ablate_x.jsonl 2>&1
timeout 300 python scripts/split_sms_sweep.py > gpurun_out/rounds_x.jsonl 2>&1
tail -5 gpurun_out/x_check.log; cat gpurun_out/ablate_x.jsonl gpurun_out/rounds_x.jsonl
