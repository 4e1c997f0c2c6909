#!/bin/bash
# §8f evidence: calibrated geometric fan-out (tau = 1) and the batch sweep on the current build.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/calibrate_fanout.py 32 3 > gpurun_out/calibrate_fanout.jsonl 2> gpurun_out/calibrate_fanout.err
timeout 900 python scripts/batch_sweep.py 24 > gpurun_out/batch_sweep.jsonl 2> gpurun_out/batch_sweep.err
cat gpurun_out/calibrate_fanout.jsonl; tail -2 gpurun_out/calibrate_fanout.err; cut -c1-220 gpurun_out/batch_sweep.jsonl; tail -2 gpurun_out/batch_sweep.err
