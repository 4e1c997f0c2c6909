"""bench.py's reference arm on the CPU (no GPU): the oracle port of
run_protocol_harness times decode rounds only, and prints the contract's
JSON line with the same `config` the GPU arm prints."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "tiny",
                          "--steps", "2", "--warmup", "1", "--cpu-rounds", "2"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "tokens/s"
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    sys.path.insert(0, ROOT)
    import argparse
    import bench
    args = argparse.Namespace(config="tiny", greedy=True, temperature=1.0, lookahead=4, fanout=4, rounds=144,
                              prompt_len=128, block_out_scale=0.06)
    assert line["config"] == bench.workload_config(args)
