"""Colocated SSD round (bench workload) under the current SSD_B200_* knobs:
ms per round (median of 3 runs of 32 rounds) plus the in-graph segment
profile (Engine.profile_ssd_round). One JSON line per process."""
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_03251_b200 as P  # noqa: E402
from paper_2603_03251_b200.configs import shapes  # noqa: E402

K = 4
ts, ds = shapes("llama8b_1b", max_ctx=1024)
eng = P.Engine(ts, ds, P.Pair(block_out_scale=0.06), max_branches=20, max_lookahead=K)
prompt = np.random.default_rng(20250809).integers(0, ts.vocab, 128).tolist()
fan = [4] * (K + 1)
cfg = P.SimConfig(lookahead=K, scheme=P.SamplingScheme.greedy(), primary_plan=P.FanOutPlan(fan, P.PRIMARY),
                  backup_plan=P.FanOutPlan(fan, P.BACKUP), primary_time=0.4, backup_time=0.0,
                  backup_kind=P.FAST_RANDOM, rounds=32, seed=20250809)
eng.run_ssd(prompt, cfg)
ms = [eng.run_ssd(prompt, cfg).device_ms / 32 for _ in range(3)]
prof = eng.profile_ssd_round(prompt, cfg)
env = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("SSD_B200_")) or "default"
print(json.dumps({"env": env, "ms_per_round": round(statistics.median(ms), 3),
                  "segments": {k: round(v, 3) for k, v in prof.items()}}), flush=True)
