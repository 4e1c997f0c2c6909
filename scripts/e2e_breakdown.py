"""Where the host-API (e2e) time of run_ssd goes on the bench workload:
wall time vs rounds (fixed cost = intercept), device loop time, and the
prefill-only cost (ssd_logits) for comparison."""
import json
import os
import sys
import time

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


def cfg(R):
    return P.SimConfig(lookahead=K, scheme=P.SamplingScheme.greedy(), primary_plan=P.FanOutPlan(fan, P.PRIMARY),
                       backup_plan=P.FanOutPlan(fan, P.BACKUP), primary_time=0.4, backup_time=0.0,
                       backup_kind=P.FAST_RANDOM, rounds=R, seed=20250809)


out = {}
for R in (1, 8, 32):
    c = cfg(R)
    eng.run_ssd(prompt, c)
    walls, devs = [], []
    for _ in range(3):
        t0 = time.perf_counter()
        r = eng.run_ssd(prompt, c)
        walls.append((time.perf_counter() - t0) * 1e3)
        devs.append(r.device_ms)
    out[R] = {"wall_ms": round(min(walls), 2), "device_loop_ms": round(min(devs), 2)}
t0 = time.perf_counter()
for _ in range(3):
    eng.logits(0, prompt)
out["logits_target_prefill_ms"] = round((time.perf_counter() - t0) / 3 * 1e3, 2)
t0 = time.perf_counter()
for _ in range(3):
    eng.logits(1, prompt)
out["logits_draft_prefill_ms"] = round((time.perf_counter() - t0) / 3 * 1e3, 2)
print(json.dumps(out))
