"""Batch-size sweep of the Saguaro loop on the 8B/1B pair:
batch in {1, 2, 4, 8} x backup in {FastRandom, SamePrimaryJIT}, greedy and
tau = 1, one B200, verifier and speculator streams colocated.

Per cell: device tokens/s (all sequences), hit rate, E_hit / E_miss, mean
accepted length. Per batch size: the measured speculator / backup latencies
in verify passes (T_p = (extend + K branch steps) / verify forward, T_b = K
JIT draft steps / verify forward, from CUDA-event forward timings) and the
Saguaro fallback policy's choice (critical batch b*, perf.cpp:57-73) next to
the measured winner.  Usage: python scripts/batch_sweep.py [rounds]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_03251_b200 as P  # noqa: E402
from paper_2603_03251_b200.configs import shapes  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 24
K, F = 4, 4
B = F * (K + 1)
BATCHES = (1, 2, 4, 8)
ts, ds = shapes("llama8b_1b", max_ctx=1024)
eng = P.Engine(ts, ds, P.Pair(block_out_scale=0.06), max_branches=B, max_lookahead=K, max_batch=max(BATCHES))
prompt = np.random.default_rng(20250809).integers(0, ts.vocab, 128).tolist()


def cfg(temp, backup, batch):
    fan = [F] * (K + 1)
    return P.SimConfig(lookahead=K, scheme=P.SamplingScheme.standard(temp),
                       primary_plan=P.FanOutPlan(fan, P.PRIMARY), backup_plan=P.FanOutPlan(fan, P.BACKUP),
                       primary_time=0.4, backup_time=0.0, backup_kind=backup, rounds=R, seed=20250809,
                       batch_size=batch)


timing = {}
for b in BATCHES:
    pos = 256
    tv = eng.profile_forward(0, b * (K + 1), pos, 5)["ms_forward"]
    tx = eng.profile_forward(1, b * (K + 1), pos, 5)["ms_forward"]
    tb = eng.profile_forward(1, b * B, pos, 5)["ms_forward"]
    tj = eng.profile_forward(1, b, pos, 5)["ms_forward"]
    timing[b] = {"verify_ms": tv, "T_p": (tx + K * tb) / tv, "T_b_jit": K * tj / tv}

for temp in (0.0, 1.0):
    for b in BATCHES:
        cells = {}
        for backup in (P.FAST_RANDOM, P.SAME_PRIMARY_JIT):
            c = cfg(temp, backup, b)
            eng.run_ssd(prompt, c)  # warm (graph capture, prefill)
            r = eng.run_ssd(prompt, c)
            cells[backup] = {"tok_s": r.tokens / (r.device_ms / 1e3), "hit_rate": r.hit_rate(),
                             "e_hit": r.hit_round_tokens / max(1, r.hit_rounds),
                             "e_miss": r.miss_round_tokens / max(1, r.miss_rounds),
                             "mean_accepted": r.accepted_sum / (R * b), "ms_per_round": r.device_ms / R}
        fr = cells[P.FAST_RANDOM]
        t = timing[b]
        p = min(max(fr["hit_rate"], 1e-6), 1 - 1e-6)
        try:
            bstar = P.critical_batch(p, fr["e_hit"], max(fr["e_miss"], 1.0), t["T_p"])
        except P.Error as e:
            bstar = f"none ({type(e).__name__})"
        choice = P.saguaro_backup(b, p, fr["e_hit"], max(fr["e_miss"], 1.0), t["T_p"], jit_time=t["T_b_jit"])
        winner = max(cells, key=lambda k: cells[k]["tok_s"])
        print(json.dumps({"temperature": temp, "batch": b, "timing": {k: round(v, 4) for k, v in t.items()},
                          "cells": {k: {kk: round(vv, 4) for kk, vv in v.items()} for k, v in cells.items()},
                          "critical_batch": bstar if isinstance(bstar, str) else round(bstar, 3),
                          "policy_choice": choice, "measured_winner": winner}), flush=True)
eng.close()
