"""Calibrated geometric fan-out on the 8B/1B pair (the
reference's sweep-fanout -> fit_powerlaw -> geometric_fanout flow,
cli.cpp:400-454, hitmodel.cpp:65-106, cache.cpp:39-113).

tau = 1 (rejection sampling, BASELINE configs[2]), K = 4, FastRandom backup,
one B200 colocated. 1) uniform fan-out F in {1, 2, 4, 8}: measured miss rate
of the cache lookups and the acceptance alpha; 2) fit miss = A F^-r; 3) the
geometric plan for the same branch budget as uniform F = 4 (20 branches)
from (alpha, r), backup plan from (0.3, r); 4) both plans run on the same
prompts / seeds: hit rate, tokens per round, device tokens/s.
Usage: python scripts/calibrate_fanout.py [rounds] [prompts]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, ROOT + "/scripts")
import paper_2603_03251_b200 as P  # noqa: E402
from paper_2603_03251_b200.configs import shapes  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 32
NP = int(sys.argv[2]) if len(sys.argv) > 2 else 3
K, BUDGET = 4, 20
ts, ds = shapes("llama8b_1b", max_ctx=1024)
eng = P.Engine(ts, ds, P.Pair(block_out_scale=0.06), max_branches=2 * BUDGET, max_lookahead=K)
prompts = [np.random.default_rng(20250809 + i).integers(0, ts.vocab, 128).tolist() for i in range(NP)]


def alpha_of(mean_accepted):
    lo, hi = 0.0, 1.0
    for _ in range(60):
        a = 0.5 * (lo + hi)
        lo, hi = (a, hi) if sum(a ** i for i in range(1, K + 1)) < mean_accepted else (lo, a)
    return lo


def run(primary, backup):
    cfg = P.SimConfig(lookahead=K, scheme=P.SamplingScheme.standard(1.0), primary_plan=primary, backup_plan=backup,
                      primary_time=0.4, backup_time=0.0, backup_kind=P.FAST_RANDOM, rounds=R, seed=7)
    tot = {"tokens": 0, "ms": 0.0, "hits": 0, "lookups": 0, "acc": 0.0}
    for i, pr in enumerate(prompts):
        cfg.seed = 7 + i
        eng.run_ssd(pr, cfg) if i == 0 else None  # warm (graph capture)
        r = eng.run_ssd(pr, cfg)
        tot["tokens"] += r.tokens
        tot["ms"] += r.device_ms
        tot["hits"] += r.hits_total()
        tot["lookups"] += r.lookups()
        tot["acc"] += r.accepted_sum
    rounds = R * len(prompts)
    return {"tok_s": tot["tokens"] / (tot["ms"] / 1e3), "hit_rate": tot["hits"] / max(1, tot["lookups"]),
            "tokens_per_round": tot["tokens"] / rounds, "mean_accepted": tot["acc"] / rounds,
            "ms_per_round": tot["ms"] / rounds}


samples, alphas = [], []
for F in (1, 2, 4, 8):
    plan = P.FanOutPlan([F] * (K + 1), P.PRIMARY)
    res = run(plan, P.FanOutPlan([F] * (K + 1), P.BACKUP))
    miss = max(1.0 - res["hit_rate"], 1e-3)
    samples.append((F, miss))
    alphas.append(alpha_of(res["mean_accepted"]))
    print(json.dumps({"stage": "uniform", "fan_out": F, **{k: round(v, 4) for k, v in res.items()}, "miss": round(miss, 4)}),
          flush=True)
r, log_amp, r2 = P.fit_powerlaw(samples)
a = float(np.clip(np.mean(alphas), 0.05, 0.95))
geo_p = P.geometric_fanout(a, r, K, BUDGET)
geo_b = P.geometric_fanout(0.3, r, K, BUDGET, P.BACKUP)
print(json.dumps({"stage": "fit", "exponent": round(r, 4), "log_amplitude": round(log_amp, 4), "r_squared": round(r2, 4),
                  "alpha": round(a, 4), "geometric_primary": geo_p.fan_out, "geometric_backup": geo_b.fan_out,
                  "predicted_hit_rate_geometric": round(P.conditional_hit_rate(geo_p, a, r), 4),
                  "predicted_hit_rate_uniform4": round(P.conditional_hit_rate(P.FanOutPlan([4] * (K + 1)), a, r), 4)}),
      flush=True)
uni = run(P.FanOutPlan([4] * (K + 1), P.PRIMARY), P.FanOutPlan([4] * (K + 1), P.BACKUP))
geo = run(geo_p, geo_b)
print(json.dumps({"stage": "compare", "budget": BUDGET, "uniform4": {k: round(v, 4) for k, v in uni.items()},
                  "geometric": {k: round(v, 4) for k, v in geo.items()}}), flush=True)
eng.close()
