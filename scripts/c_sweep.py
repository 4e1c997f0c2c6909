"""Saguaro down-weighted draft sampling sigma_{F,C} (categorical.cpp:65-92;
SURVEY §8f row 2): C sweep on the 8B/1B pair at tau = 1 (BASELINE configs[2]),
draft scheme Saguaro(F = 4, C), target Standard(1), uniform fan-out 4, K = 4,
FastRandom backup, 4 prompts x 32 rounds. Per C: cache hit rate, acceptance
(mean accepted), tokens per round, SSD and SD tokens/s. The paper's claim:
lowering C concentrates the draft on its top-F tokens, raising the hit rate
of the top-F keyed cache at some cost in acceptance."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_03251_b200 as P  # noqa: E402
from paper_2603_03251_b200.configs import shapes  # noqa: E402

R, NP, K, F = 32, 4, 4, 4
ts, ds = shapes("llama8b_1b", max_ctx=1024)
eng = P.Engine(ts, ds, P.Pair(block_out_scale=0.06), max_branches=F * (K + 1), max_lookahead=K)
prompts = [np.random.default_rng(20250809 + i).integers(0, ts.vocab, 128).tolist() for i in range(NP)]
fan = [F] * (K + 1)
for C in (1.0, 0.5, 0.2, 0.1, 0.05):
    scheme = P.SamplingScheme.saguaro(F, C, 1.0) if C < 1.0 else P.SamplingScheme.standard(1.0)
    cfg = P.SimConfig(lookahead=K, scheme=scheme, target_scheme=P.SamplingScheme.standard(1.0),
                      primary_plan=P.FanOutPlan(fan, P.PRIMARY), backup_plan=P.FanOutPlan(fan, P.BACKUP),
                      primary_time=0.4, backup_time=0.0, backup_kind=P.FAST_RANDOM, rounds=R, seed=11)
    agg = {"tok": 0, "ms": 0.0, "hits": 0, "look": 0, "acc": 0.0, "sd_tok": 0, "sd_ms": 0.0, "sd_acc": 0.0}
    for i, pr in enumerate(prompts):
        cfg.seed = 11 + i
        r = eng.run_ssd(pr, cfg)
        s = eng.run_sd(pr, cfg)
        agg["tok"] += r.tokens
        agg["ms"] += r.device_ms
        agg["hits"] += r.hits_total()
        agg["look"] += r.lookups()
        agg["acc"] += r.accepted_sum
        agg["sd_tok"] += s.tokens
        agg["sd_ms"] += s.device_ms
        agg["sd_acc"] += s.accepted_sum
    n = R * NP
    print(json.dumps({"downweight_C": C, "fan_out_F": F, "hit_rate": round(agg["hits"] / agg["look"], 4),
                      "ssd_mean_accepted": round(agg["acc"] / n, 4), "ssd_tokens_per_round": round(agg["tok"] / n, 4),
                      "ssd_tok_s": round(agg["tok"] / (agg["ms"] / 1e3), 1),
                      "sd_mean_accepted": round(agg["sd_acc"] / n, 4),
                      "sd_tok_s": round(agg["sd_tok"] / (agg["sd_ms"] / 1e3), 1)}), flush=True)
eng.close()
