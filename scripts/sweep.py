"""BASELINE configs[2] (C3): the 8B/1B pair at temperature 1.0 with
rejection-sampling verification — fan-out sweep F = 1..16 (hit rate vs round
latency), plus the Saguaro sigma_{F,C} down-weight sweep.
One JSON line per point; colocated on one GPU, device-timed."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2603_03251_b200 as P  # noqa: E402
from paper_2603_03251_b200.configs import shapes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--what", default="fanout,downweight")
ap.add_argument("--rounds", type=int, default=32)
ap.add_argument("--temperature", type=float, default=1.0)
ap.add_argument("--block-out-scale", type=float, default=0.07)
ap.add_argument("--seed", type=int, default=20250809)
a = ap.parse_args()
K = 4
ts, ds = shapes("llama8b_1b", max_ctx=1024)
eng = P.Engine(ts, ds, P.Pair(block_out_scale=a.block_out_scale), max_branches=80, max_lookahead=K)
prompt = np.random.default_rng(a.seed).integers(0, ts.vocab, 128).tolist()


def point(fan, scheme, label):
    cfg = P.SimConfig(lookahead=K, scheme=scheme, target_scheme=P.SamplingScheme.standard(a.temperature),
                      primary_plan=P.FanOutPlan([fan] * (K + 1), P.PRIMARY),
                      backup_plan=P.FanOutPlan([fan] * (K + 1), P.BACKUP), primary_time=0.4,
                      backup_kind=P.FAST_RANDOM, rounds=a.rounds, seed=a.seed)
    eng.run_ssd(prompt, cfg)  # warm (graph capture, caches)
    r = eng.run_ssd(prompt, cfg)
    sd = eng.run_sd(prompt, cfg)
    line = {"sweep": label, "fan_out": fan, "branches": fan * (K + 1), "temperature": a.temperature,
            "scheme": scheme.kind, "downweight": scheme.downweight,
            "ssd_tokens_per_s": r.tokens_per_second(), "sd_tokens_per_s": sd.tokens_per_second(),
            "round_ms": r.device_ms / r.rounds, "hit_rate": r.hit_rate(),
            "hit_rate_primary": r.hit_rate_primary(), "hit_rate_backup": r.hit_rate_backup(),
            "mean_accepted": r.accepted_sum / r.rounds, "tokens_per_round": r.tokens / r.rounds}
    print(json.dumps(line), flush=True)


if "fanout" in a.what:
    for f in (1, 2, 4, 8, 16):
        point(f, P.SamplingScheme.standard(a.temperature), "fanout")
if "downweight" in a.what:
    for c in (1.0, 0.5, 0.2, 0.05):
        point(4, P.SamplingScheme.saguaro(4, c, a.temperature), "downweight")
eng.close()
