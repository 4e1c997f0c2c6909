"""Short deterministic workload for ncu launch lists / captures:
one SSD decode of a few rounds on the 8B/1B pair (plus AR and SD rounds)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2603_03251_b200 as P  # noqa: E402
from paper_2603_03251_b200.configs import shapes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="llama8b_1b")
ap.add_argument("--rounds", type=int, default=2)
ap.add_argument("--what", default="ssd,ar,sd")
a = ap.parse_args()
ts, ds = shapes(a.config, max_ctx=1024)
eng = P.Engine(ts, ds, P.Pair(), max_branches=20, max_lookahead=4)
prompt = np.random.default_rng(0).integers(0, ts.vocab, 128).tolist()
cfg = P.SimConfig(lookahead=4, scheme=P.SamplingScheme.greedy(), primary_plan=P.FanOutPlan([4] * 5, P.PRIMARY),
                  backup_plan=P.FanOutPlan([4] * 5, P.BACKUP), rounds=a.rounds, seed=1)
for w in a.what.split(","):
    if w == "ssd":
        r = eng.run_ssd(prompt, cfg)
    elif w == "ar":
        r = eng.run_ar(prompt, P.SamplingScheme.greedy(), a.rounds, 1)
    elif w == "sd":
        r = eng.run_sd(prompt, cfg)
    print(w, r.tokens, r.device_ms, r.kernel_launches)
eng.close()
