"""Diagnostic: prefill-width logits error against the fp64-accumulating oracle
(tiny pair), per M and per summation mode, beside the fp32 oracle's own
deviation (the noise floor)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2603_03251_b200 as P  # noqa: E402
import pyoracle  # noqa: E402
from paper_2603_03251_b200.configs import shapes  # noqa: E402

ts, ds = shapes("tiny", max_ctx=1024)
pair = P.Pair()
o32 = pyoracle.TfPair(P.shape_dict(ts), P.shape_dict(ds), pair.as_dict())
o64 = pyoracle.TfPair(P.shape_dict(ts), P.shape_dict(ds), pair.as_dict(), accum="f64")
mode = os.environ.get("SSD_B200_DETERMINISTIC", "0")
eng = P.Engine(ts, ds, pair, max_branches=32, max_lookahead=8)
seeds = [int(x) for x in os.environ.get("DIAG_SEEDS", "200").split(",")]
for M in [int(x) for x in (sys.argv[1:] or ["20", "32", "33", "40", "48", "49", "64", "65", "100"])]:
  for sd in seeds:
    ctx = np.random.default_rng(sd + M).integers(0, 32000, M).tolist()
    for which in (0, 1):
        ref = o64.logits(which, ctx).astype(np.float64)
        g = eng.logits(which, ctx).astype(np.float64)
        o = o32.logits(which, ctx).astype(np.float64)
        print(json.dumps({"det": mode, "M": M, "seed": sd, "which": which, "gpu_max": round(float(np.abs(g - ref).max()), 5),
                          "gpu_rms": round(float(np.sqrt(((g - ref) ** 2).mean())), 6),
                          "noise_max": round(float(np.abs(o - ref).max()), 5)}), flush=True)
