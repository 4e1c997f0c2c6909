"""Tiny-pair logits against the fp32 and fp64-accumulating oracles (the
test_logits_match_oracle contexts): GPU-vs-fp64 and fp32-vs-fp64 deviations,
to tell a kernel error from fp32 summation-order noise."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2603_03251_b200 as P  # noqa: E402
from paper_2603_03251_b200.configs import shapes  # noqa: E402
import pyoracle  # noqa: E402

ts, ds = shapes("tiny", max_ctx=1024)
pair = P.Pair()
eng = P.Engine(ts, ds, pair, max_branches=32, max_lookahead=8)
o32 = pyoracle.TfPair(P.shape_dict(ts), P.shape_dict(ds), pair.as_dict())
o64 = pyoracle.TfPair(P.shape_dict(ts), P.shape_dict(ds), pair.as_dict(), accum="f64")
env = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("SSD_B200_")) or "default"
for which in (0, 1):
    for n in (1, 7, 40):
        ctx = np.random.default_rng(n).integers(0, 32000, n).tolist()
        g = eng.logits(which, ctx).astype(np.float64)
        a = o32.logits(which, ctx).astype(np.float64)
        b = o64.logits(which, ctx).astype(np.float64)
        rms = lambda x: float(np.sqrt((x * x).mean()))  # noqa: E731
        big = int((np.abs(g - b) > 1e-3).sum())
        print(json.dumps({"env": env, "which": which, "n": n, "gpu_vs_f32": float(np.abs(g - a).max()),
                          "gpu_vs_f64": float(np.abs(g - b).max()), "f32_vs_f64": float(np.abs(a - b).max()),
                          "gpu_vs_f64_rms": rms(g - b), "f32_vs_f64_rms": rms(a - b), "n_gt_1e-3": big}))
