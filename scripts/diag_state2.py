"""Diagnostic: replay test_errors_map_to_reference_classes, then the width
checks, printing per (M, context, model) the deviation from the fp64 oracle."""
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
o64 = pyoracle.TfPair(P.shape_dict(ts), P.shape_dict(ds), pair.as_dict(), accum="f64")
eng = P.Engine(ts, ds, pair, max_branches=32, max_lookahead=8)
if "errors" in sys.argv:
    for f in (lambda: eng.run_ar([1, 2], P.SamplingScheme.standard(-1.0), 4, 0),
              lambda: P.geometric_fanout(0.8, 1.0, 4, 3),
              lambda: eng.run_ar([1] * 10, P.SamplingScheme.greedy(), 5000, 0)):
        try:
            f()
        except P.Error as e:
            print("error:", type(e).__name__, e)
for M in (2, 5, 20, 33, 100):
    for i in range(3):
        ctx = np.random.default_rng(200 + M + 1000 * i).integers(0, 32000, M).tolist()
        row = []
        for w in (0, 1):
            g = eng.logits(w, ctx).astype(np.float64)
            row.append(float(np.abs(g - o64.logits(w, ctx).astype(np.float64)).max()))
        print(f"M={M} ctx{i}: target {row[0]:.4f} draft {row[1]:.4f}", flush=True)
