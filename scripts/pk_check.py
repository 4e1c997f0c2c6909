"""Persistent layer-block kernel (fwd_pk.cuh) vs the per-op forward: draft
logits of one M-token forward (M <= 32 takes the pk path) on the same
weights, and both paths' step times (CUDA events)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_03251_b200 as P  # noqa: E402
from paper_2603_03251_b200.configs import shapes  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "tiny"
ts, ds = shapes(cfg, max_ctx=1024)
engines = {}
for pkv in ("1", "0"):
    os.environ["SSD_B200_PK"] = pkv
    engines[pkv] = P.Engine(ts, ds, P.Pair(), max_branches=20, max_lookahead=4)
rng = np.random.default_rng(0)
for M in (1, 2, 5, 8, 17, 20, 32):
    ctx = rng.integers(0, ds.vocab, M).tolist()
    a = engines["1"].logits(1, ctx)
    b = engines["0"].logits(1, ctx)
    print(json.dumps({"cfg": cfg, "M": M, "max_abs_diff": float(np.max(np.abs(a - b))),
                      "argmax_equal": int(np.argmax(a)) == int(np.argmax(b)), "finite": bool(np.isfinite(a).all())}),
          flush=True)
if cfg != "tiny":
    for pkv, eng in engines.items():
        for w in ("d1", "d5", "d20"):
            r = eng.profile_forward(1, int(w[1:]), 256, 20)
            print(json.dumps({"pk": pkv, "fwd": w, "ms_forward": round(r["ms_forward"], 4)}), flush=True)
for e in engines.values():
    e.close()
