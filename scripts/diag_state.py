"""Diagnostic: the M=33 prefill logits after various earlier calls on the same
engine (state leaking between calls), against the fp64 oracle."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2603_03251_b200 as P  # noqa: E402
import pyoracle  # noqa: E402
from paper_2603_03251_b200.configs import shapes  # noqa: E402
from parity import sim_cfg  # noqa: E402

ts, ds = shapes("tiny", max_ctx=1024)
pair = P.Pair()
o64 = pyoracle.TfPair(P.shape_dict(ts), P.shape_dict(ds), pair.as_dict(), accum="f64")
eng = P.Engine(ts, ds, pair, max_branches=32, max_lookahead=8)
ctxs = {M: np.random.default_rng(1200 + M).integers(0, 32000, M).tolist() for M in (20, 33, 48, 100)}
refs = {(M, w): o64.logits(w, c).astype(np.float64) for M, c in ctxs.items() for w in (0, 1)}


def check(tag):
    out = []
    for M in (33, 48):
        for w in (0, 1):
            g = eng.logits(w, ctxs[M]).astype(np.float64)
            out.append(f"M{M}/{w}:{np.abs(g - refs[(M, w)]).max():.4f}")
    print(f"{tag:28s} " + " ".join(out), flush=True)


check("fresh")
prompt = np.random.default_rng(3).integers(0, 32000, 12).tolist()
eng.run_ar(prompt, P.SamplingScheme.greedy(), 20, 0)
check("after run_ar greedy")
eng.run_sd(prompt, sim_cfg(P, 4, 8, 1, 0.0, [4] * 5))
check("after run_sd greedy")
eng.run_ssd(prompt, sim_cfg(P, 4, 8, 1, 0.0, [4] * 5))
check("after run_ssd greedy")
eng.run_ssd(prompt, sim_cfg(P, 4, 8, 1, 1.0, [4] * 5))
check("after run_ssd sampled")
eng.run_ssd(prompt, sim_cfg(P, 8, 6, 1, 0.0, [4] * 9))
check("after run_ssd K=8")
for M in (2, 5, 20):
    eng.logits(0, ctxs[20][:M])
check("after logits 2/5/20")
try:
    eng.run_ar([1] * 10, P.SamplingScheme.greedy(), 5000, 0)
except P.Error as e:
    print("expected error:", type(e).__name__)
check("after TooLarge")
