"""Acceptance of the correlated random 8B/1B pair vs the block output scale
(the pair's divergence knob): greedy run_sd, mean accepted
length -> per-token acceptance alpha (E[acc] = a(1-a^K)/(1-a))."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2603_03251_b200 as P  # noqa: E402
from paper_2603_03251_b200.configs import shapes  # noqa: E402


def alpha_of(acc, K):
    lo, hi = 0.0, 1.0
    for _ in range(60):
        a = 0.5 * (lo + hi)
        e = sum(a ** i for i in range(1, K + 1))
        lo, hi = (a, hi) if e < acc else (lo, a)
    return lo


cfgname = sys.argv[1] if len(sys.argv) > 1 else "llama8b_1b"
scales = [float(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0.1", "0.06", "0.04", "0.03", "0.02"])]
ts, ds = shapes(cfgname, max_ctx=1024)
K = 4
for bos in scales:
    eng = P.Engine(ts, ds, P.Pair(block_out_scale=bos), max_branches=20, max_lookahead=K)
    accs = []
    for seed in range(4):
        prompt = np.random.default_rng(seed).integers(0, ts.vocab, 128).tolist()
        cfg = P.SimConfig(lookahead=K, scheme=P.SamplingScheme.greedy(), rounds=48, seed=seed)
        r = eng.run_sd(prompt, cfg)
        accs.append(r.accepted_sum / r.rounds)
    acc = float(np.mean(accs))
    print(f"block_out_scale={bos} mean_accepted={acc:.3f} alpha={alpha_of(acc, K):.3f} per-seed={np.round(accs, 2).tolist()}",
          flush=True)
    eng.close()
