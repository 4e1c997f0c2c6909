"""Diagnostic: wide pre-speculation (F up to 16, M = 5F branch rows) against
the CPU oracle: entry rows along each entry's prefix, greedy entries, and the
tau = 1 harness acceptance / hits per run."""
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
from parity import sim_cfg, sim_req  # noqa: E402

K = 4
ts, ds = shapes("tiny", max_ctx=1024)
pair = P.Pair()
eng = P.Engine(ts, ds, pair, max_branches=80, max_lookahead=K, max_batch=2)
orc = pyoracle.TfPair(P.shape_dict(ts), P.shape_dict(ds), pair.as_dict())
Fs = [int(x) for x in (sys.argv[1:] or ["4", "8", "12", "16"])]
for F in Fs:
    prompt = np.random.default_rng(7 + F).integers(0, 32000, 12).tolist()
    rng = P.Stream(55 + F)
    spec = eng.draft_tokens(prompt, K, P.SamplingScheme.standard(1.0), rng)
    cache = eng.build_cache_stream(prompt, spec, P.FanOutPlan([F] * (K + 1), P.PRIMARY), P.SamplingScheme.standard(1.0),
                                   K, rng)
    worst = (0.0, None)
    bad = 0
    for (k, t), toks in cache.entries.items():
        ent = cache.speculation(k, t)
        ctx = prompt + spec.tokens[:k] + [t]
        for j in range(K):
            z = orc.logits(1, ctx + ent.tokens[:j])
            e = float(np.max(np.abs(z - ent.rows[j])))
            bad += e > 5e-2
            if e > worst[0]:
                worst = (e, (k, t, j))
    print(f"F={F}: {len(cache.entries)} entries, rows vs oracle worst {worst}, bad rows {bad}", flush=True)
    # harness at tau = 1
    for rep in range(3):
        pr = np.random.default_rng(1200 + 10 * F + rep).integers(0, 32000, 12).tolist()
        g = eng.run_ssd(pr, sim_cfg(P, K, 24, 1300 + rep, 1.0, [F] * (K + 1)), transcript=True)
        o = orc.call(sim_req(pr, "harness", K, 24, 1300 + rep, 1.0, [F] * (K + 1)))
        print(f"  rep {rep}: acc gpu {g.accepted_sum} oracle {o['accepted_sum']}  hits gpu {g.hits_total()}/{g.lookups()}"
              f" oracle {o['p_hits'] + o['b_hits']}/{o['p_lookups'] + o['b_lookups']}", flush=True)
        if rep == 0 and g.transcript:
            print("  transcript[0:3]:", g.transcript[:3], flush=True)
