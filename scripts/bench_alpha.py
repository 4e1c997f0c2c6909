"""Acceptance of the correlated 8B/1B pair on the bench workload itself
(bench.py's prompt and seed) vs block_out_scale: picks the pair knob that
puts the bench near alpha ~ 0.8 (SURVEY §7 hard part 1)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2603_03251_b200 as P  # noqa: E402
from paper_2603_03251_b200.configs import shapes  # noqa: E402

sys.path.insert(0, ROOT)
from bench import alpha_of  # noqa: E402

seed = 20250809
ts, ds = shapes("llama8b_1b", max_ctx=1024)
prompt = np.random.default_rng(seed).integers(0, ts.vocab, 128).tolist()
for bos in [float(x) for x in sys.argv[1].split(",")]:
    eng = P.Engine(ts, ds, P.Pair(block_out_scale=bos), max_branches=20, max_lookahead=4)
    cfg = P.SimConfig(lookahead=4, scheme=P.SamplingScheme.greedy(), primary_plan=P.FanOutPlan([4] * 5, P.PRIMARY),
                      backup_plan=P.FanOutPlan([4] * 5, P.BACKUP), primary_time=0.4, backup_kind=P.FAST_RANDOM,
                      rounds=32, seed=seed)
    sd = eng.run_sd(prompt, cfg)
    ssd = eng.run_ssd(prompt, cfg)
    ar = eng.run_ar(prompt, P.SamplingScheme.greedy(), 64, seed)
    acc = ssd.accepted_sum / ssd.rounds
    print(f"bos={bos} SSD acc={acc:.3f} alpha={alpha_of(acc, 4):.3f} hit={ssd.hit_rate():.3f} "
          f"tok/s AR={ar.tokens_per_second():.1f} SD={sd.tokens_per_second():.1f} SSD={ssd.tokens_per_second():.1f} "
          f"SD acc={sd.accepted_sum / sd.rounds:.3f}", flush=True)
    eng.close()
