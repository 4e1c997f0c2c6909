"""L2 prefetch look-ahead sweep (SSD_B200_PF_MB): forward-step times of the
8B target (M=1, M=5) and 1B draft (M=1, M=20), and AR / SD / SSD decode
tokens/s on the bench workload."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2603_03251_b200 as P  # noqa: E402
from paper_2603_03251_b200.configs import shapes  # noqa: E402

vals = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["0", "16", "32", "64"])]
ts, ds = shapes("llama8b_1b", max_ctx=1024)
prompt = np.random.default_rng(20250809).integers(0, ts.vocab, 128).tolist()
for mb in vals:
    os.environ["SSD_B200_PF_MB"] = str(mb)
    eng = P.Engine(ts, ds, P.Pair(), max_branches=20, max_lookahead=4)
    res = {}
    for name, which, M in (("t1", 0, 1), ("t5", 0, 5), ("d1", 1, 1), ("d20", 1, 20)):
        r = eng.profile_forward(which, M, 128, 20)
        res[name] = (round(r["ms_forward"], 3), round(r["ms_gemm"], 3))
    cfg = P.SimConfig(lookahead=4, scheme=P.SamplingScheme.greedy(), primary_plan=P.FanOutPlan([4] * 5, P.PRIMARY),
                      backup_plan=P.FanOutPlan([4] * 5, P.BACKUP), primary_time=0.4, rounds=24, seed=1)
    eng.run_ar(prompt, P.SamplingScheme.greedy(), 8, 1)
    ar = eng.run_ar(prompt, P.SamplingScheme.greedy(), 48, 1)
    sd = eng.run_sd(prompt, cfg)
    ssd = eng.run_ssd(prompt, cfg)
    print(f"PF={mb}MB fwd(ms fwd, ms gemm)={res} AR={ar.tokens_per_second():.1f} SD={sd.tokens_per_second():.1f} "
          f"SSD={ssd.tokens_per_second():.1f} ssd_round_ms={ssd.device_ms / ssd.rounds:.2f} hit={ssd.hit_rate():.2f}",
          flush=True)
    eng.close()
