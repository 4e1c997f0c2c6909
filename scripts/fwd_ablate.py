"""Forward-step timings (CUDA events, direct PDL launches, 20 iterations) of
the 8B target (M=1, 5) and the 1B draft (M=1, 5, 20) under the current
environment knobs (SSD_B200_SKIP / SSD_B200_MK / ...): the ablation table
that says where a step's time goes."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_03251_b200 as P  # noqa: E402
from paper_2603_03251_b200.configs import shapes  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "t1,t5,d1,d5,d20"
ts, ds = shapes("llama8b_1b", max_ctx=1024)
eng = P.Engine(ts, ds, P.Pair(), max_branches=20, max_lookahead=4)
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("SSD_B200_")) or "default"
for w in what.split(","):
    which, M = (0 if w[0] == "t" else 1), int(w[1:])
    r = eng.profile_forward(which, M, 256, 20)
    print(json.dumps({"env": tag, "fwd": w, "ms_forward": round(r["ms_forward"], 4), "ms_gemm": round(r["ms_gemm"], 4)}),
          flush=True)
eng.close()
