"""One forward of the target (M=1 decode, M=5 verify) and of the draft
(M=20 branch step) after engine build: the window for ncu launch lists and
full captures (kernels launched directly, no graph)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_03251_b200 as P  # noqa: E402
from paper_2603_03251_b200.configs import shapes  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "t1,t5,d20"
ts, ds = shapes("llama8b_1b", max_ctx=1024)
eng = P.Engine(ts, ds, P.Pair(), max_branches=20, max_lookahead=4)
for w in what.split(","):
    which, M = (0 if w[0] == "t" else 1), int(w[1:])
    r = eng.profile_forward(which, M, 128, 1)
    print(w, r, flush=True)
eng.close()
