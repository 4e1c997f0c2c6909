"""Timeline of one persistent-kernel forward of the draft (SSD_B200_PK_TRACE=1):
for the first 16 ops of the launch (embedding + 2.5 layers), the span over
all CTAs of each phase, in us from the first CTA's entry."""
import ctypes
import os
import sys

import numpy as np

os.environ["SSD_B200_PK_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_03251_b200 as P  # noqa: E402
from paper_2603_03251_b200.configs import shapes  # noqa: E402

NAMES = ["EMBED"] + [n for _ in range(2) for n in ("QKV", "APPEND", "ATTN", "O", "NORM", "GU", "SWIGLU", "DN", "NORM")]
cfg = os.environ.get("PK_CFG", "llama8b_1b")
ts, ds = shapes(cfg, max_ctx=1024)
eng = P.Engine(ts, ds, P.Pair(), max_branches=20, max_lookahead=4)
lib = P._native.load()
lib.ssd_debug_pk_trace.restype = ctypes.c_int
SLOTS = 2 + 6 * 16
n = 148 * SLOTS
buf = (ctypes.c_ulonglong * n)()
for w in (sys.argv[1:] or ["d1", "d20"]):
    M = int(w[1:])
    eng.profile_forward(1, M, 256, 2)
    got = lib.ssd_debug_pk_trace(eng.h, buf, n)
    assert got == n, got
    t = np.array(buf, dtype=np.float64).reshape(148, SLOTS)
    ent = t[:, 0][t[:, 0] > 0]
    t0 = ent.min()
    ex = t[:, 1][t[:, 1] > 0]
    print(f"== {w}: entry +{(ent.max()-t0)/1e3:.2f}  exit {(ex.min()-t0)/1e3:.2f}..{(ex.max()-t0)/1e3:.2f} us")

    def span(v):
        v = v[v > 0]
        return f"{(v.min()-t0)/1e3:7.2f}..{(v.max()-t0)/1e3:7.2f}" if len(v) else "        -       "
    for p in range(16):
        ph = t[:, 2 + 6 * p: 8 + 6 * p]
        print(f"  op{p:2d} {NAMES[p]:6s} w {span(ph[:, 0])} -> {span(ph[:, 1])} | dep {span(ph[:, 2])} | "
              f"mma0 {span(ph[:, 3])} | mma1 {span(ph[:, 4])} | done {span(ph[:, 5])}")
for M in (1, 5, 20):
    r = eng.profile_forward(1, M, 256, 20)
    print(f"d{M}: {r['ms_forward']:.4f} ms")
eng.close()
