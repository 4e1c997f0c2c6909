"""TMA bulk-copy streaming probe sweep (pattern x block size x depth x CTAs/SM)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import ctypes as C  # noqa: E402

import paper_2603_03251_b200 as P  # noqa: E402
from paper_2603_03251_b200.configs import shapes  # noqa: E402

ts, ds = shapes("tiny", max_ctx=256)
e = P.Engine(ts, ds, P.Pair(), max_branches=4, max_lookahead=2)
lib = e.lib
res = {"read_bw": e.read_bw(2 << 30, 10)}
for mode in (0, 1):
    for blk, stages, cps in ((16384, 6, 1), (16384, 12, 1), (32768, 6, 1), (16384, 6, 2), (32768, 3, 2),
                             (65536, 3, 1), (16384, 12, 2), (8192, 24, 1)):
        g = C.c_double()
        st = lib.ssd_bench_tma_stream(e.h, 2 << 30, blk, stages, mode, cps, 10, C.byref(g))
        res[f"m{mode}_b{blk // 1024}k_s{stages}_c{cps}"] = round(g.value) if st == 0 else lib.ssd_last_error().decode()
print(json.dumps(res))
