"""Timeline of one persistent forward (fwd_mk.cuh trace): per op, the
latest B-ready / first-MMA / epilogue-done times over CTAs, relative to the
kernel's first event, and the op's duration (last arrival - previous)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2603_03251_b200 as P  # noqa: E402
from paper_2603_03251_b200.configs import shapes  # noqa: E402

KIND = ["EMBED", "QKV", "ATTN", "O", "GU", "DN", "HEAD", "NORM"]
cfgname, which, M = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
ts, ds = shapes(cfgname, max_ctx=1024)
eng = P.Engine(ts, ds, P.Pair(), max_branches=20, max_lookahead=4)
lib = P._native.load()
cap = 1000 * 148 * 4
buf = (ctypes.c_ulonglong * cap)()
kinds = (ctypes.c_int * 1000)()
uops = (ctypes.c_int * 4)(9, 11, 13, 14)  # layer 1: QKV, O, GU, DN
ubuf = (ctypes.c_ulonglong * (4 * 64 * 4))()
n = lib.ssd_debug_mk_trace(eng.h, which, M, 128, buf, cap, kinds, uops, ubuf)
assert n > 0, n
t = np.array(buf[: n * 148 * 4], dtype=np.float64).reshape(n, 148, 4)
t[t == 0] = np.nan
t0 = np.nanmin(t)
t = (t - t0) / 1e3  # us
prev = 0.0
rows = []
for p in range(n):
    done = np.nanmax(t[p, :, 2]) if p + 1 < n else np.nanmax(t[p, :, 1])
    first_w = np.nanmin(t[p, :, 3]) if not np.all(np.isnan(t[p, :, 3])) else float("nan")
    bready = np.nanmax(t[p, :, 0]) if not np.all(np.isnan(t[p, :, 0])) else float("nan")
    mma0 = np.nanmin(t[p, :, 1]) if not np.all(np.isnan(t[p, :, 1])) else float("nan")
    rows.append((p, KIND[kinds[p]], done - prev, bready, mma0, first_w, done))
    prev = done
tot = {}
for r in rows:
    tot[r[1]] = tot.get(r[1], 0) + r[2]
print("op-kind totals (us):", {k: round(v, 1) for k, v in tot.items()}, "sum", round(sum(tot.values()), 1))
for r in rows[:12] + rows[-3:]:
    print(f"op {r[0]:3d} {r[1]:5s} dur {r[2]:8.1f}  B-ready(max) {r[3]:8.1f}  MMA0(min) {r[4]:8.1f}  W0(min) {r[5]:8.1f}  done(max) {r[6]:8.1f}")
eng.close()

u = np.array(ubuf[:], dtype=np.float64).reshape(4, 64, 4)
for j in range(4):
    v = u[j]
    ok = v[:, 0] > 0
    if not ok.any():
        continue
    base = v[ok][:, :3].min()
    print(f"per-unit (CTA 0) op {uops[j]} {KIND[kinds[uops[j]]]}: us rel. [W issued, B in, MMA full, epi tile]")
    for i in np.nonzero(ok)[0][:16]:
        print("   unit", i, np.round((v[i] - base) / 1e3, 2).tolist())
