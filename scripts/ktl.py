"""Real (PDL-overlapped) timeline of decode-step kernels from the profiling
build (-DSSD_KTL=1): block 0 of each kernel stamps entry / after-PDL-wait /
exit. Usage: python scripts/ktl.py [t1|d1|d20 ...] (builds the variant)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["SSD_B200_LIB"] = os.path.join(ROOT, "paper_2603_03251_b200", "libssd_b200_ktl.so")  # before the import
from paper_2603_03251_b200 import _build  # noqa: E402

if not os.path.exists(os.environ["SSD_B200_LIB"]):
    _build.build_variant("ktl", ["SSD_KTL=1"])
import numpy as np  # noqa: E402

import paper_2603_03251_b200 as P  # noqa: E402
from paper_2603_03251_b200.configs import shapes  # noqa: E402

KIND = {1: "embed", 2: "rmsnorm", 3: "attention", 4: "attention_dec", 10: "gemm", 11: "gemm_resid", 12: "gemm_swiglu",
        20: "gemm_cl", 21: "gemm_cl_resid", 22: "gemm_cl_swiglu"}
ts, ds = shapes("llama8b_1b", max_ctx=1024)
eng = P.Engine(ts, ds, P.Pair(), max_branches=20, max_lookahead=4)
lib = P._native.load()
lib.ssd_debug_ktl.restype = ctypes.c_int
NBUF = 16384 * 4 + 16 + 64 * 160 * 8
buf = (ctypes.c_ulonglong * NBUF)()
for w in (sys.argv[1:] or ["t1", "d1", "d20"]):
    which, M = (0 if w[0] == "t" else 1), int(w[1:])
    eng.profile_forward(which, M, 128, 2)
    lib.ssd_debug_ktl(buf, NBUF)  # reset
    eng.profile_forward(which, M, 128, 1)  # warm forward + gemms + forward + gemms
    n = lib.ssd_debug_ktl(buf, NBUF)
    assert n > 0, f"no timeline records ({n}): not the SSD_KTL build?"
    sub = np.array(buf[n * 4: n * 4 + 16], dtype=np.float64)
    cta = np.array(buf[n * 4 + 16: n * 4 + 16 + 64 * 160 * 8], dtype=np.float64).reshape(64, 160, 8)
    t = np.array(buf[: n * 4], dtype=np.float64).reshape(n, 4)
    t = t[np.argsort(t[:, 1])]
    # the last full forward: from the last embed to the next embed / end, cut at the GEMM-only pass
    emb = np.nonzero(t[:, 0] == 1)[0]
    f = t[emb[-1]:]
    n_gemm = 4 * (ts.n_layers if which == 0 else ds.n_layers) + 1
    k, g = 0, 0
    while k < len(f) and g < n_gemm:
        g += f[k, 0] >= 10
        k += 1
    f = f[:k]
    t0 = f[0, 1]
    print(f"== {w}: {len(f)} kernels, block-0 span {(f[-1, 3] - t0) / 1e3:.1f} us")
    agg = {}
    prev_exit = None
    for r in f:
        kind = KIND.get(int(r[0]), str(int(r[0])))
        wait = (r[2] - r[1]) / 1e3
        work = (r[3] - r[2]) / 1e3
        gap = (r[1] - prev_exit) / 1e3 if prev_exit is not None else 0.0
        a = agg.setdefault(kind, [0, 0.0, 0.0, 0.0])
        a[0] += 1; a[1] += wait; a[2] += work; a[3] += gap
        prev_exit = r[3]
    for kind, a in agg.items():
        print(f"   {kind:12s} n={a[0]:4d} entry->ready {a[1] / a[0]:7.2f} us  ready->exit(block0) {a[2] / a[0]:7.2f} us  "
              f"prev-exit->entry {a[3] / a[0]:7.2f} us")
    print("   last attention sub-phases (us from ready; attention_dec: setup, scores, softmax, PV, out): %.2f %.2f %.2f %.2f "
          "%.2f %.2f %.2f" % tuple((sub[i] - sub[0]) / 1e3 for i in range(1, 8)))
    # per-CTA spread of the last GEMM launches of this workload (ready / MMA done / exit), us rel. to min ready
    print("   per-CTA GEMM spreads (last launches): [ready span, last MMA-done - first ready, exit span, last exit - max MMA done]")
    for j in range(64):
        c = cta[j]
        ok = c[:, 0] > 0
        if ok.sum() < 8:
            continue
        r0 = c[ok, 0].min()
        last = int(np.argmax(np.where(ok, c[:, 2], 0)))  # the CTA that exits last
        rel = lambda v: (v - c[last, 1]) / 1e3 if v > 0 else float("nan")  # noqa: E731
        print("     launch %2d mma-done %6.2f tail %6.2f | last CTA %3d: mma-complete %+.2f tfull %+.2f drained %+.2f arrived %+.2f reduced %+.2f exit %+.2f" % (
            j, (c[ok, 1].max() - r0) / 1e3, (c[ok, 2].max() - c[ok, 1].max()) / 1e3, last, rel(c[last, 7]),
            rel(c[last, 3]), rel(c[last, 4]), rel(c[last, 5]), rel(c[last, 6]), rel(c[last, 2])))
    for r in f[:24]:
        print(f"      {str(KIND.get(int(r[0]), int(r[0]))):12s} entry {(r[1] - t0) / 1e3:8.2f} ready {(r[2] - t0) / 1e3:8.2f} "
              f"exit {(r[3] - t0) / 1e3:8.2f}")
eng.close()


