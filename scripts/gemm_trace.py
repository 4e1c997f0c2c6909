"""Per-stage timeline of CTA 0 of the last GEMM of a forward (trace build)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

os.environ.setdefault("SSD_B200_LIB", os.path.join(ROOT, "paper_2603_03251_b200", "libssd_b200_trace.so"))
from paper_2603_03251_b200 import _build  # noqa: E402
if not os.path.exists(os.environ["SSD_B200_LIB"]):
    _build.build_variant("trace", ["SSD_GEMM_TRACE=1"])
import paper_2603_03251_b200 as P  # noqa: E402
from paper_2603_03251_b200.configs import shapes  # noqa: E402

ts, ds = shapes("llama8b_1b", max_ctx=1024)
e = P.Engine(ts, ds, P.Pair(), max_branches=20, max_lookahead=4)
M = int(sys.argv[1]) if len(sys.argv) > 1 else 1
e.profile_forward(0, M, 128, 3)  # last GEMM: the 8B LM head (M tokens)
buf = (C.c_ulonglong * (5 * 512))()
e.lib.ssd_debug_gemm_trace(buf)
t = np.array(buf, dtype=np.float64).reshape(5, 512)
t0 = t[4][0]
n = int((t[0] > 0).sum())
print("units traced", n, "kernel span us", (t[4][1] - t0) / 1e3)
iss, full, com, emp = [(t[r][:n] - t0) / 1e3 for r in range(4)]
for i in list(range(0, 14)) + list(range(n - 4, n)):
    print(f"unit {i:3d} issue {iss[i]:8.2f} full {full[i]:8.2f} commit {com[i]:8.2f} empty_seen {emp[i]:8.2f}")
lat = full[:n] - iss[:n]
print("issue->full latency us: median %.2f p90 %.2f" % (np.median(lat), np.percentile(lat, 90)))
gaps = np.diff(full[:n])
print("MMA-side unit interval us: median %.3f mean %.3f" % (np.median(gaps), gaps.mean()))
mma = com[:n] - full[:n]
print("MMA full->commit us: median %.3f" % np.median(mma))
rec = emp[S:n] - com[:n - S] if (S := int(os.environ.get("STAGES", "6"))) < n else np.array([0.0])
print("commit(i) -> producer saw empty (i+S) us: median %.3f" % np.median(rec))
