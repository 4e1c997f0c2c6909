"""Persistent forward kernel vs the per-op kernel path (SSD_B200_MK=0 in a
child process) on the tiny pair and the 8B/1B shapes: logits agreement and
step times."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402


def run(cfg, mk):
    code = f"""
import sys, numpy as np
sys.path.insert(0, {ROOT!r})
import paper_2603_03251_b200 as P
from paper_2603_03251_b200.configs import shapes
ts, ds = shapes({cfg!r}, max_ctx=1024)
eng = P.Engine(ts, ds, P.Pair(), max_branches=20, max_lookahead=4)
prompt = np.random.default_rng(3).integers(0, ts.vocab, 40).tolist()
try:
    lt = eng.logits(0, prompt); ld = eng.logits(1, prompt)
except Exception as e:
    import ctypes
    lib = P._native.load()
    buf = (ctypes.c_ulonglong * (8 + 8 * 256))()
    lib.ssd_debug_mk_diag(buf)
    d = list(buf)
    print("FAILED", e, "diag", d[:8], flush=True)
    import collections
    for role in range(7):
        prog = [d[8 + 8 * c + role] - 1 for c in range(148)]
        if role >= 3:
            prog = [(x // 16, x % 16) if x >= 0 else (-1, 0) for x in prog]
        print("role", role, "histogram", sorted(collections.Counter(prog).items()), flush=True)
        print("   min ctas", [c for c in range(148) if prog[c] == min(prog)][:20], flush=True)
    raise
np.save('/tmp/mk_{cfg}_{mk}_t.npy', lt); np.save('/tmp/mk_{cfg}_{mk}_d.npy', ld)
for name, which, M in (("t1", 0, 1), ("t5", 0, 5), ("d1", 1, 1), ("d20", 1, 20)):
    r = eng.profile_forward(which, M, 128, 10)
    print(name, round(r["ms_forward"], 4), round(r["ms_gemm"], 4), flush=True)
eng.close()
"""
    env = dict(os.environ, SSD_B200_MK=str(mk))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=int(os.environ.get('MK_TIMEOUT', '600')))
    print(f"--- {cfg} MK={mk} rc={out.returncode}\n{out.stdout}{out.stderr[-2000:]}", flush=True)


for cfg in sys.argv[1].split(","):
    for mk in (0, 1):
        run(cfg, mk)
    for w in "td":
        a, b = np.load(f"/tmp/mk_{cfg}_0_{w}.npy"), np.load(f"/tmp/mk_{cfg}_1_{w}.npy")
        print(cfg, w, "max|mk - per-op| =", float(np.max(np.abs(a - b))), "argmax equal:", int(a.argmax()) == int(b.argmax()))
