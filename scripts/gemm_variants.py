"""GEMM configuration sweep on the GPU: achievable read bandwidth, then the
decode-step GEMM bandwidth (8B target M=1, 1B draft M=5 / M=20) for each
compiled variant of libssd_b200 (SSD_B200_LIB selects the library)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(lib):
    code = f"""
import os, sys, json
os.environ['SSD_B200_LIB'] = {lib!r}
sys.path.insert(0, {ROOT!r})
import paper_2603_03251_b200 as P
from paper_2603_03251_b200.configs import shapes
ts, ds = shapes('llama8b_1b', max_ctx=1024)
e = P.Engine(ts, ds, P.Pair(), max_branches=20, max_lookahead=4)
out = {{'lib': os.path.basename({lib!r}), 'read_bw': e.read_bw(4 << 30, 10)}}
for name, which, M in (('t_m1', 0, 1), ('t_m5', 0, 5), ('d_m1', 1, 1), ('d_m5', 1, 5), ('d_m20', 1, 20)):
    p = e.profile_forward(which, M, 128, 10)
    out[name] = {{'gemm_gbs': p['gemm_bytes'] / (p['ms_gemm'] * 1e-3) / 1e9, 'ms_gemm': p['ms_gemm'],
                  'ms_fwd': p['ms_forward']}}
print(json.dumps(out))
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    return r.stdout.strip() or r.stderr[-2000:]


if __name__ == "__main__":
    libs = sys.argv[1:] or [os.path.join(ROOT, "paper_2603_03251_b200", "libssd_b200.so")]
    for lib in libs:
        print(one(lib), flush=True)
