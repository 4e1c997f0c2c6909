"""Forward-step time with kernel classes dropped (profiling only; the
results are numerically wrong): how much of a decode step is norms /
attention in the pipelined (PDL) setting."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = """
import os, sys, json
sys.path.insert(0, %r)
import paper_2603_03251_b200 as P
from paper_2603_03251_b200.configs import shapes
ts, ds = shapes('llama8b_1b', max_ctx=1024)
e = P.Engine(ts, ds, P.Pair(), max_branches=20, max_lookahead=4)
out = {'skip': os.environ.get('SSD_B200_SKIP', '0')}
for name, which, M in (('t_m1', 0, 1), ('t_m5', 0, 5), ('d_m1', 1, 1), ('d_m20', 1, 20)):
    p = e.profile_forward(which, M, 128, 10)
    out[name] = [round(p['ms_forward'], 3), round(p['ms_gemm'], 3)]
print(json.dumps(out))
""" % ROOT
for mask in ("0", "1", "2", "3"):
    env = dict(os.environ, SSD_B200_SKIP=mask)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
    print(r.stdout.strip() or r.stderr[-1500:], flush=True)
