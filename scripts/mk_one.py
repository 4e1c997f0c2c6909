"""One persistent-forward launch (tiny target prefill of 40 tokens) for
compute-sanitizer runs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2603_03251_b200 as P  # noqa: E402
from paper_2603_03251_b200.configs import shapes  # noqa: E402

ts, ds = shapes(sys.argv[1] if len(sys.argv) > 1 else "tiny", max_ctx=int(sys.argv[3]) if len(sys.argv) > 3 else 512)
eng = P.Engine(ts, ds, P.Pair(), max_branches=20, max_lookahead=4)
prompt = np.random.default_rng(3).integers(0, ts.vocab, int(sys.argv[2]) if len(sys.argv) > 2 else 40).tolist()
lt = eng.logits(0, prompt)
print("ok", float(lt[:4].sum()))
eng.close()
