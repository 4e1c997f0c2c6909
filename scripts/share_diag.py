"""Diagnostic: two processes sharing cuda:0, each with an UNSHARDED tiny
engine, compute the same logits repeatedly (first call included); every call
is compared with the CPU oracle. Separates GPU-sharing effects from the
tensor-parallel collectives (scripts/tp_diag.py)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import torch.multiprocessing as mp  # noqa: E402

import test_tp_gpu as T  # noqa: E402


def worker(rank, q, n):
    import paper_2603_03251_b200 as P
    from paper_2603_03251_b200.configs import shapes
    ts, ds = shapes("tiny", max_ctx=512)
    eng = P.Engine(ts, ds, P.Pair(), max_branches=8, max_lookahead=4)
    out = [eng.logits(0, T._prompt()) for _ in range(n)]
    eng.close()
    q.put((rank, out))


def main():
    import paper_2603_03251_b200 as P
    from paper_2603_03251_b200.configs import shapes
    import pyoracle
    ts, ds = shapes("tiny", max_ctx=512)
    orc = pyoracle.TfPair(P.shape_dict(ts), P.shape_dict(ds), P.Pair().as_dict())
    olg = orc.logits(0, T._prompt())
    nproc = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        procs = [ctx.Process(target=worker, args=(r, q, 3)) for r in range(nproc)]
        for p in procs:
            p.start()
        res = dict(q.get(timeout=600) for _ in range(nproc))
        for p in procs:
            p.join(timeout=120)
        print(it, [[round(float(np.max(np.abs(x - olg))), 3) for x in res[r]] for r in range(nproc)], flush=True)


if __name__ == "__main__":
    main()
