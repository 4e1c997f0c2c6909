"""Diagnostic for the tensor-parallel verifier collectives: TP=2 ranks as
processes sharing cuda:0 run the same logits call repeatedly; every call is
compared with the CPU oracle (max |diff|) to localise a failing collective."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import torch.multiprocessing as mp  # noqa: E402

import test_tp_gpu as T  # noqa: E402


def worker(rank, world, port, q, n):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2603_03251_b200 as P
    from paper_2603_03251_b200 import _native as N
    from paper_2603_03251_b200.configs import shapes
    from paper_2603_03251_b200.split import exchange_handles
    ts, ds = shapes("tiny", max_ctx=512)
    eng = P.Engine(ts, ds, P.Pair(), max_branches=8, max_lookahead=4, role=N.ROLE_VERIFIER, tp_rank=rank, tp_size=world)
    eng.tp_connect(exchange_handles(eng.tp_handle()))
    dist.barrier()
    out = [eng.logits(0, T._prompt()) for _ in range(n)]
    eng.close()
    q.put((rank, out))
    dist.destroy_process_group()


def main():
    import paper_2603_03251_b200 as P
    from paper_2603_03251_b200.configs import shapes
    import pyoracle
    ts, ds = shapes("tiny", max_ctx=512)
    orc = pyoracle.TfPair(P.shape_dict(ts), P.shape_dict(ds), P.Pair().as_dict())
    olg = orc.logits(0, T._prompt())
    for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = T._free_port()
        procs = [ctx.Process(target=worker, args=(r, 2, port, q, 6)) for r in range(2)]
        for p in procs:
            p.start()
        res = dict(q.get(timeout=600) for _ in range(2))
        for p in procs:
            p.join(timeout=120)
        h = len(olg) // 2
        print(it, [(round(float(np.max(np.abs(x[:h] - olg[:h]))), 3), round(float(np.max(np.abs(x[h:] - olg[h:]))), 3))
                   for x in res[0][:2]],
              [bool(np.array_equal(a, b)) for a, b in zip(res[0], res[1])], flush=True)


if __name__ == "__main__":
    main()
