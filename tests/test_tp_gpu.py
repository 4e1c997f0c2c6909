"""Tensor-parallel verifier: TP ranks as separate
processes (here sharing cuda:0 — the same IPC / peer-memory path NVLink
peers use), Megatron-sharded synthetic weights, all-reduces and the logits
all-gather as peer-memory kernels. Logits must match the unsharded engine to
fp32-summation noise and greedy decoding must produce the same tokens."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _prompt():
    return np.random.default_rng(21).integers(0, 32000, 24).tolist()


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2603_03251_b200 as P
        from paper_2603_03251_b200 import _native as N
        from paper_2603_03251_b200.configs import shapes
        from paper_2603_03251_b200.split import exchange_handles
        ts, ds = shapes("tiny", max_ctx=512)
        eng = P.Engine(ts, ds, P.Pair(), max_branches=8, max_lookahead=4, role=N.ROLE_VERIFIER, tp_rank=rank,
                       tp_size=world)
        eng.tp_connect(exchange_handles(eng.tp_handle()))
        dist.barrier()
        lg = eng.logits(0, _prompt())
        ar = eng.run_ar(_prompt(), P.SamplingScheme.greedy(), 12, 3)
        eng.close()
        q.put((rank, "ok", lg, ar.streams[0]))
    except Exception as e:
        q.put((rank, f"{type(e).__name__}: {e}", None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("tp", [2])
def test_tp_verifier_matches_unsharded(tp):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, tp, port, q)) for r in range(tp)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(tp):
        rank, status, lg, toks = q.get(timeout=600)
        res[rank] = (status, lg, toks)
    for p in procs:
        p.join(timeout=120)
    bad = {r: v[0] for r, v in res.items() if v[0] != "ok"}
    assert not bad, bad
    import paper_2603_03251_b200 as P
    from paper_2603_03251_b200.configs import shapes
    ts, ds = shapes("tiny", max_ctx=512)
    os.environ["SSD_B200_DETERMINISTIC"] = "1"  # the TP ranks' fixed-order forward, unsharded
    try:
        eng = P.Engine(ts, ds, P.Pair(), max_branches=8, max_lookahead=4)
    finally:
        del os.environ["SSD_B200_DETERMINISTIC"]
    ref_lg = eng.logits(0, _prompt())
    ref_toks = eng.run_ar(_prompt(), P.SamplingScheme.greedy(), 12, 3).streams[0]
    eng.close()
    # every TP rank computes the same (all-reduce sums ranks in rank order)
    for r in range(1, tp):
        assert np.array_equal(res[0][1], res[r][1]) and res[0][2] == res[r][2]
    assert float(np.max(np.abs(res[0][1] - ref_lg))) < 1e-2
    assert int(np.argmax(res[0][1])) == int(np.argmax(ref_lg))
    assert res[0][2] == ref_toks
