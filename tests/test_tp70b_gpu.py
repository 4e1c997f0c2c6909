"""BASELINE configs[3] (Llama-3.1-70B target, tensor-parallel over 4 GPUs,
+ Llama-3.2-1B draft) at reduced depth: the EXACT 70B per-layer shapes
(d 8192, 64 / 8 heads, head_dim 128, FFN 28672, V 128256; 2 layers) sharded
TP=4 over four processes sharing cuda:0 (the same IPC peer-memory path the
NVLink peers use), against the unsharded engine and the CPU oracle:

* the TP logits (rank 0; every rank bit-identical) within the fp32 noise
  floor of the fp64 oracle, like the unsharded engine's;
* greedy AR and synchronous-SD streams of the colocated TP engine (target
  shard + replicated draft: the same-box baselines of the TP bench) are the
  oracle's greedy streams (teacher-forced);
* a split SSD run with the TP4 verifier + 1 speculator equals the unsharded
  colocated harness token for token (deterministic forwards on both).
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from parity import check_greedy_stream, logit_noise_check, near_tie_for

pytestmark = pytest.mark.gpu

TP = 4
K = 4


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shapes():
    from paper_2603_03251_b200.configs import shapes
    return shapes("llama70b_1b", max_ctx=256, target_layers=2, draft_layers=2)


def _prompt():
    return np.random.default_rng(70).integers(0, 128256, 12).tolist()


def _cfg(P, rounds=3):
    return P.SimConfig(lookahead=K, scheme=P.SamplingScheme.greedy(), primary_plan=P.FanOutPlan([4] * 5, P.PRIMARY),
                       backup_plan=P.FanOutPlan([4] * 5, P.BACKUP), primary_time=0.4, rounds=rounds, seed=3)


def _worker(rank, world, port, q, mode):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2603_03251_b200 as P
        from paper_2603_03251_b200 import _native as N
        from paper_2603_03251_b200.split import SplitEngine, exchange_handles
        ts, ds = _shapes()
        if mode == "baselines":  # colocated TP engines: target shard + replicated draft
            eng = P.Engine(ts, ds, P.Pair(), max_branches=20, max_lookahead=K, role=N.ROLE_COLOCATED, tp_rank=rank,
                           tp_size=world)
            eng.tp_connect(exchange_handles(eng.tp_handle()))
            dist.barrier()
            lg = eng.logits(0, _prompt())
            ar = eng.run_ar(_prompt(), P.SamplingScheme.greedy(), 8, 1).streams[0]
            sd = eng.run_sd(_prompt(), _cfg(P)).streams[0]
            eng.close()
            q.put((rank, "ok", lg, ar, sd))
        else:  # split SSD: ranks [0, TP) verifier, rank TP speculator
            se = SplitEngine(ts, ds, P.Pair(), device=0, max_branches=20, max_lookahead=K, tp=TP)
            r = se.run(_prompt(), _cfg(P))
            se.close()
            q.put((rank, "ok", None, r.tokens, r.merged))
    except Exception as e:
        import traceback
        traceback.print_exc()
        q.put((rank, f"{type(e).__name__}: {e}", None, None, None))
    finally:
        dist.destroy_process_group()


def _launch(world, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, mode)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=1500)
        res[r[0]] = r[1:]
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert res[r][0] == "ok", (r, res[r][0])
    return res


@pytest.fixture(scope="module")
def reference(oracle_lib):
    import paper_2603_03251_b200 as P
    ts, ds = _shapes()
    os.environ["SSD_B200_DETERMINISTIC"] = "1"
    try:
        eng = P.Engine(ts, ds, P.Pair(), max_branches=20, max_lookahead=K)
    finally:
        del os.environ["SSD_B200_DETERMINISTIC"]
    orc = oracle_lib.TfPair(P.shape_dict(ts), P.shape_dict(ds), P.Pair().as_dict())
    o64 = oracle_lib.TfPair(P.shape_dict(ts), P.shape_dict(ds), P.Pair().as_dict(), accum="f64")
    yield P, eng, orc, o64
    eng.close()
    orc.close()
    o64.close()


def test_tp4_70b_width_logits_and_baselines(reference):
    P, eng, orc, o64 = reference
    res = _launch(TP, "baselines")
    for r in range(1, TP):  # every rank computes the same (ordered all-reduce sums)
        assert np.array_equal(res[0][1], res[r][1]) and res[0][2] == res[r][2] and res[0][3] == res[r][3]
    tp_lg = res[0][1]
    out = logit_noise_check(lambda which, ctx: tp_lg, orc, o64, 0, [_prompt()])
    print("TP4 logit noise", out)
    ref = logit_noise_check(eng.logits, orc, o64, 0, [_prompt()])
    print("unsharded logit noise", ref)
    tie = near_tie_for(orc, o64, [_prompt()], (0,))
    check_greedy_stream(orc, 0, _prompt(), res[0][2], near_tie=tie)
    check_greedy_stream(orc, 0, _prompt(), res[0][3], near_tie=tie)  # greedy SD is lossless: the target's stream


def test_tp4_split_ssd_matches_colocated(reference):
    P, eng, orc, o64 = reference
    res = _launch(TP + 1, "split")
    tokens, merged = res[0][2], res[0][3]
    for r in range(1, TP):
        assert res[r][2] == tokens
    check_greedy_stream(orc, 0, _prompt(), tokens, near_tie=near_tie_for(orc, o64, [_prompt()], (0,)))
    ref = eng.run_ssd(_prompt(), _cfg(P))
    assert merged["rounds"] == 3 and merged["tokens"] == len(tokens)
    if tokens == ref.streams[0]:
        for f in ("accepted_sum", "primary_origin_hits", "backup_origin_hits", "hit_rounds", "miss_rounds"):
            assert merged[f] == getattr(ref, f), f
