"""Regression for round 1's "corrupt first forward": the
first API call of a FRESH process must be exact, also while other processes
load the same GPU. Root cause (fixed): the per-call host->device copies ran
as synchronous cudaMemcpy on the legacy stream, which the engine's
non-blocking streams do not wait for, and a pageable H2D copy can return
before its DMA lands — the first forward could read the zero-initialised
history. Every copy is now stream-ordered on the engine stream.

24 fresh processes (waves of 4 sharing cuda:0, plus one process running a
decode loop as background load); each compares its FIRST `logits` call and
its first greedy `run_ssd` stream against the CPU oracle. No warm-up."""
import multiprocessing as mp
import os
import sys

import numpy as np
import pytest

from parity import check_greedy_stream

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WAVES, PER_WAVE = 6, 4
CORRUPT_TOL = 0.1


def _prompt(i):
    return np.random.default_rng(1000 + i).integers(0, 32000, 9 + i % 7).tolist()


def _cfg(P):
    return P.SimConfig(lookahead=4, scheme=P.SamplingScheme.greedy(), primary_plan=P.FanOutPlan([4] * 5, P.PRIMARY),
                       backup_plan=P.FanOutPlan([4] * 5, P.BACKUP), primary_time=0.4, rounds=4, seed=3)


def _worker(i, q):
    sys.path.insert(0, ROOT)
    try:
        import paper_2603_03251_b200 as P
        from paper_2603_03251_b200.configs import shapes
        ts, ds = shapes("tiny", max_ctx=512)
        eng = P.Engine(ts, ds, P.Pair(), max_branches=20, max_lookahead=4)
        lg = eng.logits(i % 2, _prompt(i))  # the process's first forward
        st = eng.run_ssd(_prompt(i), _cfg(P)).streams[0]
        eng.close()
        q.put((i, "ok", lg, st))
    except Exception as e:  # surface in the parent
        q.put((i, f"{type(e).__name__}: {e}", None, None))


def _load(stop):
    sys.path.insert(0, ROOT)
    import paper_2603_03251_b200 as P
    from paper_2603_03251_b200.configs import shapes
    ts, ds = shapes("tiny", max_ctx=1024)
    eng = P.Engine(ts, ds, P.Pair(), max_branches=20, max_lookahead=4)
    while not stop.is_set():
        eng.run_ar(_prompt(0), P.SamplingScheme.greedy(), 256, 1)
    eng.close()


def test_first_call_of_fresh_processes_is_exact(oracle_lib):
    import paper_2603_03251_b200 as P
    from paper_2603_03251_b200.configs import shapes
    ts, ds = shapes("tiny", max_ctx=512)
    orc = oracle_lib.TfPair(P.shape_dict(ts), P.shape_dict(ds), P.Pair().as_dict())
    ctx = mp.get_context("spawn")
    stop = ctx.Event()
    loader = ctx.Process(target=_load, args=(stop,))
    loader.start()
    bad = []
    try:
        for w in range(WAVES):
            q = ctx.Queue()
            ids = list(range(w * PER_WAVE, (w + 1) * PER_WAVE))
            procs = [ctx.Process(target=_worker, args=(i, q)) for i in ids]
            for p in procs:
                p.start()
            res = [q.get(timeout=600) for _ in ids]
            for p in procs:
                p.join(timeout=120)
            for i, status, lg, st in res:
                assert status == "ok", (i, status)
                err = float(np.max(np.abs(lg - orc.logits(i % 2, _prompt(i)))))
                # corruption (a stale history / plan) moves logits by O(1-10);
                # fp32 summation-order noise of the tiny pair is ~1e-2. The
                # greedy stream is checked teacher-forced against the oracle
                # (a divergence only at a documented near-tie: parity.py)
                try:
                    check_greedy_stream(orc, 0, _prompt(i), list(st))
                    stream_ok = True
                except AssertionError as e:
                    stream_ok = str(e)
                if err >= CORRUPT_TOL or stream_ok is not True:
                    bad.append((i, err, list(st)[:6], stream_ok))
    finally:
        stop.set()
        loader.join(timeout=120)
        orc.close()
    assert not bad, bad
