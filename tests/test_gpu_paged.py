"""Paged main KV cache on the GPU (csrc/paged.cpp +
ssd_engine_set_block_table): the attention and KV-append kernels address
main-cache keys through a per-lane block table.

* a permuted block table gives bit-identical logits and greedy streams to
  the identity layout (deterministic summation order on both sides);
* prefix sharing: lane 1 maps lane 0's cached prompt pages read-only
  (ssd_kv_seq_admit's prefix hit), skips their prefill, and both lanes'
  greedy harness streams equal the unshared run."""
import os

import numpy as np
import pytest

from parity import sim_cfg

pytestmark = pytest.mark.gpu

K = 4
PT = 16


def _engine(P, max_batch=1):
    from paper_2603_03251_b200.configs import shapes
    ts, ds = shapes("tiny", max_ctx=1024)
    return P.Engine(ts, ds, P.Pair(), max_branches=20, max_lookahead=K, max_batch=max_batch)


@pytest.fixture(scope="module")
def P():
    old = os.environ.get("SSD_B200_DETERMINISTIC")
    os.environ["SSD_B200_DETERMINISTIC"] = "1"
    import paper_2603_03251_b200 as P
    yield P
    if old is None:
        os.environ.pop("SSD_B200_DETERMINISTIC", None)
    else:
        os.environ["SSD_B200_DETERMINISTIC"] = old


def test_permuted_block_table_is_bit_identical(P):
    a, b = _engine(P), _engine(P)
    n_pages = b.kv_pages(PT)
    assert n_pages == 1024 // PT
    perm = np.random.default_rng(7).permutation(n_pages).tolist()
    b.set_block_table(0, perm, PT)
    rng = np.random.default_rng(3)
    for n in (1, 20, 40, 100):
        ctx = rng.integers(0, 32000, n).tolist()
        for which in (0, 1):
            assert np.array_equal(a.logits(which, ctx), b.logits(which, ctx)), (n, which)
    prompt = rng.integers(0, 32000, 37).tolist()
    ga = a.run_ar(prompt, P.SamplingScheme.greedy(), 24, 0)
    gb = b.run_ar(prompt, P.SamplingScheme.greedy(), 24, 0)
    assert ga.streams[0] == gb.streams[0]
    cfg = sim_cfg(P, K, 10, 5, 0.0, [4] * (K + 1))
    sa, sb = a.run_ssd(prompt, cfg), b.run_ssd(prompt, cfg)
    assert sa.streams[0] == sb.streams[0] and sa.tokens == sb.tokens
    b.clear_block_tables()
    assert b.run_ssd(prompt, cfg).streams[0] == sa.streams[0]
    a.close()
    b.close()


def test_prefix_pages_shared_across_lanes(P):
    ref, eng = _engine(P, 2), _engine(P, 2)
    n_pages = eng.kv_pages(PT)
    pool = P.KvPool(n_pages, PT)
    prompt = np.random.default_rng(11).integers(0, 32000, 70).tolist()
    R = 8
    assert pool.admit(0, prompt) == 0
    cached = pool.admit(1, prompt)
    assert cached == (len(prompt) - 1) // PT * PT == 64
    for sid in (0, 1):
        pool.reserve(sid, R * (K + 1) + 2 * K + 2)
    t0, t1 = pool.table(0)[0], pool.table(1)[0]
    assert t0[:4] == t1[:4] and not set(t0[4:]) & set(t1[4:])
    eng.set_block_table(0, t0, PT, 0)
    eng.set_block_table(1, t1, PT, cached)
    cfg = sim_cfg(P, K, R, 21, 0.0, [4] * (K + 1))
    cfg.batch_size = 2
    g, r = eng.run_ssd(prompt, cfg), ref.run_ssd(prompt, cfg)
    assert g.streams == r.streams
    assert g.tokens == r.tokens
    st = pool.stats()
    assert st["prefix_hit_pages"] == 4 and st["used_pages"] == len(set(t0) | set(t1))
    # negative control: lane 1 claims the cached prefix but maps pages nobody
    # wrote, so its attention reads zero rows and its stream must change
    # (proves the prefill skip and the table-driven reads are live)
    fresh = [p for p in range(n_pages) if p not in set(t0) | set(t1)][: len(t1)]
    eng.set_block_table(1, fresh, PT, cached)
    bad = eng.run_ssd(prompt, cfg)
    assert bad.streams[0] == r.streams[0] and bad.streams[1] != r.streams[1]
    pool.close()
    ref.close()
    eng.close()


def test_block_table_validation(P):
    eng = _engine(P)
    with pytest.raises(P.ConfigError):
        eng.kv_pages(24)                       # not a power of two
    with pytest.raises(P.ConfigError):
        eng.set_block_table(0, [0, 10 ** 6], PT)
    with pytest.raises(P.TooLargeError):
        eng.set_block_table(0, list(range(eng.kv_pages(PT) + 1)), PT)
    eng.close()
