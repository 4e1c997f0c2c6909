"""Paged KV block manager (csrc/paged.cpp)
through the C-ABI on the CPU: lookahead reservation, reconciliation after
verification (finalize + prefix hash, rollback beyond the accepted suffix),
prefix sharing, LRU eviction, and a randomized differential test against
an independent Python model (tests/kv_model.py)."""
import numpy as np
import pytest

from kv_model import KvModel, OutOfPages


@pytest.fixture
def P():
    from paper_2603_03251_b200 import _build
    _build.build()
    import paper_2603_03251_b200 as P
    return P


def test_admit_reserve_commit_rollback(P):
    pool = P.KvPool(16, 4)
    assert pool.admit(1, list(range(10))) == 0          # 10 tokens: 3 pages
    assert pool.table(1) == ([0, 1, 2], 10)
    pool.reserve(1, 5)                                   # K + 1 = 5 lookahead: 15 tokens -> 4 pages
    assert len(pool.table(1)[0]) == 4
    assert pool.commit(1, [7, 8]) == 1                   # 12 tokens fit 3 pages: one page rolled back
    assert pool.table(1) == ([0, 1, 2], 12)
    st = pool.stats()
    assert (st["used_pages"], st["free_pages"], st["rolled_back_pages"]) == (3, 13, 1)
    assert st["cached_pages"] == 3                        # 3 full pages finalized under their prefix hash
    pool.close()


def test_prefix_pages_are_shared_and_the_last_token_page_stays_private(P):
    pool = P.KvPool(32, 4)
    prompt = list(range(100, 113))                       # 13 tokens: 3 full pages + 1
    assert pool.admit(1, prompt) == 0
    assert pool.admit(2, prompt) == 12                   # 3 cached pages map read-only
    t1, t2 = pool.table(1)[0], pool.table(2)[0]
    assert t1[:3] == t2[:3] and t1[3] != t2[3]
    refs = pool.refs()
    assert [refs[p] for p in t1[:3]] == [2, 2, 2] and refs[t1[3]] == refs[t2[3]] == 1
    # a prompt of exactly 3 full pages: the page of its last token is never a hit
    assert pool.admit(3, prompt[:12]) == 8
    # divergence inside a page: only the pages before it are shared
    other = prompt[:6] + [999] + prompt[7:]
    assert pool.admit(4, other) == 4
    assert pool.stats()["prefix_hit_pages"] == 3 + 2 + 1
    pool.close()


def test_released_pages_stay_cached_until_evicted_lru(P):
    pool = P.KvPool(6, 2)
    a, b = [1, 2, 3, 4, 5], [9, 8, 7, 6, 5]
    pool.admit(1, a)                                     # 3 pages, 2 full (cached)
    pool.release(1)
    st = pool.stats()
    assert st["cached_evictable"] == 2 and st["free_pages"] == 4
    assert pool.admit(2, a) == 4                         # hits while still cached
    pool.release(2)
    pool.admit(3, b)                                     # 3 pages from the free list (1 left)
    pool.reserve(3, 5)                                   # 10 tokens need 5 pages: the free one + one eviction
    st = pool.stats()
    assert st["evictions"] == 1
    # a sequence releases its pages tail first, so the LRU victim is the end
    # of a's chain: its first page is still a prefix hit
    pool.release(3)
    assert pool.admit(4, a) == 2
    pool.close()


def test_out_of_pages_leaves_state_unchanged(P):
    pool = P.KvPool(4, 4)
    pool.admit(1, list(range(12)))
    before = (pool.table(1), pool.stats()["free_pages"])
    with pytest.raises(P.TooLargeError):
        pool.reserve(1, 9)                               # 21 tokens need 6 pages
    with pytest.raises(P.TooLargeError):
        pool.admit(2, list(range(50, 70)))
    assert (pool.table(1), pool.stats()["free_pages"]) == before
    with pytest.raises(P.ProtocolViolationError):
        pool.commit(1, list(range(5)))                   # accepted beyond the reserved pages
    with pytest.raises(P.ConfigError):
        pool.release(7)
    pool.close()


@pytest.mark.parametrize("seed", range(6))
def test_randomized_against_model(P, seed):
    rng = np.random.default_rng(seed)
    n_pages, ps = int(rng.integers(8, 40)), int(rng.integers(1, 6))
    pool, model = P.KvPool(n_pages, ps), KvModel(n_pages, ps)
    prompts = [rng.integers(0, 6, int(rng.integers(1, 20))).tolist() for _ in range(5)]
    live, next_id = [], 0
    for _ in range(300):
        op = rng.integers(0, 4)
        if op == 0 or not live:
            toks = list(prompts[int(rng.integers(0, len(prompts)))])
            toks = toks[: int(rng.integers(1, len(toks) + 1))]
            try:
                want = model.admit(next_id, toks)
            except OutOfPages:
                with pytest.raises(P.TooLargeError):
                    pool.admit(next_id, toks)
                continue
            assert pool.admit(next_id, toks) == want
            live.append(next_id)
            next_id += 1
        elif op == 1:
            sid = live[int(rng.integers(0, len(live)))]
            k = int(rng.integers(1, 6))
            try:
                model.reserve(sid, k)
            except OutOfPages:
                with pytest.raises(P.TooLargeError):
                    pool.reserve(sid, k)
                continue
            pool.reserve(sid, k)
            acc = rng.integers(0, 6, int(rng.integers(0, k + 1))).tolist()
            assert pool.commit(sid, acc) == model.commit(sid, acc)
        else:
            sid = live.pop(int(rng.integers(0, len(live))))
            pool.release(sid)
            model.release(sid)
        for sid in live:
            assert pool.table(sid) == (model.seqs[sid]["pages"], len(model.seqs[sid]["tokens"]))
        assert pool.refs() == model.ref
        st = pool.stats()
        assert st["free_pages"] == len(model.free) and st["cached_evictable"] == len(model.lru)
        assert st["evictions"] == model.evictions
        assert st["used_pages"] + st["free_pages"] + st["cached_evictable"] == n_pages
    pool.close()
