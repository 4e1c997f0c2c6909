"""The reference-facing boundary (VERDICT r1 "next" 4) on the GPU
against the CPU oracle:

* one caller-owned rng::Stream threaded through specdec::draft ->
  specdec::verify (model-driven: the target's K+1 verify forward + the fused
  decision) -> cache::build_cache, exactly as a reference caller threads its
  Stream& — same tokens, outcome, entries and the same stream position after;
* build_cache with next_lookahead != K, and the entries' draft rows, so a
  cached speculation can be verified in sampled mode;
* the asynchronous device-buffer pre-speculation (ssd_prespec_begin /
  ssd_cache_lookup / _keys / _entry) against the synchronous call.
"""
import numpy as np
import pytest

from parity import check_greedy_stream

pytestmark = pytest.mark.gpu

K = 4


@pytest.fixture(scope="module")
def tiny(oracle_lib):
    import paper_2603_03251_b200 as P
    from paper_2603_03251_b200.configs import shapes
    ts, ds = shapes("tiny", max_ctx=512)
    pair = P.Pair()
    eng = P.Engine(ts, ds, pair, max_branches=40, max_lookahead=8)
    orc = oracle_lib.TfPair(P.shape_dict(ts), P.shape_dict(ds), pair.as_dict())
    yield P, eng, orc
    eng.close()
    orc.close()


def _prompt(n, seed):
    return np.random.default_rng(seed).integers(0, 32000, n).tolist()


@pytest.mark.parametrize("next_k", [K, 2, 6])
def test_one_stream_through_draft_verify_build_cache(tiny, next_k):
    P, eng, orc = tiny
    prompt = _prompt(11, 60 + next_k)
    fan = [3, 2, 2, 1, 4]
    seed = 1234 + next_k
    rng = P.Stream(seed)
    spec = eng.draft_tokens(prompt, K, P.SamplingScheme.greedy(), rng)
    res = eng.verify(prompt, spec, rng, P.SamplingScheme.greedy(), P.SamplingScheme.greedy())
    cache = eng.build_cache_stream(prompt, spec, P.FanOutPlan(fan, P.PRIMARY), P.SamplingScheme.greedy(), next_k, rng)
    o = orc.call({"op": "chain", "context": prompt, "lookahead": K, "scheme": {"temperature": 0.0},
                  "plan": {"fan": fan}, "next_lookahead": next_k, "seed": seed})
    check_greedy_stream(orc, 1, prompt, spec.tokens)
    if spec.tokens != o["spec"]["tokens"]:
        pytest.skip("draft flipped at a documented near-tie; the rest of the chain differs legitimately")
    assert (res.accepted, res.bonus) == (o["accepted"], o["bonus"])
    assert res.emitted == o["emitted"]
    assert len(res.emitted) == res.accepted + 1  # test_specdec.cpp "emitted length is accepted plus one"
    assert sorted(cache.entries) == sorted((e[0], e[1]) for e in o["entries"])
    for k, t, toks in o["entries"]:
        assert len(cache.lookup(k, t)) == next_k
        check_greedy_stream(orc, 1, prompt + spec.tokens[:k] + [t], cache.lookup(k, t))
    # the stream advanced exactly as the reference's did (draft K + verify + one base draw)
    assert rng.next_u64() == o["next_u64"]


def test_cached_speculation_verifies_with_its_rows(tiny):
    """Sampled mode (tau = 1): an entry taken from build_cache carries the
    draft rows it was drawn from (cache.hpp:149-154), so verify applies the
    residual rule to the right laws; decisions match the oracle given the
    same laws and stream (a uniform landing within logit noise of a CDF edge
    may flip one of them)."""
    P, eng, orc = tiny
    same = 0
    trials = 8
    for trial in range(trials):
        prompt = _prompt(9, 700 + trial)
        rng = P.Stream(900 + trial)
        spec = eng.draft_tokens(prompt, K, P.SamplingScheme.standard(1.0), rng)
        cache = eng.build_cache_stream(prompt, spec, P.FanOutPlan([2] * (K + 1), P.PRIMARY),
                                       P.SamplingScheme.standard(1.0), K, rng)
        (k, t), toks = next(iter(cache.entries.items()))
        ent = cache.speculation(k, t)
        assert ent.rows is not None and ent.rows.shape == (K, eng.vocab)
        ctx = prompt + spec.tokens[:k] + [t]
        # the recorded rows are the draft's logits along the entry's own prefix
        for j in range(K):
            z = orc.logits(1, ctx + ent.tokens[:j])
            assert float(np.max(np.abs(z - ent.rows[j]))) < 5e-2
        vs = 4242 + trial
        r = eng.verify(ctx, ent, P.Stream(vs), P.SamplingScheme.standard(1.0), P.SamplingScheme.standard(1.0))
        z = ent.rows.astype(np.float64)
        dists = np.exp(z - z.max(axis=1, keepdims=True))
        dists /= dists.sum(axis=1, keepdims=True)
        o = orc.call({"op": "verify", "context": ctx, "lookahead": K,
                      "scheme": {"temperature": 1.0},
                      "spec": {"tokens": ent.tokens, "dists": dists.tolist()}, "seed": vs})
        same += (r.accepted, r.bonus) == (o["accepted"], o["bonus"])
    assert same >= trials - 1, (same, trials)


def test_async_prespeculation_matches_synchronous(tiny):
    """ssd_prespec_begin on device buffers (ordered after the caller's CUDA
    stream) gives the same keys and entries as the synchronous build_cache
    with the same stream, takes exactly one next_u64 from it, and lookups
    hit every key and miss the excluded drafted token."""
    torch = pytest.importorskip("torch")
    P, eng, orc = tiny
    prompt = _prompt(14, 81)
    fan = [4] * (K + 1)
    spec = eng.draft_tokens(prompt, K, P.SamplingScheme.greedy(), P.Stream(5))
    ref_rng = P.Stream(77)
    sync = eng.build_cache_stream(prompt, spec, P.FanOutPlan(fan, P.PRIMARY), P.SamplingScheme.greedy(), K, ref_rng)
    d_ctx = torch.tensor(prompt, dtype=torch.int32, device="cuda")
    d_spec = torch.tensor(spec.tokens, dtype=torch.int32, device="cuda")
    rng = P.Stream(77)
    stream = torch.cuda.current_stream()
    eng.prespec_begin(d_ctx.data_ptr(), len(prompt), d_spec.data_ptr(), K, P.FanOutPlan(fan, P.PRIMARY),
                      P.SamplingScheme.greedy(), K, rng, stream.cuda_stream)
    assert rng.next_u64() == ref_rng.next_u64()  # one draw, taken at begin
    keys = eng.cache_keys()
    assert sorted(keys) == sorted(sync.entries)
    for slot, (k, t) in enumerate(keys):
        assert eng.cache_lookup(k, t) == slot
        toks, rows = eng.cache_entry(slot, K, with_rows=True)
        assert toks == sync.lookup(k, t)
        assert rows.shape == (K, eng.vocab)
    assert eng.cache_lookup(0, spec.tokens[0]) == -1  # the drafted token is excluded (cache.cpp:249-270)
