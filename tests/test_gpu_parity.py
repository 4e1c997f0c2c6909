"""GPU parity: the B200 engine (through the C-ABI) against the CPU oracle on
the same synthetic weights, prompts and seeds.

Bars:
  * integer / index work — keys, lookups, RNG, weights — bit-exact;
  * greedy token streams identical to the oracle's; a divergence is only
    accepted at a documented near-tie (oracle top-2 logit gap < 1e-2);
  * logits against the fp64-accumulating oracle within the fp32 oracle's own
    deviation, floored at one bf16 activation-rounding flip
    (parity.logit_noise_check; bf16 weights, fp32 accumulation in both);
  * sampled streams: the engine draws the reference's own mt19937_64 uniforms,
    so streams match unless a uniform lands within fp32 noise of a CDF edge.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NEAR_TIE = 1e-2


@pytest.fixture(scope="module")
def tiny(oracle_lib):
    import paper_2603_03251_b200 as P
    from paper_2603_03251_b200.configs import shapes
    ts, ds = shapes("tiny", max_ctx=1024)
    pair = P.Pair()
    eng = P.Engine(ts, ds, pair, max_branches=32, max_lookahead=8)
    orc = oracle_lib.TfPair(P.shape_dict(ts), P.shape_dict(ds), pair.as_dict())
    yield P, eng, orc
    eng.close()
    orc.close()


def _prompt(n=12, V=32000, seed=3):
    return np.random.default_rng(seed).integers(0, V, n).tolist()


def test_weights_bit_identical(tiny):
    P, eng, orc = tiny
    rng = np.random.default_rng(0)
    for which, shape in ((0, eng.target), (1, eng.draft)):
        d, F, qd = shape.d_model, shape.ffn, shape.n_heads * shape.head_dim
        kvd = shape.n_kv_heads * shape.head_dim
        dims = {0: (qd, d), 1: (kvd, d), 2: (kvd, d), 3: (d, qd), 4: (F, d), 5: (F, d), 6: (d, F)}
        for layer in (0, shape.n_layers - 1):
            for kind, (R, Cc) in dims.items():
                rows = rng.integers(0, R, 64)
                cols = rng.integers(0, Cc, 64)
                g = eng.weight_bits(which, layer, kind, rows, cols)
                o = orc.weight_bits(which, layer, kind, rows.tolist(), cols.tolist())
                assert (g == o).all(), (which, layer, kind)
        for kind in (100, 101):
            rows = rng.integers(0, shape.vocab, 64)
            cols = rng.integers(0, d, 64)
            assert (eng.weight_bits(which, 0, kind, rows, cols) == orc.weight_bits(which, 0, kind, rows.tolist(),
                                                                                   cols.tolist())).all()


def test_mt19937_64_on_device_matches_std():
    import paper_2603_03251_b200 as P  # noqa: F401
    import random
    # std::mt19937_64 reference values: the 10000th output for seed 5489 is
    # 9981545732273789042 (C++ standard [rand.predef]).
    from paper_2603_03251_b200.configs import shapes
    ts, ds = shapes("tiny", max_ctx=256)
    eng = P.Engine(ts, ds, P.Pair(), max_branches=4, max_lookahead=2)
    out = eng.rng_u64(5489, 10000)
    assert out[-1] == 9981545732273789042
    eng.close()
    del random


def test_logits_match_oracle(tiny, oracle_lib):
    """Decode / short prefill logits against the fp64-accumulating oracle,
    within the fp32 oracle's own deviation floored at one activation rounding
    flip (parity.logit_noise_check). A flat 1e-2 against the fp32 oracle is
    not a stable bar even at the tiny shapes: the whole-tile SwiGLU GEMM
    (all of K in one TMEM accumulator) and the stream-K one (partials summed
    in fp32) give target logits 1.7e-2 and 1e-4 from fp64 at n = 1, while the
    fp32 oracle itself is 5.9e-3 away (scripts/diag_tiny_logits.py,
    profiles/r02g_summary.md): one bf16 rounding of an early activation flips.
    A wrong head, mask, RoPE or tile moves logits by O(1)."""
    from parity import logit_noise_check
    P, eng, orc = tiny
    orc64 = oracle_lib.TfPair(P.shape_dict(eng.target), P.shape_dict(eng.draft), P.Pair().as_dict(), accum="f64")
    try:
        for which in (0, 1):
            logit_noise_check(eng.logits, orc, orc64, which, [_prompt(n, seed=n) for n in (1, 7, 40)])
    finally:
        orc64.close()


def test_topk_keys_bit_exact_including_ties(tiny, oracle_lib):
    P, eng, orc = tiny
    rng = np.random.default_rng(1)
    V = eng.vocab
    for trial in range(6):
        K = 4
        rows = rng.standard_normal((K + 1, V)).astype(np.float32)
        # force exact ties, including around the cut
        rows = np.round(rows * (4 if trial % 2 else 1000)) / (4 if trial % 2 else 1000)
        rows[:, 17] = rows[:, 5] = rows.max(axis=1)
        fan = [4, 3, 2, 6, 5]
        excl = [int(np.argmax(rows[k])) if k % 2 == 0 else 5 for k in range(K)] + [-1]
        g = eng.topk_keys(rows, fan, excl)
        o = oracle_lib.oracle_call({"op": "keys_rows", "rows": rows.astype(np.float64).tolist(), "fan": fan,
                                    "excluded": excl})["keys"]
        for k in range(K + 1):
            assert g[k, :fan[k]].tolist() == o[k], (trial, k)


@pytest.mark.parametrize("mode", ["greedy", "sampled", "uniform_backup", "saguaro"])
def test_verify_decision_matches_oracle(tiny, oracle_lib, mode):
    P, eng, orc = tiny
    rng = np.random.default_rng(11)
    V, K = eng.vocab, 4
    same = 0
    trials = 24
    for t in range(trials):
        tr = (rng.standard_normal((K + 1, V)) * 3).astype(np.float32)
        dr = (tr[:K] + rng.standard_normal((K, V)).astype(np.float32) * 0.7).astype(np.float32)
        if mode == "greedy":
            ds = ts = P.SamplingScheme.greedy()
            toks = [int(np.argmax(dr[i])) for i in range(K)]
        elif mode == "saguaro":
            ds = P.SamplingScheme.saguaro(3, 0.5, 1.0)
            ts = P.SamplingScheme.standard(1.0)
            toks = [int(x) for x in rng.integers(0, V, K)]
        else:
            ds = ts = P.SamplingScheme.standard(1.0)
            toks = [int(np.argmax(tr[i])) if rng.random() < 0.6 else int(rng.integers(0, V)) for i in range(K)]
        seed = 1000 + t
        use_rows = mode != "uniform_backup"
        g = eng.verify_rows(tr, dr if use_rows else None, toks, ds, ts, seed)
        req = {"op": "verify_rows", "target_rows": tr.astype(np.float64).tolist(), "tokens": toks,
               "scheme": {"kind": ds.kind, "temperature": ds.temperature, "fan_out": ds.fan_out,
                          "downweight": ds.downweight},
               "target_scheme": {"kind": ts.kind, "temperature": ts.temperature}, "seed": seed}
        if use_rows:
            req["draft_rows"] = dr.astype(np.float64).tolist()
        o = oracle_lib.oracle_call(req)
        same += g == (o["accepted"], o["bonus"])
    assert same == trials


def _first_divergence(a, b):
    for i, (x, y) in enumerate(zip(a, b)):
        if x != y:
            return i
    return None if len(a) == len(b) else min(len(a), len(b))


def _assert_streams_match_or_near_tie(P, orc, prompt, g_stream, o_stream):
    i = _first_divergence(g_stream, o_stream)
    if i is None:
        return
    ctx = list(prompt) + list(o_stream[:i])
    lt = orc.logits(0, ctx)
    top2 = np.sort(lt)[-2:]
    gap = float(top2[1] - top2[0])
    assert gap < NEAR_TIE, f"streams diverge at {i} without a near-tie (gap {gap})"


def test_run_ar_greedy_matches_oracle(tiny):
    P, eng, orc = tiny
    prompt = _prompt(16, seed=5)
    g = eng.run_ar(prompt, P.SamplingScheme.greedy(), 48, seed=9)
    o = orc.call({"op": "simulate", "mode": "ar", "lookahead": 1, "rounds": 48, "seed": 9, "prompt": prompt,
                  "scheme": {"temperature": 0.0}})
    _assert_streams_match_or_near_tie(P, orc, prompt, g.streams[0], o["streams"][0])


CDF_TOL = 5e-3  # CDF shift allowed by the |logit| < 1e-2 noise


def test_run_ar_sampled_matches_oracle(tiny):
    """Same mt19937_64 uniforms on both sides: the streams agree until a
    uniform lands where logit noise can move the inverse-CDF boundary; such a
    divergence must sit within CDF_TOL of the oracle's CDF."""
    P, eng, orc = tiny
    prompt = _prompt(16, seed=6)
    g = eng.run_ar(prompt, P.SamplingScheme.standard(1.0), 32, seed=10)
    o = orc.call({"op": "simulate", "mode": "ar", "lookahead": 1, "rounds": 32, "seed": 10, "prompt": prompt,
                  "scheme": {"temperature": 1.0}})
    gs, os_ = g.streams[0], o["streams"][0]
    i = _first_divergence(gs, os_)
    if i is None:
        return
    assert i >= 1, "sampled streams diverge at the first token"
    z = orc.logits(0, list(prompt) + list(gs[:i])).astype(np.float64)
    p = np.exp(z - z.max())
    p /= p.sum()
    cdf = np.concatenate([[0.0], np.cumsum(p)])
    a, b = sorted((gs[i], os_[i]))
    assert cdf[b] - cdf[a + 1] < CDF_TOL, (i, gs[i], os_[i], cdf[b] - cdf[a + 1])


def _sim_req(prompt, mode, K, rounds, seed, temperature, fan, backup="fast_random"):
    return {"op": "simulate", "mode": mode, "lookahead": K, "rounds": rounds, "seed": seed, "prompt": prompt,
            "scheme": {"temperature": temperature}, "primary_plan": {"fan": fan}, "backup_plan": {"fan": fan},
            "timing": {"primary_time": 0.4, "backup_time": 0.0}, "backup": backup}


def _cfg(P, K, rounds, seed, temperature, fan, backup="fast_random"):
    return P.SimConfig(lookahead=K, scheme=P.SamplingScheme.standard(temperature),
                       primary_plan=P.FanOutPlan(list(fan), P.PRIMARY), backup_plan=P.FanOutPlan(list(fan), P.BACKUP),
                       primary_time=0.4, backup_time=0.0, backup_kind=backup, rounds=rounds, seed=seed)


@pytest.mark.parametrize("temperature", [0.0, 1.0])
def test_run_sd_matches_oracle(tiny, temperature):
    P, eng, orc = tiny
    prompt = _prompt(12, seed=7)
    K, R = 4, 10
    g = eng.run_sd(prompt, _cfg(P, K, R, 21, temperature, [4] * 5))
    o = orc.call(_sim_req(prompt, "sd", K, R, 21, temperature, [4] * 5))
    if temperature == 0.0:
        _assert_streams_match_or_near_tie(P, orc, prompt, g.streams[0], o["streams"][0])
    else:
        # same uniforms, but logit noise can move a sampling boundary at any
        # draw: exactness is asserted at kernel level on identical rows
        # (test_verify_decision_matches_oracle), loop statistics below
        assert len(g.streams[0]) == g.tokens and g.rounds == R
        assert all(0 <= t < eng.vocab for t in g.streams[0])


def _binom_close(k1, n1, k2, n2, z=4.0):
    p = (k1 + k2) / (n1 + n2)
    sd = np.sqrt(max(p * (1 - p), 1e-12) * (1 / n1 + 1 / n2))
    return abs(k1 / n1 - k2 / n2) <= z * sd + 1e-9


@pytest.mark.parametrize("mode", ["sd", "harness"])
def test_sampled_acceptance_and_hit_rate_statistically_match(tiny, mode):
    """tau = 1.0 (BASELINE configs[2] style): the per-position acceptance rate
    and the cache hit rate of the GPU loop match the oracle's within 4 sigma
    (binomial) over independent prompts."""
    P, eng, orc = tiny
    K, R, fan = 4, 40, [4] * 5
    acc_g = acc_o = rounds = 0
    hit_g = hit_o = look_g = look_o = 0
    for rep in range(3):
        prompt = _prompt(12, seed=100 + rep)
        cfg = _cfg(P, K, R, 500 + rep, 1.0, fan)
        req = _sim_req(prompt, mode, K, R, 500 + rep, 1.0, fan)
        g = eng.run_sd(prompt, cfg) if mode == "sd" else eng.run_ssd(prompt, cfg)
        o = orc.call(req)
        acc_g += g.accepted_sum
        acc_o += o["accepted_sum"]
        rounds += R
        if mode == "harness":
            hit_g += g.hits_total()
            look_g += g.lookups()
            hit_o += o["p_hits"] + o["b_hits"]
            look_o += o["p_lookups"] + o["b_lookups"]
    # accepted tokens out of K proposals per round
    assert _binom_close(acc_g, rounds * K, acc_o, rounds * K), (acc_g, acc_o, rounds)
    if mode == "harness":
        assert _binom_close(hit_g, look_g, hit_o, look_o), (hit_g, look_g, hit_o, look_o)


@pytest.mark.parametrize("temperature,backup", [(0.0, "fast_random"), (1.0, "fast_random"), (0.0, "same_primary_jit")])
def test_run_ssd_matches_oracle_harness(tiny, temperature, backup):
    """The Saguaro loop against the restated run_protocol_harness: streams,
    per-round (k, t*) outcomes, hit bits and the RunStats counters."""
    P, eng, orc = tiny
    prompt = _prompt(12, seed=8)
    K, R, fan = 4, 8, [4] * 5
    g = eng.run_ssd(prompt, _cfg(P, K, R, 33, temperature, fan, backup))
    o = orc.call(_sim_req(prompt, "harness", K, R, 33, temperature, fan, backup))
    gs, os_ = g.streams[0], o["streams"][0]
    i = _first_divergence(gs, os_)
    if i is None:
        assert [tuple(x) for x in g.outcomes.tolist()] == [tuple(x) for x in o["outcomes0"]]
        assert g.hits[:-1].tolist() == o["hits0"]
        for key_g, key_o in (("tokens", "tokens"), ("primary_origin_hits", "p_hits"),
                             ("backup_origin_hits", "b_hits"), ("hit_rounds", "hit_rounds"),
                             ("miss_rounds", "miss_rounds"), ("accepted_sum", "accepted_sum")):
            assert getattr(g, key_g) == o[key_o], key_g
        assert abs(g.virtual_time - o["vtime"]) < 1e-9
    elif temperature == 0.0:
        _assert_streams_match_or_near_tie(P, orc, prompt, gs, os_)
    else:  # sampled: statistics checked in test_sampled_acceptance_and_hit_rate...
        assert g.tokens == len(gs) and g.rounds == R


def test_build_cache_keys_and_entries_match_oracle(tiny):
    P, eng, orc = tiny
    prompt = _prompt(10, seed=9)
    K = 3
    spec = eng.draft_spec(prompt, K, P.SamplingScheme.greedy(), seed=1)
    o_spec = orc.call({"op": "draft", "context": prompt, "lookahead": K, "draft_seed": 1,
                       "scheme": {"temperature": 0.0}})
    assert spec.tokens == o_spec["spec"]["tokens"]
    plan = P.FanOutPlan([3, 2, 2, 4], P.PRIMARY)
    c = eng.build_cache(prompt, spec, plan, P.SamplingScheme.greedy(), K, seed=77)
    o = orc.call({"op": "build_cache", "context": prompt, "lookahead": K, "draft_seed": 1,
                  "scheme": {"temperature": 0.0}, "plan": {"fan": [3, 2, 2, 4]}, "seed": 77})
    assert sorted(c.entries) == sorted((e[0], e[1]) for e in o["entries"])
    for k, t, toks in o["entries"]:
        assert c.lookup(k, t) == toks, (k, t)


def test_errors_map_to_reference_classes(tiny):
    P, eng, orc = tiny
    with pytest.raises(P.Error):
        eng.run_ar([1, 2], P.SamplingScheme.standard(-1.0), 4, 0)
    with pytest.raises(P.BudgetTooSmallError):
        P.geometric_fanout(0.8, 1.0, 4, 3)
    with pytest.raises(P.TooLargeError):
        eng.run_ar([1] * 10, P.SamplingScheme.greedy(), 5000, 0)


@pytest.mark.parametrize("M", [2, 5, 20, 33, 100])
def test_tcgen05_forward_widths_match_oracle(tiny, oracle_lib, M):
    """The tcgen05 swap-AB GEMM at every token-operand width the engine uses
    (N = 16 / 32 / 48 / 128 tiles, cluster split-K at 17..32): logits of the
    last position of one M-token prefill forward vs the fp64-accumulating
    oracle, within the fp32 oracle's own deviation (parity.logit_noise_check:
    a wide prefill re-rounds every activation to bf16, so two fp32 summation
    orders legitimately differ by more than 1e-2 on some logits)."""
    from parity import logit_noise_check
    P, eng, orc = tiny
    orc64 = oracle_lib.TfPair(P.shape_dict(eng.target), P.shape_dict(eng.draft), P.Pair().as_dict(), accum="f64")
    try:
        ctxs = [_prompt(M, seed=200 + M + 1000 * i) for i in range(3)]
        for which in (0, 1):
            logit_noise_check(eng.logits, orc, orc64, which, ctxs)
    finally:
        orc64.close()
