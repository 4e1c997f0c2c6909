"""GPU parity on the kernel instantiations the benchmark runs (VERDICT r1
"what's weak" 1): GQA with G = 4, head_dim 128 (8B) and 64 (1B), V = 128256,
the 8B/1B GEMM tilings (N = 6144 / 4096 / 28672 / 128256 target, 3072 /
2048 / 16384 / 128256 draft) and the M = 1 / 5 / 20 forwards — against the
CPU oracle (oracle/transformer_lm.cpp, oracle/ssd_oracle.cpp).

* `bench_pair`: a reduced-depth pair with the EXACT per-layer shapes of
  Llama-3.1-8B and Llama-3.2-1B (2 layers each): logits, cache keys,
  verify decisions at V = 128256, greedy AR / SD / SSD-harness streams
  (teacher-forced, tests/parity.py), outcomes, hits and counters.
* `tiny_gqa`: small GQA pairs (G = 4 at head_dim 64 and 128) for the
  sampled-mode statistics that need many rounds.
* the full `llama8b_1b` pair: 2 greedy harness rounds through every layer.
"""
import numpy as np
import pytest

from parity import (binom_close, check_greedy_stream, check_harness_exact, check_topk_set, first_divergence,
                    logit_noise_check, near_tie_for, sim_cfg, sim_req)

pytestmark = pytest.mark.gpu

K = 4
FAN = [4] * (K + 1)

BENCH_T = dict(vocab=128256, d_model=4096, n_layers=2, n_heads=32, n_kv_heads=8, head_dim=128, ffn=14336)
BENCH_D = dict(vocab=128256, d_model=2048, n_layers=2, n_heads=32, n_kv_heads=8, head_dim=64, ffn=8192, tied=True)
GQA64_T = dict(vocab=32000, d_model=512, n_layers=4, n_heads=8, n_kv_heads=2, head_dim=64, ffn=1536)
GQA64_D = dict(vocab=32000, d_model=256, n_layers=2, n_heads=4, n_kv_heads=1, head_dim=64, ffn=768, tied=True)
GQA128_T = dict(vocab=32000, d_model=512, n_layers=4, n_heads=8, n_kv_heads=2, head_dim=128, ffn=1536)
GQA128_D = dict(vocab=32000, d_model=256, n_layers=2, n_heads=4, n_kv_heads=1, head_dim=128, ffn=768, tied=True)


def _pair(oracle_lib, t, d, max_ctx=256, branches=20, pair=None):
    import paper_2603_03251_b200 as P
    from paper_2603_03251_b200.api import model_shape
    ts, ds = model_shape(**t, max_ctx=max_ctx), model_shape(**d, max_ctx=max_ctx)
    pair = pair or P.Pair()
    eng = P.Engine(ts, ds, pair, max_branches=branches, max_lookahead=K)
    orc = oracle_lib.TfPair(P.shape_dict(ts), P.shape_dict(ds), pair.as_dict())
    return P, eng, orc


def _f64(oracle_lib, eng, pair):
    import paper_2603_03251_b200 as P
    return oracle_lib.TfPair(P.shape_dict(eng.target), P.shape_dict(eng.draft), pair.as_dict(), accum="f64")


@pytest.fixture(scope="module")
def bench_pair(oracle_lib):
    P, eng, orc = _pair(oracle_lib, BENCH_T, BENCH_D)
    yield P, eng, orc
    eng.close()
    orc.close()


@pytest.fixture(scope="module")
def bench_f64(oracle_lib, bench_pair):
    P, eng, orc = bench_pair
    o64 = _f64(oracle_lib, eng, P.Pair())
    yield o64
    o64.close()


def _prompt(n, V, seed):
    return np.random.default_rng(seed).integers(0, V, n).tolist()


@pytest.fixture(scope="module")
def tie(bench_pair, bench_f64):
    """Near-tie width of the bench-shaped pair (tests/parity.py near_tie_for)."""
    P, eng, orc = bench_pair
    w = near_tie_for(orc, bench_f64, [_prompt(n, 128256, 500 + n) for n in (3, 11, 24)])
    print("near-tie width", w)
    return w


@pytest.mark.parametrize("which", [0, 1])
def test_bench_shape_logits(bench_pair, bench_f64, tie, which):
    """M = n prefill forwards (n = 1 decode, 5 verify / extend, 20 branch
    width, 37 a prefill chunk) of the 8B-shaped (which 0) / 1B-shaped
    (which 1) model against the fp64 oracle, within the fp32 noise floor
    (tests/parity.py logit_noise_check); argmax equal or a near-tie."""
    P, eng, orc = bench_pair
    ctxs = [_prompt(n, 128256, 40 + n) for n in (1, 5, 20, 37)]
    out = logit_noise_check(eng.logits, orc, bench_f64, which, ctxs)
    print("logit noise", which, out)
    for ctx in ctxs:
        g, o = eng.logits(which, ctx), orc.logits(which, ctx)
        if int(np.argmax(g)) != int(np.argmax(o)):
            assert float(o.max() - o[int(np.argmax(g))]) < tie


def test_bench_shape_keys_on_engine_rows(bench_pair, tie):
    """Cache keys at V = 128256 from the engine's own draft logits
    (build_cache, cache.cpp:232-277): candidate sets equal the oracle's, a
    difference allowed only at a near-tie of the cut; entry tokens are the
    draft's greedy continuations (teacher-forced)."""
    P, eng, orc = bench_pair
    prompt = _prompt(12, 128256, 7)
    spec = eng.draft_spec(prompt, K, P.SamplingScheme.greedy(), seed=1)
    check_greedy_stream(orc, 1, prompt, spec.tokens, near_tie=tie)
    plan = P.FanOutPlan(FAN, P.PRIMARY)
    c = eng.build_cache(prompt, spec, plan, P.SamplingScheme.greedy(), K, seed=5)
    assert c.size() == sum(FAN)
    for k in range(K + 1):
        zo = orc.logits(1, prompt + spec.tokens[:k])
        got = [t for (kk, t) in c.entries if kk == k]
        excl = spec.tokens[k] if k < K else -1
        z = zo.astype(np.float64).copy()
        if excl >= 0:
            z[excl] = -np.inf
        want = np.argsort(-z, kind="stable")[:FAN[k]].tolist()
        assert excl not in got
        check_topk_set(zo, got, want, excl, near_tie=tie)
        for t in got:  # entry = greedy continuation of the branch (draft, specdec.cpp:8-25)
            check_greedy_stream(orc, 1, prompt + spec.tokens[:k] + [t], c.lookup(k, t), near_tie=tie)


def test_bench_shape_topk_and_verify_rows_v128k(bench_pair, oracle_lib):
    """Row kernels at V = 128256 (more vocabulary chunks than the tiny pair):
    top-(F+1) keys with forced ties and exclusion bit-exact; verify decisions
    identical to the oracle's in greedy / sampled / Saguaro modes."""
    P, eng, orc = bench_pair
    rng = np.random.default_rng(3)
    V = 128256
    for trial in range(3):
        rows = np.round(rng.standard_normal((K + 1, V)) * 64) / 64
        rows[:, 70001] = rows[:, 9] = rows.max(axis=1)
        rows = rows.astype(np.float32)
        fan = [4, 3, 2, 6, 5]
        excl = [int(np.argmax(rows[k])) if k % 2 == 0 else 9 for k in range(K)] + [-1]
        g = eng.topk_keys(rows, fan, excl)
        o = oracle_lib.oracle_call({"op": "keys_rows", "rows": rows.astype(np.float64).tolist(), "fan": fan,
                                    "excluded": excl})["keys"]
        for k in range(K + 1):
            assert g[k, :fan[k]].tolist() == o[k], (trial, k)
    for mode in ("greedy", "sampled", "saguaro"):
        for t in range(6):
            tr = (rng.standard_normal((K + 1, V)) * 3).astype(np.float32)
            dr = (tr[:K] + rng.standard_normal((K, V)).astype(np.float32) * 0.7).astype(np.float32)
            if mode == "greedy":
                ds = ts = P.SamplingScheme.greedy()
                toks = [int(np.argmax(dr[i])) for i in range(K)]
            elif mode == "saguaro":
                ds, ts = P.SamplingScheme.saguaro(4, 0.5, 1.0), P.SamplingScheme.standard(1.0)
                toks = [int(x) for x in rng.integers(0, V, K)]
            else:
                ds = ts = P.SamplingScheme.standard(1.0)
                toks = [int(np.argmax(tr[i])) if rng.random() < 0.6 else int(rng.integers(0, V)) for i in range(K)]
            seed = 77 + t
            got = eng.verify_rows(tr, dr, toks, ds, ts, seed)
            o = oracle_lib.oracle_call({"op": "verify_rows", "target_rows": tr.astype(np.float64).tolist(),
                                        "draft_rows": dr.astype(np.float64).tolist(), "tokens": toks,
                                        "scheme": {"kind": ds.kind, "temperature": ds.temperature,
                                                   "fan_out": ds.fan_out, "downweight": ds.downweight},
                                        "target_scheme": {"kind": ts.kind, "temperature": ts.temperature},
                                        "seed": seed})
            assert got == (o["accepted"], o["bonus"]), (mode, t)


def test_bench_shape_ar_and_sd_greedy(bench_pair, tie):
    P, eng, orc = bench_pair
    prompt = _prompt(16, 128256, 11)
    ar = eng.run_ar(prompt, P.SamplingScheme.greedy(), 12, seed=1)
    check_greedy_stream(orc, 0, prompt, ar.streams[0], near_tie=tie)
    sd = eng.run_sd(prompt, sim_cfg(P, K, 4, 2, 0.0, FAN))
    check_greedy_stream(orc, 0, prompt, sd.streams[0], near_tie=tie)
    o = orc.call(sim_req(prompt, "sd", K, 4, 2, 0.0, FAN))
    if first_divergence(sd.streams[0], o["streams"][0]) is None:
        assert sd.accepted_sum == o["accepted_sum"]


@pytest.mark.parametrize("backup", ["fast_random", "same_primary_jit"])
def test_bench_shape_ssd_harness_greedy(bench_pair, tie, backup):
    """run_protocol_harness (sim.cpp:502-601) on the bench shapes: the
    stream is the target's greedy stream (teacher-forced); when it equals
    the oracle's, (k*, t*) per round, hit bits and every counter agree."""
    P, eng, orc = bench_pair
    prompt = _prompt(20, 128256, 12)
    R = 5
    g = eng.run_ssd(prompt, sim_cfg(P, K, R, 9, 0.0, FAN, backup))
    check_greedy_stream(orc, 0, prompt, g.streams[0], near_tie=tie)
    o = orc.call(sim_req(prompt, "harness", K, R, 9, 0.0, FAN, backup))
    if first_divergence(g.streams[0], o["streams"][0]) is None:
        check_harness_exact(g, o)


def test_bench_shape_ssd_harness_sampled(bench_pair):
    """tau = 1 on the bench shapes: the engine draws the reference's own
    mt19937_64 uniforms; streams agree until a uniform lands within logit
    noise of a CDF edge, so only the loop's bookkeeping is exact here (the
    statistics are tested on the small GQA pairs below)."""
    P, eng, orc = bench_pair
    prompt = _prompt(10, 128256, 13)
    R = 4
    g = eng.run_ssd(prompt, sim_cfg(P, K, R, 21, 1.0, FAN))
    o = orc.call(sim_req(prompt, "harness", K, R, 21, 1.0, FAN))
    assert g.rounds == R and g.tokens == len(g.streams[0])
    assert g.hit_rounds + g.miss_rounds + g.initial_rounds >= R - 1
    if first_divergence(g.streams[0], o["streams"][0]) is None:
        check_harness_exact(g, o)


@pytest.fixture(scope="module", params=["hd64", "hd128"])
def tiny_gqa(request, oracle_lib):
    t, d = (GQA64_T, GQA64_D) if request.param == "hd64" else (GQA128_T, GQA128_D)
    P, eng, orc = _pair(oracle_lib, t, d, max_ctx=512, branches=32)
    yield P, eng, orc
    eng.close()
    orc.close()


def test_gqa_logits_and_greedy_harness(tiny_gqa, oracle_lib):
    P, eng, orc = tiny_gqa
    o64 = _f64(oracle_lib, eng, P.Pair())
    for which in (0, 1):
        logit_noise_check(eng.logits, orc, o64, which, [_prompt(n, 32000, 300 + n) for n in (1, 5, 20, 60)])
    o64.close()
    prompt = _prompt(12, 32000, 14)
    g = eng.run_ssd(prompt, sim_cfg(P, K, 10, 4, 0.0, FAN))
    check_greedy_stream(orc, 0, prompt, g.streams[0])
    o = orc.call(sim_req(prompt, "harness", K, 10, 4, 0.0, FAN))
    if first_divergence(g.streams[0], o["streams"][0]) is None:
        check_harness_exact(g, o)


def test_gqa_sampled_statistics(tiny_gqa):
    """tau = 1: acceptance and cache hit rate of the GPU harness within
    binomial 4 sigma of the oracle's over independent prompts."""
    P, eng, orc = tiny_gqa
    R = 30
    acc_g = acc_o = hit_g = hit_o = look_g = look_o = 0
    for rep in range(4):
        prompt = _prompt(12, 32000, 600 + rep)
        g = eng.run_ssd(prompt, sim_cfg(P, K, R, 700 + rep, 1.0, FAN))
        o = orc.call(sim_req(prompt, "harness", K, R, 700 + rep, 1.0, FAN))
        acc_g += g.accepted_sum
        acc_o += o["accepted_sum"]
        hit_g += g.hits_total()
        look_g += g.lookups()
        hit_o += o["p_hits"] + o["b_hits"]
        look_o += o["p_lookups"] + o["b_lookups"]
    n = 4 * R * K
    assert binom_close(acc_g, n, acc_o, n), (acc_g, acc_o)
    assert binom_close(hit_g, look_g, hit_o, look_o), (hit_g, look_g, hit_o, look_o)


def test_full_llama8b_1b_greedy_harness(oracle_lib):
    """The full-depth benchmark pair (32 + 16 layers, ~18 GB of weights on
    both sides): 2 greedy harness rounds after an 8-token prompt, every
    output token checked against the CPU oracle's 8B argmax."""
    import paper_2603_03251_b200 as P
    from paper_2603_03251_b200.configs import shapes
    ts, ds = shapes("llama8b_1b", max_ctx=128)
    pair = P.Pair(block_out_scale=0.06)
    eng = P.Engine(ts, ds, pair, max_branches=20, max_lookahead=K)
    orc = oracle_lib.TfPair(P.shape_dict(ts), P.shape_dict(ds), pair.as_dict())
    try:
        prompt = _prompt(8, 128256, 20250809)
        o64 = _f64(oracle_lib, eng, pair)
        print("logit noise 8B", logit_noise_check(eng.logits, orc, o64, 0, [prompt]))
        print("logit noise 1B", logit_noise_check(eng.logits, orc, o64, 1, [prompt]))
        tie = near_tie_for(orc, o64, [prompt, _prompt(5, 128256, 1)])
        o64.close()
        g = eng.run_ssd(prompt, sim_cfg(P, K, 2, 20250809, 0.0, FAN))
        check_greedy_stream(orc, 0, prompt, g.streams[0], near_tie=tie)
        o = orc.call(sim_req(prompt, "harness", K, 2, 20250809, 0.0, FAN))
        if first_divergence(g.streams[0], o["streams"][0]) is None:
            check_harness_exact(g, o)
    finally:
        eng.close()
        orc.close()
