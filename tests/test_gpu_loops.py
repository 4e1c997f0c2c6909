"""GPU loop semantics beyond the harness (VERDICT r1 "next" 7-8), through the
C-ABI against the CPU oracle:

* sequential `sim::run_ssd` / `run_ssd_batch` semantics (sim.cpp:123-250):
  one stream per sequence, the cache built after verify on it, the
  previous-round clock — `Engine.run_ssd(..., semantics="sequential")`;
* the harness round transcript (sim.cpp:271-317, 489-500);
* end-to-end losslessness: bigram chi-square of sampled SSD streams against
  the target's own sampled AR streams, with the reference's corrupted
  acceptance (accept_scale = 0.7, specdec.cpp:48) as the negative control
  that must be detected (test_sim.cpp:360-408);
* Saguaro sigma_{F,C} drafting inside run_sd / run_ssd (categorical.cpp:65-92);
* the tau = 1 fan-out sweep F in {1, 2, 4, 8, 16} (BASELINE configs[2]).
"""
import numpy as np
import pytest

from parity import (bigram_counts, check_greedy_stream, chi_square_two_sample, first_divergence, runs_close,
                    sim_cfg, sim_req)

pytestmark = pytest.mark.gpu

K = 4
FAN = [4] * (K + 1)
COUNTERS = (("tokens", "tokens"), ("primary_origin_lookups", "p_lookups"), ("primary_origin_hits", "p_hits"),
            ("backup_origin_lookups", "b_lookups"), ("backup_origin_hits", "b_hits"), ("hit_rounds", "hit_rounds"),
            ("miss_rounds", "miss_rounds"), ("initial_rounds", "initial_rounds"),
            ("hit_round_tokens", "hit_round_tokens"), ("miss_round_tokens", "miss_round_tokens"),
            ("accepted_sum", "accepted_sum"))


@pytest.fixture(scope="module")
def tiny(oracle_lib):
    import paper_2603_03251_b200 as P
    from paper_2603_03251_b200.configs import shapes
    ts, ds = shapes("tiny", max_ctx=1024)
    pair = P.Pair()
    eng = P.Engine(ts, ds, pair, max_branches=80, max_lookahead=K, max_batch=2)
    orc = oracle_lib.TfPair(P.shape_dict(ts), P.shape_dict(ds), pair.as_dict())
    yield P, eng, orc
    eng.close()
    orc.close()


def _prompt(n, V, seed):
    return np.random.default_rng(seed).integers(0, V, n).tolist()


@pytest.mark.parametrize("backup,batch", [("fast_random", 1), ("same_primary_jit", 1), ("fast_random", 2)])
def test_sequential_run_ssd_greedy_matches_oracle(tiny, backup, batch):
    """sim::run_ssd_batch on the GPU: every stream is the target's greedy
    stream (teacher-forced), and when the streams equal the oracle's
    run_ssd_batch, every RunStats counter and the virtual clock agree."""
    P, eng, orc = tiny
    prompt = _prompt(12, 32000, 40)
    R = 10
    cfg = sim_cfg(P, K, R, 17, 0.0, FAN, backup)
    cfg.batch_size = batch
    g = eng.run_ssd(prompt, cfg, semantics="sequential")
    req = sim_req(prompt, "ssd", K, R, 17, 0.0, FAN, backup)
    req["batch_size"] = batch
    o = orc.call(req)
    for j in range(batch):
        check_greedy_stream(orc, 0, prompt, g.streams[j])
    if all(first_divergence(g.streams[j], o["streams"][j]) is None for j in range(batch)):
        for kg, ko in COUNTERS:
            assert getattr(g, kg) == o[ko], kg
        assert abs(g.virtual_time - o["vtime"]) < 1e-9


def test_sequential_and_harness_semantics_differ_only_in_rng_order(tiny):
    """Greedy: both loops emit the target's greedy stream (identical), while
    the FastRandom backups draw from different stream positions."""
    P, eng, orc = tiny
    prompt = _prompt(12, 32000, 41)
    cfg = sim_cfg(P, K, 12, 5, 0.0, [1] * (K + 1))
    a = eng.run_ssd(prompt, cfg, semantics="sequential")
    b = eng.run_ssd(prompt, cfg, semantics="harness")
    n = min(len(a.streams[0]), len(b.streams[0]))
    assert a.streams[0][:n] == b.streams[0][:n]


def test_sequential_sampled_statistics(tiny):
    P, eng, orc = tiny
    R = 30
    acc_g, acc_o, hit_g, hit_o = [], [], [], []
    for rep in range(6):
        prompt = _prompt(12, 32000, 800 + rep)
        g = eng.run_ssd(prompt, sim_cfg(P, K, R, 900 + rep, 1.0, FAN), semantics="sequential")
        o = orc.call(sim_req(prompt, "ssd", K, R, 900 + rep, 1.0, FAN))
        acc_g.append((g.accepted_sum, R * K))
        acc_o.append((o["accepted_sum"], R * K))
        hit_g.append((g.hits_total(), g.lookups()))
        hit_o.append((o["p_hits"] + o["b_hits"], o["p_lookups"] + o["b_lookups"]))
    assert runs_close(acc_g, acc_o), (acc_g, acc_o)
    assert runs_close(hit_g, hit_o), (hit_g, hit_o)


@pytest.mark.parametrize("backup", ["fast_random", "same_primary_jit"])
def test_harness_transcript_matches_oracle(tiny, backup):
    """The JSONL round transcript of the GPU harness (one d2v / v2d message
    pair per round, draft first) equals the oracle's message for message."""
    P, eng, orc = tiny
    prompt = _prompt(10, 32000, 42)
    R = 6
    g = eng.run_ssd(prompt, sim_cfg(P, K, R, 23, 0.0, FAN, backup), transcript=True)
    o = orc.call(sim_req(prompt, "harness", K, R, 23, 0.0, FAN, backup))
    assert len(g.transcript) == 2 * R and [m["dir"] for m in g.transcript] == ["d2v", "v2d"] * R
    if first_divergence(g.streams[0], o["streams"][0]) is not None:
        pytest.skip("greedy streams diverge at a documented near-tie: message contents differ legitimately")
    for mg, mo in zip(g.transcript, o["transcript"]):
        assert mg["round"] == mo["round"] and mg["dir"] == mo["dir"]
        assert abs(mg["vclock"] - mo["vclock"]) < 1e-9
        assert mg["payload_summary"] == mo["payload_summary"], (mg, mo)


MICRO_T = dict(vocab=64, d_model=256, n_layers=2, n_heads=4, n_kv_heads=2, head_dim=64, ffn=512)
MICRO_D = dict(vocab=64, d_model=128, n_layers=1, n_heads=2, n_kv_heads=1, head_dim=64, ffn=256, tied=True)


@pytest.fixture(scope="module")
def micro(oracle_lib):
    import paper_2603_03251_b200 as P
    from paper_2603_03251_b200.api import model_shape
    ts, ds = model_shape(**MICRO_T, max_ctx=1024), model_shape(**MICRO_D, max_ctx=1024)
    eng = P.Engine(ts, ds, P.Pair(), max_branches=20, max_lookahead=K, max_batch=8)
    yield P, eng
    eng.close()


def _bigram_pvalue(P, eng, accept_scale, prompts=20, lanes=8, L=120):
    ssd, ar = [], []
    for i in range(prompts):
        prompt = _prompt(4, 64, 5000 + i)
        cfg = sim_cfg(P, K, 100, 7000 + i, 1.0, FAN, accept_scale=accept_scale)
        cfg.batch_size = lanes
        r = eng.run_ssd(prompt, cfg)
        for s in r.streams:
            assert len(s) >= L, len(s)
            ssd.append(s[:L])
        for j in range(lanes):
            ar.append(eng.run_ar(prompt, P.SamplingScheme.standard(1.0), L, 90000 + 97 * i + j).streams[0])
    return chi_square_two_sample(bigram_counts(ssd, 64), bigram_counts(ar, 64))


def test_ssd_lossless_bigram_chi_square(micro):
    """Sampled SSD (tau = 1, FastRandom backup) emits the target's own
    distribution: 160 SSD streams vs 160 target AR streams from the same
    prompts, bigram chi-square p > 0.001 (test_sim.cpp:360-375)."""
    P, eng = micro
    p, stat, dof = _bigram_pvalue(P, eng, 1.0)
    assert p > 1e-3, (p, stat, dof)


def test_corrupted_acceptance_is_detected(micro):
    """Negative control (test_sim.cpp:394-408): accept_scale = 0.7 breaks
    losslessness and the same chi-square must reject it (p < 0.001).
    Calibrated on the CPU oracle: p ~ 1e-41 at this size."""
    P, eng = micro
    p, stat, dof = _bigram_pvalue(P, eng, 0.7)
    assert p < 1e-3, (p, stat, dof)


@pytest.mark.parametrize("loop", ["sd", "harness"])
def test_saguaro_drafting_statistics(tiny, loop):
    """Draft sampling under sigma_{F,C} (F = 4, C = 0.5, tau = 1) inside the
    loops, target Standard(1): acceptance (and the harness' hit rate) within
    4 standard errors of the oracle's over independent prompts (runs as the
    independent units, parity.runs_close)."""
    P, eng, orc = tiny
    sc = P.SamplingScheme.saguaro(4, 0.5, 1.0)
    scd = {"kind": "saguaro", "temperature": 1.0, "fan_out": 4, "downweight": 0.5}
    R = 30
    acc_g, acc_o, hit_g, hit_o = [], [], [], []
    for rep in range(6):
        prompt = _prompt(12, 32000, 300 + rep)
        cfg = sim_cfg(P, K, R, 400 + rep, 1.0, FAN, scheme=sc)
        req = sim_req(prompt, loop, K, R, 400 + rep, 1.0, FAN, scheme=scd)
        req["target_scheme"] = {"kind": "standard", "temperature": 1.0}
        g = eng.run_sd(prompt, cfg) if loop == "sd" else eng.run_ssd(prompt, cfg)
        o = orc.call(req)
        acc_g.append((g.accepted_sum, R * K))
        acc_o.append((o["accepted_sum"], R * K))
        if loop == "harness":
            hit_g.append((g.hits_total(), g.lookups()))
            hit_o.append((o["p_hits"] + o["b_hits"], o["p_lookups"] + o["b_lookups"]))
    assert runs_close(acc_g, acc_o), (acc_g, acc_o)
    if loop == "harness":
        assert runs_close(hit_g, hit_o), (hit_g, hit_o)


@pytest.mark.parametrize("F", [1, 2, 4, 8, 16])
def test_fanout_sweep_tau1_statistics(tiny, F):
    """BASELINE configs[2] fan-out sweep at tau = 1 (rejection-sampling
    verification): cache hit rate and acceptance of the GPU harness within
    4 standard errors of the oracle's at every F (B = 5 F branches, up to
    M = 80), runs as the independent units (parity.runs_close). Sampled
    streams themselves diverge within a few rounds: at near-uniform tiny-pair
    laws the CDF steps (~3e-5) are below the fp32 logit noise, so the shared
    uniforms pick different tokens (scripts/diag_fanout.py: every entry's
    draft rows match the oracle to 0.03 at F = 4..16)."""
    P, eng, orc = tiny
    fan = [F] * (K + 1)
    R = 24
    acc_g, acc_o, hit_g, hit_o = [], [], [], []
    for rep in range(8):
        prompt = _prompt(12, 32000, 1200 + 10 * F + rep)
        g = eng.run_ssd(prompt, sim_cfg(P, K, R, 1300 + rep, 1.0, fan))
        o = orc.call(sim_req(prompt, "harness", K, R, 1300 + rep, 1.0, fan))
        acc_g.append((g.accepted_sum, R * K))
        acc_o.append((o["accepted_sum"], R * K))
        hit_g.append((g.hits_total(), g.lookups()))
        hit_o.append((o["p_hits"] + o["b_hits"], o["p_lookups"] + o["b_lookups"]))
    assert runs_close(acc_g, acc_o), (F, acc_g, acc_o)
    assert runs_close(hit_g, hit_o), (F, hit_g, hit_o)
