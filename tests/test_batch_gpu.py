"""Batch > 1: run_protocol_harness with
SimConfig::batch_size > 1 (sim.cpp:502-601) on the GPU, through the C-ABI
(ssd_run_ssd_batch), against the oracle's restatement of the same loop.

Every sequence shares the prompt; sequence j drafts from
Stream(derive_seed(seed, j)) and verifies from
Stream(derive_seed(derive_seed(seed, 0x5EED), j)); the whole batch stalls for
the backup when any sequence misses (the virtual clock). Bars as in
test_gpu_parity.py: greedy streams identical (or diverging only at a
documented near-tie), counters and clock exact when the streams agree,
sampled statistics within 4 sigma.
"""
import numpy as np
import pytest

from test_gpu_parity import _assert_streams_match_or_near_tie, _binom_close, _first_divergence, _prompt

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tiny_batch(oracle_lib):
    import paper_2603_03251_b200 as P
    from paper_2603_03251_b200.configs import shapes
    ts, ds = shapes("tiny", max_ctx=1024)
    pair = P.Pair()
    eng = P.Engine(ts, ds, pair, max_branches=32, max_lookahead=8, max_batch=4)
    orc = oracle_lib.TfPair(P.shape_dict(ts), P.shape_dict(ds), pair.as_dict())
    yield P, eng, orc
    eng.close()
    orc.close()


def _req(prompt, K, rounds, seed, temperature, fan, bfan, backup, batch, backup_time):
    return {"op": "simulate", "mode": "harness", "lookahead": K, "rounds": rounds, "seed": seed, "prompt": prompt,
            "scheme": {"temperature": temperature}, "primary_plan": {"fan": fan}, "backup_plan": {"fan": bfan},
            "timing": {"primary_time": 0.4, "backup_time": backup_time}, "backup": backup, "batch_size": batch}


def _cfg(P, K, rounds, seed, temperature, fan, bfan, backup, batch, backup_time):
    return P.SimConfig(lookahead=K, scheme=P.SamplingScheme.standard(temperature),
                       primary_plan=P.FanOutPlan(list(fan), P.PRIMARY), backup_plan=P.FanOutPlan(list(bfan), P.BACKUP),
                       primary_time=0.4, backup_time=backup_time, backup_kind=backup, rounds=rounds, seed=seed,
                       batch_size=batch)


COUNTERS = (("tokens", "tokens"), ("primary_origin_lookups", "p_lookups"), ("primary_origin_hits", "p_hits"),
            ("backup_origin_lookups", "b_lookups"), ("backup_origin_hits", "b_hits"), ("hit_rounds", "hit_rounds"),
            ("miss_rounds", "miss_rounds"), ("initial_rounds", "initial_rounds"),
            ("hit_round_tokens", "hit_round_tokens"), ("miss_round_tokens", "miss_round_tokens"),
            ("accepted_sum", "accepted_sum"))


@pytest.mark.parametrize("batch,backup,fan,bfan", [
    (3, "fast_random", [4] * 5, [4] * 5),
    (4, "fast_random", [2, 2, 2, 2, 2], [1, 1, 1, 1, 1]),
    (3, "same_primary_jit", [4] * 5, [4] * 5),
    (2, "fast_random", [4, 4, 4, 4, 4], [8, 4, 2, 2, 1]),  # backup-origin rounds use a different key layout
])
def test_batch_harness_greedy_matches_oracle(tiny_batch, batch, backup, fan, bfan):
    P, eng, orc = tiny_batch
    prompt = _prompt(12, seed=8)
    K, R = 4, 10
    g = eng.run_ssd(prompt, _cfg(P, K, R, 41, 0.0, fan, bfan, backup, batch, 0.5))
    o = orc.call(_req(prompt, K, R, 41, 0.0, fan, bfan, backup, batch, 0.5))
    assert g.batch == batch and len(g.streams) == batch == len(o["streams"])
    same = True
    for j in range(batch):
        if _first_divergence(g.streams[j], o["streams"][j]) is not None:
            same = False
            _assert_streams_match_or_near_tie(P, orc, prompt, g.streams[j], o["streams"][j])
    if same:
        assert [tuple(x) for x in g.outcomes.tolist()] == [tuple(x) for x in o["outcomes0"]]
        assert g.hits[:-1].tolist() == o["hits0"]
        for key_g, key_o in COUNTERS:
            assert getattr(g, key_g) == o[key_o], key_g
        assert abs(g.virtual_time - o["vtime"]) < 1e-9
        assert g.rounds == R


def test_batch_lanes_are_independent_sequences(tiny_batch):
    """Greedy with the FastRandom backup: the uniform backup tokens differ per
    sequence (own streams), so sequences diverge after their first miss, and
    lane j equals a batch-1 run whose draft / verifier streams are lane j's."""
    P, eng, orc = tiny_batch
    prompt = _prompt(12, seed=21)
    K, R, fan = 4, 8, [1] * 5  # small fan-out: misses happen
    g = eng.run_ssd(prompt, _cfg(P, K, R, 5, 0.0, fan, fan, "fast_random", 3, 0.0))
    o = orc.call(_req(prompt, K, R, 5, 0.0, fan, fan, "fast_random", 3, 0.0))
    for j in range(3):
        _assert_streams_match_or_near_tie(P, orc, prompt, g.streams[j], o["streams"][j])
    # lane 0 of a batch is the batch-1 sequence (same seeds, same streams)
    g1 = eng.run_ssd(prompt, _cfg(P, K, R, 5, 0.0, fan, fan, "fast_random", 1, 0.0))
    assert g1.streams[0] == g.streams[0]


def test_batch_sampled_statistics_match_oracle(tiny_batch):
    """tau = 1: acceptance and hit rate over a batch of 4 within 4 sigma of
    the oracle's; the whole-batch stall makes the clock at least the batch-1
    bound (every round costs max(1, T_p) or 1 + T_b)."""
    P, eng, orc = tiny_batch
    K, R, fan = 4, 20, [4] * 5
    acc_g = acc_o = hit_g = hit_o = look_g = look_o = 0
    for rep in range(2):
        prompt = _prompt(12, seed=300 + rep)
        g = eng.run_ssd(prompt, _cfg(P, K, R, 700 + rep, 1.0, fan, fan, "fast_random", 4, 0.5))
        o = orc.call(_req(prompt, K, R, 700 + rep, 1.0, fan, fan, "fast_random", 4, 0.5))
        acc_g += g.accepted_sum
        acc_o += o["accepted_sum"]
        hit_g += g.hits_total()
        look_g += g.lookups()
        hit_o += o["p_hits"] + o["b_hits"]
        look_o += o["p_lookups"] + o["b_lookups"]
        assert g.tokens == sum(len(s) for s in g.streams)
        assert g.virtual_time >= 0.4 + R - 1e-9
    n = 2 * R * 4 * K
    assert _binom_close(acc_g, n, acc_o, n), (acc_g, acc_o)
    assert _binom_close(hit_g, look_g, hit_o, look_o), (hit_g, look_g, hit_o, look_o)


def test_batch_capacity_errors(tiny_batch):
    P, eng, orc = tiny_batch
    with pytest.raises(P.TooLargeError):
        eng.run_ssd(_prompt(8), _cfg(P, 4, 4, 1, 0.0, [4] * 5, [4] * 5, "fast_random", 5, 0.0))
    with pytest.raises(P.Error):
        eng.run_ssd(_prompt(8), _cfg(P, 4, 4, 1, 0.0, [4] * 5, [4] * 5, "fast_random", 0, 0.0))


@pytest.fixture(scope="module")
def tiny_batch_det(oracle_lib):
    """The tiny pair on an engine with a fixed summation order
    (SSD_B200_DETERMINISTIC=1 at creation): bit-identical reruns, also of
    sampled configurations (the colocated default sums split GEMM tiles with
    fp32 atomics, whose order varies from run to run, and sampled tiny-pair
    streams flip at near-ties)."""
    import os

    import paper_2603_03251_b200 as P
    from paper_2603_03251_b200.configs import shapes
    ts, ds = shapes("tiny", max_ctx=1024)
    old = os.environ.get("SSD_B200_DETERMINISTIC")
    os.environ["SSD_B200_DETERMINISTIC"] = "1"
    try:
        eng = P.Engine(ts, ds, P.Pair(), max_branches=32, max_lookahead=8, max_batch=4)
    finally:
        if old is None:
            os.environ.pop("SSD_B200_DETERMINISTIC", None)
        else:
            os.environ["SSD_B200_DETERMINISTIC"] = old
    yield P, eng, None
    eng.close()


def test_round_graph_cache_invalidation(tiny_batch_det):
    """run_ssd reuses its captured round graphs while every baked-in parameter
    matches; interleaving configurations (lookahead, plans, batch, scheme,
    rounds) on one engine must give exactly the results of the first run of
    each configuration."""
    P, eng, orc = tiny_batch_det
    prompt = _prompt(12, seed=31)
    a = _cfg(P, 4, 6, 3, 0.0, [4] * 5, [4] * 5, "fast_random", 1, 0.0)
    b = _cfg(P, 3, 9, 3, 0.0, [2, 2, 2, 2], [2, 2, 2, 2], "fast_random", 2, 0.5)
    c = _cfg(P, 4, 6, 3, 1.0, [3] * 5, [3] * 5, "fast_random", 1, 0.0)
    first = {k: eng.run_ssd(prompt, cfg) for k, cfg in (("a", a), ("b", b), ("c", c))}
    for k, cfg in (("c", c), ("a", a), ("b", b), ("a", a)):
        r = eng.run_ssd(prompt, cfg)
        assert r.streams == first[k].streams, k
        assert r.outcomes.tolist() == first[k].outcomes.tolist(), k
        assert abs(r.virtual_time - first[k].virtual_time) < 1e-12, k
