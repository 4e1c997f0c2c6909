"""The colocated SSD round on disjoint SM sets (ssd_engine_sm_partition, CUDA
green contexts): the partition changes only where the two
streams' kernels run and the GEMM grid sizes, so under every partition the
greedy SSD stream is the target's greedy stream (teacher-forced against the
CPU oracle) and, where the streams agree with the oracle's run, every
RunStats counter and the virtual clock agree too."""
import numpy as np
import pytest

from parity import check_greedy_stream, first_divergence, sim_cfg, sim_req

pytestmark = pytest.mark.gpu

K = 4
FAN = [4] * (K + 1)


@pytest.fixture(scope="module")
def tiny(oracle_lib):
    import paper_2603_03251_b200 as P
    from paper_2603_03251_b200.configs import shapes
    ts, ds = shapes("tiny", max_ctx=1024)
    pair = P.Pair()
    eng = P.Engine(ts, ds, pair, max_branches=20, max_lookahead=K)
    orc = oracle_lib.TfPair(P.shape_dict(ts), P.shape_dict(ds), pair.as_dict())
    yield P, eng, orc
    eng.close()
    orc.close()


def test_default_partition_and_setter(tiny):
    import torch
    P, eng, _ = tiny
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    v, s = eng.sm_partition()
    assert v > 0 and s > 0 and v + s == sms
    assert abs(v - sms * 3 // 8) <= 8, v  # driver granularity
    assert eng.sm_partition(0) == (0, 0)
    v2, s2 = eng.sm_partition(40)
    assert abs(v2 - 40) <= 8 and v2 + s2 == sms
    with pytest.raises(P.ConfigError):
        eng.sm_partition(sms)
    assert eng.sm_partition() == (0, 0)  # a failed set leaves the round shared
    eng.sm_partition(sms * 3 // 8)


@pytest.mark.parametrize("verifier_sms", [0, 24, 56, 96])
@pytest.mark.parametrize("backup", ["fast_random", "same_primary_jit"])
def test_partitioned_round_matches_oracle(tiny, verifier_sms, backup):
    P, eng, orc = tiny
    prompt = np.random.default_rng(60 + verifier_sms).integers(0, 32000, 12).tolist()
    R = 10
    old = eng.sm_partition()
    try:
        eng.sm_partition(verifier_sms)
        g = eng.run_ssd(prompt, sim_cfg(P, K, R, 31, 0.0, FAN, backup))
    finally:
        eng.sm_partition(old[0])
    o = orc.call(sim_req(prompt, "harness", K, R, 31, 0.0, FAN, backup))
    check_greedy_stream(orc, 0, prompt, g.streams[0])
    if first_divergence(g.streams[0], o["streams"][0]) is None:
        assert g.accepted_sum == o["accepted_sum"]
        assert g.hits_total() == o["p_hits"] + o["b_hits"]
        assert abs(g.virtual_time - o["vtime"]) < 1e-9

