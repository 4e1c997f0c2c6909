"""The C-ABI library loads without a GPU, exports every symbol declared in
include/*.h, and its host-only entry points (fan-out plans, cache.cpp:13-169)
agree with the reference's golden answers bit-for-bit."""
import glob
import json
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        for m in re.finditer(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s+(ssd_[a-z_0-9]+)\s*\(", text, re.M):
            syms.add(m.group(1))
    return syms


@pytest.fixture(scope="module")
def lib():
    from paper_2603_03251_b200 import _build, _native
    _build.build()
    return _native.load()


def test_library_exports_every_declared_symbol(lib):
    from paper_2603_03251_b200 import _native
    syms = declared_symbols()
    assert len(syms) >= 15
    nm = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in nm.splitlines() if line.strip()}
    missing = syms - exported
    assert not missing, missing
    assert set(_native.SIGNATURES) == syms  # the Python binding covers the whole ABI


def test_abi_version(lib):
    assert lib.ssd_abi_version() == 1


def test_library_is_sm100a_only(lib):
    from paper_2603_03251_b200 import _native
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if ".cubin" in line)


def _golden():
    with open(os.path.join(ROOT, "tests", "golden", "ref_golden.json")) as f:
        return [c for c in json.load(f) if c["req"]["op"] == "fanout"]


@pytest.mark.parametrize("case", _golden(), ids=lambda c: c["name"])
def test_native_fanout_plans_match_reference(lib, case):
    import paper_2603_03251_b200 as P
    req, ref = case["req"], case["out"]
    K = req["lookahead"]
    if "error" in ref:
        with pytest.raises(P.BudgetTooSmallError if ref["code"] == 5 else P.Error):
            if "uniform" in req:
                P.uniform_fanout(K, req["uniform"])
            else:
                P.geometric_fanout(*req["geometric"][:2], K, req["geometric"][2])
        return
    if "uniform" in req:
        plan = P.uniform_fanout(K, req["uniform"])
    else:
        a, r, b = req["geometric"]
        plan = P.geometric_fanout(a, r, K, b)
    assert plan.fan_out == ref["fan"]


def test_conditional_hit_rate_endpoints(lib):
    import paper_2603_03251_b200 as P
    # cache.cpp:150-169: a = 0 -> only position 0 counts; huge fan-out -> ~1
    assert P.conditional_hit_rate(P.FanOutPlan([2, 1, 1]), 0.0, 1.0) == pytest.approx(0.5)
    assert P.conditional_hit_rate(P.FanOutPlan([10 ** 6] * 4), 0.7, 1.0) == pytest.approx(1.0, abs=1e-5)


def test_engine_fails_loudly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2603_03251_b200 as P
    from paper_2603_03251_b200.configs import shapes
    ts, ds = shapes("tiny", max_ctx=128)
    with pytest.raises(P.CudaError):
        P.Engine(ts, ds, P.Pair())


def _perf_cases():
    with open(os.path.join(ROOT, "tests", "golden", "ref_golden.json")) as f:
        return [c for c in json.load(f) if c["req"]["op"] == "perf"]


@pytest.mark.parametrize("case", _perf_cases(), ids=lambda c: c["name"])
def test_perf_model_matches_reference_golden(lib, case):
    """ssd_speedup_batch / ssd_critical_batch (the batch-size crossover that
    drives the Saguaro fallback policy) against the compiled reference's
    perf.cpp:19-73 on the same inputs."""
    import paper_2603_03251_b200 as P
    r, out = case["req"], case["out"]
    args = (r["hit_rate"], r["hit_tokens"], r["miss_tokens"], r["primary_time"])
    if "error" in out:
        if out["code"] == 9:  # NoCrossoverError from critical_batch
            with pytest.raises(P.NoCrossoverError):
                P.critical_batch(*args)
        else:
            with pytest.raises(P.Error):
                P.speedup_batch(*args, r.get("backup_time", 0.0), r.get("batch", 1))
        return
    if "batch" in r:
        assert P.speedup_batch(*args, r.get("backup_time", 0.0), r["batch"]) == pytest.approx(out["speedup_batch"],
                                                                                             rel=1e-14)
    # batch 1 is speedup_ssd (perf.cpp:19-27)
    assert P.speedup_batch(*args, r.get("backup_time", 0.0), 1) == pytest.approx(out["speedup_ssd"], rel=1e-14)
    if r.get("critical"):
        if "critical_batch" in out:
            assert P.critical_batch(*args) == pytest.approx(out["critical_batch"], rel=1e-14)
        else:
            with pytest.raises(P.NoCrossoverError):
                P.critical_batch(*args)


def test_saguaro_fallback_policy(lib):
    """JIT backup below b*, FastRandom at or above it; without a crossover the
    strategy with the larger batch speedup."""
    import paper_2603_03251_b200 as P
    p, eh, em, tp = 0.8, 3.0, 1.0, 0.4
    b = P.critical_batch(p, eh, em, tp)
    assert 2.0 < b < 3.0
    assert P.saguaro_backup(1, p, eh, em, tp) == P.SAME_PRIMARY_JIT
    assert P.saguaro_backup(2, p, eh, em, tp) == P.SAME_PRIMARY_JIT
    assert P.saguaro_backup(3, p, eh, em, tp) == P.FAST_RANDOM
    assert P.saguaro_backup(8, p, eh, em, tp) == P.FAST_RANDOM
    assert P.saguaro_backup(4, 0.5, 1.0, 3.0, 0.5) in (P.SAME_PRIMARY_JIT, P.FAST_RANDOM)


def _fit_cases():
    with open(os.path.join(ROOT, "tests", "golden", "ref_golden.json")) as f:
        return [c for c in json.load(f) if c["req"]["op"] == "fit_powerlaw"]


@pytest.mark.parametrize("case", _fit_cases(), ids=lambda c: c["name"])
def test_fit_powerlaw_matches_reference_golden(lib, case):
    """ssd_fit_powerlaw against the compiled reference's hitmodel.cpp:65-106."""
    import paper_2603_03251_b200 as P
    out = case["out"]
    if "error" in out:
        with pytest.raises(P.InsufficientDataError if out["code"] == 7 else P.Error):
            P.fit_powerlaw(case["req"]["samples"])
        return
    r, la, r2 = P.fit_powerlaw(case["req"]["samples"])
    assert r == pytest.approx(out["exponent"], rel=1e-13, abs=1e-15)
    assert la == pytest.approx(out["log_amplitude"], rel=1e-13, abs=1e-15)
    assert r2 == pytest.approx(out["r_squared"], rel=1e-13, abs=1e-15)


def test_host_stream_is_std_mt19937_64():
    """ssd_rng_stream (the C form of rng::Stream, rng.hpp:29-48) is host
    code: std::mt19937_64's 10000th output for the default seed is
    9981545732273789042 ([rand.predef]); next_uniform takes the top 53 bits
    (rng.hpp:39-41); derive_seed is rng.hpp:24-26."""
    import paper_2603_03251_b200 as P
    s = P.Stream(5489)
    c = s.copy()
    for _ in range(9999):
        s.next_u64()
    assert s.next_u64() == 9981545732273789042
    x = c.copy().next_u64()
    assert c.next_uniform() == (x >> 11) * 2.0 ** -53
    m = 0xFFFFFFFFFFFFFFFF
    z = (7 + (3 + 1) * 0x9E3779B97F4A7C15) & m
    z = (z + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    assert P.derive_seed(7, 3) == z ^ (z >> 31)
