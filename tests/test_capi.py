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
