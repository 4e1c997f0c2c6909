"""The C++ shim (include/ssdlab_b200.hpp) — the reference-style ssdlab
interface over the C-ABI — compiled with g++ and driven like a reference
caller (tests/cpp/shim_smoke.cpp)."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2603_03251_b200")


@pytest.fixture(scope="module")
def shim_bin(tmp_path_factory):
    if not os.path.exists(os.path.join(LIBDIR, "libssd_b200.so")):
        pytest.fail("libssd_b200.so missing: run __graft_entry__.build()")
    out = str(tmp_path_factory.mktemp("shim") / "shim_smoke")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "shim_smoke.cpp"), "-L", LIBDIR, "-lssd_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", out], check=True)
    return out


def test_shim_compiles_links_and_plans_on_host(shim_bin):
    r = subprocess.run([shim_bin, "--no-gpu"], capture_output=True, text=True, check=True)
    assert json.loads(r.stdout)["uniform"] == [4, 4, 4, 4, 4]


@pytest.mark.gpu
def test_shim_drives_engine_like_reference_caller(shim_bin):
    import paper_2603_03251_b200 as P
    from paper_2603_03251_b200.configs import shapes
    r = subprocess.run([shim_bin], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    got = json.loads(r.stdout)
    assert got["consistent"] and got["lookups"] and got["too_large"] and got["cache_size"] == 20
    # the same run through the Python mirror of the C-ABI
    ts, ds = shapes("tiny", max_ctx=512)
    eng = P.Engine(ts, ds, P.Pair(), max_branches=32, max_lookahead=4)
    prompt = [(i * 7919 + 13) % 32000 for i in range(8)]
    cfg = P.SimConfig(lookahead=4, scheme=P.SamplingScheme.greedy(), target_scheme=P.SamplingScheme.greedy(),
                      primary_plan=P.FanOutPlan([4] * 5, P.PRIMARY), backup_plan=P.FanOutPlan([4] * 5, P.BACKUP),
                      primary_time=0.4, rounds=6, seed=1)
    py = eng.run_ssd(prompt, cfg)
    eng.close()
    assert py.streams[0] == got["tokens"]
    assert abs(py.hit_rate() - got["hit_rate"]) < 1e-9


REF_CASES = os.path.join(ROOT, "tests", "cpp", "ref_cases.cpp")


@pytest.fixture(scope="module")
def ref_cases_bin(tmp_path_factory):
    """The reference's own specdec / cache known-answer cases (test_specdec.cpp
    :43-153, test_cache.cpp:221-302) restated against the shim, compiled
    with a doctest stand-in (tests/cpp/doctest_shim.h)."""
    out = str(tmp_path_factory.mktemp("refcases") / "ref_cases")
    cuda = "/usr/local/cuda"
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    "-I", os.path.join(cuda, "include"), REF_CASES, "-L", LIBDIR, "-lssd_b200",
                    "-L", os.path.join(cuda, "lib64"), "-lcudart", f"-Wl,-rpath,{LIBDIR}",
                    f"-Wl,-rpath,{os.path.join(cuda, 'lib64')}", "-o", out], check=True)
    return out


def test_reference_cases_compile_against_shim(ref_cases_bin):
    assert os.path.exists(ref_cases_bin)


@pytest.mark.gpu
def test_reference_cases_pass_on_gpu(ref_cases_bin):
    r = subprocess.run([ref_cases_bin], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]
    got = json.loads(r.stdout.strip().splitlines()[-1])
    assert got["failed"] == 0 and got["cases"] >= 13, got
