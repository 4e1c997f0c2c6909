"""TEST INFRASTRUCTURE ONLY — freeze golden vectors from the UNMODIFIED
reference (oracle/_ref/libssdref.so, compiled from /root/reference/proj/src).

Run in the build container (the reference tree is not on the GPU box):
    python oracle/make_golden.py
Writes tests/golden/ref_golden.json: a list of {"name", "req", "out"} where
`out` is the reference's answer to `req` (request schema: oracle_capi.cpp).
tests/test_oracle_golden.py replays every request through the restated
oracle and requires bit-identical answers.

The cases mirror the reference's own tests (proj/tests/test_*.cpp) and the
shipped configs (proj/configs/*.json); each name cites its source.
"""
from __future__ import annotations

import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import pyoracle as po  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "ref_golden.json")


def log_of(ps):
    return [math.log(max(p, 1e-300)) for p in ps]


def base_config(vocab, order, alpha, K, budget, seed, **kw):
    """test_sim.cpp:30-45 base_config."""
    req = {"op": "simulate",
           "lm": {"vocab": vocab, "order": order, "concentration": 0.5, "seed": seed, "alpha_goal": alpha},
           "lookahead": K,
           "primary_plan": {"geometric": [alpha, 1.0, budget]},
           "backup_plan": {"geometric": [0.3, 1.0, budget]},
           "seed": seed}
    req.update(kw)
    return req


def shift_chain_rows(V):
    """test_sim.cpp:20-28 shift_chain_lm: near-deterministic c -> c+1."""
    rows = []
    for c in range(V):
        p = [1e-12] * V
        p[(c + 1) % V] = 1.0
        rows.append(log_of(p))
    return rows


def cases():
    cs = []
    add = lambda name, req: cs.append({"name": name, "req": req})  # noqa: E731
    # ---- categorical.cpp KATs (test_categorical.cpp)
    add("top_indices ties (test_categorical.cpp:73-77)", {"op": "top_indices", "z": [1, 3, 3, 0.5], "count": 2})
    add("top_indices full", {"op": "top_indices", "z": [0.1, -2, 0.1, 5, 5, 0.1, 3], "count": 7})
    add("saguaro worked example (test_categorical.cpp:79-88)",
        {"op": "apply_scheme", "z": log_of([0.49, 0.49, 0.01, 0.01]),
         "scheme": {"kind": "saguaro", "fan_out": 2, "downweight": 47 / 147, "temperature": 1.0}})
    add("saguaro with temperature", {"op": "apply_scheme", "z": [0.3, -1.2, 2.5, 0.0, 1.1],
                                     "scheme": {"kind": "saguaro", "fan_out": 2, "downweight": 0.4, "temperature": 0.7}})
    add("softmax temperature", {"op": "apply_scheme", "z": [0.3, -1.2, 2.5, 0.0, 1.1],
                                "scheme": {"kind": "standard", "temperature": 1.7}})
    add("residual worked example (test_categorical.cpp:166-182)",
        {"op": "residual", "target": [0.48, 0.48, 0.02, 0.02], "draft": [0.49, 0.49, 0.01, 0.01]})
    add("residual degenerate (test_categorical.cpp:184-187)",
        {"op": "residual", "target": [0.5, 0.5], "draft": [0.5, 0.5]})
    add("sample frequencies (test_categorical.cpp:244-258)", {"op": "sample", "p": [0.25] * 4, "seed": 11, "n": 400})
    add("sample one-hot (test_categorical.cpp:238-242)", {"op": "sample", "p": [0, 0, 1, 0], "seed": 3, "n": 5})
    # ---- fan-out plans (test_cache.cpp:52-185)
    for a, r, K, B in [(0.8, 1.0, 4, 24), (0.3, 1.0, 4, 24), (0.8, 1.0, 3, 12), (0.6, 0.5, 5, 40),
                       (0.9, 2.0, 4, 8), (0.75, 1.0, 4, 20), (0.5, 50.0, 3, 16)]:
        add(f"geometric_fanout a={a} r={r} K={K} B={B}", {"op": "fanout", "lookahead": K, "geometric": [a, r, B]})
    add("geometric budget too small (test_cache.cpp:105-109)", {"op": "fanout", "lookahead": 4, "geometric": [0.8, 1.0, 4]})
    for K, B in [(4, 24), (3, 10), (4, 5)]:
        add(f"uniform_fanout K={K} B={B}", {"op": "fanout", "lookahead": K, "uniform": B})
    # ---- models: make_lm + calibrate_pair (lm.cpp:91-172)
    add("models V=8 m=1 alpha 0.8", {"op": "models", "lm": {"vocab": 8, "order": 1, "concentration": 0.5, "seed": 101, "alpha_goal": 0.8}})
    add("models V=6 m=2 alpha 0.85 (test_sim.cpp order-2)", {"op": "models", "lm": {"vocab": 6, "order": 2, "concentration": 0.6, "seed": 140, "alpha_goal": 0.85}})
    add("models V=12 m=0 eps 0.35 (test_sim.cpp:76-86)", {"op": "models", "lm": {"vocab": 12, "order": 0, "concentration": 0.6, "seed": 104, "epsilon": 0.35}})
    add("models concentration 1", {"op": "models", "lm": {"vocab": 16, "order": 1, "concentration": 1.0, "seed": 5, "epsilon": 0.2}})
    # ---- specdec (test_specdec.cpp)
    chain = {"order": 1, "target_rows": shift_chain_rows(5), "seed": 102}
    add("draft follows the argmax chain (test_specdec.cpp:43-50)",
        {"op": "draft", "lm": chain, "context": [0], "lookahead": 4, "draft_seed": 9})
    add("verify on the chain from ctx {2} (test_specdec.cpp:144-153)",
        {"op": "verify", "lm": chain, "context": [2], "lookahead": 4, "draft_seed": 4, "seed": 5})
    one_row = {"order": 0, "target_rows": [log_of([0.3, 0.7])], "draft_rows": [log_of([0.6, 0.4])], "seed": 1}
    add("verify accept law p_t=0.3 p_d=0.6 (test_specdec.cpp:84-102)",
        {"op": "verify", "lm": one_row, "context": [], "lookahead": 1,
         "spec": {"tokens": [0], "dists": [[0.6, 0.4]]}, "seed": 77})
    lm8 = {"vocab": 8, "order": 1, "concentration": 0.5, "seed": 49, "epsilon": 0.7, "noise_seed": 50}
    for s in range(6):
        add(f"verify make_lm V=8 seed {s}", {"op": "verify", "lm": lm8, "context": [s % 8], "lookahead": 3,
                                             "draft_seed": 1000 + s, "seed": 2000 + s, "with_dists": True})
    add("verify with corrupted acceptance 0.7", {"op": "verify", "lm": lm8, "context": [1], "lookahead": 3,
                                                 "draft_seed": 3, "seed": 4, "accept_scale": 0.7})
    add("verify saguaro draft", {"op": "verify", "lm": lm8, "context": [2], "lookahead": 3, "draft_seed": 5, "seed": 6,
                                 "scheme": {"kind": "saguaro", "fan_out": 2, "downweight": 0.5, "temperature": 1.0}})
    # ---- build_cache (test_cache.cpp:209-302)
    row4 = {"order": 0, "target_rows": [log_of([0.6, 0.25, 0.1, 0.05])], "seed": 43}
    add("build_cache excludes the in-flight token (test_cache.cpp:221-237)",
        {"op": "build_cache", "lm": row4, "context": [], "lookahead": 1,
         "spec": {"tokens": [0], "dists": [[0.6, 0.25, 0.1, 0.05]]}, "plan": {"fan": [2, 0]}, "seed": 44})
    add("build_cache zero plan (test_cache.cpp:209-219)",
        {"op": "build_cache", "lm": {"vocab": 8, "order": 1, "concentration": 0.8, "seed": 41, "epsilon": 0.0},
         "context": [5], "lookahead": 2, "draft_seed": 42, "plan": {"fan": [0, 0, 0]}, "seed": 42})
    add("build_cache lookup entries (test_cache.cpp:263-280)",
        {"op": "build_cache", "lm": {"vocab": 10, "order": 1, "concentration": 0.9, "seed": 47, "epsilon": 0.0},
         "context": [3], "lookahead": 2, "draft_seed": 48, "plan": {"fan": [3, 3, 3]}, "seed": 48})
    for t in range(5):
        add(f"build_cache random plan {t} (test_cache.cpp:239-261)",
            {"op": "build_cache", "lm": {"vocab": 12, "order": 1, "concentration": 0.7, "seed": 46, "epsilon": 0.3},
             "context": [t % 12], "lookahead": 1 + t % 3, "draft_seed": 300 + t,
             "plan": {"fan": [(3 * t + k) % 11 for k in range(2 + t % 3)]}, "seed": 400 + t})
    add("build_cache saguaro scheme",
        {"op": "build_cache", "lm": {"vocab": 16, "order": 1, "concentration": 0.5, "seed": 9, "alpha_goal": 0.7},
         "context": [4], "lookahead": 3, "draft_seed": 1, "plan": {"geometric": [0.7, 1.0, 12]}, "seed": 2,
         "scheme": {"kind": "saguaro", "fan_out": 3, "downweight": 0.3, "temperature": 1.0}})
    # ---- sim loops (test_sim.cpp)
    add("run_ar chain (test_sim.cpp:58-63)",
        {"op": "simulate", "mode": "ar", "lm": chain, "lookahead": 1, "rounds": 10, "seed": 8})
    add("run_ar make_lm (test_sim.cpp:50-56)",
        {"op": "simulate", "mode": "ar", "lm": {"vocab": 8, "order": 1, "concentration": 0.5, "seed": 101, "epsilon": 0.0},
         "lookahead": 1, "rounds": 100, "seed": 7})
    add("run_sd base_config(12,1,0.8,4,10,130)", {**base_config(12, 1, 0.8, 4, 10, 130), "mode": "sd", "rounds": 300})
    add("run_ssd base_config(10,1,0.8,3,12,117) (SURVEY 8c)", {**base_config(10, 1, 0.8, 3, 12, 117), "mode": "ssd", "rounds": 50})
    add("harness base_config(10,1,0.8,3,12,117) (SURVEY 8c)", {**base_config(10, 1, 0.8, 3, 12, 117), "mode": "harness", "rounds": 50})
    add("exhaustive plans never miss (test_sim.cpp:136-155)",
        {**base_config(8, 1, 0.7, 3, 8, 110), "mode": "ssd", "rounds": 200, "timing": {"primary_time": 0.6},
         "primary_plan": {"fan": [7, 7, 7, 8]}, "backup_plan": {"fan": [7, 7, 7, 8]}})
    add("ssd jit backup (test_sim.cpp:173-185)",
        {**base_config(12, 1, 0.8, 3, 16, 200), "mode": "ssd", "rounds": 300, "timing": {"primary_time": 0.3, "backup_time": 0.3},
         "backup": "same_primary_jit"})
    add("ssd batch 2 (test_sim.cpp:219-230)", {**base_config(10, 1, 0.8, 3, 12, 114), "mode": "ssd", "rounds": 200, "batch_size": 2})
    add("ssd synthetic iid batch 3 (test_sim.cpp:261-278)",
        {**base_config(10, 1, 0.8, 2, 9, 116), "mode": "ssd", "rounds": 300, "batch_size": 3, "timing": {"primary_time": 0.5},
         "synthetic_hit_rate": 0.8})
    add("ssd order-2 (test_sim.cpp:280-297)",
        {"op": "simulate", "mode": "ssd", "lm": {"vocab": 6, "order": 2, "concentration": 0.6, "seed": 140, "alpha_goal": 0.85, "noise_seed": 141},
         "lookahead": 3, "primary_plan": {"geometric": [0.85, 1.0, 10]}, "backup_plan": {"geometric": [0.3, 1.0, 10]},
         "seed": 142, "rounds": 300})
    add("ssd corrupted acceptance (test_sim.cpp:393-408)",
        {**base_config(16, 1, 0.75, 4, 20, 122), "mode": "ssd", "rounds": 300, "accept_scale": 0.7})
    add("ssd saguaro scheme t=0.8",
        {**base_config(16, 1, 0.75, 4, 20, 131), "mode": "ssd", "rounds": 300,
         "scheme": {"kind": "saguaro", "fan_out": 3, "downweight": 0.5, "temperature": 0.8}})
    add("harness overlap tp=0.7 (test_sim.cpp:326-336)",
        {**base_config(10, 1, 0.8, 3, 12, 119), "mode": "harness", "rounds": 60, "timing": {"primary_time": 0.7}})
    add("harness slow prespec tp=1.2 (test_sim.cpp:338-351)",
        {**base_config(8, 1, 0.7, 2, 8, 120), "mode": "harness", "rounds": 30, "timing": {"primary_time": 1.2},
         "primary_plan": {"fan": [7, 7, 8]}, "backup_plan": {"fan": [7, 7, 8]}})
    add("harness jit batch 2", {**base_config(10, 1, 0.8, 3, 12, 123), "mode": "harness", "rounds": 80, "batch_size": 2,
                                "backup": "same_primary_jit", "timing": {"primary_time": 0.4, "backup_time": 0.4}})
    add("harness fast_random batch 4 backup 0.5", {**base_config(10, 1, 0.8, 3, 12, 124), "mode": "harness", "rounds": 80,
                                                   "batch_size": 4, "timing": {"primary_time": 0.4, "backup_time": 0.5}})
    add("harness batch 3 differing primary and backup plans",
        {**base_config(12, 1, 0.75, 3, 10, 125), "mode": "harness", "rounds": 60, "batch_size": 3,
         "primary_plan": {"fan": [4, 3, 2, 1]}, "backup_plan": {"fan": [1, 1, 4, 4]}})
    # ---- perf model (perf.cpp:19-73): batch speedup and the backup crossover b*
    for p_, eh, em, tp, tb, b in ((0.9, 3.2, 1.6, 0.8, 0.8, 4), (0.7, 2.5, 1.2, 0.5, 0.0, 16), (0.95, 3.5, 2.0, 1.0, 1.0, 2),
                                  (0.6, 2.0, 1.5, 0.3, 0.3, 1), (0.8, 3.0, 1.0, 0.4, 0.4, 8)):
        add(f"perf p={p_} Eh={eh} Em={em} tp={tp} tb={tb} b={b}",
            {"op": "perf", "hit_rate": p_, "hit_tokens": eh, "miss_tokens": em, "primary_time": tp, "backup_time": tb,
             "batch": b, "critical": True})
    # ---- miss-rate power law (hitmodel.cpp:65-106) feeding geometric_fanout's exponent
    add("fit_powerlaw exact r=0.8", {"op": "fit_powerlaw", "samples": [[f, 0.6 * f ** -0.8] for f in (1, 2, 4, 8, 16)]})
    add("fit_powerlaw noisy", {"op": "fit_powerlaw", "samples": [[1, 0.58], [2, 0.41], [4, 0.22], [4, 0.25], [8, 0.14],
                                                                 [16, 0.061]]})
    add("fit_powerlaw one fan-out (InsufficientData)", {"op": "fit_powerlaw", "samples": [[4, 0.2], [4, 0.3]]})
    add("fit_powerlaw zero miss rejected", {"op": "fit_powerlaw", "samples": [[1, 0.5], [2, 0.0]]})
    add("perf no crossover", {"op": "perf", "hit_rate": 0.5, "hit_tokens": 1.0, "miss_tokens": 3.0, "primary_time": 0.5,
                              "critical": True})
    add("perf hit rate out of range", {"op": "perf", "hit_rate": 1.5, "hit_tokens": 2.0, "miss_tokens": 1.0,
                                       "primary_time": 0.5})
    add("harness synthetic rejected (test_sim.cpp:353-358)",
        {**base_config(8, 1, 0.8, 2, 8, 121), "mode": "harness", "rounds": 10, "synthetic_hit_rate": 0.5})
    # ---- shipped configs (proj/configs/simulate_*.json), shortened
    cfg_lm = {"vocab": 32, "order": 1, "concentration": 0.5, "seed": 7, "alpha_goal": 0.8}
    add("configs/simulate_ssd.json (2000 rounds)",
        {"op": "simulate", "mode": "ssd", "lm": cfg_lm, "lookahead": 4, "scheme": {"kind": "standard", "temperature": 1.0},
         "primary_plan": {"geometric": [0.8, 1.0, 24]}, "backup_plan": {"geometric": [0.3, 1.0, 24]},
         "timing": {"primary_time": 0.4, "backup_time": 0.0}, "backup": "fast_random", "rounds": 2000, "seed": 20250809})
    add("configs/simulate_sd.json (2000 rounds)",
        {"op": "simulate", "mode": "sd", "lm": cfg_lm, "lookahead": 4, "timing": {"primary_time": 0.4},
         "rounds": 2000, "seed": 20250809})
    add("configs/simulate_ssd.json harness (300 rounds)",
        {"op": "simulate", "mode": "harness", "lm": cfg_lm, "lookahead": 4,
         "primary_plan": {"geometric": [0.8, 1.0, 24]}, "backup_plan": {"geometric": [0.3, 1.0, 24]},
         "timing": {"primary_time": 0.4, "backup_time": 0.0}, "rounds": 300, "seed": 20250809})
    return cs


def main():
    po.build(with_ref=True)
    out = []
    for c in cases():
        res = po.reference().call(c["req"])  # errors are golden too
        out.append({**c, "out": res})
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(f"wrote {len(out)} cases to {OUT} ({os.path.getsize(OUT) / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
