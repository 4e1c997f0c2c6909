#!/usr/bin/env python
"""Batch-1 Saguaro (SSD) decode benchmark on B200 — BASELINE.json's metric
(batch-1 decode tokens/sec + speedup vs AR and SD; cache hit rate; HBM GB/s).

Workload (N=1): BASELINE.json configs[1] shapes — Llama-3.1-8B target +
Llama-3.2-1B draft, random-init correlated pair, greedy, lookahead K=4,
fan-out 4 at every position (20 branches), FastRandom backup, batch 1;
verifier and speculator on two streams of one GPU (SURVEY §8e "1-GPU
colocated"). A step = one decode of `--rounds` SSD rounds from a 128-token
synthetic prompt. N>1: independent replicas, one per GPU ("weak").

`--impl reference` times the reference algorithm on host cores instead:
the CPU oracle port of run_protocol_harness over the same transformer pair
(oracle/, test infrastructure), a bounded sample per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.stop = index, [], threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) == 6:
                    self.rows.append(vals)
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload(args, prompt_index: int = 0):
    """The N=1 workload (BASELINE configs[1]): the prompt of step i is a
    fresh uniform-random 128-token prompt (seeded by the root seed and i)."""
    import numpy as np
    import paper_2603_03251_b200 as P
    from paper_2603_03251_b200.configs import shapes
    ts, ds = shapes(args.config, max_ctx=args.max_ctx)
    K = args.lookahead
    fan = [args.fanout] * (K + 1)
    temp = 0.0 if args.greedy else args.temperature
    cfg = P.SimConfig(lookahead=K, scheme=P.SamplingScheme.standard(temp),
                      primary_plan=P.FanOutPlan(list(fan), P.PRIMARY), backup_plan=P.FanOutPlan(list(fan), P.BACKUP),
                      primary_time=0.4, backup_time=0.0, backup_kind=P.FAST_RANDOM, rounds=args.rounds,
                      seed=args.seed + prompt_index)
    prompt = np.random.default_rng([args.seed, prompt_index]).integers(0, ts.vocab, args.prompt_len).tolist()
    return P, ts, ds, cfg, prompt, fan, temp


def workload_config(args) -> dict:
    """`config` of the JSON line — identical in both arms."""
    desc = {"llama8b_1b": " (Llama-3.1-8B/Llama-3.2-1B shapes)", "llama70b_1b": " (Llama-3.1-70B/Llama-3.2-1B shapes)"}
    return {"workload": f"{args.config}{desc.get(args.config, '')} ssd "
                        f"{'greedy' if args.greedy else f'tau={args.temperature}'} K={args.lookahead} "
                        f"F={args.fanout} batch1, one 128-token synthetic prompt per step, {args.rounds} rounds",
            "prompt_len": args.prompt_len, "rounds_per_step": args.rounds,
            "branches": args.fanout * (args.lookahead + 1), "pair_block_out_scale": args.block_out_scale,
            "l2": "no flush: 18 GB of weights streamed per round >> 126 MB L2"}


def cpu_sample(args, threads, prompt_index, rounds, pair=None):
    """The reference algorithm (oracle port of run_protocol_harness,
    test infrastructure) on host cores over the same transformer pair:
    `rounds` decode rounds of step `prompt_index`'s prompt. The prompt is
    prefilled first (untimed, as the GPU value excludes prefill) and only
    the rounds are timed (the oracle's decode_seconds)."""
    import pyoracle
    P, ts, ds, cfg, prompt, fan, temp = workload(args, prompt_index)
    own = pair is None
    t0 = time.perf_counter()
    if own:
        pair = pyoracle.TfPair(P.shape_dict(ts), P.shape_dict(ds), pair_for(args, P).as_dict(), threads=threads)
    build_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    pair.logits(0, prompt[:-1])  # prefill (KV reused by the harness: common prefix)
    pair.logits(1, prompt[:-1])
    prefill_s = time.perf_counter() - t0
    req = {"op": "simulate", "mode": "harness", "lookahead": cfg.lookahead, "rounds": rounds, "seed": cfg.seed,
           "prompt": prompt, "scheme": {"temperature": temp}, "primary_plan": {"fan": fan},
           "backup_plan": {"fan": fan}, "timing": {"primary_time": 0.4}}
    out = pair.call(req)
    if own:
        pair.close()
    return {"tokens": out["tokens"], "seconds": out["decode_seconds"], "build_s": build_s, "prefill_s": prefill_s,
            "rounds": rounds}


def cpu_pair(args, threads):
    import pyoracle
    P, ts, ds, *_ = workload(args)
    return pyoracle.TfPair(P.shape_dict(ts), P.shape_dict(ds), pair_for(args, P).as_dict(), threads=threads)


def run_reference(args):
    """--impl reference: the reference algorithm (oracle port of
    run_protocol_harness) on all host cores, same workload config; a step =
    `--cpu-rounds` decode rounds of that step's prompt (prefill untimed)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    pair = cpu_pair(args, threads)
    toks, secs = 0, 0.0
    for i in range(args.warmup + args.steps):
        s = cpu_sample(args, threads, i, rounds=1 if i < args.warmup else args.cpu_rounds, pair=pair)
        if i >= args.warmup:
            toks += s["tokens"]
            secs += s["seconds"]
    pair.close()
    v = toks / secs if secs > 0 else 0.0
    line = {"impl": "reference", "metric": "batch-1 decode tokens/sec (SSD)", "value": v, "unit": "tokens/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * secs / max(1, args.steps), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16 weights, fp32 compute", "data": "synthetic",
            "config": workload_config(args),
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": threads, "kind": "port",
                             "sample": f"{args.cpu_rounds} decode rounds per step (prompt i of step i, prefill and "
                                       f"initial draft untimed) of the oracle run_protocol_harness port"},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_split(args):
    """N > 1: the split SSD run of DESIGN.md §6 — rank 0 verifier (target on
    its own GPU), ranks 1..N-1 speculators (draft replicas, branch-sharded),
    messages GPU -> GPU through NVLink-mapped mailboxes. One decode stream:
    total work is fixed as N grows ("strong")."""
    import torch
    import torch.distributed as dist
    from paper_2603_03251_b200.split import SplitEngine
    ws, rank, local = dist_env()
    ndev = max(1, torch.cuda.device_count())
    dev = local % ndev
    torch.cuda.set_device(dev)
    # NCCL needs one GPU per rank; fewer GPUs than ranks (a functional run of
    # the split protocol on one GPU) falls back to gloo for the plumbing
    backend = "nccl" if ndev >= ws else "gloo"
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
    else:
        dist.init_process_group("gloo")
    P, ts, ds, cfg, prompt, fan, temp = workload(args)
    B = sum(fan)
    tp = max(1, min(args.tp, ws - 1))
    se = SplitEngine(ts, ds, pair_for(args, P), device=dev, max_branches=max(B, 1), max_lookahead=cfg.lookahead, tp=tp)
    for _ in range(args.warmup):
        se.run(prompt, cfg)
    torch.cuda.synchronize()
    dist.barrier()
    runs, walls = [], []
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            t0 = time.perf_counter()
            r = se.run(prompt, cfg)
            walls.append(time.perf_counter() - t0)
            runs.append(r)
    torch.cuda.synchronize()
    dist.barrier()
    se.close()
    # device time: each run's merged device_ms is already the max over ranks
    dev_ms = sum(r.merged["device_ms"] for r in runs) if rank == 0 else 0.0
    wall = sum(walls)
    t = torch.tensor([wall], device="cuda" if backend == "nccl" else "cpu", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    wall = float(t[0])
    # same-box baselines (AR, synchronous SD) at the verifier's tensor parallelism
    per_run = max(16, sum(r.merged["tokens"] for r in runs) // len(runs)) if rank == 0 else 0
    t = torch.tensor([per_run], dtype=torch.int64, device="cuda" if backend == "nccl" else "cpu")
    dist.broadcast(t, 0)
    if tp > 1:
        from paper_2603_03251_b200.split import tp_baselines
        base = tp_baselines(ts, ds, pair_for(args, P), dev, tp, prompt, cfg, int(t[0]), max(B, 1))
    elif rank == 0:
        eng = P.Engine(ts, ds, pair_for(args, P), device=dev, max_branches=max(B, 1), max_lookahead=cfg.lookahead)
        base = {"ar": eng.run_ar(prompt, cfg.target_scheme or P.SamplingScheme.standard(temp), int(t[0]), cfg.seed),
                "sd": eng.run_sd(prompt, cfg)}
        eng.close()
    if rank == 0:
        m = [r.merged for r in runs]
        tokens = sum(x["tokens"] for x in m)
        hits = sum(x["primary_origin_hits"] + x["backup_origin_hits"] for x in m)
        lookups = sum(x["primary_origin_lookups"] + x["backup_origin_lookups"] for x in m)
        acc = sum(x["accepted_sum"] for x in m) / sum(x["rounds"] for x in m)
        value = tokens / (dev_ms * 1e-3)
        ar, sd = base["ar"], base["sd"]
        ar_tps = ar.tokens / (ar.device_ms * 1e-3)
        sd_tps = sd.tokens / (sd.device_ms * 1e-3)
        line = {"metric": "batch-1 decode tokens/sec (SSD)", "value": value, "unit": "tokens/s", "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / len(runs),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (random-init correlated pair, random prompt)",
                "config": {"workload": f"{args.config} ssd greedy K={cfg.lookahead} F={args.fanout} batch1 "
                                       f"split verifier TP{tp} + {ws - tp} speculators (branch-sharded); AR / SD "
                                       f"baselines at TP{tp} (draft replicated)",
                           "prompt_len": args.prompt_len, "rounds_per_step": args.rounds, "branches": B,
                           "l2": "no flush: weights streamed per round >> 126 MB L2",
                           "parallelism": f"verifier TP{tp} + speculator x{ws - tp}, NVLink mailboxes",
                           "gpus_visible": ndev},
                "e2e": {"value": tokens / wall, "unit": "tokens/s", "h2d_bytes_per_step": 4 * len(prompt),
                        "d2h_bytes_per_step": 4 * (tokens // len(runs))},
                "gpu_launches": sum(x["kernel_launches"] for x in m) // len(m),
                "ssd_tokens_per_s": value, "ar_tokens_per_s": ar_tps, "sd_tokens_per_s": sd_tps,
                "speedup_vs_ar": value / ar_tps, "speedup_vs_sd": value / sd_tps,
                "hit_rate": hits / lookups if lookups else None, "mean_accepted": acc,
                "alpha": alpha_of(acc, cfg.lookahead),
                "tokens_per_round": tokens / sum(x["rounds"] for x in m), "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def path_roofline(tw, dw, K, hbm_gbs, ssd_tokens_per_round, sd_tokens_per_round, ssd_tps, ar_tps, sd_tps):
    """tokens/s each loop would reach if every forward streamed
    its weights at the measured HBM bandwidth (bytes per round / bandwidth,
    times the measured tokens per round), and the achieved fraction. One GPU
    (colocated): an SSD round streams the target once (verify) and the draft
    K + 1 times (extend + K branch steps); SD streams the draft K times and
    the target once; AR the target once per token."""
    bw = hbm_gbs * 1e9
    ssd_s = (tw + (K + 1) * dw) / bw
    sd_s = (tw + K * dw) / bw
    ar_s = tw / bw
    out = {"ssd_round_bytes": tw + (K + 1) * dw, "ssd_tokens_per_s": ssd_tokens_per_round / ssd_s,
           "sd_tokens_per_s": sd_tokens_per_round / sd_s, "ar_tokens_per_s": 1.0 / ar_s}
    out["ssd_frac"] = ssd_tps / out["ssd_tokens_per_s"]
    out["sd_frac"] = sd_tps / out["sd_tokens_per_s"]
    out["ar_frac"] = ar_tps / out["ar_tokens_per_s"]
    return out


def alpha_of(mean_accepted: float, K: int) -> float:
    """Per-token acceptance alpha from the mean accepted length
    (E[accepted] = sum_{i=1..K} alpha^i)."""
    lo, hi = 0.0, 1.0
    for _ in range(60):
        a = 0.5 * (lo + hi)
        lo, hi = (a, hi) if sum(a ** i for i in range(1, K + 1)) < mean_accepted else (lo, a)
    return lo


def pair_for(args, P):
    """The correlated random pair; --block-out-scale is the divergence knob
     that sets the acceptance rate."""
    return P.Pair(block_out_scale=args.block_out_scale)


def _ci95(xs):
    import math
    xs = [x for x in xs if x is not None]
    if not xs:
        return None
    m = sum(xs) / len(xs)
    if len(xs) < 2:
        return {"mean": m, "ci95": None, "n": len(xs)}
    sd = math.sqrt(sum((x - m) ** 2 for x in xs) / (len(xs) - 1))
    return {"mean": m, "ci95": 1.96 * sd / math.sqrt(len(xs)), "n": len(xs)}


def _ratio(a, b):
    return a / b if b else None


def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    if ws > 1 and args.multi == "split":
        return run_split(args)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    P, ts, ds, cfg0, prompt0, fan, temp = workload(args)
    B = sum(fan)
    K = cfg0.lookahead
    eng = P.Engine(ts, ds, pair_for(args, P), device=local, max_branches=max(B, 1), max_lookahead=K)

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # step i decodes prompt i (rank r: prompts offset by r * 1000, replicas)
    def step_work(i):
        return workload(args, 1000 * rank + i)

    for i in range(args.warmup):
        _, _, _, cfg, prompt, _, _ = step_work(i)
        eng.run_ssd(prompt, cfg)
    barrier()
    runs, walls, prompts = [], [], []
    with ClockSampler(local) as clk:
        for i in range(args.warmup, args.warmup + args.steps):
            _, _, _, cfg, prompt, _, _ = step_work(i)
            t0 = time.perf_counter()
            r = eng.run_ssd(prompt, cfg)  # host prompt in, host tokens out (the public API call)
            walls.append(time.perf_counter() - t0)
            runs.append(r)
            prompts.append((prompt, cfg))
    barrier()
    tokens = sum(r.tokens for r in runs)
    dev_ms = sum(r.device_ms for r in runs)
    live_round_ms = dev_ms / max(1, sum(r.rounds for r in runs))  # CUDA events around the round graphs
    wall = sum(walls)
    launches = sum(r.kernel_launches for r in runs) // max(1, len(runs))
    if ws > 1:
        t = torch.tensor([dev_ms, wall], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        dev_ms, wall = float(t[0]), float(t[1])
    value = ws * tokens / (dev_ms * 1e-3)
    e2e = ws * tokens / wall
    ssd_tps = tokens / (dev_ms * 1e-3)
    # same-box baselines on the same prompts: AR (the same token count) and synchronous SD (same rounds)
    ar_tok = ar_ms = sd_tok = sd_ms = sd_acc = sd_rounds = 0
    for (prompt, cfg), r in zip(prompts, runs):
        ar = eng.run_ar(prompt, cfg.target_scheme or P.SamplingScheme.standard(temp), max(16, r.tokens), cfg.seed)
        sd = eng.run_sd(prompt, cfg)
        ar_tok += ar.tokens
        ar_ms += ar.device_ms
        sd_tok += sd.tokens
        sd_ms += sd.device_ms
        sd_acc += sd.accepted_sum
        sd_rounds += sd.rounds
    ar_tps = ar_tok / (ar_ms * 1e-3)
    sd_tps = sd_tok / (sd_ms * 1e-3)
    # segment breakdown of the colocated round (a separate profiled run: globaltimer stamp kernels in the
    # round graph, one host sync per round; the roofline below uses the live timed-region round time)
    rp = eng.profile_ssd_round(prompts[0][0], prompts[0][1])
    prof_t = eng.profile_forward(0, 1, args.prompt_len, 10)
    prof_x = eng.profile_forward(1, K + 1, args.prompt_len, 10)
    prof_b = eng.profile_forward(1, B, args.prompt_len, 10)
    pk, pk_kind = peaks()
    hbm = float(pk.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
    read_peak = eng.read_bw(4 << 30, 10)
    tw, dw = eng.weight_bytes(0), eng.weight_bytes(1)
    round_bytes = tw + (K + 1) * dw
    achieved = round_bytes / (live_round_ms * 1e-3) / 1e9
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "round_traffic.json")
    if os.path.exists(tfile):
        with open(tfile) as f:
            traffic = json.load(f).get("bytes_per_round")
    per = [{"alpha": alpha_of(r.accepted_sum / r.rounds, K), "hit": r.hit_rate(), "hit_p": r.hit_rate_primary(),
            "hit_b": r.hit_rate_backup(), "tpr": r.tokens / r.rounds,
            "e_hit": _ratio(r.hit_round_tokens, r.hit_rounds), "e_miss": _ratio(r.miss_round_tokens, r.miss_rounds),
            "tps": r.tokens / (r.device_ms * 1e-3)} for r in runs]
    hits = sum(r.hits_total() for r in runs)
    lookups = sum(r.lookups() for r in runs)
    acc = sum(r.accepted_sum for r in runs) / sum(r.rounds for r in runs)
    line = {"metric": "batch-1 decode tokens/sec (SSD)", "value": value, "unit": "tokens/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / len(runs),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init correlated pair, uniform-random prompts, one per step)",
            "config": {**workload_config(args),
                       "parallelism": f"replicas{ws}" if ws > 1 else "verifier+speculator streams on 1 GPU"},
            "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": 4 * args.prompt_len + 1024,
                    "d2h_bytes_per_step": 4 * (tokens // len(runs)) + 4 * 3 * args.rounds},
            "gpu_launches": launches,
            "ssd_tokens_per_s": ssd_tps, "ar_tokens_per_s": ar_tps, "sd_tokens_per_s": sd_tps,
            "speedup_vs_ar": ssd_tps / ar_tps, "speedup_vs_sd": ssd_tps / sd_tps,
            "decode_tokens": tokens, "prompts": len(runs),
            "hit_rate": hits / lookups if lookups else None,
            "p_hit_primary": _ratio(sum(r.primary_origin_hits for r in runs),
                                    sum(r.primary_origin_lookups for r in runs)),
            "p_hit_backup": _ratio(sum(r.backup_origin_hits for r in runs), sum(r.backup_origin_lookups for r in runs)),
            "e_hit": _ratio(sum(r.hit_round_tokens for r in runs), sum(r.hit_rounds for r in runs)),
            "e_miss": _ratio(sum(r.miss_round_tokens for r in runs), sum(r.miss_rounds for r in runs)),
            "mean_accepted": acc, "alpha": alpha_of(acc, K),
            "sd_mean_accepted": sd_acc / max(1, sd_rounds),
            "tokens_per_round": tokens / sum(r.rounds for r in runs),
            "per_prompt": {k: _ci95([x[k] for x in per]) for k in per[0]},
            "round_ms": rp,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": traffic, "peak_kind": pk_kind, "read_only_peak": read_peak,
                         "frac_of_read_peak": achieved / read_peak,
                         "kernel": "weight-streaming tcgen05 GEMM forwards of the colocated SSD round "
                                   "(8B verify M=K+1 on one stream || 1B extend M=K+1 + K branch steps M=B on "
                                   "the other); ms per round = CUDA events around the timed region's round "
                                   "graphs / rounds",
                         "bytes_per_round": round_bytes, "ms_per_round": live_round_ms,
                         "profiled_round_ms": rp["round"],
                         "verify_forward_gbs": tw / (rp["verify_forward"] * 1e-3) / 1e9,
                         "branch_forward_gbs": K * dw / (rp["branch_forwards"] * 1e-3) / 1e9,
                         "standalone": {
                             "t1_gemm_gbs": prof_t["gemm_bytes"] / (prof_t["ms_gemm"] * 1e-3) / 1e9,
                             "t1_forward_ms": prof_t["ms_forward"], "t1_gemm_ms": prof_t["ms_gemm"],
                             "d5_forward_ms": prof_x["ms_forward"], "d20_forward_ms": prof_b["ms_forward"],
                             "d20_gemm_gbs": prof_b["gemm_bytes"] / (prof_b["ms_gemm"] * 1e-3) / 1e9}},
            "model_bytes": {"target_step": tw, "draft_step": dw},
            "path_roofline": path_roofline(tw, dw, K, hbm, tokens / sum(r.rounds for r in runs),
                                           sd_acc / max(1, sd_rounds) + 1.0, ssd_tps, ar_tps, sd_tps),
            "clocks": clk.summary()}
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        s = cpu_sample(args, os.cpu_count() or 1, args.warmup, rounds=args.cpu_rounds)
        line["cpu_baseline"] = {"value": s["tokens"] / s["seconds"], "unit": "tokens/s", "cores": os.cpu_count(),
                                "kind": "port",
                                "sample": f"{args.cpu_rounds} decode rounds of the first timed prompt through the "
                                          f"oracle run_protocol_harness port (same pair, config and seed); prefill "
                                          f"{s['prefill_s']:.1f}s and model build {s['build_s']:.1f}s untimed"}
    eng.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="llama8b_1b")
    # ~512 decode tokens per prompt at ~3.5 tokens per round
    ap.add_argument("--rounds", type=int, default=144)
    ap.add_argument("--cpu-rounds", type=int, default=3, help="decode rounds per CPU-baseline sample")
    ap.add_argument("--lookahead", type=int, default=4)
    ap.add_argument("--fanout", type=int, default=4)
    ap.add_argument("--prompt-len", type=int, default=128)
    ap.add_argument("--max-ctx", type=int, default=1024)
    ap.add_argument("--temperature", type=float, default=1.0)
    ap.add_argument("--sampled", dest="greedy", action="store_false")
    ap.add_argument("--seed", type=int, default=20250809)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # pair divergence knob calibrated on this workload to alpha ~ 0.8 (
    # scripts/bench_alpha.py, profiles/r01_summary.md); alpha is reported
    ap.add_argument("--block-out-scale", type=float, default=0.06)
    ap.add_argument("--tp", type=int, default=1, help="N>1 split mode: tensor-parallel verifier ranks")
    ap.add_argument("--multi", default="split", choices=["split", "replicas"],
                    help="N>1: split verifier/speculator processes (default) or independent replicas")
    ap.set_defaults(greedy=True)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
