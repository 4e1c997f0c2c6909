"""Host side of a split SSD run: the reference's
VerifierProcess and DraftProcess (sim.cpp:321-485) as one OS process each,
rank 0 = verifier (target model), ranks 1..G = speculators (draft model,
branch-sharded). torch.distributed is plumbing only: it exchanges the
64-byte CUDA IPC handles of the device mailboxes once and merges the
counters at the end. Every per-round message travels GPU -> GPU inside the
round graphs (split.cuh), never through the host.

Launch: `python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N`
(rank r on cuda:(local_rank % device_count)) or tests/test_split.py.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

from . import _native as N
from .api import ConfigError, Engine, Pair, RunStats, SimConfig

VERIFIER_RANK = 0


def role_of(rank: int, world_size: int, tp: int = 1) -> int:
    """Ranks [0, tp) verify (a tensor-parallel verifier when tp > 1); every
    other rank speculates."""
    if tp < 1 or world_size < tp + 1:
        raise ConfigError("split: needs the verifier ranks + at least one speculator")
    if not 0 <= rank < world_size:
        raise ConfigError("split: rank out of range")
    return N.ROLE_VERIFIER if rank < tp else N.ROLE_SPECULATOR


def branch_block(B: int, rank: int, G: int) -> tuple[int, int]:
    """Contiguous block [lo, lo + n) of the B keyed branches decoded by
    speculator `rank` of G (mirror of engine.cu branch_block)."""
    lo = B * rank // G
    return lo, B * (rank + 1) // G - lo


def branch_owner(b: int, B: int, G: int) -> int:
    """Speculator that decodes (and, on a hit, sends) branch b."""
    for g in range(G):
        lo, n = branch_block(B, g, G)
        if lo <= b < lo + n:
            return g
    raise ValueError("branch out of range")


def exchange_handles(handle: bytes, group=None) -> list[bytes]:
    """All-gather every process's mailbox handle, ordered by rank."""
    import torch.distributed as dist
    out: list = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, handle, group=group)
    if any(not isinstance(h, bytes) or len(h) != N.MAILBOX_HANDLE_BYTES for h in out):
        raise ConfigError("split: malformed mailbox handle")
    return out


COUNTERS = ("rounds", "tokens", "virtual_time", "primary_origin_lookups", "primary_origin_hits",
            "backup_origin_lookups", "backup_origin_hits", "hit_rounds", "miss_rounds", "initial_rounds",
            "hit_round_tokens", "miss_round_tokens", "accepted_sum")


def merge_stats(per_rank: Sequence[dict], tp: int = 1) -> dict:
    """RunStats of a split run from every rank's own counters ([verifier
    ranks 0..tp-1, speculator 0, ...]). The verifier knows tokens / accepted;
    each speculator rebuilds the same history from (k*, t*) and keeps the
    lookup / hit / clock counters, so every counter must agree across
    speculators (and across the ranks of a tensor-parallel verifier), and
    tokens / accepted with the verifier. Device time = the slowest rank."""
    if len(per_rank) < tp + 1:
        raise ConfigError("split: need the verifier and at least one speculator")
    v, s0 = per_rank[0], per_rank[tp]
    for vr in per_rank[1:tp]:
        for k in ("tokens", "accepted_sum", "rounds"):
            if vr[k] != v[k]:
                raise ConfigError(f"split: tensor-parallel verifier ranks disagree on {k}")
    for s in per_rank[tp + 1:]:
        for k in COUNTERS:
            if s[k] != s0[k]:
                raise ConfigError(f"split: speculators disagree on {k}")
    for k in ("tokens", "accepted_sum", "rounds"):
        if v[k] != s0[k]:
            raise ConfigError(f"split: verifier and speculator disagree on {k}")
    out = dict(s0)
    out["device_ms"] = max(r["device_ms"] for r in per_rank)
    out["kernel_launches"] = sum(r["kernel_launches"] for r in per_rank)
    return out


@dataclass
class SplitRun:
    rank: int
    world_size: int
    stats: RunStats             # this process's own counters
    merged: Optional[dict]      # rank 0: the whole run's RunStats fields
    tokens: Optional[list]      # rank 0: the emitted token stream


class SplitEngine:
    """One process of a split run: builds its role's model on `device`,
    exchanges mailbox handles with the other ranks (collective), and runs
    rounds of the protocol."""

    def __init__(self, target, draft, pair: Pair = Pair(), device: int = 0, max_branches: int = 64,
                 max_lookahead: int = 8, group=None, tp: int = 1):
        """tp > 1: ranks [0, tp) form a tensor-parallel verifier (tp.cuh)."""
        import torch.distributed as dist
        self.group = group
        self.tp = tp
        self.rank = dist.get_rank(group)
        self.world_size = dist.get_world_size(group)
        self.role = role_of(self.rank, self.world_size, tp)
        vrank = self.rank if self.role == N.ROLE_VERIFIER else 0
        self.engine = Engine(target, draft, pair, device=device, max_branches=max_branches,
                             max_lookahead=max_lookahead, role=self.role, tp_rank=vrank,
                             tp_size=tp if self.role == N.ROLE_VERIFIER else 1)
        if tp > 1:  # map the verifier ranks' collective regions
            mine = self.engine.tp_handle() if self.role == N.ROLE_VERIFIER else bytes(N.MAILBOX_HANDLE_BYTES)
            tph = exchange_handles(mine, group)
            if self.role == N.ROLE_VERIFIER:
                self.engine.tp_connect(tph[:tp])
        handles = exchange_handles(self.engine.mailbox_handle(), group)
        self.engine.connect(handles, self.rank)
        dist.barrier(group)  # every inbox is mapped and clean before anyone sends

    @property
    def n_spec(self) -> int:
        return self.world_size - self.tp

    def run(self, prompt: Sequence[int], cfg: SimConfig) -> SplitRun:
        import torch.distributed as dist
        if self.role == N.ROLE_VERIFIER:
            r = self.engine.run_ssd_verifier(prompt, cfg, self.n_spec)
        else:
            r = self.engine.run_ssd_speculator(prompt, cfg, self.rank - self.tp, self.n_spec, self.tp)
        fields = [f for f, _ in N.RunStatsC._fields_]
        mine = {f: getattr(r, f) for f in fields}
        allst: list = [None] * self.world_size
        dist.all_gather_object(allst, mine, group=self.group)
        merged = merge_stats(allst, self.tp) if self.rank == VERIFIER_RANK else None
        return SplitRun(self.rank, self.world_size, r, merged, r.streams[0] if r.streams else None)

    def close(self):
        self.engine.close()


def tp_baselines(target, draft, pair: Pair, device: int, tp: int, prompt: Sequence[int], cfg: SimConfig,
                 ar_tokens: int, max_branches: int, group=None) -> Optional[dict]:
    """Same-box AR and synchronous SD baselines of a tensor-parallel target
    (BASELINE configs[3]): ranks [0, tp) each build a colocated TP engine
    (target shard + replicated draft), connect their collective regions and
    run run_ar / run_sd in lock step (every rank computes the same tokens);
    other ranks only take part in the handle exchange. Rank 0 returns
    {"ar": RunStats, "sd": RunStats}; every other rank None."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    mine = rank < tp
    eng = None
    if mine:
        eng = Engine(target, draft, pair, device=device, max_branches=max_branches, max_lookahead=cfg.lookahead,
                     role=N.ROLE_COLOCATED, tp_rank=rank, tp_size=tp)
    h = eng.tp_handle() if mine else bytes(N.MAILBOX_HANDLE_BYTES)
    handles = exchange_handles(h, group)
    if mine:
        eng.tp_connect(handles[:tp])
    dist.barrier(group)
    out = None
    if mine:
        from .api import SamplingScheme
        ar = eng.run_ar(prompt, cfg.target_scheme or SamplingScheme.standard(cfg.scheme.temperature), ar_tokens,
                        cfg.seed)
        sd = eng.run_sd(prompt, cfg)
        out = {"ar": ar, "sd": sd} if rank == VERIFIER_RANK else None
        eng.close()
    dist.barrier(group)
    return out
