"""Python mirror of the reference's speculator / verifier / speculation-cache
interface (ssd-lab proj/include/ssdlab: categorical.hpp, cache.hpp,
specdec.hpp, sim.hpp, errors.hpp), calling the B200 engine through the C-ABI
(include/ssd_b200.h). Names, argument meaning and error classes follow the
reference so the parity tests read like the reference's own tests.

Host code here only marshals arguments; every decode step, verification,
key selection, lookup and backup runs in the native library on the GPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _native as N

# ------------------------------------------------------------------ errors
# errors.hpp:9-61


class Error(RuntimeError):
    """ssdlab::Error"""


class AllZeroError(Error): pass  # noqa: E701
class DegenerateResidualError(Error): pass  # noqa: E701
class TooLargeError(Error): pass  # noqa: E701
class BudgetTooSmallError(Error): pass  # noqa: E701
class DivergentError(Error): pass  # noqa: E701
class InsufficientDataError(Error): pass  # noqa: E701
class UnreachableError(Error): pass  # noqa: E701
class NoCrossoverError(Error): pass  # noqa: E701
class ProtocolViolationError(Error): pass  # noqa: E701
class ConfigError(Error): pass  # noqa: E701
class CudaError(Error): pass  # noqa: E701


_BY_CODE = {1: Error, 2: AllZeroError, 3: DegenerateResidualError, 4: TooLargeError, 5: BudgetTooSmallError,
            6: DivergentError, 7: InsufficientDataError, 8: UnreachableError, 9: NoCrossoverError,
            10: ProtocolViolationError, 11: ConfigError, 100: CudaError}


def _check(status: int) -> None:
    if status != 0:
        msg = N.load().ssd_last_error().decode(errors="replace")
        raise _BY_CODE.get(status, Error)(msg)


# ------------------------------------------------------------------ types
@dataclass(frozen=True)
class SamplingScheme:
    """dist::SamplingScheme (categorical.hpp:43-60); temperature 0 = greedy."""
    kind: str = "standard"
    temperature: float = 1.0
    fan_out: int = 0
    downweight: float = 1.0

    @staticmethod
    def standard(temperature: float = 1.0) -> "SamplingScheme":
        return SamplingScheme("standard", temperature)

    @staticmethod
    def saguaro(fan_out: int, downweight: float, temperature: float = 1.0) -> "SamplingScheme":
        return SamplingScheme("saguaro", temperature, fan_out, downweight)

    @staticmethod
    def greedy() -> "SamplingScheme":
        return SamplingScheme("standard", 0.0)

    def c(self) -> N.Scheme:
        return N.Scheme(1 if self.kind == "saguaro" else 0, self.fan_out, self.temperature, self.downweight)


PRIMARY, BACKUP = 0, 1  # specdec::Origin


@dataclass
class FanOutPlan:
    """cache::FanOutPlan (cache.hpp:18-25)."""
    fan_out: list
    role: int = PRIMARY
    budget: int = 0

    @property
    def lookahead(self) -> int:
        return len(self.fan_out) - 1

    def total(self) -> int:
        return int(sum(self.fan_out))

    def c(self) -> N.Plan:
        p = N.Plan()
        p.lookahead = self.lookahead
        p.role = self.role
        p.budget = self.budget or self.total()
        for k, f in enumerate(self.fan_out):
            p.fan_out[k] = int(f)
        return p


def _plan_from_c(p: N.Plan) -> FanOutPlan:
    return FanOutPlan([p.fan_out[k] for k in range(p.lookahead + 1)], p.role, p.budget)


def geometric_fanout(acceptance: float, exponent: float, lookahead: int, budget: int, role: int = PRIMARY) -> FanOutPlan:
    """cache::geometric_fanout (cache.cpp:39-113), evaluated natively."""
    p = N.Plan()
    _check(N.load().ssd_geometric_fanout(acceptance, exponent, lookahead, budget, role, C.byref(p)))
    return _plan_from_c(p)


def uniform_fanout(lookahead: int, budget: int, role: int = PRIMARY) -> FanOutPlan:
    """cache::uniform_fanout (cache.cpp:115-127)."""
    p = N.Plan()
    _check(N.load().ssd_uniform_fanout(lookahead, budget, role, C.byref(p)))
    return _plan_from_c(p)


def conditional_hit_rate(plan: FanOutPlan, acceptance: float, exponent: float) -> float:
    return N.load().ssd_conditional_hit_rate(C.byref(plan.c()), acceptance, exponent)


FAST_RANDOM, SAME_PRIMARY_JIT = "fast_random", "same_primary_jit"  # sim::BackupKind


def speedup_batch(hit_rate: float, hit_tokens: float, miss_tokens: float, primary_time: float,
                  backup_time: float, batch: float) -> float:
    """perf::speedup_batch (perf.cpp:44-55): per-sequence speedup under
    whole-batch stalls; times in units of one verification pass."""
    out = C.c_double()
    _check(N.load().ssd_speedup_batch(hit_rate, hit_tokens, miss_tokens, primary_time, backup_time, batch,
                                      C.byref(out)))
    return out.value


def fit_powerlaw(samples) -> tuple:
    """hitmodel::fit_powerlaw (hitmodel.cpp:65-106): (exponent r,
    log_amplitude, r_squared) of miss = A F^-r over (fan-out, miss) pairs."""
    f = np.ascontiguousarray([float(a) for a, _ in samples], dtype=np.float64)
    m = np.ascontiguousarray([float(b) for _, b in samples], dtype=np.float64)
    r, la, r2 = C.c_double(), C.c_double(), C.c_double()
    _check(N.load().ssd_fit_powerlaw(f.ctypes.data_as(C.POINTER(C.c_double)), m.ctypes.data_as(C.POINTER(C.c_double)),
                                     len(f), C.byref(r), C.byref(la), C.byref(r2)))
    return r.value, la.value, r2.value


def critical_batch(hit_rate: float, hit_tokens: float, miss_tokens: float, primary_time: float) -> float:
    """perf::critical_batch (perf.cpp:57-73): the batch size b* where the
    free backup overtakes the JIT re-draft (NoCrossoverError if none)."""
    out = C.c_double()
    _check(N.load().ssd_critical_batch(hit_rate, hit_tokens, miss_tokens, primary_time, C.byref(out)))
    return out.value


def saguaro_backup(batch: int, hit_rate: float, hit_tokens: float, miss_tokens: float, primary_time: float,
                   jit_time: Optional[float] = None, fast_time: float = 0.0) -> str:
    """The Saguaro fallback policy (PAPER §5): re-use the
    primary speculator as a just-in-time backup below the crossover batch
    b*, the free FastRandom backup at or above it. Without a crossover the
    strategy with the larger speedup_batch at this batch size wins."""
    jt = primary_time if jit_time is None else jit_time
    try:
        return SAME_PRIMARY_JIT if batch < critical_batch(hit_rate, hit_tokens, miss_tokens, primary_time) \
            else FAST_RANDOM
    except (NoCrossoverError, Error):
        j = speedup_batch(hit_rate, hit_tokens, miss_tokens, primary_time, jt, batch)
        f = speedup_batch(hit_rate, hit_tokens, miss_tokens, primary_time, fast_time, batch)
        return SAME_PRIMARY_JIT if j > f else FAST_RANDOM


@dataclass
class SimConfig:
    """sim::SimConfig (sim.hpp:28-53); the models live in the Engine."""
    lookahead: int = 4
    scheme: SamplingScheme = field(default_factory=SamplingScheme.standard)
    target_scheme: Optional[SamplingScheme] = None  # default: standard(scheme.temperature) as cli.cpp:211
    primary_plan: Optional[FanOutPlan] = None
    backup_plan: Optional[FanOutPlan] = None
    primary_time: float = 0.3
    backup_time: float = 0.0
    backup_kind: str = FAST_RANDOM
    rounds: int = 1000
    seed: int = 0
    accept_scale: float = 1.0
    batch_size: int = 1  # sim.hpp:40; run_ssd only (whole-batch stall semantics)

    def c(self) -> N.SimConfigC:
        ts = self.target_scheme or SamplingScheme.standard(self.scheme.temperature)
        pp = self.primary_plan or uniform_fanout(self.lookahead, self.lookahead + 1, PRIMARY)
        bp = self.backup_plan or FanOutPlan(list(pp.fan_out), BACKUP, pp.budget)
        return N.SimConfigC(self.lookahead, self.scheme.c(), ts.c(), pp.c(), bp.c(),
                            0 if self.backup_kind == SAME_PRIMARY_JIT else 1, self.primary_time, self.backup_time,
                            self.rounds, self.seed, self.accept_scale)


@dataclass
class RunStats:
    """sim::RunStats (sim.hpp:55-104) plus device time."""
    rounds: int
    tokens: int
    virtual_time: float
    primary_origin_lookups: int
    primary_origin_hits: int
    backup_origin_lookups: int
    backup_origin_hits: int
    hit_rounds: int
    miss_rounds: int
    initial_rounds: int
    hit_round_tokens: int
    miss_round_tokens: int
    accepted_sum: float
    device_ms: float
    kernel_launches: int
    streams: list = field(default_factory=list)
    batch: int = 1
    outcomes: Optional[np.ndarray] = None  # [rounds, 2] (accepted, bonus)
    hits: Optional[np.ndarray] = None      # [rounds] 1/0, -1 on the last round
    transcript: Optional[list] = None      # harness round transcript (sim.cpp:489-500), parsed JSONL

    @classmethod
    def _from_c(cls, s: N.RunStatsC, stream=None):
        return cls(*[getattr(s, f) for f, _ in N.RunStatsC._fields_], streams=[stream] if stream is not None else [])

    def speed(self) -> float:
        return self.tokens / self.virtual_time

    def lookups(self) -> int:
        return self.primary_origin_lookups + self.backup_origin_lookups

    def hits_total(self) -> int:
        return self.primary_origin_hits + self.backup_origin_hits

    def hit_rate(self) -> float:
        return self.hits_total() / self.lookups() if self.lookups() else 0.0

    def hit_rate_primary(self):
        return self.primary_origin_hits / self.primary_origin_lookups if self.primary_origin_lookups else None

    def hit_rate_backup(self):
        return self.backup_origin_hits / self.backup_origin_lookups if self.backup_origin_lookups else None

    def mean_accepted(self) -> float:
        return self.accepted_sum / self.rounds

    def tokens_per_second(self) -> float:
        return self.tokens / (self.device_ms * 1e-3) if self.device_ms > 0 else 0.0


class Stream:
    """rng::Stream (rng.hpp:29-48): a caller-owned mt19937_64 stream. Engine
    calls that take it advance it exactly as the reference advances the
    Stream& it is given (one uniform per draw, one next_u64 per build_cache)."""

    def __init__(self, seed: int):
        self.c = N.RngStream()
        N.load().ssd_rng_stream_seed(C.byref(self.c), int(seed) & 0xFFFFFFFFFFFFFFFF)

    def next_u64(self) -> int:
        return int(N.load().ssd_rng_stream_next_u64(C.byref(self.c)))

    def next_uniform(self) -> float:
        return float(N.load().ssd_rng_stream_next_uniform(C.byref(self.c)))

    def copy(self) -> "Stream":
        s = Stream.__new__(Stream)
        s.c = N.RngStream()
        C.memmove(C.byref(s.c), C.byref(self.c), C.sizeof(N.RngStream))
        return s


def derive_seed(root: int, index: int) -> int:
    """rng::derive_seed (rng.hpp:24-26)."""
    return int(N.load().ssd_derive_seed(int(root) & 0xFFFFFFFFFFFFFFFF, int(index) & 0xFFFFFFFFFFFFFFFF))


@dataclass
class RoundResult:
    """specdec::RoundResult (specdec.hpp:44-52): outcome (k, t*) and the
    emitted tokens (accepted prefix + bonus)."""
    accepted: int
    bonus: int
    emitted: list


@dataclass
class Speculation:
    """specdec::Speculation (specdec.hpp:22-28): tokens plus the draft logit
    rows they were drawn from (the recorded laws are the scheme applied to
    these rows)."""
    tokens: list
    rows: Optional[np.ndarray] = None
    origin: int = PRIMARY


@dataclass
class SpeculationCache:
    """cache::SpeculationCache (cache.hpp:114-135): (accepted, bonus) -> tokens."""
    entries: dict
    round_origin: int = PRIMARY
    rows: Optional[dict] = None  # (k, t) -> [next_K][V] draft logit rows (build_cache_stream)

    def lookup(self, accepted: int, bonus: int):
        return self.entries.get((accepted, bonus))

    def speculation(self, accepted: int, bonus: int) -> Optional["Speculation"]:
        """The stored Speculation (tokens + the rows they were drawn from)."""
        t = self.entries.get((accepted, bonus))
        if t is None:
            return None
        return Speculation(list(t), None if self.rows is None else self.rows[(accepted, bonus)], PRIMARY)

    def size(self) -> int:
        return len(self.entries)


# ------------------------------------------------------------------ shapes
def model_shape(vocab, d_model, n_layers, n_heads, n_kv_heads, head_dim, ffn, tied=False, max_ctx=4096,
                rope_theta=500000.0, norm_eps=1e-5) -> N.ModelShape:
    return N.ModelShape(vocab, d_model, n_layers, n_heads, n_kv_heads, head_dim, ffn, 1 if tied else 0, max_ctx,
                        rope_theta, norm_eps)


def shape_dict(s: N.ModelShape) -> dict:
    """Oracle-side (oracle/oracle_capi.cpp parse_shape) description."""
    return {"vocab": s.vocab, "d": s.d_model, "layers": s.n_layers, "heads": s.n_heads, "kv_heads": s.n_kv_heads,
            "head_dim": s.head_dim, "ffn": s.ffn, "tied": bool(s.tied), "rope_theta": s.rope_theta,
            "norm_eps": s.norm_eps, "max_ctx": s.max_ctx}


@dataclass
class Pair:
    """Correlated random pair parameters."""
    seed: int = 20250809
    embed_scale: float = 1.0
    shared_mlp_scale: float = 8.0
    block_out_scale: float = 0.1
    target_private_embed: float = 0.1
    target_private_head: float = 0.25
    draft_gain_mix: float = 0.0
    logit_scale: float = 0.25

    def c(self) -> N.PairParams:
        return N.PairParams(self.seed, self.embed_scale, self.shared_mlp_scale, self.block_out_scale,
                            self.target_private_embed, self.target_private_head, self.draft_gain_mix,
                            self.logit_scale)

    def as_dict(self) -> dict:
        return dict(self.__dict__)


def _i32(seq) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(seq, dtype=np.int32))


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class Engine:
    """A (target, draft) pair resident on one B200 plus its decode loops."""

    def __init__(self, target: N.ModelShape, draft: N.ModelShape, pair: Pair = Pair(), device: int = 0,
                 max_branches: int = 64, max_lookahead: int = 8, role: int = N.ROLE_COLOCATED, tp_rank: int = 0,
                 tp_size: int = 1, max_batch: int = 1):
        """role: ROLE_COLOCATED (both models), ROLE_VERIFIER (target only) or
        ROLE_SPECULATOR (draft only) — the processes of a split run. A
        verifier may be tensor-parallel: rank tp_rank of tp_size (connect the
        ranks with tp_handle / tp_connect)."""
        self.lib = N.load()
        self.target, self.draft, self.pair = target, draft, pair
        self.vocab = target.vocab
        self.role = role
        self.tp_rank, self.tp_size = tp_rank, tp_size
        self.max_batch = max_batch
        h = C.c_void_p()
        if max_batch > 1:  # batch lanes (colocated engine)
            _check(self.lib.ssd_engine_create_batch(C.byref(target), C.byref(draft), C.byref(pair.c()), device,
                                                    max_batch, max_branches, max_lookahead, C.byref(h)))
        else:
            _check(self.lib.ssd_engine_create_tp(C.byref(target), C.byref(draft), C.byref(pair.c()), device, role,
                                                 tp_rank, tp_size, max_branches, max_lookahead, C.byref(h)))
        self.h = h

    def tp_handle(self) -> bytes:
        buf = (C.c_uint8 * N.MAILBOX_HANDLE_BYTES)()
        _check(self.lib.ssd_tp_export(self.h, buf))
        return bytes(buf)

    def tp_connect(self, handles: Sequence[bytes]):
        """Map the TP ranks' collective regions (handles ordered by TP rank)."""
        blob = b"".join(handles)
        if len(handles) != self.tp_size or len(blob) != N.MAILBOX_HANDLE_BYTES * self.tp_size:
            raise ConfigError("tensor parallel: one 64-byte handle per rank")
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        _check(self.lib.ssd_tp_connect(self.h, buf))

    def close(self):
        if getattr(self, "h", None):
            self.lib.ssd_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def weight_bytes(self, which: int) -> int:
        return int(self.lib.ssd_engine_weight_bytes(self.h, which))

    # ---- decode loops (sim.hpp)
    def run_ar(self, prompt: Sequence[int], target_scheme: SamplingScheme, tokens: int, seed: int) -> RunStats:
        p = _i32(prompt)
        out = np.zeros(tokens, dtype=np.int32)
        st = N.RunStatsC()
        _check(self.lib.ssd_run_ar(self.h, _ptr(p, C.c_int32), len(p), C.byref(target_scheme.c()), tokens, seed,
                                   _ptr(out, C.c_int32), tokens, C.byref(st)))
        return RunStats._from_c(st, out.tolist())

    def run_sd(self, prompt: Sequence[int], cfg: SimConfig) -> RunStats:
        p = _i32(prompt)
        cap = cfg.rounds * (cfg.lookahead + 1)
        out = np.zeros(cap, dtype=np.int32)
        n = C.c_int64()
        st = N.RunStatsC()
        _check(self.lib.ssd_run_sd(self.h, _ptr(p, C.c_int32), len(p), C.byref(cfg.c()), _ptr(out, C.c_int32), cap,
                                   C.byref(n), C.byref(st)))
        return RunStats._from_c(st, out[: n.value].tolist())

    def run_ssd(self, prompt: Sequence[int], cfg: SimConfig, semantics: str = "harness",
                transcript: bool = False) -> RunStats:
        """semantics "harness": sim::run_protocol_harness (sim.cpp:502-601);
        "sequential": sim::run_ssd / run_ssd_batch (sim.cpp:123-250, one
        stream per sequence, the cache built after verify). cfg.batch_size
        sequences (whole-batch stall: any miss delays the round for the
        backup). streams[j] is sequence j's output; outcomes / hits are
        sequence 0's. transcript=True (harness): r.transcript is the JSONL
        round transcript (Transcript::to_jsonl, sim.cpp:489-500), parsed."""
        import json
        p = _i32(prompt)
        b = int(cfg.batch_size)
        cap = cfg.rounds * (cfg.lookahead + 1)
        out = np.zeros(b * cap, dtype=np.int32)
        oc = np.zeros(2 * cfg.rounds, dtype=np.int32)
        hits = np.zeros(cfg.rounds, dtype=np.int32)
        lens = np.zeros(b, dtype=np.int64)
        st = N.RunStatsC()
        opt = N.RunOptionsC()
        opt.semantics = {"harness": N.SEMANTICS_HARNESS, "sequential": N.SEMANTICS_SEQUENTIAL}[semantics]
        tlen = C.c_int64(0)
        tbuf = None
        if transcript:
            tcap = 4096 + cfg.rounds * b * (64 + 16 * (cfg.lookahead + 4)) + 256 * cfg.rounds
            tbuf = C.create_string_buffer(tcap)
            opt.transcript = C.cast(tbuf, C.c_char_p)
            opt.transcript_cap = tcap
            opt.transcript_len = C.pointer(tlen)
        _check(self.lib.ssd_run_ssd_ex(self.h, _ptr(p, C.c_int32), len(p), C.byref(cfg.c()), b, C.byref(opt),
                                       _ptr(out, C.c_int32), cap, _ptr(lens, C.c_int64), _ptr(oc, C.c_int32),
                                       _ptr(hits, C.c_int32), C.byref(st)))
        r = RunStats._from_c(st, out[: int(lens[0])].tolist())
        if transcript:
            if tlen.value >= tcap:
                raise Error("transcript: buffer too small")
            r.transcript = [json.loads(x) for x in tbuf.value.decode().splitlines() if x]
        r.streams = [out[j * cap: j * cap + int(lens[j])].tolist() for j in range(b)]
        r.batch = b
        r.outcomes = oc.reshape(-1, 2)
        r.hits = hits
        return r

    # ---- split processes (sim.cpp:258-601 over NVLink mailboxes; paper_2603_03251_b200/split.py)
    def mailbox_handle(self) -> bytes:
        buf = (C.c_uint8 * N.MAILBOX_HANDLE_BYTES)()
        _check(self.lib.ssd_mailbox_export(self.h, buf))
        return bytes(buf)

    def connect(self, handles: Sequence[bytes], self_index: int):
        """Map the peers' mailboxes; order [verifier, speculator 0, ...]."""
        blob = b"".join(handles)
        if len(blob) != N.MAILBOX_HANDLE_BYTES * len(handles):
            raise ConfigError("mailbox: every handle must be 64 bytes")
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        _check(self.lib.ssd_mailbox_connect(self.h, len(handles), buf, self_index))

    def run_ssd_verifier(self, prompt: Sequence[int], cfg: SimConfig, n_spec: int) -> RunStats:
        """VerifierProcess side of run_protocol_harness (sim.cpp:321-351)."""
        p = _i32(prompt)
        cap = cfg.rounds * (cfg.lookahead + 1)
        out = np.zeros(cap, dtype=np.int32)
        oc = np.zeros(2 * cfg.rounds, dtype=np.int32)
        n = C.c_int64()
        st = N.RunStatsC()
        _check(self.lib.ssd_run_ssd_verifier(self.h, _ptr(p, C.c_int32), len(p), C.byref(cfg.c()), n_spec,
                                             _ptr(out, C.c_int32), cap, C.byref(n), _ptr(oc, C.c_int32),
                                             C.byref(st)))
        r = RunStats._from_c(st, out[:n.value].tolist())
        r.outcomes = oc.reshape(-1, 2)
        return r

    def run_ssd_speculator(self, prompt: Sequence[int], cfg: SimConfig, rank: int, n_spec: int,
                           n_verifiers: int = 1) -> RunStats:
        """DraftProcess side (sim.cpp:376-485) for speculator `rank` of n_spec;
        n_verifiers = ranks of a tensor-parallel verifier."""
        p = _i32(prompt)
        hits = np.zeros(cfg.rounds, dtype=np.int32)
        st = N.RunStatsC()
        _check(self.lib.ssd_run_ssd_speculator(self.h, _ptr(p, C.c_int32), len(p), C.byref(cfg.c()), rank, n_spec,
                                               n_verifiers, _ptr(hits, C.c_int32), C.byref(st)))
        r = RunStats._from_c(st)
        r.hits = hits
        return r

    # ---- single operations (specdec.hpp / cache.hpp / lm.hpp)
    def logits(self, which: int, context: Sequence[int]) -> np.ndarray:
        c = _i32(context)
        out = np.zeros(self.vocab, dtype=np.float32)
        _check(self.lib.ssd_logits(self.h, which, _ptr(c, C.c_int32), len(c), _ptr(out, C.c_float)))
        return out

    def draft_spec(self, context: Sequence[int], lookahead: int, scheme: SamplingScheme, seed: int,
                   with_rows: bool = True) -> Speculation:
        c = _i32(context)
        toks = np.zeros(lookahead, dtype=np.int32)
        rows = np.zeros((lookahead, self.vocab), dtype=np.float32) if with_rows else None
        _check(self.lib.ssd_draft(self.h, _ptr(c, C.c_int32), len(c), lookahead, C.byref(scheme.c()), seed,
                                  _ptr(toks, C.c_int32), _ptr(rows, C.c_float) if with_rows else None))
        return Speculation(toks.tolist(), rows)

    def build_cache(self, context: Sequence[int], spec: Speculation, plan: FanOutPlan, scheme: SamplingScheme,
                    next_lookahead: int, seed: int) -> SpeculationCache:
        c = _i32(context)
        s = _i32(spec.tokens)
        K = len(spec.tokens)
        tot = plan.total()
        keys = np.zeros(2 * max(tot, 1), dtype=np.int32)
        toks = np.zeros(max(tot, 1) * next_lookahead, dtype=np.int32)
        cnt = C.c_int32()
        _check(self.lib.ssd_build_cache(self.h, _ptr(c, C.c_int32), len(c), _ptr(s, C.c_int32), K,
                                        C.byref(plan.c()), C.byref(scheme.c()), next_lookahead, seed,
                                        _ptr(keys, C.c_int32), _ptr(toks, C.c_int32), C.byref(cnt)))
        entries = {}
        for i in range(cnt.value):
            entries[(int(keys[2 * i]), int(keys[2 * i + 1]))] = toks[i * next_lookahead:(i + 1) * next_lookahead].tolist()
        return SpeculationCache(entries, plan.role)

    # ---- the reference's Stream&-taking interface (specdec.hpp / cache.hpp)
    def draft_tokens(self, context: Sequence[int], lookahead: int, scheme: SamplingScheme, rng: Stream,
                     origin: int = PRIMARY) -> Speculation:
        """specdec::draft (specdec.hpp:59-61) with the caller's stream (named
        draft_tokens here: `Engine.draft` is the draft model's shape)."""
        c = _i32(context)
        toks = np.zeros(lookahead, dtype=np.int32)
        rows = np.zeros((lookahead, self.vocab), dtype=np.float32)
        _check(self.lib.ssd_draft_stream(self.h, _ptr(c, C.c_int32), len(c), lookahead, C.byref(scheme.c()),
                                         C.byref(rng.c), _ptr(toks, C.c_int32), _ptr(rows, C.c_float)))
        return Speculation(toks.tolist(), rows, origin)

    def verify(self, context: Sequence[int], spec: Speculation, rng: Stream,
               draft_scheme: Optional[SamplingScheme] = None, target_scheme: Optional[SamplingScheme] = None,
               accept_scale: float = 1.0) -> RoundResult:
        """specdec::verify (specdec.hpp:81-83): target forward over context ||
        spec + the fused decision, with the caller's stream. spec.rows None =
        uniform dists (the FastRandom backup)."""
        ds = draft_scheme or SamplingScheme.standard()
        ts = target_scheme or SamplingScheme.standard(ds.temperature)
        c = _i32(context)
        t = _i32(spec.tokens)
        K = len(t)
        rows = None if spec.rows is None else np.ascontiguousarray(spec.rows, dtype=np.float32)
        acc, bonus = C.c_int32(), C.c_int32()
        em = np.zeros(K + 1, dtype=np.int32)
        _check(self.lib.ssd_verify(self.h, _ptr(c, C.c_int32), len(c), _ptr(t, C.c_int32), K,
                                   None if rows is None else _ptr(rows, C.c_float), C.byref(ds.c()), C.byref(ts.c()),
                                   accept_scale, C.byref(rng.c), C.byref(acc), C.byref(bonus), _ptr(em, C.c_int32)))
        return RoundResult(acc.value, bonus.value, em[: acc.value + 1].tolist())

    def build_cache_stream(self, context: Sequence[int], spec: Speculation, plan: FanOutPlan, scheme: SamplingScheme,
                           next_lookahead: int, rng: Stream, with_rows: bool = True) -> SpeculationCache:
        """cache::build_cache (cache.hpp:149-154) with the caller's stream,
        any next_lookahead, and each entry's draft rows."""
        c = _i32(context)
        s = _i32(spec.tokens)
        tot = plan.total()
        keys = np.zeros(2 * max(tot, 1), dtype=np.int32)
        toks = np.zeros(max(tot, 1) * next_lookahead, dtype=np.int32)
        rows = np.zeros((max(tot, 1), next_lookahead, self.vocab), dtype=np.float32) if with_rows else None
        cnt = C.c_int32()
        _check(self.lib.ssd_build_cache_stream(self.h, _ptr(c, C.c_int32), len(c), _ptr(s, C.c_int32), len(s),
                                               C.byref(plan.c()), C.byref(scheme.c()), next_lookahead, C.byref(rng.c),
                                               _ptr(keys, C.c_int32), _ptr(toks, C.c_int32),
                                               _ptr(rows, C.c_float) if with_rows else None, C.byref(cnt)))
        entries, erows = {}, ({} if with_rows else None)
        for i in range(cnt.value):
            key = (int(keys[2 * i]), int(keys[2 * i + 1]))
            entries[key] = toks[i * next_lookahead:(i + 1) * next_lookahead].tolist()
            if with_rows:
                erows[key] = rows[i]
        return SpeculationCache(entries, plan.role, erows)

    # ---- asynchronous pre-speculation on device buffers
    def prespec_begin(self, d_context, n: int, d_spec, lookahead: int, plan: FanOutPlan, scheme: SamplingScheme,
                      next_lookahead: int, rng: Stream, cuda_stream: int = 0):
        """d_context / d_spec: device pointers (int32); cuda_stream: a
        cudaStream_t handle whose queued work produces them (0 = none)."""
        _check(self.lib.ssd_prespec_begin(self.h, C.c_void_p(int(d_context)), n, C.c_void_p(int(d_spec)), lookahead,
                                          C.byref(plan.c()), C.byref(scheme.c()), next_lookahead, C.byref(rng.c),
                                          C.c_void_p(int(cuda_stream)) if cuda_stream else None))

    def cache_lookup(self, accepted: int, bonus: int) -> int:
        slot = C.c_int32()
        _check(self.lib.ssd_cache_lookup(self.h, accepted, bonus, C.byref(slot)))
        return slot.value

    def cache_keys(self) -> list:
        n = C.c_int32()
        _check(self.lib.ssd_cache_keys(self.h, None, C.byref(n)))
        keys = np.zeros(2 * max(n.value, 1), dtype=np.int32)
        _check(self.lib.ssd_cache_keys(self.h, _ptr(keys, C.c_int32), C.byref(n)))
        return [(int(keys[2 * i]), int(keys[2 * i + 1])) for i in range(n.value)]

    def cache_entry(self, slot: int, next_lookahead: int, with_rows: bool = False):
        toks = np.zeros(next_lookahead, dtype=np.int32)
        rows = np.zeros((next_lookahead, self.vocab), dtype=np.float32) if with_rows else None
        _check(self.lib.ssd_cache_entry(self.h, slot, _ptr(toks, C.c_int32),
                                        _ptr(rows, C.c_float) if with_rows else None))
        return toks.tolist(), rows

    # ---- kernel-level hooks
    def topk_keys(self, rows: np.ndarray, fan_out: Sequence[int], excluded: Sequence[int]) -> np.ndarray:
        rows = np.ascontiguousarray(rows, dtype=np.float32)
        n, V = rows.shape
        f = _i32(fan_out)
        e = _i32(excluded)
        max_f = max(1, int(f.max()))
        keys = np.zeros(n * max_f, dtype=np.int32)
        _check(self.lib.ssd_topk_keys(self.h, _ptr(rows, C.c_float), n, V, _ptr(f, C.c_int32), _ptr(e, C.c_int32),
                                      max_f, _ptr(keys, C.c_int32)))
        return keys.reshape(n, max_f)

    def verify_rows(self, target_rows: np.ndarray, draft_rows: Optional[np.ndarray], tokens: Sequence[int],
                    draft_scheme: SamplingScheme, target_scheme: SamplingScheme, seed: int,
                    accept_scale: float = 1.0):
        t = np.ascontiguousarray(target_rows, dtype=np.float32)
        d = None if draft_rows is None else np.ascontiguousarray(draft_rows, dtype=np.float32)
        tk = _i32(tokens)
        acc, bonus = C.c_int32(), C.c_int32()
        _check(self.lib.ssd_verify_rows(self.h, _ptr(t, C.c_float), None if d is None else _ptr(d, C.c_float),
                                        _ptr(tk, C.c_int32), len(tk), t.shape[1], C.byref(draft_scheme.c()),
                                        C.byref(target_scheme.c()), accept_scale, seed, C.byref(acc), C.byref(bonus)))
        return acc.value, bonus.value

    # ---- paged KV cache (ssd_engine_set_block_table)
    def kv_pages(self, page_tokens: int) -> int:
        """Pages of this engine's main caches (the KvPool size)."""
        n = C.c_int32()
        _check(self.lib.ssd_engine_kv_pages(self.h, page_tokens, C.byref(n)))
        return n.value

    def set_block_table(self, lane: int, pages: Sequence[int], page_tokens: int, cached_tokens: int = 0) -> None:
        p = _i32(pages)
        _check(self.lib.ssd_engine_set_block_table(self.h, lane, _ptr(p, C.c_int32) if len(p) else None, len(p),
                                                   page_tokens, cached_tokens))

    def clear_block_tables(self) -> None:
        _check(self.lib.ssd_engine_clear_block_tables(self.h))

    # ---- B200 knob: disjoint SM sets for the colocated round's two streams
    def sm_partition(self, verifier_sms: int | None = None) -> tuple[int, int]:
        """(verifier SMs, speculator SMs) of the colocated SSD round; with
        verifier_sms set first (0 = both streams share every SM)."""
        v, s = C.c_int32(), C.c_int32()
        _check(self.lib.ssd_engine_sm_partition(self.h, -1 if verifier_sms is None else int(verifier_sms),
                                                C.byref(v), C.byref(s)))
        return v.value, s.value

    def profile_forward(self, which: int, M: int, pos: int, iters: int) -> dict:
        f, g = C.c_double(), C.c_double()
        b, n = C.c_int64(), C.c_int32()
        _check(self.lib.ssd_profile_forward(self.h, which, M, pos, iters, C.byref(f), C.byref(g), C.byref(b),
                                            C.byref(n)))
        return {"ms_forward": f.value, "ms_gemm": g.value, "gemm_bytes": b.value, "gemm_launches": n.value}

    ROUND_SEGMENTS = ("round", "verify_forward", "verify_decision", "extend_forward", "keys_streams",
                      "branch_forwards", "branch_picks", "lookup", "fork_lag")

    def profile_ssd_round(self, prompt: Sequence[int], cfg: SimConfig) -> dict:
        """ms per segment of the colocated SSD round, measured by event nodes
        inside the round graph (ssd_profile_ssd_round)."""
        p = _i32(prompt)
        out = (C.c_double * 9)()
        st = N.RunStatsC()
        _check(self.lib.ssd_profile_ssd_round(self.h, _ptr(p, C.c_int32), len(p), C.byref(cfg.c()), out,
                                              C.byref(st)))
        return {k: float(out[i]) for i, k in enumerate(self.ROUND_SEGMENTS)}

    def read_bw(self, nbytes: int = 4 << 30, iters: int = 10) -> float:
        g = C.c_double()
        _check(self.lib.ssd_bench_read_bw(self.h, nbytes, iters, C.byref(g)))
        return g.value

    def rng_u64(self, seed: int, n: int) -> list:
        out = np.zeros(n, dtype=np.uint64)
        _check(self.lib.ssd_rng_u64(self.h, seed, n, _ptr(out, C.c_uint64)))
        return [int(x) for x in out]

    def weight_bits(self, which: int, layer: int, kind: int, rows, cols) -> np.ndarray:
        r = np.ascontiguousarray(rows, dtype=np.int64)
        c = np.ascontiguousarray(cols, dtype=np.int64)
        out = np.zeros(len(r), dtype=np.uint16)
        _check(self.lib.ssd_weight_bits(self.h, which, layer, kind, _ptr(r, C.c_int64), _ptr(c, C.c_int64), len(r),
                                        _ptr(out, C.c_uint16)))
        return out


class KvPool:
    """Paged KV block manager (csrc/paged.cpp, the paper's
    engine PAPER.md:1000-1002): lookahead reservation, reconciliation after
    verification (finalize + prefix hash, rollback of pages beyond the
    accepted suffix) and a prefix cache with LRU eviction."""

    def __init__(self, n_pages: int, page_tokens: int):
        self.lib = N.load()
        self.h = C.c_void_p()
        _check(self.lib.ssd_kv_pool_create(n_pages, page_tokens, C.byref(self.h)))
        self.n_pages, self.page_tokens = n_pages, page_tokens

    def close(self) -> None:
        if self.h:
            self.lib.ssd_kv_pool_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def admit(self, seq: int, tokens: Sequence[int]) -> int:
        """Returns the number of leading prompt tokens whose KV is cached."""
        t = _i32(tokens)
        cached = C.c_int32()
        _check(self.lib.ssd_kv_seq_admit(self.h, seq, _ptr(t, C.c_int32), len(t), C.byref(cached)))
        return cached.value

    def reserve(self, seq: int, lookahead: int) -> None:
        _check(self.lib.ssd_kv_seq_reserve(self.h, seq, lookahead))

    def commit(self, seq: int, accepted: Sequence[int]) -> int:
        """Append the accepted tokens; returns the pages rolled back."""
        t = _i32(accepted)
        rel = C.c_int32()
        _check(self.lib.ssd_kv_seq_commit(self.h, seq, _ptr(t, C.c_int32) if len(t) else None, len(t),
                                          C.byref(rel)))
        return rel.value

    def release(self, seq: int) -> None:
        _check(self.lib.ssd_kv_seq_release(self.h, seq))

    def table(self, seq: int) -> tuple:
        """(block table, committed tokens)."""
        n, ntok = C.c_int32(), C.c_int32()
        _check(self.lib.ssd_kv_seq_table(self.h, seq, None, 0, C.byref(n), C.byref(ntok)))
        out = np.zeros(max(n.value, 1), dtype=np.int32)
        _check(self.lib.ssd_kv_seq_table(self.h, seq, _ptr(out, C.c_int32), len(out), C.byref(n), C.byref(ntok)))
        return out[: n.value].tolist(), ntok.value

    def stats(self) -> dict:
        st = N.KvStats()
        _check(self.lib.ssd_kv_pool_stats(self.h, C.byref(st)))
        return {f: getattr(st, f) for f, _ in N.KvStats._fields_}

    def refs(self) -> list:
        out = np.zeros(self.n_pages, dtype=np.int32)
        _check(self.lib.ssd_kv_page_refs(self.h, _ptr(out, C.c_int32), self.n_pages))
        return out.tolist()
