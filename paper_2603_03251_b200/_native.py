"""ctypes declarations of include/ssd_b200.h (the C-ABI). Loading fails loudly
when the in-tree libssd_b200.so is missing: there is no fallback path."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SSD_B200_LIB", os.path.join(HERE, "libssd_b200.so"))
MAX_LOOKAHEAD = 16
MAILBOX_HANDLE_BYTES = 64
ROLE_COLOCATED, ROLE_VERIFIER, ROLE_SPECULATOR = 0, 1, 2

# ---------------------------------------------------------------- structs


class ModelShape(C.Structure):
    _fields_ = [("vocab", C.c_int32), ("d_model", C.c_int32), ("n_layers", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn", C.c_int32), ("tied", C.c_int32),
                ("max_ctx", C.c_int32), ("rope_theta", C.c_double), ("norm_eps", C.c_float)]


class PairParams(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("embed_scale", C.c_float), ("shared_mlp_scale", C.c_float),
                ("block_out_scale", C.c_float), ("target_private_embed", C.c_float),
                ("target_private_head", C.c_float), ("draft_gain_mix", C.c_float), ("logit_scale", C.c_float)]


class Scheme(C.Structure):
    _fields_ = [("kind", C.c_int32), ("fan_out", C.c_int32), ("temperature", C.c_double), ("downweight", C.c_double)]


class Plan(C.Structure):
    _fields_ = [("lookahead", C.c_int32), ("role", C.c_int32), ("budget", C.c_int32),
                ("fan_out", C.c_int32 * (MAX_LOOKAHEAD + 1))]


class SimConfigC(C.Structure):
    _fields_ = [("lookahead", C.c_int32), ("scheme", Scheme), ("target_scheme", Scheme), ("primary_plan", Plan),
                ("backup_plan", Plan), ("backup_kind", C.c_int32), ("primary_time", C.c_double),
                ("backup_time", C.c_double), ("rounds", C.c_int64), ("seed", C.c_uint64),
                ("accept_scale", C.c_double)]


class RunStatsC(C.Structure):
    _fields_ = [("rounds", C.c_int64), ("tokens", C.c_int64), ("virtual_time", C.c_double),
                ("primary_origin_lookups", C.c_int64), ("primary_origin_hits", C.c_int64),
                ("backup_origin_lookups", C.c_int64), ("backup_origin_hits", C.c_int64),
                ("hit_rounds", C.c_int64), ("miss_rounds", C.c_int64), ("initial_rounds", C.c_int64),
                ("hit_round_tokens", C.c_int64), ("miss_round_tokens", C.c_int64), ("accepted_sum", C.c_double),
                ("device_ms", C.c_double), ("kernel_launches", C.c_int64)]


SEMANTICS_HARNESS, SEMANTICS_SEQUENTIAL = 0, 1


class RngStream(C.Structure):
    """ssd_rng_stream: the mt19937_64 state of rng::Stream (rng.hpp:29-48)."""
    _fields_ = [("state", C.c_uint64 * 312), ("index", C.c_int32), ("reserved_", C.c_int32)]


class RunOptionsC(C.Structure):
    _fields_ = [("semantics", C.c_int32), ("transcript", C.c_char_p), ("transcript_cap", C.c_int64),
                ("transcript_len", C.POINTER(C.c_int64))]


class KvStats(C.Structure):
    _fields_ = [("n_pages", C.c_int32), ("free_pages", C.c_int32), ("used_pages", C.c_int32),
                ("cached_pages", C.c_int32), ("cached_evictable", C.c_int32), ("sequences", C.c_int32),
                ("allocated", C.c_int64), ("evictions", C.c_int64), ("finalized", C.c_int64),
                ("prefix_hit_pages", C.c_int64), ("prefix_miss_pages", C.c_int64), ("reserved_pages", C.c_int64),
                ("rolled_back_pages", C.c_int64)]


P = C.POINTER
i32p, i64p, u64p, f32p, u16p = P(C.c_int32), P(C.c_int64), P(C.c_uint64), P(C.c_float), P(C.c_uint16)
EngineP = C.c_void_p

# name -> (restype, argtypes); every symbol declared in include/ssd_b200.h
SIGNATURES = {
    "ssd_last_error": (C.c_char_p, []),
    "ssd_abi_version": (C.c_int, []),
    "ssd_geometric_fanout": (C.c_int, [C.c_double, C.c_double, C.c_int32, C.c_int32, C.c_int32, P(Plan)]),
    "ssd_uniform_fanout": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, P(Plan)]),
    "ssd_conditional_hit_rate": (C.c_double, [P(Plan), C.c_double, C.c_double]),
    "ssd_speedup_batch": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                    P(C.c_double)]),
    "ssd_fit_powerlaw": (C.c_int, [P(C.c_double), P(C.c_double), C.c_int32, P(C.c_double), P(C.c_double),
                                   P(C.c_double)]),
    "ssd_critical_batch": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double, P(C.c_double)]),
    "ssd_engine_create": (C.c_int, [P(ModelShape), P(ModelShape), P(PairParams), C.c_int32, C.c_int32, C.c_int32,
                                    P(EngineP)]),
    "ssd_engine_create_role": (C.c_int, [P(ModelShape), P(ModelShape), P(PairParams), C.c_int32, C.c_int32,
                                         C.c_int32, C.c_int32, P(EngineP)]),
    "ssd_engine_create_tp": (C.c_int, [P(ModelShape), P(ModelShape), P(PairParams), C.c_int32, C.c_int32, C.c_int32,
                                       C.c_int32, C.c_int32, C.c_int32, P(EngineP)]),
    "ssd_engine_create_batch": (C.c_int, [P(ModelShape), P(ModelShape), P(PairParams), C.c_int32, C.c_int32,
                                          C.c_int32, C.c_int32, P(EngineP)]),
    "ssd_engine_destroy": (C.c_int, [EngineP]),
    "ssd_tp_export": (C.c_int, [EngineP, P(C.c_uint8)]),
    "ssd_tp_connect": (C.c_int, [EngineP, P(C.c_uint8)]),
    "ssd_mailbox_export": (C.c_int, [EngineP, P(C.c_uint8)]),
    "ssd_mailbox_connect": (C.c_int, [EngineP, C.c_int32, P(C.c_uint8), C.c_int32]),
    "ssd_run_ssd_verifier": (C.c_int, [EngineP, i32p, C.c_int32, P(SimConfigC), C.c_int32, i32p, C.c_int64, i64p,
                                       i32p, P(RunStatsC)]),
    "ssd_run_ssd_speculator": (C.c_int, [EngineP, i32p, C.c_int32, P(SimConfigC), C.c_int32, C.c_int32, C.c_int32,
                                         i32p, P(RunStatsC)]),
    "ssd_engine_weight_bytes": (C.c_int64, [EngineP, C.c_int32]),
    "ssd_run_ar": (C.c_int, [EngineP, i32p, C.c_int32, P(Scheme), C.c_int64, C.c_uint64, i32p, C.c_int64,
                             P(RunStatsC)]),
    "ssd_run_sd": (C.c_int, [EngineP, i32p, C.c_int32, P(SimConfigC), i32p, C.c_int64, i64p, P(RunStatsC)]),
    "ssd_run_ssd": (C.c_int, [EngineP, i32p, C.c_int32, P(SimConfigC), i32p, C.c_int64, i64p, i32p, i32p,
                              P(RunStatsC)]),
    "ssd_run_ssd_ex": (C.c_int, [EngineP, i32p, C.c_int32, P(SimConfigC), C.c_int32, P(RunOptionsC), i32p, C.c_int64,
                                 i64p, i32p, i32p, P(RunStatsC)]),
    "ssd_run_ssd_batch": (C.c_int, [EngineP, i32p, C.c_int32, P(SimConfigC), C.c_int32, i32p, C.c_int64, i64p, i32p,
                                    i32p, P(RunStatsC)]),
    "ssd_logits": (C.c_int, [EngineP, C.c_int32, i32p, C.c_int32, f32p]),
    "ssd_draft": (C.c_int, [EngineP, i32p, C.c_int32, C.c_int32, P(Scheme), C.c_uint64, i32p, f32p]),
    "ssd_build_cache": (C.c_int, [EngineP, i32p, C.c_int32, i32p, C.c_int32, P(Plan), P(Scheme), C.c_int32,
                                  C.c_uint64, i32p, i32p, i32p]),
    "ssd_topk_keys": (C.c_int, [EngineP, f32p, C.c_int32, C.c_int32, i32p, i32p, C.c_int32, i32p]),
    "ssd_verify_rows": (C.c_int, [EngineP, f32p, f32p, i32p, C.c_int32, C.c_int32, P(Scheme), P(Scheme), C.c_double,
                                  C.c_uint64, i32p, i32p]),
    "ssd_profile_forward": (C.c_int, [EngineP, C.c_int32, C.c_int32, C.c_int32, C.c_int32, P(C.c_double),
                                      P(C.c_double), i64p, i32p]),
    "ssd_bench_read_bw": (C.c_int, [EngineP, C.c_int64, C.c_int32, P(C.c_double)]),
    "ssd_profile_ssd_round": (C.c_int, [EngineP, i32p, C.c_int32, P(SimConfigC), P(C.c_double), P(RunStatsC)]),
    "ssd_rng_stream_seed": (None, [P(RngStream), C.c_uint64]),
    "ssd_rng_stream_next_u64": (C.c_uint64, [P(RngStream)]),
    "ssd_rng_stream_next_uniform": (C.c_double, [P(RngStream)]),
    "ssd_derive_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "ssd_draft_stream": (C.c_int, [EngineP, i32p, C.c_int32, C.c_int32, P(Scheme), P(RngStream), i32p, f32p]),
    "ssd_verify": (C.c_int, [EngineP, i32p, C.c_int32, i32p, C.c_int32, f32p, P(Scheme), P(Scheme), C.c_double,
                             P(RngStream), i32p, i32p, i32p]),
    "ssd_build_cache_stream": (C.c_int, [EngineP, i32p, C.c_int32, i32p, C.c_int32, P(Plan), P(Scheme), C.c_int32,
                                         P(RngStream), i32p, i32p, f32p, i32p]),
    "ssd_prespec_begin": (C.c_int, [EngineP, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, P(Plan), P(Scheme),
                                    C.c_int32, P(RngStream), C.c_void_p]),
    "ssd_cache_lookup": (C.c_int, [EngineP, C.c_int32, C.c_int32, i32p]),
    "ssd_cache_keys": (C.c_int, [EngineP, i32p, i32p]),
    "ssd_cache_entry": (C.c_int, [EngineP, C.c_int32, i32p, f32p]),
    "ssd_rng_u64": (C.c_int, [EngineP, C.c_uint64, C.c_int32, u64p]),
    "ssd_weight_bits": (C.c_int, [EngineP, C.c_int32, C.c_int32, C.c_int32, i64p, i64p, C.c_int32, u16p]),
    # paged KV block manager (csrc/paged.cpp)
    "ssd_kv_pool_create": (C.c_int, [C.c_int32, C.c_int32, P(C.c_void_p)]),
    "ssd_kv_pool_destroy": (None, [C.c_void_p]),
    "ssd_kv_seq_admit": (C.c_int, [C.c_void_p, C.c_int64, i32p, C.c_int32, i32p]),
    "ssd_kv_seq_reserve": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32]),
    "ssd_kv_seq_commit": (C.c_int, [C.c_void_p, C.c_int64, i32p, C.c_int32, i32p]),
    "ssd_kv_seq_release": (C.c_int, [C.c_void_p, C.c_int64]),
    "ssd_kv_seq_table": (C.c_int, [C.c_void_p, C.c_int64, i32p, C.c_int32, i32p, i32p]),
    "ssd_kv_pool_stats": (C.c_int, [C.c_void_p, P(KvStats)]),
    "ssd_kv_page_refs": (C.c_int, [C.c_void_p, i32p, C.c_int32]),
    "ssd_engine_kv_pages": (C.c_int, [EngineP, C.c_int32, i32p]),
    "ssd_engine_sm_partition": (C.c_int, [EngineP, C.c_int32, i32p, i32p]),
    "ssd_engine_set_block_table": (C.c_int, [EngineP, C.c_int32, i32p, C.c_int32, C.c_int32, C.c_int32]),
    "ssd_engine_clear_block_tables": (C.c_int, [EngineP]),
}

_lib = None


def load() -> C.CDLL:
    """Load the in-tree C-ABI library. Raises when it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2603_03251_b200._build` "
                              "(there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib
