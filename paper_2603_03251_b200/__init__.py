"""B200-native Saguaro (speculative speculative decoding) hot path.

The product is the native library libssd_b200.so (include/ssd_b200.h): CUDA
kernels for sm_100a plus the C++ round loops. This package is the thin
Python mirror of the reference's interface used by tests and bench.py.
"""
from .api import (  # noqa: F401
    BACKUP, FAST_RANDOM, PRIMARY, SAME_PRIMARY_JIT, AllZeroError, BudgetTooSmallError, ConfigError, CudaError,
    DegenerateResidualError, DivergentError, Engine, Error, FanOutPlan, InsufficientDataError, KvPool, NoCrossoverError, Pair,
    ProtocolViolationError, RoundResult, RunStats, SamplingScheme, Stream, SimConfig, Speculation, SpeculationCache, TooLargeError,
    UnreachableError, conditional_hit_rate, critical_batch, derive_seed, fit_powerlaw, geometric_fanout, model_shape, saguaro_backup, shape_dict,
    speedup_batch, uniform_fanout)
from .configs import CONFIGS, TINY_DRAFT, TINY_TARGET, LLAMA_1B, LLAMA_8B  # noqa: F401
