"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU oracle and to the
compiled reference (oracle/_ref). Imported by tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline legs only; the product never imports this.
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libssdref.so")
REFERENCE_SRC = "/root/reference/proj"


def build(with_ref: bool | None = None) -> None:
    """Compile the oracle (always) and the reference driver (when the
    reference tree is present, i.e. in the build container)."""
    targets = ["all"]
    if with_ref is None:
        with_ref = os.path.isdir(REFERENCE_SRC)
    if with_ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


class _Lib:
    def __init__(self, path: str, call: str, free: str):
        self.lib = ctypes.CDLL(path)
        self._call = getattr(self.lib, call)
        self._call.restype = ctypes.c_void_p
        self._call.argtypes = [ctypes.c_char_p]
        self._free = getattr(self.lib, free)
        self._free.argtypes = [ctypes.c_void_p]

    def call(self, req: dict) -> dict:
        ptr = self._call(json.dumps(req).encode())
        try:
            out = json.loads(ctypes.string_at(ptr).decode())
        finally:
            self._free(ptr)
        return out


_oracle = None
_ref = None


class OracleError(RuntimeError):
    def __init__(self, msg: str, code: int):
        super().__init__(msg)
        self.code = code


def _check(out: dict) -> dict:
    if "error" in out:
        raise OracleError(out["error"], out.get("code", 1))
    return out


def oracle() -> _Lib:
    global _oracle
    if _oracle is None:
        _oracle = _Lib(ORACLE_SO, "oracle_call", "oracle_free")
        lib = _oracle.lib
        lib.oracle_tf_create.restype = ctypes.c_int
        lib.oracle_tf_create.argtypes = [ctypes.c_char_p]
        lib.oracle_tf_destroy.argtypes = [ctypes.c_int]
        lib.oracle_tf_logits.restype = ctypes.c_int
        lib.oracle_tf_logits.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_float)]
        lib.oracle_tf_weight_bits.restype = ctypes.c_int
        lib.oracle_tf_weight_bits.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                              ctypes.POINTER(ctypes.c_long), ctypes.POINTER(ctypes.c_long),
                                              ctypes.c_int, ctypes.POINTER(ctypes.c_ushort)]
        lib.oracle_tf_final_gain.restype = ctypes.c_float
        lib.oracle_tf_final_gain.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def reference() -> _Lib:
    global _ref
    if _ref is None:
        _ref = _Lib(REF_SO, "ref_call", "ref_free")
    return _ref


def oracle_call(req: dict) -> dict:
    return _check(oracle().call(req))


def ref_call(req: dict) -> dict:
    return _check(reference().call(req))


class TfPair:
    """A (target, draft) CPU transformer pair held by the oracle library."""

    def __init__(self, target: dict, draft: dict, pair: dict | None = None, threads: int = 0, accum: str = "f32"):
        """accum "f64": fp64 sums with the same bf16 rounding points — the
        noise-floor reference of the logit parity tests."""
        self.spec = {"target": target, "draft": draft, "pair": pair or {}, "threads": threads, "accum": accum}
        self.handle = oracle().lib.oracle_tf_create(json.dumps(self.spec).encode())
        if self.handle < 0:
            raise OracleError("oracle_tf_create failed", 1)
        self.vocab = target["vocab"]

    def logits(self, which: int, ctx) -> "list[float]":
        import numpy as np
        arr = (ctypes.c_int * len(ctx))(*[int(t) for t in ctx])
        out = np.empty(self.vocab, dtype=np.float32)
        rc = oracle().lib.oracle_tf_logits(self.handle, which, arr, len(ctx),
                                           out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)))
        if rc:
            raise OracleError("oracle_tf_logits failed", 1)
        return out

    def weight_bits(self, which: int, layer: int, kind: int, rows, cols):
        import numpy as np
        n = len(rows)
        r = (ctypes.c_long * n)(*rows)
        c = (ctypes.c_long * n)(*cols)
        out = np.empty(n, dtype=np.uint16)
        rc = oracle().lib.oracle_tf_weight_bits(self.handle, which, layer, kind, r, c, n,
                                                out.ctypes.data_as(ctypes.POINTER(ctypes.c_ushort)))
        if rc:
            raise OracleError("oracle_tf_weight_bits failed", 1)
        return out

    def final_gain(self, which: int, i: int) -> float:
        return oracle().lib.oracle_tf_final_gain(self.handle, which, i)

    def call(self, req: dict) -> dict:
        return oracle_call({**req, "tf_pair": self.handle})

    def close(self):
        if self.handle > 0:
            oracle().lib.oracle_tf_destroy(self.handle)
            self.handle = -1
