"""Build the native engine in-tree: paper_2603_03251_b200/libssd_b200.so
(sm_100a only). Used by __graft_entry__.build() and `python -m
paper_2603_03251_b200._build`."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libssd_b200.so")
SOURCES = ["engine.cu", "plans.cpp", "paged.cpp"]
# every header under csrc/ (a missing entry once left a stale library in place)
DEPS = SOURCES + sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".h", ".hpp")))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-diag-suppress", "177"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in DEPS if os.path.exists(os.path.join(CSRC, f))]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "ssd_b200.h"))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    cmd = [NVCC, *FLAGS, "-o", LIB, *[os.path.join(CSRC, s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True, cwd=CSRC)
    return LIB


def build_variant(name: str, defines: list[str], verbose: bool = False) -> str:
    """A profiling variant of the library (e.g. -DSSD_KTL=1 kernel timeline),
    loaded with SSD_B200_LIB=<path>; never the product build."""
    out = os.path.join(HERE, f"libssd_b200_{name}.so")
    cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-o", out, *[os.path.join(CSRC, s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True, cwd=CSRC)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
