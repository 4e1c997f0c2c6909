"""tcgen05.mma rate at the GEMM's shapes (M=128 x N, K-major SW128 smem
operands): cycles per 32 KB weight unit (8 MMAs), and the completion latency."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_03251_b200 as P  # noqa: E402

lib = P._native.load()
import torch  # noqa: E402,F401  (context)
torch.cuda.init()
out = (ctypes.c_ulonglong * 2)()
for np_ in (16, 32, 64, 128, 256):
    for iters in (1, 64):
        rc = lib.ssd_debug_mma_rate(np_, iters, out)
        print(f"N={np_:3d} units={iters:3d}: {out[0] / iters:9.1f} cycles/unit ({out[0] / iters / 1.965e3:6.3f} us @1.965GHz), "
              f"final wait {out[1]} cycles rc={rc}", flush=True)
