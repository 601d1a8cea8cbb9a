"""Launch landmarks (gstats build) of rdx_gemm_pair at the C2 MLP shape, and the same
gate|up GEMM alone with the default raster and with row-block-major raster.
RDX_LIB_VARIANT=gstats python scripts/pair_times.py"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("RDX_LIB_VARIANT", "gstats")
import scripts.pair_bench as pb  # noqa: E402  (builds the args)
from paper_2601_15013_b200 import _native  # noqa: E402

lib = _native.lib()
names = ["entry_first", "entry_last", "prologue_done", "first_stage", "last_mma", "epi_done", "exit"]


def landmarks(fn):
    torch.cuda.synchronize()
    st = (ctypes.c_ulonglong * 8)()
    lib.rdx_gemm_debug_stats(st, 2)
    fn()
    torch.cuda.synchronize()
    lib.rdx_gemm_debug_stats(st, 2)
    t = list(st)
    return "  ".join(f"{n}={(t[k] - t[0]) / 1e3:.1f}" for k, n in enumerate(names))


print("pair        :", landmarks(lambda: pb.run(1)))
lib.rdx_gemm_debug_pair(1)
print("gate_up     :", landmarks(lambda: _native.check(lib.rdx_gemm(pb.g, pb.st), "g")))
prev = lib.rdx_gemm_debug_group_m(1)
print("gate_up rbm :", landmarks(lambda: _native.check(lib.rdx_gemm(pb.g, pb.st), "g")))
lib.rdx_gemm_debug_group_m(prev)
print("down        :", landmarks(lambda: _native.check(lib.rdx_gemm(pb.dd, pb.st), "d")))

st = (ctypes.c_ulonglong * 8)()
lib.rdx_gemm_debug_stats(None, 1)
pb.run(1)
torch.cuda.synchronize()
lib.rdx_gemm_debug_stats(st, 0)
v = list(st)
print(f"pair: producer dep-wait cycles total {v[6]} over {v[7]} tiles (avg {v[6] / max(v[7], 1):.0f});"
      f" MMA loop {v[2] / 74:.0f} cycles/pair, tempty wait {v[0] / 74:.0f}, full wait {v[1] / 74:.0f}")
