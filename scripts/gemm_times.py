"""Launch landmarks of single GEMM launches (stats build, RDX_LIB_VARIANT=gstats): entry skew,
prologue, first operand stage, last MMA commit, last epilogue store, exit (us from first entry).
VARIANT=pos|store|swiglu|gateup|resid M=7024 python scripts/gemm_times.py"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("RDX_LIB_VARIANT", "gstats")
import scripts.gemm_stats as gs  # noqa: E402  (builds fn for VARIANT, runs once)
from paper_2601_15013_b200 import _native  # noqa: E402

lib = _native.lib()
names = ["entry_first", "entry_last", "prologue_done", "first_stage", "last_mma", "epi_done", "exit"]
res = []
for _ in range(5):
    torch.cuda.synchronize()
    st = (ctypes.c_ulonglong * 8)()
    lib.rdx_gemm_debug_stats(st, 2)  # reset
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    gs.fn()
    e.record()
    torch.cuda.synchronize()
    lib.rdx_gemm_debug_stats(st, 2)
    t = list(st)
    res.append((s.elapsed_time(e) * 1e3, [(t[k] - t[0]) / 1e3 for k in range(7)]))
for ev, t in res[1:]:
    print(f"{gs.V}: event {ev:6.1f} us | " + "  ".join(f"{n}={v:.1f}" for n, v in zip(names, t)))
