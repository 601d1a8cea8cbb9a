"""Where the exposed rmsnorm tail goes (stats build: RDX_LIB_VARIANT=nstats): the C2 o_proj GEMM
with slab counters + rdx_rmsnorm_rows_after, %globaltimer landmarks of the GEMM and per-block
entry/exit of the norm, relative to the GEMM's last CTA exit.  NORM_W=4|8: warps per norm block."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("RDX_LIB_VARIANT", "nstats")
from paper_2601_15013_b200 import _native  # noqa: E402

lib = _native.lib()
st = _native.stream_handle()
M, d, K = 7024, 1024, int(os.environ.get("K", "2048"))
bf = torch.bfloat16
a = torch.randn(M, K, device="cuda").to(bf)
w = (torch.randn(d, K, device="cuda") * 0.05).to(bf)
h = torch.zeros(M, d, device="cuda")
ln = torch.ones(d, device="cuda")
hn = torch.empty(M, d, dtype=bf, device="cuda")
ctr = torch.zeros(-(-M // 32), dtype=torch.int32, device="cuda")
args = _native.GemmArgs()
args.a, args.b, args.m, args.n, args.k = a.data_ptr(), w.data_ptr(), M, d, K
args.lda, args.ldb, args.epi, args.out, args.ldo = K, K, _native.EPI_RESID_F32, h.data_ptr(), d
args.done_ctr = ctr.data_ptr()
W = int(os.environ.get("NORM_W", "8"))  # warps per norm block (rdx_norm_debug_warps)
_native.check(lib.rdx_norm_debug_warps(W), "warps")
nb = min(-(-M // W), 4096)
for it in range(4):
    ctr.zero_()
    torch.cuda.synchronize()
    gt = (ctypes.c_ulonglong * 8)()
    lib.rdx_gemm_debug_stats(gt, 2)  # reset landmarks
    _native.check(lib.rdx_gemm(args, st), "gemm")
    _native.check(lib.rdx_rmsnorm_rows_after(h.data_ptr(), d, M, d, ln.data_ptr(), 1e-6, hn.data_ptr(), d,
                                             ctr.data_ptr(), d, None, st), "norm")
    torch.cuda.synchronize()
    lib.rdx_gemm_debug_stats(gt, 2)
    g = list(gt)
    buf = (ctypes.c_ulonglong * (2 * nb))()
    _native.check(lib.rdx_norm_debug_times(buf, nb), "times")
    t = np.array(list(buf), dtype=np.float64).reshape(nb, 2)
    ex = g[6]  # GEMM last CTA exit
    s_rel, e_rel = (t[:, 0] - ex) / 1e3, (t[:, 1] - ex) / 1e3
    print(f"iter {it}: gemm span {(ex - g[0]) / 1e3:.1f} us (last mma {(g[4] - g[0]) / 1e3:.1f}, epi done "
          f"{(g[5] - g[0]) / 1e3:.1f});  norm blocks started before gemm exit: {(s_rel < 0).sum()}/{nb}; "
          f"start rel exit: min {s_rel.min():.1f} median {np.median(s_rel):.1f} max {s_rel.max():.1f} us; "
          f"end rel exit: median {np.median(e_rel):.1f} p90 {np.percentile(e_rel, 90):.1f} max {e_rel.max():.1f} us",
          flush=True)
