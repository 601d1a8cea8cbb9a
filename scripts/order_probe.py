"""Tile order A/B on the residual GEMMs (C3/C4 shapes): n-major (default) vs row-block-major
(what done_ctr selects), interleaved, median us."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_15013_b200 import _native  # noqa: E402

lib = _native.lib()
st = _native.stream_handle()
bf = torch.bfloat16
for name, M, d, K in (("c3 o_proj", 28168, 2560, 4096), ("c3 down", 28168, 2560, 9728),
                      ("c4 o_proj", 34816, 4096, 4096), ("c4 down", 34816, 4096, 12288), ("c2 down", 7024, 1024, 3072)):
    a = torch.randn(M, K, device="cuda").to(bf)
    w = (torch.randn(d, K, device="cuda") * 0.05).to(bf)
    h = torch.zeros(M, d, device="cuda")
    ctr = torch.zeros(-(-M // 32), dtype=torch.int32, device="cuda")

    def run(mm):
        args = _native.GemmArgs()
        args.a, args.b, args.m, args.n, args.k = a.data_ptr(), w.data_ptr(), M, d, K
        args.lda, args.ldb, args.epi, args.out, args.ldo = K, K, _native.EPI_RESID_F32, h.data_ptr(), d
        if mm:
            args.done_ctr = ctr.data_ptr()
        _native.check(lib.rdx_gemm(args, st), "gemm")

    res = {False: [], True: []}
    for _ in range(5):
        for mm in (False, True):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(3):
                run(mm)
            e.record()
            e.synchronize()
            res[mm].append(s.elapsed_time(e) / 3 * 1e3)
    print(f"{name}: n-major {statistics.median(res[False]):.1f} us   row-block-major {statistics.median(res[True]):.1f} us",
          flush=True)
