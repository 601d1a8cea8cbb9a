"""rdx_gemm call builder shared by the GEMM probe scripts."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_15013_b200 import _native  # noqa: E402


def gemm(a, w, epi, out, bn=0, **kw):
    args = _native.GemmArgs()
    args.a, args.b = a.data_ptr(), w.data_ptr()
    args.m, args.n, args.k = a.shape[0], w.shape[0], w.shape[1]
    args.lda, args.ldb = a.stride(0), w.stride(0)
    args.epi, args.block_n = epi, bn
    args.out, args.ldo = out.data_ptr(), out.stride(0)
    for k, v in kw.items():
        setattr(args, k, v)
    lib = _native.lib()
    st = _native.stream_handle()
    return lambda: _native.check(lib.rdx_gemm(args, st), "rdx_gemm")
