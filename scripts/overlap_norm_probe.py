"""C2 o_proj / down shapes: RESID_F32 GEMM with vs without the slab counters, and GEMM + rmsnorm
stream-ordered vs GEMM(counters) + rdx_rmsnorm_rows_after (programmatic dependent)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_15013_b200 import _native  # noqa: E402

lib = _native.lib()
st = _native.stream_handle()
M, d = 7024, 1024
bf = torch.bfloat16


def t(fn, it=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / it * 1e3


for K in (2048, 3072):
    a = torch.randn(M, K, device="cuda").to(bf)
    w = (torch.randn(d, K, device="cuda") * 0.05).to(bf)
    h = torch.zeros(M, d, device="cuda")
    ln = torch.ones(d, device="cuda")
    hn = torch.empty(M, d, dtype=bf, device="cuda")
    ctr = torch.zeros(-(-M // 32), dtype=torch.int32, device="cuda")
    use = [0]

    def gemm(with_ctr):
        args = _native.GemmArgs()
        args.a, args.b, args.m, args.n, args.k = a.data_ptr(), w.data_ptr(), M, d, K
        args.lda, args.ldb, args.epi, args.out, args.ldo = K, K, _native.EPI_RESID_F32, h.data_ptr(), d
        if with_ctr:
            args.done_ctr = ctr.data_ptr()
        _native.check(lib.rdx_gemm(args, st), "gemm")

    def rms():
        _native.check(lib.rdx_rmsnorm_rows(h.data_ptr(), d, None, M, d, ln.data_ptr(), 1e-6, hn.data_ptr(), d, st), "r")

    def rms_after():
        use[0] += 1
        _native.check(lib.rdx_rmsnorm_rows_after(h.data_ptr(), d, M, d, ln.data_ptr(), 1e-6, hn.data_ptr(), d,
                                                 ctr.data_ptr(), use[0] * d, None, st), "ra")

    r = {
        "gemm": t(lambda: gemm(False)),
        "gemm+ctr": t(lambda: gemm(True)),
        "rms": t(rms),
        "gemm;rms": t(lambda: (gemm(False), rms())),
        "gemm+ctr;rms": t(lambda: (gemm(True), rms())),
        "gemm+ctr;rms_after": t(lambda: (gemm(True), rms_after())),
    }
    print(f"K={K}: " + "  ".join(f"{k} {v:.1f}" for k, v in r.items()), flush=True)

# the same pairs captured in a CUDA graph (8 GEMM+norm pairs per graph)
for K in (2048,):
    a = torch.randn(M, K, device="cuda").to(bf)
    w = (torch.randn(d, K, device="cuda") * 0.05).to(bf)
    h = torch.zeros(M, d, device="cuda")
    ln = torch.ones(d, device="cuda")
    hn = torch.empty(M, d, dtype=bf, device="cuda")
    ctr = torch.zeros(-(-M // 32), dtype=torch.int32, device="cuda")

    def body(overlap):
        ctr.zero_()
        for u in range(1, 9):
            args = _native.GemmArgs()
            args.a, args.b, args.m, args.n, args.k = a.data_ptr(), w.data_ptr(), M, d, K
            args.lda, args.ldb, args.epi, args.out, args.ldo = K, K, _native.EPI_RESID_F32, h.data_ptr(), d
            if overlap:
                args.done_ctr = ctr.data_ptr()
            s_ = _native.stream_handle()
            _native.check(lib.rdx_gemm(args, s_), "gemm")
            if overlap:
                _native.check(lib.rdx_rmsnorm_rows_after(h.data_ptr(), d, M, d, ln.data_ptr(), 1e-6, hn.data_ptr(), d,
                                                         ctr.data_ptr(), u * d, None, s_), "ra")
            else:
                _native.check(lib.rdx_rmsnorm_rows(h.data_ptr(), d, None, M, d, ln.data_ptr(), 1e-6, hn.data_ptr(), d,
                                                   s_), "r")

    graphs = {}
    for ov in (False, True):
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            body(ov)
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            body(ov)
        graphs[ov] = g
    res = {False: [], True: []}
    for _ in range(10):
        for ov in (False, True):
            res[ov].append(t(graphs[ov].replay, 5))
    import statistics
    print(f"[RDX_NORM_AFTER_PDL={os.environ.get('RDX_NORM_AFTER_PDL', '1')}] graph of 8 pairs K={K}: stream-ordered {statistics.median(res[False]):.1f} us  "
          f"overlapped {statistics.median(res[True]):.1f} us")
    print("eager of 8 pairs:", f"stream-ordered {t(lambda: body(False), 5):.1f} us  overlapped {t(lambda: body(True), 5):.1f} us")
