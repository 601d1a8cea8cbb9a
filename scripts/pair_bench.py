"""rdx_gemm_pair (one launch) vs two rdx_gemm launches at the C2 MLP shape: CUDA-event time.
python scripts/pair_bench.py [m d di]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_15013_b200 import _native  # noqa: E402

m, d, di = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (7024, 1024, 3072)
lib = _native.lib()
st = _native.stream_handle()
bf = torch.bfloat16
x = torch.randn(m, d, device="cuda").to(bf)
wgu = (torch.randn(2 * di, d, device="cuda") * 0.05).to(bf)
wd = (torch.randn(d, di, device="cuda") * 0.05).to(bf)
act = torch.empty(m, di, dtype=bf, device="cuda")
h = torch.zeros(m, d, device="cuda")
slabs = -(-m // 32)
dep = torch.zeros(slabs, dtype=torch.int32, device="cuda")
done = torch.zeros(slabs, dtype=torch.int32, device="cuda")


def args(a, w, epi, out, dn=None):
    g = _native.GemmArgs()
    g.a, g.b, g.m, g.n, g.k = a.data_ptr(), w.data_ptr(), m, w.shape[0], w.shape[1]
    g.lda, g.ldb, g.epi, g.out, g.ldo = a.stride(0), w.stride(0), epi, out.data_ptr(), out.stride(0)
    if dn is not None:
        g.done_ctr = dn.data_ptr()
    return g


g = args(x, wgu, _native.EPI_SWIGLU, act)
dd = args(act, wd, _native.EPI_RESID_F32, h)


def run(pair):
    lib.rdx_gemm_debug_pair(pair)
    dep.zero_()
    _native.check(lib.rdx_gemm_pair(g, dd, dep.data_ptr(), st), "pair")


for p in (1, 0):
    run(p)
torch.cuda.synchronize()
res = {1: [], 0: []}
for _ in range(20):
    for p in (1, 0):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        run(p)
        e.record()
        e.synchronize()
        res[p].append(s.elapsed_time(e) * 1e3)
print({("pair" if k else "two launches"): round(sorted(v)[10], 1) for k, v in res.items()}, "us")
