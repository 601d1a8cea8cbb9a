"""Interleaved A/B of GEMM tile shapes (rdx_gemm_debug_shape) for every C2/C3/C4 GEMM; median us per shape."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_15013_b200 import _native  # noqa: E402
from paper_2601_15013_b200.model import SWIGLU_UNIT  # noqa: E402
from scripts.gemm_epi_bench_lib import gemm  # noqa: E402

CONFIGS = {"c2": (7024, 1024, 3072, 16, 8), "c2nd": (11056, 1024, 3072, 16, 8), "c3": (28168, 2560, 9728, 32, 8),
           "c4": (34816, 4096, 12288, 32, 8)}
SHAPES = [(0, 0), (2, 256), (2, 128), (1, 256), (1, 128)]
bf = torch.bfloat16
hd = 128
lib = _native.lib()
only = sys.argv[1:] or list(CONFIGS)


def t(fn, it):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / it * 1e3


for name in only:
    M, d, di, H, KV = CONFIGS[name]
    di_pad = -(-di // SWIGLU_UNIT) * SWIGLU_UNIT
    a = torch.randn(M, max(d, di_pad, H * hd), device="cuda").to(bf)
    wqkv = (torch.randn((H + 2 * KV) * hd, d, device="cuda") * 0.05).to(bf)
    qkv = torch.empty(M, (H + 2 * KV) * hd, dtype=bf, device="cuda")
    qn = torch.ones(hd, device="cuda")
    pos = torch.randint(0, 2048, (M,), device="cuda", dtype=torch.int32)
    wgu = (torch.randn(2 * di_pad, d, device="cuda") * 0.05).to(bf)
    act = torch.empty(M, di_pad, dtype=bf, device="cuda")
    wo = (torch.randn(d, H * hd, device="cuda") * 0.05).to(bf)
    wd = (torch.randn(d, di_pad, device="cuda") * 0.05).to(bf)
    h = torch.zeros(M, d, device="cuda")
    ad, ah, ai = a[:, :d], a[:, :H * hd], a[:, :di_pad]
    kinds = {
        "qkv": lambda: gemm(ad, wqkv, _native.EPI_QKV, qkv, q_norm_w=qn.data_ptr(), k_norm_w=qn.data_ptr(),
                            rope_pos=pos.data_ptr(), rope_theta=1e6, head_dim=hd, q_heads=H, kv_heads=KV, eps=1e-6),
        "gate_up": lambda: gemm(ad, wgu, _native.EPI_SWIGLU, act),
        "o_proj": lambda: gemm(ah, wo, _native.EPI_RESID_F32, h),
        "down": lambda: gemm(ai, wd, _native.EPI_RESID_F32, h),
    }
    it = 10 if M < 20000 else 3
    for kind, mk in kinds.items():
        res = {sh: [] for sh in SHAPES}
        fns = {}
        for sh in SHAPES:
            lib.rdx_gemm_debug_shape(*sh)
            fns[sh] = mk()  # args struct built now; shape is read at launch time
        for sh in SHAPES:
            lib.rdx_gemm_debug_shape(*sh)
            t(fns[sh], 2)
        for _ in range(5):
            for sh in SHAPES:
                lib.rdx_gemm_debug_shape(*sh)
                res[sh].append(t(fns[sh], it))
        lib.rdx_gemm_debug_shape(0, 0)
        med = {sh: statistics.median(v) for sh, v in res.items()}
        best = min((v, sh) for sh, v in med.items() if sh != (0, 0))
        print(f"{name} {kind:8s} auto {med[(0, 0)]:8.1f} | " + "  ".join(f"{sh[0]},{sh[1]}: {med[sh]:8.1f}" for sh in SHAPES[1:])
              + f"   best {best[1]} {'(auto ok)' if med[(0, 0)] <= best[0] * 1.01 else '(AUTO LOSES %.1f%%)' % (100 * (med[(0, 0)] / best[0] - 1))}",
              flush=True)
