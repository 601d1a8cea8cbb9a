"""GEMM tile raster A/B (rdx_gemm_debug_group_m): every C2/C3/C4 GEMM under group_m in GROUPS,
interleaved, median us (group_m 1000 = legacy column-block-major, 1 = row-block-major)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_15013_b200 import _native  # noqa: E402
from paper_2601_15013_b200.model import SWIGLU_UNIT  # noqa: E402
from scripts.gemm_epi_bench_lib import gemm  # noqa: E402

CONFIGS = {"c2": (7024, 1024, 3072, 16, 8), "c3": (28168, 2560, 9728, 32, 8), "c4": (34816, 4096, 12288, 32, 8)}
GROUPS = [int(x) for x in os.environ.get("GROUPS", "1000,1,2,4,8,16").split(",")]
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
        "qkv": gemm(ad, wqkv, _native.EPI_QKV, qkv, q_norm_w=qn.data_ptr(), k_norm_w=qn.data_ptr(),
                    rope_pos=pos.data_ptr(), rope_theta=1e6, head_dim=hd, q_heads=H, kv_heads=KV, eps=1e-6),
        "gate_up": gemm(ad, wgu, _native.EPI_SWIGLU, act),
        "o_proj": gemm(ah, wo, _native.EPI_RESID_F32, h),
        "down": gemm(ai, wd, _native.EPI_RESID_F32, h),
    }
    it = 5 if M < 20000 else 2
    for kind, fn in kinds.items():
        res = {g: [] for g in GROUPS}
        for g in GROUPS:
            lib.rdx_gemm_debug_group_m(g)
            t(fn, 1)
        for _ in range(5):
            for g in GROUPS:
                lib.rdx_gemm_debug_group_m(g)
                res[g].append(t(fn, it))
        lib.rdx_gemm_debug_group_m(0)
        med = {g: statistics.median(v) for g, v in res.items()}
        best = min(med, key=med.get)
        print(f"{name} {kind:8s} " + "  ".join(f"g{g}: {med[g]:8.1f}" for g in GROUPS) + f"   best g{best}", flush=True)
