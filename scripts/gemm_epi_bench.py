"""Time rdx_gemm at the C2 (Qwen3-0.6B, M=7024) shapes per epilogue: QKV vs plain store, etc."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_15013_b200 import _native  # noqa: E402
from scripts.gemm_epi_bench_lib import gemm  # noqa: E402

M = int(os.environ.get("M", "7024"))


def t(fn, it=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / it * 1e3


bf = torch.bfloat16
d, hd, H, KV, di = 1024, 128, 16, 8, 3072
a = torch.randn(M, d, device="cuda").to(bf)
wqkv = (torch.randn((H + 2 * KV) * hd, d, device="cuda") * 0.05).to(bf)
qkv = torch.empty(M, (H + 2 * KV) * hd, dtype=bf, device="cuda")
qn = torch.ones(hd, device="cuda")
rope = torch.randn(M, hd // 2, 2, device="cuda")
fl = 2 * M * wqkv.shape[0] * d
for bn in (0,):
    us_store = t(gemm(a, wqkv, _native.EPI_STORE_BF16, qkv, bn))
    us_qkv = t(gemm(a, wqkv, _native.EPI_QKV, qkv, bn, q_norm_w=qn.data_ptr(), k_norm_w=qn.data_ptr(),
                    rope_table=rope.data_ptr(), head_dim=hd, q_heads=H, kv_heads=KV, eps=1e-6))
    rope_bl = torch.randn(-(-M // 32) * 32 * hd, device="cuda")
    us_bl = t(gemm(a, wqkv, _native.EPI_QKV, qkv, bn, q_norm_w=qn.data_ptr(), k_norm_w=qn.data_ptr(),
                   rope_table=rope_bl.data_ptr(), rope_blocked=1, head_dim=hd, q_heads=H, kv_heads=KV, eps=1e-6))
    posd = torch.randint(0, 2048, (M,), device="cuda", dtype=torch.int32)
    us_pos = t(gemm(a, wqkv, _native.EPI_QKV, qkv, bn, q_norm_w=qn.data_ptr(), k_norm_w=qn.data_ptr(),
                    rope_pos=posd.data_ptr(), rope_theta=1e6, head_dim=hd, q_heads=H, kv_heads=KV, eps=1e-6))
    print(f"  rope from positions {us_pos:.1f} us ({fl / us_pos / 1e6:.0f} TF/s)", flush=True)
    print(f"qkv shape M={M}: store_bf16 {us_store:.1f} us ({fl / us_store / 1e6:.0f} TF/s)  "
          f"EPI_QKV {us_qkv:.1f} us ({fl / us_qkv / 1e6:.0f} TF/s)  "
          f"blocked rope {us_bl:.1f} us ({fl / us_bl / 1e6:.0f} TF/s)", flush=True)
wgu = (torch.randn(2 * di, d, device="cuda") * 0.05).to(bf)
act = torch.empty(M, di, dtype=bf, device="cuda")
gu = torch.empty(M, 2 * di, dtype=bf, device="cuda")
fl = 2 * M * 2 * di * d
print(f"gate_up: store_bf16 {t(gemm(a, wgu, _native.EPI_STORE_BF16, gu)):.1f} us  "
      f"EPI_SWIGLU {t(gemm(a, wgu, _native.EPI_SWIGLU, act)):.1f} us  ({fl / 1e6:.0f} MFLOP)", flush=True)
wo = (torch.randn(d, H * hd, device="cuda") * 0.05).to(bf)
ao = torch.randn(M, H * hd, device="cuda").to(bf)
h = torch.zeros(M, d, device="cuda")
fl = 2 * M * d * H * hd
us = t(gemm(ao, wo, _native.EPI_RESID_F32, h))
print(f"o_proj: EPI_RESID_F32 {us:.1f} us ({fl / us / 1e6:.0f} TF/s)", flush=True)
wd = (torch.randn(d, di, device="cuda") * 0.05).to(bf)
us = t(gemm(act, wd, _native.EPI_RESID_F32, h))
print(f"down: EPI_RESID_F32 {us:.1f} us ({2 * M * d * di / us / 1e6:.0f} TF/s)", flush=True)
