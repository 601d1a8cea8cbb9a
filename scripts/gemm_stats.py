"""Role counters of the stats build (RDX_LIB_VARIANT=gstats): one QKV-shaped GEMM variant, per-tile cycles."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_15013_b200 import _native  # noqa: E402
from scripts.gemm_epi_bench_lib import gemm  # noqa: E402

M = int(os.environ.get("M", "6912"))
bf = torch.bfloat16
d, hd, H, KV = 1024, 128, 16, 8
a = torch.randn(M, d, device="cuda").to(bf)
w = (torch.randn((H + 2 * KV) * hd, d, device="cuda") * 0.05).to(bf)
out = torch.empty(M, (H + 2 * KV) * hd, dtype=bf, device="cuda")
qn = torch.ones(hd, device="cuda")
pos = torch.randint(0, 2048, (M,), device="cuda", dtype=torch.int32)
V = os.environ.get("VARIANT", "pos")
if V in ("resid", "residnorm"):  # o_proj shape: K = H * hd, N = d
    ao = torch.randn(M, H * hd, device="cuda").to(bf)
    wo = (torch.randn(d, H * hd, device="cuda") * 0.05).to(bf)
    hres = torch.zeros(M, d, device="cuda")
    hb = torch.empty(M, d, dtype=bf, device="cuda")
    ss = torch.empty(M, d // 64, device="cuda")
    if V == "resid":
        fn = gemm(ao, wo, _native.EPI_RESID_F32, hres)
    else:
        fn = gemm(ao, wo, _native.EPI_RESID_NORM, hres, out_bf16=hb.data_ptr(), ldo_bf16=hb.stride(0),
                  ss_out=ss.data_ptr())
elif V == "store":
    fn = gemm(a, w, _native.EPI_STORE_BF16, out)
elif V == "swiglu":  # QKV-shaped mainloop, half the output columns (gate_up's epilogue)
    fn = gemm(a, w, _native.EPI_SWIGLU, out[:, : w.shape[0] // 2])
elif V == "gateup":  # the real gate_up shape (N = 2 x 3072)
    wgu = (torch.randn(6144, d, device="cuda") * 0.05).to(bf)
    gu = torch.empty(M, 3072, dtype=bf, device="cuda")
    fn = gemm(a, wgu, _native.EPI_SWIGLU, gu)
else:
    fn = gemm(a, w, _native.EPI_QKV, out, q_norm_w=qn.data_ptr(), k_norm_w=qn.data_ptr(), rope_pos=pos.data_ptr(),
          rope_theta=1e6, head_dim=hd, q_heads=H, kv_heads=KV, eps=1e-6)
lib = _native.lib()
fn()
torch.cuda.synchronize()


def main():
    lib.rdx_gemm_debug_stats(None, 1)
    it = 20
    s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s_ev.record()
    for _ in range(it):
        fn()
    e_ev.record()
    torch.cuda.synchronize()
    print(f"{V}: {s_ev.elapsed_time(e_ev) / it * 1e3:.1f} us per launch")
    st = (ctypes.c_ulonglong * 8)()
    _native.check(lib.rdx_gemm_debug_stats(st, 0), "stats")
    st = list(st)
    mma_units = 74 if os.environ.get("RDX_GEMM_SHAPE", "2,256")[0] == "2" else 148
    print(f"M={M}: per MMA warp per launch: tempty wait {st[0] / it / mma_units:.0f}  full wait {st[1] / it / mma_units:.0f}"
          f"  loop {st[2] / it / mma_units:.0f} cycles")
    if st[5]:
      print(f"epilogue per warp-tile: wait {st[3] / st[5]:.0f}  busy {st[4] / st[5]:.0f}  (tiles {st[5] // it})")


if __name__ == "__main__":
    main()
