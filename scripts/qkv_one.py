"""Three launches of one C2 QKV-shaped GEMM variant (for ncu -s 2 -c 1): VARIANT=store|qkv|qkvb, M env."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_15013_b200 import _native  # noqa: E402
from scripts.gemm_epi_bench_lib import gemm  # noqa: E402

M = int(os.environ.get("M", "6912"))
V = os.environ.get("VARIANT", "qkvb")
bf = torch.bfloat16
d, hd, H, KV = 1024, 128, 16, 8
a = torch.randn(M, d, device="cuda").to(bf)
w = (torch.randn((H + 2 * KV) * hd, d, device="cuda") * 0.05).to(bf)
out = torch.empty(M, (H + 2 * KV) * hd, dtype=bf, device="cuda")
qn = torch.ones(hd, device="cuda")
rope = torch.randn(-(-M // 32) * 32 * hd, device="cuda")
if V == "store":
    fn = gemm(a, w, _native.EPI_STORE_BF16, out)
elif V == "pos":
    pos = torch.randint(0, 2048, (M,), device="cuda", dtype=torch.int32)
    fn = gemm(a, w, _native.EPI_QKV, out, q_norm_w=qn.data_ptr(), k_norm_w=qn.data_ptr(), rope_pos=pos.data_ptr(),
              rope_theta=1e6, head_dim=hd, q_heads=H, kv_heads=KV, eps=1e-6)
else:
    fn = gemm(a, w, _native.EPI_QKV, out, q_norm_w=qn.data_ptr(), k_norm_w=qn.data_ptr(), rope_table=rope.data_ptr(),
              rope_blocked=int(V == "qkvb"), head_dim=hd, q_heads=H, kv_heads=KV, eps=1e-6)
for _ in range(3):
    fn()
torch.cuda.synchronize()
