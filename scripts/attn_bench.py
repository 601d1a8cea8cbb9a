"""Scratch: time rdx_attention vs FA2 on the C2 suffix / plain shapes."""
import math, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_15013_b200 import build_plan, _native
from paper_2601_15013_b200.plan import host_plan_cu_q
from paper_2601_15013_b200.workloads import RerankSpec, msmarco_rerank_batch
b = msmarco_rerank_batch(RerankSpec())
plan = build_plan(b)
cu = b.cu_seqlens; cu_q = host_plan_cu_q(plan, cu)
m, n = plan.n_compact, b.num_tokens
H, KV, hd = 16, 8, 128
qkv = torch.randn(m, (H + 2 * KV) * hd, device="cuda").to(torch.bfloat16)
scatter = torch.from_numpy(np.array(plan.scatter_indices).view(np.int32)).cuda()
cu32 = torch.tensor(cu, dtype=torch.int32, device="cuda"); cuq32 = torch.tensor(cu_q, dtype=torch.int32, device="cuda")
out = torch.empty(m, H * hd, dtype=torch.bfloat16, device="cuda")
maxq = int(np.diff(cu_q).max()); maxk = int(np.diff(cu).max())
lib = _native.lib()
def ours():
    lib.rdx_attention(qkv.data_ptr(), qkv.stride(0), scatter.data_ptr(), cu32.data_ptr(), cuq32.data_ptr(), len(cu)-1, maxq, H, KV, hd, 1/math.sqrt(hd), out.data_ptr(), out.stride(0), torch.cuda.current_stream().cuda_stream)
qkv_full = torch.randn(n, (H + 2 * KV) * hd, device="cuda").to(torch.bfloat16)
out_full = torch.empty(n, H * hd, dtype=torch.bfloat16, device="cuda")
def ours_plain():
    lib.rdx_attention(qkv_full.data_ptr(), qkv_full.stride(0), None, cu32.data_ptr(), cu32.data_ptr(), len(cu)-1, maxk, H, KV, hd, 1/math.sqrt(hd), out_full.data_ptr(), out_full.stride(0), torch.cuda.current_stream().cuda_stream)
from flash_attn import flash_attn_varlen_func
kvf = qkv_full[:, H*hd:]
def fa2():
    flash_attn_varlen_func(qkv[:, :H*hd].view(m, H, hd), kvf[:, :KV*hd].view(n, KV, hd), kvf[:, KV*hd:].view(n, KV, hd), cuq32, cu32, maxq, maxk, causal=True)
def t(fn, it=50):
    for _ in range(5): fn()
    torch.cuda.synchronize(); s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it): fn()
    e.record(); e.synchronize(); return s.elapsed_time(e)/it*1e3
print("ours suffix us", round(t(ours),1), "ours plain us", round(t(ours_plain),1), "fa2 suffix us", round(t(fa2),1), flush=True)
