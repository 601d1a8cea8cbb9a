"""Scratch probe: FA2 varlen vs flashinfer fmha_varlen (CUTLASS sm100) on the C2 suffix-attention shapes."""
import time, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_15013_b200.workloads import RerankSpec, msmarco_rerank_batch
from paper_2601_15013_b200 import build_plan
b = msmarco_rerank_batch(RerankSpec())
plan = build_plan(b)
from paper_2601_15013_b200.plan import host_plan_cu_q
cu = b.cu_seqlens; cu_q = host_plan_cu_q(plan, cu)
m, n = plan.n_compact, b.num_tokens
H, KV, hd = 16, 8, 128
q = torch.randn(m, H, hd, device="cuda", dtype=torch.bfloat16)
k = torch.randn(n, KV, hd, device="cuda", dtype=torch.bfloat16)
v = torch.randn(n, KV, hd, device="cuda", dtype=torch.bfloat16)
cuq = torch.tensor(cu_q, dtype=torch.int32, device="cuda"); cuk = torch.tensor(cu, dtype=torch.int32, device="cuda")
maxq = int(np.diff(cu_q).max()); maxk = int(np.diff(cu).max())
from flash_attn import flash_attn_varlen_func
def t(fn, it=50):
    for _ in range(5): fn()
    torch.cuda.synchronize(); s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it): fn()
    e.record(); e.synchronize(); return s.elapsed_time(e)/it*1e3
o1 = flash_attn_varlen_func(q, k, v, cuq, cuk, maxq, maxk, causal=True)
print("fa2 us", t(lambda: flash_attn_varlen_func(q, k, v, cuq, cuk, maxq, maxk, causal=True)), flush=True)
t0=time.time()
try:
    import flashinfer
    from flashinfer.prefill import fmha_varlen
    o2 = fmha_varlen(q, k, v, cuq, cuk, causal=True, max_qo_len=maxq)
    torch.cuda.synchronize()
    print("flashinfer first call (jit) s", time.time()-t0, flush=True)
    print("max diff", (o1.float()-o2.float()).abs().max().item(), flush=True)
    print("fi us", t(lambda: fmha_varlen(q, k, v, cuq, cuk, causal=True, max_qo_len=maxq)), flush=True)
except Exception as ex:
    import traceback; traceback.print_exc()
    print("flashinfer failed", ex, time.time()-t0)
