"""Library sm_100 attention on the C2 / C4 shapes, as the bar for rdx_attention.

  python scripts/attn_lib_bench.py [c2|c4]

Times flashinfer's ragged prefill (backends cutlass = the sm100 FMHA, cudnn,
fa2) and torch SDPA (cuDNN / flash backends on a padded dense batch) on the
suffix-query shape (Q = compact suffix rows, cu_seqlens_q = cu_q; K/V = the
full sequences, materialised in the original layout) and on the plain shape
(no dedup), beside rdx_attention.  Library code is measurement-only here; no
product path imports it.
"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_15013_b200 import _native, build_plan  # noqa: E402
from paper_2601_15013_b200.plan import host_plan_cu_q  # noqa: E402
from paper_2601_15013_b200.workloads import RerankSpec, long_prefix_batch, msmarco_rerank_batch  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
if cfg == "c2":
    b, H, KV, hd = msmarco_rerank_batch(RerankSpec()), 16, 8, 128
else:
    b, H, KV, hd = long_prefix_batch(seed=0), 32, 8, 128
plan = build_plan(b)
cu = b.cu_seqlens
cu_q = host_plan_cu_q(plan, cu)
m, n, B = plan.n_compact, b.num_tokens, b.num_sequences
lens = np.diff(cu).astype(np.float64)
lcp = lens - np.diff(cu_q)
pairs_suffix = float(np.sum(lens * (lens + 1) / 2 - lcp * (lcp + 1) / 2))
pairs_full = float(np.sum(lens * (lens + 1) / 2))
g = torch.Generator(device="cuda").manual_seed(0)
qkv = torch.randn(m, (H + 2 * KV) * hd, device="cuda", generator=g).to(torch.bfloat16)
sc = torch.from_numpy(np.array(plan.scatter_indices).astype(np.int64)).cuda()
qkv_full = qkv[sc].contiguous()
q_c = qkv[:, :H * hd].reshape(m, H, hd).contiguous()
q_f = qkv_full[:, :H * hd].reshape(n, H, hd).contiguous()
k_f = qkv_full[:, H * hd:(H + KV) * hd].reshape(n, KV, hd).contiguous()
v_f = qkv_full[:, (H + KV) * hd:].reshape(n, KV, hd).contiguous()
cu_t = torch.tensor(cu, dtype=torch.int32, device="cuda")
cuq_t = torch.tensor(cu_q, dtype=torch.int32, device="cuda")


def t(fn, it=20):
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


def report(name, us, pairs):
    print(f"{cfg} {name:38s} {us:9.1f} us  {4 * H * hd * pairs / (us * 1e-6) / 1e12:7.0f} TF/s", flush=True)


# ours
lib = _native.lib()
scatter32 = torch.from_numpy(np.array(plan.scatter_indices).view(np.int32)).cuda()
out = torch.empty(m, H * hd, dtype=torch.bfloat16, device="cuda")
out_full = torch.empty(n, H * hd, dtype=torch.bfloat16, device="cuda")
maxq, maxk = int(np.diff(cu_q).max()), int(np.diff(cu).max())
st = torch.cuda.current_stream().cuda_stream
report("rdx_attention suffix", t(lambda: lib.rdx_attention(
    qkv.data_ptr(), qkv.stride(0), m, scatter32.data_ptr(), cu_t.data_ptr(), cuq_t.data_ptr(), B, maxq, maxk, H, KV,
    hd, 1 / math.sqrt(hd), out.data_ptr(), out.stride(0), st)), pairs_suffix)
report("rdx_attention plain", t(lambda: lib.rdx_attention(
    qkv_full.data_ptr(), qkv_full.stride(0), n, None, cu_t.data_ptr(), cu_t.data_ptr(), B, maxk, maxk, H, KV,
    hd, 1 / math.sqrt(hd), out_full.data_ptr(), out_full.stride(0), st)), pairs_full)
ref_suffix = out.clone()

try:
    import flashinfer

    ws = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for backend in ("cutlass", "cudnn", "fa2", "auto"):
        for shape, qo, q, pairs in (("suffix", cuq_t, q_c, pairs_suffix), ("plain", cu_t, q_f, pairs_full)):
            try:
                w = flashinfer.BatchPrefillWithRaggedKVCacheWrapper(ws, "NHD", backend=backend)
                w.plan(qo, cu_t, H, KV, hd, causal=True, q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
                o = w.run(q, k_f, v_f)
                us = t(lambda: w.run(q, k_f, v_f))
                report(f"flashinfer ragged [{backend}] {shape}", us, pairs)
                if shape == "suffix":
                    err = (o.reshape(m, -1).float() - ref_suffix.float()).abs().max().item()
                    print(f"   max|diff| vs rdx suffix: {err:.3e}", flush=True)
            except Exception as e:  # noqa: BLE001
                print(f"{cfg} flashinfer [{backend}] {shape}: unavailable ({type(e).__name__}: {str(e)[:160]})",
                      flush=True)
except ImportError as e:
    print("flashinfer import failed", e)

# torch SDPA on a padded dense batch (plain shape only; padding inflates work, FLOPs counted unpadded)
L = maxk
qd = torch.zeros(B, H, L, hd, dtype=torch.bfloat16, device="cuda")
kd = torch.zeros(B, KV, L, hd, dtype=torch.bfloat16, device="cuda")
vd = torch.zeros_like(kd)
for s in range(B):
    lo, hi = int(cu[s]), int(cu[s + 1])
    qd[s, :, :hi - lo] = q_f[lo:hi].transpose(0, 1)
    kd[s, :, :hi - lo] = k_f[lo:hi].transpose(0, 1)
    vd[s, :, :hi - lo] = v_f[lo:hi].transpose(0, 1)
kd_r = kd.repeat_interleave(H // KV, dim=1)
vd_r = vd.repeat_interleave(H // KV, dim=1)
from torch.nn.attention import SDPBackend, sdpa_kernel  # noqa: E402

for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION):
    try:
        with sdpa_kernel([be]):
            fn = lambda: torch.nn.functional.scaled_dot_product_attention(qd, kd_r, vd_r, is_causal=True)  # noqa
            fn()
            report(f"torch sdpa [{be.name}] padded plain", t(fn), pairs_full)
    except Exception as e:  # noqa: BLE001
        print(f"{cfg} sdpa {be.name}: unavailable ({type(e).__name__}: {str(e)[:160]})", flush=True)
