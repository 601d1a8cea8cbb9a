"""Interleaved A/B of an rdx_attention debug switch (bk64 | split), same process and inputs, suffix
and plain layouts, plus the max difference between the two outputs and an fp32 reference on a few
sequences.  python scripts/attn_switch_ab.py <bk64|split> [c2|c2lit] [iters]"""
import ctypes
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_15013_b200 import _native, build_plan  # noqa: E402
from paper_2601_15013_b200.plan import host_plan_cu_q  # noqa: E402
from paper_2601_15013_b200.workloads import RerankSpec, msmarco_rerank_batch  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "split"
cfg = sys.argv[2] if len(sys.argv) > 2 else "c2"
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 30
spec = RerankSpec() if cfg == "c2" else RerankSpec(template_len=0, query_len=32, tail_len=0)
b, H, KV, hd = msmarco_rerank_batch(spec), 16, 8, 128
plan = build_plan(b)
cu = b.cu_seqlens
lib = _native.lib()
switch = getattr(lib, f"rdx_attention_debug_{which}")
st = torch.cuda.current_stream().cuda_stream
g = torch.Generator(device="cuda").manual_seed(0)
for layout in ("suffix", "plain"):
    if layout == "suffix":
        cu_q = host_plan_cu_q(plan, cu)
        m = plan.n_compact
        sc = torch.from_numpy(np.array(plan.scatter_indices).view(np.int32)).cuda()
    else:
        cu_q, m, sc = cu, b.num_tokens, None
    qkv = torch.randn(m, (H + 2 * KV) * hd, device="cuda", generator=g).to(torch.bfloat16)
    cu_t = torch.tensor(cu, dtype=torch.int32, device="cuda")
    cuq_t = torch.tensor(cu_q, dtype=torch.int32, device="cuda")
    maxq, maxk = int(np.diff(cu_q).max()), int(np.diff(cu).max())
    outs = {v: torch.empty(m, H * hd, dtype=torch.bfloat16, device="cuda") for v in (1, 0)}

    def call(v):
        switch(v)
        return lib.rdx_attention(ctypes.c_void_p(qkv.data_ptr()), ctypes.c_int64(qkv.stride(0)), ctypes.c_int64(m),
                                 ctypes.c_void_p(sc.data_ptr() if sc is not None else 0), ctypes.c_void_p(cu_t.data_ptr()),
                                 ctypes.c_void_p(cuq_t.data_ptr()), ctypes.c_int64(len(cu) - 1), ctypes.c_int32(maxq),
                                 ctypes.c_int32(maxk), ctypes.c_int32(H), ctypes.c_int32(KV), ctypes.c_int32(hd),
                                 ctypes.c_float(1 / math.sqrt(hd)), ctypes.c_void_p(outs[v].data_ptr()),
                                 ctypes.c_int64(outs[v].stride(0)), ctypes.c_void_p(st))

    res = {1: [], 0: []}
    for v in (1, 0):
        for _ in range(3):
            assert call(v) == 0
    torch.cuda.synchronize()
    for _ in range(iters):
        for v in (1, 0):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            switch(v)
            s.record()
            for _ in range(5):
                call(v)
            e.record()
            e.synchronize()
            res[v].append(s.elapsed_time(e) / 5 * 1e3)
    switch(0)
    diff = (outs[1].float() - outs[0].float()).abs().max().item()
    # fp32 reference on the first 4 sequences (suffix queries attend to all keys of their sequence)
    qf = qkv.float()
    sc_np = np.arange(b.num_tokens) if sc is None else np.array(plan.scatter_indices, dtype=np.int64)
    err = 0.0
    for s_ in range(4):
        k0, k1, q0, q1 = int(cu[s_]), int(cu[s_ + 1]), int(cu_q[s_]), int(cu_q[s_ + 1])
        rows = torch.from_numpy(sc_np[k0:k1]).cuda()
        L, nq = k1 - k0, q1 - q0
        for hh in range(H):
            g_ = hh // (H // KV)
            q = qf[q0:q1, hh * hd:(hh + 1) * hd]
            k = qf[rows, H * hd + g_ * hd:H * hd + (g_ + 1) * hd]
            vv = qf[rows, (H + KV) * hd + g_ * hd:(H + KV) * hd + (g_ + 1) * hd]
            sco = (q @ k.T) / math.sqrt(hd)
            qpos = torch.arange(L - nq, L, device="cuda")[:, None]
            sco = sco.masked_fill(torch.arange(L, device="cuda")[None, :] > qpos, float("-inf"))
            ref = torch.softmax(sco, -1) @ vv
            err = max(err, (outs[1][q0:q1, hh * hd:(hh + 1) * hd].float() - ref).abs().max().item())
    med = {k: round(sorted(v)[len(v) // 2], 2) for k, v in res.items()}
    print(f"{cfg} {layout}: {which} on {med[1]} us, off {med[0]} us; max|on - off| {diff:.3e}; "
          f"max|on - fp32 ref| {err:.3e}", flush=True)
