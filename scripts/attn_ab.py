"""Interleaved A/B of rdx_attention between the in-tree _rdx.so and _rdx_<tag>.so (same process,
same box, same inputs): python scripts/attn_ab.py <tag> [c2|c4] [iters]"""
import ctypes
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_15013_b200 import _native, build_plan  # noqa: E402
from paper_2601_15013_b200.plan import host_plan_cu_q  # noqa: E402
from paper_2601_15013_b200.workloads import RerankSpec, long_prefix_batch, msmarco_rerank_batch  # noqa: E402

tag = sys.argv[1]
cfg = sys.argv[2] if len(sys.argv) > 2 else "c2"
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 30
b, H, KV, hd = ((msmarco_rerank_batch(RerankSpec()), 16, 8, 128) if cfg == "c2" else (long_prefix_batch(seed=0), 32, 8, 128))
plan = build_plan(b)
cu = b.cu_seqlens
cu_q = host_plan_cu_q(plan, cu)
m, n, B = plan.n_compact, b.num_tokens, b.num_sequences
g = torch.Generator(device="cuda").manual_seed(0)
qkv = torch.randn(m, (H + 2 * KV) * hd, device="cuda", generator=g).to(torch.bfloat16)
sc = torch.from_numpy(np.array(plan.scatter_indices).view(np.int32)).cuda()
cu_t = torch.tensor(cu, dtype=torch.int32, device="cuda")
cuq_t = torch.tensor(cu_q, dtype=torch.int32, device="cuda")
maxq, maxk = int(np.diff(cu_q).max()), int(np.diff(cu).max())
libs = {"main": _native.lib(), tag: ctypes.CDLL(os.path.join(os.path.dirname(_native.SO_PATH), f"_rdx_{tag}.so"))}
outs = {k: torch.empty(m, H * hd, dtype=torch.bfloat16, device="cuda") for k in libs}
st = torch.cuda.current_stream().cuda_stream


def call(k):
    return libs[k].rdx_attention(ctypes.c_void_p(qkv.data_ptr()), ctypes.c_int64(qkv.stride(0)), ctypes.c_int64(m),
                          ctypes.c_void_p(sc.data_ptr()), ctypes.c_void_p(cu_t.data_ptr()),
                          ctypes.c_void_p(cuq_t.data_ptr()), ctypes.c_int64(B), ctypes.c_int32(maxq),
                          ctypes.c_int32(maxk), ctypes.c_int32(H), ctypes.c_int32(KV), ctypes.c_int32(hd),
                          ctypes.c_float(1 / math.sqrt(hd)), ctypes.c_void_p(outs[k].data_ptr()),
                          ctypes.c_int64(outs[k].stride(0)), ctypes.c_void_p(st))


res = {k: [] for k in libs}
for k in libs:
    for _ in range(3):
        rc = call(k)
        assert rc == 0, (k, rc)
torch.cuda.synchronize()
for it in range(iters):
    for k in libs:
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            call(k)
        e.record()
        e.synchronize()
        res[k].append(s.elapsed_time(e) / 5 * 1e3)
same = torch.equal(outs["main"], outs[tag])
print(cfg, {k: round(sorted(v)[len(v) // 2], 2) for k, v in res.items()}, "us (median); outputs identical:", same)
