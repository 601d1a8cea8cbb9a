"""Scratch: time each Qwen3-0.6B GEMM at the C2 shapes for every (CTA group, BN) choice."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, torch
sys.path.insert(0, %r)
from paper_2601_15013_b200 import _native
from paper_2601_15013_b200.model import DeviceWeights
res = {}
for M in (7024, 11056):
    for name, N, K, epi in (("qkv", 4096, 1024, 4), ("o_proj", 1024, 2048, 2), ("gate_up", 6144, 1024, 3), ("down", 1024, 3072, 2)):
        a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        w = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
        if epi == 2: out = torch.zeros(M, N, device="cuda")
        elif epi == 3: out = torch.empty(M, N // 2, dtype=torch.bfloat16, device="cuda")
        else: out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        qn = torch.ones(128, device="cuda"); rope = torch.zeros(M, 64, 2, device="cuda")
        args = _native.GemmArgs(); args.a=a.data_ptr(); args.b=w.data_ptr(); args.m=M; args.n=N; args.k=K
        args.lda=K; args.ldb=K; args.epi=epi; args.block_n=0; args.out=out.data_ptr(); args.ldo=out.stride(0)
        args.q_norm_w=qn.data_ptr(); args.k_norm_w=qn.data_ptr(); args.rope_table=rope.data_ptr(); args.head_dim=128; args.q_heads=16; args.kv_heads=8; args.eps=1e-6
        lib = _native.lib(); st = torch.cuda.current_stream().cuda_stream
        for _ in range(5): lib.rdx_gemm(args, st)
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(50): lib.rdx_gemm(args, st)
        e.record(); e.synchronize()
        us = s.elapsed_time(e) / 50 * 1e3
        res[f"{name}@{M}"] = round(us, 1)
print(json.dumps(res))
''' % ROOT
out = {}
for shape in ("auto", "2,256", "2,128", "1,256", "1,128"):
    env = dict(os.environ)
    if shape != "auto": env["RDX_GEMM_SHAPE"] = shape
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
    out[shape] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-300:]
    print(shape, out[shape], flush=True)
