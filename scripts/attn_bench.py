"""Time rdx_attention (suffix and plain layouts) on the C2 / C4 shapes; FA2 varlen beside it for context.

  python scripts/attn_bench.py [c2|c4] [--no-fa2] [--iters N]
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

cfg = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "c2"
iters = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else 20
if cfg == "c2":
    b, H, KV, hd = msmarco_rerank_batch(RerankSpec()), 16, 8, 128
elif cfg == "c4":
    b, H, KV, hd = long_prefix_batch(seed=0), 32, 8, 128
else:
    raise SystemExit(cfg)
plan = build_plan(b)
cu = b.cu_seqlens
cu_q = host_plan_cu_q(plan, cu)
m, n = plan.n_compact, b.num_tokens
g = torch.Generator(device="cuda").manual_seed(0)
qkv = torch.randn(m, (H + 2 * KV) * hd, device="cuda", generator=g).to(torch.bfloat16)
scatter = torch.from_numpy(np.array(plan.scatter_indices).view(np.int32)).cuda()
cu32 = torch.tensor(cu, dtype=torch.int32, device="cuda")
cuq32 = torch.tensor(cu_q, dtype=torch.int32, device="cuda")
out = torch.empty(m, H * hd, dtype=torch.bfloat16, device="cuda")
maxq = int(np.diff(cu_q).max())
maxk = int(np.diff(cu).max())
maxk_arg = 0 if os.environ.get("ATTN_LONG") == "1" else maxk  # 0: force the long-unit pipeline
lib = _native.lib()
lens = np.diff(cu).astype(np.float64)
lcp = lens - np.diff(cu_q)
pairs_suffix = float(np.sum(lens * (lens + 1) / 2 - lcp * (lcp + 1) / 2))
pairs_full = float(np.sum(lens * (lens + 1) / 2))


def ours():
    lib.rdx_attention(qkv.data_ptr(), qkv.stride(0), qkv.shape[0], scatter.data_ptr(), cu32.data_ptr(), cuq32.data_ptr(),
                      len(cu) - 1, maxq, maxk_arg, H, KV, hd, 1 / math.sqrt(hd), out.data_ptr(), out.stride(0),
                      torch.cuda.current_stream().cuda_stream)


qkv_full = qkv[torch.from_numpy(np.array(plan.scatter_indices).astype(np.int64)).cuda()].contiguous()
out_full = torch.empty(n, H * hd, dtype=torch.bfloat16, device="cuda")


def ours_plain():
    lib.rdx_attention(qkv_full.data_ptr(), qkv_full.stride(0), qkv_full.shape[0], None, cu32.data_ptr(), cu32.data_ptr(), len(cu) - 1,
                      maxk, maxk_arg, H, KV, hd, 1 / math.sqrt(hd), out_full.data_ptr(), out_full.stride(0),
                      torch.cuda.current_stream().cuda_stream)


def t(fn, it=iters):
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


us_s = t(ours)
us_p = t(ours_plain)
tf_s = 4 * H * hd * pairs_suffix / (us_s * 1e-6) / 1e12
tf_p = 4 * H * hd * pairs_full / (us_p * 1e-6) / 1e12
print(f"{cfg}: N={n} N'={m} ours suffix {us_s:.1f} us ({tf_s:.0f} TF/s)  plain {us_p:.1f} us ({tf_p:.0f} TF/s)", flush=True)
# parity of suffix vs plain (same math, different layouts)
ours(); ours_plain(); torch.cuda.synchronize()
sc = torch.from_numpy(np.array(plan.scatter_indices).astype(np.int64)).cuda()
diff = (out[sc].float() - out_full.float()).abs().max().item()
print(f"suffix-vs-plain max|diff| {diff:.3e}", flush=True)
if "--no-fa2" not in sys.argv:
    try:
        from flash_attn import flash_attn_varlen_func

        kvf = qkv_full[:, H * hd:]

        def fa2():
            flash_attn_varlen_func(qkv[:, :H * hd].view(m, H, hd), kvf[:, :KV * hd].view(n, KV, hd),
                                   kvf[:, KV * hd:].view(n, KV, hd), cuq32, cu32, maxq, maxk, causal=True)

        us_f = t(fa2)
        print(f"fa2 suffix {us_f:.1f} us ({4 * H * hd * pairs_suffix / (us_f * 1e-6) / 1e12:.0f} TF/s)", flush=True)
        ref = flash_attn_varlen_func(qkv[:, :H * hd].view(m, H, hd), kvf[:, :KV * hd].view(n, KV, hd),
                                     kvf[:, KV * hd:].view(n, KV, hd), cuq32, cu32, maxq, maxk, causal=True)
        print(f"ours-vs-fa2 max|diff| {(ref.reshape(m, -1).float() - out.float()).abs().max().item():.3e}")
    except Exception as ex:  # library context only
        print("fa2 unavailable:", ex)
if os.environ.get("RDX_ATTN_STATS") == "1":
    import ctypes

    names = ["mma_wait_kv", "mma_wait_p", "mma_wait_q", "mma_wait_ofree", "mma_total", "sm_wait_s", "sm_total",
             "epi_wait", "ld_wait_free", "ld_total", "sm_rescales", "mma_issue", "epi_total", "sm_exp"]
    for label, fn in (("suffix", ours), ("plain", ours_plain)):
        buf = (ctypes.c_ulonglong * 16)()
        lib.rdx_attention_debug_stats(buf, 16)  # reset
        fn()
        torch.cuda.synchronize()
        lib.rdx_attention_debug_stats(buf, 16)
        v = list(buf)
        den = {"mma": v[4], "sm": v[6], "ld": v[9], "epi": v[12]}
        print(label, "per-role clock fractions:",
              {n: round(x / max(den[n.split("_")[0]], 1), 3) for n, x in zip(names, v) if n != "sm_rescales"},
              "sm_rescales", v[10], flush=True)
if os.environ.get("RDX_ATTN_TRACE") == "1":
    import ctypes

    ours()
    torch.cuda.synchronize()
    buf = (ctypes.c_uint32 * (2 + 2 * 4096))()
    lib.rdx_attention_debug_trace(buf, len(buf))
    n = min(buf[0], 4096)
    ev = sorted((buf[2 + 2 * i], buf[3 + 2 * i]) for i in range(n))
    t0 = ev[0][0] if ev else 0
    roles = {0: "LOAD", 1: "MMA ", 2: "SOFT", 3: "EPI "}
    names = {(0, 1): "K tile", (0, 2): "V tile", (1, 1): "issue S", (1, 2): "got P", (1, 3): "K ready",
             (1, 4): "V ready", (2, 1): "got S",
             (2, 2): "pub P", (2, 3): "S in regs", (2, 4): "max done", (2, 5): "exp done", (3, 1): "O ready",
             (3, 2): "O stored"}
    for tt, code in ev[:int(os.environ.get("TRACE_N", "160"))]:
        role, e, pl = code >> 12, (code >> 8) & 15, code & 255
        print(f"{(tt - t0) & 0xffffffff:9d} {roles.get(role, role)} {names.get((role, e), e):9s} h={pl >> 4} j={pl & 15}"
              + (f" [{'box' if pl & 0x80 else 'r16' if pl & 0x40 else 'g4'}]" if role == 0 else ""))
if os.environ.get("RDX_ATTN_STATS") == "1":
    import ctypes

    ours()
    torch.cuda.synchronize()
    nct = torch.cuda.get_device_properties(0).multi_processor_count
    buf = (ctypes.c_ulonglong * (3 * nct))()
    if lib.rdx_attention_debug_cta_times(buf, nct) == 0:
        st = np.array([buf[3 * i] for i in range(nct)], dtype=np.float64)
        en = np.array([buf[3 * i + 1] for i in range(nct)], dtype=np.float64)
        un = np.array([buf[3 * i + 2] for i in range(nct)])
        t0 = st.min()
        print("CTA start us: min 0 max %.2f | end us: min %.2f median %.2f max %.2f (CTA %d)" %
              ((st.max() - t0) / 1e3, (en.min() - t0) / 1e3, np.median(en - t0) / 1e3, (en.max() - t0) / 1e3,
               int(en.argmax())))
        for u in sorted(set(un.tolist())):
            sel = un == u
            print(f"  {int(sel.sum()):4d} CTAs with {u} units: end us median {np.median(en[sel] - t0) / 1e3:.2f} "
                  f"max {(en[sel] - t0).max() / 1e3:.2f}; busy us median {np.median(en[sel] - st[sel]) / 1e3:.2f}")
