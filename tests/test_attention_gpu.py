"""rdx_attention (tcgen05 attention with the scatter fused into its loads) vs a
plain PyTorch fp32 reference of the reference's boundary (model.py:368-383:
scatter Q/K/V to the original layout, exact causal softmax per sequence with
GQA contiguous grouping, gather back).  Tolerance: bf16 P/V rounding."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _reference(qkv, scatter, cu, H, KV, hd):
    import torch

    full = qkv.float()[scatter.long()] if scatter is not None else qkv.float()
    n = full.shape[0]
    q = full[:, : H * hd].view(n, H, hd)
    k = full[:, H * hd:(H + KV) * hd].view(n, KV, hd)
    v = full[:, (H + KV) * hd:(H + 2 * KV) * hd].view(n, KV, hd)
    out = torch.zeros(n, H, hd, device=qkv.device)
    grp = H // KV
    for s in range(len(cu) - 1):
        lo, hi = int(cu[s]), int(cu[s + 1])
        L = hi - lo
        if L == 0:
            continue
        mask = torch.ones(L, L, dtype=torch.bool, device=qkv.device).tril()
        for h in range(H):
            sc = (q[lo:hi, h] @ k[lo:hi, h // grp].T) / math.sqrt(hd)
            sc = sc.masked_fill(~mask, float("-inf"))
            out[lo:hi, h] = torch.softmax(sc, -1) @ v[lo:hi, h // grp]
    return out.reshape(n, H * hd)


def _run(qkv, scatter, cu, cu_q, H, KV, hd, m_out, max_k=None):
    """max_k=None: the true longest sequence (short-unit pipeline when <= 512 keys); 0: long-unit pipeline."""
    import torch

    from paper_2601_15013_b200 import _native

    cu32 = torch.tensor(np.asarray(cu), dtype=torch.int32, device="cuda")
    cuq32 = torch.tensor(np.asarray(cu_q), dtype=torch.int32, device="cuda")
    out = torch.full((m_out, H * hd), float("nan"), dtype=torch.bfloat16, device="cuda")
    max_q = int(np.diff(np.asarray(cu_q)).max())
    max_k = int(np.diff(np.asarray(cu)).max()) if max_k is None else max_k
    code = _native.lib().rdx_attention(qkv.data_ptr(), qkv.stride(0), qkv.shape[0],
                                       None if scatter is None else scatter.data_ptr(), cu32.data_ptr(),
                                       cuq32.data_ptr(), len(cu) - 1, max_q, max_k, H, KV, hd, 1.0 / math.sqrt(hd),
                                       out.data_ptr(), out.stride(0), _native.stream_handle())
    _native.check(code, "rdx_attention")
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("hd,H,KV", [(128, 16, 8), (128, 32, 8), (64, 4, 2), (16, 4, 2), (32, 2, 1), (128, 4, 4)])
def test_plain_layout(hd, H, KV):
    import torch

    rng = np.random.default_rng(hd + H)
    lens = rng.integers(1, 300, size=6)
    cu = np.concatenate([[0], np.cumsum(lens)])
    n = int(cu[-1])
    g = torch.Generator(device="cuda").manual_seed(1)
    qkv = torch.randn(n, (H + 2 * KV) * hd, device="cuda", generator=g).to(torch.bfloat16)
    out = _run(qkv, None, cu, cu, H, KV, hd, n)
    ref = _reference(qkv, None, cu, H, KV, hd)
    err = (out.float() - ref).abs().max().item()
    assert err <= 2e-2 * ref.abs().max().item() + 1e-3, err


@pytest.mark.parametrize("pipeline", ["auto", "long", "bk64", "split"])
@pytest.mark.parametrize("hd,H,KV", [(128, 16, 8), (128, 32, 8), (64, 4, 2), (16, 4, 2)])
def test_suffix_queries_through_scatter(hd, H, KV, pipeline):
    """Compact Q rows + K/V gathered through the plan's scatter map == full-layout attention."""
    import torch

    from paper_2601_15013_b200 import build_plan
    from paper_2601_15013_b200.plan import host_plan_cu_q
    from paper_2601_15013_b200.workloads import RerankSpec, msmarco_rerank_batch

    b = msmarco_rerank_batch(RerankSpec(queries=2, passages_per_query=12, template_len=40, query_len=50,
                                        vocab=1000, seed=hd))
    plan = build_plan(b)
    cu_q = host_plan_cu_q(plan, b.cu_seqlens)
    m = plan.n_compact
    g = torch.Generator(device="cuda").manual_seed(2)
    qkv = torch.randn(m, (H + 2 * KV) * hd, device="cuda", generator=g).to(torch.bfloat16)
    scatter = torch.from_numpy(np.array(plan.scatter_indices).view(np.int32)).cuda()
    from paper_2601_15013_b200 import _native

    lib = _native.lib()
    prev = lib.rdx_attention_debug_bk64(1 if pipeline == "bk64" else 0)  # 64-key double-buffered S
    prev_s = lib.rdx_attention_debug_split(1 if pipeline == "split" else 0)  # half units in the last round
    try:
        out = _run(qkv, scatter, b.cu_seqlens, cu_q, H, KV, hd, m, max_k=0 if pipeline == "long" else None)
    finally:
        lib.rdx_attention_debug_bk64(prev)
        lib.rdx_attention_debug_split(prev_s)
    ref_full = _reference(qkv, scatter, b.cu_seqlens, H, KV, hd)
    gather = torch.from_numpy(np.array(plan.gather_indices).astype(np.int64)).cuda()
    ref = ref_full[gather]
    err = (out.float() - ref).abs().max().item()
    assert err <= 2e-2 * ref.abs().max().item() + 1e-3, err


def test_long_prefix_c4_slice():
    """2048-token shared prefix + 256-token suffixes: 36+ key tiles, 4-8 query blocks."""
    import torch

    from paper_2601_15013_b200 import build_plan
    from paper_2601_15013_b200.plan import host_plan_cu_q
    from paper_2601_15013_b200.workloads import long_prefix_batch

    b = long_prefix_batch(B=3, prefix_len=2048, suffix_len=256, vocab=151936)
    plan = build_plan(b)
    cu_q = host_plan_cu_q(plan, b.cu_seqlens)
    H, KV, hd = 8, 2, 128
    g = torch.Generator(device="cuda").manual_seed(3)
    qkv = torch.randn(plan.n_compact, (H + 2 * KV) * hd, device="cuda", generator=g).to(torch.bfloat16)
    scatter = torch.from_numpy(np.array(plan.scatter_indices).view(np.int32)).cuda()
    out = _run(qkv, scatter, b.cu_seqlens, cu_q, H, KV, hd, plan.n_compact)
    ref = _reference(qkv, scatter, b.cu_seqlens, H, KV, hd)[
        torch.from_numpy(np.array(plan.gather_indices).astype(np.int64)).cuda()]
    err = (out.float() - ref).abs().max().item()
    assert err <= 2e-2 * ref.abs().max().item() + 1e-3, err


@pytest.mark.parametrize("hd,H,KV,maxlen", [(128, 16, 8, 900), (128, 8, 1, 400), (64, 8, 8, 700), (96, 6, 3, 500)])
def test_plain_long_and_ragged(hd, H, KV, maxlen):
    """Many query-tile pairs per sequence, GQA groups 1..8, a non-power-of-two head dim,
    and empty sequences in the batch (no work units, no output rows)."""
    import torch

    rng = np.random.default_rng(maxlen + H)
    lens = rng.integers(1, maxlen, size=5)
    lens[1] = 0
    lens[3] = maxlen
    cu = np.concatenate([[0], np.cumsum(lens)])
    n = int(cu[-1])
    g = torch.Generator(device="cuda").manual_seed(4)
    qkv = torch.randn(n, (H + 2 * KV) * hd, device="cuda", generator=g).to(torch.bfloat16)
    out = _run(qkv, None, cu, cu, H, KV, hd, n)
    ref = _reference(qkv, None, cu, H, KV, hd)
    err = (out.float() - ref).abs().max().item()
    assert err <= 2e-2 * ref.abs().max().item() + 1e-3, err


def test_large_logit_range_rescale():
    """Scores spanning > 2^8 between key tiles exercise the lazy O rescale path."""
    import torch

    H, KV, hd = 4, 2, 64
    lens = np.array([700, 300])
    cu = np.concatenate([[0], np.cumsum(lens)])
    n = int(cu[-1])
    g = torch.Generator(device="cuda").manual_seed(5)
    qkv = torch.randn(n, (H + 2 * KV) * hd, device="cuda", generator=g)
    ramp = torch.linspace(0.1, 6.0, n, device="cuda")[:, None]  # later keys dominate more and more
    qkv[:, H * hd:(H + KV) * hd] *= ramp
    qkv[:, : H * hd] *= 3.0
    qkv = qkv.to(torch.bfloat16)
    out = _run(qkv, None, cu, cu, H, KV, hd, n)
    ref = _reference(qkv, None, cu, H, KV, hd)
    err = (out.float() - ref).abs().max().item()
    assert torch.isfinite(out.float()).all()
    assert err <= 2e-2 * ref.abs().max().item() + 1e-3, err
