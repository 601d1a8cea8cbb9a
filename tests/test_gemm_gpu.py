"""tcgen05 GEMM + fused epilogues vs a plain PyTorch fp32 reference of the same op.

Inputs are bf16; the reference computes in fp32 from the same bf16 values, so
the only difference is accumulation order (fp32) and the final bf16 rounding.
Tolerances are stated per epilogue.
"""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gemm(a, w, epi, out, block_n=0, **qkv):
    from paper_2601_15013_b200 import _native

    args = _native.GemmArgs()
    args.a, args.b = a.data_ptr(), w.data_ptr()
    args.m, args.n, args.k = a.shape[0], w.shape[0], w.shape[1]
    args.lda, args.ldb = a.stride(0), w.stride(0)
    args.epi, args.block_n = epi, block_n
    args.out, args.ldo = out.data_ptr(), out.stride(0)
    if qkv:
        args.q_norm_w = qkv["qn"].data_ptr()
        args.k_norm_w = qkv["kn"].data_ptr()
        args.rope_table = qkv["rope"].data_ptr()
        args.rope_blocked = int(qkv.get("blocked", 0))
        if qkv.get("pos") is not None:
            args.rope_pos, args.rope_theta = qkv["pos"].data_ptr(), qkv.get("theta", 1e6)
        args.head_dim, args.q_heads, args.kv_heads = qkv["hd"], qkv["H"], qkv["KV"]
        args.eps = qkv["eps"]
    _native.check(_native.lib().rdx_gemm(args, _native.stream_handle()), "rdx_gemm")


def _rand(m, k, seed, scale=1.0):
    import torch

    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(m, k, generator=g, device="cuda") * scale).to(torch.bfloat16)


@pytest.mark.parametrize("m,n,k", [(128, 256, 64), (1, 128, 64), (300, 384, 256), (7040, 4096, 1024),
                                   (129, 200, 72), (1000, 1024, 2048)])
@pytest.mark.parametrize("block_n", [128, 256])
def test_store_bf16_and_f32(m, n, k, block_n):
    import torch

    from paper_2601_15013_b200 import _native

    a, w = _rand(m, k, 1), _rand(n, k, 2)
    ref = a.float() @ w.float().T
    out = torch.full((m, n), float("nan"), dtype=torch.bfloat16, device="cuda")
    _gemm(a, w, _native.EPI_STORE_BF16, out, block_n)
    torch.cuda.synchronize()
    tol = 2e-2 * ref.abs().max().item() + 1e-3
    assert (out.float() - ref).abs().max().item() <= tol
    out32 = torch.full((m, n), float("nan"), dtype=torch.float32, device="cuda")
    _gemm(a, w, _native.EPI_STORE_F32, out32, block_n)
    assert (out32 - ref).abs().max().item() <= 1e-3 * math.sqrt(k) * ref.abs().max().item() / 8 + 1e-4


def test_rows_batch_invariant():
    """Row r of the output is bit-identical whatever M is (no split-K, fixed tiles)."""
    import torch

    from paper_2601_15013_b200 import _native

    a, w = _rand(1000, 512, 3), _rand(768, 512, 4)
    full = torch.empty(1000, 768, dtype=torch.float32, device="cuda")
    _gemm(a, w, _native.EPI_STORE_F32, full)
    sub = torch.empty(37, 768, dtype=torch.float32, device="cuda")
    _gemm(a[500:537], w, _native.EPI_STORE_F32, sub)
    assert torch.equal(full[500:537], sub)


def test_resid_f32():
    import torch

    from paper_2601_15013_b200 import _native

    a, w = _rand(333, 512, 5), _rand(1024, 512, 6)
    h0 = torch.randn(333, 1024, device="cuda")
    h = h0.clone()
    _gemm(a, w, _native.EPI_RESID_F32, h)
    ref = h0 + a.float() @ w.float().T
    assert (h - ref).abs().max().item() <= 1e-3


@pytest.mark.parametrize("block_n", [128, 256])
def test_swiglu(block_n):
    import torch

    from paper_2601_15013_b200 import _native
    from paper_2601_15013_b200.model import DeviceWeights

    m, d, di = 515, 256, 384
    a = _rand(m, d, 7)
    wg, wu = _rand(di, d, 8, 0.1), _rand(di, d, 9, 0.1)
    wgu = DeviceWeights._interleave_gate_up(wg, wu, di)
    out = torch.empty(m, di, dtype=torch.bfloat16, device="cuda")
    _gemm(a, wgu, _native.EPI_SWIGLU, out, block_n)
    g = a.float() @ wg.float().T
    u = a.float() @ wu.float().T
    ref = g / (1 + torch.exp(-g)) * u
    assert (out.float() - ref).abs().max().item() <= 2e-2 * ref.abs().max().item() + 1e-3


@pytest.mark.parametrize("hd,H,KV", [(128, 16, 8), (16, 4, 2), (64, 4, 2)])
def test_qkv_norm_rope(hd, H, KV):
    import torch

    from paper_2601_15013_b200 import _native

    m, d = 300, 256
    a = _rand(m, d, 10)
    n = (H + 2 * KV) * hd
    w = _rand(n, d, 11, 0.2)
    qn = torch.rand(hd, device="cuda") + 0.5
    kn = torch.rand(hd, device="cuda") + 0.5
    pos = torch.randint(0, 4000, (m,), device="cuda", dtype=torch.int32)
    rope = torch.empty(m, hd // 2, 2, device="cuda")
    _native.check(_native.lib().rdx_rope_table(pos.data_ptr(), m, hd, 1e6, rope.data_ptr(),
                                               _native.stream_handle()), "rope")
    out = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    _gemm(a, w, _native.EPI_QKV, out, 0, qn=qn, kn=kn, rope=rope, hd=hd, H=H, KV=KV, eps=1e-6)
    # fp32 torch reference of model.py:356-366 with fp64 rope tables
    x = a.float() @ w.float().T
    inv = 1e6 ** (-torch.arange(0, hd, 2, dtype=torch.float64, device="cuda") / hd)
    ang = pos.double()[:, None] * inv[None, :]
    cos = torch.cat([ang.cos(), ang.cos()], 1).float()[:, None, :]
    sin = torch.cat([ang.sin(), ang.sin()], 1).float()[:, None, :]

    def norm_rope(t, wgt):
        t = t / torch.sqrt((t * t).mean(-1, keepdim=True) + 1e-6) * wgt
        rot = torch.cat([-t[..., hd // 2:], t[..., : hd // 2]], -1)
        return t * cos + rot * sin

    q = norm_rope(x[:, : H * hd].view(m, H, hd), qn).reshape(m, -1)
    k = norm_rope(x[:, H * hd:(H + KV) * hd].view(m, KV, hd), kn).reshape(m, -1)
    v = x[:, (H + KV) * hd:]
    ref = torch.cat([q, k, v], 1)
    err = (out.float() - ref).abs().max().item()
    assert err <= 2e-2 * ref.abs().max().item(), err


def _blocked_rope(pos, hd, theta=1e6):
    import torch

    from paper_2601_15013_b200 import _native

    m = pos.shape[0]
    t = torch.full((-(-m // 32) * 32 * (hd // 2) * 2,), float("nan"), device="cuda")
    _native.check(_native.lib().rdx_rope_table_blocked(pos.data_ptr(), m, hd, theta, t.data_ptr(),
                                                       _native.stream_handle()), "rope_blocked")
    return t


@pytest.mark.parametrize("m,hd", [(1, 16), (45, 64), (300, 128), (4097, 128)])
def test_rope_table_blocked_layout(m, hd):
    """rdx_rope_table_blocked holds rdx_rope_table's values at the documented indices."""
    import torch

    from paper_2601_15013_b200 import _native

    pos = torch.randint(0, 40000, (m,), device="cuda", dtype=torch.int32)
    rm = torch.empty(m, hd // 2, 2, device="cuda")
    _native.check(_native.lib().rdx_rope_table(pos.data_ptr(), m, hd, 1e6, rm.data_ptr(),
                                               _native.stream_handle()), "rope")
    bl = _blocked_rope(pos, hd).view(-1, 2)
    j = torch.arange(m, device="cuda")[:, None]
    i = torch.arange(hd // 2, device="cuda")[None, :]
    idx = 2 * (((j // 32) * (hd // 4) + i // 2) * 32 + j % 32) + i % 2
    assert torch.equal(bl[idx.reshape(-1)].view(m, hd // 2, 2), rm)


@pytest.mark.parametrize("m,hd,H,KV", [(300, 128, 16, 8), (7024, 128, 16, 8), (77, 16, 4, 2), (129, 64, 4, 2),
                                       (1000, 32, 6, 2)])
def test_qkv_blocked_rope_bit_identical(m, hd, H, KV):
    """The lane-blocked RoPE table gives the same bits as the row-major one."""
    import torch

    from paper_2601_15013_b200 import _native

    d = 256
    a = _rand(m, d, 12)
    n = (H + 2 * KV) * hd
    w = _rand(n, d, 13, 0.2)
    qn = torch.rand(hd, device="cuda") + 0.5
    kn = torch.rand(hd, device="cuda") + 0.5
    pos = torch.randint(0, 4000, (m,), device="cuda", dtype=torch.int32)
    rope = torch.empty(m, hd // 2, 2, device="cuda")
    _native.check(_native.lib().rdx_rope_table(pos.data_ptr(), m, hd, 1e6, rope.data_ptr(),
                                               _native.stream_handle()), "rope")
    out_rm = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    out_bl = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    kw = dict(qn=qn, kn=kn, hd=hd, H=H, KV=KV, eps=1e-6)
    _gemm(a, w, _native.EPI_QKV, out_rm, 0, rope=rope, **kw)
    _gemm(a, w, _native.EPI_QKV, out_bl, 0, rope=_blocked_rope(pos, hd), blocked=1, **kw)
    torch.cuda.synchronize()
    assert torch.equal(out_rm, out_bl)


@pytest.mark.parametrize("m,hd,H,KV,maxpos", [(300, 128, 16, 8, 4000), (7024, 128, 16, 8, 40000),
                                              (129, 64, 4, 2, 1 << 20), (1000, 64, 6, 2, 300)])
def test_qkv_rope_from_positions(m, hd, H, KV, maxpos):
    """(cos, sin) computed in the epilogue from positions: same result as the fp64-derived
    table within the bf16 output rounding (|angle error| < 1e-6 by construction)."""
    import torch

    from paper_2601_15013_b200 import _native

    d = 256
    a = _rand(m, d, 14)
    n = (H + 2 * KV) * hd
    w = _rand(n, d, 15, 0.2)
    qn = torch.rand(hd, device="cuda") + 0.5
    kn = torch.rand(hd, device="cuda") + 0.5
    g = torch.Generator(device="cuda").manual_seed(16)
    pos = torch.randint(0, maxpos, (m,), device="cuda", dtype=torch.int32, generator=g)
    pos[0] = maxpos - 1
    rope = torch.empty(m, hd // 2, 2, device="cuda")
    _native.check(_native.lib().rdx_rope_table(pos.data_ptr(), m, hd, 1e6, rope.data_ptr(),
                                               _native.stream_handle()), "rope")
    kw = dict(qn=qn, kn=kn, hd=hd, H=H, KV=KV, eps=1e-6)
    out_t = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    out_p = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    _gemm(a, w, _native.EPI_QKV, out_t, 0, rope=rope, **kw)
    _gemm(a, w, _native.EPI_QKV, out_p, 0, rope=rope, pos=pos, theta=1e6, **kw)
    torch.cuda.synchronize()
    t, p = out_t.float(), out_p.float()
    # v columns never see RoPE: bit-identical
    assert torch.equal(out_t[:, (H + KV) * hd:], out_p[:, (H + KV) * hd:])
    # q/k: at most one bf16 rounding step apart (2^-8 relative), almost always equal
    diff = (t - p).abs()
    # one bf16 step of the result, plus the ~1e-6 rad angle error times the term size
    # (a*cos - b*sin can cancel, so the absolute floor scales with the tensor, not the result)
    assert (diff <= t.abs() * 2.0 ** -7 + 1e-5 * t.abs().max()).all(), diff.max().item()
    # |angle error| ~1e-6 flips a bf16 rounding only for values within ~1e-6 of a rounding boundary
    eq = (diff == 0).float().mean().item()
    print(f"equal fraction {eq:.4f}")
    assert eq > 0.9, eq


def test_gemm_error_codes():
    import torch

    from paper_2601_15013_b200 import ShapeMismatch, _native

    a = torch.zeros(4, 12, dtype=torch.bfloat16, device="cuda")
    w = torch.zeros(8, 12, dtype=torch.bfloat16, device="cuda")
    out = torch.zeros(4, 8, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ShapeMismatch):
        _gemm(a, w, _native.EPI_STORE_BF16, out)
    # rdx_rmsnorm_rows_after: unsupported width, missing counters, QKV rope_pos head_dim
    lib, st = _native.lib(), _native.stream_handle()
    x = torch.zeros(64, 384, device="cuda")
    wn = torch.ones(384, device="cuda")
    o = torch.empty(64, 384, dtype=torch.bfloat16, device="cuda")
    ctr = torch.zeros(2, dtype=torch.int32, device="cuda")
    assert lib.rdx_rmsnorm_rows_after(x.data_ptr(), 384, 64, 384, wn.data_ptr(), 1e-6, o.data_ptr(), 384,
                                      ctr.data_ptr(), 384, None, st) == 13  # RDX_ERR_UNSUPPORTED
    assert lib.rdx_rmsnorm_rows_after(x.data_ptr(), 384, 64, 384, wn.data_ptr(), 1e-6, o.data_ptr(), 384,
                                      None, 384, None, st) == 12  # RDX_ERR_INVALID_ARGUMENT
    assert lib.rdx_rmsnorm_rows_after(x.data_ptr(), 384, 0, 384, wn.data_ptr(), 1e-6, o.data_ptr(), 384,
                                      None, 0, None, st) == 0  # no rows: nothing to do
    aq = torch.zeros(8, 64, dtype=torch.bfloat16, device="cuda")
    wq = torch.zeros(6 * 32, 64, dtype=torch.bfloat16, device="cuda")
    oq = torch.zeros(8, 6 * 32, dtype=torch.bfloat16, device="cuda")
    pos = torch.zeros(8, dtype=torch.int32, device="cuda")
    qn = torch.ones(32, device="cuda")
    args = _native.GemmArgs()
    args.a, args.b, args.m, args.n, args.k, args.lda, args.ldb = aq.data_ptr(), wq.data_ptr(), 8, 192, 64, 64, 64
    args.epi, args.out, args.ldo = _native.EPI_QKV, oq.data_ptr(), 192
    args.q_norm_w = args.k_norm_w = qn.data_ptr()
    args.head_dim, args.q_heads, args.kv_heads, args.eps = 32, 2, 2, 1e-6
    args.rope_pos, args.rope_theta = pos.data_ptr(), 1e6  # positions mode needs head_dim 64 or 128
    assert lib.rdx_gemm(args, st) == 12
    # slab counters only exist on the residual reduce-add epilogue
    a2 = torch.zeros(64, 64, dtype=torch.bfloat16, device="cuda")
    w2 = torch.zeros(128, 64, dtype=torch.bfloat16, device="cuda")
    o2 = torch.zeros(64, 128, dtype=torch.bfloat16, device="cuda")
    args = _native.GemmArgs()
    args.a, args.b, args.m, args.n, args.k, args.lda, args.ldb = a2.data_ptr(), w2.data_ptr(), 64, 128, 64, 64, 64
    args.epi, args.out, args.ldo, args.done_ctr = _native.EPI_STORE_BF16, o2.data_ptr(), 128, ctr.data_ptr()
    assert lib.rdx_gemm(args, st) == 12
    assert lib.rdx_device_status(st) == 0


@pytest.mark.timeout(120)
def test_rmsnorm_after_timeout_reports_status():
    """A slab counter that never reaches its target stops the wait after ~8 s and is
    reported by rdx_device_status (RDX_ERR_DEVICE_TIMEOUT) instead of killing the context."""
    import torch

    from paper_2601_15013_b200 import _native
    from paper_2601_15013_b200.errors import NativeLibraryError

    lib, st = _native.lib(), _native.stream_handle()
    assert lib.rdx_device_status(st) == 0
    x = torch.ones(32, 256, device="cuda")
    wn = torch.ones(256, device="cuda")
    o = torch.empty(32, 256, dtype=torch.bfloat16, device="cuda")
    ctr = torch.zeros(1, dtype=torch.int32, device="cuda")  # never incremented
    _native.check(lib.rdx_rmsnorm_rows_after(x.data_ptr(), 256, 32, 256, wn.data_ptr(), 1e-6, o.data_ptr(), 256,
                                             ctr.data_ptr(), 256, None, st), "rmsnorm_after")
    with pytest.raises(NativeLibraryError):
        _native.check_device_status()
    assert lib.rdx_device_status(st) == 0  # cleared by the read
    torch.cuda.synchronize()  # the context is still usable
    assert torch.isfinite(o.float()).all()


def _gemm_norm(a, w, epi, out, block_n=0, row_ss=None, norm_dim=0, eps=1e-6, hb=None, ss_out=None):
    from paper_2601_15013_b200 import _native

    args = _native.GemmArgs()
    args.a, args.b = a.data_ptr(), w.data_ptr()
    args.m, args.n, args.k = a.shape[0], w.shape[0], w.shape[1]
    args.lda, args.ldb = a.stride(0), w.stride(0)
    args.epi, args.block_n = epi, block_n
    args.out, args.ldo = out.data_ptr(), out.stride(0)
    if row_ss is not None:
        args.row_ss, args.ss_parts, args.norm_dim, args.norm_eps = row_ss.data_ptr(), row_ss.shape[1], norm_dim, eps
    if hb is not None:
        args.out_bf16, args.ldo_bf16, args.ss_out = hb.data_ptr(), hb.stride(0), ss_out.data_ptr()
    _native.check(_native.lib().rdx_gemm(args, _native.stream_handle()), "rdx_gemm")


@pytest.mark.parametrize("m,n,k", [(300, 1024, 2048), (7024, 1024, 3072), (129, 64, 128), (1000, 2560, 512)])
@pytest.mark.parametrize("block_n", [128, 256])
def test_resid_norm_epilogue(m, n, k, block_n):
    """RDX_EPI_RESID_NORM: h += acc, hb = bf16(h), ss = per-64-column sums of h^2 (model.py:387-392 fused)."""
    import torch

    from paper_2601_15013_b200 import _native

    a, w = _rand(m, k, 11), _rand(n, k, 12, 0.05)
    h0 = torch.randn(m, n, device="cuda")
    h = h0.clone()
    hb = torch.full((m, n), float("nan"), dtype=torch.bfloat16, device="cuda")
    ss = torch.full((m, n // 64), float("nan"), device="cuda")
    _gemm_norm(a, w, _native.EPI_RESID_NORM, h, block_n, hb=hb, ss_out=ss)
    torch.cuda.synchronize()
    ref = h0 + a.float() @ w.float().T
    assert (h - ref).abs().max().item() <= 1e-3 * ref.abs().max().item()
    assert torch.equal(hb, h.to(torch.bfloat16))  # exactly the bf16 of the stored residual
    ref_ss = (h * h).view(m, n // 64, 64).sum(-1)
    assert torch.allclose(ss, ref_ss, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("block_n", [128, 256])
def test_row_norm_fused_swiglu_and_qkv(block_n):
    """row_ss scaling == RMSNorm of the A rows with the weight folded into B."""
    import torch

    from paper_2601_15013_b200 import _native

    m, d, di = 517, 1024, 1536
    x = torch.randn(m, d, device="cuda") * 3
    ln = torch.rand(d, device="cuda") + 0.5
    ss = (x * x).view(m, d // 64, 64).sum(-1)
    xb = x.to(torch.bfloat16)
    # SwiGLU: gate/up interleaved in 64-column units (csrc/gemm.cu)
    wg, wu = _rand(di, d, 21, 0.05), _rand(di, d, 22, 0.05)
    w_gu = torch.cat([wg.view(di // 64, 1, 64, d), wu.view(di // 64, 1, 64, d)], 1).reshape(2 * di, d)
    w_fold = (w_gu.float() * ln[None, :]).to(torch.bfloat16)
    out = torch.full((m, di), float("nan"), dtype=torch.bfloat16, device="cuda")
    _gemm_norm(xb, w_fold, _native.EPI_SWIGLU, out, block_n, row_ss=ss, norm_dim=d, eps=1e-6)
    torch.cuda.synchronize()
    xn = x / torch.sqrt((x * x).mean(1, keepdim=True) + 1e-6) * ln
    g, u = xn @ wg.float().T, xn @ wu.float().T
    ref = torch.nn.functional.silu(g) * u
    assert (out.float() - ref).abs().max().item() <= 3e-2 * ref.abs().max().item()


@pytest.mark.parametrize("epi_name,m,n,k", [("EPI_RESID_F32", 7024, 1536, 2048), ("EPI_SWIGLU", 7024, 6144, 1024),
                                            ("EPI_STORE_BF16", 7024, 2560, 3072), ("EPI_STORE_F32", 5000, 2048, 512)])
def test_tail_split_bit_identical(epi_name, m, n, k):
    """The last partial round runs as half-width tiles (e.g. the C2 gate-up shape): every
    element is still one CTA's full K reduction -> identical bits."""
    import torch

    from paper_2601_15013_b200 import _native

    lib = _native.lib()
    epi = getattr(_native, epi_name)
    a, w = _rand(m, k, 31), _rand(n, k, 32, 0.05)
    if epi == _native.EPI_SWIGLU:
        shape, dt = (m, n // 2), torch.bfloat16
    elif epi == _native.EPI_STORE_BF16:
        shape, dt = (m, n), torch.bfloat16
    else:
        shape, dt = (m, n), torch.float32
    base = torch.randn(shape, device="cuda").to(dt) if epi == _native.EPI_RESID_F32 else torch.zeros(shape, dtype=dt,
                                                                                                      device="cuda")
    outs = []
    for on in (1, 0):
        prev = lib.rdx_gemm_debug_tail_split(on)
        try:
            o = base.clone()
            _gemm(a, w, epi, o)
            torch.cuda.synchronize()
        finally:
            lib.rdx_gemm_debug_tail_split(prev)
        outs.append(o)
    assert torch.equal(outs[0], outs[1])
    if epi == _native.EPI_STORE_F32:
        ref = a.float() @ w.float().T
        assert (outs[0] - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()


@pytest.mark.parametrize("epi_name,m,n,k,shape,counters", [
    ("EPI_RESID_F32", 7024, 1024, 2048, (0, 0), True),    # C2 o_proj (slab counters: row-block-major)
    ("EPI_RESID_F32", 7024, 1024, 3072, (0, 0), False),   # C2 down, column-block-major raster
    ("EPI_RESID_F32", 5000, 1024, 2048, (0, 0), True),    # 7 column tiles of 160/128
    ("EPI_STORE_BF16", 6026, 1024, 1024, (0, 0), False),  # 6 column tiles of 192/160
    ("EPI_STORE_F32", 7024, 1024, 512, (0, 0), False),
    ("EPI_STORE_F32", 3500, 1024, 512, (1, 256), False),  # 1-CTA tiles
    ("EPI_RESID_F32", 7000, 1056, 640, (0, 0), True),     # N not a multiple of 256
])
def test_column_partition_bit_identical(epi_name, m, n, k, shape, counters):
    """Few-round launches cut N into column tiles of two widths (multiples of 32): same
    bits as the plain 256-wide schedule, every slab counter reaches N, STORE_F32 == torch."""
    import torch

    from paper_2601_15013_b200 import _native

    lib = _native.lib()
    epi = getattr(_native, epi_name)
    a, w = _rand(m, k, 41), _rand(n, k, 42, 0.05)
    dt = torch.bfloat16 if epi == _native.EPI_STORE_BF16 else torch.float32
    base = torch.randn(m, n, device="cuda").to(dt) if epi == _native.EPI_RESID_F32 else torch.zeros(m, n, dtype=dt,
                                                                                                   device="cuda")
    outs, ncols = [], []
    lib.rdx_gemm_debug_shape(*shape)
    try:
        for on in (1, 0):
            prev = lib.rdx_gemm_debug_colpart(on)
            try:
                o = base.clone()
                ctr = torch.zeros(-(-m // 32), dtype=torch.int32, device="cuda")
                args = _native.GemmArgs()
                args.a, args.b, args.m, args.n, args.k = a.data_ptr(), w.data_ptr(), m, n, k
                args.lda, args.ldb, args.epi, args.out, args.ldo = k, k, epi, o.data_ptr(), n
                if counters:
                    args.done_ctr = ctr.data_ptr()
                _native.check(lib.rdx_gemm(args, _native.stream_handle()), "gemm")
                ncols.append(lib.rdx_gemm_debug_colpart(-1))
                torch.cuda.synchronize()
            finally:
                lib.rdx_gemm_debug_colpart(prev)
            outs.append(o)
            if counters:
                assert (ctr == n).all()
    finally:
        lib.rdx_gemm_debug_shape(0, 0)
    assert ncols[0] > 0 and ncols[1] == 0, ncols  # the partition ran, then the plain schedule
    assert torch.equal(outs[0], outs[1])
    if epi == _native.EPI_STORE_F32:
        ref = a.float() @ w.float().T
        assert (outs[0] - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()


@pytest.mark.parametrize("m,hd,H,KV", [(7024, 128, 16, 8), (34816, 128, 32, 8), (7024, 64, 16, 8)])
def test_qkv_tail_split_bit_identical(m, hd, H, KV):
    """QKV tail tiles one head wide go to one warp per lane quarter: same bits as unsplit."""
    import torch

    from paper_2601_15013_b200 import _native

    lib = _native.lib()
    d = 1024
    a = _rand(m, d, 41)
    n = (H + 2 * KV) * hd
    w = _rand(n, d, 42, 0.05)
    qn = torch.rand(hd, device="cuda") + 0.5
    kn = torch.rand(hd, device="cuda") + 0.5
    pos = torch.randint(0, 4096, (m,), device="cuda", dtype=torch.int32)
    outs = []
    for on in (1, 0):
        prev = lib.rdx_gemm_debug_tail_split(on)
        try:
            o = torch.full((m, n), float("nan"), dtype=torch.bfloat16, device="cuda")
            _gemm(a, w, _native.EPI_QKV, o, 0, qn=qn, kn=kn, rope=pos, pos=pos, hd=hd, H=H, KV=KV, eps=1e-6)
            torch.cuda.synchronize()
        finally:
            lib.rdx_gemm_debug_tail_split(prev)
        outs.append(o)
    assert not torch.isnan(outs[0].float()).any()
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("m,d,k", [(7024, 1024, 2048), (1000, 2560, 512), (33, 1024, 256)])
def test_resid_done_counter_and_rmsnorm_after(m, d, k):
    """RESID_F32 with a slab completion counter (row-block-major tiles) feeding
    rdx_rmsnorm_rows_after as a programmatic dependent: same h and same bf16 rows as
    the stream-ordered GEMM + rdx_rmsnorm_rows, counters = d per slab."""
    import torch

    from paper_2601_15013_b200 import _native

    lib = _native.lib()
    st = _native.stream_handle()
    a, w = _rand(m, k, 51), _rand(d, k, 52, 0.05)
    h0 = torch.randn(m, d, device="cuda")
    ln = torch.rand(d, device="cuda") + 0.5
    # reference path
    h_ref = h0.clone()
    _gemm(a, w, _native.EPI_RESID_F32, h_ref)
    n_ref = torch.empty(m, d, dtype=torch.bfloat16, device="cuda")
    _native.check(lib.rdx_rmsnorm_rows(h_ref.data_ptr(), d, None, m, d, ln.data_ptr(), 1e-6, n_ref.data_ptr(), d, st),
                  "rms")
    # overlapped path, twice in a row on the same counters (targets d and 2d)
    h = h0.clone()
    ctr = torch.zeros(-(-m // 32), dtype=torch.int32, device="cuda")
    out = torch.empty(m, d, dtype=torch.bfloat16, device="cuda")
    for use in (1, 2):
        args = _native.GemmArgs()
        args.a, args.b = a.data_ptr(), w.data_ptr()
        args.m, args.n, args.k = m, d, k
        args.lda, args.ldb = a.stride(0), w.stride(0)
        args.epi, args.out, args.ldo = _native.EPI_RESID_F32, h.data_ptr(), h.stride(0)
        args.done_ctr = ctr.data_ptr()
        _native.check(lib.rdx_gemm(args, st), "gemm")
        _native.check(lib.rdx_rmsnorm_rows_after(h.data_ptr(), d, m, d, ln.data_ptr(), 1e-6, out.data_ptr(), d,
                                                 ctr.data_ptr(), use * d, None, st), "rms_after")
        if use == 1:
            torch.cuda.synchronize()
            assert torch.equal(h, h_ref)
            assert torch.equal(out, n_ref)
            assert (ctr == d).all()
    torch.cuda.synchronize()
    assert (ctr == 2 * d).all()


@pytest.mark.parametrize("epi_name", ["EPI_RESID_F32", "EPI_SWIGLU", "EPI_STORE_BF16"])
def test_tile_raster_bit_identical(epi_name):
    """The tile raster (groups of row blocks) only reorders whole tiles: same bits."""
    import torch

    from paper_2601_15013_b200 import _native

    lib = _native.lib()
    epi = getattr(_native, epi_name)
    m, n, k = 17000, 2048, 512  # 67 pair row blocks: the grouped raster is the default here
    a, w = _rand(m, k, 61), _rand(n, k, 62, 0.05)
    shape = (m, n // 2) if epi == _native.EPI_SWIGLU else (m, n)
    dt = torch.float32 if epi == _native.EPI_RESID_F32 else torch.bfloat16
    base = torch.randn(shape, device="cuda").to(dt)
    outs = []
    for g in (0, 1, 3, 16, 1000):
        prev = lib.rdx_gemm_debug_group_m(g)
        try:
            o = base.clone()
            _gemm(a, w, epi, o)
            torch.cuda.synchronize()
        finally:
            lib.rdx_gemm_debug_group_m(prev)
        outs.append(o)
    for o in outs[1:]:
        assert torch.equal(outs[0], o)


def test_gemm_shape_fuzz():
    """Seeded random shapes through every tile shape, raster and the slab counters:
    STORE_F32 / RESID_F32 against torch fp32, counters == N per slab."""
    import torch

    from paper_2601_15013_b200 import _native

    lib = _native.lib()
    rng = np.random.default_rng(7)
    for trial in range(14):
        m = int(rng.integers(1, 20000))
        n = int(rng.integers(1, 96)) * 64
        k = int(rng.integers(1, 40)) * 64
        shape = [(0, 0), (1, 128), (1, 256), (2, 128), (2, 256)][trial % 5]
        group = [0, 1, 3, 16][trial % 4]
        a, w = _rand(m, k, 100 + trial), _rand(n, k, 200 + trial, 0.05)
        ref = a.float() @ w.float().T
        lib.rdx_gemm_debug_shape(*shape)
        prev_g = lib.rdx_gemm_debug_group_m(group)
        try:
            out = torch.full((m, n), float("nan"), device="cuda")
            _gemm(a, w, _native.EPI_STORE_F32, out)
            h0 = torch.randn(m, n, device="cuda")
            h = h0.clone()
            ctr = torch.zeros(-(-m // 32), dtype=torch.int32, device="cuda")
            args = _native.GemmArgs()
            args.a, args.b, args.m, args.n, args.k = a.data_ptr(), w.data_ptr(), m, n, k
            args.lda, args.ldb, args.epi, args.out, args.ldo = k, k, _native.EPI_RESID_F32, h.data_ptr(), n
            args.done_ctr = ctr.data_ptr()
            _native.check(lib.rdx_gemm(args, _native.stream_handle()), "gemm")
            torch.cuda.synchronize()
        finally:
            lib.rdx_gemm_debug_shape(0, 0)
            lib.rdx_gemm_debug_group_m(prev_g)
        tol = 1e-3 * ref.abs().max().item() + 1e-4
        assert (out - ref).abs().max().item() <= tol, (m, n, k, shape, group)
        assert (h - (h0 + ref)).abs().max().item() <= tol, (m, n, k, shape, group)
        assert (ctr == n).all(), (m, n, k, shape, group)


def _unweave(gu):
    """[m, 2 di] gate|up output interleaved in 64-column units -> (gate, up), each [m, di]."""
    m, n = gu.shape
    v = gu.view(m, n // 128, 2, 64)
    return v[:, :, 0, :].reshape(m, n // 2), v[:, :, 1, :].reshape(m, n // 2)


@pytest.mark.parametrize("m,d,di", [(7024, 1024, 3072), (5000, 1024, 3072), (300, 512, 1536), (20000, 2560, 9728)])
def test_gemm_pair_bit_identical(m, d, di):
    """rdx_gemm_pair (gate|up SwiGLU then down residual in one persistent launch, down tiles
    gated on per-slab counters of act) == the two rdx_gemm launches, bit for bit; the slab
    counters of the down GEMM's own done_ctr still reach N."""
    import torch

    from paper_2601_15013_b200 import _native

    lib = _native.lib()
    st = _native.stream_handle()
    x = _rand(m, d, 51)
    wgu = _rand(2 * di, d, 52, 0.05)
    wd = _rand(d, di, 53, 0.05)
    h0 = torch.randn(m, d, device="cuda")
    slabs = -(-m // 32)

    def args(a, w, epi, out, done=None):
        g = _native.GemmArgs()
        g.a, g.b, g.m, g.n, g.k = a.data_ptr(), w.data_ptr(), m, w.shape[0], w.shape[1]
        g.lda, g.ldb, g.epi, g.out, g.ldo = a.stride(0), w.stride(0), epi, out.data_ptr(), out.stride(0)
        if done is not None:
            g.done_ctr = done.data_ptr()
        return g

    outs = []
    for pair in (1, 0):
        prev = lib.rdx_gemm_debug_pair(pair)
        try:
            act = torch.full((m, di), float("nan"), device="cuda").to(torch.bfloat16)
            h = h0.clone()
            done = torch.zeros(slabs, dtype=torch.int32, device="cuda")
            dep = torch.zeros(slabs, dtype=torch.int32, device="cuda")
            g = args(x, wgu, _native.EPI_SWIGLU, act)
            dn = args(act, wd, _native.EPI_RESID_F32, h, done)
            _native.check(lib.rdx_gemm_pair(g, dn, dep.data_ptr(), st), "rdx_gemm_pair")
            torch.cuda.synchronize()
        finally:
            lib.rdx_gemm_debug_pair(prev)
        assert (done == d).all()
        if pair and bool(dep.any()):  # the one-launch path ran (not the two-launch fallback)
            assert (dep == di).all()  # every act column of every slab was published
        outs.append((act, h))
    _native.check_device_status()
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])
    # and against torch (fp32 reference of the SwiGLU MLP on the bf16 act)
    gu = x.float() @ wgu.float().T
    gate, up = _unweave(gu)
    ref_act = (torch.nn.functional.silu(gate) * up)
    assert (outs[0][0].float() - ref_act).abs().max().item() <= 2e-2 * ref_act.abs().max().item()
