"""RadixMLP training step on the GPU: ``loss_and_grads``.

Reference: pkg/src/radix_compact/model.py:419-531 (``loss_and_grads``: mean
cross-entropy over all N positions, full backward through the compact path)
and PAPER.md:191-223 (the backward of a gather is a scatter-add).  Same
signature, same parameter names, same result types (Python float loss, dict of
numpy arrays in the params' dtype).

What runs where:
  * every RadixMLP row movement -- the compact-row token gather, the Q/K/V
    scatter N' -> N, the attention-output gather N -> N', the logits scatter --
    is ``rdx_gather_rows`` forward and ``rdx_gather_rows_backward`` (the
    deterministic ascending-index scatter-add, bit-identical to np.add.at)
    backward, via the ``RowGather`` autograd function;
  * ``precision="fp64"`` (default, the reference's contract): the dense math
    (GEMMs, norms, RoPE, per-sequence causal softmax) is fp64 CUDA tensors
    under torch autograd: the reference computes gradients in fp64 and its
    tests hold them to 1e-6 relative (tests/test_model.py:233-247);
  * ``precision="bf16"``: every projection GEMM -- forward (q/k/v/o, gate/up/down,
    LM head), activation gradient dX = dY W and weight gradient dW = dY^T X --
    runs on the tcgen05 GEMM (``rdx_gemm``, bf16 operands, fp32 accumulation in
    TMEM); the K-major operands W^T, dY^T, X^T are built by
    ``rdx_transpose_f32_bf16`` (fused fp32 -> bf16 cast, zero-padded to the
    GEMM's 8-element K multiple).  Norms, RoPE, SwiGLU, the causal softmax and
    the loss stay fp32 torch autograd.  Stated tolerance vs the reference's
    fp64 gradients: max |g - g_ref| / max |g_ref| <= 2.5e-2 per parameter (measured 1.1e-2 on C1), loss
    to 1e-2 relative (tests/test_training_gpu.py).
The forward follows ``_forward_cached`` (model.py:322-416) op for op, in
compact space: position-wise work on the N' rows, attention on the original
layout, exactly as the reference.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .errors import ShapeMismatch
from .model import FlopLedger, ModelConfig
from .plan import CompactionPlan
from .ragged import RaggedBatch, validate_batch


class RowGather:
    """out[j] = x[idx[j]] with the scatter-add adjoint, both on the sm_100a kernels."""

    _fn = None

    @classmethod
    def apply(cls, x, idx):
        if cls._fn is None:
            import torch

            from .ops import gather_rows_backward_device, gather_rows_device

            class _F(torch.autograd.Function):
                @staticmethod
                def forward(ctx, x_, idx_):
                    ctx.save_for_backward(idx_)
                    ctx.n_rows = x_.shape[0]
                    return gather_rows_device(x_.contiguous(), idx_)

                @staticmethod
                def backward(ctx, grad):
                    (idx_,) = ctx.saved_tensors
                    return gather_rows_backward_device(grad.contiguous(), idx_, ctx.n_rows), None

            cls._fn = _F
        return cls._fn.apply(x, idx)


def _tc_gemm(a, b):
    """fp32 [M, N] = a [M, K] @ b [N, K]^T on the tcgen05 GEMM (rdx_gemm, EPI_STORE_F32)."""
    import torch

    m, k = a.shape
    n = b.shape[0]
    npad = -(-n // 4) * 4  # 16-byte fp32 output rows
    out = torch.empty(m, npad, dtype=torch.float32, device=a.device)
    args = _native.GemmArgs()
    args.a, args.b, args.m, args.n, args.k = a.data_ptr(), b.data_ptr(), m, n, k
    args.lda, args.ldb = a.stride(0), b.stride(0)
    args.epi = _native.EPI_STORE_F32
    args.block_n = 0
    args.out, args.ldo = out.data_ptr(), npad
    _native.check(_native.lib().rdx_gemm(args, _native.stream_handle()), "rdx_gemm")
    return out[:, :n]


def _bf16_rows(x, k_pad):
    """fp32 [M, K] -> bf16 [M, k_pad] (zero-padded K), the K-major A/B operand as is."""
    import torch

    out = torch.zeros(x.shape[0], k_pad, dtype=torch.bfloat16, device=x.device)
    out[:, : x.shape[1]] = x
    return out


def _bf16_t(x, ld):
    """fp32 [R, C] -> bf16 [C, ld] = x^T zero-padded (rdx_transpose_f32_bf16)."""
    import torch

    x = x.contiguous()
    out = torch.empty(x.shape[1], ld, dtype=torch.bfloat16, device=x.device)
    _native.check(_native.lib().rdx_transpose_f32_bf16(x.data_ptr(), x.shape[0], x.shape[1], x.stride(0),
                                                       out.data_ptr(), ld, _native.stream_handle()),
                  "rdx_transpose_f32_bf16")
    return out


def _pad8(k):
    return -(-int(k) // 8) * 8


class TcLinear:
    """y = x W^T with forward, dX and dW all on the tcgen05 GEMM (bf16 operands, fp32 accumulate)."""

    _fn = None

    @classmethod
    def apply(cls, x, w):
        if cls._fn is None:
            import torch

            class _F(torch.autograd.Function):
                @staticmethod
                def forward(ctx, x_, w_):
                    x32, w32 = x_.float().contiguous(), w_.float().contiguous()
                    ctx.save_for_backward(x32, w32)
                    ctx.w_dtype = w_.dtype
                    k8 = _pad8(x32.shape[1])
                    return _tc_gemm(_bf16_rows(x32, k8), _bf16_rows(w32, k8))

                @staticmethod
                def backward(ctx, gy):
                    x32, w32 = ctx.saved_tensors
                    gy = gy.float().contiguous()
                    m, n = gy.shape
                    n8, m8 = _pad8(n), _pad8(m)
                    gx = _tc_gemm(_bf16_rows(gy, n8), _bf16_t(w32, n8))          # [M, K] = dY W
                    gw = _tc_gemm(_bf16_t(gy, m8), _bf16_t(x32, m8))             # [N, K] = dY^T X
                    return gx, gw.to(ctx.w_dtype)

            cls._fn = _F
        return cls._fn.apply(x, w)


def _rmsnorm(x, w, eps):
    import torch

    rms = torch.sqrt(torch.mean(x * x, dim=1, keepdim=True) + eps)
    return x / rms * w


def _rotate_half(x):
    import torch

    h = x.shape[-1] // 2
    return torch.cat([-x[..., h:], x[..., :h]], dim=-1)


def _attention(qf, kf, vf, cu, heads, kv, hd):
    """Exact causal softmax per sequence (model.py:228-265), GQA contiguous grouping."""
    import torch

    n = qf.shape[0]
    group = heads // kv
    q = qf.reshape(n, heads, hd)
    k = kf.reshape(n, kv, hd)
    v = vf.reshape(n, kv, hd)
    outs = []
    for s in range(len(cu) - 1):
        lo, hi = int(cu[s]), int(cu[s + 1])
        L = hi - lo
        if L == 0:
            continue
        qs = q[lo:hi].transpose(0, 1)                                    # [H, L, hd]
        ks = k[lo:hi].transpose(0, 1).repeat_interleave(group, dim=0)    # [H, L, hd]
        vs = v[lo:hi].transpose(0, 1).repeat_interleave(group, dim=0)
        sc = qs @ ks.transpose(1, 2) / np.sqrt(hd)
        mask = torch.ones(L, L, dtype=torch.bool, device=qf.device).tril()
        sc = sc.masked_fill(~mask, float("-inf"))
        outs.append((torch.softmax(sc, dim=-1) @ vs).transpose(0, 1).reshape(L, heads * hd))
    return torch.cat(outs, 0) if outs else qf.new_zeros(0, heads * hd)


def loss_and_grads(config: ModelConfig, params: dict, batch: RaggedBatch, plan: CompactionPlan | None, targets,
                   ledger: FlopLedger | None = None, *, precision: str = "fp64"):
    """Mean cross-entropy over all N positions and the gradient of every parameter
    (model.py:419-531); ``plan`` None = dense pass, else the compact (RadixMLP) pass.
    ``precision``: "fp64" (the reference's contract) or "bf16" (tcgen05 GEMMs)."""
    import torch

    if precision not in ("fp64", "bf16"):
        raise ValueError("precision must be 'fp64' or 'bf16'")
    tc = precision == "bf16"

    def mm(x, w):  # x @ w.T
        return TcLinear.apply(x, w) if tc else x @ w.T

    validate_batch(batch)
    targets = np.asarray(targets, dtype=np.int64)
    n = batch.num_tokens
    if targets.shape[0] != n:
        raise ShapeMismatch(f"{targets.shape[0]} targets for {n} tokens")
    if ledger is None:
        ledger = FlopLedger()
    dev = torch.device("cuda")
    _native.lib()  # no CPU fallback
    dtype = np.asarray(params["embed"]).dtype
    tdt = torch.float64 if (dtype == np.float64 and not tc) else torch.float32
    P = {k: torch.tensor(np.asarray(v), dtype=tdt, device=dev, requires_grad=True) for k, v in params.items()}
    tok = torch.from_numpy(np.asarray(batch.token_ids, dtype=np.int64)).to(dev)
    cu = np.asarray(batch.cu_seqlens, dtype=np.int64)
    hd, heads, kv, eps = config.head_dim, config.num_heads, config.num_kv_heads, config.norm_eps

    if plan is not None:
        if plan.n_original != n or plan.scatter_indices.shape[0] != n:
            from .errors import PlanBatchMismatch

            raise PlanBatchMismatch(f"plan built for {plan.n_original} tokens, batch has {n}")
        gather = torch.from_numpy(np.array(plan.gather_indices, copy=True).view(np.int32)).to(dev)
        scatter = torch.from_numpy(np.array(plan.scatter_indices, copy=True).view(np.int32)).to(dev)
        positions = np.asarray(plan.compact_positions, dtype=np.int64)
        token_rows = tok[gather.long()]
        ledger.index_copy(int(gather.shape[0]))
    else:
        gather = scatter = None
        positions = np.asarray(batch.position_ids, dtype=np.int64)
        token_rows = tok
    m = int(token_rows.shape[0])

    # embedding rows: a gather of the table by token id (adjoint = ordered scatter-add)
    h = RowGather.apply(P["embed"], token_rows.to(torch.int32))
    ledger.positionwise("embed", m)
    inv = config.rope_theta ** (-np.arange(0, hd, 2, dtype=np.float64) / hd)
    ang = positions.astype(np.float64)[:, None] * inv[None, :]
    cos = torch.from_numpy(np.concatenate([np.cos(ang)] * 2, 1)).to(dev, tdt)[:, None, :]
    sin = torch.from_numpy(np.concatenate([np.sin(ang)] * 2, 1)).to(dev, tdt)[:, None, :]
    for i in range(config.num_layers):
        p = f"layers.{i}."
        hn = _rmsnorm(h, P[p + "ln1"], eps)
        ledger.positionwise(f"l{i}.ln1", m)
        q = mm(hn, P[p + "wq"])
        k = mm(hn, P[p + "wk"])
        v = mm(hn, P[p + "wv"])
        ledger.positionwise(f"l{i}.qkv_proj", m)
        qn = _rmsnorm(q.reshape(-1, hd), P[p + "q_norm"], eps).reshape(m, heads, hd)
        kn = _rmsnorm(k.reshape(-1, hd), P[p + "k_norm"], eps).reshape(m, kv, hd)
        ledger.positionwise(f"l{i}.qk_norm_rope", m)
        qf = (qn * cos + _rotate_half(qn) * sin).reshape(m, heads * hd)
        kf = (kn * cos + _rotate_half(kn) * sin).reshape(m, kv * hd)
        vf = v
        if plan is not None:
            qf, kf, vf = (RowGather.apply(x, scatter) for x in (qf, kf, vf))
            ledger.index_copy(3 * n)
        ledger.attention(n)
        attn = _attention(qf, kf, vf, cu, heads, kv, hd)
        if plan is not None:
            attn = RowGather.apply(attn, gather)
            ledger.index_copy(m)
        h = h + mm(attn, P[p + "wo"])
        ledger.positionwise(f"l{i}.o_proj", m)
        ledger.positionwise(f"l{i}.attn_residual", m)
        hn2 = _rmsnorm(h, P[p + "ln2"], eps)
        g = mm(hn2, P[p + "w_gate"])
        u = mm(hn2, P[p + "w_up"])
        h = h + mm(g * torch.sigmoid(g) * u, P[p + "w_down"])
        ledger.positionwise(f"l{i}.mlp", m)
        ledger.positionwise(f"l{i}.mlp_residual", m)
    hf = _rmsnorm(h, P["final_norm"], eps)
    ledger.positionwise("final_norm", m)
    logits = mm(hf, P["lm_head"])
    ledger.positionwise("lm_head", m)
    if plan is not None:
        logits = RowGather.apply(logits, scatter)
        ledger.index_copy(n)
    tt = torch.from_numpy(targets).to(dev)
    loss = torch.nn.functional.cross_entropy(logits, tt, reduction="mean")
    loss.backward()
    grads = {name: (t.grad if t.grad is not None else torch.zeros_like(t)).detach().cpu().numpy().astype(dtype)
             for name, t in P.items()}
    return float(loss.item()), grads
