"""The reference's exported model primitives, as thin wrappers over the GPU kernels.

Reference: pkg/src/radix_compact/model.py:147 (``rmsnorm``), 180 (``apply_rope``),
204 (``swiglu_mlp``), 210 (``attention_ragged``); same names, arguments,
``ShapeMismatch`` / ``OddHeadDim`` errors.  Inputs may be numpy arrays (returned
as numpy, in the input dtype) or CUDA tensors (returned as CUDA tensors).  The
arithmetic is the hot path's: bf16 operands, fp32 accumulation / statistics,
so results match the reference's fp64 within bf16 tolerance (tests state it).

  rmsnorm          rdx_rmsnorm_rows
  apply_rope       rdx_rope_table (fp64 angles on the device) + rotate-half
  swiglu_mlp       rdx_gemm EPI_SWIGLU (gate|up interleaved) + rdx_gemm EPI_STORE_F32
  attention_ragged rdx_attention (plain layout: scatter = NULL, cu_q = cu)
"""

from __future__ import annotations

import math

import numpy as np

from . import _native
from .errors import OddHeadDim, ShapeMismatch


def _to_dev(x, dtype=None):
    import torch

    if isinstance(x, torch.Tensor):
        t = x if x.is_cuda else x.cuda()
    else:
        t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    if dtype is not None:
        t = t.to(dtype)
    return t.contiguous()


def _back(out, like):
    import torch

    if isinstance(like, torch.Tensor):
        return out.to(like.dtype) if like.dtype.is_floating_point else out
    arr = out.float().cpu().numpy()
    return arr.astype(np.asarray(like).dtype, copy=False)


def rmsnorm(x, weight, eps: float):
    """x / sqrt(mean(x^2) + eps) * weight per row (model.py:147-152)."""
    import torch

    shape = tuple(x.shape)
    if len(shape) != 2 or shape[1] != tuple(weight.shape)[0]:
        raise ShapeMismatch(f"rmsnorm: x {shape} vs weight {tuple(weight.shape)}")
    n, d = shape
    xd, wd = _to_dev(x, torch.float32), _to_dev(weight, torch.float32)
    pad = (-d) % 8  # kernel contract: rows of whole 16-byte vectors
    if pad:
        xd = torch.nn.functional.pad(xd, (0, pad))
        wd = torch.nn.functional.pad(wd, (0, pad))
    out = torch.empty(n, d + pad, dtype=torch.bfloat16, device=xd.device)
    if n:
        code = _native.lib().rdx_rmsnorm_rows(xd.data_ptr(), xd.stride(0), None, n, d + pad, wd.data_ptr(),
                                              float(eps) * (d + pad) / d if pad else float(eps), out.data_ptr(),
                                              out.stride(0), _native.stream_handle())
        _native.check(code, "rdx_rmsnorm_rows")
    res = out[:, :d].float()
    if pad:  # the kernel averaged over d + pad columns: rescale to the mean over d
        res = res * math.sqrt(d / (d + pad))
    return _back(res, x)


def rope_tables(positions, head_dim: int, theta: float):
    """(cos, sin) [rows, head_dim] with duplicated halves (model.py:165-172), from rdx_rope_table."""
    import torch

    if head_dim % 2:
        raise OddHeadDim(f"head_dim {head_dim} is odd")
    pos = _to_dev(np.asarray(positions, dtype=np.uint32).view(np.int32) if not isinstance(positions, torch.Tensor)
                  else positions.to(torch.int32))
    n = pos.shape[0]
    table = torch.empty(n, head_dim // 2, 2, dtype=torch.float32, device=pos.device)
    if n:
        code = _native.lib().rdx_rope_table(pos.data_ptr(), n, head_dim, float(theta), table.data_ptr(),
                                            _native.stream_handle())
        _native.check(code, "rdx_rope_table")
    cos, sin = table[..., 0], table[..., 1]
    return torch.cat([cos, cos], 1), torch.cat([sin, sin], 1)


def _rotate_half(x):
    import torch

    half = x.shape[-1] // 2
    return torch.cat([-x[..., half:], x[..., :half]], dim=-1)


def apply_rope(q, k, positions, theta: float = 10000.0):
    """Rotate-half rotary embedding of (rows, heads, head_dim) q and k (model.py:180-190)."""
    import torch

    if tuple(np.shape(positions))[:1] != tuple(q.shape)[:1]:
        raise ShapeMismatch("positions length must match q rows")
    cos, sin = rope_tables(positions, q.shape[-1], theta)
    qd, kd = _to_dev(q, torch.float32), _to_dev(k, torch.float32)
    c, s = cos[:, None, :], sin[:, None, :]
    qo = qd * c + _rotate_half(qd) * s
    ko = kd * c + _rotate_half(kd) * s
    return _back(qo, q), _back(ko, k)


def _gemm(a, w, epi, out, **extra):
    args = _native.GemmArgs()
    args.a, args.b = a.data_ptr(), w.data_ptr()
    args.m, args.n, args.k = a.shape[0], w.shape[0], w.shape[1]
    args.lda, args.ldb = a.stride(0), w.stride(0)
    args.epi, args.block_n = epi, 0
    args.out, args.ldo = out.data_ptr(), out.stride(0)
    for key, val in extra.items():
        setattr(args, key, val)
    _native.check(_native.lib().rdx_gemm(args, _native.stream_handle()), "rdx_gemm")


def swiglu_mlp(h, w_gate, w_up, w_down):
    """silu(h Wg^T) * (h Wu^T) Wd^T (model.py:204-207) with the fused SwiGLU GEMM epilogue."""
    import torch

    from .model import DeviceWeights, SWIGLU_UNIT

    hs, gs = tuple(h.shape), tuple(w_gate.shape)
    if len(hs) != 2 or hs[1] != gs[1]:
        raise ShapeMismatch(f"swiglu: h {hs} vs w_gate {gs}")
    if tuple(w_up.shape) != gs or tuple(w_down.shape) != (gs[1], gs[0]):
        raise ShapeMismatch("swiglu: w_up / w_down shapes")
    bf = torch.bfloat16
    d, di = gs[1], gs[0]
    if d % 8:
        raise ShapeMismatch("swiglu: hidden size must be a multiple of 8 (16-byte TMA rows)")
    di_pad = -(-di // SWIGLU_UNIT) * SWIGLU_UNIT
    hd_ = _to_dev(h, bf)
    w_gu = DeviceWeights._interleave_gate_up(_to_dev(w_gate, bf), _to_dev(w_up, bf), di_pad)
    wd = _to_dev(w_down, bf)
    if di_pad != di:
        wd = torch.cat([wd, torch.zeros(d, di_pad - di, dtype=bf, device=wd.device)], 1).contiguous()
    m = hs[0]
    act = torch.empty(m, di_pad, dtype=bf, device=hd_.device)
    out = torch.empty(m, -(-d // 4) * 4, dtype=torch.float32, device=hd_.device)[:, :d]
    if m:
        _gemm(hd_, w_gu, _native.EPI_SWIGLU, act)
        _gemm(act, wd, _native.EPI_STORE_F32, out)
    return _back(out, h)


def attention_ragged(q, k, v, cu_seqlens, num_heads: int, num_kv_heads: int, head_dim: int):
    """Exact causal GQA softmax attention over a packed batch (model.py:210-225), rdx_attention."""
    import torch

    n = q.shape[0]
    if tuple(q.shape) != (n, num_heads * head_dim):
        raise ShapeMismatch(f"q shape {tuple(q.shape)}")
    if tuple(k.shape) != (n, num_kv_heads * head_dim) or tuple(v.shape) != tuple(k.shape):
        raise ShapeMismatch(f"k/v shape {tuple(k.shape)}/{tuple(v.shape)}")
    bf = torch.bfloat16
    qkv = torch.cat([_to_dev(q, bf), _to_dev(k, bf), _to_dev(v, bf)], 1).contiguous()
    cu = np.asarray(cu_seqlens, dtype=np.int64)
    cu32 = torch.from_numpy(cu.astype(np.int32)).to(qkv.device)
    out = torch.zeros(n, num_heads * head_dim, dtype=bf, device=qkv.device)
    lens = np.diff(cu)
    if n and lens.size:
        code = _native.lib().rdx_attention(qkv.data_ptr(), qkv.stride(0), n, None, cu32.data_ptr(), cu32.data_ptr(),
                                           lens.size, int(lens.max()), int(lens.max()), num_heads, num_kv_heads,
                                           head_dim, 1.0 / math.sqrt(head_dim), out.data_ptr(), out.stride(0),
                                           _native.stream_handle())
        _native.check(code, "rdx_attention")
    return _back(out, q)
