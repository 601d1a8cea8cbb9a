"""Row gather / scatter on the GPU (reference: pkg/src/radix_compact/ops.py:29-66).

``gather_rows(x, idx)`` returns ``out[j] = x[idx[j]]`` as a bit-exact row copy
(any dtype; the kernel moves bytes in 16-byte vectors), ``scatter_rows`` is
the same operation with the scatter map.  Device tensors in -> device tensor
out; host numpy in -> host numpy out (H2D + kernel + D2H).  Errors match the
reference: non-2-D input -> ShapeMismatch, index outside [0, rows) ->
IndexOutOfRange (checked on the device, surfaced after the launch).
``num_threads`` is accepted for signature compatibility and ignored (the
reference's RADIX_COMPACT_THREADS pool, ops.py:23-26, has no GPU meaning).
"""

from __future__ import annotations

import numpy as np

from . import _native
from .errors import IndexOutOfRange, ShapeMismatch


def gather_rows_device(x, idx, out=None, err=None, stream=None):
    """Device gather: x [rows, cols] (any dtype, row-contiguous), idx int32/u32 [n]."""
    import torch

    if x.dim() != 2:
        raise ShapeMismatch(f"expected a 2-D matrix, got shape {tuple(x.shape)}")
    if idx.dim() != 1:
        raise ShapeMismatch(f"indices must be 1-D, got shape {tuple(idx.shape)}")
    if x.stride(1) != 1:
        x = x.contiguous()
    n = int(idx.shape[0])
    cols = int(x.shape[1])
    if out is None:
        out = torch.empty((n, cols), dtype=x.dtype, device=x.device)
    esz = x.element_size()
    code = _native.lib().rdx_gather_rows(
        x.data_ptr(), int(x.shape[0]), x.stride(0) * esz, idx.data_ptr(), n,
        out.data_ptr(), out.stride(0) * esz, cols * esz,
        None if err is None else err.data_ptr(), _native.stream_handle(stream),
    )
    _native.check(code, "rdx_gather_rows")
    return out


def _check_host_indices(indices, limit: int) -> np.ndarray:
    idx = np.asarray(indices)
    if idx.ndim != 1:
        raise ShapeMismatch(f"indices must be 1-D, got shape {idx.shape}")
    idx64 = idx.astype(np.int64, copy=False)
    if idx64.size and (int(idx64.min()) < 0 or int(idx64.max()) >= limit):
        raise IndexOutOfRange(f"index outside [0, {limit})")
    return idx64


def gather_rows(x, gather_indices, num_threads: int | None = None):
    """out[j, :] = x[gather_indices[j], :] (ops.py:50-61), on the GPU."""
    del num_threads
    import torch

    if isinstance(x, torch.Tensor):
        if x.dim() != 2:
            raise ShapeMismatch(f"expected a 2-D matrix, got shape {tuple(x.shape)}")
        idx = gather_indices
        if not isinstance(idx, torch.Tensor):
            idx = torch.from_numpy(_check_host_indices(idx, x.shape[0]).astype(np.int32))
        idx = idx.to(device=x.device, dtype=torch.int32)
        err = torch.zeros(1, dtype=torch.int32, device=x.device)
        out = gather_rows_device(x, idx, err=err)
        if int(err.item()):
            raise IndexOutOfRange(f"index outside [0, {x.shape[0]})")
        return out
    xh = np.asarray(x)
    if xh.ndim != 2:
        raise ShapeMismatch(f"expected a 2-D matrix, got shape {xh.shape}")
    idx = _check_host_indices(gather_indices, xh.shape[0])
    if idx.size == 0 or xh.shape[1] == 0:
        return np.empty((idx.size, xh.shape[1]), dtype=xh.dtype)
    xd = torch.from_numpy(np.ascontiguousarray(xh)).cuda()
    idd = torch.from_numpy(idx.astype(np.int32)).cuda()
    return gather_rows_device(xd, idd).cpu().numpy()


def scatter_rows(y, scatter_indices, num_threads: int | None = None):
    """out[i, :] = y[scatter_indices[i], :] (ops.py:64-66), on the GPU."""
    return gather_rows(y, scatter_indices, num_threads=num_threads)


def gather_rows_backward_device(grad, idx, n: int, out=None, err=None, stream=None):
    """Device adjoint of the row gather: out[n, cols] = 0; out[idx[j]] += grad[j] in
    ascending j (ops.py:69-99).  grad fp32/fp64 [len(idx), cols], idx int32/u32."""
    import torch

    if grad.dim() != 2:
        raise ShapeMismatch(f"expected a 2-D matrix, got shape {tuple(grad.shape)}")
    if grad.dtype not in (torch.float32, torch.float64):
        raise TypeError(f"gather_rows_backward: float32/float64 gradients only, got {grad.dtype}")
    if idx.dim() != 1 or idx.shape[0] != grad.shape[0]:
        raise ShapeMismatch(f"{idx.shape[0] if idx.dim() == 1 else tuple(idx.shape)} indices vs "
                            f"{grad.shape[0]} gradient rows")
    if grad.stride(1) != 1:
        grad = grad.contiguous()
    cols = int(grad.shape[1])
    if out is None:
        out = torch.empty((int(n), cols), dtype=grad.dtype, device=grad.device)
    lib = _native.lib()
    from .plan import _WORKSPACE

    nbytes = int(lib.rdx_gather_rows_backward_scratch_bytes(int(idx.shape[0]), int(n)))
    scratch = _WORKSPACE.get(grad.device, nbytes)
    esz = grad.element_size()
    dtype = _native.RDX_DTYPE_F32 if grad.dtype == torch.float32 else _native.RDX_DTYPE_F64
    code = lib.rdx_gather_rows_backward(
        grad.data_ptr(), grad.stride(0) * esz, idx.data_ptr(), int(idx.shape[0]), int(n), out.data_ptr(),
        out.stride(0) * esz, cols, dtype, None if err is None else err.data_ptr(), scratch.data_ptr(),
        scratch.numel(), _native.stream_handle(stream))
    _native.check(code, "rdx_gather_rows_backward")
    return out


def gather_rows_backward(grad_out, gather_indices, n: int, num_threads: int | None = None):
    """Adjoint of gather_rows (ops.py:69-99): zero-init scatter-add into n rows with
    ascending-j accumulation (bit-identical to the reference's np.add.at path)."""
    del num_threads
    import torch

    if isinstance(grad_out, torch.Tensor):
        idx = gather_indices
        if not isinstance(idx, torch.Tensor):
            idx = torch.from_numpy(_check_host_indices(idx, n).astype(np.int32))
        idx = idx.to(device=grad_out.device, dtype=torch.int32)
        err = torch.zeros(1, dtype=torch.int32, device=grad_out.device)
        out = gather_rows_backward_device(grad_out, idx, n, err=err)
        if int(err.item()):
            raise IndexOutOfRange(f"index outside [0, {n})")
        return out
    g = np.asarray(grad_out)
    if g.ndim != 2:
        raise ShapeMismatch(f"expected a 2-D matrix, got shape {g.shape}")
    idx = _check_host_indices(gather_indices, n)
    if idx.size != g.shape[0]:
        raise ShapeMismatch(f"{idx.size} indices vs {g.shape[0]} gradient rows")
    if g.dtype not in (np.float32, np.float64):
        raise TypeError(f"gather_rows_backward: float32/float64 gradients only, got {g.dtype}")
    if n == 0 or g.shape[1] == 0:
        return np.zeros((n, g.shape[1]), dtype=g.dtype)
    gd = torch.from_numpy(np.ascontiguousarray(g)).cuda()
    idd = torch.from_numpy(idx.astype(np.int32)).cuda()
    return gather_rows_backward_device(gd, idd, n).cpu().numpy()


def scatter_rows_backward(grad_out, scatter_indices, n_compact: int, num_threads: int | None = None):
    """Adjoint of scatter_rows (ops.py:102-107): duplicated originals summed into their
    compact representative, ascending-i accumulation."""
    return gather_rows_backward(grad_out, scatter_indices, n_compact, num_threads=num_threads)
