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
