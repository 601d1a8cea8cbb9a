"""Compaction plans: the GPU prefix-trie planner behind the reference API.

Python surface mirrors pkg/src/radix_compact/trie.py:36-233:
``CompactionPlan``, ``build_plan``, ``build_plan_fast_paths``,
``build_plan_auto``, ``should_enable`` and ``pad_plan`` keep their names,
argument meaning, outputs and exceptions.  The index computation itself runs
on the GPU (csrc/plan_build.cu, ``rdx_plan_build``), bit-exact to the
reference's trie; there is no CPU planner in this package.

``build_plan_device`` is the hot-path entry: device-resident inputs in,
device-resident :class:`DevicePlan` out, with a single small D2H read of
(N', status, cu_q) so the host can size the compact buffers.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from . import _native
from .errors import CapacityExceeded, EmptyPlan, NativeLibraryError, raise_for_status
from .ragged import RaggedBatch, validate_batch


@dataclass(frozen=True)
class CompactionPlan:
    """Host copy of a plan; same fields and properties as trie.py:36-70."""

    gather_indices: np.ndarray
    scatter_indices: np.ndarray
    compact_positions: np.ndarray
    n_original: int
    n_compact: int

    def __post_init__(self):
        for name in ("gather_indices", "scatter_indices", "compact_positions"):
            arr = np.ascontiguousarray(getattr(self, name), dtype=np.uint32)
            arr.flags.writeable = False
            object.__setattr__(self, name, arr)

    @property
    def n_padded(self) -> int:
        return int(self.gather_indices.shape[0])

    @property
    def gamma(self) -> float:
        return self.n_compact / self.n_original if self.n_original else 1.0

    @property
    def gamma_exact(self) -> Fraction:
        return Fraction(self.n_compact, self.n_original) if self.n_original else Fraction(1)


@dataclass
class DevicePlan:
    """Device-resident plan produced by :func:`build_plan_device`.

    ``gather`` / ``compact_positions`` have exactly ``n_compact`` rows,
    ``scatter`` has ``n_original``; all int32 views of the u32 maps.
    ``cu_q`` (device, int32 [B+1]) delimits each sequence's compact suffix
    (finding 2 of SURVEY.md: compact rows of sequence s are the contiguous
    range [cu_q[s], cu_q[s+1]) ); ``cu_q_host`` is its host copy, read on first
    use (the planner returns N', the status and max_q without copying cu_q).
    """

    gather: "object"
    scatter: "object"
    compact_positions: "object"
    cu_q: "object"
    lcp: "object"
    n_original: int
    n_compact: int
    attempts: int = 1
    max_q: int = -1  # longest compact suffix (rows of one sequence), from the planner
    extras: dict = field(default_factory=dict)
    _cu_q_host: object = field(default=None, repr=False)

    @property
    def cu_q_host(self) -> np.ndarray:
        if self._cu_q_host is None:
            self._cu_q_host = self.cu_q.cpu().numpy().astype(np.int64)
        return self._cu_q_host

    @property
    def n_padded(self) -> int:
        return int(self.gather.shape[0])

    @property
    def gamma(self) -> float:
        return self.n_compact / self.n_original if self.n_original else 1.0

    @property
    def max_q_len(self) -> int:
        if self.max_q >= 0:
            return self.max_q
        return int(np.diff(self.cu_q_host).max()) if self.cu_q_host.size > 1 else 0

    def to_host(self) -> CompactionPlan:
        return CompactionPlan(
            gather_indices=self.gather.cpu().numpy().view(np.uint32),
            scatter_indices=self.scatter.cpu().numpy().view(np.uint32),
            compact_positions=self.compact_positions.cpu().numpy().view(np.uint32),
            n_original=self.n_original,
            n_compact=self.n_compact,
        )


class _Workspace:
    """Grow-only per-device scratch arena for the planner."""

    def __init__(self):
        self._buf = {}
        self._lock = threading.Lock()

    def get(self, device, nbytes: int):
        import torch

        key = str(device)
        with self._lock:
            buf = self._buf.get(key)
            if buf is None or buf.numel() < nbytes:
                buf = torch.empty(max(nbytes, 1 << 16), dtype=torch.uint8, device=device)
                self._buf[key] = buf
            return buf


_WORKSPACE = _Workspace()


_PINNED = threading.local()


_SCRATCH_BYTES: dict = {}


def _info_buffer():
    """Thread-local pinned 4-word buffer (tensor, numpy view) the planner kernel writes
    (N', status, attempts, max_q) into directly: host memory allocated by cudaHostAlloc is
    device-addressable under unified addressing, so no device-to-host copy is queued."""
    import torch

    buf = getattr(_PINNED, "info", None)
    if buf is None:
        t = torch.zeros(4, dtype=torch.int32, pin_memory=True)
        buf = (t, t.numpy())
        _PINNED.info = buf
    return buf


def build_plan_device(tok, pos, cu, *, allow_empty: bool = False, stream=None,
                      n_original: int | None = None) -> DevicePlan:
    """GPU planner on device tensors (tok/pos int32-viewed u32 [N], cu int64 [B+1]).

    One kernel computes gather/scatter/compact_positions/cu_q and writes
    (N', status, attempts, max_q) straight into pinned host memory; the call
    returns after one stream synchronisation.
    """
    import torch

    lib = _native.lib()
    dev = tok.device
    n = int(tok.shape[0]) if n_original is None else int(n_original)
    b = int(cu.shape[0]) - 1
    if n >= (1 << 32) - 1:
        raise CapacityExceeded(f"{n} tokens exceed 32-bit index range")
    # one allocation for every output: gather | scatter | compact_positions | cu_q | lcp
    nn, nb = max(n, 1), max(b, 1)
    buf = torch.empty(3 * nn + (b + 1) + nb, dtype=torch.int32, device=dev)
    o = 3 * nn
    key = (n, b)
    sb = _SCRATCH_BYTES.get(key)
    if sb is None:
        sb = _SCRATCH_BYTES[key] = int(lib.rdx_plan_scratch_bytes(n, b))
    scratch = _WORKSPACE.get(dev, sb)
    flags = _native.RDX_PLAN_ALLOW_EMPTY if allow_empty else 0
    sh = (stream.cuda_stream if stream is not None else
          torch._C._cuda_getCurrentRawStream(dev.index if dev.index is not None else torch.cuda.current_device()))
    info, iv = _info_buffer()
    iv[1] = -1  # status sentinel: a kernel that never ran cannot leave a stale RDX_OK behind
    p0 = buf.data_ptr()
    code = lib.rdx_plan_build(
        tok.data_ptr(), pos.data_ptr(), cu.data_ptr(), b, n, flags,
        p0, p0 + 4 * nn, p0 + 8 * nn, p0 + 4 * o, p0 + 4 * (o + b + 1), info.data_ptr(),
        scratch.data_ptr(), ctypes.c_size_t(scratch.numel()), sh,
    )
    _native.check(code, "rdx_plan_build")
    # the one host wait (GIL released in the ctypes call): (N', status, attempts, max_q) are in `info`
    _native.check(lib.rdx_stream_synchronize(sh), "rdx_stream_synchronize")
    n_compact, status, attempts, max_q = (int(x) for x in iv)
    if status == -1:
        raise NativeLibraryError("rdx_plan_build: the planner kernel did not report a status")
    raise_for_status(status, "rdx_plan_build")
    # every view in one call (five separate slices cost ~13 us of host time at C2)
    gather, _, scatter, _, cpos, _, cu_q, lcp = buf.split(
        [n_compact, nn - n_compact, n, nn - n, n_compact, nn - n_compact, b + 1, nb])
    return DevicePlan(
        gather=gather,
        scatter=scatter,
        compact_positions=cpos,
        cu_q=cu_q,
        lcp=lcp if b else lcp[:0],
        n_original=n,
        n_compact=n_compact,
        attempts=attempts,
        max_q=max_q,
    )


def upload_batch(batch: RaggedBatch, device="cuda"):
    """Host batch -> (tok, pos, cu) device tensors (u32 stored as int32)."""
    import torch

    _native.lib()  # fail loudly (NativeLibraryError) before touching CUDA
    tok = torch.from_numpy(np.array(batch.token_ids, dtype=np.uint32).view(np.int32))
    pos = torch.from_numpy(np.array(batch.position_ids, dtype=np.uint32).view(np.int32))
    cu = torch.from_numpy(np.array(batch.cu_seqlens, dtype=np.int64))
    return tok.to(device), pos.to(device), cu.to(device)


def build_plan(batch: RaggedBatch, allow_empty: bool = False) -> CompactionPlan:
    """Reference ``build_plan`` (trie.py:125-148), computed on the GPU."""
    validate_batch(batch, allow_empty=allow_empty)
    n = batch.num_tokens
    if n >= 2**32:
        raise CapacityExceeded(f"{n} tokens exceed 32-bit index range")
    if n == 0:
        z = np.zeros(0, np.uint32)
        return CompactionPlan(z, z, z, 0, 0)
    tok, pos, cu = upload_batch(batch)
    return build_plan_device(tok, pos, cu, allow_empty=allow_empty).to_host()


def build_plan_fast_paths(batch: RaggedBatch) -> CompactionPlan | None:
    """Reference fast paths (trie.py:151-188): B == 1 or all-identical batches.

    Returns None when neither applies.  The GPU planner produces the same
    identity / tiled plan for those batches, so the plan is built there.
    """
    validate_batch(batch)
    b, n = batch.num_sequences, batch.num_tokens
    if b == 1:
        return build_plan(batch)
    if b > 1:
        lengths = batch.seq_lengths()
        length = int(lengths[0])
        if np.all(lengths == length):
            t = batch.token_ids.reshape(b, length)
            p = batch.position_ids.reshape(b, length)
            if np.all(t == t[0]) and np.all(p == p[0]):
                return build_plan(batch)
    del n
    return None


def build_plan_auto(batch: RaggedBatch) -> CompactionPlan:
    """Reference ``build_plan_auto`` (trie.py:191-194): one GPU build covers all cases."""
    return build_plan(batch)


def should_enable(plan, threshold) -> bool:
    """gamma <= threshold, inclusive, exact rational (trie.py:197-203)."""
    n, m = int(plan.n_original), int(plan.n_compact)
    gamma = Fraction(m, n) if n else Fraction(1)
    return gamma <= Fraction(threshold).limit_denominator(10**9)


def pad_plan(plan: CompactionPlan, bucket_size: int) -> CompactionPlan:
    """Pad N' to a multiple of bucket_size by repeating row 0 (trie.py:206-233)."""
    if bucket_size < 1:
        raise ValueError("bucket_size must be >= 1")
    if plan.n_compact == 0:
        raise EmptyPlan("cannot pad a plan with zero compact tokens")
    target = -(-plan.n_compact // bucket_size) * bucket_size
    if target == plan.n_padded:
        return plan
    extra = target - plan.n_compact
    g = plan.gather_indices[: plan.n_compact]
    p = plan.compact_positions[: plan.n_compact]
    return CompactionPlan(
        gather_indices=np.concatenate([g, np.repeat(g[:1], extra)]),
        scatter_indices=plan.scatter_indices,
        compact_positions=np.concatenate([p, np.repeat(p[:1], extra)]),
        n_original=plan.n_original,
        n_compact=plan.n_compact,
    )


def host_plan_cu_q(plan: CompactionPlan, cu_seqlens) -> np.ndarray | None:
    """cu_q of a host plan if it has the per-sequence-suffix structure, else None.

    Plans from build_plan always have it (compact rows of sequence s are
    [cu[s] + lcp_s, cu[s+1]) in order); hand-made plans may not.
    """
    cu = np.asarray(cu_seqlens, dtype=np.int64)
    n, m = plan.n_original, plan.n_compact
    g = plan.gather_indices[:m].astype(np.int64)
    s = plan.scatter_indices.astype(np.int64)
    if n == 0:
        return np.zeros(cu.shape[0], dtype=np.int64)
    if s.size != n or (m and (g.max() >= n or s.max() >= m)):
        return None
    is_rep = g[s] == np.arange(n)
    csum = np.concatenate([[0], np.cumsum(is_rep.astype(np.int64))])
    counts = csum[cu[1:]] - csum[cu[:-1]]
    cu_q = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    if cu_q[-1] != m:
        return None
    lcp = np.diff(cu) - counts
    expect = np.concatenate([np.arange(cu[i] + lcp[i], cu[i + 1]) for i in range(cu.shape[0] - 1)]) \
        if cu.shape[0] > 1 else np.zeros(0, np.int64)
    if expect.shape[0] != m or not np.array_equal(expect, g):
        return None
    return cu_q
