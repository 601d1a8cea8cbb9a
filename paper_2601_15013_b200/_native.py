"""ctypes binding of the sm_100a C-ABI library (include/radix_b200.h).

The library is built in-tree (``python -m paper_2601_15013_b200.build`` or
``__graft_entry__.build()``) into ``paper_2601_15013_b200/_rdx.so``.  There is
no fallback: :func:`lib` raises :class:`NativeLibraryError` when the shared
object is missing or no CUDA device is visible, and every call's status code
is turned into the reference exception of the same name.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import NativeLibraryError, raise_for_status

SO_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_rdx.so")
# Developer experiments only: RDX_LIB_VARIANT=<tag> loads the in-tree _rdx_<tag>.so
# built by build_library(variant=<tag>) (same sources, extra compile flags).
if os.environ.get("RDX_LIB_VARIANT"):
    SO_PATH = os.path.join(os.path.dirname(SO_PATH), f"_rdx_{os.environ['RDX_LIB_VARIANT']}.so")

# Every symbol include/radix_b200.h declares (tests check the export list).
EXPORTS = (
    "rdx_version",
    "rdx_status_name",
    "rdx_last_cuda_error",
    "rdx_plan_scratch_bytes",
    "rdx_plan_build",
    "rdx_plan_debug_smem",
    "rdx_plan_debug_trace",
    "rdx_gather_rows",
    "rdx_gather_rows_backward_scratch_bytes",
    "rdx_gather_rows_backward",
    "rdx_embed_rmsnorm",
    "rdx_embed_rows",
    "rdx_rmsnorm_rows",
    "rdx_rmsnorm_rows_after",
    "rdx_device_status",
    "rdx_stream_synchronize",
    "rdx_rope_table",
    "rdx_rope_table_blocked",
    "rdx_gemm",
    "rdx_gemm_pair",
    "rdx_gemm_debug_pair",
    "rdx_gemm_debug_tail_split",
    "rdx_gemm_debug_colpart",
    "rdx_norm_debug_times",
    "rdx_norm_debug_warps",
    "rdx_norm_debug_backoff",
    "rdx_gemm_debug_stats",
    "rdx_gemm_debug_shape",
    "rdx_gemm_debug_group_m",
    "rdx_debug_pdl",
    "rdx_attention",
    "rdx_attention_debug_bk64",
    "rdx_attention_debug_split",
    "rdx_attention_debug_stats",
    "rdx_attention_debug_trace",
    "rdx_attention_debug_cta_times",
    "rdx_gemm_debug_group_m_bigk",
    "rdx_rerank_scores",
    "rdx_transpose_f32_bf16",
    "rdx_num_sms",
)

RDX_PLAN_ALLOW_EMPTY = 0x1
RDX_DTYPE_F32 = 0
RDX_DTYPE_F64 = 1

EPI_STORE_BF16 = 0
EPI_STORE_F32 = 1
EPI_RESID_F32 = 2
EPI_SWIGLU = 3
EPI_QKV = 4
EPI_RESID_NORM = 5

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_u32 = ctypes.c_uint32
_f32 = ctypes.c_float
_f64 = ctypes.c_double


class GemmArgs(ctypes.Structure):
    """Mirror of ``rdx_gemm_args``."""

    _fields_ = [
        ("a", _vp),
        ("b", _vp),
        ("m", _i64),
        ("n", _i64),
        ("k", _i64),
        ("lda", _i64),
        ("ldb", _i64),
        ("epi", _i32),
        ("block_n", _i32),
        ("out", _vp),
        ("ldo", _i64),
        ("q_norm_w", _vp),
        ("k_norm_w", _vp),
        ("rope_table", _vp),
        ("head_dim", _i32),
        ("q_heads", _i32),
        ("kv_heads", _i32),
        ("eps", _f32),
        ("row_ss", _vp),
        ("ss_parts", _i32),
        ("norm_dim", _i32),
        ("norm_eps", _f32),
        ("out_bf16", _vp),
        ("ldo_bf16", _i64),
        ("ss_out", _vp),
        ("rope_blocked", _i32),
        ("rope_pos", _vp),
        ("rope_theta", _f64),
        ("done_ctr", _vp),
        ("a_ready", _vp),
        ("a_ready_use", _u32),
    ]


_SIGNATURES = {
    "rdx_version": (ctypes.c_int, []),
    "rdx_status_name": (ctypes.c_char_p, [ctypes.c_int]),
    "rdx_last_cuda_error": (ctypes.c_char_p, []),
    "rdx_plan_scratch_bytes": (ctypes.c_size_t, [_i64, _i64]),
    "rdx_plan_build": (
        ctypes.c_int,
        [_vp, _vp, _vp, _i64, _i64, _u32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp],
    ),
    "rdx_gather_rows": (ctypes.c_int, [_vp, _i64, _i64, _vp, _i64, _vp, _i64, _i64, _vp, _vp]),
    "rdx_gather_rows_backward_scratch_bytes": (ctypes.c_size_t, [_i64, _i64]),
    "rdx_gather_rows_backward": (ctypes.c_int, [_vp, _i64, _vp, _i64, _i64, _vp, _i64, _i64, _i32, _vp, _vp,
                                                ctypes.c_size_t, _vp]),
    "rdx_embed_rmsnorm": (
        ctypes.c_int,
        [_vp, _vp, _i64, _vp, _i64, _i64, _vp, _f32, _vp, _vp, _vp, _vp],
    ),
    "rdx_embed_rows": (ctypes.c_int, [_vp, _vp, _i64, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp]),
    "rdx_rmsnorm_rows": (ctypes.c_int, [_vp, _i64, _vp, _i64, _i64, _vp, _f32, _vp, _i64, _vp]),
    "rdx_device_status": (ctypes.c_int, [_vp]),
    "rdx_stream_synchronize": (ctypes.c_int, [_vp]),
    "rdx_rmsnorm_rows_after": (ctypes.c_int, [_vp, _i64, _i64, _i64, _vp, _f32, _vp, _i64, _vp, _u32, _vp, _vp]),
    "rdx_rope_table": (ctypes.c_int, [_vp, _i64, _i32, _f64, _vp, _vp]),
    "rdx_rope_table_blocked": (ctypes.c_int, [_vp, _i64, _i32, _f64, _vp, _vp]),
    "rdx_gemm": (ctypes.c_int, [ctypes.POINTER(GemmArgs), _vp]),
    "rdx_gemm_pair": (ctypes.c_int, [ctypes.POINTER(GemmArgs), ctypes.POINTER(GemmArgs), _vp, _vp]),
    "rdx_gemm_debug_tail_split": (ctypes.c_int, [ctypes.c_int]),
    "rdx_gemm_debug_colpart": (ctypes.c_int, [ctypes.c_int]),
    "rdx_norm_debug_times": (ctypes.c_int, [_vp, ctypes.c_int]),
    "rdx_norm_debug_warps": (ctypes.c_int, [ctypes.c_int]),
    "rdx_norm_debug_backoff": (ctypes.c_int, [ctypes.c_uint]),
    "rdx_gemm_debug_pair": (ctypes.c_int, [ctypes.c_int]),
    "rdx_plan_debug_smem": (ctypes.c_int, [ctypes.c_int]),
    "rdx_attention_debug_bk64": (ctypes.c_int, [ctypes.c_int]),
    "rdx_attention_debug_split": (ctypes.c_int, [ctypes.c_int]),
    "rdx_plan_debug_trace": (ctypes.c_int, [_vp]),
    "rdx_gemm_debug_stats": (ctypes.c_int, [_vp, ctypes.c_int]),
    "rdx_gemm_debug_shape": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "rdx_gemm_debug_group_m": (ctypes.c_int, [ctypes.c_int]),
    "rdx_debug_pdl": (ctypes.c_int, [ctypes.c_int]),
    "rdx_rerank_scores": (ctypes.c_int, [_vp, _i64, _i64, _i64, _i64, _vp, _vp]),
    "rdx_transpose_f32_bf16": (ctypes.c_int, [_vp, _i64, _i64, _i64, _vp, _i64, _vp]),
    "rdx_attention": (ctypes.c_int, [_vp, _i64, _i64, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _i32, _i32, _f32, _vp, _i64,
                                      _vp]),
    "rdx_attention_debug_stats": (ctypes.c_int, [_vp, _i32]),
    "rdx_attention_debug_trace": (ctypes.c_int, [_vp, _i32]),
    "rdx_attention_debug_cta_times": (ctypes.c_int, [_vp, _i32]),
    "rdx_gemm_debug_group_m_bigk": (ctypes.c_int, [_i32]),
    "rdx_num_sms": (ctypes.c_int, []),
}

_lock = threading.Lock()
_lib = None


def load_library(path: str = SO_PATH) -> ctypes.CDLL:
    """dlopen the library and bind signatures (no device needed)."""
    if not os.path.exists(path):
        raise NativeLibraryError(
            f"sm_100a library not built: {path} missing (run __graft_entry__.build())"
        )
    handle = ctypes.CDLL(path)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    return handle


def lib() -> ctypes.CDLL:
    """The loaded library; requires a visible CUDA device (no CPU fallback)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                import torch

                if not torch.cuda.is_available():
                    raise NativeLibraryError("no CUDA device: the RadixMLP hot path runs on sm_100a only")
                _lib = load_library()
    return _lib


class _Counter:
    """C-ABI calls that reached the device (each launches one kernel); bench.py reads it."""

    launches = 0


LAUNCHES = _Counter()


def check(code: int, what: str) -> None:
    """Raise the mapped exception for a non-zero status; count successful launches."""
    if code == 0:
        LAUNCHES.launches += 1
    if code:
        detail = ""
        if code == 100:
            detail = (lib().rdx_last_cuda_error() or b"").decode()
        raise_for_status(code, what, detail)


def check_device_status(stream=None) -> None:
    """Raise if an asynchronous device-side contract failed since the last check
    (rdx_device_status; synchronises the stream)."""
    check_status = lib().rdx_device_status(stream_handle(stream))
    if check_status:
        raise_for_status(check_status, "device status")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch

    if stream is not None:
        return stream.cuda_stream
    # the current stream's raw handle without building a torch.cuda.Stream object (~4 us less)
    return torch._C._cuda_getCurrentRawStream(torch.cuda.current_device())
