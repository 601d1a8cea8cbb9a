"""B200-native RadixMLP hot path (arxiv 2601.15013), drop-in for radix_compact.

Re-exports the reference's hot-path API (pkg/src/radix_compact/__init__.py:8-95)
with the index build, row operators and the Qwen3 prefill running as sm_100a
kernels behind a C ABI (include/radix_b200.h).  Importing the package needs no
GPU; calling a hot-path function without a CUDA device or without the built
library raises NativeLibraryError (there is no CPU fallback).
"""

from .errors import (
    BoundaryMismatch,
    CapacityExceeded,
    EmptyPlan,
    HashRetriesExhausted,
    IndexOutOfRange,
    MismatchedLengths,
    NativeLibraryError,
    NonMonotoneOffsets,
    OddHeadDim,
    OverflowId,
    PlanBatchMismatch,
    RadixCompactError,
    ShapeMismatch,
)
from .model import (
    QWEN3_PRESETS,
    TINY_C1,
    DeviceBatch,
    DeviceWeights,
    FlopLedger,
    ModelConfig,
    Qwen3Config,
    RadixQwen3,
    forward,
    forward_scores,
    init_params,
)
from .ops import (gather_rows, gather_rows_backward, gather_rows_backward_device, gather_rows_device, scatter_rows,
                  scatter_rows_backward)
from .pipeline import PipelineReport, pipelined_run, score_stream
from .primitives import apply_rope, attention_ragged, rmsnorm, swiglu_mlp
from .training import loss_and_grads
from .plan import (
    CompactionPlan,
    DevicePlan,
    build_plan,
    build_plan_auto,
    build_plan_device,
    build_plan_fast_paths,
    pad_plan,
    should_enable,
)
from .ragged import (
    BatchStats,
    RaggedBatch,
    batch_from_json,
    batch_to_json,
    default_positions,
    validate_batch,
)
from .serialization import load_plan, plan_from_bytes, plan_from_json, plan_to_bytes, plan_to_json, save_plan

__version__ = "0.1.0"

__all__ = [
    "BatchStats", "BoundaryMismatch", "CapacityExceeded", "CompactionPlan", "DeviceBatch", "DevicePlan",
    "DeviceWeights", "EmptyPlan", "FlopLedger", "HashRetriesExhausted", "IndexOutOfRange",
    "MismatchedLengths", "ModelConfig", "NativeLibraryError", "NonMonotoneOffsets", "OddHeadDim",
    "OverflowId", "PlanBatchMismatch", "QWEN3_PRESETS", "Qwen3Config", "RadixCompactError", "RadixQwen3",
    "RaggedBatch", "ShapeMismatch", "TINY_C1", "batch_from_json", "batch_to_json", "build_plan",
    "build_plan_auto", "build_plan_device", "build_plan_fast_paths", "default_positions", "forward",
    "forward_scores", "loss_and_grads", "apply_rope", "attention_ragged", "rmsnorm", "swiglu_mlp", "pipelined_run", "PipelineReport", "score_stream", "gather_rows", "gather_rows_backward", "gather_rows_backward_device", "gather_rows_device", "init_params", "load_plan", "pad_plan",
    "plan_from_bytes", "plan_from_json", "plan_to_bytes", "plan_to_json", "save_plan", "scatter_rows", "scatter_rows_backward",
    "should_enable", "validate_batch",
]
