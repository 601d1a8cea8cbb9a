"""RadixMLP-wrapped Qwen3 prefill on B200 (reference: pkg/src/radix_compact/model.py).

Algorithm 1 of the paper as the reference's
``_forward_cached`` runs it (model.py:322-416): every position-wise stage
(embedding, RMSNorms, Q/K/V/O projections, q/k norm + RoPE, SwiGLU MLP,
residuals, LM head) runs on the N' compact rows; only attention sees the
original ragged layout.  Here each stage is an sm_100a kernel behind the C ABI
(include/radix_b200.h):

  embed + ln1          rdx_embed_rmsnorm       (gathers tok[gather[j]])
  QKV + q/k-norm+RoPE  rdx_gemm EPI_QKV        (tcgen05, fused epilogue)
  attention boundary   rdx_attention           (tcgen05; K/V read through the
                                                scatter map, Q/O stay compact)
  O-proj + residual    rdx_gemm EPI_RESID_F32  (TMA reduce-add into h)
  ln2                  rdx_rmsnorm_rows
  gate|up + SiLU*mul   rdx_gemm EPI_SWIGLU
  down + residual      rdx_gemm EPI_RESID_F32
  final norm + head    rdx_rmsnorm_rows (+ last-token row select) + rdx_gemm

Attention boundary modes:
  ``attention="full"``   exactly the reference: scatter Q/K/V to N rows
                         (rdx_gather_rows), attention over the original
                         layout, gather N -> N' (model.py:368-383).
  ``attention="suffix"`` (default) SURVEY §8f-1: compact rows of sequence s
                         are its suffix [lcp_s, L_s), so Q stays compact
                         (cu_seqlens_q = cu_q), K/V are read in place through
                         the scatter map and the causal mask is bottom-right
                         aligned.  Mathematically identical; no row copies.

Numerics: weights/activations bf16, fp32 accumulation (TMEM), fp32 residual
stream and norm statistics.  Parity vs the fp64 reference is a tolerance
(tests/test_model_gpu.py), dedup-on vs dedup-off differs only through the
attention kernel's row blocking.

Scoring contract (no reference counterpart; SURVEY finding 5): full-vocab
logits for all N rows are infeasible at Qwen3 scale, so ``logits="last"``
returns the last-token logits [B, vocab] of each sequence (the reranker
read-out); ``logits="all"`` returns the reference's [N, vocab].
"""

from __future__ import annotations

import math
import os
from collections import OrderedDict
from dataclasses import dataclass, fields

import numpy as np

from . import _native
from .errors import NativeLibraryError, OddHeadDim, PlanBatchMismatch, ShapeMismatch
from .ops import gather_rows_device
from .plan import CompactionPlan, DevicePlan, build_plan_device, host_plan_cu_q, upload_batch
from .ragged import RaggedBatch, validate_batch

SWIGLU_UNIT = 64  # gate/up interleave unit of the SwiGLU epilogue (csrc/gemm.cu)


@dataclass(frozen=True)
class ModelConfig:
    """Hyper-parameters (model.py:31-67), same fields and validation."""

    num_layers: int = 2
    hidden_size: int = 256
    intermediate_size: int = 512
    num_heads: int = 4
    num_kv_heads: int = 2
    head_dim: int = 64
    vocab_size: int = 128
    rope_theta: float = 10000.0
    norm_eps: float = 1e-6

    def __post_init__(self):
        if self.hidden_size != self.num_heads * self.head_dim:
            raise ShapeMismatch("hidden_size must equal num_heads * head_dim")
        self._check_common()

    def _check_common(self):
        if self.num_kv_heads < 1 or self.num_heads % self.num_kv_heads:
            raise ShapeMismatch("num_heads must be divisible by num_kv_heads")
        for name in ("num_layers", "hidden_size", "intermediate_size", "vocab_size"):
            if getattr(self, name) < 1:
                raise ShapeMismatch(f"{name} must be >= 1")

    @property
    def q_dim(self) -> int:
        return self.num_heads * self.head_dim

    @property
    def kv_dim(self) -> int:
        return self.num_kv_heads * self.head_dim

    def to_json(self) -> dict:
        return {f.name: getattr(self, f.name) for f in fields(self)}


@dataclass(frozen=True)
class Qwen3Config(ModelConfig):
    """ModelConfig that admits q_dim != hidden (real Qwen3 head layouts).

    The reference's check (model.py:44-45) rejects Qwen3-0.6B/4B/8B although
    the rest of its model already handles q_dim != hidden (SURVEY finding 3).
    """

    def __post_init__(self):
        self._check_common()


# Public HF config.json values (SURVEY §8 notation), random-init only.
QWEN3_PRESETS = {
    "qwen3-0.6b": Qwen3Config(28, 1024, 3072, 16, 8, 128, 151936, 1e6, 1e-6),
    "qwen3-4b": Qwen3Config(36, 2560, 9728, 32, 8, 128, 151936, 1e6, 1e-6),
    "qwen3-8b": Qwen3Config(36, 4096, 12288, 32, 8, 128, 151936, 1e6, 1e-6),
}
# C1 of BASELINE.json: 2 layers, d=64, 4 heads
TINY_C1 = Qwen3Config(2, 64, 192, 4, 2, 16, 1024, 10000.0, 1e-6)


class FlopLedger:
    """Row counters per stage (model.py:70-91), same fields and methods."""

    def __init__(self):
        self.positionwise_row_ops = 0
        self.attention_row_ops = 0
        self.gather_scatter_rows = 0
        self.phases: list[tuple[str, int]] = []

    def positionwise(self, name: str, rows: int) -> None:
        self.positionwise_row_ops += rows
        self.phases.append((name, rows))

    def attention(self, rows: int) -> None:
        self.attention_row_ops += rows

    def index_copy(self, rows: int) -> None:
        self.gather_scatter_rows += rows


def init_params(config: ModelConfig, seed: int = 0, dtype=np.float64) -> dict:
    """Seeded uniform[-0.05, 0.05] init, norms = 1 (model.py:94-119).

    Same parameter names, shapes ([out, in]) and RNG draw order as the
    reference, so the oracle and the GPU model see identical weights.
    """
    rng = np.random.default_rng(seed)
    d, di = config.hidden_size, config.intermediate_size

    def u(*shape):
        return rng.uniform(-0.05, 0.05, size=shape).astype(dtype)

    p = {"embed": u(config.vocab_size, d)}
    for i in range(config.num_layers):
        pre = f"layers.{i}."
        p[pre + "ln1"] = np.ones(d, dtype=dtype)
        p[pre + "wq"] = u(config.q_dim, d)
        p[pre + "wk"] = u(config.kv_dim, d)
        p[pre + "wv"] = u(config.kv_dim, d)
        p[pre + "wo"] = u(d, config.q_dim)
        p[pre + "q_norm"] = np.ones(config.head_dim, dtype=dtype)
        p[pre + "k_norm"] = np.ones(config.head_dim, dtype=dtype)
        p[pre + "ln2"] = np.ones(d, dtype=dtype)
        p[pre + "w_gate"] = u(di, d)
        p[pre + "w_up"] = u(di, d)
        p[pre + "w_down"] = u(d, di)
    p["final_norm"] = np.ones(d, dtype=dtype)
    p["lm_head"] = u(config.vocab_size, d)
    return p


def padded_intermediate(config: ModelConfig) -> int:
    return -(-config.intermediate_size // SWIGLU_UNIT) * SWIGLU_UNIT


def _check_kernel_shapes(config: ModelConfig) -> None:
    hd = config.head_dim
    if hd % 2:
        raise OddHeadDim(f"head_dim {hd} is odd")
    if hd % 16 or hd > 128:
        raise ShapeMismatch(f"head_dim {hd}: the fused QKV epilogue needs a multiple of 16, <= 128")
    if config.hidden_size % 8:
        raise ShapeMismatch("hidden_size must be a multiple of 8 (16-byte TMA rows)")


class DeviceWeights:
    """Kernel-ready weights on one GPU.

    w_qkv  bf16 [q+2kv, d]  (wq | wk | wv stacked, model.py:352-354)
    w_gu   bf16 [2*di_pad, d] gate/up rows interleaved in units of 64 so each
           GEMM tile holds matching gate and up columns (EPI_SWIGLU)
    w_down bf16 [d, di_pad] zero-padded columns
    norms  fp32
    """

    def __init__(self, config: ModelConfig, tensors: dict):
        self.config = config
        self.t = tensors

    @staticmethod
    def _interleave_gate_up(gate, up, di_pad):
        import torch

        d = gate.shape[1]
        pad = di_pad - gate.shape[0]
        if pad:
            z = torch.zeros(pad, d, dtype=gate.dtype, device=gate.device)
            gate, up = torch.cat([gate, z]), torch.cat([up, z])
        g = gate.view(di_pad // SWIGLU_UNIT, 1, SWIGLU_UNIT, d)
        u = up.view(di_pad // SWIGLU_UNIT, 1, SWIGLU_UNIT, d)
        return torch.cat([g, u], dim=1).reshape(2 * di_pad, d).contiguous()

    @classmethod
    def from_tensors(cls, config: ModelConfig, get, device="cuda"):
        """Build from a callable name -> torch tensor (any float dtype, any device)."""
        import torch

        _check_kernel_shapes(config)
        bf, f32 = torch.bfloat16, torch.float32
        di_pad = padded_intermediate(config)

        def dev(name, dtype):
            return get(name).to(device=device, dtype=dtype).contiguous()

        t = {"embed": dev("embed", bf), "final_norm": dev("final_norm", f32), "lm_head": dev("lm_head", bf)}
        for i in range(config.num_layers):
            pre = f"layers.{i}."
            t[pre + "w_qkv"] = torch.cat(
                [dev(pre + "wq", bf), dev(pre + "wk", bf), dev(pre + "wv", bf)]).contiguous()
            t[pre + "wo"] = dev(pre + "wo", bf)
            t[pre + "w_gu"] = cls._interleave_gate_up(dev(pre + "w_gate", bf), dev(pre + "w_up", bf), di_pad)
            wd = dev(pre + "w_down", bf)
            if di_pad != config.intermediate_size:
                wd = torch.cat([wd, torch.zeros(wd.shape[0], di_pad - wd.shape[1], dtype=bf, device=device)],
                               dim=1).contiguous()
            t[pre + "w_down"] = wd
            for nm in ("ln1", "ln2", "q_norm", "k_norm"):
                t[pre + nm] = dev(pre + nm, f32)
        return cls(config, t)

    def fold_norms(self) -> None:
        """w_qkv_n = w_qkv * ln1, w_gu_n = w_gu * ln2 (per input column), bf16; idempotent.

        RMSNorm(x) W^T = rstd(x) * (x (W diag(w))^T): the weight half of the norm
        moves into the GEMM operand, the row scale into the GEMM epilogue.
        """
        import torch

        for i in range(self.config.num_layers):
            pre = f"layers.{i}."
            for wname, nname in (("w_qkv", "ln1"), ("w_gu", "ln2")):
                key = pre + wname + "_n"
                if key not in self.t:
                    w = self.t[pre + wname].float() * self.t[pre + nname].float()[None, :]
                    self.t[key] = w.to(torch.bfloat16).contiguous()

    @classmethod
    def from_params(cls, config: ModelConfig, params: dict, device="cuda"):
        import torch

        return cls.from_tensors(config, lambda n: torch.from_numpy(np.ascontiguousarray(params[n])), device)

    @classmethod
    def random(cls, config: ModelConfig, seed: int = 0, device="cuda"):
        """On-device seeded uniform[-0.05, 0.05] init (norms = 1), for benchmarks."""
        import torch

        gen = torch.Generator(device=device)
        gen.manual_seed(seed)
        d, di = config.hidden_size, config.intermediate_size
        shapes = {"embed": (config.vocab_size, d), "lm_head": (config.vocab_size, d), "final_norm": (d,)}
        for i in range(config.num_layers):
            pre = f"layers.{i}."
            shapes.update({pre + "ln1": (d,), pre + "ln2": (d,), pre + "q_norm": (config.head_dim,),
                           pre + "k_norm": (config.head_dim,), pre + "wq": (config.q_dim, d),
                           pre + "wk": (config.kv_dim, d), pre + "wv": (config.kv_dim, d),
                           pre + "wo": (d, config.q_dim), pre + "w_gate": (di, d), pre + "w_up": (di, d),
                           pre + "w_down": (d, di)})

        def get(name):
            shape = shapes[name]
            if len(shape) == 1:
                return torch.ones(shape, dtype=torch.float32, device=device)
            w = torch.empty(shape, dtype=torch.float32, device=device)
            w.uniform_(-0.05, 0.05, generator=gen)
            return w

        return cls.from_tensors(config, get, device)


@dataclass
class DeviceBatch:
    """A ragged batch resident on the GPU (u32 ids stored as int32)."""

    tok: object
    pos: object
    cu: object        # int64 [B+1]
    cu32: object      # int32 [B+1] (attention kernel)
    cu_host: np.ndarray
    n: int
    b: int
    max_len: int
    max_token: int = -1  # host-known max token id (-1: unknown, checked on device)

    @classmethod
    def from_batch(cls, batch: RaggedBatch, device="cuda", non_blocking=False):
        import torch

        tok, pos, cu = upload_batch(batch, device)
        cu_host = np.asarray(batch.cu_seqlens, dtype=np.int64)
        lens = np.diff(cu_host)
        mt = int(batch.token_ids.max()) if batch.num_tokens else -1
        return cls(tok, pos, cu, cu.to(torch.int32), cu_host, int(batch.num_tokens),
                   int(batch.num_sequences), int(lens.max()) if lens.size else 0, mt)


@dataclass
class _Layout:
    m: int                 # rows computed by position-wise stages
    n_compact: int
    gather: object         # int32 [m] or None (identity)
    scatter: object        # int32 [n] or None
    positions: object      # int32 [m]
    cu_q32: object         # int32 [B+1] compact-suffix offsets (suffix mode)
    max_q: int
    suffix_ok: bool
    dedup: bool
    cu_q_host: object = None  # host cu_q (np.ndarray) or the DevicePlan that reads it lazily


class _Graph:
    """One captured prefill body plus its static input buffers."""

    def __init__(self, graph, inputs: dict, output, err):
        self.graph = graph
        self.inputs = inputs
        self.output = output
        self.err = err


class RadixQwen3:
    """Qwen3 prefill whose position-wise work runs on the compact rows.

    ``prefill`` resolves the plan (GPU planner: one small D2H read for N'),
    then runs the layer stack.  With ``use_graphs=True`` the layer stack is
    captured into a CUDA graph per shape BUCKET and replayed, removing
    per-launch host overhead: N' is padded to a multiple of 256 rows the way
    ``pad_plan`` pads (repeating gather[0] / compact_positions[0]), the batch
    to a multiple of 16 sequences with empty ones, and the index buffers /
    attention grid to bucketed token counts and lengths.  All captures share
    one memory pool, at most ``max_graphs`` graphs are kept (least recently
    used evicted) and ``graph_captures`` counts captures.  A graph's output
    is valid until the next ``prefill`` call on the same model.
    """

    def __init__(self, config: ModelConfig, weights: DeviceWeights, use_graphs: bool = False,
                 fused_norm: bool | None = None, max_graphs: int = 8):
        _check_kernel_shapes(config)
        self.config = config
        self.w = weights
        self.di_pad = padded_intermediate(config)
        self.use_graphs = use_graphs
        # fused_norm: ln1/ln2 folded into the QKV / gate-up weights, row statistics from the
        # residual GEMM epilogue (RDX_EPI_RESID_NORM) -> no standalone rmsnorm passes.
        # Off by default: measured on B200 it does not beat the TMA reduce-add epilogue +
        # rmsnorm pass (C2 7.48-7.58 vs 7.66-7.68 ms, C4 551 vs 556 ms).
        self.fused_norm = False if fused_norm is None else fused_norm
        # rmsnorm passes overlap the residual GEMM's last round (RDX_NORM_OVERLAP=0: stream-ordered)
        self.norm_overlap = os.environ.get("RDX_NORM_OVERLAP", "1") != "0"
        # chained norm -> next GEMM on ready counters: correct (tests) but measured slower
        # (C2 -6.7 %, C3 -4.5 %), so off unless RDX_NORM_CHAIN=1
        self.norm_chain = os.environ.get("RDX_NORM_CHAIN", "0") == "1"
        # gate|up -> down as one persistent launch (rdx_gemm_pair); RDX_GEMM_PAIR=0: two launches
        self.mlp_pair = os.environ.get("RDX_GEMM_PAIR", "1") != "0"
        if self.fused_norm:
            if config.hidden_size % 64:
                raise ShapeMismatch("fused_norm needs hidden_size % 64 == 0")
            weights.fold_norms()
        self.op_hook = None  # optional callable(name, launch_fn, flops) (bench.py per-op CUDA events)
        self._graphs: OrderedDict = OrderedDict()  # bucket key -> _Graph, least recently used first
        self._graph_pool = None
        self.max_graphs = max_graphs
        self.graph_captures = 0

    # ------------------------------------------------------------ launches
    def _op(self, name, fn, flops=0.0):
        if self.op_hook is not None:
            return self.op_hook(name, fn, flops)
        return fn()

    def _gemm(self, name, a, w, epi, out, *, m, stream, qkv=False, rope=None, layer=None, row_ss=None,
              hb=None, ss_out=None, done=None, ready=None, build_only=False):
        cfg = self.config
        args = _native.GemmArgs()
        args.a = a.data_ptr()
        args.b = w.data_ptr()
        args.m = m
        args.n = w.shape[0]
        args.k = w.shape[1]
        args.lda = a.stride(0)
        args.ldb = w.stride(0)
        args.epi = epi
        args.block_n = 0
        args.out = out.data_ptr()
        args.ldo = out.stride(0)
        if qkv:
            args.q_norm_w = self.w.t[layer + "q_norm"].data_ptr()
            args.k_norm_w = self.w.t[layer + "k_norm"].data_ptr()
            if rope[0] == "pos":  # (cos, sin) computed in the epilogue from the row positions
                args.rope_pos = rope[1].data_ptr()
                args.rope_theta = float(cfg.rope_theta)
            else:  # lane-blocked fp64-derived table
                args.rope_table = rope[1].data_ptr()
                args.rope_blocked = 1
            args.head_dim = cfg.head_dim
            args.q_heads = cfg.num_heads
            args.kv_heads = cfg.num_kv_heads
            args.eps = cfg.norm_eps
        if done is not None:  # per-32-row-slab completion counter for rdx_rmsnorm_rows_after
            args.done_ctr = done.data_ptr()
        if ready is not None:  # chained A: (the norm's ready counters, use number)
            args.a_ready = ready[0].data_ptr()
            args.a_ready_use = ready[1]
        if row_ss is not None:  # RMSNorm of the A rows fused in (weight folded into w)
            args.row_ss = row_ss.data_ptr()
            args.ss_parts = row_ss.shape[1]
            args.norm_dim = cfg.hidden_size
            args.norm_eps = cfg.norm_eps
        if hb is not None:  # RDX_EPI_RESID_NORM outputs
            args.out_bf16 = hb.data_ptr()
            args.ldo_bf16 = hb.stride(0)
            args.ss_out = ss_out.data_ptr()
        if build_only:  # the caller launches it (rdx_gemm_pair)
            return args
        lib = _native.lib()

        def launch():
            _native.check(lib.rdx_gemm(args, stream), f"rdx_gemm[{name}]")

        self._op("gemm." + name, launch, 2.0 * m * args.n * args.k)

    def _gemm_pair(self, first, second, dep, stream):
        """gate|up and down in one persistent launch (rdx_gemm_pair, dep: zeroed slab counters)."""
        lib = _native.lib()

        def launch():
            _native.check(lib.rdx_gemm_pair(first, second, dep.data_ptr(), stream), "rdx_gemm_pair")

        self._op("gemm.mlp", launch, 2.0 * first.m * first.n * first.k + 2.0 * second.m * second.n * second.k)

    def _rmsnorm(self, x, w, out, rows=None, n_rows=None, stream=None):
        lib = _native.lib()
        n_rows = x.shape[0] if n_rows is None else n_rows

        def launch():
            code = lib.rdx_rmsnorm_rows(x.data_ptr(), x.stride(0), None if rows is None else rows.data_ptr(),
                                        n_rows, x.shape[1], w.data_ptr(), self.config.norm_eps,
                                        out.data_ptr(), out.stride(0), stream)
            _native.check(code, "rdx_rmsnorm_rows")

        self._op("rmsnorm", launch)

    def _rmsnorm_after(self, x, w, out, ctr, target, stream=None, ready=None):
        """rmsnorm overlapping the tail of the residual GEMM that feeds it (slab counters);
        with ``ready`` it publishes finished rows for a chained consumer GEMM."""
        lib = _native.lib()

        def launch():
            code = lib.rdx_rmsnorm_rows_after(x.data_ptr(), x.stride(0), x.shape[0], x.shape[1], w.data_ptr(),
                                              self.config.norm_eps, out.data_ptr(), out.stride(0), ctr.data_ptr(),
                                              target, None if ready is None else ready.data_ptr(), stream)
            _native.check(code, "rdx_rmsnorm_rows_after")

        self._op("rmsnorm", launch)

    def _gather(self, name, x, idx, stream_obj):
        return self._op(name, lambda: gather_rows_device(x, idx, stream=stream_obj))

    def _attn(self, qkv, scatter, cu32, cu_q32, b, max_q, max_k, out, flops, stream):
        """rdx_attention: Q compact rows, K/V read through ``scatter`` (None = plain layout)."""
        cfg = self.config
        lib = _native.lib()

        def launch():
            code = lib.rdx_attention(qkv.data_ptr(), qkv.stride(0), qkv.shape[0],
                                     None if scatter is None else scatter.data_ptr(), cu32.data_ptr(),
                                     cu_q32.data_ptr(), b, max(int(max_q), 1), int(max_k), cfg.num_heads,
                                     cfg.num_kv_heads, cfg.head_dim, 1.0 / math.sqrt(cfg.head_dim),
                                     out.data_ptr(), out.stride(0), stream)
            _native.check(code, "rdx_attention")

        self._op("attention", launch, flops)
        return out

    # ------------------------------------------------------------ layout
    def _layout(self, db: DeviceBatch, plan, attention: str) -> _Layout:
        import torch

        if plan is None:
            return _Layout(db.n, db.n, None, None, db.pos, db.cu32, db.max_len, True, False)
        if isinstance(plan, str) and plan == "auto":
            plan = self._op("plan_build", lambda: build_plan_device(db.tok, db.pos, db.cu))
        if isinstance(plan, DevicePlan):
            if plan.n_original != db.n or plan.scatter.shape[0] != db.n:
                raise PlanBatchMismatch(f"plan built for {plan.n_original} tokens, batch has {db.n}")
            return _Layout(plan.n_padded, plan.n_compact, plan.gather, plan.scatter, plan.compact_positions,
                           plan.cu_q, plan.max_q_len, True, True, plan)  # cu_q host copy read only if needed
        if isinstance(plan, CompactionPlan):
            if plan.n_original != db.n:
                raise PlanBatchMismatch(f"plan built for {plan.n_original} tokens, batch has {db.n}")
            if plan.scatter_indices.shape[0] != db.n:
                raise PlanBatchMismatch("scatter index length disagrees with batch")
            dev = db.tok.device
            g = torch.from_numpy(np.array(plan.gather_indices).view(np.int32)).to(dev)
            s = torch.from_numpy(np.array(plan.scatter_indices).view(np.int32)).to(dev)
            p = torch.from_numpy(np.array(plan.compact_positions).view(np.int32)).to(dev)
            cu_q = host_plan_cu_q(plan, db.cu_host) if attention == "suffix" else None
            if cu_q is None:
                return _Layout(plan.n_padded, plan.n_compact, g, s, p, None, 0, False, True)
            cu_q32 = torch.from_numpy(cu_q.astype(np.int32)).to(dev)
            max_q = int(np.diff(cu_q).max()) if cu_q.size > 1 else 0
            return _Layout(plan.n_padded, plan.n_compact, g, s, p, cu_q32, max_q, True, True, cu_q)
        raise TypeError(f"unsupported plan type {type(plan).__name__}")

    # ------------------------------------------------------------ forward
    def prefill(self, db: DeviceBatch, plan=None, *, attention: str = "suffix", logits: str = "all",
                ledger: FlopLedger | None = None, stream=None):
        """Run the prefill; returns fp32 logits [N, vocab] ("all") or [B, vocab] ("last")."""
        if attention not in ("suffix", "full"):
            raise ValueError("attention must be 'suffix' or 'full'")
        if logits not in ("all", "last"):
            raise ValueError("logits must be 'all' or 'last'")
        if db.max_token >= self.config.vocab_size:
            from .errors import IndexOutOfRange

            raise IndexOutOfRange("token id outside [0, vocab_size)")
        lay = self._layout(db, plan, attention)
        mode = "plain" if not lay.dedup else ("suffix" if attention == "suffix" and lay.suffix_ok else "full")
        if ledger is not None:  # row accounting only when the caller asked for it (host time on the hot path)
            self._fill_ledger(ledger, lay, db, mode, logits)
        eager = not self.use_graphs or self.op_hook is not None or db.n == 0
        if eager or self._graph_key(db, lay, mode, logits) not in self._graphs:
            self._att_pairs = self._attention_pairs(db, lay, mode)  # FLOP accounting of the launches
        if eager:
            out, err = self._body(db.tok, lay.gather, lay.scatter, lay.positions, db.cu32, db.cu, lay.cu_q32,
                                  lay.m, db.n, db.b, lay.n_compact, lay.max_q, db.max_len, mode, logits, stream)
            if db.max_token < 0 and int(err.item()):
                from .errors import IndexOutOfRange

                raise IndexOutOfRange("token id outside [0, vocab_size)")
            return out
        return self._replay(db, lay, mode, logits, stream)

    # CUDA-graph buckets (pad_plan semantics, trie.py:206-233): one graph
    # serves every batch whose padded shape falls in the same bucket.  M_BUCKET = 256 is the
    # CTA-pair GEMM row tile, so padding N' up to it adds no GEMM tile; the other buckets
    # only size index buffers and the attention unit grid (empty units cost a skip).
    M_BUCKET, N_BUCKET, B_BUCKET, LEN_BUCKET = 256, 2048, 16, 64

    @staticmethod
    def _round(x, q):
        return -(-max(int(x), 1) // q) * q

    def _graph_shape(self, db, lay, mode):
        """(m_b, n_b, b_b, max_q_b, max_k_b) of the bucket a batch falls in."""
        r = self._round
        # the row bucket grows with M (256 below 16K rows, 512 below 32K, ...): at most ~1.6 %
        # padding, and a distribution of large batches maps onto a few graphs
        def mq(m):
            return self.M_BUCKET << max(0, int(m).bit_length() - 14)

        if mode == "plain":
            m_b = n_b = r(db.n, mq(db.n))
        else:
            m_b, n_b = r(lay.m, mq(lay.m)), r(db.n, self.N_BUCKET)
        max_k = r(db.max_len, self.LEN_BUCKET)
        max_q = max_k if mode == "plain" else r(lay.max_q, self.LEN_BUCKET)
        return m_b, n_b, r(db.b, self.B_BUCKET), max_q, max_k

    def _graph_key(self, db, lay, mode, logits):
        return (mode, logits) + self._graph_shape(db, lay, mode)

    @staticmethod
    def _fill(dst, src, pad_from_end=False):
        """dst[:len(src)] = src; the rest repeats src[0] (or src[-1]): device-side, no sync."""
        k = src.shape[0]
        dst[:k].copy_(src, non_blocking=True)
        if k < dst.shape[0]:
            edge = src[k - 1:k] if pad_from_end else src[:1]
            dst[k:].copy_(edge.expand(dst.shape[0] - k), non_blocking=True)

    def _replay(self, db, lay, mode, logits, stream):
        import torch

        key = self._graph_key(db, lay, mode, logits)
        m_b, n_b, b_b, max_q_b, max_k_b = key[2:]
        g = self._graphs.get(key)
        if g is None:
            dev = db.tok.device
            i32 = dict(dtype=torch.int32, device=dev)
            inputs = {"tok": torch.zeros(n_b, **i32), "pos": torch.zeros(m_b, **i32),
                      "cu32": torch.zeros(b_b + 1, **i32), "cu": torch.zeros(b_b + 1, dtype=torch.int64, device=dev),
                      "gather": None, "scatter": None, "cu_q32": None}
            if mode != "plain":
                inputs.update(gather=torch.zeros(m_b, **i32), scatter=torch.zeros(n_b, **i32),
                              cu_q32=torch.zeros(b_b + 1, **i32))
            self._stage(inputs, db, lay, mode)
            cu_q = inputs["cu32"] if mode == "plain" else inputs["cu_q32"]
            args = (inputs["tok"], inputs["gather"], inputs["scatter"], inputs["pos"], inputs["cu32"], inputs["cu"],
                    cu_q, m_b, n_b, b_b, 0, max_q_b, max_k_b, mode, logits, None)
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):  # warm-up outside capture (allocator, lazy init)
                self._body(*args)
            torch.cuda.current_stream().wait_stream(side)
            if self._graph_pool is None:  # one memory pool shared by every captured bucket
                self._graph_pool = torch.cuda.graph_pool_handle()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, pool=self._graph_pool):
                out, err = self._body(*args)
            g = _Graph(graph, inputs, out, err)
            self._graphs[key] = g
            self.graph_captures += 1
            while len(self._graphs) > self.max_graphs:  # LRU bound
                self._graphs.popitem(last=False)
        else:
            self._graphs.move_to_end(key)
            # always copy: device buffers written through the C ABI do not bump torch's
            # version counters, so "same tensor" cannot prove "same contents"
            self._stage(g.inputs, db, lay, mode)
        g.graph.replay()
        if db.max_token < 0 and int(g.err.item()):
            from .errors import IndexOutOfRange

            raise IndexOutOfRange("token id outside [0, vocab_size)")
        rows = db.b if logits == "last" else db.n
        return g.output[:rows]

    def _stage(self, inputs, db, lay, mode):
        """Copy one batch into a bucket's static buffers, padding as pad_plan does."""
        self._fill(inputs["tok"], db.tok)
        self._fill(inputs["cu32"], db.cu32, pad_from_end=True)   # padded sequences are empty
        self._fill(inputs["cu"], db.cu, pad_from_end=True)
        if mode == "plain":
            self._fill(inputs["pos"], db.pos)
        else:
            self._fill(inputs["gather"], lay.gather)              # pad rows repeat gather[0] ...
            self._fill(inputs["pos"], lay.positions)              # ... and compact_positions[0]
            self._fill(inputs["scatter"], lay.scatter)
            if lay.cu_q32 is not None:
                self._fill(inputs["cu_q32"], lay.cu_q32, pad_from_end=True)

    def _fill_ledger(self, ledger, lay, db, mode, logits):
        """Row counters exactly as the reference's forward records them (model.py:331-411)."""
        m, n = lay.m, db.n
        if lay.dedup:
            ledger.index_copy(m)
        ledger.positionwise("embed", m)
        for i in range(self.config.num_layers):
            ledger.positionwise(f"l{i}.ln1", m)
            ledger.positionwise(f"l{i}.qkv_proj", m)
            ledger.positionwise(f"l{i}.qk_norm_rope", m)
            if mode == "plain":
                ledger.attention(n)
            elif mode == "suffix":
                ledger.index_copy(2 * n)          # K/V only
                ledger.attention(lay.n_compact)   # query rows stay compact
            else:
                ledger.index_copy(3 * n)
                ledger.attention(n)
                ledger.index_copy(m)
            for ph in ("o_proj", "attn_residual", "mlp", "mlp_residual"):
                ledger.positionwise(f"l{i}.{ph}", m)
        rows = db.b if logits == "last" else m
        ledger.positionwise("final_norm", rows)
        ledger.positionwise("lm_head", rows)
        if lay.dedup and logits == "all":
            ledger.index_copy(n)

    @staticmethod
    def _attention_pairs(db, lay, mode) -> float:
        """Causal (query, key) pairs per head (host arithmetic, for FLOP accounting)."""
        lens = np.diff(db.cu_host).astype(np.float64)
        full = float(np.sum(lens * (lens + 1) / 2))
        if mode != "suffix":
            return full
        cu_q = getattr(lay, "cu_q_host", None)
        if cu_q is not None and not isinstance(cu_q, np.ndarray):
            cu_q = cu_q.cu_q_host  # a DevicePlan: its lazily read host copy
        if cu_q is None:
            return full
        lcp = lens - np.diff(cu_q)
        return float(np.sum(lens * (lens + 1) / 2 - lcp * (lcp + 1) / 2))

    def _body(self, tok, gather, scatter, positions, cu32, cu64, cu_q32, m, n, b, n_compact, max_q, max_k,
              mode, logits, stream):
        """The layer stack as pure launches (CUDA-graph capturable)."""
        import torch

        cfg, T = self.config, self.w.t
        lib = _native.lib()
        st = _native.stream_handle(stream)
        dev = tok.device
        d, hd, H, KV = cfg.hidden_size, cfg.head_dim, cfg.num_heads, cfg.num_kv_heads
        qd, kvd = cfg.q_dim, cfg.kv_dim
        bf = torch.bfloat16
        h = torch.empty(m, d, dtype=torch.float32, device=dev)
        hn = torch.empty(m, d, dtype=bf, device=dev)  # fused_norm: bf16(h), unnormalised
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        fused = self.fused_norm
        ss = torch.empty(m, d // 64, dtype=torch.float32, device=dev) if fused else None

        def embed():
            if fused:
                code = lib.rdx_embed_rows(tok.data_ptr(), None if gather is None else gather.data_ptr(), m,
                                          T["embed"].data_ptr(), cfg.vocab_size, d, h.data_ptr(), hn.data_ptr(),
                                          ss.data_ptr(), err.data_ptr(), st)
                _native.check(code, "rdx_embed_rows")
                return
            code = lib.rdx_embed_rmsnorm(tok.data_ptr(), None if gather is None else gather.data_ptr(), m,
                                         T["embed"].data_ptr(), cfg.vocab_size, d, T["layers.0.ln1"].data_ptr(),
                                         cfg.norm_eps, h.data_ptr(), hn.data_ptr(), err.data_ptr(), st)
            _native.check(code, "rdx_embed_rmsnorm")

        self._op("embed_rmsnorm", embed)
        resid_epi = _native.EPI_RESID_NORM if fused else _native.EPI_RESID_F32
        sfx = "_n" if fused else ""
        if hd in (64, 128):
            rope = ("pos", positions)  # the QKV epilogue computes (cos, sin) itself: no table pass
        else:
            # lane-blocked (cos, sin) table: the QKV epilogue's 32 lanes read contiguous runs
            table = torch.empty(-(-m // 32) * 32 * (hd // 2) * 2, dtype=torch.float32, device=dev)
            rope = ("table", table)

            def rope_fn():
                _native.check(lib.rdx_rope_table_blocked(positions.data_ptr(), m, hd, float(cfg.rope_theta),
                                                         table.data_ptr(), st), "rdx_rope_table_blocked")

            self._op("rope_table", rope_fn)
        qkv = torch.empty(m, qd + 2 * kvd, dtype=bf, device=dev)
        act = torch.empty(m, self.di_pad, dtype=bf, device=dev)
        attn_out = torch.empty(m, qd, dtype=bf, device=dev)
        if mode != "full" and m > n_compact:
            attn_out[n_compact:] = 0  # padded rows are never attention queries (n_compact = 0: graph buckets)
        last_rows = None
        if logits == "last":
            ends = cu64[1:] - 1
            last_rows = (scatter[ends] if mode != "plain" else ends).to(torch.int32).contiguous()
        att_flops = 4.0 * qd * getattr(self, "_att_pairs", 0.0)
        # ln2 / next ln1 start on the row blocks the residual GEMM has finished (its last
        # round leaves SMs idle): 32-row slab counters, one target step of d per use
        overlap = self.norm_overlap and not fused and d in (256, 512, 1024, 2048, 2560, 4096)
        # chained (RDX_NORM_CHAIN=1): that norm also publishes finished rows and the next GEMM
        # (gate_up / the next layer's QKV) starts on them as its programmatic dependent
        chain = overlap and self.norm_chain
        slabs = -(-m // 32)
        # (rdx_gemm_pair runs two launches itself at >= 64 pair row blocks; decided here too so
        # launch counts and the per-op breakdown name what runs)
        pair = self.mlp_pair and not fused and -(-m // 256) < 64
        n_dep = cfg.num_layers * slabs if pair else 0
        n_ctr = (2 * slabs if chain else slabs) if overlap else 0
        ctrs = torch.zeros(n_ctr + n_dep, dtype=torch.int32, device=dev) if n_ctr + n_dep else None  # one memset
        ctr = ctrs[:slabs] if overlap else None
        rdy = ctrs[slabs:2 * slabs] if chain else None
        deps = ctrs[n_ctr:] if pair else None
        uses = 0

        def norm_after(wt):
            nonlocal uses
            if overlap:
                uses += 1
                self._rmsnorm_after(h, wt, hn, ctr, uses * d, stream=st, ready=rdy)
            else:
                self._rmsnorm(h, wt, hn, stream=st)

        def ready_arg():  # the consumer of the norm just launched (None before the first one)
            return (rdy, uses) if chain and uses > 0 else None

        for i in range(cfg.num_layers):
            pre = f"layers.{i}."
            self._gemm("qkv", hn, T[pre + "w_qkv" + sfx], _native.EPI_QKV, qkv, m=m, stream=st, qkv=True,
                       rope=rope, layer=pre, row_ss=ss, ready=ready_arg())
            if mode == "plain":
                a = self._attn(qkv, None, cu32, cu32, b, max_k, max_k, attn_out, att_flops, st)
            elif mode == "suffix":
                a = self._attn(qkv, scatter, cu32, cu_q32, b, max_q, max_k, attn_out, att_flops, st)
            else:
                qkv_full = self._gather("scatter_qkv", qkv, scatter, stream)
                a_full = torch.empty(n, qd, dtype=bf, device=dev)
                self._attn(qkv_full, None, cu32, cu32, b, max_k, max_k, a_full, att_flops, st)
                a = self._gather("gather_attn", a_full, gather, stream)
            a = a.reshape(m, qd)
            self._gemm("o_proj", a, T[pre + "wo"], resid_epi, h, m=m, stream=st, hb=hn if fused else None,
                       ss_out=ss, done=ctr)
            if not fused:
                norm_after(T[pre + "ln2"])
            last = i + 1 == cfg.num_layers
            if pair:
                g_args = self._gemm("gate_up", hn, T[pre + "w_gu"], _native.EPI_SWIGLU, act, m=m, stream=st,
                                    ready=ready_arg(), build_only=True)
                d_args = self._gemm("down", act, T[pre + "w_down"], resid_epi, h, m=m, stream=st,
                                    done=None if last else ctr, build_only=True)
                self._gemm_pair(g_args, d_args, deps[i * slabs:(i + 1) * slabs], st)
            else:
                self._gemm("gate_up", hn, T[pre + "w_gu" + sfx], _native.EPI_SWIGLU, act, m=m, stream=st,
                           row_ss=ss, ready=ready_arg())
                self._gemm("down", act, T[pre + "w_down"], resid_epi, h, m=m, stream=st,
                           hb=hn if fused else None, ss_out=ss, done=None if last else ctr)
            if not fused and not last:
                norm_after(T[f"layers.{i + 1}.ln1"])

        vocab = cfg.vocab_size
        vpad = -(-vocab // 8) * 8  # 16-byte aligned logits rows
        if logits == "last":
            hl = torch.empty(b, d, dtype=bf, device=dev)
            self._rmsnorm(h, T["final_norm"], hl, rows=last_rows, n_rows=b, stream=st)
            out = torch.empty(b, vpad, dtype=torch.float32, device=dev)[:, :vocab]
            self._gemm("lm_head", hl, T["lm_head"], _native.EPI_STORE_F32, out, m=b, stream=st)
            result = out if vpad == vocab else out.contiguous()
        else:
            self._rmsnorm(h, T["final_norm"], hn, stream=st)
            out = torch.empty(m, vpad, dtype=torch.float32, device=dev)[:, :vocab]
            self._gemm("lm_head", hn, T["lm_head"], _native.EPI_STORE_F32, out, m=m, stream=st)
            if mode != "plain":
                result = self._gather("scatter_logits", out, scatter, stream)
            else:
                result = out if vpad == vocab else out.contiguous()
        return result, err


def _model_for(config: ModelConfig, params) -> RadixQwen3:
    """No implicit weight cache: the reference's forward is pure in ``params``
    (its tests edit arrays in place between calls, test_model.py:304-313), so a
    numpy dict is converted on every call.  Callers that reuse weights pass a
    :class:`DeviceWeights` or a :class:`RadixQwen3`."""
    if isinstance(params, RadixQwen3):
        return params
    if isinstance(params, DeviceWeights):
        return RadixQwen3(config, params)
    return RadixQwen3(config, DeviceWeights.from_params(config, params))


def forward(config: ModelConfig, params, batch: RaggedBatch, plan=None, ledger: FlopLedger | None = None,
            *, attention: str = "suffix", logits: str = "all"):
    """Reference-compatible entry (model.py:310-319) returning device fp32 logits.

    ``params`` is the reference's numpy dict (converted on every call), a
    :class:`DeviceWeights` or a :class:`RadixQwen3`.  ``plan`` is None (dedup
    off), a host :class:`CompactionPlan`, a :class:`DevicePlan` or "auto"
    (GPU planner).
    """
    validate_batch(batch, allow_empty=True)
    model = _model_for(config, params)
    db = DeviceBatch.from_batch(batch)
    return model.prefill(db, plan, attention=attention, logits=logits, ledger=ledger)


def forward_scores(config: ModelConfig, params, batch: RaggedBatch, plan="auto"):
    """Last-token logits [B, vocab] (the scoring contract), device fp32."""
    return forward(config, params, batch, plan=plan, logits="last")
