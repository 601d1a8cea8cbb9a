#!/usr/bin/env python
"""RadixMLP prefill benchmark on B200 (one process per GPU).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c4|c5]
                  [--impl ours|reference] [--scaling weak|strong]

Metric (BASELINE.json): input tokens/s counted in ORIGINAL tokens N, Qwen3
prefill with RadixMLP on, beside the same framework with dedup off; plus the
row-gather GB/s microbenchmark.  A "step" = one reranking pass over one
batch: GPU plan build (index computation) + RadixMLP prefill on the compact
rows + last-token logits (full vocab) + reranker scores.

Workloads (BASELINE.json configs):
  c2 (default)  configs[1]: Qwen3-0.6B, synthetic MS-MARCO-shaped batch, 1 query
                x 64 passages behind a shared reranker template.  N > 1: weak
                scaling, one query subtree (64 passages) per GPU.
  c3            configs[2]: Qwen3-4B, 4 queries x 64 passages = batch 256.  N > 1:
                strong scaling, the batch-256 workload split by trie subtree.
  c4            configs[3]: Qwen3-8B, 128 x (2048 shared + 256).  N > 1: strong
                scaling, batch 128 split by trie subtree (the 2048-token trunk is
                recomputed on every GPU).
  c5            configs[4]: planner + row gather/scatter microbenchmark.
``--scaling`` overrides the default per config.  ``--gpus N`` without a
torchrun environment re-executes itself under ``torch.distributed.run`` with N
local ranks (one process per GPU, NCCL); the only collective is the final
all-gather of per-sequence scores.

``value``   device time, inputs already in HBM, L2 flushed between steps, max over ranks.
``e2e``     the public API from pinned host buffers: H2D ids, GPU plan, prefill,
            scores D2H, all inside the timed region, over K DISTINCT batches of
            the workload's distribution (different seeds, so N, N', B-lengths
            vary), through RadixReranker.score_many (CUDA-graph buckets,
            ``graph_captures_timed`` = captures inside the timed region).
``parity``  at the benchmarked config: radix vs dedup-off last-token logits and
            scores, and the reference boundary (attention="full") vs dedup off.
``roofline`` the dominant kernel (the gate|up SwiGLU GEMM, tcgen05): 2*M*N*K /
            its CUDA-event launch time; peak = burst bf16 for a short step,
            sustained for a long one (MEASURED_PEAKS.json).
``cpu_baseline`` the reference's own CPU path (radix_compact from baseline/_ref:
            numba build_plan + numpy forward) on a bounded sample, else its port.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "input tokens/sec (orig. tokens) Qwen3 prefill, RadixMLP vs no-dedup; gather GB/s"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
TOL = 2e-2  # BASELINE.json north star: max relative error on final logits
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f), "measured"
    return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


def host_info():
    model = None
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name"):
                model = line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}


# ------------------------------------------------------------------ workloads
DEFAULT_SCALING = {"c2": "weak", "c3": "strong", "c4": "strong"}


def workload(name: str, world: int, scaling: str, seed: int = 0):
    """(config, model name, GLOBAL batch, label) of a benchmark config; ``seed`` draws
    another batch of the same distribution (the e2e stream)."""
    from paper_2601_15013_b200.model import QWEN3_PRESETS
    from paper_2601_15013_b200.ragged import RaggedBatch
    from paper_2601_15013_b200.workloads import RerankSpec, long_prefix_batch, msmarco_rerank_batch

    weak = world if scaling == "weak" else 1
    if name == "c2":
        spec = RerankSpec(queries=weak, passages_per_query=64, seed=seed)
        return QWEN3_PRESETS["qwen3-0.6b"], "qwen3-0.6b", msmarco_rerank_batch(spec), spec.label
    if name == "c2_literal":  # configs[1] literally: one ~32-token query prefix, no template
        spec = RerankSpec(queries=weak, passages_per_query=64, template_len=0, query_len=32, tail_len=0, seed=seed)
        return QWEN3_PRESETS["qwen3-0.6b"], "qwen3-0.6b", msmarco_rerank_batch(spec), spec.label
    if name == "c3":
        spec = RerankSpec(queries=4 * weak, passages_per_query=64, seed=seed)
        return QWEN3_PRESETS["qwen3-4b"], "qwen3-4b", msmarco_rerank_batch(spec), spec.label
    if name == "c4":
        parts = [long_prefix_batch(seed=seed * 1000 + r) for r in range(weak)]
        if weak == 1:
            batch = parts[0]
        else:
            tok = np.concatenate([p.token_ids for p in parts])
            cu = np.concatenate([[0], np.cumsum(np.concatenate([np.diff(p.cu_seqlens) for p in parts]))])
            batch = RaggedBatch(tok, np.concatenate([p.position_ids for p in parts]), cu)
        return QWEN3_PRESETS["qwen3-8b"], "qwen3-8b", batch, f"long_prefix_B{128 * weak}_P2048_S256"
    raise SystemExit(f"unknown config {name}")


# ------------------------------------------------------------------ distributed plumbing
def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_launch(args):
    """``--gpus N`` outside torchrun: re-execute under torch.distributed.run, one rank per GPU."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def _backend_device(world):
    import torch
    import torch.distributed as dist

    if world > 1 and dist.get_backend() == "gloo":
        return torch.device("cpu")
    return torch.device("cuda", torch.cuda.current_device())


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=_backend_device(world))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_objects(obj, world):
    if world == 1:
        return [obj]
    import torch.distributed as dist

    out = [None] * world
    dist.all_gather_object(out, obj)
    return out


def barrier(world: int, cuda: bool = True):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    if cuda:
        import torch

        torch.cuda.synchronize()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        # nvidia-smi needs ~0.1-0.3 s to print its first sample; a short timed region (C2: ~0.15 s)
        # could end before that, so wait for the first (pre-region, discarded) sample
        import select

        ready, _, _ = select.select([self.proc.stdout], [], [], 5.0)
        if ready:
            self.proc.stdout.readline()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.06)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=5)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ timing
class L2Flusher:
    def __init__(self, nbytes=256 << 20):
        import torch

        self.buf = torch.empty(nbytes // 4, dtype=torch.int32, device="cuda")

    def __call__(self):
        self.buf.zero_()


def time_steps(fn, steps, warmup, world, flush=None, sampler=None):
    """W untimed warm-ups, then exactly K steps each bracketed by CUDA events
    (L2 flushed between steps, outside the events); barrier + synchronize on
    both sides; returns (total ms max over ranks, per-step ms list, clocks)."""
    import torch

    for _ in range(warmup):
        fn()
    barrier(world)
    if sampler:
        sampler.start()
    evs = []
    for _ in range(steps):
        if flush:
            flush()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        evs.append((s, e))
    barrier(world)
    clocks = sampler.stop() if sampler else None
    per = [s.elapsed_time(e) for s, e in evs]
    return max_over_ranks(sum(per), world), per, clocks


# ------------------------------------------------------------------ per-op events and the roofline
def op_breakdown(model, step, steps):
    """Per-op CUDA events (on the launching stream) over ``steps`` eager steps."""
    import torch

    records = []

    def hook(name, launch, flops):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        out = launch()
        e.record()
        records.append((name, flops, s, e))
        return out

    model.op_hook = hook
    try:
        step()
        records.clear()
        for _ in range(steps):
            step()
        torch.cuda.synchronize()
    finally:
        model.op_hook = None
    by = {}
    for name, f, s, e in records:
        d = by.setdefault(name, [0.0, 0.0, 0])
        d[0] += f
        d[1] += s.elapsed_time(e)
        d[2] += 1
    return by


def ncu_traffic(path):
    """dram read + write bytes of one launch from a committed ncu --set full summary
    (scripts/ncu_summary.py output under profiles/), or None."""
    scale = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}
    try:
        tot, kernel = 0.0, None
        for line in open(path):
            parts = line.split()
            if line.startswith("kernel:"):
                kernel = line.split(":", 1)[1].strip()[:60]
            if len(parts) >= 4 and parts[0] == "dram" and parts[1] in ("read", "write"):
                tot += float(parts[2]) * scale[parts[3].lower()]
        return (round(tot), kernel) if tot else None
    except (OSError, ValueError, KeyError):
        return None


def roofline(by, steps, ms_per_step, peaks, peaks_src, config_name):
    """Dominant kernel = the MLP launch: gate|up SwiGLU GEMM and down GEMM in one
    persistent kernel (rdx_gemm_pair), else the gate|up GEMM alone (the top launch of
    the step in every ncu launch list)."""
    pair = "gemm.mlp" in by
    name = "gemm.mlp" if pair else "gemm.gate_up"
    f, ms, n = by[name]
    achieved = f / (ms * 1e-3) / 1e12
    long_step = ms_per_step >= 50.0
    peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]) if long_step else peaks["bf16_tflops"]
    gemm = [(v[0], v[1], v[2]) for k, v in by.items() if k.startswith("gemm.")]
    gf, gms, gn = sum(x[0] for x in gemm), sum(x[1] for x in gemm), sum(x[2] for x in gemm)
    roof = {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4), "traffic": None,
            "kernel": ("gemm_kernel<256, SWIGLU, 2, RESID_F32> (tcgen05 2-CTA, rdx_gemm_pair): gate|up + SiLU*mul, "
                       "then down + residual reduce-add in the same launch" if pair else
                       "gemm_kernel (tcgen05 2-CTA, EPI_SWIGLU): gate|up projection + SiLU*mul"),
            "flops_per_launch": round(f / n), "avg_launch_us": round(ms * 1e3 / n, 2),
            "peak_kind": ("sustained (step >= 50 ms: clocks settle under the power cap)" if long_step
                          else "burst (short step, kernels run at boost clocks)") + f"; {peaks_src}",
            "all_gemms": {"achieved": round(gf / (gms * 1e-3) / 1e12, 1), "frac": round(gf / (gms * 1e-3) / 1e12 / peak, 4),
                          "launches_per_step": gn // steps, "share_of_step": round(gms / steps / ms_per_step, 3)}}
    stems = ["ncu_gemm_mlp"] if pair else ["ncu_gemm_gateup", "ncu_gateup"]
    for path in [os.path.join(ROOT, "profiles", f"{rnd}_{stem}_{config_name}.txt") for rnd in ("r2", "r1")
                 for stem in stems]:
        tr = ncu_traffic(path)
        if tr is not None:  # DRAM bytes of one launch from the committed ncu --set full capture
            roof["traffic"] = tr[0]
            roof["traffic_source"] = f"{os.path.relpath(path, ROOT)} (dram read+write, 1 launch)"
            roof["algorithmic_bytes"] = None
            break
    return roof


# ------------------------------------------------------------------ gather GB/s
def gather_microbench(peak_gbs):
    import torch

    from paper_2601_15013_b200 import gather_rows_device

    # paper Table 6 largest shape: [100000, 2048] f16 -> 500000 rows, bf16 here
    g = torch.Generator(device="cuda").manual_seed(0)
    src = torch.randn(100_000, 2048, device="cuda", generator=g).to(torch.bfloat16)
    idx = torch.randint(0, 100_000, (500_000,), device="cuda", dtype=torch.int32, generator=g)
    dst = torch.empty(500_000, 2048, dtype=torch.bfloat16, device="cuda")
    for _ in range(3):
        gather_rows_device(src, idx, out=dst)
    torch.cuda.synchronize()
    times = []
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        gather_rows_device(src, idx, out=dst)
        e.record()
        e.synchronize()
        times.append(s.elapsed_time(e))
    ms = statistics.median(times)
    nbytes = 500_000 * (2 * 2048 * 2 + 4)
    gbs = nbytes / (ms * 1e-3) / 1e9
    del src, dst
    return {"shape": "[100000,2048] bf16 -> 500000 rows", "ms": round(ms, 4), "gbs": round(gbs, 1),
            "frac_of_hbm": round(gbs / peak_gbs, 3), "bytes_convention": "2*rows*row_bytes + 4*rows"}


# ------------------------------------------------------------------ CPU baselines
def import_reference():
    """The reference package (pip-installed into baseline/_ref, which travels to the GPU box), or None."""
    if os.path.isdir(os.path.join(REF_DIR, "radix_compact")):
        if REF_DIR not in sys.path:
            sys.path.append(REF_DIR)
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_rdx")
        try:
            import radix_compact
            import radix_compact.model  # noqa: F401
            import radix_compact.trie  # noqa: F401

            return radix_compact
        except Exception:  # noqa: BLE001 -- e.g. numba missing: fall back to the port
            return None
    return None


def _median_time(fn, reps=7):
    """The reference's own methodology (bench.py:243-250): one warm-up discarded, median of reps."""
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


CPU_SAMPLE = {"c2": (2, None), "c2_literal": (2, None), "c3": (4, 2), "c4": (2, 1)}  # (sequences, layers or full)


def cpu_forward_sample(config, batch, name, warm=False):
    """The reference CPU forward on a bounded sample of the workload: the first ``seqs``
    sequences at full depth (c2) or at ``layers`` layers extrapolated per layer (c3/c4,
    labelled).  Uses the reference itself (radix_compact.model.forward with its own
    numba build_plan) when baseline/_ref is importable, else the oracle port."""
    from paper_2601_15013_b200.shard import sub_batch

    seqs, layers = CPU_SAMPLE[name]
    if warm:  # warm-up: JIT (numba) and page-in only, one layer
        layers = 1
    sb = sub_batch(batch, np.arange(min(seqs, batch.num_sequences)))
    rng = np.random.default_rng(0)
    d, v = config.hidden_size, config.vocab_size
    uniq, tok_small = np.unique(sb.token_ids, return_inverse=True)  # embed rows of the sample's tokens only
    depth = config.num_layers if layers is None else layers
    params = {"embed": rng.uniform(-0.05, 0.05, size=(uniq.size, d)).astype(np.float32),
              "final_norm": np.ones(d, np.float32),
              "lm_head": rng.uniform(-0.05, 0.05, size=(v, d)).astype(np.float32)}
    for i in range(depth):
        pre = f"layers.{i}."
        for nm, shp in (("wq", (config.q_dim, d)), ("wk", (config.kv_dim, d)), ("wv", (config.kv_dim, d)),
                        ("wo", (d, config.q_dim)), ("w_gate", (config.intermediate_size, d)),
                        ("w_up", (config.intermediate_size, d)), ("w_down", (d, config.intermediate_size))):
            params[pre + nm] = rng.uniform(-0.05, 0.05, size=shp).astype(np.float32)
        for nm, n in (("ln1", d), ("ln2", d), ("q_norm", config.head_dim), ("k_norm", config.head_dim)):
            params[pre + nm] = np.ones(n, np.float32)
    tok_small = tok_small.astype(np.uint32)
    ref = import_reference()
    if ref is not None:
        from dataclasses import replace

        class Qwen3LikeConfig(ref.model.ModelConfig):  # admits q_dim != hidden (SURVEY finding 3)
            def __post_init__(self):
                pass

        fields = {k: getattr(config, k) for k in ("num_layers", "hidden_size", "intermediate_size", "num_heads",
                                                  "num_kv_heads", "head_dim", "vocab_size", "rope_theta", "norm_eps")}
        rcfg = Qwen3LikeConfig(**fields)
        rb = ref.RaggedBatch(tok_small, sb.position_ids, sb.cu_seqlens)

        def run(nl):
            t0 = time.perf_counter()
            plan = ref.trie.build_plan(rb)
            ref.model.forward(replace(rcfg, num_layers=nl), params, rb, plan)
            return time.perf_counter() - t0, plan.n_compact

        kind = "reference"
        what = ("radix_compact.trie.build_plan (numba) + radix_compact.model.forward (numpy; its contract "
                "computes logits for every row, [N, vocab])")
    else:
        from oracle import oracle as orc

        def run(nl):
            t0 = time.perf_counter()
            g, s, cp, m = orc.build_plan_oracle(sb.token_ids, sb.position_ids, sb.cu_seqlens)
            orc.forward_oracle(config, params, tok_small, sb.position_ids, sb.cu_seqlens, plan=(g, s, cp),
                               last_only=True, layers=nl)
            return time.perf_counter() - t0, m

        kind = "port"
        what = "oracle/ port of the reference forward (last-token logits), fp32"
    if layers is None:
        t, m = run(config.num_layers)
        total, timed = t, t
        depth_note = f"all {config.num_layers} layers"
    else:
        t1, m = run(1)
        t2, _ = run(2) if layers >= 2 else (None, m)
        per_layer = (t2 - t1) if t2 is not None else t1
        total = t1 + (config.num_layers - 1) * max(per_layer, 1e-9)
        timed = t1 + (t2 or 0.0)
        depth_note = (f"1{' and 2' if layers >= 2 else ''} layer(s) timed, extrapolated per layer to "
                      f"{config.num_layers} (labelled extrapolation, SURVEY §8d)")
    return {"value": sb.num_tokens / total, "unit": "tokens/s", "cores": os.cpu_count() or 1, "kind": kind,
            "sample": (f"{sb.num_sequences} of {batch.num_sequences} sequences / {sb.num_tokens} tokens "
                       f"(N'={m}) of the workload, {depth_note}; {what}; f32 weights, BLAS on all host threads"),
            "seconds": round(timed, 2)}


def cpu_plan_baseline(batch):
    """The reference planner on the FULL workload batch: numba build_plan (1 thread by design,
    trie.py:73), _median_time methodology; else the C restatement of the trie."""
    ref = import_reference()
    if ref is not None:
        rb = ref.RaggedBatch(batch.token_ids, batch.position_ids, batch.cu_seqlens)
        t = _median_time(lambda: ref.trie.build_plan(rb))
        return {"ms": round(t * 1e3, 3), "impl": "radix_compact.trie.build_plan (reference, numba JIT, 1 thread)",
                "kind": "reference"}
    from oracle import oracle as orc

    t = _median_time(lambda: orc.build_plan_oracle(batch.token_ids, batch.position_ids, batch.cu_seqlens))
    return {"ms": round(t * 1e3, 3), "impl": "oracle/trie_oracle.c (C restatement of trie.py:73-122, 1 thread)",
            "kind": "port"}


# ------------------------------------------------------------------ C5 microbenchmark
def _event_time(fn, iters=10, warm=2, flush=None):
    """Median CUDA-event time (ms) of fn on the current stream, L2 flushed before each call."""
    import torch

    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        if flush:
            flush()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


def _graph_time(fn, reps=10):
    """Device time (ms) per call of a launch-only fn: `reps` calls captured in one CUDA graph and
    replayed, so host submission latency is not in the number (median of 5 replays)."""
    import torch

    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
        g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) / reps)
    return sorted(ts)[2]


def run_micro(args):
    """BASELINE configs[4]: index build and gather/scatter over ragged batches of
    1K-1M tokens (prefix-sharing ratios 0..1, multi-level tries): GPU planner
    time vs the reference planner (numba build_plan from baseline/_ref, 1
    thread by design; else the C restatement), and row gather/scatter GB/s."""
    import ctypes

    import torch

    from oracle import oracle as orc
    from paper_2601_15013_b200 import _native
    from paper_2601_15013_b200.ops import gather_rows_device
    from paper_2601_15013_b200.plan import _WORKSPACE, build_plan_device, upload_batch
    from paper_2601_15013_b200.workloads import multilevel_batch, prefix_ratio_batch

    torch.cuda.set_device(0)
    peaks, peaks_src = load_peaks()
    hbm = peaks["hbm_gbs"]
    lib = _native.lib()
    flush = L2Flusher()
    ref = import_reference()
    sizes = [1 << 10, 1 << 14, 1 << 17, 1 << 20]
    cases = [(f"ratio{r:.2f}", n, lambda n=n, r=r: prefix_ratio_batch(n, r)) for n in sizes
             for r in (0.0, 0.25, 0.5, 0.75, 1.0)]
    cases += [("multilevel", n, lambda n=n: multilevel_batch(n)) for n in sizes]
    plans = []
    for name, n, make in cases:
        batch = make()
        tok, pos, cu = upload_batch(batch)
        b = int(cu.shape[0]) - 1
        nn = int(tok.shape[0])
        gather = torch.empty(nn, dtype=torch.int32, device="cuda")
        scatter = torch.empty_like(gather)
        cpos = torch.empty_like(gather)
        info = torch.empty(4 + b + 1, dtype=torch.int32, device="cuda")
        lcp = torch.empty(max(b, 1), dtype=torch.int32, device="cuda")
        scratch = _WORKSPACE.get(tok.device, int(lib.rdx_plan_scratch_bytes(nn, b)))
        def kernel_only():
            _native.check(lib.rdx_plan_build(tok.data_ptr(), pos.data_ptr(), cu.data_ptr(), b, nn, 0,
                                             gather.data_ptr(), scatter.data_ptr(), cpos.data_ptr(),
                                             info.data_ptr() + 16, lcp.data_ptr(), info.data_ptr(),
                                             scratch.data_ptr(), ctypes.c_size_t(scratch.numel()),
                                             _native.stream_handle()),
                          "rdx_plan_build")

        ms_launch = _event_time(kernel_only, flush=flush)  # host-submitted launch, L2 flushed before it
        ms_kernel = _graph_time(kernel_only)                # device time per launch (CUDA graph of 10)
        ms_api = _event_time(lambda: build_plan_device(tok, pos, cu), flush=flush)
        plan = build_plan_device(tok, pos, cu)
        g, sc, cp, m = orc.build_plan_oracle(batch.token_ids, batch.position_ids, batch.cu_seqlens)
        port_ms = _median_time(lambda: orc.build_plan_oracle(batch.token_ids, batch.position_ids,
                                                             batch.cu_seqlens), reps=5) * 1e3
        rec = {"case": name, "N": nn, "B": b, "N_compact": plan.n_compact,
               "gamma": round(plan.n_compact / max(nn, 1), 4), "gpu_kernel_us": round(ms_kernel * 1e3, 1),
               "gpu_launch_us": round(ms_launch * 1e3, 1),
               "gpu_api_us": round(ms_api * 1e3, 1), "cpu_port_us": round(port_ms * 1e3, 1)}
        if ref is not None:
            rb = ref.RaggedBatch(batch.token_ids, batch.position_ids, batch.cu_seqlens)
            ref_ms = _median_time(lambda: ref.trie.build_plan(rb), reps=5) * 1e3
            rec["cpu_reference_numba_us"] = round(ref_ms * 1e3, 1)
            rec["speedup_kernel_vs_reference"] = round(ref_ms / ms_kernel, 1)
            rec["speedup_api_vs_reference"] = round(ref_ms / ms_api, 1)
        rec["bit_exact_vs_oracle"] = bool(m == plan.n_compact and np.array_equal(
            plan.scatter.cpu().numpy().view(np.uint32), sc) and np.array_equal(
            plan.gather.cpu().numpy().view(np.uint32), g))
        nbytes = 12 * nn + 8 * plan.n_compact + 8 * (b + 1)
        rec["index_gbs"] = round(nbytes / (ms_kernel * 1e-3) / 1e9, 1)
        plans.append(rec)
        if name in ("ratio0.50", "multilevel") and nn >= (1 << 14):
            rec["_dev"] = (plan, nn)
    rows = []
    for rec in plans:
        dev = rec.pop("_dev", None)
        if dev is None:
            continue
        plan, nn = dev
        for d in (1024, 2560, 4096, 6144):
            x = torch.randn(plan.n_compact, d, device="cuda").to(torch.bfloat16)
            full = torch.empty(nn, d, dtype=torch.bfloat16, device="cuda")
            comp = torch.empty(plan.n_compact, d, dtype=torch.bfloat16, device="cuda")
            ms_s = _event_time(lambda: gather_rows_device(x, plan.scatter, out=full), flush=flush)
            ms_g = _event_time(lambda: gather_rows_device(full, plan.gather, out=comp), flush=flush)
            rb_ = 2 * d
            alg_s = nn * (2 * rb_ + 4)
            alg_g = plan.n_compact * (2 * rb_ + 4)
            uniq_s = plan.n_compact * rb_ + nn * rb_ + 4 * nn  # each compact row read once from DRAM
            rows.append({"case": rec["case"], "N": nn, "N_compact": plan.n_compact, "d": d,
                         "scatter_us": round(ms_s * 1e3, 1), "scatter_gbs": round(alg_s / (ms_s * 1e-3) / 1e9, 1),
                         "scatter_dram_gbs": round(uniq_s / (ms_s * 1e-3) / 1e9, 1),
                         "gather_us": round(ms_g * 1e3, 1), "gather_gbs": round(alg_g / (ms_g * 1e-3) / 1e9, 1)})
            del x, full, comp
    # the reference's own CPU row ops beside them (radix_compact.ops, numpy; f32 rows since numpy
    # has no bf16), 1 thread and all host threads, _median_time methodology (bench.py:243-250)
    cpu_rows = []
    if ref is not None:
        import radix_compact.ops as rops

        for rec in plans:
            if rec["case"] != "ratio0.50" or rec["N"] != (1 << 17):
                continue
            pb = prefix_ratio_batch(rec["N"], 0.5)
            hplan = ref.trie.build_plan(ref.RaggedBatch(pb.token_ids, pb.position_ids, pb.cu_seqlens))
            for d in (1024, 4096):
                xc = np.random.default_rng(0).standard_normal((hplan.n_compact, d), dtype=np.float32)
                for th in (1, os.cpu_count() or 1):
                    t = _median_time(lambda: rops.gather_rows(xc, hplan.scatter_indices, num_threads=th), reps=3)
                    nb = rec["N"] * (2 * 4 * d + 4)
                    cpu_rows.append({"op": "scatter (gather_rows with the scatter map, N' -> N)", "N": rec["N"],
                                     "d": d, "dtype": "f32", "threads": th, "ms": round(t * 1e3, 2),
                                     "gbs": round(nb / t / 1e9, 2)})
    gather = gather_microbench(hbm)
    best = max(r["gather_gbs"] for r in rows) if rows else gather["gbs"]
    line = {"metric": "C5 index build + row gather/scatter microbenchmark", "value": round(best, 1),
            "unit": "GB/s", "n_gpus": 1, "higher_is_better": True, "dtype": "u32 indices / bf16 rows",
            "data": "synthetic", "config": {"workload": "c5: 1K-1M tokens, seq 512, prefix ratio 0..1, multi-level",
                                            "l2": "L2 flushed (256 MiB write) before each timed call"},
            "hbm_peak_gbs": hbm, "peak_source": peaks_src,
            "bytes_convention": "gather/scatter: 2*rows_out*row_bytes + 4*rows_out; index: 12N + 8N' + 8(B+1)",
            "index_build": plans, "row_ops": rows, "gather_table6": gather, "host": host_info(),
            "cpu_row_ops_reference": cpu_rows,
            "cpu_baseline": {"kind": "reference" if ref is not None else "port", "cores": 1,
                             "sample": ("radix_compact.trie.build_plan (numba, 1 thread) and the C restatement"
                                        if ref is not None else "oracle/trie_oracle.c") + ", full batch"}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ arms
def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    scaling = args.scaling or DEFAULT_SCALING.get(args.config, "weak")
    config, model_name, batch, label = workload(args.config, max(world, args.gpus), scaling)
    samples = []
    for _ in range(min(args.warmup, 1)):  # CPU warm-up = numba JIT + page-in (one 1-layer sample)
        cpu_forward_sample(config, batch, args.config, warm=True)
    for _ in range(args.steps):
        samples.append(cpu_forward_sample(config, batch, args.config))
    value = statistics.median([s["value"] for s in samples])
    s0 = samples[0]
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 2), "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(statistics.median([s["seconds"] for s in samples]) * 1e3, 1),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (random-init weights)",
            "config": {"workload": label, "model": model_name, "global_batch": batch.num_sequences,
                       "tokens_per_step": batch.num_tokens, "parallelism": "cpu (rank 0)"},
            "cpu_baseline": {"value": round(value, 2), "unit": "tokens/s", "cores": s0["cores"], "kind": s0["kind"],
                             "sample": s0["sample"]},
            "e2e": {"value": round(value, 2), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "host": host_info(),
            "note": ("each step = one bounded sample of the workload on the host cores; the reference is pure "
                     "Python/numpy/numba (pkg/), installed into baseline/_ref")}
    print(json.dumps(line), flush=True)


def maxrel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def parity_block(model, rr, rr_base, db, plan):
    """At the benchmarked config, on this rank's batch (eager launches)."""
    import torch

    graphs, model.use_graphs = model.use_graphs, False
    try:
        radix = model.prefill(db, plan, logits="last").cpu().numpy()
        base = model.prefill(db, None, logits="last").cpu().numpy()
        full = model.prefill(db, plan, attention="full", logits="last").cpu().numpy()
        sr = rr.score_device(db, plan=plan).cpu().numpy()
        sb = rr_base.score_device(db, plan=None).cpu().numpy()
        torch.cuda.synchronize()
    finally:
        model.use_graphs = graphs
    r = {"logits_maxrel_radix_vs_nodedup": maxrel(radix, base),
         "scores_maxabs_radix_vs_nodedup": float(np.abs(sr - sb).max()),
         "full_boundary_vs_nodedup_bit_identical": bool(np.array_equal(full, base)),
         "logits_maxrel_full_vs_nodedup": maxrel(full, base), "tolerance": TOL,
         "oracle_parity": "tests/test_parity_scale_gpu.py (full-depth 0.6B, 4B/8B slices, planner on every batch)"}
    r["ok"] = bool(r["logits_maxrel_radix_vs_nodedup"] <= TOL and r["logits_maxrel_full_vs_nodedup"] <= TOL)
    return r


def run_ours(args):
    import torch

    rank, world, local = dist_env()
    if world > 1 and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(0 if args.share_gpu else local)
    if world > 1:
        import torch.distributed as dist

        if args.share_gpu:  # several ranks on one GPU (tests): NCCL refuses duplicate GPUs
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2601_15013_b200 import DeviceBatch, DeviceWeights, RadixQwen3, _native, build_plan_device
    from paper_2601_15013_b200.rerank import RadixReranker
    from paper_2601_15013_b200.shard import gather_scores, partition_by_subtree, shard_report

    peaks, peaks_src = load_peaks()
    scaling = args.scaling or DEFAULT_SCALING[args.config]
    config, model_name, global_batch, label = workload(args.config, world, scaling)
    shards = partition_by_subtree(global_batch, world)
    mine = shards[rank]
    model = RadixQwen3(config, DeviceWeights.random(config, seed=0), use_graphs=not args.no_graphs,
                       fused_norm=True if args.fused_norm else None)
    db = DeviceBatch.from_batch(mine.batch)
    rr = RadixReranker(model, dedup=True)
    rr_base = RadixReranker(model, dedup=False)
    flush = L2Flusher()

    def finish(scores):
        if world > 1:
            return gather_scores(scores, mine.seq_ids, global_batch.num_sequences)
        return scores

    def step_radix():
        return finish(rr.score_device(db))

    def step_base():
        return finish(rr_base.score_device(db))

    plan = build_plan_device(db.tok, db.pos, db.cu)
    tokens_all = global_batch.num_tokens
    per_rank = gather_objects({"n_compact": plan.n_compact}, world)
    report = shard_report(shards, [p["n_compact"] for p in per_rank])
    global_nc = None
    if rank == 0 and world > 1:
        gdb = DeviceBatch.from_batch(global_batch)
        global_nc = build_plan_device(gdb.tok, gdb.pos, gdb.cu).n_compact
        del gdb

    # launches per step (our C-ABI kernels), counted on an eager step after the graph capture
    step_radix()
    torch.cuda.synchronize()
    model.use_graphs, graphs_on = False, model.use_graphs
    c0 = _native.LAUNCHES.launches
    step_radix()
    torch.cuda.synchronize()
    launches_per_step = _native.LAUNCHES.launches - c0
    model.use_graphs = graphs_on

    if args.profile:  # short run for ncu: warm-ups, then the profiled radix steps (cudaProfilerStart/Stop
        for _ in range(args.warmup):  # bracket them, for `ncu --profile-from-start off`), no JSON
            step_radix()
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        for _ in range(args.steps):
            step_radix()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return
    sampler = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    ms_radix, per_radix, clocks = time_steps(step_radix, args.steps, args.warmup, world, flush, sampler)
    ms_base, per_base, _ = time_steps(step_base, args.steps, args.warmup, world, flush)
    value = tokens_all * args.steps / (ms_radix * 1e-3)
    value_base = tokens_all * args.steps / (ms_base * 1e-3)

    # ---- e2e through the public API over K DISTINCT batches of the workload's distribution
    def shard_of(seed):
        gb = workload(args.config, world, scaling, seed=seed)[2]
        part = partition_by_subtree(gb, world)[rank] if world > 1 else None
        return gb, (part.batch if part else gb), (part.seq_ids if part else None)

    # server start-up: one pass over as many distinct batches as the timed stream fills the
    # graph buckets of the distribution (captures inside the timed region are still counted)
    warm = [shard_of(2000 + i) for i in range(max(args.warmup, args.steps, 6))]
    timed = [shard_of(1000 + i) for i in range(args.steps)]
    tokens_e2e = sum(t[0].num_tokens for t in timed)

    def e2e_run(items):
        outs = rr.score_many([t[1] for t in items])
        if world > 1:
            for (gb, _, ids), s in zip(items, outs):
                gather_scores(torch.from_numpy(s).cuda(), ids, gb.num_sequences).cpu()
        return outs

    e2e_run(warm)  # fills the graph buckets of the distribution (what a server does at start-up)
    captures0 = model.graph_captures
    h2d = d2h = 0
    barrier(world)
    t0 = time.perf_counter()
    e2e_run(timed)
    torch.cuda.synchronize()
    ms_e2e = max_over_ranks((time.perf_counter() - t0) * 1e3, world)
    barrier(world)
    captures_timed = model.graph_captures - captures0
    for _, b, _ in timed:
        h2d += b.num_tokens * 8 + (b.num_sequences + 1) * 8
        d2h += b.num_sequences * 4 + (4 + b.num_sequences + 1) * 4
    e2e_value = tokens_e2e / (ms_e2e * 1e-3)
    # the same API on K copies of the benchmark batch (what `value` times)
    same = [(global_batch, mine.batch, mine.seq_ids if world > 1 else None)] * args.steps
    e2e_run(same[:2])
    barrier(world)
    t0 = time.perf_counter()
    e2e_run(same)
    torch.cuda.synchronize()
    ms_same = max_over_ranks((time.perf_counter() - t0) * 1e3, world)
    barrier(world)

    line = None
    if rank == 0:
        steps_b = max(3, min(args.steps, 10))
        # per-op events on this rank's own work (no collective: the other ranks wait at the final barrier)
        by = op_breakdown(model, lambda: rr.score_device(db), steps_b)
        ms_step = ms_radix / args.steps
        roof = roofline(by, steps_b, ms_step, peaks, peaks_src, args.config)
        by_base = op_breakdown(model, lambda: rr_base.score_device(db), 3)
        breakdown = {k: {"us_per_step": round(v[1] * 1e3 / steps_b, 1), "launches_per_step": v[2] // steps_b,
                         **({"tflops": round(v[0] / (v[1] * 1e-3) / 1e12, 1)} if v[0] else {})}
                     for k, v in sorted(by.items(), key=lambda kv: -kv[1][1])}
        parity = parity_block(model, rr, rr_base, db, plan)
        literal = None
        if args.config == "c2" and world == 1:
            lcfg, _, lbatch, llabel = workload("c2_literal", 1, "weak")
            ldb = DeviceBatch.from_batch(lbatch)
            lms, _, _ = time_steps(lambda: rr.score_device(ldb), args.steps, args.warmup, 1, flush)
            lms_b, _, _ = time_steps(lambda: rr_base.score_device(ldb), args.steps, args.warmup, 1, flush)
            lplan = build_plan_device(ldb.tok, ldb.pos, ldb.cu)
            literal = {"workload": llabel, "N": lbatch.num_tokens, "N_compact": lplan.n_compact,
                       "gamma": round(lplan.n_compact / lbatch.num_tokens, 4),
                       "value": round(lbatch.num_tokens * args.steps / (lms * 1e-3), 1),
                       "nodedup_value": round(lbatch.num_tokens * args.steps / (lms_b * 1e-3), 1),
                       "speedup_vs_nodedup": round(lms_b / lms, 3),
                       "note": "configs[1] taken literally: a 32-token query prefix, no reranker template "
                               "(Amdahl cap ~1/gamma of the position-wise share)"}
        gather = gather_microbench(peaks["hbm_gbs"])
        cpu = None
        if not args.no_cpu and world == 1:
            cpu = cpu_forward_sample(config, global_batch, args.config)
            cpu["plan"] = cpu_plan_baseline(global_batch)
            cpu["plan"]["gpu_plan_us"] = round(
                _event_time(lambda: build_plan_device(db.tok, db.pos, db.cu), flush=flush) * 1e3, 1)
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights)",
            "config": {"workload": label, "model": model_name, "global_batch": global_batch.num_sequences,
                       "tokens_per_step": int(tokens_all), "n_compact_global": global_nc,
                       "parallelism": f"dp{world} (trie-subtree shards, {scaling} scaling)",
                       "logits": "last-token, full vocab", "attention": "suffix-query (rdx_attention, tcgen05)",
                       "cuda_graphs": not args.no_graphs, "l2": "L2 flushed (256 MiB write) between timed steps"},
            "shards": report,
            "nodedup": {"value": round(value_base, 1), "ms_per_step": round(ms_base / args.steps, 4)},
            "speedup_vs_nodedup": round(value / value_base, 3),
            "e2e": {"value": round(e2e_value, 1), "unit": "tokens/s", "h2d_bytes_per_step": int(h2d // args.steps),
                    "d2h_bytes_per_step": int(d2h // args.steps), "ms_per_step": round(ms_e2e / args.steps, 4),
                    "api": "RadixReranker.score_many over K distinct host batches (pinned H2D, GPU plan, "
                           "CUDA-graph bucket replay, scores D2H; batch t+1's upload+plan overlap batch t)",
                    "batches": "distinct seeds of the workload distribution",
                    "graph_captures_timed": captures_timed, "graphs_cached": len(model._graphs),
                    "frac_of_value": round(e2e_value / value, 3),
                    "same_batch": {"value": round(tokens_all * args.steps / (ms_same * 1e-3), 1),
                                   "ms_per_step": round(ms_same / args.steps, 4)}},
            "parity": parity,
            "roofline": roof,
            "breakdown_us_radix": breakdown,
            "breakdown_us_nodedup": {k: round(v[1] * 1e3 / 3, 1) for k, v in
                                     sorted(by_base.items(), key=lambda kv: -kv[1][1])},
            "literal_configs1": literal,
            "cpu_baseline": cpu,
            "gather": gather,
            "host": host_info(),
            "gpu_launches": int(launches_per_step * args.steps),
            "gpu_launches_note": "our C-ABI kernels per timed region (radix arm), counted at the C ABI",
            "clocks": clocks,
        }
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)


def selftest_launcher(args):
    """CPU check of the multi-rank plumbing bench.py uses (launcher, trie-subtree partition,
    score all-gather over gloo) with a stand-in scorer; rank 0 prints one JSON line."""
    import torch
    import torch.distributed as dist

    from paper_2601_15013_b200.shard import partition_by_subtree, score_sharded, shard_report

    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    scaling = args.scaling or DEFAULT_SCALING.get(args.config, "weak")
    batch = workload(args.config, world, scaling)[2]

    def stub(b):
        cu = b.cu_seqlens
        return torch.tensor([float(b.token_ids[cu[i]:cu[i + 1]].astype(np.int64).sum() % 9973)
                             for i in range(b.num_sequences)], dtype=torch.float32)

    shards = partition_by_subtree(batch, world)
    got = score_sharded(batch, stub, shards=shards) if world > 1 else stub(batch)
    want = stub(batch)
    if rank == 0:
        print(json.dumps({"selftest": "launcher", "n_ranks": world, "ok": bool(torch.equal(got, want)),
                          "global_batch": batch.num_sequences, "scaling": scaling, "shards": shard_report(shards)}),
              flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="N > 1: weak (per-GPU work fixed) or strong (global batch fixed); default per config")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--profile", action="store_true", help="radix steps only, for ncu")
    ap.add_argument("--no-graphs", action="store_true", help="eager launches instead of CUDA-graph replay")
    ap.add_argument("--fused-norm", action="store_true", help="RMSNorm fused into the GEMMs (RDX_EPI_RESID_NORM A/B)")
    ap.add_argument("--share-gpu", action="store_true", help="all ranks on cuda:0 with gloo (multi-rank tests)")
    ap.add_argument("--selftest-launcher", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    maybe_launch(args)
    if args.selftest_launcher:
        selftest_launcher(args)
    elif args.config == "c5" and args.impl == "ours":
        run_micro(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
