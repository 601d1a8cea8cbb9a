#!/usr/bin/env python
"""RadixMLP prefill benchmark on B200 (one process per GPU).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c4] [--impl ours|reference]

Metric (BASELINE.json): input tokens/s counted in ORIGINAL tokens N, Qwen3
prefill with RadixMLP on, beside the same framework with dedup off; plus the
row-gather GB/s microbenchmark.  A "step" = one reranking pass over one
batch: GPU plan build (index computation) + RadixMLP prefill on the compact
rows + last-token logits (full vocab) + reranker scores.  Default workload
(configs[1]): Qwen3-0.6B, random-init bf16 weights, synthetic MS-MARCO-shaped
batch (1 query x 64 passages behind a shared reranker template).  N > 1:
weak scaling, each GPU gets one query's 64-passage subtree (trie-subtree
partition, paper_2601_15013_b200/shard.py); the only collective is the final
all-gather of scores.

``value``   device time, inputs already in HBM, L2 flushed between steps.
``e2e``     the public API from pinned host buffers: H2D ids, plan, prefill,
            scores D2H, all inside the timed region; value = the streaming
            call RadixReranker.score_many over the K batches (upload + plan of
            batch t+1 overlap the prefill of batch t), ``e2e.sequential`` = one
            RadixReranker.score call per batch.
``roofline`` the tcgen05 GEMMs (the dominant kernels): algorithmic FLOPs /
            CUDA-event time of every GEMM launch, vs measured sustained bf16.
``cpu_baseline`` the CPU oracle port (oracle/oracle.py) on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "input tokens/sec (orig. tokens) Qwen3 prefill, RadixMLP vs no-dedup; gather GB/s"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return p, "measured"
    return PEAKS_FALLBACK, "fallback"


def build_config(name: str, world: int):
    from paper_2601_15013_b200.model import QWEN3_PRESETS
    from paper_2601_15013_b200.workloads import RerankSpec, long_prefix_batch, msmarco_rerank_batch

    if name == "c2":
        spec = RerankSpec(queries=world, passages_per_query=64)
        return QWEN3_PRESETS["qwen3-0.6b"], "qwen3-0.6b", msmarco_rerank_batch(spec), spec.label
    if name == "c3":
        spec = RerankSpec(queries=4 * world, passages_per_query=64)
        return QWEN3_PRESETS["qwen3-4b"], "qwen3-4b", msmarco_rerank_batch(spec), spec.label
    if name == "c4":
        from paper_2601_15013_b200.ragged import RaggedBatch

        parts = [long_prefix_batch(seed=r) for r in range(world)]
        if world == 1:
            batch = parts[0]
        else:
            tok = np.concatenate([p.token_ids for p in parts])
            cu = np.concatenate([[0], np.cumsum(np.concatenate([np.diff(p.cu_seqlens) for p in parts]))])
            batch = RaggedBatch(tok, np.concatenate([p.position_ids for p in parts]), cu)
        return QWEN3_PRESETS["qwen3-8b"], "qwen3-8b", batch, "long_prefix_B128_P2048_S256"
    raise SystemExit(f"unknown config {name}")


# ------------------------------------------------------------------ distributed plumbing
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    import torch

    if world > 1:
        import torch.distributed as dist

        dist.barrier()
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
    both sides; returns (total ms max over ranks, per-step ms list)."""
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
    total = max_over_ranks(sum(per), world)
    return total, per, clocks


def time_wall_steps(fn, steps, warmup, world):
    """End-to-end through the host API: host timer around K synchronous calls."""
    import torch

    for _ in range(warmup):
        fn()
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(steps):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) * 1e3
    barrier(world)
    return max_over_ranks(dt, world)


# ------------------------------------------------------------------ roofline of the GEMMs
def op_breakdown(model, step, steps, peak_tflops):
    """Per-op CUDA events over ``steps`` eager steps; the GEMM roofline comes from
    the gemm.* launches (algorithmic 2*M*N*K FLOPs / event time)."""
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
    gemm = [(f, s.elapsed_time(e)) for name, f, s, e in records if name.startswith("gemm.")]
    flops = sum(g[0] for g in gemm)
    ms = sum(g[1] for g in gemm)
    achieved = flops / (ms * 1e-3) / 1e12
    breakdown = {k: {"us_per_step": round(v[1] * 1e3 / steps, 1), "launches_per_step": v[2] // steps,
                     **({"tflops": round(v[0] / (v[1] * 1e-3) / 1e12, 1)} if v[0] else {})}
                 for k, v in sorted(by.items(), key=lambda kv: -kv[1][1])}
    roof = {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak_tflops, "unit": "TFLOP/s",
            "frac": round(achieved / peak_tflops, 4), "traffic": None,
            "kernel": "rdx gemm_kernel (tcgen05, every GEMM launch of a step)",
            "flops_per_launch": round(flops / max(len(gemm), 1)), "avg_launch_us": round(ms * 1e3 / max(len(gemm), 1), 2)}
    return roof, ms / steps, breakdown


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


# ------------------------------------------------------------------ gather GB/s
def gather_microbench(peak_gbs):
    import torch

    from paper_2601_15013_b200 import gather_rows_device

    out = {}
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
    out = {"shape": "[100000,2048] bf16 -> 500000 rows", "ms": round(ms, 4), "gbs": round(gbs, 1),
           "frac_of_hbm": round(gbs / peak_gbs, 3), "bytes_convention": "2*rows*row_bytes + 4*rows"}
    del src, dst
    return out


# ------------------------------------------------------------------ CPU baseline (oracle port)
def cpu_sample(config, batch, seqs=8, layers=(1, 2)):
    """Time the oracle port of the reference forward (radix plan, fp32, all host
    threads) on ``seqs`` sequences of the workload; extrapolate to the full
    depth: t = t(1 layer) + (L-1) * (t(2) - t(1))."""
    from oracle import oracle as orc
    from paper_2601_15013_b200.shard import sub_batch

    sb = sub_batch(batch, np.arange(min(seqs, batch.num_sequences)))
    rng = np.random.default_rng(0)
    d, v = config.hidden_size, config.vocab_size
    uniq, tok_small = np.unique(sb.token_ids, return_inverse=True)
    params = {"embed": rng.uniform(-0.05, 0.05, size=(uniq.size, d)).astype(np.float32),
              "final_norm": np.ones(d, np.float32),
              "lm_head": rng.uniform(-0.05, 0.05, size=(v, d)).astype(np.float32)}
    for i in range(max(layers)):
        pre = f"layers.{i}."
        for nm, shp in (("wq", (config.q_dim, d)), ("wk", (config.kv_dim, d)), ("wv", (config.kv_dim, d)),
                        ("wo", (d, config.q_dim)), ("w_gate", (config.intermediate_size, d)),
                        ("w_up", (config.intermediate_size, d)), ("w_down", (d, config.intermediate_size))):
            params[pre + nm] = rng.uniform(-0.05, 0.05, size=shp).astype(np.float32)
        for nm, n in (("ln1", d), ("ln2", d), ("q_norm", config.head_dim), ("k_norm", config.head_dim)):
            params[pre + nm] = np.ones(n, np.float32)
    t0 = time.perf_counter()
    g, s, cp, m = orc.build_plan_oracle(sb.token_ids, sb.position_ids, sb.cu_seqlens)
    t_plan = time.perf_counter() - t0
    ts = {}
    for nl in layers:
        t0 = time.perf_counter()
        orc.forward_oracle(config, params, tok_small, sb.position_ids, sb.cu_seqlens, plan=(g, s, cp),
                           last_only=True, layers=nl)
        ts[nl] = time.perf_counter() - t0
    per_layer = max(ts[2] - ts[1], 1e-9)
    total = t_plan + ts[1] + (config.num_layers - 1) * per_layer
    try:
        from threadpoolctl import threadpool_info

        cores = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        cores = os.cpu_count() or 1
    return {"value": sb.num_tokens / total, "unit": "tokens/s", "cores": int(cores), "kind": "port",
            "sample": (f"{sb.num_sequences} seqs / {sb.num_tokens} tokens (N'={m}) of the workload; oracle "
                       f"plan + radix forward fp32, 1 and 2 layers timed, extrapolated to "
                       f"{config.num_layers} layers + last-token LM head over {config.vocab_size} vocab"),
            "seconds": round(ts[1] + ts[2] + t_plan, 2)}


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


def run_micro(args):
    """BASELINE configs[4]: index build and gather/scatter over ragged batches of
    1K-1M tokens (prefix-sharing ratios 0..1, multi-level tries): GPU planner
    time vs the CPU restatement of the reference trie (1 thread, as the
    reference's numba build), and row gather/scatter GB/s vs measured HBM."""
    import ctypes

    import torch

    from oracle import oracle as orc
    from paper_2601_15013_b200 import _native
    from paper_2601_15013_b200.plan import _WORKSPACE, build_plan_device, upload_batch
    from paper_2601_15013_b200.ops import gather_rows_device
    from paper_2601_15013_b200.workloads import multilevel_batch, prefix_ratio_batch

    torch.cuda.set_device(0)
    peaks, peaks_src = load_peaks()
    hbm = peaks["hbm_gbs"]
    lib = _native.lib()
    flush = L2Flusher()
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
        st = _native.stream_handle()

        def kernel_only():
            _native.check(lib.rdx_plan_build(tok.data_ptr(), pos.data_ptr(), cu.data_ptr(), b, nn, 0,
                                             gather.data_ptr(), scatter.data_ptr(), cpos.data_ptr(),
                                             info.data_ptr() + 16, lcp.data_ptr(), info.data_ptr(),
                                             scratch.data_ptr(), ctypes.c_size_t(scratch.numel()), st),
                          "rdx_plan_build")

        ms_kernel = _event_time(kernel_only, flush=flush)
        ms_api = _event_time(lambda: build_plan_device(tok, pos, cu), flush=flush)
        plan = build_plan_device(tok, pos, cu)
        t0 = time.perf_counter()
        reps = 0
        while True:
            g, sc, cp, m = orc.build_plan_oracle(batch.token_ids, batch.position_ids, batch.cu_seqlens)
            reps += 1
            if time.perf_counter() - t0 > 0.2 or reps >= 20:
                break
        cpu_ms = (time.perf_counter() - t0) * 1e3 / reps
        ok = (m == plan.n_compact and np.array_equal(plan.scatter.cpu().numpy().view(np.uint32), sc))
        nbytes = 12 * nn + 8 * plan.n_compact + 8 * (b + 1)
        plans.append({"case": name, "N": nn, "B": b, "N_compact": plan.n_compact,
                      "gamma": round(plan.n_compact / max(nn, 1), 4), "gpu_kernel_us": round(ms_kernel * 1e3, 1),
                      "gpu_api_us": round(ms_api * 1e3, 1), "cpu_ref_port_us": round(cpu_ms * 1e3, 1),
                      "speedup_kernel_vs_cpu": round(cpu_ms / ms_kernel, 1),
                      "index_gbs": round(nbytes / (ms_kernel * 1e-3) / 1e9, 1), "bit_exact_vs_oracle": bool(ok)})
        if name == "ratio0.50" or name == "multilevel":
            plans[-1]["_dev"] = (plan, nn)
    rows = []
    for rec in plans:
        dev = rec.pop("_dev", None)
        if dev is None or rec["N"] < (1 << 14):
            continue
        plan, nn = dev
        for d in (1024, 2560, 4096, 6144):
            x = torch.randn(plan.n_compact, d, device="cuda").to(torch.bfloat16)
            full = torch.empty(nn, d, dtype=torch.bfloat16, device="cuda")
            comp = torch.empty(plan.n_compact, d, dtype=torch.bfloat16, device="cuda")
            ms_s = _event_time(lambda: gather_rows_device(x, plan.scatter, out=full), flush=flush)
            ms_g = _event_time(lambda: gather_rows_device(full, plan.gather, out=comp), flush=flush)
            rb = 2 * d
            alg_s = nn * (2 * rb + 4)
            alg_g = plan.n_compact * (2 * rb + 4)
            uniq_s = plan.n_compact * rb + nn * rb + 4 * nn  # each compact row read once from DRAM
            rows.append({"case": rec["case"], "N": nn, "N_compact": plan.n_compact, "d": d,
                         "scatter_us": round(ms_s * 1e3, 1), "scatter_gbs": round(alg_s / (ms_s * 1e-3) / 1e9, 1),
                         "scatter_dram_gbs": round(uniq_s / (ms_s * 1e-3) / 1e9, 1),
                         "gather_us": round(ms_g * 1e3, 1), "gather_gbs": round(alg_g / (ms_g * 1e-3) / 1e9, 1)})
            del x, full, comp
    gather = gather_microbench(hbm)
    best = max(r["gather_gbs"] for r in rows) if rows else gather["gbs"]
    line = {"metric": "C5 index build + row gather/scatter microbenchmark", "value": round(best, 1),
            "unit": "GB/s", "n_gpus": 1, "higher_is_better": True, "dtype": "u32 indices / bf16 rows",
            "data": "synthetic", "config": {"workload": "c5: 1K-1M tokens, seq 512, prefix ratio 0..1, multi-level",
                                            "l2": "L2 flushed (256 MiB write) before each timed call"},
            "hbm_peak_gbs": hbm, "peak_source": peaks_src,
            "bytes_convention": "gather/scatter: 2*rows_out*row_bytes + 4*rows_out; index: 12N + 8N' + 8(B+1)",
            "index_build": plans, "row_ops": rows, "gather_table6": gather,
            "cpu_baseline": {"kind": "port", "cores": 1,
                             "sample": "oracle/trie_oracle.c (C restatement of trie.py:73-122), full batch"}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ arms
def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    config, model_name, batch, label = build_config(args.config, 1)
    samples = []
    for _ in range(args.warmup):
        cpu_sample(config, batch)
    for _ in range(args.steps):
        samples.append(cpu_sample(config, batch))
    vals = [s["value"] for s in samples]
    value = statistics.median(vals)
    s0 = samples[0]
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 2), "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": label, "model": model_name + " (random init)", "global_batch": batch.num_sequences,
                       "seq_tokens": batch.num_tokens, "parallelism": "cpu"},
            "cpu_baseline": {"value": round(value, 2), "unit": "tokens/s", "cores": s0["cores"], "kind": "port",
                             "sample": s0["sample"]},
            "e2e": {"value": round(value, 2), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "reference is pure Python (pkg/), not runnable on the GPU box; oracle/oracle.py is its port"}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2601_15013_b200 import DeviceBatch, DeviceWeights, RadixQwen3, _native, build_plan_device
    from paper_2601_15013_b200.rerank import RadixReranker
    from paper_2601_15013_b200.shard import gather_scores, partition_by_subtree

    peaks, peaks_src = load_peaks()
    config, model_name, global_batch, label = build_config(args.config, world)
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
    n_tok, n_comp = db.n, plan.n_compact
    tokens_all = max_over_ranks(0, 1) + global_batch.num_tokens

    # launches per step (our C-ABI kernels)
    step_radix()  # captures the CUDA graph (if enabled) outside the count
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
    sampler = ClockSampler(local) if rank == 0 else None
    ms_radix, per_radix, clocks = time_steps(step_radix, args.steps, args.warmup, world, flush, sampler)
    ms_base, per_base, _ = time_steps(step_base, args.steps, args.warmup, world, flush)
    value = tokens_all * args.steps / (ms_radix * 1e-3)
    value_base = tokens_all * args.steps / (ms_base * 1e-3)

    # e2e through the public API (host buffers, H2D + D2H inside the timed region)
    host_batch = mine.batch

    def e2e_step():
        s = rr.score(host_batch)
        if world > 1:
            finish(torch.from_numpy(s).cuda()).cpu()
        return s

    ms_e2e_seq = time_wall_steps(e2e_step, args.steps, args.warmup, world)

    # the same K host batches through the streaming API (RadixReranker.score_many): batch t+1's
    # H2D copy and GPU plan build overlap batch t's prefill (pipeline.score_stream)
    def e2e_stream():
        outs = rr.score_many([host_batch] * args.steps)
        if world > 1:
            for s in outs:
                finish(torch.from_numpy(s).cuda()).cpu()

    rr.score_many([host_batch] * max(args.warmup, 1))
    barrier(world)
    t0 = time.perf_counter()
    e2e_stream()
    torch.cuda.synchronize()
    ms_e2e = max_over_ranks((time.perf_counter() - t0) * 1e3, world)
    barrier(world)
    e2e_value = tokens_all * args.steps / (ms_e2e * 1e-3)
    e2e_seq_value = tokens_all * args.steps / (ms_e2e_seq * 1e-3)

    roof, gemm_ms_per_step, breakdown = op_breakdown(model, step_radix, max(3, min(args.steps, 10)),
                                                     peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]))
    roof["peak_source"] = f"{peaks_src} bf16_tflops_sustained (kernels inside a long step)"
    roof["gemm_share_of_step"] = round(gemm_ms_per_step / (ms_radix / args.steps), 3)
    tr = ncu_traffic(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                  f"r1_ncu_gemm_gateup_{args.config}.txt"))
    if tr is not None:  # DRAM bytes of one gate_up launch (the largest GEMM) from the committed ncu capture
        roof["traffic"] = tr[0]
        roof["traffic_source"] = f"profiles/r1_ncu_gemm_gateup_{args.config}.txt ({tr[1]}; dram read+write, 1 launch)"
    _, _, breakdown_base = op_breakdown(model, step_base, 3, 1.0)

    gather = gather_microbench(peaks["hbm_gbs"]) if rank == 0 else None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_sample(config, global_batch)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_radix / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights)",
            "config": {"workload": label, "model": model_name, "global_batch": global_batch.num_sequences,
                       "tokens_per_step": int(tokens_all), "n_compact_rank0": int(n_comp),
                       "gamma_rank0": round(n_comp / n_tok, 4), "parallelism": f"dp{world} (trie-subtree shards)",
                       "logits": "last-token, full vocab", "attention": "suffix-query (rdx_attention, tcgen05)",
                       "cuda_graphs": not args.no_graphs,
                       "l2": "L2 flushed (256 MiB write) between timed steps"},
            "nodedup": {"value": round(value_base, 1), "ms_per_step": round(ms_base / args.steps, 4)},
            "speedup_vs_nodedup": round(value / value_base, 3),
            "e2e": {"value": round(e2e_value, 1), "unit": "tokens/s", "h2d_bytes_per_step": int(rr.h2d_bytes),
                    "d2h_bytes_per_step": int(rr.d2h_bytes), "ms_per_step": round(ms_e2e / args.steps, 4),
                    "api": "RadixReranker.score_many (pipelined stream of K host batches)",
                    "sequential": {"value": round(e2e_seq_value, 1), "api": "RadixReranker.score per batch",
                                   "ms_per_step": round(ms_e2e_seq / args.steps, 4)}},
            "roofline": roof,
            "breakdown_us_radix": breakdown,
            "breakdown_us_nodedup": {k: v["us_per_step"] for k, v in breakdown_base.items()},
            "cpu_baseline": cpu,
            "gather": gather,
            "gpu_launches": int(launches_per_step * args.steps),
            "gpu_launches_note": "our C-ABI kernels per timed region (radix arm), counted at the C ABI",
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--profile", action="store_true", help="radix steps only, for ncu")
    ap.add_argument("--no-graphs", action="store_true", help="eager launches instead of CUDA-graph replay")
    ap.add_argument("--fused-norm", action="store_true", help="RMSNorm fused into the GEMMs (RDX_EPI_RESID_NORM A/B)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.config == "c5" and args.impl == "ours":
        run_micro(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
