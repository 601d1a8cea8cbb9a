"""GPU planner on the benchmark batches: kernel time (CUDA events), API time (build_plan_device,
including its one D2H read), reference numba build_plan (baseline/_ref) beside it.
python scripts/plan_bench.py"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2601_15013_b200 import _native  # noqa: E402
from paper_2601_15013_b200.plan import _WORKSPACE, build_plan_device, upload_batch  # noqa: E402

lib = _native.lib()
flush = bench.L2Flusher()
ref = bench.import_reference()
for name in ("c2", "c2_literal", "c3", "c4"):  # c5 sizes: bench.py --config c5
    batch = bench.workload(name, 1, "weak")[2]
    tok, pos, cu = upload_batch(batch)
    b, nn = int(cu.shape[0]) - 1, int(tok.shape[0])
    gather, scatter, cpos = (torch.empty(nn, dtype=torch.int32, device="cuda") for _ in range(3))
    info = torch.empty(4 + b + 1, dtype=torch.int32, device="cuda")
    lcp = torch.empty(max(b, 1), dtype=torch.int32, device="cuda")
    scratch = _WORKSPACE.get(tok.device, int(lib.rdx_plan_scratch_bytes(nn, b)))
    st = _native.stream_handle()

    def kernel_only():
        _native.check(lib.rdx_plan_build(tok.data_ptr(), pos.data_ptr(), cu.data_ptr(), b, nn, 0, gather.data_ptr(),
                                         scatter.data_ptr(), cpos.data_ptr(), info.data_ptr() + 16, lcp.data_ptr(),
                                         info.data_ptr(), scratch.data_ptr(), ctypes.c_size_t(scratch.numel()), st),
                      "rdx_plan_build")

    def graph_time(reps=20):
        # device time per launch without host submission in the way: `reps` launches
        # captured in one CUDA graph, replayed (L2 warm between launches)
        s2 = torch.cuda.Stream()
        with torch.cuda.stream(s2):
            kernel_only()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s2):
                for _ in range(reps):
                    _native.check(lib.rdx_plan_build(tok.data_ptr(), pos.data_ptr(), cu.data_ptr(), b, nn, 0,
                                                     gather.data_ptr(), scatter.data_ptr(), cpos.data_ptr(),
                                                     info.data_ptr() + 16, lcp.data_ptr(), info.data_ptr(),
                                                     scratch.data_ptr(), ctypes.c_size_t(scratch.numel()),
                                                     _native.stream_handle(s2)), "plan")
            g.replay()
            torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s2)
                g.replay()
                e1.record(s2)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3 / reps)
        return sorted(ts)[2]

    gk = graph_time()
    prev = lib.rdx_plan_debug_smem(0)
    gk_l2 = graph_time()
    lib.rdx_plan_debug_smem(prev)
    import time as _t
    t0 = _t.perf_counter()
    for _ in range(50):
        kernel_only()
    host_launch = (_t.perf_counter() - t0) / 50 * 1e6
    torch.cuda.synchronize()
    print(f"{name:11s} device time per launch (CUDA graph of 20): cluster-smem {gk:6.1f} us, L2-resident {gk_l2:6.1f} us;"
          f" host submit of one rdx_plan_build via ctypes {host_launch:6.1f} us", flush=True)
    prev = lib.rdx_plan_debug_smem(0)
    k_l2 = bench._event_time(kernel_only, iters=20, flush=flush) * 1e3
    lib.rdx_plan_debug_smem(prev)
    k = bench._event_time(kernel_only, iters=20, flush=flush) * 1e3
    k_warm = bench._event_time(kernel_only, iters=20) * 1e3
    api = bench._event_time(lambda: build_plan_device(tok, pos, cu), iters=20, flush=flush) * 1e3
    line = (f"{name:11s} N={nn:7d} kernel {k:7.1f} us (L2 warm {k_warm:6.1f}; L2-resident planner {k_l2:6.1f})"
            f"  api {api:7.1f} us")
    if ref is not None:
        rb = ref.RaggedBatch(batch.token_ids, batch.position_ids, batch.cu_seqlens)
        t = bench._median_time(lambda: ref.trie.build_plan(rb)) * 1e6
        line += f"  reference numba {t:8.1f} us  (kernel {t / k:5.1f}x, api {t / api:5.1f}x)"
    print(line, flush=True)
