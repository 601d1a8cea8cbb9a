"""Host-side breakdown of one build_plan_device call at C2 (perf_counter_ns, median of 200):
allocation, launch submit, stream sync, result slicing.  python scripts/plan_api_breakdown.py"""
import ctypes
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2601_15013_b200 import _native  # noqa: E402
from paper_2601_15013_b200.plan import _WORKSPACE, _info_buffer, build_plan_device, upload_batch  # noqa: E402

b = bench.workload("c2", 1, "weak")[2]
tok, pos, cu = upload_batch(b)
lib = _native.lib()
for _ in range(20):
    build_plan_device(tok, pos, cu)
torch.cuda.synchronize()
n, nb = int(tok.shape[0]), int(cu.shape[0]) - 1
sb = int(lib.rdx_plan_scratch_bytes(n, nb))
parts = {k: [] for k in ("alloc", "submit", "sync", "slices", "total")}
for _ in range(200):
    t0 = time.perf_counter_ns()
    buf = torch.empty(3 * n + (nb + 1) + nb, dtype=torch.int32, device="cuda")
    scratch = _WORKSPACE.get(tok.device, sb)
    sh = torch._C._cuda_getCurrentRawStream(0)
    info, iv = _info_buffer()
    iv[1] = -1
    t1 = time.perf_counter_ns()
    p0 = buf.data_ptr()
    o = 3 * n
    lib.rdx_plan_build(tok.data_ptr(), pos.data_ptr(), cu.data_ptr(), nb, n, 0, p0, p0 + 4 * n, p0 + 8 * n,
                       p0 + 4 * o, p0 + 4 * (o + nb + 1), info.data_ptr(), scratch.data_ptr(),
                       ctypes.c_size_t(scratch.numel()), sh)
    t2 = time.perf_counter_ns()
    lib.rdx_stream_synchronize(sh)
    t3 = time.perf_counter_ns()
    m = int(iv[0])
    views = buf.split([m, n - m, n, 0, m, n - m, nb + 1, nb])
    t4 = time.perf_counter_ns()
    for k, v in zip(parts, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0)):
        v and parts[k].append(v / 1e3)
print("C2 build_plan_device parts (us, median):", {k: round(statistics.median(v), 1) for k, v in parts.items()})
t0 = time.perf_counter()
for _ in range(200):
    build_plan_device(tok, pos, cu)
print("build_plan_device us:", round((time.perf_counter() - t0) / 200 * 1e6, 1))
