"""Phase timestamps (%globaltimer) of the cluster-resident planner at the C2/C3 shapes.
python scripts/plan_trace.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2601_15013_b200 import _native  # noqa: E402
from paper_2601_15013_b200.plan import build_plan_device, upload_batch  # noqa: E402

lib = _native.lib()
buf = torch.zeros(64, dtype=torch.int64, device="cuda")
names = ["start", "staged", "B1", "P0", "B2", "P2", "B3", "P3", "B4", "P4", "P5", "end"]
from paper_2601_15013_b200.workloads import prefix_ratio_batch  # noqa: E402

cases = [(name, bench.workload(name, 1, "weak")[2]) for name in ("c2", "c3")]
cases += [(f"{n // 1024}K", prefix_ratio_batch(n, 0.5)) for n in (1024, 4096)]
for name, b in cases:
    tok, pos, cu = upload_batch(b)
    for _ in range(5):
        build_plan_device(tok, pos, cu)
    lib.rdx_plan_debug_trace(buf.data_ptr())
    for _ in range(3):
        buf.zero_()
        build_plan_device(tok, pos, cu)
    lib.rdx_plan_debug_trace(None)
    t = buf.cpu().tolist()
    t0 = t[0]
    starts = [x - t0 for x in t[16:32] if x]
    print(name, "CTA starts (ns rel. CTA 0):", starts)
    print(name, " ".join(f"{names[k]}={(t[k] - t0) / 1e3:.2f}" for k in range(12) if t[k]), "us")
    for nm, off in (("P2 end", 32), ("P3 end", 48)):
        v = [(x - t0) / 1e3 for x in t[off:off + 16] if x]
        print(name, f"per-CTA {nm} (us):", " ".join(f"{x:.2f}" for x in v))
