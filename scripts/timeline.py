"""Kernel timeline of CUDA-graph prefill steps via torch.profiler (CUPTI activity
records: one record per kernel node, start/end on the GPU clock).  Prints per-kernel
duration, the gap to the previous kernel's end (negative = overlap), and the per-kind
totals of one step, so exposed (critical-path) time can be told from overlapped time.

  python scripts/timeline.py [c2|c3|c4] [--json out.json]
"""
import json
import os
import sys
from collections import defaultdict

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2601_15013_b200 import DeviceBatch, DeviceWeights, RadixQwen3  # noqa: E402
from paper_2601_15013_b200.rerank import RadixReranker  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "c2"
config, _, batch, _ = bench.workload(cfg_name, 1, "weak")
rr = RadixReranker(RadixQwen3(config, DeviceWeights.random(config, seed=0), use_graphs=True))
db = DeviceBatch.from_batch(batch)
for _ in range(4):
    rr.score_device(db)
torch.cuda.synchronize()
flush = bench.L2Flusher()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        flush()
        rr.score_device(db)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
kern = []
for e in evs:
    nm = e.name
    if "Memcpy" in nm or "Memset" in nm:
        continue
    kern.append((e.time_range.start, e.time_range.end, nm))
kern.sort()


def kind(nm):
    if "gemm_kernel" in nm:
        return "gemm<" + nm.split("gemm_kernel<")[1].split(">")[0] + ">"
    for k in ("attention_kernel", "rmsnorm_rows_after", "rmsnorm_rows", "embed_rmsnorm", "plan_build", "rerank",
              "fill", "elementwise", "flush"):
        if k in nm:
            return k
    return nm[:40]


# the second step: from the last flush kernel on
idx = [i for i, k in enumerate(kern) if "fill" in k[2].lower() or "elementwise" in k[2].lower()]
start = idx[-1] + 1 if idx else len(kern) // 2
step = kern[start:]
tot = defaultdict(float)
cnt = defaultdict(int)
exposed = defaultdict(float)
prev_end = step[0][0]
for s, e, nm in step:
    k = kind(nm)
    tot[k] += e - s
    cnt[k] += 1
    exposed[k] += max(0.0, e - max(s, prev_end))  # time this kernel extends the busy frontier
    prev_end = max(prev_end, e)
span = step[-1][1] - step[0][0]
print(f"{cfg_name}: {len(step)} kernels, span {span:.1f} us (first start -> last end)")
print(f"{'kind':28s} {'n':>4s} {'sum_us':>9s} {'avg_us':>8s} {'exposed_us':>10s}")
for k in sorted(tot, key=lambda x: -exposed[x]):
    print(f"{k:28s} {cnt[k]:4d} {tot[k]:9.1f} {tot[k] / cnt[k]:8.2f} {exposed[k]:10.1f}")
gaps = sum(max(0.0, step[i][0] - max(e for _, e, _ in step[:i])) for i in range(1, len(step)))
print(f"idle gaps between kernels: {gaps:.1f} us")
print("first layer:")
for s, e, nm in step[:10]:
    print(f"  {s - step[0][0]:9.1f} {e - s:8.1f}  {kind(nm)}")
if "--json" in sys.argv:
    with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
        json.dump([{"start_us": s - step[0][0], "dur_us": e - s, "kernel": kind(nm)} for s, e, nm in step], f)
