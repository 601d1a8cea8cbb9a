"""Kernel timeline of one C2 CUDA-graph step (torch.profiler / CUPTI): busy time, idle gaps between
kernels, and the largest gaps by the kernel pair around them."""
import collections
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2601_15013_b200 import DeviceBatch, DeviceWeights, RadixQwen3  # noqa: E402
from paper_2601_15013_b200.rerank import RadixReranker  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
config, _, batch, _ = bench.workload(cfg_name, 1, "weak")
rr = RadixReranker(RadixQwen3(config, DeviceWeights.random(config, seed=0), use_graphs=True))
db = DeviceBatch.from_batch(batch)
plan = rr.plan(db)
for _ in range(5):
    rr.score_device(db, plan=plan)
torch.cuda.synchronize()
a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a_ev.record()
for _ in range(20):
    rr.score_device(db, plan=plan)
b_ev.record()
b_ev.synchronize()
print(f"event-timed step (precomputed plan, back to back): {a_ev.elapsed_time(b_ev) / 20:.3f} ms")
a_ev.record()
for _ in range(20):
    rr.score_device(db)
b_ev.record()
b_ev.synchronize()
print(f"event-timed step (plan built each step): {a_ev.elapsed_time(b_ev) / 20:.3f} ms")
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        rr.score_device(db, plan=plan)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.end > e.time_range.start]
ev.sort(key=lambda e: e.time_range.start)
# keep the last step: split at gaps > 200 us
steps, cur = [], [ev[0]]
for a, b in zip(ev, ev[1:]):
    if b.time_range.start - a.time_range.end > 200:
        steps.append(cur)
        cur = []
    cur.append(b)
steps.append(cur)
print("kernels per profiled chunk:", [len(x) for x in steps])
st = max(steps, key=len)
t0, t1 = st[0].time_range.start, max(e.time_range.end for e in st)
busy = sum(e.time_range.end - e.time_range.start for e in st)
gaps = []
for a, b in zip(st, st[1:]):
    g = b.time_range.start - a.time_range.end
    gaps.append((g, a.name[:40], b.name[:40]))
print(f"{cfg_name}: kernels {len(st)}  span {t1 - t0:.1f} us  busy {busy:.1f} us  idle {t1 - t0 - busy:.1f} us "
      f"({100 * (1 - busy / (t1 - t0)):.1f} %)")
agg = collections.defaultdict(lambda: [0, 0.0])
for g, a, b in gaps:
    k = (a.split("<")[0].split("(")[0][-28:], b.split("<")[0].split("(")[0][-28:])
    agg[k][0] += 1
    agg[k][1] += g
for k, (n, tot) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:12]:
    print(f"  {n:4d} x  {tot / n:6.2f} us  total {tot:8.1f} us   {k[0]} -> {k[1]}")
