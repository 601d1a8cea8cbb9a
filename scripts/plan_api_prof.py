import time, torch, sys, os
sys.path.insert(0, '/root/repo')
import bench
from paper_2601_15013_b200.plan import build_plan_device, upload_batch
b = bench.workload("c2", 1, "weak")[2]
tok, pos, cu = upload_batch(b)
for _ in range(20): build_plan_device(tok, pos, cu)
torch.cuda.synchronize()
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(200): build_plan_device(tok, pos, cu)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
t0=time.perf_counter()
for _ in range(200): build_plan_device(tok, pos, cu)
print("api us", (time.perf_counter()-t0)/200*1e6)
