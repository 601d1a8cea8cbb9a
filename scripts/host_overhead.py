"""Host-side cost of one C2 score_device step: plan build (+ its one sync), prefill launch path, read-out."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2601_15013_b200 import DeviceBatch, DeviceWeights, RadixQwen3  # noqa: E402
from paper_2601_15013_b200.rerank import RadixReranker  # noqa: E402

config, _, batch, _ = bench.workload("c2", 1, "weak")
rr = RadixReranker(RadixQwen3(config, DeviceWeights.random(config, seed=0), use_graphs=True))
db = DeviceBatch.from_batch(batch)
for _ in range(5):
    rr.score_device(db)
torch.cuda.synchronize()
T = {"plan": 0.0, "prefill_host": 0.0, "scores_host": 0.0}
n = 20
for _ in range(n):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = rr.plan(db)
    t1 = time.perf_counter()
    logits = rr.model.prefill(db, plan, attention=rr.attention, logits="last")
    t2 = time.perf_counter()
    s = torch.empty(db.b, dtype=torch.float32, device=logits.device)
    rr.model  # noqa
    from paper_2601_15013_b200 import _native
    _native.lib().rdx_rerank_scores(logits.data_ptr(), db.b, logits.stride(0), rr.yes_id, rr.no_id, s.data_ptr(),
                                    _native.stream_handle())
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    T["plan"] += t1 - t0
    T["prefill_host"] += t2 - t1
    T["scores_host"] += t3 - t2
print({k: round(v / n * 1e6, 1) for k, v in T.items()}, "us per step (host)")
