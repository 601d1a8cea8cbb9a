"""Does running two half-batches on two streams (CUDA graphs) fill each other's kernel tails?

full: the C2 batch as one graph; seq: two half-batch graphs back to back on one stream;
conc: the two half graphs on two streams."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_15013_b200 import DeviceBatch, DeviceWeights, RadixQwen3  # noqa: E402
from paper_2601_15013_b200.model import QWEN3_PRESETS  # noqa: E402
from paper_2601_15013_b200.rerank import RadixReranker  # noqa: E402
from paper_2601_15013_b200.shard import partition_by_subtree  # noqa: E402
from paper_2601_15013_b200.workloads import RerankSpec, msmarco_rerank_batch  # noqa: E402

cfg = QWEN3_PRESETS[os.environ.get("MODEL", "qwen3-0.6b")]
w = DeviceWeights.random(cfg, seed=0)
batch = msmarco_rerank_batch(RerankSpec(queries=int(os.environ.get("Q", "1")), passages_per_query=64))
halves = [s.batch for s in partition_by_subtree(batch, 2)]
runs = []
for b in [batch] + halves:
    m = RadixQwen3(cfg, w, use_graphs=True)
    rr = RadixReranker(m)
    db = DeviceBatch.from_batch(b)
    plan = rr.plan(db)
    runs.append((rr, db, plan))
    print("rows", b.num_tokens, "compact", plan.n_compact, flush=True)


def step(i):
    rr, db, plan = runs[i]
    return rr.score_device(db, plan=plan)


s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def full():
    step(0)


def seq():
    step(1)
    step(2)


def conc():
    main = torch.cuda.current_stream()
    s1.wait_stream(main)
    s2.wait_stream(main)
    with torch.cuda.stream(s1):
        step(1)
    with torch.cuda.stream(s2):
        step(2)
    main.wait_stream(s1)
    main.wait_stream(s2)


def timeit(fn, it=30):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / it


for rep in range(2):
    print({name: round(timeit(f), 3) for name, f in (("full", full), ("seq", seq), ("conc", conc))}, flush=True)
