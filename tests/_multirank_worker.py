"""torchrun worker for tests/test_multirank_gpu.py: every rank on cuda:0 (one GPU box),
gloo for the score all-gather.  Rank r scores its trie-subtree shard with the real
RadixReranker (GPU planner + tcgen05 prefill); rank 0 compares the gathered scores with
one single-process pass over the whole batch and writes the verdict."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2601_15013_b200 import DeviceWeights, RadixQwen3  # noqa: E402
from paper_2601_15013_b200.model import Qwen3Config  # noqa: E402
from paper_2601_15013_b200.rerank import RadixReranker  # noqa: E402
from paper_2601_15013_b200.shard import partition_by_subtree, score_sharded, shard_report  # noqa: E402
from paper_2601_15013_b200.workloads import RerankSpec, long_prefix_batch, msmarco_rerank_batch  # noqa: E402


def main(out_path):
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    cfg = Qwen3Config(2, 512, 1024, 8, 4, 64, 8192, 1e6, 1e-6)
    model = RadixQwen3(cfg, DeviceWeights.random(cfg, seed=1), use_graphs=True)
    rr = RadixReranker(model)
    results = {}
    for name, batch in (("rerank_3q", msmarco_rerank_batch(RerankSpec(queries=3, passages_per_query=12, vocab=8192))),
                        ("long_prefix", long_prefix_batch(B=8, prefix_len=300, suffix_len=40, vocab=8192))):
        shards = partition_by_subtree(batch, world)
        got = score_sharded(batch, lambda b: torch.from_numpy(rr.score(b)).cuda(), shards=shards).cpu().numpy()
        if rank == 0:
            want = rr.score(batch)
            results[name] = {"bit_identical": bool(np.array_equal(got, want)),
                             "maxabs": float(np.abs(got - want).max()), "shards": shard_report(shards)}
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump(results, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
