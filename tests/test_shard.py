"""Multi-GPU partitioning by trie subtree, host logic + the final
all-gather, exercised with world_size 2 on the gloo backend (CPU)."""

import os
import socket

import numpy as np
import pytest


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_partition_covers_every_sequence_once():
    from paper_2601_15013_b200.shard import partition_by_subtree
    from paper_2601_15013_b200.workloads import RerankSpec, msmarco_rerank_batch

    b = msmarco_rerank_batch(RerankSpec(queries=4, passages_per_query=16, vocab=5000))
    for world in (1, 2, 3, 4, 8):
        shards = partition_by_subtree(b, world)
        ids = np.sort(np.concatenate([s.seq_ids for s in shards]))
        assert np.array_equal(ids, np.arange(b.num_sequences))
        assert sum(s.batch.num_tokens for s in shards) == b.num_tokens


def test_cuts_land_between_query_subtrees(oracle):
    """4 queries behind a shared template: 4 shards = 4 query subtrees, only the template is duplicated."""
    from paper_2601_15013_b200.shard import partition_by_subtree
    from paper_2601_15013_b200.workloads import RerankSpec, msmarco_rerank_batch

    spec = RerankSpec(queries=4, passages_per_query=16, vocab=5000)
    b = msmarco_rerank_batch(spec)
    m_global = oracle.build_plan_oracle(b.token_ids, b.position_ids, b.cu_seqlens)[3]
    shards = partition_by_subtree(b, 4)
    m_sum = 0
    for s in shards:
        assert s.seq_ids.size == 16
        q = set((s.seq_ids // 16).tolist())
        assert len(q) == 1  # one query subtree per shard
        m = oracle.build_plan_oracle(s.batch.token_ids, s.batch.position_ids, s.batch.cu_seqlens)[3]
        assert m == s.est_compact_rows
        m_sum += m
    assert m_sum - m_global == 3 * spec.template_len


def test_distinct_roots_no_duplication(oracle):
    from paper_2601_15013_b200.ragged import RaggedBatch, default_positions
    from paper_2601_15013_b200.shard import partition_by_subtree

    rng = np.random.default_rng(0)
    seqs = []
    for root in range(6):
        stem = rng.integers(0, 50, size=10)
        for _ in range(5):
            seqs.append(np.concatenate([[1000 + root], stem, rng.integers(0, 50, size=7)]))
    cu = np.cumsum([0] + [len(x) for x in seqs])
    b = RaggedBatch(np.concatenate(seqs), default_positions(cu), cu)
    m_global = oracle.build_plan_oracle(b.token_ids, b.position_ids, b.cu_seqlens)[3]
    shards = partition_by_subtree(b, 3)
    total = sum(oracle.build_plan_oracle(s.batch.token_ids, s.batch.position_ids, s.batch.cu_seqlens)[3]
                for s in shards)
    assert total == m_global


def _worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist

    from paper_2601_15013_b200.shard import gather_scores, partition_by_subtree
    from paper_2601_15013_b200.workloads import RerankSpec, msmarco_rerank_batch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b = msmarco_rerank_batch(RerankSpec(queries=2, passages_per_query=8, vocab=3000))
    mine = partition_by_subtree(b, world)[rank]
    # stand-in per-sequence score: a deterministic function of the sequence tokens
    cu = mine.batch.cu_seqlens
    local = torch.tensor([float(mine.batch.token_ids[cu[i]:cu[i + 1]].astype(np.int64).sum() % 9973)
                          for i in range(mine.batch.num_sequences)], dtype=torch.float32)
    out = gather_scores(local, mine.seq_ids, b.num_sequences)
    if rank == 0:
        np.save(result_path, out.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_gather_scores_world2_gloo(tmp_path):
    import torch.multiprocessing as mp

    from paper_2601_15013_b200.workloads import RerankSpec, msmarco_rerank_batch

    path = str(tmp_path / "scores.npy")
    mp.spawn(_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    got = np.load(path)
    b = msmarco_rerank_batch(RerankSpec(queries=2, passages_per_query=8, vocab=3000))
    cu = b.cu_seqlens
    want = np.array([float(b.token_ids[cu[i]:cu[i + 1]].astype(np.int64).sum() % 9973)
                     for i in range(b.num_sequences)], dtype=np.float32)
    assert np.array_equal(got, want)


def _brute_makespan(lens, lcps, world):
    """Exhaustive minimum over all contiguous splits (small cases)."""
    import itertools

    b = len(lens)
    best = None
    for cut in itertools.combinations(range(1, b), world - 1):
        cuts = [0, *cut, b]
        costs = []
        for r in range(world):
            lo, hi = cuts[r], cuts[r + 1]
            costs.append(int(lens[lo:hi].sum() - lcps[lo:hi - 1].sum()))
        mk = max(costs)
        best = mk if best is None else min(best, mk)
    return best


def test_partition_minimises_makespan():
    from paper_2601_15013_b200.shard import _makespan_cuts

    rng = np.random.default_rng(4)
    for _ in range(40):
        b = int(rng.integers(2, 9))
        world = int(rng.integers(1, b + 1))
        lens = rng.integers(5, 40, size=b)
        lcps = np.array([rng.integers(0, min(lens[i], lens[i + 1]) + 1) for i in range(b - 1)], dtype=np.int64)
        cuts = _makespan_cuts(lens.astype(np.int64), lcps, world)
        assert cuts[0] == 0 and cuts[-1] == b and all(cuts[i] < cuts[i + 1] for i in range(world))
        costs = [int(lens[cuts[r]:cuts[r + 1]].sum() - lcps[cuts[r]:cuts[r + 1] - 1].sum()) for r in range(world)]
        assert max(costs) == _brute_makespan(lens, lcps, world)


def test_strong_scaling_shards_balanced_c4():
    """C4 (128 x (2048 + 256)) at 8 GPUs: 16 sequences each, N'_g = 2048 + 16*256."""
    from paper_2601_15013_b200.shard import partition_by_subtree, shard_report
    from paper_2601_15013_b200.workloads import long_prefix_batch

    rep = shard_report(partition_by_subtree(long_prefix_batch(seed=0), 8))
    assert [r["sequences"] for r in rep] == [16] * 8
    assert all(r["N_compact"] == 2048 + 16 * 256 for r in rep)


@pytest.mark.parametrize("argv", [["--gpus", "2"], ["--gpus", "4", "--config", "c4"],
                                  ["--gpus", "3", "--config", "c3"]])
def test_bench_launcher_selftest(argv):
    """bench.py --gpus N re-executes itself under torch.distributed.run (N ranks, gloo here),
    partitions the workload by trie subtree and all-gathers per-sequence scores."""
    import json
    import subprocess
    import sys

    from conftest import ROOT

    r = subprocess.run([sys.executable, "bench.py", *argv, "--selftest-launcher"], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["ok"] and line["n_ranks"] == int(argv[1])
    assert sum(s["sequences"] for s in line["shards"]) == line["global_batch"]
