"""Pipelined scheduling (reference bench.py:346-405 pipelined_run).

CPU tests: the producer/consumer contract with a host plan builder (identical
results to sequential, WorkerPanic with the batch index, producer errors
re-raised).  GPU tests: the planner as producer, and RadixReranker.score_many
(side-stream upload + plan build overlapping the prefill) == score() per batch."""

import numpy as np
import pytest


def _batches(n=5):
    from paper_2601_15013_b200.workloads import SyntheticSpec, make_synthetic_batch

    return [make_synthetic_batch(SyntheticSpec(B=4 + i, prefix_len=8 + i, suffix_len=4, vocab=64, seed=i))
            for i in range(n)]


def _host_planner(batch):
    from oracle import oracle as orc

    return orc.build_plan_oracle(batch.token_ids, batch.position_ids, batch.cu_seqlens)


def test_pipelined_run_matches_sequential_cpu():
    from paper_2601_15013_b200 import pipelined_run

    batches = _batches()
    seen = []
    rep = pipelined_run(batches, lambda b, p: seen.append(p), plan_builder=_host_planner)
    assert len(seen) == len(batches) and rep.tokens == sum(b.num_tokens for b in batches)
    for b, p in zip(batches, seen):
        ref = _host_planner(b)
        assert all(np.array_equal(x, y) for x, y in zip(p[:3], ref[:3])) and p[3] == ref[3]
    assert 0.0 <= rep.hidden_fraction <= 1.0 and rep.tokens_per_s > 0


def test_pipelined_run_errors_cpu():
    from paper_2601_15013_b200 import pipelined_run
    from paper_2601_15013_b200.errors import WorkerPanic

    batches = _batches(4)

    def worker(b, p):
        if b is batches[2]:
            raise RuntimeError("boom")

    with pytest.raises(WorkerPanic) as ei:
        pipelined_run(batches, worker, plan_builder=_host_planner)
    assert ei.value.batch_index == 2

    def bad_builder(b):
        raise ValueError("planner failed")

    with pytest.raises(ValueError):
        pipelined_run(batches, lambda b, p: None, plan_builder=bad_builder)


@pytest.mark.gpu
def test_pipelined_run_gpu_planner():
    from paper_2601_15013_b200 import build_plan, pipelined_run

    batches = _batches()
    got = []
    pipelined_run(batches, lambda b, p: got.append(p))  # default plan_builder = GPU build_plan
    for b, p in zip(batches, got):
        ref = _host_planner(b)
        assert np.array_equal(p.scatter_indices, ref[1]) and p.n_compact == ref[3]
        assert np.array_equal(build_plan(b).gather_indices, p.gather_indices)


@pytest.mark.gpu
@pytest.mark.parametrize("graphs", [False, True])
def test_score_many_equals_score(graphs):
    from paper_2601_15013_b200 import TINY_C1, DeviceWeights, RadixQwen3
    from paper_2601_15013_b200.rerank import RadixReranker
    from paper_2601_15013_b200.workloads import RerankSpec, msmarco_rerank_batch

    model = RadixQwen3(TINY_C1, DeviceWeights.random(TINY_C1, seed=1), use_graphs=graphs)
    rr = RadixReranker(model)
    batches = [msmarco_rerank_batch(RerankSpec(queries=1, passages_per_query=6 + (i % 3), template_len=12,
                                               query_len=10, passage_min=20, passage_max=40, tail_len=5,
                                               vocab=1000, seed=i)) for i in range(6)]
    seq = [rr.score(b) for b in batches]
    pipe = rr.score_many(batches)
    assert len(pipe) == len(seq)
    for a, b in zip(seq, pipe):
        assert a.shape == b.shape and np.array_equal(a, b)
