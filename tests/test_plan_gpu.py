"""GPU planner parity: rdx_plan_build vs the reference's golden plans and the C oracle.

Bit-exact for every index (gather, scatter, compact_positions, N').  Sizes
up to 1M tokens are checked against the oracle trie; the long-prefix C4
shape is checked through its closed form N' = P + B*S and the plan
invariants (tests/test_trie.py:95-112 of the reference).
"""

import numpy as np
import pytest

from conftest import unpack

pytestmark = pytest.mark.gpu


def _gpu_plan(tok, pos, cu, allow_empty=False):
    from paper_2601_15013_b200 import RaggedBatch, build_plan

    return build_plan(RaggedBatch(tok, pos, cu), allow_empty=allow_empty)


def _assert_plan(plan, gather, scatter, m, pos=None):
    assert plan.n_compact == m
    np.testing.assert_array_equal(plan.gather_indices, gather)
    np.testing.assert_array_equal(plan.scatter_indices, scatter)
    if pos is not None:
        np.testing.assert_array_equal(plan.compact_positions, np.asarray(pos)[np.asarray(gather, np.int64)])


@pytest.mark.parametrize("prefix", ["known", "rand", "arbpos", "pattern"])
def test_golden_plans_bit_exact(golden_plans, prefix):
    count = 0
    for tok, pos, cu, gather, scatter, m in unpack(golden_plans, prefix):
        _assert_plan(_gpu_plan(tok, pos, cu), gather, scatter, m, pos)
        count += 1
    assert count > 0


def test_toy_known_answer():
    plan = _gpu_plan(np.array([1, 2, 3, 1, 2, 4]), np.array([0, 1, 2, 0, 1, 2]), np.array([0, 3, 6]))
    assert plan.gather_indices.tolist() == [0, 1, 2, 5]
    assert plan.scatter_indices.tolist() == [0, 1, 2, 0, 1, 3]
    assert plan.compact_positions.tolist() == [0, 1, 2, 2]
    assert plan.gamma == pytest.approx(4 / 6)


def test_table_rows(golden_plans):
    from paper_2601_15013_b200.workloads import SyntheticSpec, make_synthetic_batch

    for p, s, n, m in golden_plans["table"]:
        b = make_synthetic_batch(SyntheticSpec(B=32, prefix_len=int(p), suffix_len=int(s)))
        plan = _gpu_plan(b.token_ids, b.position_ids, b.cu_seqlens)
        assert plan.n_original == n and plan.n_compact == m


@pytest.mark.parametrize("n_target,prefix_ratio", [(1024, 0.0), (16384, 0.25), (131072, 0.5), (1 << 20, 0.75),
                                                   (1 << 20, 1.0)])
def test_vs_oracle_large(oracle, n_target, prefix_ratio):
    """C5 microbench shapes: L=512, B=N/512, shared prefix ratio, bit-exact vs the oracle."""
    from paper_2601_15013_b200.workloads import SyntheticSpec, make_synthetic_batch

    L = 512
    p = int(L * prefix_ratio)
    b = make_synthetic_batch(SyntheticSpec(B=n_target // L, prefix_len=p, suffix_len=L - p, vocab=151936, seed=3))
    g, s, cp, m = oracle.build_plan_oracle(b.token_ids, b.position_ids, b.cu_seqlens)
    plan = _gpu_plan(b.token_ids, b.position_ids, b.cu_seqlens)
    _assert_plan(plan, g, s, m)
    np.testing.assert_array_equal(plan.compact_positions, cp)


def test_multilevel_trie_vs_oracle(oracle):
    """Branching at many depths with a tiny alphabet (deep shared structure)."""
    rng = np.random.default_rng(11)
    for _ in range(20):
        bsz = int(rng.integers(50, 400))
        lens = rng.integers(1, 300, size=bsz)
        cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        tok = rng.integers(0, 2, size=int(cu[-1])).astype(np.uint32)
        starts = np.repeat(cu[:-1], lens)
        pos = (np.arange(int(cu[-1])) - starts).astype(np.uint32)
        g, s, cp, m = oracle.build_plan_oracle(tok, pos, cu)
        _assert_plan(_gpu_plan(tok, pos, cu), g, s, m)


def test_long_prefix_c4_closed_form():
    from paper_2601_15013_b200.workloads import long_prefix_batch

    b = long_prefix_batch()
    plan = _gpu_plan(b.token_ids, b.position_ids, b.cu_seqlens)
    assert plan.n_original == 294_912 and plan.n_compact == 2048 + 128 * 256
    g = plan.gather_indices.astype(np.int64)
    s = plan.scatter_indices.astype(np.int64)
    assert np.all(np.diff(g) > 0)
    assert np.array_equal(s[g], np.arange(plan.n_compact))
    rep = g[s]
    assert np.array_equal(b.token_ids[rep], b.token_ids)
    assert np.array_equal(b.position_ids[rep], b.position_ids)


def test_empty_sequences_allowed(oracle):
    tok = np.array([1, 2, 1, 2, 3], dtype=np.uint32)
    cu = np.array([0, 2, 2, 5, 5], dtype=np.int64)
    pos = np.array([0, 1, 0, 1, 2], dtype=np.uint32)
    g, s, cp, m = oracle.build_plan_oracle(tok, pos, cu)
    _assert_plan(_gpu_plan(tok, pos, cu, allow_empty=True), g, s, m)


def test_validation_errors():
    from paper_2601_15013_b200 import BoundaryMismatch, MismatchedLengths, NonMonotoneOffsets

    with pytest.raises(NonMonotoneOffsets):
        _gpu_plan(np.array([1, 2, 3]), np.array([0, 1, 0]), np.array([0, 3, 2]))
    with pytest.raises(NonMonotoneOffsets):
        _gpu_plan(np.array([1, 2]), np.array([0, 1]), np.array([0, 2, 2]))
    with pytest.raises(BoundaryMismatch):
        _gpu_plan(np.array([1, 2]), np.array([0, 1]), np.array([1, 2]))
    with pytest.raises(MismatchedLengths):
        _gpu_plan(np.array([1, 2]), np.array([0]), np.array([0, 2]))


def test_device_side_validation_codes():
    """The C ABI reports bad offsets itself (no host pre-check)."""
    import torch

    from paper_2601_15013_b200 import NonMonotoneOffsets, build_plan_device

    tok = torch.tensor([1, 2, 3], dtype=torch.int32, device="cuda")
    cu = torch.tensor([0, 3, 2], dtype=torch.int64, device="cuda")
    with pytest.raises(NonMonotoneOffsets):
        build_plan_device(tok, tok, cu)


def test_cu_q_matches_suffix_structure():
    from paper_2601_15013_b200 import RaggedBatch, build_plan_device
    from paper_2601_15013_b200.plan import host_plan_cu_q, upload_batch
    from paper_2601_15013_b200.workloads import RerankSpec, msmarco_rerank_batch

    b = msmarco_rerank_batch(RerankSpec(queries=2, passages_per_query=16))
    tok, pos, cu = upload_batch(b)
    dp = build_plan_device(tok, pos, cu)
    assert np.array_equal(dp.cu_q_host, host_plan_cu_q(dp.to_host(), b.cu_seqlens))
    lcp = dp.lcp.cpu().numpy()
    assert np.array_equal(np.diff(dp.cu_q_host), np.diff(b.cu_seqlens) - lcp)
    assert isinstance(b, RaggedBatch)


def _device_plan_arrays(b, allow_empty=False):
    from paper_2601_15013_b200 import build_plan_device
    from paper_2601_15013_b200.plan import upload_batch

    tok, pos, cu = upload_batch(b)
    dp = build_plan_device(tok, pos, cu, allow_empty=allow_empty)
    return (dp.n_compact, dp.gather.cpu().numpy(), dp.scatter.cpu().numpy(), dp.compact_positions.cpu().numpy(),
            dp.cu_q_host.copy(), dp.lcp.cpu().numpy())


def _batches_for_both_planners():
    from paper_2601_15013_b200 import RaggedBatch
    from paper_2601_15013_b200.workloads import RerankSpec, SyntheticSpec, make_synthetic_batch, msmarco_rerank_batch

    out = [msmarco_rerank_batch(RerankSpec()), msmarco_rerank_batch(RerankSpec(queries=4)),
           msmarco_rerank_batch(RerankSpec(template_len=0, query_len=32, tail_len=0))]
    for n, p in ((1000, 0.5), (4096, 0.0), (16384, 0.25), (65536, 0.75), (65536 + 512, 0.5)):
        out.append(make_synthetic_batch(SyntheticSpec(B=max(n // 512, 1), prefix_len=int(512 * p),
                                                      suffix_len=512 - int(512 * p), seed=5)))
    rng = np.random.default_rng(19)
    for n_seq, maxlen in ((6000, 8), (300, 300), (2, 30000)):  # many short / deep multi-level / two long
        lens = rng.integers(1, maxlen, size=n_seq)
        cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        tok = rng.integers(0, 3, size=int(cu[-1])).astype(np.uint32)
        pos = (np.arange(int(cu[-1])) - np.repeat(cu[:-1], lens)).astype(np.uint32)
        out.append(RaggedBatch(tok, pos, cu))
    return out


def test_smem_planner_matches_l2_planner(oracle):
    """The cluster-resident planner (whole working set in shared memory, <= 64K tokens)
    and the L2-resident planners give the same bits on every batch shape; both match
    the oracle."""
    from paper_2601_15013_b200 import _native

    lib = _native.lib()
    for b in _batches_for_both_planners():
        res = []
        for on in (1, 0):
            prev = lib.rdx_plan_debug_smem(on)
            try:
                res.append(_device_plan_arrays(b))
            finally:
                lib.rdx_plan_debug_smem(prev)
        for x, y in zip(res[0], res[1]):
            np.testing.assert_array_equal(np.asarray(x), np.asarray(y))
        g, s, cp, m = oracle.build_plan_oracle(b.token_ids, b.position_ids, b.cu_seqlens)
        assert res[0][0] == m
        np.testing.assert_array_equal(res[0][1], g)
        np.testing.assert_array_equal(res[0][2], s)
        np.testing.assert_array_equal(res[0][3], cp)


@pytest.mark.parametrize("smem", [1, 0])
def test_validation_codes_both_planners(smem):
    import torch

    from paper_2601_15013_b200 import BoundaryMismatch, NonMonotoneOffsets, _native, build_plan_device

    lib = _native.lib()
    prev = lib.rdx_plan_debug_smem(smem)
    try:
        tok = torch.arange(3000, dtype=torch.int32, device="cuda")
        for cu, exc in (([0, 3000, 2000], NonMonotoneOffsets), ([0, 1000, 1000, 3000], NonMonotoneOffsets),
                        ([5, 1000, 3000], BoundaryMismatch), ([0, 1000, 2999], BoundaryMismatch)):
            cu_t = torch.tensor(cu, dtype=torch.int64, device="cuda")
            with pytest.raises(exc):
                build_plan_device(tok, tok, cu_t)
        # empty sequences are fine when allowed
        cu_t = torch.tensor([0, 1000, 1000, 3000], dtype=torch.int64, device="cuda")
        dp = build_plan_device(tok, tok, cu_t, allow_empty=True)
        assert dp.n_compact == 3000
    finally:
        lib.rdx_plan_debug_smem(prev)


def test_planner_fuzz_both_kernels(oracle):
    """Seeded random batches across the cluster-planner's whole range (1 CTA .. 16 CTAs, chunks
    ending mid-sequence, sequence starts on chunk boundaries, duplicated and empty-suffix
    sequences, tiny alphabets = deep shared structure) and beyond it (grid planner): both
    kernels bit-exact vs the oracle."""
    from paper_2601_15013_b200 import RaggedBatch, _native

    lib = _native.lib()
    rng = np.random.default_rng(2026)
    for trial in range(40):
        n_target = int(rng.choice([1, 7, 300, 1024, 1025, 4096, 9000, 16383, 33000, 65536, 70000]))
        nseq = int(rng.integers(1, max(2, min(n_target, 3000))))
        lens = rng.multinomial(n_target - nseq, np.ones(nseq) / nseq) + 1 if n_target >= nseq else np.ones(nseq, int)
        cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        n = int(cu[-1])
        alphabet = int(rng.choice([2, 3, 50, 151936]))
        tok = rng.integers(0, alphabet, size=n).astype(np.uint32)
        # copy whole earlier sequences / prefixes into later ones (shared trunks, exact duplicates)
        for s in range(1, nseq):
            if rng.random() < 0.5:
                src = int(rng.integers(0, s))
                k = int(min(lens[s], lens[src], rng.integers(0, lens[src] + 1)))
                tok[cu[s]:cu[s] + k] = tok[cu[src]:cu[src] + k]
        pos = (np.arange(n) - np.repeat(cu[:-1], lens)).astype(np.uint32)
        b = RaggedBatch(tok, pos, cu)
        g, s_, cp, m = oracle.build_plan_oracle(tok, pos, cu)
        for on in (1, 0):
            prev = lib.rdx_plan_debug_smem(on)
            try:
                res = _device_plan_arrays(b)
            finally:
                lib.rdx_plan_debug_smem(prev)
            assert res[0] == m, (trial, on, n, nseq)
            np.testing.assert_array_equal(res[1], g)
            np.testing.assert_array_equal(res[2], s_)
            np.testing.assert_array_equal(res[3], cp)
            assert int(np.diff(res[4]).max()) == int(np.max(np.diff(cu) - res[5]))
