"""Host-side logic (no GPU): validation order, gating, padding, wire formats,
workload generators (pinned to the reference's draws), bindings type checks."""

import os

import numpy as np
import pytest

from conftest import GOLDEN


def _batch(tok, cu, pos=None):
    from paper_2601_15013_b200 import RaggedBatch, default_positions

    cu = np.asarray(cu, dtype=np.int64)
    return RaggedBatch(np.asarray(tok), default_positions(cu) if pos is None else np.asarray(pos), cu)


def test_validation_order():
    from paper_2601_15013_b200 import (BoundaryMismatch, MismatchedLengths, NonMonotoneOffsets, OverflowId,
                                       RaggedBatch, validate_batch)

    with pytest.raises(MismatchedLengths):
        validate_batch(RaggedBatch(np.array([1, 2]), np.array([0]), np.array([0, 2])))
    with pytest.raises(BoundaryMismatch):
        validate_batch(RaggedBatch(np.array([1, 2]), np.array([0, 1]), np.array([1, 2])))
    with pytest.raises(NonMonotoneOffsets):
        validate_batch(RaggedBatch(np.array([1, 2, 3]), np.array([0, 1, 0]), np.array([0, 3, 2])))
    with pytest.raises(NonMonotoneOffsets):
        validate_batch(RaggedBatch(np.array([1, 2]), np.array([0, 1]), np.array([0, 2, 2])))
    validate_batch(RaggedBatch(np.array([1, 2]), np.array([0, 1]), np.array([0, 2, 2])), allow_empty=True)
    with pytest.raises(BoundaryMismatch):
        validate_batch(RaggedBatch(np.array([1, 2]), np.array([0, 1]), np.array([0, 1])))
    with pytest.raises(OverflowId):
        validate_batch(RaggedBatch(np.array([1, 2**32]), np.array([0, 1]), np.array([0, 2])))
    with pytest.raises(OverflowId):
        validate_batch(RaggedBatch(np.array([1, 2]), np.array([0, -1]), np.array([0, 2])))
    stats = validate_batch(_batch([1, 2, 3, 4, 5], [0, 2, 5]))
    assert (stats.total_tokens, stats.num_sequences, stats.max_seq_len, stats.min_seq_len) == (5, 2, 3, 2)


def test_default_positions_and_immutability():
    from paper_2601_15013_b200 import default_positions

    assert default_positions([0, 3, 5]).tolist() == [0, 1, 2, 0, 1]
    assert default_positions([0]).tolist() == []
    b = _batch([1, 2, 3], [0, 3])
    with pytest.raises(ValueError):
        b.token_ids[0] = 9
    assert b.token_ids.dtype == np.uint32 and b.cu_seqlens.dtype == np.int64


def test_should_enable_and_pad_plan():
    from paper_2601_15013_b200 import CompactionPlan, EmptyPlan, pad_plan, should_enable

    plan = CompactionPlan(np.array([0, 1, 2, 5]), np.array([0, 1, 2, 0, 1, 3]), np.array([0, 1, 2, 2]), 6, 4)
    exact = CompactionPlan(np.arange(19), np.arange(20) % 19, np.arange(19), 20, 19)
    assert should_enable(exact, 0.95) and not should_enable(exact, 0.94) and not should_enable(exact, 0.0)
    padded = pad_plan(plan, 8)
    assert padded.gather_indices.tolist() == [0, 1, 2, 5, 0, 0, 0, 0]
    assert padded.compact_positions.tolist()[4:] == [0, 0, 0, 0]
    assert padded.n_padded == 8 and padded.n_compact == 4 and padded.gamma == plan.gamma
    assert pad_plan(plan, 4) is plan and pad_plan(plan, 1) is plan and pad_plan(padded, 8) is padded
    with pytest.raises(EmptyPlan):
        pad_plan(CompactionPlan(np.zeros(0), np.zeros(0), np.zeros(0), 0, 0), 8)
    with pytest.raises(ValueError):
        pad_plan(plan, 0)


def test_serialization_byte_identical_to_reference():
    from paper_2601_15013_b200 import CompactionPlan, load_plan, pad_plan, plan_from_bytes, plan_to_bytes

    plan = CompactionPlan(np.array([0, 1, 2, 5]), np.array([0, 1, 2, 0, 1, 3]), np.array([0, 1, 2, 2]), 6, 4)
    with open(os.path.join(GOLDEN, "plan_toy.rdxp"), "rb") as f:
        ref = f.read()
    assert plan_to_bytes(plan) == ref
    assert plan_to_bytes(pad_plan(plan, 16)) == ref  # padding is not serialised
    again = plan_from_bytes(ref)
    assert again.gather_indices.tolist() == [0, 1, 2, 5] and plan_to_bytes(again) == ref
    js = load_plan(os.path.join(GOLDEN, "plan_toy.json"))
    assert js.scatter_indices.tolist() == [0, 1, 2, 0, 1, 3] and js.n_compact == 4
    with pytest.raises(ValueError):
        plan_from_bytes(b"XXXX" + b"\x00" * 64)


def test_generators_match_reference_draws(golden_synthetic):
    from paper_2601_15013_b200.workloads import Pattern, SyntheticSpec, make_pattern_batch, make_synthetic_batch

    i = 0
    while f"spec{i}" in golden_synthetic:
        b, p, s, v, seed = golden_synthetic[f"spec{i}"].tolist()
        batch = make_synthetic_batch(SyntheticSpec(B=b, prefix_len=p, suffix_len=s, vocab=v, seed=seed))
        assert np.array_equal(batch.token_ids, golden_synthetic[f"spec{i}_tok"])
        i += 1
    assert i == 5
    for pat in Pattern:
        for seed, vocab in ((3, 97), (3, 11), (0, 97)):
            b = make_pattern_batch(pat, seed=seed, vocab=vocab)
            assert np.array_equal(b.token_ids, golden_synthetic[f"pat_{pat.value}_{seed}_{vocab}_tok"])
            assert np.array_equal(b.cu_seqlens, golden_synthetic[f"pat_{pat.value}_{seed}_{vocab}_cu"])


def test_rerank_workload_shape(oracle):
    from paper_2601_15013_b200.workloads import RerankSpec, msmarco_rerank_batch

    spec = RerankSpec()
    b = msmarco_rerank_batch(spec)
    lens = np.diff(b.cu_seqlens)
    assert b.num_sequences == 64 and lens.min() >= 72 + 77 and lens.max() <= 120 + 77
    m = oracle.build_plan_oracle(b.token_ids, b.position_ids, b.cu_seqlens)[3]
    shared = spec.template_len + spec.query_len
    assert m == shared + (b.num_tokens - 64 * shared)


def test_host_plan_cu_q(oracle):
    from paper_2601_15013_b200 import CompactionPlan
    from paper_2601_15013_b200.plan import host_plan_cu_q

    rng = np.random.default_rng(5)
    for _ in range(50):
        tok, pos, cu = oracle.random_small_batch(rng)
        g, s, cp, m = oracle.build_plan_oracle(tok, pos, cu)
        cu_q = host_plan_cu_q(CompactionPlan(g, s, cp, len(tok), m), cu)
        assert cu_q is not None and cu_q[-1] == m
    bad = CompactionPlan(np.array([1, 0]), np.array([1, 0]), np.array([0, 0]), 2, 2)
    assert host_plan_cu_q(bad, np.array([0, 2])) is None


def test_bindings_type_check_before_gpu():
    from paper_2601_15013_b200 import bindings

    with pytest.raises(TypeError):
        bindings.gather_rows(np.zeros((2, 2), dtype=np.int32), [0, 1])


def test_config_validation():
    from paper_2601_15013_b200 import QWEN3_PRESETS, ModelConfig, Qwen3Config, ShapeMismatch

    with pytest.raises(ShapeMismatch):
        ModelConfig(hidden_size=100)
    with pytest.raises(ShapeMismatch):
        ModelConfig(num_heads=4, num_kv_heads=3)
    q = QWEN3_PRESETS["qwen3-0.6b"]
    assert q.q_dim == 2048 and q.hidden_size == 1024 and isinstance(q, Qwen3Config)


def test_init_params_matches_reference_layout():
    from paper_2601_15013_b200 import TINY_C1, init_params

    p = init_params(TINY_C1, seed=0)
    assert p["layers.0.wq"].shape == (64, 64) and p["layers.1.w_down"].shape == (64, 192)
    assert p["lm_head"].shape == (1024, 64) and np.all(p["final_norm"] == 1.0)
    assert np.abs(p["embed"]).max() <= 0.05


def test_gate_up_interleave_layout():
    import torch

    from paper_2601_15013_b200.model import DeviceWeights

    gate = torch.arange(192 * 2, dtype=torch.float32).view(192, 2)
    up = -gate
    out = DeviceWeights._interleave_gate_up(gate, up, 192)
    assert out.shape == (384, 2)
    assert torch.equal(out[:64], gate[:64]) and torch.equal(out[64:128], up[:64])
    assert torch.equal(out[128:192], gate[64:128])
