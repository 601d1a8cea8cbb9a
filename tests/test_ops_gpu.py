"""Row gather/scatter (rdx_gather_rows) and bindings parity on the GPU.

Bit-exact: the kernels are byte copies.  Mirrors the reference's
tests/test_ops.py:18-143 and bindings/tests/test_bindings.py.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_toy_gather_scatter():
    from paper_2601_15013_b200 import gather_rows, scatter_rows

    x = np.array([[1.0], [2.0], [3.0], [1.0], [2.0], [4.0]])
    assert gather_rows(x, [0, 1, 2, 5]).tolist() == [[1.0], [2.0], [3.0], [4.0]]
    y = np.array([[1.0], [2.0], [3.0], [4.0]])
    assert scatter_rows(y, [0, 1, 2, 0, 1, 3]).tolist() == [[1.0], [2.0], [3.0], [1.0], [2.0], [4.0]]


@pytest.mark.parametrize("dtype", [np.float32, np.float64, np.int8, np.uint16, np.int32])
@pytest.mark.parametrize("cols", [1, 3, 8, 64, 1000, 6144])
def test_bit_exact_all_dtypes(rng, dtype, cols):
    from paper_2601_15013_b200 import gather_rows

    rows = 257
    x = (rng.normal(size=(rows, cols)) * 100).astype(dtype)
    idx = rng.integers(0, rows, size=999)
    out = gather_rows(x, idx)
    assert out.dtype == x.dtype
    assert np.array_equal(out, x[idx])


def test_bf16_device_strided_source():
    import torch

    from paper_2601_15013_b200 import gather_rows_device

    x = torch.randn(500, 6144, device="cuda").to(torch.bfloat16)
    idx = torch.randint(0, 500, (2000,), device="cuda", dtype=torch.int32)
    sub = x[:, 2048:]  # strided K/V view, as the attention boundary uses it
    out = gather_rows_device(sub, idx)
    assert torch.equal(out, sub[idx.long()])


def test_errors():
    from paper_2601_15013_b200 import IndexOutOfRange, ShapeMismatch, gather_rows

    x = np.zeros((3, 2))
    with pytest.raises(IndexOutOfRange):
        gather_rows(x, [0, 3])
    with pytest.raises(IndexOutOfRange):
        gather_rows(x, [-1])
    with pytest.raises(ShapeMismatch):
        gather_rows(np.zeros(3), [0])


def test_device_out_of_range_flag():
    import torch

    from paper_2601_15013_b200 import IndexOutOfRange, gather_rows

    x = torch.ones(4, 16, device="cuda")
    with pytest.raises(IndexOutOfRange):
        gather_rows(x, torch.tensor([0, 7], dtype=torch.int32, device="cuda"))


def test_round_trip_through_plan(rng, oracle):
    from paper_2601_15013_b200 import build_plan, gather_rows, scatter_rows
    from paper_2601_15013_b200.ragged import RaggedBatch

    for _ in range(20):
        tok, pos, cu = oracle.random_small_batch(rng)
        plan = build_plan(RaggedBatch(tok, pos, cu))
        xc = rng.normal(size=(plan.n_compact, 4))
        x = scatter_rows(xc, plan.scatter_indices)
        assert np.array_equal(scatter_rows(gather_rows(x, plan.gather_indices), plan.scatter_indices), x)


def test_bindings_parity_100_batches(tmp_path, oracle):
    """Acceptance criterion 12 (test_acceptance.py:302-339) with the oracle as the other side."""
    from paper_2601_15013_b200 import bindings, serialization
    from paper_2601_15013_b200.plan import CompactionPlan

    rng = np.random.default_rng(99)
    for i in range(100):
        tok, pos, cu = oracle.random_small_batch(rng)
        d = bindings.compute_plan(tok, pos, cu)
        g, s, cp, m = oracle.build_plan_oracle(tok, pos, cu)
        for key in ("gather", "scatter", "compact_positions"):
            assert d[key].dtype == np.uint32 and d[key].flags["C_CONTIGUOUS"]
        assert np.array_equal(d["gather"], g) and np.array_equal(d["scatter"], s)
        path = tmp_path / f"p{i}.rdxp"
        bindings.save_plan(d, path)
        ref_bytes = serialization.plan_to_bytes(CompactionPlan(g, s, cp, len(tok), m))
        assert path.read_bytes() == ref_bytes
        x = rng.normal(size=(len(tok), 4))
        assert np.array_equal(bindings.gather_rows(x, d["gather"]), x[g.astype(np.int64)])
        y = rng.normal(size=(m, 4)).astype(np.float32)
        assert np.array_equal(bindings.scatter_rows(y, d["scatter"]), y[s.astype(np.int64)])


def test_bindings_delegation(monkeypatch):
    from paper_2601_15013_b200 import bindings
    from paper_2601_15013_b200 import plan as planmod

    calls = []
    original = planmod.build_plan_auto

    def spy(batch):
        calls.append(batch.num_tokens)
        return original(batch)

    monkeypatch.setattr(bindings, "_plan_builder", spy)
    d = bindings.compute_plan([1, 2, 3, 1, 2, 4], [0, 1, 2, 0, 1, 2], [0, 3, 6])
    assert calls == [6] and d["n_compact"] == 4
    assert d["compact_positions"].tolist() == [0, 1, 2, 2]
