"""gather_rows_backward / scatter_rows_backward (ops.py:69-107) on the GPU vs the
reference's np.add.at path: bit-identical (ascending-j accumulation), fp32 and fp64,
duplicated / empty / out-of-range indices, and the compact-path use in a trie plan."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ref(grad, idx, n):
    out = np.zeros((n, grad.shape[1]), dtype=grad.dtype)
    np.add.at(out, np.asarray(idx, dtype=np.int64), grad)
    return out


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("cols", [1, 3, 4, 64, 1000])
def test_bit_identical_to_add_at(dtype, cols):
    from paper_2601_15013_b200 import gather_rows_backward

    rng = np.random.default_rng(cols)
    n_idx, n = 5000, 700
    idx = rng.integers(0, n, size=n_idx).astype(np.uint32)  # heavy duplication, some rows empty
    grad = rng.standard_normal((n_idx, cols)).astype(dtype) * rng.uniform(1e-3, 1e3, size=(n_idx, 1)).astype(dtype)
    out = gather_rows_backward(grad, idx, n)
    ref = _ref(grad, idx, n)
    assert out.dtype == ref.dtype
    assert np.array_equal(out.view(np.uint8), ref.view(np.uint8))  # bitwise


def test_toy_values_and_errors():
    """ops tests toy values (tests/test_ops.py:18-38 style) + error contract."""
    from paper_2601_15013_b200 import gather_rows_backward, scatter_rows_backward
    from paper_2601_15013_b200.errors import IndexOutOfRange, ShapeMismatch

    g = np.array([[1.0, 2.0], [3.0, 4.0], [5.0, 6.0]])
    out = gather_rows_backward(g, [2, 0, 2], 4)
    assert np.array_equal(out, [[3.0, 4.0], [0.0, 0.0], [6.0, 8.0], [0.0, 0.0]])
    assert np.array_equal(scatter_rows_backward(g, [1, 1, 0], 2), [[5.0, 6.0], [4.0, 6.0]])
    with pytest.raises(IndexOutOfRange):
        gather_rows_backward(g, [0, 1, 4], 4)
    with pytest.raises(ShapeMismatch):
        gather_rows_backward(g, [0, 1], 4)
    with pytest.raises(ShapeMismatch):
        gather_rows_backward(g[0], [0], 4)
    with pytest.raises(TypeError):
        gather_rows_backward(g.astype(np.float16), [0, 1, 2], 4)
    assert gather_rows_backward(np.zeros((0, 2)), [], 3).shape == (3, 2)


def test_device_error_flag_and_compact_plan():
    """Device path: out-of-range flag; scatter adjoint over a real trie plan equals add.at."""
    import torch

    from paper_2601_15013_b200 import build_plan, gather_rows_backward, scatter_rows_backward
    from paper_2601_15013_b200.errors import IndexOutOfRange
    from paper_2601_15013_b200.workloads import SyntheticSpec, make_synthetic_batch

    b = make_synthetic_batch(SyntheticSpec(B=16, prefix_len=40, suffix_len=12, vocab=1000, seed=3))
    plan = build_plan(b)
    rng = np.random.default_rng(0)
    d_full = rng.standard_normal((plan.n_original, 96))
    d_comp = scatter_rows_backward(torch.from_numpy(d_full).cuda(), plan.scatter_indices, plan.n_compact)
    assert np.array_equal(d_comp.cpu().numpy(), _ref(d_full, plan.scatter_indices, plan.n_compact))
    # gather adjoint: distinct indices -> plain placement, zeros elsewhere
    d_c = rng.standard_normal((plan.n_compact, 8)).astype(np.float32)
    d_f = gather_rows_backward(d_c, plan.gather_indices, plan.n_original)
    assert np.array_equal(d_f, _ref(d_c, plan.gather_indices, plan.n_original))
    with pytest.raises(IndexOutOfRange):
        gather_rows_backward(torch.ones(2, 4, device="cuda"), torch.tensor([0, 9], device="cuda"), 5)


def test_large_ragged_deterministic():
    """1M-row scatter adjoint with a long-prefix plan: two runs bitwise equal and equal to add.at."""
    import torch

    from paper_2601_15013_b200 import build_plan, scatter_rows_backward
    from paper_2601_15013_b200.workloads import prefix_ratio_batch

    b = prefix_ratio_batch(1 << 20, 0.5)
    plan = build_plan(b)
    g = torch.randn(plan.n_original, 16, device="cuda")
    a = scatter_rows_backward(g, plan.scatter_indices, plan.n_compact)
    c = scatter_rows_backward(g, plan.scatter_indices, plan.n_compact)
    assert torch.equal(a, c)
    ref = _ref(g.cpu().numpy(), plan.scatter_indices, plan.n_compact)
    assert np.array_equal(a.cpu().numpy(), ref)
