"""The reference's exported primitives (model.py:147, 180, 204, 210) on the GPU kernels,
per-op against the CPU oracle's restatement (tests/test_model.py:49-195 style).
Tolerance: bf16 operands / fp32 accumulation vs fp64 -> max-relative 2e-2."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / max(np.abs(b).max(), 1e-30))


def test_rmsnorm():
    from oracle import oracle as orc
    from paper_2601_15013_b200 import rmsnorm
    from paper_2601_15013_b200.errors import ShapeMismatch

    rng = np.random.default_rng(0)
    for d in (64, 1000, 1024, 36):
        x = rng.standard_normal((37, d)) * 3
        w = rng.uniform(0.5, 1.5, d)
        out = rmsnorm(x, w, 1e-6)
        assert out.dtype == x.dtype and out.shape == x.shape
        assert _rel(out, orc.rmsnorm(x, w, 1e-6)) <= 1e-2
    with pytest.raises(ShapeMismatch):
        rmsnorm(np.ones((3, 4)), np.ones(5), 1e-6)


def test_apply_rope_matches_tables_and_positions():
    from oracle import oracle as orc
    from paper_2601_15013_b200 import apply_rope
    from paper_2601_15013_b200.errors import OddHeadDim, ShapeMismatch

    rng = np.random.default_rng(1)
    n, h, kvh, hd = 50, 4, 2, 64
    q, k = rng.standard_normal((n, h, hd)), rng.standard_normal((n, kvh, hd))
    pos = rng.integers(0, 100000, n).astype(np.uint32)
    qo, ko = apply_rope(q, k, pos, theta=1e6)
    cos, sin = orc.rope_tables(pos, hd, 1e6, np.float64)
    c, s = cos[:, None, :], sin[:, None, :]
    assert _rel(qo, q * c + orc._rotate_half(q) * s) <= 1e-5
    assert _rel(ko, k * c + orc._rotate_half(k) * s) <= 1e-5
    with pytest.raises(ShapeMismatch):
        apply_rope(q, k, pos[:-1])
    with pytest.raises(OddHeadDim):
        apply_rope(np.ones((2, 1, 3)), np.ones((2, 1, 3)), [0, 1])


def test_swiglu_mlp():
    from oracle import oracle as orc
    from paper_2601_15013_b200 import swiglu_mlp
    from paper_2601_15013_b200.errors import ShapeMismatch

    rng = np.random.default_rng(2)
    for m, d, di in ((300, 256, 512), (7, 64, 192), (129, 1024, 3000)):
        h = rng.standard_normal((m, d))
        wg, wu = rng.uniform(-0.05, 0.05, (di, d)), rng.uniform(-0.05, 0.05, (di, d))
        wd = rng.uniform(-0.05, 0.05, (d, di))
        out = swiglu_mlp(h, wg, wu, wd)
        ref = (orc.silu(h @ wg.T) * (h @ wu.T)) @ wd.T
        assert out.shape == (m, d) and _rel(out, ref) <= 2e-2
    with pytest.raises(ShapeMismatch):
        swiglu_mlp(np.ones((3, 8)), np.ones((4, 16)), np.ones((4, 16)), np.ones((16, 4)))


def test_attention_ragged():
    from oracle import oracle as orc
    from paper_2601_15013_b200 import attention_ragged
    from paper_2601_15013_b200.errors import ShapeMismatch

    rng = np.random.default_rng(3)
    H, KV, hd = 4, 2, 64
    cu = np.array([0, 5, 5, 40, 97])
    n = int(cu[-1])
    q, k, v = (rng.standard_normal((n, x * hd)) for x in (H, KV, KV))
    out = attention_ragged(q, k, v, cu, H, KV, hd)
    assert _rel(out, orc.attention(q, k, v, cu, H, KV, hd)) <= 2e-2
    with pytest.raises(ShapeMismatch):
        attention_ragged(q, k[:, :-1], v, cu, H, KV, hd)
