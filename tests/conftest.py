"""Shared fixtures.  GPU tests carry @pytest.mark.gpu; everything else runs on CPU."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")


@pytest.fixture(scope="session")
def native_lib():
    """Build (if stale) and load the C-ABI library; no device needed."""
    from paper_2601_15013_b200 import _native
    from paper_2601_15013_b200.build import build_library

    build_library()
    return _native.load_library()


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as orc

    orc.build_oracle_lib()
    return orc


@pytest.fixture(scope="session")
def golden_plans():
    return dict(np.load(os.path.join(GOLDEN, "plans.npz")))


@pytest.fixture(scope="session")
def golden_forward():
    return dict(np.load(os.path.join(GOLDEN, "forward.npz")))


@pytest.fixture(scope="session")
def golden_synthetic():
    return dict(np.load(os.path.join(GOLDEN, "synthetic.npz")))


def unpack(g: dict, prefix: str):
    """Iterate (tok, pos, cu, gather, scatter, n_compact) of a packed golden set."""
    n_off, b_off, m_off = g[prefix + "_n_off"], g[prefix + "_b_off"], g[prefix + "_m_off"]
    for i in range(len(n_off) - 1):
        yield (g[prefix + "_tok"][n_off[i]:n_off[i + 1]], g[prefix + "_pos"][n_off[i]:n_off[i + 1]],
               g[prefix + "_cu"][b_off[i]:b_off[i + 1]], g[prefix + "_gather"][m_off[i]:m_off[i + 1]],
               g[prefix + "_scatter"][n_off[i]:n_off[i + 1]], int(g[prefix + "_n_compact"][i]))


@pytest.fixture
def rng():
    return np.random.default_rng(0)
