"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
symbol include/radix_b200.h declares; no compute calls here."""

import os
import re
import subprocess

import pytest

from conftest import ROOT


def _header_functions():
    with open(os.path.join(ROOT, "include", "radix_b200.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(rdx_\w+)\s*\(", text, re.M)))


def test_header_declarations_match_binding():
    from paper_2601_15013_b200 import _native

    assert _header_functions() == sorted(_native.EXPORTS)


def test_library_exports_every_symbol(native_lib):
    for name in _header_functions():
        assert hasattr(native_lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2601_15013_b200", "_rdx.so")],
                         capture_output=True, text=True, check=True).stdout
    for name in _header_functions():
        assert re.search(rf"\bT {name}\b", out), name


def test_status_names(native_lib):
    assert native_lib.rdx_version() == 300
    assert native_lib.rdx_status_name(0) == b"RDX_OK"
    assert native_lib.rdx_status_name(7) == b"IndexOutOfRange"
    assert native_lib.rdx_status_name(2) == b"NonMonotoneOffsets"


def test_status_to_exception_mapping():
    from paper_2601_15013_b200 import errors

    for code, name in ((1, "MismatchedLengths"), (2, "NonMonotoneOffsets"), (3, "BoundaryMismatch"),
                       (7, "IndexOutOfRange"), (8, "ShapeMismatch"), (9, "PlanBatchMismatch")):
        with pytest.raises(errors.RadixCompactError) as ei:
            errors.raise_for_status(code, "x")
        assert type(ei.value).__name__ == name


def test_sass_contains_tcgen05_and_tma(native_lib):
    """The GEMM is tcgen05 (UTCHMMA) fed by TMA (UTMALDG), accumulators read with LDTM."""
    so = os.path.join(ROOT, "paper_2601_15013_b200", "_rdx.so")
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    if not sass:
        pytest.skip("cuobjdump unavailable")
    for mnem in ("UTCHMMA", "UTMALDG", "LDTM"):
        assert mnem in sass, mnem
    assert "HMMA" not in sass.replace("UTCHMMA", "")


def test_no_gpu_raises_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2601_15013_b200 import NativeLibraryError, build_plan
    from paper_2601_15013_b200.ragged import RaggedBatch

    import numpy as np

    with pytest.raises(NativeLibraryError):
        build_plan(RaggedBatch(np.array([1, 2]), np.array([0, 1]), np.array([0, 2])))
