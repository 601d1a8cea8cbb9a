"""Drop-in boundary with the reference installed.

The reference package ``radix_compact`` (+ ``radix_bindings``) is found at
/root/reference/pkg (this container) or ``baseline/_ref`` (the pip install
that travels to the GPU box).  Each check runs in a fresh
interpreter so that ``paper_2601_15013_b200.errors`` binds the reference's
own exception classes (it does so only when ``radix_compact`` is importable
at its first import).

CPU: the validation path raises before any device work, so the reference's
``test_errors_carry_primary_names`` (bindings/tests/test_bindings.py:36-38)
runs here with the GPU planner swapped in.  GPU: the whole binding contract
(toy plan, identity, errors, gather/scatter, RDXP round trip, 25 random
batches against the reference's own numba planner) with the swap applied.
"""

from __future__ import annotations

import os
import subprocess
import sys
import textwrap

import pytest

from conftest import ROOT

REF_SRC = [("/root/reference/pkg/src", "/root/reference/pkg/bindings/src"),
           (os.path.join(ROOT, "baseline", "_ref"),)]
REF_TEST = "/root/reference/pkg/bindings/tests/test_bindings.py"

SWAP = textwrap.dedent("""
    import radix_bindings as rb
    from paper_2601_15013_b200.plan import build_plan_auto as _gpu_plan_builder
    rb._plan_builder = _gpu_plan_builder          # INTEGRATION.md section 1
""")


def _ref_paths():
    for paths in REF_SRC:
        if all(os.path.isdir(os.path.join(p, "radix_compact")) or os.path.isdir(os.path.join(p, "radix_bindings"))
               for p in paths) and any(os.path.isdir(os.path.join(p, "radix_compact")) for p in paths):
            return list(paths)
    return None


def _run(code: str, timeout=600):
    paths = _ref_paths()
    if paths is None:
        pytest.skip("reference package not installed (neither /root/reference nor baseline/_ref)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join(paths + [ROOT] + [env.get("PYTHONPATH", "")])
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_rdx")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=timeout,
                       cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return r.stdout


def test_errors_are_reference_classes():
    out = _run(textwrap.dedent("""
        import radix_compact.errors as ref
        import paper_2601_15013_b200 as pkg
        import paper_2601_15013_b200.errors as ours
        for name in ("RadixCompactError", "MismatchedLengths", "NonMonotoneOffsets", "BoundaryMismatch",
                     "OverflowId", "CapacityExceeded", "EmptyPlan", "IndexOutOfRange", "ShapeMismatch",
                     "OddHeadDim", "PlanBatchMismatch", "VocabTooSmall", "WorkerPanic"):
            assert getattr(ours, name) is getattr(ref, name), name
        assert issubclass(ours.HashRetriesExhausted, ref.RadixCompactError)
        assert issubclass(ours.NativeLibraryError, ref.RadixCompactError)
        assert ours.STATUS_CLASSES[2] is ref.NonMonotoneOffsets
        assert pkg.NonMonotoneOffsets is ref.NonMonotoneOffsets
        print("PASS")
    """))
    assert "PASS" in out


def test_swap_reference_error_test_cpu():
    """INTEGRATION §1's swap, then the reference's own error test (validation runs on the host)."""
    code = SWAP + textwrap.dedent("""
        import radix_compact.errors as ref
        try:
            rb.compute_plan([1, 2, 3], [0, 1, 0], [0, 3, 2])
        except ref.NonMonotoneOffsets as e:
            assert type(e).__name__ == "NonMonotoneOffsets"
        else:
            raise AssertionError("no exception")
        print("PASS")
    """)
    if os.path.exists(REF_TEST):  # the reference's test file itself, with the swap applied
        code += textwrap.dedent(f"""
            import pytest, sys
            rc = pytest.main(["-q", "-p", "no:cacheprovider", {REF_TEST!r} + "::test_errors_carry_primary_names"])
            assert rc == 0, rc
            print("PASS-REF-TEST")
        """)
    out = _run(code)
    assert "PASS" in out
    if os.path.exists(REF_TEST):
        assert "PASS-REF-TEST" in out


@pytest.mark.gpu
def test_swap_reference_binding_contract_gpu():
    """Every contract of bindings/tests/test_bindings.py with the GPU planner swapped in."""
    code = SWAP + textwrap.dedent("""
        import os, tempfile
        import numpy as np
        import radix_compact
        import radix_compact.trie as trie
        from radix_compact.errors import NonMonotoneOffsets
        from radix_compact.ragged import default_positions

        calls = []
        orig = rb._plan_builder
        def spy(batch):
            calls.append(batch.num_tokens)
            return orig(batch)
        rb._plan_builder = spy
        plan = rb.compute_plan([1, 2, 3, 1, 2, 4], [0, 1, 2, 0, 1, 2], [0, 3, 6])
        assert calls == [6], calls          # the binding delegated to the GPU planner
        rb._plan_builder = orig
        assert plan["gather"].tolist() == [0, 1, 2, 5]
        assert plan["scatter"].tolist() == [0, 1, 2, 0, 1, 3]
        assert plan["compact_positions"].tolist() == [0, 1, 2, 2]
        assert plan["n_original"] == 6 and plan["n_compact"] == 4
        assert abs(plan["gamma"] - 4 / 6) < 1e-12
        for k in ("gather", "scatter", "compact_positions"):
            assert plan[k].dtype == np.uint32 and plan[k].flags["C_CONTIGUOUS"]
        ident = rb.compute_plan([7, 8, 9], [0, 1, 2], [0, 3])
        assert ident["gather"].tolist() == [0, 1, 2] and ident["scatter"].tolist() == [0, 1, 2]
        try:
            rb.compute_plan([1, 2, 3], [0, 1, 0], [0, 3, 2])
            raise AssertionError("no exception")
        except NonMonotoneOffsets:
            pass
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "plan.rdxp")
            rb.save_plan(plan, path)
            again = rb.load_plan(path)
            for k in ("gather", "scatter", "compact_positions"):
                assert np.array_equal(again[k], plan[k])
            lib_plan = trie.load_plan(path)
            assert trie.plan_to_bytes(lib_plan) == open(path, "rb").read()
        rng = np.random.default_rng(17)
        for _ in range(25):
            b = int(rng.integers(1, 6))
            cu = np.concatenate([[0], np.cumsum(rng.integers(1, 10, size=b))]).astype(np.int64)
            tokens = rng.integers(0, 5, size=int(cu[-1]))
            pos = default_positions(cu)
            got = rb.compute_plan(tokens, pos, cu)
            ref = trie.build_plan_auto(radix_compact.RaggedBatch(tokens, pos, cu))   # reference numba trie
            assert np.array_equal(got["gather"], ref.gather_indices)
            assert np.array_equal(got["scatter"], ref.scatter_indices)
            assert np.array_equal(got["compact_positions"], ref.compact_positions)
        # acceptance criterion 12 (test_acceptance.py:302-339): the reference CLI `plan --binary`
        # (CPU numba planner) and the binding's save_plan of the GPU plan write identical bytes
        from radix_compact import save_batch
        from radix_compact.cli import main as cli_main
        with tempfile.TemporaryDirectory() as d:
            for i in range(100):
                b = int(rng.integers(1, 7))
                cu = np.concatenate([[0], np.cumsum(rng.integers(1, 12, size=b))]).astype(np.int64)
                tokens = rng.integers(0, 4, size=int(cu[-1])).astype(np.uint32)
                batch = radix_compact.RaggedBatch(tokens, default_positions(cu), cu)
                bfile, pfile, qfile = (os.path.join(d, n) for n in ("b.json", "p.rdxp", "q.rdxp"))
                save_batch(batch, bfile)
                assert cli_main(["plan", bfile, "-o", pfile, "--binary"]) == 0
                rb.save_plan(rb.compute_plan(batch.token_ids, batch.position_ids, batch.cu_seqlens), qfile)
                assert open(pfile, "rb").read() == open(qfile, "rb").read(), i
        print("PASS")
    """)
    out = _run(code)
    assert "PASS" in out
