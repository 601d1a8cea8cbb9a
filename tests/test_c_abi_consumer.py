"""A plain-C program (tests/c_abi/plan_consumer.c) against include/radix_b200.h and _rdx.so:
the header compiles as C99 with -Wall -Wextra -Werror and the program links (CPU); on a B200
it builds the reference's toy plan and gathers rows through the ABI alone (no Python, no torch)."""
import os
import shutil
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "c_abi", "plan_consumer.c")
PKG = os.path.join(ROOT, "paper_2601_15013_b200")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _build(out):
    if not shutil.which("gcc"):
        pytest.skip("gcc unavailable")
    if not os.path.exists(os.path.join(PKG, "_rdx.so")):
        pytest.skip("_rdx.so not built")
    cmd = ["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA, "include"), SRC, "-o", out,
           "-L", PKG, "-l:_rdx.so", f"-Wl,-rpath,{PKG}",
           "-L", os.path.join(CUDA, "lib64"), "-lcudart", f"-Wl,-rpath,{os.path.join(CUDA, 'lib64')}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_c_consumer_compiles_and_links(tmp_path):
    _build(str(tmp_path / "plan_consumer"))


@pytest.mark.gpu
def test_c_consumer_runs(tmp_path):
    exe = _build(str(tmp_path / "plan_consumer"))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c-abi ok: N'=4 gather=[0,1,2,5]" in r.stdout
