"""Build the sm_100a C-ABI library in-tree (no JIT cache, so it travels).

``python -m paper_2601_15013_b200.build [--force]``
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_rdx.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
              "--expt-relaxed-constexpr", "-diag-suppress", "177"]


def nvcc_path() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    out_t = os.path.getmtime(OUT)
    return any(os.path.getmtime(p) > out_t for p in deps)


def build_library(force: bool = False, verbose: bool = False, variant: str | None = None,
                  extra_flags: list[str] | None = None) -> str:
    """Compile every csrc/*.cu for sm_100a into _rdx.so (or _rdx_<variant>.so); returns its path."""
    out = OUT if variant is None else os.path.join(HERE, f"_rdx_{variant}.so")
    if variant is None and not force and not _stale():
        return OUT
    tmp = out + ".tmp"
    extra = os.environ.get("RDX_NVCC_EXTRA", "").split() + list(extra_flags or [])  # e.g. -DRDX_ATTN_STATS_BUILD=1
    cmd = [nvcc_path(), *ARCH_FLAGS, *NVCC_FLAGS, *extra, "-I", INCLUDE, "-o", tmp, *sources()]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose=True))
