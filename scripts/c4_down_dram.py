"""C4 down GEMM (M=34816, N=4096, K=12288, RDX_EPI_RESID_F32) alone: CUDA-event time per launch for
raster groups of 16/8/4/2 row blocks (rdx_gemm_debug_group_m_bigk).  Run under
`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum` for the DRAM bytes per launch.
python scripts/c4_down_dram.py [group ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_15013_b200 import _native  # noqa: E402
from scripts.gemm_epi_bench_lib import gemm  # noqa: E402

M, N, K = 34816, 4096, 12288
a = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
w = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
h = torch.zeros(M, N, device="cuda")
fn = gemm(a, w, _native.EPI_RESID_F32, h)
lib = _native.lib()
groups = [int(g) for g in sys.argv[1:]] or [16, 8, 4, 2]
for g in groups:
    lib.rdx_gemm_debug_group_m_bigk(g)
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):
        fn()
    e.record()
    e.synchronize()
    ms = s.elapsed_time(e) / 3
    print(f"group {g:2d}: {ms * 1e3:8.1f} us  {2 * M * N * K / (ms * 1e-3) / 1e12:7.1f} TF/s", flush=True)
