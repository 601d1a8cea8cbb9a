"""rdx_rmsnorm_rows at the C2 shape: L2-warm (input just written) vs L2-cold."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_15013_b200 import _native  # noqa: E402

M, D = int(os.environ.get("M", "7024")), 1024
lib = _native.lib()
h = torch.randn(M, D, device="cuda")
src = torch.randn(M, D, device="cuda")
w = torch.ones(D, device="cuda")
out = torch.empty(M, D, dtype=torch.bfloat16, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def rms():
    _native.check(lib.rdx_rmsnorm_rows(h.data_ptr(), D, None, M, D, w.data_ptr(), 1e-6, out.data_ptr(), D, st), "rms")


def timed(pre, it=50):
    tot = 0.0
    for i in range(it + 3):
        pre()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rms()
        b.record()
        b.synchronize()
        if i >= 3:
            tot += a.elapsed_time(b)
    return tot / it * 1e3


warm = timed(lambda: h.copy_(src))
cold = timed(lambda: flush.zero_())
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    rms()
a.record()
for _ in range(50):
    rms()
b.record()
b.synchronize()
back = a.elapsed_time(b) / 50 * 1e3
gb = M * D * 6 / 1e9
print(f"rmsnorm M={M}: warm(h just written) {warm:.1f} us ({gb / warm * 1e6:.0f} GB/s)  cold {cold:.1f} us "
      f"({gb / cold * 1e6:.0f} GB/s)  back-to-back {back:.1f} us")
