"""One row-gather launch at the paper's Table-6 shape ([100000, 2048] bf16 -> 500000 rows) for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_15013_b200 import gather_rows_device  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
src = torch.randn(100_000, 2048, device="cuda", generator=g).to(torch.bfloat16)
idx = torch.randint(0, 100_000, (500_000,), device="cuda", dtype=torch.int32, generator=g)
dst = torch.empty(500_000, 2048, dtype=torch.bfloat16, device="cuda")
for _ in range(5):
    gather_rows_device(src, idx, out=dst)
torch.cuda.synchronize()
