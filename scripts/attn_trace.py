"""Scratch: per-step event timeline of rdx_attention CTA 0 (debug trace)."""
import ctypes, math, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "attn_bench.py")).read().split("from flash_attn")[0])
lib.rdx_attention_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
lib.rdx_attention_trace(None, 0)
for _ in range(3): ours()
torch.cuda.synchronize()
buf = np.zeros((4096, 64), dtype=np.uint64)
lib.rdx_attention_trace(buf.ctypes.data, buf.nbytes)
names = ["kv_full", "s_free", "pfull(pv issue)", "S ready(softmax)", "computed", "pv_done", "P published"]
for c in (0, 77):
    r = buf[c].astype(np.int64); t0 = r[0]
    print("CTA", c)
    for st in range(8):
        vals = [(int(r[8 + st * 7 + k]) - t0) if r[8 + st * 7 + k] > 0 else None for k in range(7)]
        print("  step", st, {n: v for n, v in zip(names, vals)})
