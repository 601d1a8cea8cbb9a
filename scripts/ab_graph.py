"""A/B of a library switch on the C2 CUDA-graph step: two models captured with the switch on / off,
replays interleaved (same box, same clocks).  python scripts/ab_graph.py [pdl|tail|norm] [c2|c3|c4]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2601_15013_b200 import DeviceBatch, DeviceWeights, RadixQwen3, _native  # noqa: E402
from paper_2601_15013_b200.rerank import RadixReranker  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "pdl"
cfg_name = sys.argv[2] if len(sys.argv) > 2 else "c2"
lib = _native.lib()
if what == "group":  # GEMM raster: G_ON vs G_OFF row blocks per group (captured into each arm's graph)
    def setter(on):
        lib.rdx_gemm_debug_group_m(int(os.environ.get("G_ON", "16") if on else os.environ.get("G_OFF", "0")))
elif what == "groupk":  # raster group of the K >= 8192 GEMMs only (C4 down): G_ON vs G_OFF
    def setter(on):
        lib.rdx_gemm_debug_group_m_bigk(int(os.environ.get("G_ON", "6") if on else os.environ.get("G_OFF", "16")))
elif what == "norm":  # model-level switch: rmsnorm overlapping the residual GEMM's tail
    def setter(on):
        os.environ["RDX_NORM_OVERLAP"] = str(on)
elif what == "pair":  # gate|up + down as one launch (rdx_gemm_pair) vs two launches
    setter = lib.rdx_gemm_debug_pair
elif what == "chain":  # model-level switch: norm -> next GEMM chained on ready counters
    def setter(on):
        os.environ["RDX_NORM_CHAIN"] = str(on)
elif what == "normw":  # rmsnorm_rows_after blocks of 4 warps (fit beside a GEMM CTA) vs 8
    def setter(on):
        lib.rdx_norm_debug_warps(4 if on else 8)
elif what == "backoff":  # norm slab-poller backoff cap B_ON vs B_OFF ns (device variable: set per replay)
    def setter(on):
        lib.rdx_norm_debug_backoff(int(os.environ.get("B_ON", "512") if on else os.environ.get("B_OFF", "2048")))
elif what == "colpart":  # GEMM column partition of few-round launches
    setter = lib.rdx_gemm_debug_colpart
else:
    setter = lib.rdx_debug_pdl if what == "pdl" else lib.rdx_gemm_debug_tail_split
config, _, batch, _ = bench.workload(cfg_name, 1, "weak")
w = DeviceWeights.random(config, seed=0)
db = DeviceBatch.from_batch(batch)
arms = {}
for on in (1, 0):
    setter(on)
    rr = RadixReranker(RadixQwen3(config, w, use_graphs=True))
    for _ in range(3):
        rr.score_device(db)  # captures this arm's graph with the switch in this state
    torch.cuda.synchronize()
    arms[on] = rr
flush = bench.L2Flusher()
res = {1: [], 0: []}
for it in range(int(os.environ.get("AB_ITERS", "20"))):
    for on in (1, 0):
        flush()
        if what == "backoff":
            setter(on)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        arms[on].score_device(db)
        e.record()
        e.synchronize()
        res[on].append(s.elapsed_time(e))
med = {k: sorted(v)[len(v) // 2] for k, v in res.items()}
print(f"{what} on: median {med[1]:.4f} ms   off: median {med[0]:.4f} ms   ({(med[0] / med[1] - 1) * 100:+.1f}% from on)")
