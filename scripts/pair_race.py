"""Determinism probe of the MLP pair launch: the same prefill repeated (pair on / off),
radix vs no-dedup, eager; prints max |diff| of last-token logits."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_15013_b200 import DeviceWeights, RadixQwen3, _native  # noqa: E402
from paper_2601_15013_b200.model import QWEN3_PRESETS, DeviceBatch, Qwen3Config  # noqa: E402
from paper_2601_15013_b200.plan import build_plan_device  # noqa: E402
from paper_2601_15013_b200.workloads import RerankSpec, msmarco_rerank_batch  # noqa: E402

base = QWEN3_PRESETS["qwen3-0.6b"]
L = int(os.environ.get("LAYERS", "4"))
cfg = Qwen3Config(L, base.hidden_size, base.intermediate_size, base.num_heads, base.num_kv_heads, base.head_dim,
                  base.vocab_size, base.rope_theta, base.norm_eps)
w = DeviceWeights.random(cfg, seed=7)
db = DeviceBatch.from_batch(msmarco_rerank_batch(RerankSpec(passages_per_query=64)))
plan = build_plan_device(db.tok, db.pos, db.cu)
res = {}
for pair in (True, False):
    m = RadixQwen3(cfg, w, use_graphs=False)
    m.mlp_pair = pair
    for p in (plan, None):
        outs = [m.prefill(db, p, logits="last").clone() for _ in range(4)]
        torch.cuda.synchronize()
        res[(pair, p is None)] = outs
        spread = max((o - outs[0]).abs().max().item() for o in outs)
        print(f"pair={pair} nodedup={p is None}: run-to-run max|diff| {spread:.3e}", flush=True)
ref = res[(False, False)][0]
for k, v in res.items():
    print(k, "vs two-launch radix:", (v[0] - ref).abs().max().item())
