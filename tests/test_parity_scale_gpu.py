"""Parity at the benchmarked configurations (BASELINE.json configs[1]-[3]).

* Planner: the GPU plan of the FULL C2 (template and literal shapes), C3 and C4
  batches is bit-identical to the C restatement of the reference trie
  (oracle/trie_oracle.c, trie.py:73-148).
* Forward: the real Qwen3 dimensions against the oracle (model.py:322-416 restated,
  fp32 numpy) on sub-batches of the benchmark workloads:
    - Qwen3-0.6B, all 28 layers, vocab 151936, last-token logits, read out
      after 1, 2, 4, 7, 14 and 28 layers (error vs depth);
    - Qwen3-4B dimensions, 2 layers, on 4 sequences of the C3 batch (2 queries);
    - Qwen3-8B dimensions, 2 layers, on 2 sequences of the C4 batch (2048+256).
  Weights are drawn once (seeded uniform +-0.05, the init_params law), rounded
  to bf16 (what the GPU computes with) and handed to both sides, so the
  difference measured is the bf16 activation path against fp32 math.
  Tolerance: max |gpu - oracle| / max |oracle| <= 2e-2 on final logits
  (BASELINE.json north star), at every depth.
* Dedup on vs off on the same GPU at full depth: max-rel <= 2e-2 (suffix-query
  attention rounds differently), and the reference-algorithm boundary
  (attention="full") equal to dedup off (tests/test_model.py:201-209).
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 2e-2


def maxrel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def _record(name, payload):
    """Keep the measured errors (RDX_PARITY_LOG=<path>: appended as JSON lines)."""
    path = os.environ.get("RDX_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps({"test": name, **payload}) + "\n")
    print(name, payload)


# ------------------------------------------------------------------ planner
def _bench_batches():
    from paper_2601_15013_b200.workloads import RerankSpec, long_prefix_batch, msmarco_rerank_batch

    return {
        "c2_template": msmarco_rerank_batch(RerankSpec()),
        "c2_literal": msmarco_rerank_batch(RerankSpec(template_len=0, query_len=32, tail_len=0)),
        "c3": msmarco_rerank_batch(RerankSpec(queries=4)),
        "c4": long_prefix_batch(seed=0),
    }


@pytest.mark.parametrize("name", ["c2_template", "c2_literal", "c3", "c4"])
def test_planner_bit_exact_on_benchmark_batch(name, oracle):
    from paper_2601_15013_b200 import build_plan

    batch = _bench_batches()[name]
    plan = build_plan(batch)
    g, s, cp, m = oracle.build_plan_oracle(batch.token_ids, batch.position_ids, batch.cu_seqlens)
    assert plan.n_compact == m
    assert np.array_equal(plan.gather_indices, g)
    assert np.array_equal(plan.scatter_indices, s)
    assert np.array_equal(plan.compact_positions, cp)
    _record("planner_" + name, {"N": batch.num_tokens, "N_compact": m, "gamma": round(m / batch.num_tokens, 4)})


# ------------------------------------------------------------------ forward
def _weights(cfg, seed, layers):
    """(DeviceWeights, oracle params, token remap) from one seeded bf16 draw."""
    import torch

    from paper_2601_15013_b200 import DeviceWeights

    gen = torch.Generator(device="cuda").manual_seed(seed)
    d, di = cfg.hidden_size, cfg.intermediate_size
    dev = {}

    def u(*shape):
        w = torch.empty(shape, dtype=torch.float32, device="cuda")
        w.uniform_(-0.05, 0.05, generator=gen)
        return w.to(torch.bfloat16)

    dev["embed"], dev["lm_head"] = u(cfg.vocab_size, d), u(cfg.vocab_size, d)
    dev["final_norm"] = torch.ones(d, device="cuda")
    for i in range(layers):
        p = f"layers.{i}."
        dev.update({p + "wq": u(cfg.q_dim, d), p + "wk": u(cfg.kv_dim, d), p + "wv": u(cfg.kv_dim, d),
                    p + "wo": u(d, cfg.q_dim), p + "w_gate": u(di, d), p + "w_up": u(di, d),
                    p + "w_down": u(d, di)})
        for nm, n in (("ln1", d), ("ln2", d), ("q_norm", cfg.head_dim), ("k_norm", cfg.head_dim)):
            dev[p + nm] = torch.ones(n, device="cuda")
    from dataclasses import replace

    dw = DeviceWeights.from_tensors(replace(cfg, num_layers=layers), lambda n: dev[n])
    host = {k: v.float().cpu().numpy() for k, v in dev.items() if k != "embed"}
    return dw, host, dev["embed"]


def _oracle_logits(oracle, cfg, host, embed_dev, batch, depths):
    """Oracle last-token logits (radix plan of the oracle itself) at each depth."""
    import torch

    uniq, tok_small = np.unique(batch.token_ids, return_inverse=True)
    params = dict(host)
    params["embed"] = embed_dev[torch.from_numpy(uniq.astype(np.int64)).cuda()].float().cpu().numpy()
    g, s, cp, _ = oracle.build_plan_oracle(batch.token_ids, batch.position_ids, batch.cu_seqlens)
    return oracle.forward_oracle(cfg, params, tok_small, batch.position_ids, batch.cu_seqlens, plan=(g, s, cp),
                                 last_only=True, depths=depths)


def _gpu_logits(cfg, dw, batch, depth, plan="auto", attention="suffix"):
    from dataclasses import replace

    from paper_2601_15013_b200 import DeviceBatch, RadixQwen3

    model = RadixQwen3(replace(cfg, num_layers=depth), dw)
    return model.prefill(DeviceBatch.from_batch(batch), plan, attention=attention, logits="last").cpu().numpy()


def test_qwen3_06b_full_depth_vs_oracle(oracle):
    """All 28 layers at 0.6B dims, real vocab, 6 sequences of the C2 batch."""
    from paper_2601_15013_b200.model import QWEN3_PRESETS
    from paper_2601_15013_b200.shard import sub_batch
    from paper_2601_15013_b200.workloads import RerankSpec, msmarco_rerank_batch

    cfg = QWEN3_PRESETS["qwen3-0.6b"]
    batch = sub_batch(msmarco_rerank_batch(RerankSpec()), np.arange(6))
    dw, host, emb = _weights(cfg, 11, cfg.num_layers)
    depths = [1, 2, 4, 7, 14, 28]
    ref = _oracle_logits(oracle, cfg, host, emb, batch, depths)
    errs = {}
    for dep in depths:
        got = _gpu_logits(cfg, dw, batch, dep)
        errs[dep] = maxrel(got, ref[dep])
    nodedup = _gpu_logits(cfg, dw, batch, 28, plan=None)
    full = _gpu_logits(cfg, dw, batch, 28, attention="full")
    radix = _gpu_logits(cfg, dw, batch, 28)
    _record("qwen3_0.6b_depth", {"N": batch.num_tokens, "maxrel_by_depth": errs,
                                 "radix_vs_nodedup": maxrel(radix, nodedup),
                                 "full_vs_nodedup_bit_identical": bool(np.array_equal(full, nodedup))})
    assert all(e <= TOL for e in errs.values()), errs
    # RadixMLP is exact: every compact row is computed exactly as its original rows are
    # (same GEMM K order, same attention key tiles), so on and off agree bit for bit
    assert np.array_equal(radix, nodedup), maxrel(radix, nodedup)
    assert np.array_equal(full, nodedup)


@pytest.mark.parametrize("which", ["qwen3-4b", "qwen3-8b"])
def test_wide_slices_vs_oracle(which, oracle):
    """2-layer slices at 4B / 8B dimensions on sub-batches of the C3 / C4 workloads."""
    from paper_2601_15013_b200.model import QWEN3_PRESETS
    from paper_2601_15013_b200.shard import sub_batch
    from paper_2601_15013_b200.workloads import RerankSpec, long_prefix_batch, msmarco_rerank_batch

    cfg = QWEN3_PRESETS[which]
    if which == "qwen3-4b":
        batch = sub_batch(msmarco_rerank_batch(RerankSpec(queries=4)), np.array([0, 1, 64, 65]))
    else:
        batch = sub_batch(long_prefix_batch(seed=0), np.array([0, 1]))
    dw, host, emb = _weights(cfg, 13, 2)
    ref = _oracle_logits(oracle, cfg, host, emb, batch, [1, 2])
    errs = {dep: maxrel(_gpu_logits(cfg, dw, batch, dep), ref[dep]) for dep in (1, 2)}
    nodedup = _gpu_logits(cfg, dw, batch, 2, plan=None)
    full = _gpu_logits(cfg, dw, batch, 2, attention="full")
    radix = _gpu_logits(cfg, dw, batch, 2)
    _record(which + "_slice", {"N": batch.num_tokens, "maxrel_by_depth": errs,
                               "radix_vs_nodedup": maxrel(radix, nodedup),
                               "full_vs_nodedup_bit_identical": bool(np.array_equal(full, nodedup))})
    assert all(e <= TOL for e in errs.values()), errs
    # RadixMLP is exact: every compact row is computed exactly as its original rows are
    # (same GEMM K order, same attention key tiles), so on and off agree bit for bit
    assert np.array_equal(radix, nodedup), maxrel(radix, nodedup)
    assert np.array_equal(full, nodedup)
