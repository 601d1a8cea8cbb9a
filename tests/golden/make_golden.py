"""Generate golden fixtures by importing the REFERENCE implementation.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/bindings/src \
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Outputs (committed, small):
  plans.npz      reference build_plan on the known-answer batches of
                 tests/test_trie.py, 1000 random_small_batch seeds
                 (test_acceptance.py:129-140), 200 batches with arbitrary
                 position ids, the fanout>8 case, the 15-row table
                 (test_acceptance.py:65-82) and the six patterns.
  synthetic.npz  reference make_synthetic_batch / make_pattern_batch tokens.
  forward.npz    reference forward() logits: six patterns on ModelConfig()
                 (seed 7), C1 (2L, d=64, 4 heads, 8x(32+16)), and a 1-layer
                 Qwen3-0.6B-dimension slice (q_dim != hidden via a subclass
                 that overrides only __post_init__, SURVEY finding 3).
  grads.npz      reference loss_and_grads() on C1: loss + every parameter gradient
                 (fp32) with the plan, loss without it.
  plan_toy.rdxp / plan_toy.json  reference serialisation of the toy plan.
"""

from __future__ import annotations

import os
import sys
from dataclasses import dataclass

import numpy as np

import radix_compact as rc
from radix_compact import trie
from radix_compact.bench import Pattern, SyntheticSpec, make_pattern_batch, make_synthetic_batch

OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/tests")
from conftest import random_small_batch  # noqa: E402  (reference test helper)


def make(tokens, cu):
    cu = np.asarray(cu, dtype=np.int64)
    return rc.RaggedBatch(np.asarray(tokens), rc.default_positions(cu), cu)


def pack(batches):
    """Concatenate a list of (batch, plan) into flat arrays + offsets."""
    tok, pos, cu, gat, sca = [], [], [], [], []
    n_off, b_off, m_off, ncomp = [0], [0], [0], []
    for batch, plan in batches:
        tok.append(batch.token_ids.astype(np.uint32))
        pos.append(batch.position_ids.astype(np.uint32))
        cu.append(batch.cu_seqlens.astype(np.int64))
        gat.append(plan.gather_indices)
        sca.append(plan.scatter_indices)
        n_off.append(n_off[-1] + batch.num_tokens)
        b_off.append(b_off[-1] + batch.cu_seqlens.shape[0])
        m_off.append(m_off[-1] + plan.n_compact)
        ncomp.append(plan.n_compact)
    return dict(tok=np.concatenate(tok), pos=np.concatenate(pos), cu=np.concatenate(cu),
                gather=np.concatenate(gat), scatter=np.concatenate(sca), n_off=np.array(n_off),
                b_off=np.array(b_off), m_off=np.array(m_off), n_compact=np.array(ncomp))


def plans():
    out = {}
    known = {
        "toy": make([1, 2, 3, 1, 2, 4], [0, 3, 6]),
        "single": make([7, 8, 9], [0, 3]),
        "identical": make([4, 5, 6, 4, 5, 6], [0, 3, 6]),
        "position_matters": make([3, 3, 1, 3], [0, 2, 4]),
        "divergence": make([1, 2, 9, 1, 3, 9], [0, 3, 6]),
        "gating_19_20": make([1, 2, 3, 1] + [9] * 16, [0, 3, 20]),
        "fanout_wide": make(np.concatenate([[i % 40, 7] for i in range(64)]), np.arange(65) * 2),
    }
    items = []
    for name, b in known.items():
        items.append((b, trie.build_plan(b)))
    out.update({f"known_{k}": v for k, v in pack(items).items()})
    out["known_names"] = np.array(list(known))

    rand = []
    for seed in range(1000):
        b = random_small_batch(np.random.default_rng(seed))
        rand.append((b, trie.build_plan(b)))
    out.update({f"rand_{k}": v for k, v in pack(rand).items()})

    # arbitrary position ids (the key is (pos << 32) ^ tok, trie.py:87)
    arb = []
    rng = np.random.default_rng(4242)
    for _ in range(200):
        bsz = int(rng.integers(1, 9))
        lens = rng.integers(1, 13, size=bsz)
        cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        tok = rng.integers(0, 3, size=int(cu[-1])).astype(np.uint32)
        pos = rng.integers(0, 3, size=int(cu[-1])).astype(np.uint32)
        b = rc.RaggedBatch(tok, pos, cu)
        arb.append((b, trie.build_plan(b)))
    out.update({f"arbpos_{k}": v for k, v in pack(arb).items()})

    # patterns (seed 3, vocab 97) -> plans
    pats = [(make_pattern_batch(p, seed=3), None) for p in Pattern]
    pats = [(b, trie.build_plan(b)) for b, _ in pats]
    out.update({f"pattern_{k}": v for k, v in pack(pats).items()})

    table = [(1, 256), (16, 256), (32, 256), (128, 256), (256, 256), (512, 256), (1024, 256), (2048, 256),
             (1, 1024), (32, 1024), (128, 1024), (256, 1024), (512, 1024), (1024, 1024), (2048, 1024)]
    rows = []
    for p, s in table:
        plan = trie.build_plan(make_synthetic_batch(SyntheticSpec(B=32, prefix_len=p, suffix_len=s)))
        rows.append((p, s, plan.n_original, plan.n_compact))
    out["table"] = np.array(rows, dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "plans.npz"), **out)


def synthetic():
    out = {}
    specs = [(32, 16, 8, 1024, 0), (8, 32, 16, 1024, 0), (5, 9, 4, 11, 2), (4, 6, 5, 1024, 1), (3, 0, 4, 64, 7)]
    for i, (b, p, s, v, seed) in enumerate(specs):
        batch = make_synthetic_batch(SyntheticSpec(B=b, prefix_len=p, suffix_len=s, vocab=v, seed=seed))
        out[f"spec{i}"] = np.array([b, p, s, v, seed])
        out[f"spec{i}_tok"] = batch.token_ids.astype(np.uint32)
    for pat in Pattern:
        for seed, vocab in ((3, 97), (3, 11), (0, 97)):
            b = make_pattern_batch(pat, seed=seed, vocab=vocab)
            out[f"pat_{pat.value}_{seed}_{vocab}_tok"] = b.token_ids.astype(np.uint32)
            out[f"pat_{pat.value}_{seed}_{vocab}_cu"] = b.cu_seqlens.astype(np.int64)
    np.savez_compressed(os.path.join(OUT, "synthetic.npz"), **out)


@dataclass(frozen=True)
class Qwen3Like(rc.ModelConfig):
    def __post_init__(self):  # only relax hidden == heads * head_dim (SURVEY finding 3)
        pass


def forward():
    out = {}
    cfg = rc.ModelConfig()
    params = rc.init_params(cfg, seed=7)
    for pat in Pattern:
        b = make_pattern_batch(pat, seed=3)
        base = rc.forward(cfg, params, b)
        radix = rc.forward(cfg, params, b, plan=trie.build_plan(b))
        assert np.array_equal(base, radix)
        out[f"pattern_{pat.value}_logits"] = base

    c1 = rc.ModelConfig(num_layers=2, hidden_size=64, intermediate_size=192, num_heads=4, num_kv_heads=2,
                        head_dim=16, vocab_size=1024)
    p1 = rc.init_params(c1, seed=0)
    b1 = make_synthetic_batch(SyntheticSpec(B=8, prefix_len=32, suffix_len=16, vocab=1024, seed=0))
    plan1 = trie.build_plan(b1)
    l1 = rc.forward(c1, p1, b1)
    assert np.array_equal(l1, rc.forward(c1, p1, b1, plan=plan1))
    out["c1_logits"] = l1.astype(np.float32)
    out["c1_n_compact"] = np.array(plan1.n_compact)

    q = Qwen3Like(num_layers=1, hidden_size=1024, intermediate_size=3072, num_heads=16, num_kv_heads=8,
                  head_dim=128, vocab_size=512, rope_theta=1e6, norm_eps=1e-6)
    pq = rc.init_params(q, seed=0)
    bq = make_synthetic_batch(SyntheticSpec(B=4, prefix_len=48, suffix_len=16, vocab=512, seed=5))
    lq = rc.forward(q, pq, bq)
    assert np.array_equal(lq, rc.forward(q, pq, bq, plan=trie.build_plan(bq)))
    out["q06_slice_logits"] = lq.astype(np.float32)
    np.savez_compressed(os.path.join(OUT, "forward.npz"), **out)


def grads():
    """Reference loss_and_grads (model.py:419-531) on C1 with seeded targets: loss and
    every gradient with the plan, loss without it."""
    out = {}
    c1 = rc.ModelConfig(num_layers=2, hidden_size=64, intermediate_size=192, num_heads=4, num_kv_heads=2,
                        head_dim=16, vocab_size=1024)
    p1 = rc.init_params(c1, seed=0)
    b1 = make_synthetic_batch(SyntheticSpec(B=8, prefix_len=32, suffix_len=16, vocab=1024, seed=0))
    t1 = np.random.default_rng(11).integers(0, c1.vocab_size, size=b1.num_tokens)
    out["c1_targets"] = t1
    loss, g = rc.loss_and_grads(c1, p1, b1, trie.build_plan(b1), t1)
    out["c1_radix_loss"] = np.array(loss)
    for name, val in g.items():  # fp32 storage: 6e-8 relative, far inside the 1e-6 check
        out[f"c1_radix_grad:{name}"] = val.astype(np.float32)
    loss_base, _ = rc.loss_and_grads(c1, p1, b1, None, t1)
    out["c1_base_loss"] = np.array(loss_base)
    np.savez_compressed(os.path.join(OUT, "grads.npz"), **out)


def serial():
    plan = trie.build_plan(make([1, 2, 3, 1, 2, 4], [0, 3, 6]))
    trie.save_plan(plan, os.path.join(OUT, "plan_toy.rdxp"), binary=True)
    trie.save_plan(plan, os.path.join(OUT, "plan_toy.json"))


if __name__ == "__main__":
    plans()
    synthetic()
    forward()
    grads()
    serial()
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))
