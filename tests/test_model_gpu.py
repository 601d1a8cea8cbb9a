"""RadixQwen3 prefill on the GPU vs the reference's golden logits (fp64).

Tolerance (BASELINE.json north star): max |gpu - ref| / max |ref| <= 2e-2 on
final logits, bf16 weights/activations vs the fp64 reference.  Dedup on vs
off, and both attention-boundary modes, are compared against each other too.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 2e-2


def maxrel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def test_patterns_vs_reference(golden_forward):
    from paper_2601_15013_b200 import ModelConfig, forward, init_params
    from paper_2601_15013_b200.workloads import Pattern, make_pattern_batch

    cfg = ModelConfig()
    params = init_params(cfg, seed=7)
    for pat in Pattern:
        b = make_pattern_batch(pat, seed=3)
        ref = golden_forward[f"pattern_{pat.value}_logits"]
        for plan in (None, "auto"):
            for attention in ("suffix", "full"):
                out = forward(cfg, params, b, plan=plan, attention=attention).cpu().numpy()
                assert out.shape == ref.shape
                assert maxrel(out, ref) <= TOL, (pat.value, plan, attention, maxrel(out, ref))


def test_c1_vs_reference(golden_forward):
    from paper_2601_15013_b200 import TINY_C1, forward, init_params
    from paper_2601_15013_b200.workloads import SyntheticSpec, make_synthetic_batch

    params = init_params(TINY_C1, seed=0)
    b = make_synthetic_batch(SyntheticSpec(B=8, prefix_len=32, suffix_len=16, vocab=1024, seed=0))
    ref = golden_forward["c1_logits"]
    base = forward(TINY_C1, params, b).cpu().numpy()
    radix = forward(TINY_C1, params, b, plan="auto").cpu().numpy()
    full = forward(TINY_C1, params, b, plan="auto", attention="full").cpu().numpy()
    assert maxrel(base, ref) <= TOL
    assert maxrel(radix, ref) <= TOL
    assert maxrel(full, ref) <= TOL
    # full-layout attention boundary = the reference's algorithm; rows are bit-identical to dedup off
    assert np.array_equal(full, base)


def test_qwen3_06b_slice_vs_reference(golden_forward):
    from paper_2601_15013_b200 import Qwen3Config, forward, init_params
    from paper_2601_15013_b200.workloads import SyntheticSpec, make_synthetic_batch

    cfg = Qwen3Config(1, 1024, 3072, 16, 8, 128, 512, 1e6, 1e-6)
    params = init_params(cfg, seed=0)
    b = make_synthetic_batch(SyntheticSpec(B=4, prefix_len=48, suffix_len=16, vocab=512, seed=5))
    ref = golden_forward["q06_slice_logits"]
    for plan in (None, "auto"):
        out = forward(cfg, params, b, plan=plan).cpu().numpy()
        assert maxrel(out, ref) <= TOL, (plan, maxrel(out, ref))


def test_last_token_logits_match_full(golden_forward):
    from paper_2601_15013_b200 import TINY_C1, forward, init_params
    from paper_2601_15013_b200.workloads import SyntheticSpec, make_synthetic_batch

    params = init_params(TINY_C1, seed=0)
    b = make_synthetic_batch(SyntheticSpec(B=8, prefix_len=32, suffix_len=16, vocab=1024, seed=0))
    last = forward(TINY_C1, params, b, plan="auto", logits="last").cpu().numpy()
    ref = golden_forward["c1_logits"][b.cu_seqlens[1:] - 1]
    assert maxrel(last, ref) <= TOL


def test_ledger_law():
    """tests/test_model.py:265-283: m + L*(3n + m) + n row copies with the full boundary."""
    from paper_2601_15013_b200 import FlopLedger, ModelConfig, build_plan, forward, init_params
    from paper_2601_15013_b200.workloads import Pattern, make_pattern_batch

    cfg = ModelConfig(num_layers=1, hidden_size=64, intermediate_size=128, num_heads=2, num_kv_heads=1,
                      head_dim=32, vocab_size=11)
    params = init_params(cfg, seed=0)
    b = make_pattern_batch(Pattern.COMPLEX_SHARING, seed=3, vocab=11)
    plan = build_plan(b)
    n, m = plan.n_original, plan.n_compact
    base, radix = FlopLedger(), FlopLedger()
    forward(cfg, params, b, ledger=base)
    forward(cfg, params, b, plan=plan, ledger=radix, attention="full")
    assert all(rows == n for _, rows in base.phases)
    assert all(rows == m for _, rows in radix.phases)
    assert base.attention_row_ops == radix.attention_row_ops == n * cfg.num_layers
    assert base.gather_scatter_rows == 0
    assert radix.gather_scatter_rows == m + cfg.num_layers * (3 * n + m) + n


def test_padded_plan_identical():
    from paper_2601_15013_b200 import ModelConfig, build_plan, forward, init_params, pad_plan
    from paper_2601_15013_b200.workloads import Pattern, make_pattern_batch

    cfg = ModelConfig(num_layers=1, hidden_size=64, intermediate_size=128, num_heads=2, num_kv_heads=1,
                      head_dim=32, vocab_size=11)
    params = init_params(cfg, seed=1)
    b = make_pattern_batch(Pattern.SHARED_PREFIX, seed=3, vocab=11)
    plan = build_plan(b)
    a = forward(cfg, params, b, plan=plan).cpu().numpy()
    p = forward(cfg, params, b, plan=pad_plan(plan, 16)).cpu().numpy()
    assert np.array_equal(a, p)


def test_plan_batch_mismatch():
    from paper_2601_15013_b200 import ModelConfig, PlanBatchMismatch, build_plan, forward, init_params
    from paper_2601_15013_b200.ragged import RaggedBatch, default_positions

    cfg = ModelConfig(num_layers=1, hidden_size=64, intermediate_size=128, num_heads=2, num_kv_heads=1,
                      head_dim=32, vocab_size=11)
    params = init_params(cfg, seed=0)
    cu = np.array([0, 3, 6])
    b = RaggedBatch(np.array([1, 2, 3, 1, 2, 4]), default_positions(cu), cu)
    cu2 = np.array([0, 2, 4])
    other = RaggedBatch(np.array([1, 2, 1, 2]), default_positions(cu2), cu2)
    with pytest.raises(PlanBatchMismatch):
        forward(cfg, params, b, plan=build_plan(other))


def test_causality():
    from paper_2601_15013_b200 import ModelConfig, forward, init_params
    from paper_2601_15013_b200.ragged import RaggedBatch, default_positions

    cfg = ModelConfig(num_layers=1, hidden_size=64, intermediate_size=128, num_heads=2, num_kv_heads=1,
                      head_dim=32, vocab_size=11)
    params = init_params(cfg, seed=2)
    cu = np.array([0, 3, 7])
    a_b = RaggedBatch(np.array([1, 2, 3, 1, 2, 4, 5]), default_positions(cu), cu)
    p_b = RaggedBatch(np.array([1, 2, 3, 1, 9, 4, 5]), default_positions(cu), cu)
    for plan, att in ((None, "suffix"), ("auto", "full")):
        a = forward(cfg, params, a_b, plan=plan, attention=att).cpu().numpy()
        p = forward(cfg, params, p_b, plan=plan, attention=att).cpu().numpy()
        diff = np.abs(a - p).max(axis=1)
        assert np.all(diff[:4] == 0.0)
        assert np.all(diff[4:] > 0.0)


def test_fused_norm_path_matches_reference():
    """RMSNorm folded into the GEMMs (RDX_EPI_RESID_NORM + row_ss) gives the reference's logits."""
    import torch

    from oracle import oracle as orc
    from paper_2601_15013_b200 import TINY_C1, DeviceWeights, RadixQwen3, build_plan, init_params
    from paper_2601_15013_b200.model import DeviceBatch
    from paper_2601_15013_b200.workloads import SyntheticSpec, make_synthetic_batch

    batch = make_synthetic_batch(SyntheticSpec(B=8, prefix_len=32, suffix_len=16, vocab=1024, seed=0))
    params = init_params(TINY_C1, seed=0)
    model = RadixQwen3(TINY_C1, DeviceWeights.from_params(TINY_C1, params), fused_norm=True)
    out = model.prefill(DeviceBatch.from_batch(batch), build_plan(batch)).float().cpu().numpy()
    ref = orc.forward_oracle(TINY_C1, params, batch.token_ids, batch.position_ids, batch.cu_seqlens)
    err = float(np.abs(out - ref).max() / np.abs(ref).max())
    assert err <= 2e-2, err
    torch.cuda.synchronize()


def test_norm_overlap_bit_identical():
    """rmsnorm overlapped with the residual GEMM (slab counters + programmatic dependent
    launch, the default) gives the same logits as the stream-ordered passes, eager and
    under CUDA graphs, dedup on and off."""
    import torch

    from paper_2601_15013_b200 import DeviceWeights, RadixQwen3
    from paper_2601_15013_b200.model import QWEN3_PRESETS, DeviceBatch, Qwen3Config
    from paper_2601_15013_b200.plan import build_plan_device
    from paper_2601_15013_b200.workloads import RerankSpec, msmarco_rerank_batch

    base = QWEN3_PRESETS["qwen3-0.6b"]
    cfg = Qwen3Config(3, base.hidden_size, base.intermediate_size, base.num_heads, base.num_kv_heads, base.head_dim,
                      base.vocab_size, base.rope_theta, base.norm_eps)
    w = DeviceWeights.random(cfg, seed=3)
    batch = msmarco_rerank_batch(RerankSpec(passages_per_query=16))
    db = DeviceBatch.from_batch(batch)
    plan = build_plan_device(db.tok, db.pos, db.cu)
    outs = {}
    for graphs in (False, True):
        for overlap, chain in ((True, True), (True, False), (False, False)):
            m = RadixQwen3(cfg, w, use_graphs=graphs)
            m.norm_overlap, m.norm_chain = overlap, chain
            for p in (plan, None):
                o = m.prefill(db, p, logits="last")
                o = m.prefill(db, p, logits="last").clone()  # second call: graph replay
                torch.cuda.synchronize()
                outs[(graphs, overlap, chain, p is None)] = o
    for key, o in outs.items():
        assert torch.equal(o, outs[(False, False, False, key[3])]), key
    from paper_2601_15013_b200 import _native

    _native.check_device_status()  # no slab wait timed out on the way


@pytest.mark.parametrize("graphs", [False, True])
def test_mlp_pair_bit_identical(graphs):
    """gate|up and down in one persistent launch (rdx_gemm_pair) == two launches, bit for
    bit, with the overlapped norms on, eager and under CUDA graphs, dedup on and off."""
    import torch

    from paper_2601_15013_b200 import DeviceWeights, RadixQwen3, _native
    from paper_2601_15013_b200.model import QWEN3_PRESETS, DeviceBatch, Qwen3Config
    from paper_2601_15013_b200.plan import build_plan_device
    from paper_2601_15013_b200.workloads import RerankSpec, msmarco_rerank_batch

    base = QWEN3_PRESETS["qwen3-0.6b"]
    cfg = Qwen3Config(4, base.hidden_size, base.intermediate_size, base.num_heads, base.num_kv_heads, base.head_dim,
                      base.vocab_size, base.rope_theta, base.norm_eps)
    w = DeviceWeights.random(cfg, seed=7)
    db = DeviceBatch.from_batch(msmarco_rerank_batch(RerankSpec(passages_per_query=64)))
    plan = build_plan_device(db.tok, db.pos, db.cu)
    outs = {}
    for pair in (True, False):
        m = RadixQwen3(cfg, w, use_graphs=graphs)
        m.mlp_pair = pair
        for p in (plan, None):
            m.prefill(db, p, logits="last")
            outs[(pair, p is None)] = m.prefill(db, p, logits="last").clone()
    torch.cuda.synchronize()
    _native.check_device_status()
    for nd in (False, True):
        assert torch.equal(outs[(True, nd)], outs[(False, nd)])


@pytest.mark.parametrize("preset,layers", [("qwen3-0.6b", 4), ("qwen3-4b", 2), ("qwen3-8b", 2)])
def test_norm_chain_bit_identical_widths(preset, layers):
    """The chained norm -> GEMM pipeline (the GEMM streams rows the norm publishes on
    ready counters) at every model width (d = 1024 / 2560 / 4096: 4, 2 and 1 warps per
    norm block beside the GEMM CTA) equals the stream-ordered passes bit for bit."""
    import torch

    from paper_2601_15013_b200 import DeviceWeights, RadixQwen3, _native
    from paper_2601_15013_b200.model import QWEN3_PRESETS, DeviceBatch, Qwen3Config
    from paper_2601_15013_b200.plan import build_plan_device
    from paper_2601_15013_b200.workloads import RerankSpec, msmarco_rerank_batch

    base = QWEN3_PRESETS[preset]
    cfg = Qwen3Config(layers, base.hidden_size, base.intermediate_size, base.num_heads, base.num_kv_heads,
                      base.head_dim, base.vocab_size, base.rope_theta, base.norm_eps)
    w = DeviceWeights.random(cfg, seed=5)
    db = DeviceBatch.from_batch(msmarco_rerank_batch(RerankSpec(queries=2, passages_per_query=32)))
    plan = build_plan_device(db.tok, db.pos, db.cu)
    outs = []
    for overlap, chain in ((True, True), (False, False)):
        m = RadixQwen3(cfg, w, use_graphs=False)
        m.norm_overlap, m.norm_chain = overlap, chain
        outs.append(m.prefill(db, plan, logits="last").clone())
    torch.cuda.synchronize()
    _native.check_device_status()
    assert torch.equal(outs[0], outs[1])


def test_graph_buckets_distinct_batches():
    """A stream of DISTINCT batches (different N, N', B, lengths) through CUDA-graph buckets:
    every result equals the eager forward bit for bit, batches of one bucket share a graph,
    the cache stays within max_graphs (LRU) and out-of-vocab ids raise on the graph path."""
    import torch

    from paper_2601_15013_b200 import DeviceWeights, IndexOutOfRange, RadixQwen3
    from paper_2601_15013_b200.model import DeviceBatch, Qwen3Config
    from paper_2601_15013_b200.plan import build_plan_device
    from paper_2601_15013_b200.workloads import RerankSpec, msmarco_rerank_batch

    cfg = Qwen3Config(2, 256, 512, 4, 2, 64, 4096, 1e6, 1e-6)
    w = DeviceWeights.random(cfg, seed=5)
    eager = RadixQwen3(cfg, w)
    graphs = RadixQwen3(cfg, w, use_graphs=True, max_graphs=3)
    specs = [RerankSpec(passages_per_query=p, vocab=4096, seed=s) for s, p in
             ((0, 16), (1, 16), (2, 17), (3, 30), (4, 16), (5, 33), (6, 9), (7, 16))]
    keys = set()
    for spec in specs:
        db = DeviceBatch.from_batch(msmarco_rerank_batch(spec))
        plan = build_plan_device(db.tok, db.pos, db.cu)
        for p in (plan, None):
            ref = eager.prefill(db, p, logits="last")
            got = graphs.prefill(db, p, logits="last")
            torch.cuda.synchronize()
            assert got.shape == ref.shape
            assert torch.equal(got, ref), (spec, p is None)
            lay = graphs._layout(db, p, "suffix")
            keys.add(graphs._graph_key(db, lay, "suffix" if p is not None else "plain", "last"))
        assert len(graphs._graphs) <= 3
    assert graphs.graph_captures >= len(keys) and len(keys) < 2 * len(specs)
    # all-logits output through a bucket (padded rows sliced off)
    db = DeviceBatch.from_batch(msmarco_rerank_batch(specs[0]))
    plan = build_plan_device(db.tok, db.pos, db.cu)
    assert torch.equal(graphs.prefill(db, plan), eager.prefill(db, plan))
    # device batch with an unknown max token id and an out-of-vocab id: the graph path checks on device
    bad = DeviceBatch(db.tok.clone(), db.pos, db.cu, db.cu32, db.cu_host, db.n, db.b, db.max_len, -1)
    bad.tok[5] = cfg.vocab_size + 3
    with pytest.raises(IndexOutOfRange):
        graphs.prefill(bad, build_plan_device(bad.tok, bad.pos, bad.cu), logits="last")
