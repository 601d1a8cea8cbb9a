"""Row kernels (rmsnorm, embed+rmsnorm, RoPE table, rerank read-out) vs torch fp32 references,
and CUDA-graph replay == eager launches."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _call(name, *args):
    from paper_2601_15013_b200 import _native

    _native.check(getattr(_native.lib(), name)(*args, _native.stream_handle()), name)


@pytest.mark.parametrize("d", [64, 256, 1024, 2560, 4096, 1000])
def test_rmsnorm_rows(d):
    import torch

    if d % 8:
        pytest.skip("kernel contract: d % 8 == 0")
    x = torch.randn(333, d, device="cuda") * 3
    w = torch.rand(d, device="cuda") + 0.5
    rows = torch.randint(0, 333, (57,), device="cuda", dtype=torch.int32)
    out = torch.empty(57, d, dtype=torch.bfloat16, device="cuda")
    _call("rdx_rmsnorm_rows", x.data_ptr(), x.stride(0), rows.data_ptr(), 57, d, w.data_ptr(), 1e-6,
          out.data_ptr(), out.stride(0))
    xs = x[rows.long()]
    ref = xs / torch.sqrt((xs * xs).mean(1, keepdim=True) + 1e-6) * w
    assert (out.float() - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()


def test_embed_rmsnorm_gather():
    import torch

    V, d, n = 500, 1024, 300
    emb = (torch.randn(V, d, device="cuda") * 0.05).to(torch.bfloat16)
    w = torch.rand(d, device="cuda") + 0.5
    tok = torch.randint(0, V, (n,), device="cuda", dtype=torch.int32)
    gather = torch.randint(0, n, (200,), device="cuda", dtype=torch.int32)
    h = torch.empty(200, d, device="cuda")
    hn = torch.empty(200, d, dtype=torch.bfloat16, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    _call("rdx_embed_rmsnorm", tok.data_ptr(), gather.data_ptr(), 200, emb.data_ptr(), V, d, w.data_ptr(), 1e-6,
          h.data_ptr(), hn.data_ptr(), err.data_ptr())
    rows = emb[tok[gather.long()].long()].float()
    assert torch.equal(h, rows)
    ref = rows / torch.sqrt((rows * rows).mean(1, keepdim=True) + 1e-6) * w
    assert (hn.float() - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()
    assert int(err.item()) == 0


def test_rope_table_fp64_accurate():
    import torch

    pos = torch.tensor([0, 1, 7, 2303, 40000], dtype=torch.int32, device="cuda")
    hd, theta = 128, 1e6
    t = torch.empty(5, hd // 2, 2, device="cuda")
    _call("rdx_rope_table", pos.data_ptr(), 5, hd, theta, t.data_ptr())
    inv = theta ** (-np.arange(0, hd, 2, dtype=np.float64) / hd)
    ang = pos.cpu().numpy().astype(np.float64)[:, None] * inv[None, :]
    ref = np.stack([np.cos(ang), np.sin(ang)], -1).astype(np.float32)
    assert np.abs(t.cpu().numpy() - ref).max() <= 1e-6


def test_rerank_scores():
    import torch

    logits = torch.randn(7, 300, device="cuda")
    out = torch.empty(7, device="cuda")
    _call("rdx_rerank_scores", logits.data_ptr(), 7, 300, 11, 5, out.data_ptr())
    ref = torch.sigmoid(logits[:, 11] - logits[:, 5])
    assert (out - ref).abs().max().item() <= 1e-5


def test_cuda_graph_replay_matches_eager():
    from paper_2601_15013_b200 import TINY_C1, DeviceBatch, DeviceWeights, RadixQwen3, init_params
    from paper_2601_15013_b200.workloads import SyntheticSpec, make_synthetic_batch

    params = init_params(TINY_C1, seed=0)
    w = DeviceWeights.from_params(TINY_C1, params)
    eager = RadixQwen3(TINY_C1, w, use_graphs=False)
    graphed = RadixQwen3(TINY_C1, w, use_graphs=True)
    for seed in (0, 1, 0):
        b = make_synthetic_batch(SyntheticSpec(B=8, prefix_len=32, suffix_len=16, vocab=1024, seed=seed))
        db = DeviceBatch.from_batch(b)
        for plan in (None, "auto"):
            for logits in ("last", "all"):
                a = eager.prefill(db, plan, logits=logits).cpu().numpy()
                g = graphed.prefill(db, plan, logits=logits).cpu().numpy()
                assert np.array_equal(a, g), (seed, plan, logits)
    assert len(graphed._graphs) == 4
