"""Public reranking API: host batch in, per-sequence scores out.

``RadixReranker.score(batch)`` is the call a user makes (and what bench.py's
``e2e`` number measures): pinned-host -> HBM copy of the packed ids, GPU
plan build, RadixMLP prefill with last-token logits (the scoring contract of
model.py), the Qwen3-reranker read-out ``sigmoid(logit_yes - logit_no)``
(= softmax([no, yes])[yes]) in ``rdx_rerank_scores``, and a D2H copy of the
B scores.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .model import DeviceBatch, ModelConfig, RadixQwen3
from .plan import build_plan_device
from .ragged import RaggedBatch, validate_batch

# Qwen3 tokenizer ids of "yes" / "no" (the Qwen3-Reranker read-out tokens)
QWEN3_YES_ID = 9693
QWEN3_NO_ID = 2152


class _Pinned:
    """Grow-only pinned staging buffers for the packed batch."""

    def __init__(self):
        self.bufs = {}

    def get(self, name, n, dtype):
        import torch

        buf = self.bufs.get(name)
        if buf is None or buf.numel() < n or buf.dtype != dtype:
            buf = torch.empty(max(n, 1), dtype=dtype, pin_memory=True)
            self.bufs[name] = buf
        return buf[:n]


class RadixReranker:
    def __init__(self, model: RadixQwen3, yes_id: int = QWEN3_YES_ID, no_id: int = QWEN3_NO_ID,
                 dedup: bool = True, attention: str = "suffix"):
        cfg: ModelConfig = model.config
        self.model = model
        self.yes_id = min(yes_id, cfg.vocab_size - 1)
        self.no_id = min(no_id, cfg.vocab_size - 1)
        self.dedup = dedup
        self.attention = attention
        self._pinned = _Pinned()
        self.last_plan = None
        self.h2d_bytes = 0
        self.d2h_bytes = 0

    def upload(self, batch: RaggedBatch, slot: int = 0) -> DeviceBatch:
        """Pinned staging (slot = double-buffer index for pipelined streams) -> HBM, async."""
        import torch

        n, b = batch.num_tokens, batch.num_sequences
        tok = self._pinned.get(f"tok{slot}", n, torch.int32)
        pos = self._pinned.get(f"pos{slot}", n, torch.int32)
        cu = self._pinned.get(f"cu{slot}", b + 1, torch.int64)
        tok.numpy()[:] = batch.token_ids.view(np.int32)
        pos.numpy()[:] = batch.position_ids.view(np.int32)
        cu.numpy()[:] = batch.cu_seqlens
        dt, dp, dc = (x.to("cuda", non_blocking=True) for x in (tok, pos, cu))
        cu_host = np.asarray(batch.cu_seqlens, dtype=np.int64)
        lens = np.diff(cu_host)
        self.h2d_bytes = tok.numel() * 4 + pos.numel() * 4 + cu.numel() * 8
        # host max token id (O(N) next to the copy): out-of-vocab ids raise IndexOutOfRange before
        # any launch, on the eager and the CUDA-graph path alike
        max_token = int(batch.token_ids.max()) if n else -1
        return DeviceBatch(dt, dp, dc, dc.to(torch.int32), cu_host, n, b, int(lens.max()) if lens.size else 0,
                           max_token)

    def plan(self, db: DeviceBatch):
        """GPU plan of a device batch (None when dedup is off)."""
        return build_plan_device(db.tok, db.pos, db.cu) if self.dedup else None

    def score_device(self, db: DeviceBatch, plan="build"):
        """Device-resident batch -> device scores [B] (float32).  ``plan``: "build" (GPU
        planner now), or a plan prepared earlier (pipelined streams)."""
        import torch

        if isinstance(plan, str) and plan == "build":
            plan = self.plan(db)
        self.last_plan = plan
        logits = self.model.prefill(db, plan, attention=self.attention, logits="last")
        scores = torch.empty(db.b, dtype=torch.float32, device=logits.device)
        code = _native.lib().rdx_rerank_scores(logits.data_ptr(), db.b, logits.stride(0), self.yes_id,
                                               self.no_id, scores.data_ptr(), _native.stream_handle())
        _native.check(code, "rdx_rerank_scores")
        return scores

    def score(self, batch: RaggedBatch) -> np.ndarray:
        """Host batch -> host scores [B]."""
        validate_batch(batch)
        scores = self.score_device(self.upload(batch))
        out = scores.cpu().numpy()
        _native.check_device_status()  # an overlapped-norm wait that timed out fails here, not silently
        # D2H: the plan's (N', status, cu_q) read (dedup only) and the scores
        self.d2h_bytes = out.nbytes + ((4 + batch.num_sequences + 1) * 4 if self.dedup else 0)
        return out

    def score_many(self, batches) -> list:
        """Scores of a stream of host batches; batch t+1's upload and plan build overlap
        batch t's prefill (pipeline.score_stream).  Same results as ``score`` per batch."""
        from .pipeline import score_stream

        out = score_stream(self, batches)
        if out:
            last = batches[-1]
            self.d2h_bytes = out[-1].nbytes + ((4 + last.num_sequences + 1) * 4 if self.dedup else 0)
        return out
