"""Multi-GPU partitioning by trie subtree.

RadixMLP is per-batch and stateless, so the batch shards into
independent sub-batches of whole sequences; each GPU builds the plan of its
own sub-batch (bit-exact to the reference's build_plan on that sub-batch)
and runs the full prefill on it.  No collective runs on the hot path; only
the per-sequence scores are all-gathered at the end.

Partition: sort sequences lexicographically by their (token, position) path
(trie DFS order), so every trie subtree is a contiguous run; then cut the
sorted order into ``world`` chunks of balanced compact-row cost, moving each
cut to the adjacent pair with the smallest shared prefix inside a window
around the balanced cut point.  Shared rows are duplicated only at cuts, and
a cut at LCP 0 (distinct root subtrees) duplicates nothing.  When the root
has a single child (a common system prompt), the same rule descends to the
first level with fanout: cuts land between different queries.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .ragged import RaggedBatch


def _seq_keys(batch: RaggedBatch):
    cu = batch.cu_seqlens
    keys = []
    for s in range(batch.num_sequences):
        lo, hi = int(cu[s]), int(cu[s + 1])
        pair = (batch.position_ids[lo:hi].astype(np.uint64) << np.uint64(32)) | batch.token_ids[lo:hi].astype(np.uint64)
        keys.append(pair)
    return keys


def _lcp(a: np.ndarray, b: np.ndarray) -> int:
    n = min(a.shape[0], b.shape[0])
    if n == 0:
        return 0
    neq = np.flatnonzero(a[:n] != b[:n])
    return int(neq[0]) if neq.size else n


def trie_order(batch: RaggedBatch):
    """Sequence indices in trie (lexicographic path) order and adjacent LCPs."""
    keys = _seq_keys(batch)
    order = sorted(range(len(keys)), key=lambda s: tuple(keys[s].tolist()))
    lcps = np.array([_lcp(keys[order[i]], keys[order[i + 1]]) for i in range(len(order) - 1)], dtype=np.int64)
    return np.array(order, dtype=np.int64), lcps


@dataclass
class Shard:
    rank: int
    seq_ids: np.ndarray      # original sequence indices, in original order
    batch: RaggedBatch       # the sub-batch
    est_compact_rows: int    # compact rows this shard computes


def sub_batch(batch: RaggedBatch, seq_ids) -> RaggedBatch:
    cu = batch.cu_seqlens
    seq_ids = np.asarray(seq_ids, dtype=np.int64)
    toks, poss, lens = [], [], []
    for s in seq_ids:
        lo, hi = int(cu[s]), int(cu[s + 1])
        toks.append(batch.token_ids[lo:hi])
        poss.append(batch.position_ids[lo:hi])
        lens.append(hi - lo)
    new_cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    tok = np.concatenate(toks) if toks else np.zeros(0, np.uint32)
    pos = np.concatenate(poss) if poss else np.zeros(0, np.uint32)
    return RaggedBatch(tok, pos, new_cu)


def partition_by_subtree(batch: RaggedBatch, world: int, window: float = 0.25) -> list[Shard]:
    """Split ``batch`` into ``world`` shards along trie-subtree boundaries."""
    if world < 1:
        raise ValueError("world must be >= 1")
    b = batch.num_sequences
    order, lcps = trie_order(batch)
    lens = np.diff(batch.cu_seqlens)[order]
    # compact rows each sequence adds in trie order = L - lcp(prev)
    unique = lens - np.concatenate([[0], lcps]) if b else np.zeros(0, np.int64)
    csum = np.concatenate([[0], np.cumsum(unique)])
    total = int(csum[-1])
    cuts = [0]
    for g in range(1, world):
        target = total * g / world
        ideal = int(np.searchsorted(csum, target))
        lo = max(cuts[-1] + 1, int(ideal - window * b / world))
        hi = min(b - (world - g), int(ideal + window * b / world))
        if lo > hi:
            cut = min(max(ideal, cuts[-1] + 1), b - (world - g))
        else:
            cand = np.arange(lo, hi + 1)
            # prefer the smallest LCP across the cut, then closeness to the balanced point
            lcp_at = lcps[np.clip(cand - 1, 0, max(len(lcps) - 1, 0))] if len(lcps) else np.zeros_like(cand)
            score = lcp_at * (b + 1) + np.abs(cand - ideal)
            cut = int(cand[np.argmin(score)])
        cuts.append(max(cut, cuts[-1]))
    cuts.append(b)
    shards = []
    for r in range(world):
        ids = np.sort(order[cuts[r]:cuts[r + 1]])
        sb = sub_batch(batch, ids)
        rows = 0
        if ids.size:
            seg = order[cuts[r]:cuts[r + 1]]
            seg_lens = np.diff(batch.cu_seqlens)[seg]
            inner = lcps[cuts[r]:cuts[r + 1] - 1] if seg.size > 1 else np.zeros(0, np.int64)
            rows = int(seg_lens.sum() - inner.sum())
        shards.append(Shard(r, ids, sb, rows))
    return shards


def gather_scores(local_scores, seq_ids, total_seqs: int, group=None):
    """All-gather per-sequence scores (the only collective) and restore batch order."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    counts = torch.tensor([local_scores.shape[0]], device=local_scores.device, dtype=torch.int64)
    all_counts = [torch.zeros_like(counts) for _ in range(world)]
    dist.all_gather(all_counts, counts, group=group)
    cmax = int(max(int(c.item()) for c in all_counts))
    pad = torch.zeros(cmax, dtype=local_scores.dtype, device=local_scores.device)
    pad[: local_scores.shape[0]] = local_scores
    ids = torch.full((cmax,), -1, dtype=torch.int64, device=local_scores.device)
    ids[: local_scores.shape[0]] = torch.as_tensor(np.asarray(seq_ids), device=local_scores.device)
    bufs = [torch.empty_like(pad) for _ in range(world)]
    idbufs = [torch.empty_like(ids) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    dist.all_gather(idbufs, ids, group=group)
    vals, idx = torch.cat(bufs), torch.cat(idbufs)
    out = torch.zeros(total_seqs, dtype=local_scores.dtype, device=local_scores.device)
    keep = idx >= 0
    out[idx[keep]] = vals[keep]
    return out
