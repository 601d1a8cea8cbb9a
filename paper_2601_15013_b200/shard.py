"""Multi-GPU partitioning by trie subtree.

RadixMLP is per-batch and stateless, so the batch shards into
independent sub-batches of whole sequences; each GPU builds the plan of its
own sub-batch (bit-exact to the reference's build_plan on that sub-batch)
and runs the full prefill on it.  No collective runs on the hot path; only
the per-sequence scores are all-gathered at the end.

Partition: sort sequences lexicographically by their (token, position) path
(trie DFS order), so every trie subtree is a contiguous run; then cut the
sorted order into ``world`` runs minimising the largest per-GPU compact-row
count (each run's plan recomputes the prefix it shares with the run before
it), ties broken by the fewest duplicated rows.  A cut at LCP 0 (distinct
root subtrees) duplicates nothing; when the root has a single child (a
common system prompt), cuts between different queries duplicate only the
prompt.
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


def partition_by_subtree(batch: RaggedBatch, world: int, window: float | None = None) -> list[Shard]:
    """Split ``batch`` into ``world`` shards of whole trie subtrees, minimising the makespan.

    Sequences are taken in trie order (every subtree contiguous) and cut into
    ``world`` contiguous runs.  A run's cost is the compact rows its own plan
    will have: sum of L - lcp(previous) inside the run, with the run's first
    sequence paying its full length (the shared trunk is recomputed on each
    GPU that holds part of it).  An exact DP over cut positions minimises the
    largest run cost (the step time of the slowest GPU), ties broken by the
    least duplicated prefix rows, so cuts land between root subtrees whenever
    that does not lengthen the slowest shard.  ``window`` is accepted for API
    compatibility and ignored.
    """
    del window
    if world < 1:
        raise ValueError("world must be >= 1")
    b = batch.num_sequences
    order, lcps = trie_order(batch)
    lens = np.diff(batch.cu_seqlens)[order].astype(np.int64)
    if b == 0:
        cuts = [0] * (world + 1)
    else:
        cuts = _makespan_cuts(lens, lcps.astype(np.int64), world)
    shards = []
    for r in range(world):
        seg = order[cuts[r]:cuts[r + 1]]
        ids = np.sort(seg)
        sb = sub_batch(batch, ids)
        rows = 0
        if seg.size:
            inner = lcps[cuts[r]:cuts[r + 1] - 1] if seg.size > 1 else np.zeros(0, np.int64)
            rows = int(lens[cuts[r]:cuts[r + 1]].sum() - inner.sum())
        shards.append(Shard(r, ids, sb, rows))
    return shards


def _makespan_cuts(lens: np.ndarray, lcps: np.ndarray, world: int) -> list[int]:
    """cuts[0]=0 < ... < cuts[world]=B (non-empty runs while B >= world) minimising
    (max run cost, total duplicated rows); run cost(i, j) = U[j] - U[i] + lcp_before(i)."""
    b = lens.shape[0]
    lcp_before = np.concatenate([[0], lcps])            # shared rows of sequence i with i-1
    unique = lens - lcp_before                          # rows sequence i adds in trie order
    U = np.concatenate([[0], np.cumsum(unique)]).astype(np.float64)
    big = float(U[-1] + lens.sum() + 1)                 # > any duplication total
    inf = np.inf
    g_max = min(world, b)
    # best[g][j]: lexicographic (makespan, dup) of splitting the first j sequences into g runs
    prev = np.full(b + 1, inf)
    prev[0] = 0.0
    choice = np.zeros((g_max + 1, b + 1), dtype=np.int64)
    for g in range(1, g_max + 1):
        cur = np.full(b + 1, inf)
        for j in range(g, b + 1):
            i = np.arange(g - 1, j)                     # last run = sequences [i, j)
            i = i[np.isfinite(prev[i])]
            cost = U[j] - U[i] + lcp_before[i]
            pm = np.floor(prev[i] / big)                # previous makespan
            pd = prev[i] - pm * big                     # previous duplication
            dup = pd + np.where(i > 0, lcp_before[i], 0)
            val = np.maximum(pm, cost) * big + dup
            k = int(np.argmin(val))
            cur[j] = val[k]
            choice[g, j] = i[k]
        prev = cur
    cuts = [b]
    j = b
    for g in range(g_max, 0, -1):
        j = int(choice[g, j])
        cuts.append(j)
    cuts = cuts[::-1]
    cuts += [b] * (world - g_max)                       # more ranks than sequences: empty shards
    return cuts


def gather_scores(local_scores, seq_ids, total_seqs: int, group=None):
    """All-gather per-sequence scores (the only collective) and restore batch order.

    NCCL gathers device tensors over NVLink; with the gloo backend (CPU tests,
    or several ranks sharing one GPU) the exchange goes through host tensors and
    the result comes back on ``local_scores``' device.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    home = local_scores.device
    dev = torch.device("cpu") if dist.get_backend(group) == "gloo" else home
    local_scores = local_scores.to(dev)
    counts = torch.tensor([local_scores.shape[0]], device=dev, dtype=torch.int64)
    all_counts = [torch.zeros_like(counts) for _ in range(world)]
    dist.all_gather(all_counts, counts, group=group)
    cmax = int(max(int(c.item()) for c in all_counts))
    pad = torch.zeros(cmax, dtype=local_scores.dtype, device=dev)
    pad[: local_scores.shape[0]] = local_scores
    ids = torch.full((cmax,), -1, dtype=torch.int64, device=dev)
    ids[: local_scores.shape[0]] = torch.as_tensor(np.asarray(seq_ids), device=dev)
    bufs = [torch.empty_like(pad) for _ in range(world)]
    idbufs = [torch.empty_like(ids) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    dist.all_gather(idbufs, ids, group=group)
    vals, idx = torch.cat(bufs), torch.cat(idbufs)
    out = torch.zeros(total_seqs, dtype=local_scores.dtype, device=dev)
    keep = idx >= 0
    out[idx[keep]] = vals[keep]
    return out.to(home)


def shard_report(shards, n_compact=None) -> list[dict]:
    """Per-rank workload summary: sequences, tokens N_g, compact rows N'_g, gamma_g.

    ``n_compact`` (optional, per shard) overrides the host estimate with the
    planner's exact N'_g; the two agree for plans of whole sequences.
    """
    out = []
    for i, s in enumerate(shards):
        m = int(s.est_compact_rows if n_compact is None else n_compact[i])
        n = int(s.batch.num_tokens)
        out.append({"rank": s.rank, "sequences": int(s.seq_ids.size), "N": n, "N_compact": m,
                    "gamma": round(m / n, 4) if n else 1.0})
    return out


def score_sharded(batch: RaggedBatch, scorer, group=None, shards=None):
    """Score ``batch`` across the ranks of ``group``: rank r scores shard r of the trie-subtree
    partition with ``scorer(sub_batch) -> tensor [B_r]`` and the scores are all-gathered back
    into the batch's sequence order.  Every rank returns the full [B] scores."""
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    shards = partition_by_subtree(batch, world) if shards is None else shards
    mine = shards[rank]
    return gather_scores(scorer(mine.batch), mine.seq_ids, batch.num_sequences, group=group)
