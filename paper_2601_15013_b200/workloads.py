"""Synthetic ragged batches for parity tests and benchmarks.

``make_synthetic_batch`` / ``make_pattern_batch`` reproduce the reference
generators draw-for-draw (pkg/src/radix_compact/bench.py:24-144; pinned by
tests/golden/synthetic.npz).  ``msmarco_rerank_batch`` and
``long_prefix_batch`` are the BASELINE.json workloads:

  C2/C3  MS-MARCO-shaped reranking: a shared prefix (reranker system /
         instruction template + query), one passage per sequence with
         length ~ U[passage_min, passage_max], and a fixed template tail that
         follows the passage (never shareable: its history differs).
  C4     long shared prefix: SyntheticSpec(B=128, prefix_len=2048,
         suffix_len=256, vocab=151936).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

from .errors import VocabTooSmall
from .ragged import RaggedBatch, default_positions


@dataclass(frozen=True)
class SyntheticSpec:
    """B sequences sharing a P-token prefix with S-token unique suffixes (bench.py:24-41)."""

    B: int
    prefix_len: int
    suffix_len: int
    vocab: int = 1024
    seed: int = 0

    def __post_init__(self):
        if self.B < 1 or self.prefix_len + self.suffix_len < 1:
            raise ValueError("need B >= 1 and at least one token per sequence")

    @property
    def label(self) -> str:
        return f"B{self.B}_P{self.prefix_len}_S{self.suffix_len}"


def make_synthetic_batch(spec: SyntheticSpec) -> RaggedBatch:
    """Shared prefix, suffixes forced to diverge at their first token, so N' = P + B*S."""
    b, p, s = spec.B, spec.prefix_len, spec.suffix_len
    if s > 0 and spec.vocab < b:
        raise VocabTooSmall(f"vocab {spec.vocab} < batch size {b}")
    rng = np.random.default_rng(spec.seed)
    prefix = rng.integers(0, spec.vocab, size=p, dtype=np.uint32)
    rows = np.empty((b, p + s), dtype=np.uint32)
    rows[:, :p] = prefix
    if s > 0:
        rows[:, p:] = rng.integers(0, spec.vocab, size=(b, s), dtype=np.uint32)
        rows[:, p] = rng.permutation(spec.vocab)[:b]
    cu = np.arange(b + 1, dtype=np.int64) * (p + s)
    return RaggedBatch(rows.reshape(-1), default_positions(cu), cu)


class Pattern(Enum):
    SINGLE_SEQUENCE = "single_sequence"
    IDENTICAL_SEQUENCES = "identical_sequences"
    SHARED_PREFIX = "shared_prefix"
    NO_SHARING = "no_sharing"
    MIXED_LENGTHS = "mixed_lengths"
    COMPLEX_SHARING = "complex_sharing"


def make_pattern_batch(pattern: Pattern, seed: int = 0, vocab: int = 97) -> RaggedBatch:
    """The six Appendix-C sharing patterns (bench.py:85-144), same draws."""
    rng = np.random.default_rng((seed, list(Pattern).index(pattern)))

    def distinct(k):
        return rng.permutation(vocab)[:k].astype(np.uint32)

    def draw(k):
        return rng.integers(0, vocab, size=k, dtype=np.uint32)

    cat = np.concatenate
    if pattern is Pattern.SINGLE_SEQUENCE:
        seqs = [draw(5)]
    elif pattern is Pattern.IDENTICAL_SEQUENCES:
        one = draw(5)
        seqs = [one, one.copy()]
    elif pattern is Pattern.SHARED_PREFIX:
        shared, tails = draw(3), distinct(2)
        seqs = [cat([shared, [tails[0]], draw(1)]), cat([shared, [tails[1]], draw(1)])]
    elif pattern is Pattern.NO_SHARING:
        heads = distinct(2)
        seqs = [cat([[heads[0]], draw(2)]), cat([[heads[1]], draw(2)])]
    elif pattern is Pattern.MIXED_LENGTHS:
        a, forks, deeper = draw(1), distinct(2), distinct(2)
        seqs = [cat([a, [forks[0]]]), cat([a, [forks[1]], [deeper[0]]]),
                cat([a, [forks[1]], [deeper[1]], draw(2)])]
    else:  # COMPLEX_SHARING
        a, d1, d2, d3 = draw(1), distinct(2), distinct(2), distinct(2)
        seqs = [cat([a, [d1[0]], draw(3)]), cat([a, [d1[1]], [d2[0]], draw(2)]),
                cat([a, [d1[1]], [d2[1]], [d3[0]], draw(1)]),
                cat([a, [d1[1]], [d2[1]], [d3[1]], draw(1)])]
    tokens = cat(seqs).astype(np.uint32)
    cu = np.cumsum([0] + [len(x) for x in seqs]).astype(np.int64)
    return RaggedBatch(tokens, default_positions(cu), cu)


@dataclass(frozen=True)
class RerankSpec:
    """MS-MARCO-v1.1-shaped reranking batch (BASELINE.json configs[1], [2])."""

    queries: int = 1
    passages_per_query: int = 64
    template_len: int = 32     # reranker system + instruction template (shared by all)
    query_len: int = 32        # "~32-token query prefix"
    passage_min: int = 72
    passage_max: int = 120     # mean 96
    tail_len: int = 13         # "<|im_end|> ... assistant ... </think>" tail after the passage
    vocab: int = 151936
    seed: int = 0

    @property
    def label(self) -> str:
        return (f"rerank_q{self.queries}x{self.passages_per_query}_T{self.template_len}"
                f"_Q{self.query_len}_P{self.passage_min}-{self.passage_max}_tail{self.tail_len}")


def msmarco_rerank_batch(spec: RerankSpec = RerankSpec()) -> RaggedBatch:
    rng = np.random.default_rng(spec.seed)
    template = rng.integers(0, spec.vocab, size=spec.template_len, dtype=np.uint32)
    tail = rng.integers(0, spec.vocab, size=spec.tail_len, dtype=np.uint32)
    seqs = []
    for _ in range(spec.queries):
        query = rng.integers(0, spec.vocab, size=spec.query_len, dtype=np.uint32)
        for _ in range(spec.passages_per_query):
            plen = int(rng.integers(spec.passage_min, spec.passage_max + 1))
            passage = rng.integers(0, spec.vocab, size=plen, dtype=np.uint32)
            seqs.append(np.concatenate([template, query, passage, tail]))
    tokens = np.concatenate(seqs).astype(np.uint32)
    cu = np.cumsum([0] + [len(x) for x in seqs]).astype(np.int64)
    return RaggedBatch(tokens, default_positions(cu), cu)


def long_prefix_batch(B: int = 128, prefix_len: int = 2048, suffix_len: int = 256, vocab: int = 151936,
                      seed: int = 0) -> RaggedBatch:
    """C4: SyntheticSpec(B, 2048, 256, vocab 151936) -> N'=P+B*S exactly."""
    return make_synthetic_batch(SyntheticSpec(B=B, prefix_len=prefix_len, suffix_len=suffix_len,
                                              vocab=vocab, seed=seed))


def prefix_ratio_batch(n_tokens: int, ratio: float, seq_len: int = 512, vocab: int = 151936,
                       seed: int = 0) -> RaggedBatch:
    """C5 (Table 5 of the paper): n_tokens / seq_len sequences of
    seq_len tokens whose first round(ratio * seq_len) tokens are shared."""
    b = max(1, n_tokens // seq_len)
    p = int(round(ratio * seq_len))
    return make_synthetic_batch(SyntheticSpec(B=b, prefix_len=p, suffix_len=seq_len - p, vocab=vocab, seed=seed))


def multilevel_batch(n_tokens: int, levels=((64, 1), (64, 4), (128, 4)), leaf_len: int = 256,
                     vocab: int = 151936, seed: int = 0) -> RaggedBatch:
    """C5 multi-level trie: a tree whose level i has `fanout` children of `length`
    tokens each (each child diverges at its first token); every root-to-leaf
    path gets its own leaf_len-token unique tail.  Paths repeat the tree until
    n_tokens is reached (distinct trees per repetition)."""
    rng = np.random.default_rng(seed)
    seq_len = sum(length for length, _ in levels) + leaf_len
    seqs = []
    while sum(len(s) for s in seqs) + seq_len <= max(n_tokens, seq_len):
        paths = [np.zeros(0, dtype=np.uint32)]
        for length, fanout in levels:
            nxt = []
            for pth in paths:
                firsts = rng.permutation(vocab)[:fanout]
                for f in firsts:
                    seg = rng.integers(0, vocab, size=length, dtype=np.uint32)
                    seg[0] = f
                    nxt.append(np.concatenate([pth, seg]))
            paths = nxt
        for pth in paths:
            seqs.append(np.concatenate([pth, rng.integers(0, vocab, size=leaf_len, dtype=np.uint32)]))
            if sum(len(s) for s in seqs) + seq_len > max(n_tokens, seq_len):
                break
    tokens = np.concatenate(seqs).astype(np.uint32)
    cu = np.cumsum([0] + [len(x) for x in seqs]).astype(np.int64)
    return RaggedBatch(tokens, default_positions(cu), cu)
