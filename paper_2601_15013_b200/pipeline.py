"""Pipelined scheduling of a stream of batches.

Reference: pkg/src/radix_compact/bench.py:346-405 (``pipelined_run``) and the
paper's pipelining note: the index build of batch t+1 runs
while batch t is computed, so the planner's latency leaves the critical path.

Two forms:

* ``pipelined_run(batches, worker, plan_builder, queue_capacity)`` keeps the
  reference's contract (same name, arguments, ``PipelineReport`` fields,
  ``WorkerPanic`` on a worker failure, producer errors re-raised, results
  identical to sequential construction).  The producer thread calls the GPU
  planner.
* ``score_stream(reranker, batches)`` is the B200-native form used by the
  serving path: batch t+1's pinned-host -> HBM copy and GPU plan build run on
  a side CUDA stream while batch t's prefill (CUDA-graph replay) runs on the
  main stream; only the planner's 4-word info read and the B scores cross
  back to the host.
"""

from __future__ import annotations

import queue
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from .errors import WorkerPanic
from .plan import build_plan


@dataclass
class PipelineReport:
    """Same fields as the reference's report (bench.py:326-341)."""

    total_s: float
    build_s: list = field(default_factory=list)
    compute_s: list = field(default_factory=list)
    tokens: int = 0
    hidden_fraction: float = 0.0

    @property
    def tokens_per_s(self) -> float:
        return self.tokens / self.total_s if self.total_s else float("inf")


_SENTINEL = object()


def pipelined_run(batches, worker, plan_builder=build_plan, queue_capacity: int = 2) -> PipelineReport:
    """Producer thread builds plan t+1 while ``worker(batch, plan)`` consumes batch t."""
    batches = list(batches)
    handoff: queue.Queue = queue.Queue(maxsize=max(1, queue_capacity))
    build_times: list[float] = []
    producer_error: list[BaseException] = []

    def produce():
        try:
            for idx, batch in enumerate(batches):
                t0 = time.perf_counter()
                plan = plan_builder(batch)
                build_times.append(time.perf_counter() - t0)
                handoff.put((idx, batch, plan))
        except BaseException as exc:  # surfaced on the consumer side
            producer_error.append(exc)
        finally:
            handoff.put(_SENTINEL)

    compute_times = []
    start = time.perf_counter()
    thread = threading.Thread(target=produce, daemon=True)
    thread.start()
    while True:
        item = handoff.get()
        if item is _SENTINEL:
            break
        idx, batch, plan = item
        t0 = time.perf_counter()
        try:
            worker(batch, plan)
        except Exception as exc:
            while handoff.get() is not _SENTINEL:  # let the producer finish
                pass
            thread.join()
            raise WorkerPanic(idx, str(exc)) from exc
        compute_times.append(time.perf_counter() - t0)
    thread.join()
    if producer_error:
        raise producer_error[0]
    total = time.perf_counter() - start
    sequential = sum(build_times) + sum(compute_times)
    hidden = max(0.0, sequential - total)
    denom = sum(build_times)
    return PipelineReport(total_s=total, build_s=build_times, compute_s=compute_times,
                          tokens=sum(b.num_tokens for b in batches),
                          hidden_fraction=min(1.0, hidden / denom) if denom > 0 else 0.0)


def score_stream(reranker, batches):
    """Scores of every batch (host numpy arrays, in order), with batch t+1's upload
    and plan build on a side stream overlapping batch t's prefill.  Results are
    bit-identical to calling ``reranker.score`` on each batch in turn."""
    import torch

    from . import _native
    from .ragged import validate_batch

    batches = list(batches)
    if not batches:
        return []
    main = torch.cuda.current_stream()
    side = getattr(reranker, "_side_stream", None)
    if side is None:
        side = reranker._side_stream = torch.cuda.Stream()

    def prepare(batch, slot):
        validate_batch(batch)
        with torch.cuda.stream(side):
            db = reranker.upload(batch, slot=slot)
            plan = reranker.plan(db)  # blocks only on the side stream's 4-word info read
        ready = torch.cuda.Event()
        ready.record(side)
        return db, plan, ready

    results = [None] * len(batches)
    pending = None  # (index, pinned buffer, event) of the batch whose scores are still in flight
    nxt = prepare(batches[0], 0)
    for t in range(len(batches)):
        db, plan, ready = nxt
        main.wait_event(ready)
        for x in (db.tok, db.pos, db.cu, db.cu32):
            x.record_stream(main)
        if plan is not None:
            for x in (plan.gather, plan.scatter, plan.compact_positions, plan.cu_q):
                x.record_stream(main)
        scores = reranker.score_device(db, plan=plan)
        b = scores.shape[0]
        buf = reranker._pinned.get(f"scores{t & 1}", b, torch.float32)  # grow-only, reused across calls
        buf.copy_(scores, non_blocking=True)
        done = torch.cuda.Event()
        done.record(main)
        if t + 1 < len(batches):
            nxt = prepare(batches[t + 1], (t + 1) & 1)  # overlaps the prefill of batch t
        # collect batch t-1 only now: batch t's prefill is already queued behind it, so the
        # GPU never idles on the host's read-back (slot (t-1)&1 is reused by batch t+1)
        if pending is not None:
            pt, pbuf, pdone = pending
            pdone.synchronize()
            results[pt] = np.array(pbuf.numpy(), copy=True)
        pending = (t, buf, done)
    pt, pbuf, pdone = pending
    pdone.synchronize()
    results[pt] = np.array(pbuf.numpy(), copy=True)
    _native.check_device_status(main)  # once per stream: an overlapped-norm wait that timed out
    return results
