"""Plan wire formats (reference: pkg/src/radix_compact/trie.py:238-314).

JSON ``{gather, scatter, compact_positions, n_original, n_compact}`` and the
RDXP binary layout: magic ``RDXP``, ``<HQQ`` (version, N, N'), then u32
gather[N'], compact_positions[N'], scatter[N], little endian.  Padding is a
runtime transform and is not serialised.  Byte-identical to the reference
writer (tests/test_serialization.py checks against golden files).
"""

from __future__ import annotations

import json
import struct

import numpy as np

from .plan import CompactionPlan

MAGIC = b"RDXP"
VERSION = 1
_HEAD = struct.Struct("<HQQ")


def plan_to_json(plan: CompactionPlan) -> dict:
    return {
        "gather": plan.gather_indices.tolist(),
        "scatter": plan.scatter_indices.tolist(),
        "compact_positions": plan.compact_positions.tolist(),
        "n_original": plan.n_original,
        "n_compact": plan.n_compact,
    }


def plan_from_json(obj: dict) -> CompactionPlan:
    return CompactionPlan(
        gather_indices=np.asarray(obj["gather"], dtype=np.uint32),
        scatter_indices=np.asarray(obj["scatter"], dtype=np.uint32),
        compact_positions=np.asarray(obj["compact_positions"], dtype=np.uint32),
        n_original=int(obj["n_original"]),
        n_compact=int(obj["n_compact"]),
    )


def plan_to_bytes(plan: CompactionPlan) -> bytes:
    m = plan.n_compact
    parts = [
        MAGIC,
        _HEAD.pack(VERSION, plan.n_original, m),
        plan.gather_indices[:m].astype("<u4").tobytes(),
        plan.compact_positions[:m].astype("<u4").tobytes(),
        plan.scatter_indices.astype("<u4").tobytes(),
    ]
    return b"".join(parts)


def plan_from_bytes(data: bytes) -> CompactionPlan:
    if data[:4] != MAGIC:
        raise ValueError("bad magic, not a plan file")
    version, n, m = _HEAD.unpack_from(data, 4)
    if version != VERSION:
        raise ValueError(f"unsupported plan version {version}")
    off = 4 + _HEAD.size
    arrays = []
    for count in (m, m, n):
        arrays.append(np.frombuffer(data, dtype="<u4", count=count, offset=off))
        off += 4 * count
    gather, cpos, scatter = arrays
    return CompactionPlan(gather, scatter, cpos, int(n), int(m))


def save_plan(plan: CompactionPlan, path, binary: bool = False) -> None:
    if binary:
        with open(path, "wb") as f:
            f.write(plan_to_bytes(plan))
    else:
        with open(path, "w") as f:
            json.dump(plan_to_json(plan), f)


def load_plan(path) -> CompactionPlan:
    with open(path, "rb") as f:
        data = f.read()
    if data[:4] == MAGIC:
        return plan_from_bytes(data)
    return plan_from_json(json.loads(data.decode()))
