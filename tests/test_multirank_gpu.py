"""The N > 1 path on real kernels: several ranks (one process each, torch.distributed.run)
share the single GPU of the test box and use gloo for the only collective (the score
all-gather; NCCL refuses two ranks on one device).  Sharded scores equal one
single-process pass bit for bit (GEMMs are batch invariant and attention sees the same
K/V rows), and bench.py --gpus 2 runs end to end through its own launcher."""

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_scores_match_single_pass(world, tmp_path):
    out = str(tmp_path / "res.json")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                        "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
                        os.path.join(ROOT, "tests", "_multirank_worker.py"), out],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    res = json.load(open(out))
    for name, v in res.items():
        assert v["bit_identical"], (name, v)
        assert len(v["shards"]) == world


def test_bench_two_ranks_one_gpu():
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--share-gpu", "--steps", "3", "--warmup", "3",
                        "--no-cpu"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "weak"
    assert line["config"]["global_batch"] == 128 and len(line["shards"]) == 2
    assert line["parity"]["ok"] and line["value"] > 0 and line["e2e"]["value"] > 0
