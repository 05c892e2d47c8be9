"""bench.py under torchrun with two ranks (gloo emulation on one GPU): the pole-, row- and
batch-sharded timed regions, the max-over-ranks timing, the N > 1 e2e leg and rank 0's
single JSON line."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("workload,shard,tag", [("C1", "pole", "pole-shard x2"), ("C2", "rows", "row-shard x2"),
                                               ("C2", "pole", "pole-shard x2"), ("C3", "batch", "batch-shard x2"),
                                               ("C3", "pole", "pole-shard x2")])
def test_two_rank_bench_line(workload, shard, tag):
    env = dict(os.environ, PFX_BENCH_GLOO="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--workload", workload, "--shard", shard, "--steps", "3", "--warmup", "3",
           "--e2e-steps", "2", "--check"]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["e2e"] is not None and d["e2e"]["value"] > 0
    assert tag in d["config"]["parallelism"]
    # parity: rank 0's part of the sharded result equals the unsharded computation (the pole
    # shards' partial sums meet in a different order, so to rounding, not bitwise)
    assert d["check_rel"] is not None and d["check_rel"] <= 1e-12, d["check_rel"]


def test_c4_colsplit_five_ranks():
    # 12 pairs on 5 ranks: two whole pairs per rank, the two leftover pairs split by inverse
    # columns (sharding.colsplit_plan); rank 0's reduced result equals the unsharded exp(A)
    env = dict(os.environ, PFX_BENCH_GLOO="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "5",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "5", "--workload", "C4", "--steps", "1", "--warmup", "3", "--e2e-steps", "1",
           "--prof-steps", "1", "--check"]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 5 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert "split by inverse columns" in d["config"]["parallelism"]
    assert d["check_rel"] is not None and d["check_rel"] <= 1e-12, d["check_rel"]
