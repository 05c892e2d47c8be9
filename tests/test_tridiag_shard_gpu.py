"""Row-sharded tridiagonal path (pfx_expm_tridiag_shard): 2-4 ranks under torchrun (gloo
all-gathers, every rank on the one visible GPU) reproduce the unsharded call to rounding and
the oracle to the north-star 1e-10; the rank row spans tile [0, N)."""
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


@pytest.mark.parametrize("N,nrhs,n,ranks,shift", [
    (4096, 4, 24, 2, 0.0),      # C2 recipe, several chunks per rank
    (1 << 16, 16, 24, 4, 0.0),  # C2 recipe at 2^16 rows
    (20000, 17, 16, 3, 0.0),    # two RHS tiles, ragged chunk split
    (257, 3, 20, 2, 0.5),       # random SPD-negative tridiagonal, shifted (e^c on the rank's rows)
    (40, 2, 12, 4, 0.0),        # fewer chunks than ranks: some ranks own no rows
])
def test_row_shard(N, nrhs, n, ranks, shift):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(ranks),
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tests", "shard_worker.py"),
           str(N), str(nrhs), str(n), str(shift)]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    spans = sorted(tuple(s) for s in d["spans"])
    assert spans[0][0] == 0 and spans[-1][1] == N
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert d["vs_unsharded"] <= 1e-12, d
    assert d["vs_oracle"] <= 1e-10, d
