"""ExpOptions(distributed=True) through the real library on gloo ranks sharing the one GPU:
pole sharding of the public API (reference engine.py:217-228, the n/2 pair fan-out and the
ascending reduction) and, for matexp_full on the blocked large path, the column split of the
leftover pairs."""
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


@pytest.mark.parametrize("d,n,cplx,ranks", [
    (640, 6, 1, 2),    # 3 pairs on 2 ranks: one whole pair each + half the columns of the third
    (704, 10, 1, 3),   # 5 pairs on 3 ranks
    (576, 6, 0, 2),    # real symmetric: the split path returns float64
    (200, 8, 1, 3),    # d <= 512: plain pole blocks on the batched kernel
])
def test_engine_distributed(d, n, cplx, ranks):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(ranks),
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "engine_dist_worker.py"), str(d), str(n), str(cplx)]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    r = json.loads(lines[0])
    assert r["full_vs_unsharded"] <= 1e-12, r
    assert r["full_vs_oracle"] <= 1e-10 and r["action_vs_oracle"] <= 1e-10, r
    assert r["times"] == n // 2 and r["t_para_ok"]
    assert r["dtype"] == ("complex128" if cplx else "float64")
