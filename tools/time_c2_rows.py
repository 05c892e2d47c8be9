"""Expected row-sharded C2 scaling on one GPU: time one rank's share of an eval (its chunk
range, both scan exchanges) for 1/2/4/8 ranks.  The all-gather is a local stand-in (every
rank's block = this rank's), so the numbers are right and the results are not; the real
collective adds two small all-gathers (~KB) per eval."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2306_16778_b200 import _native, workloads as W  # noqa: E402
from paper_2306_16778_b200.roots import default_table  # noqa: E402

dev = torch.device("cuda:0")
d, o = W.c2_matrix()
V = W.c2_rhs()
t2, c2 = default_table(24).interleaved()
D, O, Vd = (torch.from_numpy(x).to(dev) for x in (d, o, V))
out = torch.zeros_like(Vd)
for R in (1, 2, 4, 8):
    for r in sorted({0, R // 2}):
        ag = (lambda R_: (lambda mine: np.tile(mine, R_)))(R)
        for _ in range(3):
            _native.expm_tridiag_shard(D, O, Vd, t2, c2, 0.0, r, R, ag, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        t0 = time.perf_counter()
        e0.record()
        for _ in range(reps):
            _native.expm_tridiag_shard(D, O, Vd, t2, c2, 0.0, r, R, ag, out=out)
        e1.record()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / reps * 1e3
        r0, r1 = _native.tridiag_shard_rows(1 << 20, 16, r, R)
        print(f"ranks={R} rank={r} rows={r1 - r0} device_ms={e0.elapsed_time(e1) / reps:.3f} wall_ms={wall:.3f}")
if len(sys.argv) > 1:  # kernel breakdown of one rank's share at R ranks
    R = int(sys.argv[1])
    ag = lambda mine: np.tile(mine, R)  # noqa: E731
    _native.prof_enable(True)
    _native.prof_read()
    for _ in range(5):
        _native.expm_tridiag_shard(D, O, Vd, t2, c2, 0.0, 0, R, ag, out=out)
    torch.cuda.synchronize()
    for k, (cnt, ms, _) in _native.prof_read().items():
        print(f"R={R} {k:24s} launches={cnt // 5} ms_per_eval={ms / 5:.4f}")
    _native.prof_enable(False)
