"""Kernel breakdown of one rank's column-split share of C4 (8 ranks: one whole pair + part of a
shared pair): per-kernel launch counts and device time from the library's profiling events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2306_16778_b200 import _native, workloads as W  # noqa: E402
from paper_2306_16778_b200.roots import default_table  # noqa: E402
from paper_2306_16778_b200.sharding import colsplit_plan  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 8
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 0
dev = torch.device("cuda:0")
A, _ = W.c4_matrix()
t2, c2 = default_table(24).interleaved()
Ad = torch.from_numpy(A).to(dev)
tasks = colsplit_plan(12, A.shape[0], rank, R)
idx = [k for k, _, _ in tasks]
th = np.concatenate([t2[2 * k: 2 * k + 2] for k in idx])
co = np.concatenate([c2[2 * k: 2 * k + 2] for k in idx])
rg = [(a, b) for _, a, b in tasks]
out = None
for _ in range(2):
    out = _native.expm_dense_cols_device(Ad, th, co, rg, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    _native.expm_dense_cols_device(Ad, th, co, rg, out=out)
e1.record()
torch.cuda.synchronize()
print(f"ranks={R} rank={rank} tasks={tasks}: {e0.elapsed_time(e1) / 3:.2f} ms")
_native.prof_enable(True)
_native.prof_read()
_native.expm_dense_cols_device(Ad, th, co, rg, out=out)
torch.cuda.synchronize()
k = _native.prof_read()
_native.prof_enable(False)
for name, (c, t, f) in sorted(k.items(), key=lambda kv: -kv[1][1]):
    print(f"  {name:28s} {c:5d} launches {t:8.2f} ms  {f / t / 1e9 if t else 0:8.1f} TF/s")
print(f"  total (sum of launches) {sum(v[1] for v in k.values()):.2f} ms")
