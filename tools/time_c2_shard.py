"""Device time of C2 with the first np pole pairs only: the per-rank work of pole sharding
at 1/2/4/8 GPUs (12/6/3/1-2 pairs)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_16778_b200 import _native, workloads as W
from paper_2306_16778_b200.roots import default_table
from paper_2306_16778_b200.sharding import slice_poles
d, o = W.c2_matrix(); V = W.c2_rhs()
dev = torch.device("cuda:0")
Dd, Od, Vd = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (d, o, V))
t2, c2 = default_table(24).interleaved()
for npr in (12, 6, 3, 2, 1):
    a, b = slice_poles(t2, c2, 0, npr)
    for _ in range(3):
        _native.expm_tridiag_device(Dd, Od, Vd, a, b, 0.0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        _native.expm_tridiag_device(Dd, Od, Vd, a, b, 0.0)
    e1.record(); torch.cuda.synchronize()
    print(f"pairs={npr:2d}  {e0.elapsed_time(e1) / 10:.3f} ms")
