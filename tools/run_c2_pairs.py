"""C2 with the first np pole pairs on cuda:0 (device mode), for profiling sharded ranks."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_16778_b200 import _native, workloads as W
from paper_2306_16778_b200.roots import default_table
from paper_2306_16778_b200.sharding import slice_poles
npr = int(sys.argv[1]) if len(sys.argv) > 1 else 1
d, o = W.c2_matrix(); V = W.c2_rhs()
dev = torch.device("cuda:0")
Dd, Od, Vd = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (d, o, V))
a, b = slice_poles(*default_table(24).interleaved(), 0, npr)
for _ in range(2):
    _native.expm_tridiag_device(Dd, Od, Vd, a, b, 0.0)
torch.cuda.synchronize()
print("ok")
