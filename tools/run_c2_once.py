"""One C2 evaluation on cuda:0 through the device entry (profiling helper)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_16778_b200 import _native, workloads as W
from paper_2306_16778_b200.roots import default_table
dev = torch.device("cuda:0")
d, o = W.c2_matrix(); V = W.c2_rhs()
t2, c2 = default_table(24).interleaved()
D, O, Vd = (torch.from_numpy(x).to(dev) for x in (d, o, V))
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for _ in range(reps):
    out = _native.expm_tridiag_device(D, O, Vd, t2, c2, 0.0)
torch.cuda.synchronize()
print("ok", float(out[0, 0]))
