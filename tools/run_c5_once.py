"""C5 (or a smaller grid) once on cuda:0 through the device entry (profiling helper)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_16778_b200 import _native, workloads as W
from paper_2306_16778_b200.roots import default_table
m = int(sys.argv[1]) if len(sys.argv) > 1 else 512
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda:0")
band = W.c5_band(m); V = W.c5_rhs(m, 8)
t2, c2 = default_table(16).interleaved()
B, Vd = torch.from_numpy(band).to(dev), torch.from_numpy(V).to(dev)
for _ in range(reps):
    out = _native.expm_banded_device(B, Vd, t2, c2, 0.0)
torch.cuda.synchronize()
print("ok", out.shape)
