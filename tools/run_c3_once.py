"""One C3 batch (or a prefix of it) on cuda:0 through the device entry (profiling helper)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_16778_b200 import _native, workloads as W
from paper_2306_16778_b200.roots import default_table
batch = int(sys.argv[1]) if len(sys.argv) > 1 else 148
dev = torch.device("cuda:0")
A = np.stack([W.c3_matrix(b) for b in range(batch)]); V = np.stack([W.c3_vector(b) for b in range(batch)])
t2, c2 = default_table(20).interleaved()
Ad, Vd = torch.from_numpy(A).to(dev), torch.from_numpy(V).to(dev)
for _ in range(2):
    out = _native.expm_dense_device(Ad, Vd, t2, c2, 0.0)
torch.cuda.synchronize()
print("ok", out.shape)
