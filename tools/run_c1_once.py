"""C1 once on cuda:0 through the device entry (profiling helper; PFX_DENSE_PHASES=1 prints phases)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_16778_b200 import _native, workloads as W
from paper_2306_16778_b200.roots import default_table
A, v, _ = W.c1_inputs()
t2, c2 = default_table(16).interleaved()
Ad, vd = torch.from_numpy(A).cuda(), torch.from_numpy(v).cuda()
for _ in range(3):
    _native.expm_dense_device(Ad, vd, t2, c2, 0.0)
torch.cuda.synchronize()
