"""C4 (or a smaller d) once on cuda:0 through the device entry (profiling helper)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_16778_b200 import _native, workloads as W
from paper_2306_16778_b200.roots import default_table
d = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
A, _ = W.c4_matrix(d)
t2, c2 = default_table(24).interleaved()
Ad = torch.from_numpy(A).cuda()
for _ in range(reps):
    out = _native.expm_dense_device(Ad, None, t2, c2, 0.0)
torch.cuda.synchronize()
print("ok", out.shape)
