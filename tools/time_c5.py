"""Device time of one C5 evaluation (after one warm-up), for PFX_BD_SKIP experiments."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_16778_b200 import _native, workloads as W
from paper_2306_16778_b200.roots import default_table
m = int(sys.argv[1]) if len(sys.argv) > 1 else 512
dev = torch.device("cuda:0")
band = W.c5_band(m); V = W.c5_rhs(m, 8)
t2, c2 = default_table(16).interleaved()
B, Vd = torch.from_numpy(band).to(dev), torch.from_numpy(V).to(dev)
_native.expm_banded_device(B, Vd, t2, c2, 0.0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(2):
    _native.expm_banded_device(B, Vd, t2, c2, 0.0)
e1.record(); torch.cuda.synchronize()
print(f"skip={os.environ.get('PFX_BD_SKIP', '0'):>3s}  {e0.elapsed_time(e1) / 2:8.1f} ms")
