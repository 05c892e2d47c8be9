"""Wall time of C2 through the host entry (pinned buffers), as bench.py's e2e leg."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_16778_b200 import _native, workloads as W
from paper_2306_16778_b200.roots import default_table
d, o = W.c2_matrix(); V = W.c2_rhs()
t2, c2 = default_table(24).interleaved()
pd, po, pv = (torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in (d, o, V))
out = torch.empty(V.size, dtype=torch.float64).pin_memory()
for _ in range(3):
    _native.expm_tridiag_host(pd.numpy(), po.numpy(), pv.numpy(), t2, c2, 0.0, out=out.numpy())
for rep in range(3):
    t = time.perf_counter()
    for _ in range(10):
        _native.expm_tridiag_host(pd.numpy(), po.numpy(), pv.numpy(), t2, c2, 0.0, out=out.numpy())
    print(f"host-entry C2: {(time.perf_counter() - t) / 10 * 1e3:.2f} ms/eval")
if "--check" in sys.argv:
    from oracle import restate  # parity of the pipelined host path at full size (slow: CPU oracle on 2 columns)
    dev = torch.device("cuda:0")
    full = _native.expm_tridiag_device(*(torch.from_numpy(x).to(dev) for x in (d, o, V)), t2, c2, 0.0).cpu().numpy()
    got = out.numpy().reshape(V.shape)
    print("host vs device rel", np.linalg.norm(got - full) / np.linalg.norm(full))
