"""Per-call wall time of C1 through the device and host entries (host-overhead check)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_16778_b200 import _native, workloads as W
from paper_2306_16778_b200.roots import default_table
A, v, _ = W.c1_inputs()
t2, c2 = default_table(16).interleaved()
Ad, vd = torch.from_numpy(A).cuda(), torch.from_numpy(v).cuda()
s = torch.cuda.Stream()
def bench(name, fn, n=200):
    for _ in range(10): fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize()
    print(f"{name:40s} {(time.perf_counter() - t) / n * 1e6:8.1f} us/call")
bench("device, default stream", lambda: _native.expm_dense_device(Ad, vd, t2, c2, 0.0))
bench("device, side stream", lambda: _native.expm_dense_device(Ad, vd, t2, c2, 0.0, stream=s))
out = torch.empty(128, dtype=torch.float64, device="cuda")
bench("device, side stream, out=", lambda: _native.expm_dense_device(Ad, vd, t2, c2, 0.0, stream=s, out=out))
bench("host", lambda: _native.expm_dense_host(A, v, t2, c2, 0.0))
bench("torch sync only", lambda: torch.cuda.current_stream().synchronize())
