"""Pinned host <-> device copy bandwidth (134 MB, the size of C2's V / out)."""
import time
import torch
n = 16 << 20
h = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def bw(fn, reps=10):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps
t_h2d = bw(lambda: d.copy_(h, non_blocking=True))
t_d2h = bw(lambda: h.copy_(d, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
t_both = bw(both)
GB = n * 8 / 1e9
print(f"H2D {GB / t_h2d:.1f} GB/s ({t_h2d*1e3:.2f} ms)  D2H {GB / t_d2h:.1f} GB/s ({t_d2h*1e3:.2f} ms)  "
      f"concurrent {2 * GB / t_both:.1f} GB/s total ({t_both*1e3:.2f} ms)")
