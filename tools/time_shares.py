"""Expected multi-GPU scaling on one B200: the device time of ONE rank's share of an eval for
1/2/4/8 ranks, per config and sharding mode (bench.py --shard): pole shards (the largest
rank's contiguous block of pairs), batch shards (C3: batch / R matrices).  The collective
that joins the shares is not included (pole: one reduce of the output; batch: none)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2306_16778_b200 import _native, workloads as W  # noqa: E402
from paper_2306_16778_b200.roots import default_table  # noqa: E402

dev = torch.device("cuda:0")


def timeit(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def largest_block(npairs, R):
    return max((r + 1) * npairs // R - r * npairs // R for r in range(R))


which = sys.argv[1:] or ["C3", "C4", "C5"]
if "C3" in which:
    A, V = W.c3_batch()
    t2, c2 = default_table(20).interleaved()
    Ad, Vd = torch.from_numpy(A).to(dev), torch.from_numpy(V).to(dev)
    for R in (1, 2, 4, 8):
        nb = 512 // R
        ms = timeit(lambda: _native.expm_dense_device(Ad[:nb], Vd[:nb], t2, c2, 0.0), 3)
        npr = largest_block(10, R)
        msp = timeit(lambda: _native.expm_dense_device(Ad, Vd, t2[:2 * npr], c2[:2 * npr], 0.0), 3)
        print(f"C3 ranks={R} batch-shard {ms:.2f} ms  pole-shard ({npr} pairs) {msp:.2f} ms", flush=True)
if "C4" in which:
    A, _ = W.c4_matrix()
    t2, c2 = default_table(24).interleaved()
    Ad = torch.from_numpy(A).to(dev)
    for R in (1, 2, 4, 8, 5):
        npr = largest_block(12, R)
        ms = timeit(lambda: _native.expm_dense_device(Ad, None, t2[:2 * npr], c2[:2 * npr], 0.0), 1)
        line = f"C4 ranks={R} pole-shard ({npr} pairs) {ms:.1f} ms"
        if 12 % R:
            # leftover pairs split by inverse columns (sharding.colsplit_plan): every rank's share
            from paper_2306_16778_b200.sharding import colsplit_plan

            worst = 0.0
            for r in range(R):
                tasks = colsplit_plan(12, A.shape[0], r, R)
                idx = [k for k, _, _ in tasks]
                th = np.concatenate([t2[2 * k: 2 * k + 2] for k in idx])
                co = np.concatenate([c2[2 * k: 2 * k + 2] for k in idx])
                rg = [(a, b) for _, a, b in tasks]
                t = timeit(lambda: _native.expm_dense_cols_device(Ad, th, co, rg), 1)
                worst = max(worst, t)
                line += f"\n   colsplit rank {r}: {tasks} {t:.1f} ms"
            line += f"\n   colsplit worst rank {worst:.1f} ms"
        print(line, flush=True)
if "C5" in which:
    band, V = W.c5_band(), W.c5_rhs()
    t2, c2 = default_table(16).interleaved()
    B, Vd = torch.from_numpy(band).to(dev), torch.from_numpy(V).to(dev)
    for R in (1, 2, 4, 8):
        npr = largest_block(8, R)
        ms = timeit(lambda: _native.expm_banded_device(B, Vd, t2[:2 * npr], c2[:2 * npr], 0.0), 1)
        print(f"C5 ranks={R} pole-shard ({npr} pairs) {ms:.1f} ms", flush=True)
