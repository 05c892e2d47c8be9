"""Golden fixtures for the banded config C5 at its real size — generated here (build container,
8 vCPUs, OpenBLAS) by the CPU oracle restatement, committed, and read by
tests/test_configs_gpu.py on the GPU box (where the zgbsv restatement of a whole C5 eval would
cost minutes of host time per test run).

    python tests/golden/make_config_fixtures.py [c5_rect] [c5_full]

The reference has no banded path; the restatement
oracle/restate.py::banded_action follows engine.py:194-201,226-228 (default_table pairs,
2 Re(a y), ascending reduction) with LAPACK zgbsv (kl = ku = kb) as the per-pair solve.

Outputs (rows sampled to keep the files small; the full-result Frobenius norm is stored
so the test can bound the relative error of the whole block):
  c5_rect_512x64.npz   C5 recipe on a 512 x 64 grid (N = 32,768, kb = 512 = C5's bandwidth)
  c5_full.npz          C5 itself (512 x 512 grid, N = 262,144, kb = 512, 8 RHS, n = 16)
each holding rows (sorted sample), value[rows] (R_n(A) V from the restatement),
oracle[rows] (DST-I closed form of exp(A) V), fro (||R_n(A) V||_F of the whole block),
err_ref (||R_n(A)V - exp(A)V||_F of the restatement, for P2).
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

from oracle import closed, restate  # noqa: E402
from paper_2306_16778_b200 import workloads as W  # noqa: E402


def sample_rows(N: int, edge: int, stride: int) -> np.ndarray:
    rows = set(range(min(edge, N))) | set(range(max(0, N - edge), N)) | set(range(0, N, stride))
    return np.array(sorted(rows), dtype=np.int64)


def make(name: str, nx: int, ny: int, edge: int, stride: int) -> None:
    n, s = W.C5["n"], W.C5["scale"]
    band = W.c5_band_rect(nx, ny, s)
    N = nx * ny
    V = np.random.default_rng([0, 0, 1]).standard_normal((N, W.C5["nrhs"]))
    t0 = time.time()
    Y = restate.banded_action(band, V, n)
    t1 = time.time()
    E = closed.dst_exp_lap2d(nx, s, V, ny)
    rows = sample_rows(N, edge, stride)
    np.savez_compressed(
        os.path.join(HERE, f"{name}.npz"), rows=rows, value=Y[rows], oracle=E[rows],
        fro=np.linalg.norm(Y), err_ref=np.linalg.norm(Y - E), nx=nx, ny=ny, n=n, scale=s,
    )
    print(f"{name}: N={N} restatement {t1 - t0:.1f} s, rows kept {rows.size}, "
          f"||Y||_F={np.linalg.norm(Y):.6e}, ||Y-E||_F/||E||_F={np.linalg.norm(Y - E) / np.linalg.norm(E):.3e}")


if __name__ == "__main__":
    which = sys.argv[1:] or ["c5_rect", "c5_full"]
    if "c5_rect" in which:
        make("c5_rect_512x64", 512, 64, edge=1024, stride=32)
    if "c5_full" in which:
        make("c5_full", 512, 512, edge=1024, stride=128)
