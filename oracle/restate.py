"""CPU restatement of the reference hot path — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Every function follows /root/reference/pkg/src/pfexpm/engine.py:178-230 (`_run_tasks`):
  * poles/residues = default_table(n).thetas_f8()/coeffs_f8() at even indices
    (engine.py:180-182,196) — read here from the reference-generated golden
    fixture tests/golden/tables_f8.npz;
  * one shifted solve per conjugate pair (engine.py:197-213);
  * real path combine 2*Re(a*y) (engine.py:201,210), complex path
    a*y + conj(a)*yc with yc from the conjugate-transposed factorization
    (engine.py:202-206) or aX + (aX)^H (engine.py:211-213);
  * slots reduced in ascending pair order (engine.py:225-228).
The dense restatement uses the same numpy/scipy calls as the reference and so
reproduces it bit-for-bit (checked in tests/test_oracle.py).  The structured
restatements replace the dense solve by LAPACK zgtsv / zgbsv (partial
pivoting, the LAPACK analogue of np.linalg.solve).
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.linalg
import scipy.linalg.lapack as lapack

_GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "tables_f8.npz")
_TABLES = None


def pairs(n: int):
    """(theta, a) complex128 arrays of the n/2 representatives (roots.py:222-226, engine.py:196)."""
    global _TABLES
    if _TABLES is None:
        z = np.load(_GOLDEN)
        _TABLES = {k: z[k] for k in z.files}
    return _TABLES[f"theta_{n}"][0::2].copy(), _TABLES[f"coef_{n}"][0::2].copy()


def _reduce(slots):
    acc = slots[0]
    for s in slots[1:]:
        acc = acc + s
    return acc


def _pool_map(fn, count, threads):
    if threads <= 1:
        return [fn(i) for i in range(count)]
    with ThreadPoolExecutor(max_workers=threads) as pool:
        return list(pool.map(fn, range(count)))


def run_tasks_dense(A: np.ndarray, v, n: int, threads: int = 1):
    """Restatement of engine._run_tasks for a dense Hermitian A (engine.py:178-230)."""
    A = np.asarray(A, dtype=complex)
    theta, coef = pairs(n)
    d = A.shape[0]
    action = v is not None
    real_path = bool(np.all(A.imag == 0.0)) and (not action or bool(np.isrealobj(v)))
    if action:
        v = np.asarray(v, dtype=complex)

    def task(slot):
        a = coef[slot]
        M = A + theta[slot] * np.eye(d)
        if action:
            if real_path:
                y = np.linalg.solve(M, v)
                return 2.0 * (a * y).real
            lu = scipy.linalg.lu_factor(M, check_finite=False)
            y = scipy.linalg.lu_solve(lu, v, trans=0, check_finite=False)
            yc = scipy.linalg.lu_solve(lu, v, trans=2, check_finite=False)
            return a * y + np.conj(a) * yc
        X = np.linalg.solve(M, np.eye(d, dtype=complex))
        if real_path:
            return 2.0 * (a * X).real
        aX = a * X
        return aX + aX.conj().T

    return _reduce(_pool_map(task, len(theta), threads))


def resolve_shift(A: np.ndarray, shift, bounds=None) -> float:
    """engine._resolve_shift (engine.py:276-280): 'auto' -> alpha from exact bounds else Gershgorin hi."""
    if shift == "auto":
        if bounds is not None:
            return float(bounds[1])
        a = np.asarray(A)
        centers = np.real(np.diag(a))
        radii = np.sum(np.abs(a), axis=1) - np.abs(np.diag(a))
        return float(np.max(centers + radii))
    return float(shift)


def matexp_dense(A: np.ndarray, v, n: int, shift=None, bounds=None, threads: int = 1):
    """Value of matexp_full/matexp_action/matexp_shifted (engine.py:233-320)."""
    A = np.asarray(A, dtype=complex)
    if shift is None:
        return run_tasks_dense(A, v, n, threads)
    c = resolve_shift(A, shift, bounds)
    B = A - c * np.eye(A.shape[0])
    return math.exp(c) * run_tasks_dense(B, v, n, threads)


def tridiag_action(diag, off, V, n: int, threads: int = 1, cols=None):
    """R_n(T) V for real symmetric tridiagonal T via zgtsv per pair, 2Re(a y), ascending sum."""
    theta, coef = pairs(n)
    diag = np.asarray(diag, dtype=np.float64)
    off = np.asarray(off, dtype=np.float64).astype(complex)
    V = np.asarray(V, dtype=np.float64)
    if cols is not None:
        V = V[:, cols]
    squeeze = V.ndim == 1
    B = (V[:, None] if squeeze else V).astype(complex)

    def task(slot):
        if diag.shape[0] == 1:  # zgtsv wrapper rejects empty off-diagonals
            return 2.0 * (coef[slot] * (B / (diag[0] + theta[slot]))).real
        _, _, _, y, info = lapack.zgtsv(off, diag + theta[slot], off, B)
        if info != 0:
            raise np.linalg.LinAlgError(f"zgtsv info={info}")
        return 2.0 * (coef[slot] * y).real

    out = _reduce(_pool_map(task, len(theta), threads))
    return out[:, 0] if squeeze else out


def sym_band_to_general(band: np.ndarray):
    """Lower symmetric band storage (band[r,j] = A[j+r,j]) -> LAPACK gb storage with
    kl = ku = kb and 2*kl + ku + 1 rows (ab[kl+ku+i-j, j] = A[i,j]), complex128."""
    kb = band.shape[0] - 1
    N = band.shape[1]
    ab = np.zeros((3 * kb + 1, N), dtype=complex)
    for r in range(kb + 1):
        if r >= N:
            break
        vals = band[r, : N - r]
        ab[2 * kb + r, : N - r] = vals  # A[j+r, j], i - j = r
        ab[2 * kb - r, r:] = vals  # A[j, j+r] at column j+r, i - j = -r
    return ab


def banded_action(band, V, n: int, threads: int = 1, cols=None):
    """R_n(A) V for real symmetric banded A via zgbsv per pair, 2Re(a y), ascending sum."""
    theta, coef = pairs(n)
    band = np.asarray(band, dtype=np.float64)
    kb = band.shape[0] - 1
    V = np.asarray(V, dtype=np.float64)
    if cols is not None:
        V = V[:, cols]
    B = V.astype(complex)
    base = sym_band_to_general(band)

    def task(slot):
        ab = base.copy()
        ab[2 * kb, :] += theta[slot]
        _, _, y, info = lapack.zgbsv(kb, kb, ab, B, overwrite_ab=1)
        if info != 0:
            raise np.linalg.LinAlgError(f"zgbsv info={info}")
        return 2.0 * (coef[slot] * y).real

    return _reduce(_pool_map(task, len(theta), threads))
