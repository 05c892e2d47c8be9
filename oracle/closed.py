"""Exact (truncation-free) oracles — TEST INFRASTRUCTURE ONLY.

exp_eig:        U e^Lambda U^H via eigh (reference linalg.py:111-123).
dst_exp_lap1d:  exp(s*tridiag(1,-2,1)) V through the orthonormal DST-I
                eigenbasis, lambda_k = -4 s sin^2(k pi / (2(N+1)))
                (closed form used by reference tests/test_linalg.py:145-151,177-184).
dst_exp_lap2d:  same for s*(kron(T,I) + kron(I,T)) on an m x m grid
                (Kronecker-sum spectrum, reference tests/test_bench.py:78-87).
"""
from __future__ import annotations

import numpy as np
import scipy.fft


def exp_eig(A: np.ndarray) -> np.ndarray:
    w, U = np.linalg.eigh(np.asarray(A, dtype=complex))
    return (U * np.exp(w)) @ U.conj().T


def _lam(N: int, s: float) -> np.ndarray:
    k = np.arange(1, N + 1)
    return -4.0 * s * np.sin(k * np.pi / (2.0 * (N + 1))) ** 2


def dst_exp_lap1d(N: int, s: float, V: np.ndarray) -> np.ndarray:
    W = scipy.fft.dst(V, type=1, norm="ortho", axis=0)
    lam = _lam(N, s)
    W = W * (np.exp(lam)[:, None] if W.ndim == 2 else np.exp(lam))
    return scipy.fft.dst(W, type=1, norm="ortho", axis=0)


def dst_exp_lap2d(m: int, s: float, V: np.ndarray, ny: int | None = None) -> np.ndarray:
    """exp(s (kron(T_ny, I_m) + kron(I_ny, T_m))) V on an m x ny grid (x = m fastest);
    ny = None: the square m x m grid."""
    ny = m if ny is None else ny
    nrhs = V.shape[1]
    X = V.reshape(ny, m, nrhs)
    W = scipy.fft.dstn(X, type=1, norm="ortho", axes=(0, 1))
    W = W * np.exp(_lam(ny, s)[:, None] + _lam(m, s)[None, :])[:, :, None]
    return scipy.fft.dstn(W, type=1, norm="ortho", axes=(0, 1)).reshape(m * ny, nrhs)
