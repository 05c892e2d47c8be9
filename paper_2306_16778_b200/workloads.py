"""Seeded synthetic inputs for the five BASELINE configurations.

No public dataset is involved: the reference's own benchmark matrices are
synthetic (random spectrum, Laplacians; /root/reference/pkg/src/pfexpm/bench.py:1-10),
and these recipes reproduce them bit-for-bit with numpy's default_rng using the
reference's list-seed protocol (bench.py:174,186).

C1  dense real symmetric, d=128, spectrum U[-50,0], exp(A)v, n=16      (bench.py:171-188)
C2  1-D Dirichlet Laplacian, N=2^20, spectrum (-100,0), 16 RHS, n=24   (tridiagonal)
C3  512 dense complex Hermitian, d=256, U[-200,0], exp(A)v, n=20       (batched)
C4  dense complex Hermitian, d=4096, U[-500,0], full exp(A), n=24
C5  2-D 5-point Laplacian on 512^2 (bandwidth 512), (-400,0), 8 RHS, n=16 (banded)
"""
from __future__ import annotations

import numpy as np

C1 = dict(name="C1", d=128, lo=-50.0, hi=0.0, n=16)
C2 = dict(name="C2", N=1 << 20, nrhs=16, n=24, scale=25.0)
C3 = dict(name="C3", d=256, batch=512, lo=-200.0, hi=0.0, n=20)
C4 = dict(name="C4", d=4096, lo=-500.0, hi=0.0, n=24)
C5 = dict(name="C5", m=512, nrhs=8, n=16, scale=50.0)


def random_real_symmetric(d: int, lo: float, hi: float, seed: int = 0, trial: int = 0):
    """Q diag(lam) Q^T with sign-fixed QR (recipe of bench.gen_matrix, bench.py:173-182).

    Returns (A, lam_min, lam_max)."""
    rng = np.random.default_rng([seed, trial])
    lam = np.sort(rng.uniform(lo, hi, d))
    Q, R = np.linalg.qr(rng.standard_normal((d, d)))
    Q = Q * np.sign(np.diag(R))
    A = (Q * lam) @ Q.T
    A = (A + A.T) / 2.0
    return A, float(lam[0]), float(lam[-1])


def unit_vector(d: int, seed: int = 0, trial: int = 0) -> np.ndarray:
    """Seeded Gaussian unit vector (recipe of bench._unit_vector, bench.py:185-188)."""
    rng = np.random.default_rng([seed, trial, 1])
    v = rng.standard_normal(d)
    return v / np.linalg.norm(v)


def random_complex_hermitian(d: int, lo: float, hi: float, seed: int = 0, trial: int = 0):
    """U diag(lam) U^H, U from the phase-fixed QR of a complex Gaussian.

    Draw order (real part first) is part of the recipe.  Returns (A, lam_min, lam_max)."""
    rng = np.random.default_rng([seed, trial])
    lam = np.sort(rng.uniform(lo, hi, d))
    Gr = rng.standard_normal((d, d))
    Gi = rng.standard_normal((d, d))
    Q, R = np.linalg.qr(Gr + 1j * Gi)
    dr = np.diag(R)
    Q = Q * (dr / np.abs(dr))
    A = (Q * lam) @ Q.conj().T
    A = (A + A.conj().T) / 2.0
    return A, float(lam[0]), float(lam[-1])


# -- C1 ----------------------------------------------------------------------

def c1_inputs():
    A, lo, hi = random_real_symmetric(C1["d"], C1["lo"], C1["hi"], 0, 0)
    return A, unit_vector(C1["d"], 0, 0), (lo, hi)


# -- C2 ----------------------------------------------------------------------

def c2_matrix(N: int = C2["N"], scale: float = C2["scale"]):
    """tA = scale * tridiag(1,-2,1): diag (N,), off-diagonal (N-1,), float64.

    scale = 25 puts the spectrum -100 sin^2(k pi / (2(N+1))) inside (-100, 0)."""
    diag = np.full(N, -2.0 * scale)
    off = np.full(N - 1, scale)
    return diag, off


def c2_rhs(N: int = C2["N"], nrhs: int = C2["nrhs"]):
    return np.random.default_rng([0, 0, 1]).standard_normal((N, nrhs))


# -- C3 ----------------------------------------------------------------------

def c3_matrix(b: int, d: int = C3["d"]):
    A, _, _ = random_complex_hermitian(d, C3["lo"], C3["hi"], 0, b)
    return A


def c3_bounds(b: int, d: int = C3["d"]):
    """Exact spectral bounds of c3_matrix(b) (known by construction)."""
    from .linalg import SpectralBounds
    rng = np.random.default_rng([0, b])
    lam = np.sort(rng.uniform(C3["lo"], C3["hi"], d))
    return SpectralBounds(float(lam[0]), float(lam[-1]), exact=True)


def c3_vector(b: int, d: int = C3["d"]):
    return unit_vector(d, 0, b)


def c3_batch(batch: int = C3["batch"], d: int = C3["d"]):
    A = np.empty((batch, d, d), dtype=np.complex128)
    V = np.empty((batch, d), dtype=np.float64)
    for b in range(batch):
        A[b] = c3_matrix(b, d)
        V[b] = c3_vector(b, d)
    return A, V


# -- C4 ----------------------------------------------------------------------

def c4_matrix(d: int = C4["d"]):
    A, lo, hi = random_complex_hermitian(d, C4["lo"], C4["hi"], 0, 0)
    return A, (lo, hi)


def c4_eigen(d: int = C4["d"]):
    """(A, Q, lam) of the C4 recipe: A = Q diag(lam) Q^H (symmetrised), so exp(A) is known
    by construction (Q e^lam Q^H), the eigen-oracle of SURVEY §8d P2 without an eigh."""
    rng = np.random.default_rng([0, 0])
    lam = np.sort(rng.uniform(C4["lo"], C4["hi"], d))
    Gr = rng.standard_normal((d, d))
    Gi = rng.standard_normal((d, d))
    Q, R = np.linalg.qr(Gr + 1j * Gi)
    dr = np.diag(R)
    Q = Q * (dr / np.abs(dr))
    A = (Q * lam) @ Q.conj().T
    A = (A + A.conj().T) / 2.0
    return A, Q, lam


# -- C5 ----------------------------------------------------------------------

def c5_band(m: int = C5["m"], scale: float = C5["scale"]):
    """A = scale*(kron(T,I) + kron(I,T)), T = tridiag(1,-2,1) of size m, natural ordering.

    Returned in symmetric lower band storage: band[r, j] = A[j + r, j] for
    r = 0..m (kb = m), zero where j + r >= N.  Spectrum inside (-8*scale, 0)."""
    return c5_band_rect(m, m, scale)


def c5_band_rect(nx: int, ny: int, scale: float = C5["scale"]):
    """5-point Dirichlet Laplacian on an nx x ny grid (x fastest, natural ordering):
    A = scale*(kron(T_ny, I_nx) + kron(I_ny, T_nx)), bandwidth kb = nx, N = nx*ny, in the
    lower band storage of c5_band.  The C5 recipe at a reduced row count (full bandwidth)."""
    N = nx * ny
    band = np.zeros((nx + 1, N))
    band[0, :] = -4.0 * scale
    j = np.arange(N - 1)
    band[1, : N - 1] = np.where((j % nx) != nx - 1, scale, 0.0)
    band[nx, : N - nx] = scale
    return band


def c5_rhs(m: int = C5["m"], nrhs: int = C5["nrhs"]):
    return np.random.default_rng([0, 0, 1]).standard_normal((m * m, nrhs))
