"""Matrix types consumed by the engine, plus the single-shift solve API.

Dense `HermitianMatrix`/`SpectralBounds`/`gershgorin_bounds` keep the reference's
input contract (/root/reference/pkg/src/pfexpm/linalg.py:37-89,137-146): entries are
coerced to complex128, Hermitian-checked against tol_herm * max|a|, frozen.

`TridiagonalHermitian` and `BandedHermitian` are additive structured types (the
reference is dense-only) so configs C2/C5 are reachable through the
same `matexp_action` entry point.  They hold real symmetric matrices in compact
storage and are never densified.

`shifted_solve` / `shifted_inverse` (linalg.py:92-108) run on the GPU through the
same native dense kernels as the engine.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import BadSpec, InvariantViolation

RESIDUAL_FACTOR = 10.0
_EPS = float(np.finfo(np.float64).eps)


@dataclass(frozen=True)
class SpectralBounds:
    """[lo, hi] encloses the spectrum; exact=True when the ends are eigenvalues."""

    lo: float
    hi: float
    exact: bool = False

    def __post_init__(self):
        if not self.lo <= self.hi:
            raise InvariantViolation("bounds-order", f"lo = {self.lo} > hi = {self.hi}")

    def rho(self) -> float:
        return max(abs(self.lo), abs(self.hi))

    def alpha(self) -> float:
        return self.hi


@dataclass(frozen=True)
class HermitianMatrix:
    """Validated dense Hermitian matrix (complex128, read-only)."""

    entries: np.ndarray
    tol_herm: float = 1e-12
    bounds: SpectralBounds | None = field(default=None, compare=False)

    def __post_init__(self):
        a = np.asarray(self.entries, dtype=complex)
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise InvariantViolation("square", f"shape {a.shape}")
        if a.size:
            scale = max(1.0, float(np.max(np.abs(a))))
            dev = float(np.max(np.abs(a - a.conj().T)))
        else:
            scale, dev = 1.0, 0.0
        if dev > self.tol_herm * scale:
            raise InvariantViolation(
                "hermitian", f"max |A - A^H| = {dev:.3e} > {self.tol_herm:.1e} * {scale:.3e}"
            )
        if not a.flags.c_contiguous:
            a = np.ascontiguousarray(a)
        a.setflags(write=False)
        object.__setattr__(self, "entries", a)

    @property
    def d(self) -> int:
        return self.entries.shape[0]

    def is_real(self) -> bool:
        return bool(np.all(self.entries.imag == 0.0))

    def shifted_by(self, c: float) -> "HermitianMatrix":
        """A - cI with bounds moved accordingly (reference engine.py:296-301)."""
        b = None
        if self.bounds is not None:
            b = SpectralBounds(self.bounds.lo - c, self.bounds.hi - c, self.bounds.exact)
        return HermitianMatrix(self.entries - c * np.eye(self.d), tol_herm=self.tol_herm, bounds=b)


@dataclass(frozen=True)
class TridiagonalHermitian:
    """Real symmetric tridiagonal matrix: diag (N,), off (N-1,) float64."""

    diag: np.ndarray
    off: np.ndarray
    bounds: SpectralBounds | None = field(default=None, compare=False)

    def __post_init__(self):
        d = np.ascontiguousarray(np.asarray(self.diag, dtype=np.float64))
        o = np.ascontiguousarray(np.asarray(self.off, dtype=np.float64))
        if d.ndim != 1 or o.ndim != 1 or o.shape[0] != max(d.shape[0] - 1, 0):
            raise InvariantViolation("tridiagonal-shape", f"diag {d.shape}, off {o.shape}")
        if not (np.all(np.isfinite(d)) and np.all(np.isfinite(o))):
            raise InvariantViolation("finite", "non-finite tridiagonal entries")
        d.setflags(write=False)
        o.setflags(write=False)
        object.__setattr__(self, "diag", d)
        object.__setattr__(self, "off", o)

    @property
    def d(self) -> int:
        return self.diag.shape[0]

    def is_real(self) -> bool:
        return True

    def shifted_by(self, c: float) -> "TridiagonalHermitian":
        b = None
        if self.bounds is not None:
            b = SpectralBounds(self.bounds.lo - c, self.bounds.hi - c, self.bounds.exact)
        return TridiagonalHermitian(self.diag - c, self.off, bounds=b)


@dataclass(frozen=True)
class BandedHermitian:
    """Real symmetric band matrix in lower band storage.

    band[r, j] = A[j + r, j] for r = 0..kb; entries with j + r >= N are ignored.
    """

    band: np.ndarray
    bounds: SpectralBounds | None = field(default=None, compare=False)

    def __post_init__(self):
        b = np.ascontiguousarray(np.asarray(self.band, dtype=np.float64))
        if b.ndim != 2 or b.shape[0] < 1:
            raise InvariantViolation("band-shape", f"{b.shape}")
        if not np.all(np.isfinite(b)):
            raise InvariantViolation("finite", "non-finite band entries")
        b.setflags(write=False)
        object.__setattr__(self, "band", b)

    @property
    def d(self) -> int:
        return self.band.shape[1]

    @property
    def kb(self) -> int:
        return self.band.shape[0] - 1

    def is_real(self) -> bool:
        return True

    def shifted_by(self, c: float) -> "BandedHermitian":
        nb = np.array(self.band)
        nb[0] -= c
        b = None
        if self.bounds is not None:
            b = SpectralBounds(self.bounds.lo - c, self.bounds.hi - c, self.bounds.exact)
        return BandedHermitian(nb, bounds=b)


def gershgorin_bounds(A) -> SpectralBounds:
    """Gershgorin enclosure (reference linalg.py:137-146), for every matrix type."""
    if isinstance(A, HermitianMatrix):
        a = A.entries
        centers = np.real(np.diag(a))
        radii = np.sum(np.abs(a), axis=1) - np.abs(np.diag(a))
    elif isinstance(A, TridiagonalHermitian):
        centers = A.diag
        radii = np.zeros_like(centers)
        if A.d > 1:
            ao = np.abs(A.off)
            radii[:-1] += ao
            radii[1:] += ao
    elif isinstance(A, BandedHermitian):
        N, kb = A.d, A.kb
        centers = A.band[0].copy()
        radii = np.zeros(N)
        for r in range(1, kb + 1):
            if r >= N:
                break
            col = np.abs(A.band[r, : N - r])
            radii[: N - r] += col  # A[j+r, j] sits in row j+r and (by symmetry) row j
            radii[r:] += col
    else:
        raise BadSpec(f"unsupported matrix type {type(A).__name__}")
    if centers.size == 0:
        return SpectralBounds(0.0, 0.0, exact=False)
    return SpectralBounds(float(np.min(centers - radii)), float(np.max(centers + radii)), exact=False)


def shifted_solve(A: HermitianMatrix, theta: complex, V: np.ndarray) -> np.ndarray:
    """Solve (A + theta I) Y = V on the GPU (partial-pivoted LU; reference linalg.py:92-103)."""
    from . import _native

    return _native.shifted_solve(A, complex(theta), V)


def shifted_inverse(A: HermitianMatrix, theta: complex) -> np.ndarray:
    """(A + theta I)^{-1} on the GPU (reference linalg.py:106-108)."""
    return shifted_solve(A, theta, np.eye(A.d, dtype=complex))


def solve_residual_bound(A: HermitianMatrix, theta: complex, y: np.ndarray) -> float:
    """Right side of the residual contract (reference linalg.py:30-32,149-153)."""
    M = A.entries + np.asarray(theta, dtype=complex) * np.eye(A.d)
    return RESIDUAL_FACTOR * A.d * _EPS * float(np.linalg.norm(M, "fro")) * float(np.linalg.norm(y))
