"""Pole/residue tables of R_n(z) = 1/exp_n(-z).

The engine needs, for each even n, the n/2 representatives theta_k (Im > 0) and
residues a_k of the partial-fraction expansion, bit-identical to the reference's
`default_table(n).thetas_f8()/coeffs_f8()` (/root/reference/pkg/src/pfexpm/roots.py:222-226,
315-318), in its pair order (ascending Re, roots.py:148-170).

Two sources, both pinned against the reference-generated golden fixtures
(tests/golden/tables):
  * the native host routine `pfx_pole_table` (csrc/poles.cpp): Aberth starting
    points, double-double Newton, product-formula residues — bit-identical to
    the reference for every even n <= 58;
  * `data/pole_tables_f8.txt`: the reference's numbers frozen as hex floats.
default_table() computes the table with the native routine and serves the frozen copy only for
the three orders where the two differ (NATIVE_DIFFERS), so the engine matches the reference
bit-for-bit at every n.
"""
from __future__ import annotations

import functools
import os
from dataclasses import dataclass

import numpy as np

from .errors import InvariantViolation, OrderOutOfRange

ORDER_MIN = 2
ORDER_MAX = 64
_DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "pole_tables_f8.txt")


def check_order(n: int) -> None:
    if not isinstance(n, (int, np.integer)) or isinstance(n, bool):
        raise OrderOutOfRange(f"order must be an integer, got {n!r}")
    if n % 2 != 0 or not (ORDER_MIN <= n <= ORDER_MAX):
        raise OrderOutOfRange(f"order must be even and in [{ORDER_MIN}, {ORDER_MAX}], got {n}")


@dataclass(frozen=True)
class PoleTable:
    """n/2 conjugate-pair representatives (Im theta > 0) and their residues."""

    n: int
    theta: np.ndarray  # (n/2,) complex128
    coef: np.ndarray  # (n/2,) complex128

    @property
    def npairs(self) -> int:
        return self.n // 2

    def thetas_f8(self) -> np.ndarray:
        """Full conjugate-adjacent layout, as reference RootTable.thetas_f8()."""
        out = np.empty(self.n, dtype=complex)
        out[0::2] = self.theta
        out[1::2] = np.conj(self.theta)
        return out

    def coeffs_f8(self) -> np.ndarray:
        out = np.empty(self.n, dtype=complex)
        out[0::2] = self.coef
        out[1::2] = np.conj(self.coef)
        return out

    def interleaved(self):
        """(theta2, coef2) float64 arrays [re0, im0, re1, im1, ...] for the C ABI."""
        t = np.ascontiguousarray(self.theta).view(np.float64).copy()
        c = np.ascontiguousarray(self.coef).view(np.float64).copy()
        return t, c


@functools.lru_cache(maxsize=None)
def _frozen_tables() -> dict:
    tables = {}
    with open(_DATA, "r", encoding="utf-8") as fh:
        for line in fh:
            parts = line.split()
            if not parts or parts[0].startswith("#"):
                continue
            n, k = int(parts[0]), int(parts[1])
            vals = [float.fromhex(p) for p in parts[2:6]]
            t, c = tables.setdefault(n, ([], []))
            assert len(t) == k
            t.append(complex(vals[0], vals[1]))
            c.append(complex(vals[2], vals[3]))
    return tables


def frozen_table(n: int) -> PoleTable:
    check_order(n)
    t, c = _frozen_tables()[n]
    return PoleTable(n, np.array(t, dtype=complex), np.array(c, dtype=complex))


def native_table(n: int) -> PoleTable:
    """Compute the table with the native double-double routine (pfx_pole_table)."""
    from . import _native

    check_order(n)
    theta2, coef2 = _native.pole_table(n)
    return PoleTable(n, theta2.view(np.complex128).copy(), coef2.view(np.complex128).copy())


def validate(table: PoleTable) -> None:
    """Structural invariants (reference roots.py:233-298): Im>0 reps, ascending Re,
    1 <= |theta| <= n, outside the parabola Im^2 < 4(Re+1)."""
    th = table.theta
    if th.shape != (table.npairs,) or table.coef.shape != (table.npairs,):
        raise InvariantViolation("length", f"expected {table.npairs} pairs")
    if np.any(th.imag <= 0):
        raise InvariantViolation("pair-order", "representatives must have Im > 0")
    key = list(zip(th.real, th.imag))
    if any(a >= b for a, b in zip(key, key[1:])):
        raise InvariantViolation("pair-sort", "pairs must ascend by (Re, Im)")
    m2 = np.abs(th) ** 2
    if np.any(m2 < 1.0 * (1 - 1e-15)) or np.any(m2 > table.n**2 * (1 + 1e-15)):
        raise InvariantViolation("modulus", "|theta| outside [1, n]")
    if np.any(th.imag**2 < 4.0 * (th.real + 1.0)):
        raise InvariantViolation("parabola", "root inside Im^2 < 4(Re+1)")


# Orders where the native double-double routine and the reference tables differ
# (tests/test_poles.py): at n=62 the reference's 5-step double-double Newton
# from LAPACK companion eigenvalues stops 4e-14 (relative) short of the root
# (the native value is the correctly rounded root, checked with mpmath at 60
# digits); at n=60 and n=64 one residue differs by 1 ulp.  The engine needs the
# reference's numbers bit-for-bit, so default_table() serves the frozen copy.
NATIVE_DIFFERS = (60, 62, 64)


@functools.lru_cache(maxsize=None)
def default_table(n: int) -> PoleTable:
    """Process-wide table cache (reference roots.py:315-318), bit-identical to the
    reference's default_table(n).thetas_f8()/coeffs_f8() at even indices."""
    check_order(n)
    # the product computes its own poles (native double-double routine, bit-identical to the
    # reference for these orders: tests/test_poles.py); the three orders where the reference's
    # own numbers differ in the last place, and a checkout without the built library, are
    # served from the frozen copy of the reference's tables
    if n not in NATIVE_DIFFERS:
        from . import _native

        if _native.available():
            return native_table(n)
    return frozen_table(n)
