"""Scalar pieces the engine needs for its certified bound (host-only, tiny).

Restates err_n(x) = R_n(x) - exp(x) on x <= 0 from the reference
(/root/reference/pkg/src/pfexpm/scalar.py:380-423): for y = -x < n+1 it uses the
all-positive tail identity err_n = tail_n(y) e^{-y} / exp_n(y), otherwise the
direct difference.  exp_trunc is Horner on the truncated Taylor series
(scalar.py:80-100).
"""
from __future__ import annotations

from functools import lru_cache

import numpy as np

from .roots import check_order


@lru_cache(maxsize=None)
def _inv_fact(n: int) -> tuple:
    vals, f = [1.0], 1.0
    for k in range(1, n + 1):
        f *= k
        vals.append(1.0 / f)
    return tuple(vals)


def exp_trunc(n: int, z):
    c = _inv_fact(n)
    p = z * 0 + c[n]
    for k in range(n - 1, -1, -1):
        p = p * z + c[k]
    return p


def approx_error(n: int, x):
    check_order(n)
    is_scalar = np.isscalar(x) or (isinstance(x, np.ndarray) and x.ndim == 0)
    y = np.atleast_1d(-np.asarray(x, dtype=np.float64))
    if np.any(y < 0.0):
        raise ValueError("x must be <= 0")
    p = exp_trunc(n, y)
    res = np.empty_like(y)
    far = y >= n + 1.0
    if np.any(far):
        res[far] = 1.0 / p[far] - np.exp(-y[far])
    near = ~far
    if np.any(near):
        yn = y[near]
        term = np.ones_like(yn)
        for k in range(1, n + 2):
            term = term * yn / k
        acc = term.copy()
        k = n + 1
        while True:
            k += 1
            term = term * yn / k
            acc = acc + term
            if np.all(term <= 1e-20 * acc) or k > n + 200:
                break
        res[near] = acc * np.exp(-yn) / p[near]
    return float(res[0]) if is_scalar else res.reshape(np.shape(x))
