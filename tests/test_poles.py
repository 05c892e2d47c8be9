"""Native pole/residue table (pfx_pole_table, csrc/poles.cpp) vs the reference tables."""
import numpy as np
import pytest

from paper_2306_16778_b200 import roots


@pytest.mark.parametrize("n", list(range(2, 65, 2)))
def test_native_table(n):
    nat = roots.native_table(n)
    ref = roots.frozen_table(n)
    roots.validate(nat)
    if n not in roots.NATIVE_DIFFERS:
        assert np.array_equal(nat.theta.view(np.float64), ref.theta.view(np.float64))
        assert np.array_equal(nat.coef.view(np.float64), ref.coef.view(np.float64))
    else:
        # reference n=62 root is 4e-14 short of convergence; n=60/64 residues differ by 1 ulp
        assert np.max(np.abs(nat.theta - ref.theta) / np.abs(ref.theta)) <= 1e-13
        assert np.max(np.abs(nat.coef - ref.coef) / np.abs(ref.coef)) <= 1e-11


def test_residue_identity():
    # sum_k a_k / theta_k = R_n(0) = 1 over all n roots (reference tests/test_roots.py:62-69)
    for n in (8, 16, 24, 32):
        t = roots.native_table(n)
        s = np.sum(t.coeffs_f8() / t.thetas_f8())
        assert abs(s - 1.0) < 1e-12


def test_bad_order_rejected():
    from paper_2306_16778_b200 import _native
    from paper_2306_16778_b200.errors import BadSpec

    with pytest.raises(BadSpec):
        _native.pole_table(7)
