"""Host-side logic of the engine API (reference tests/test_engine.py:80-163 patterns)."""
import math

import numpy as np
import pytest

from paper_2306_16778_b200 import (
    BadSpec,
    BandedHermitian,
    ExpOptions,
    ExpResult,
    HermitianMatrix,
    InvariantViolation,
    OrderOutOfRange,
    OrderTooSmall,
    PfexpmError,
    SingularSystem,
    SpectralBounds,
    TridiagonalHermitian,
    apriori_bound,
    approx_error,
    gershgorin_bounds,
    matexp_action,
    matexp_full,
)
from paper_2306_16778_b200.errors import raise_for_status
from paper_2306_16778_b200 import workloads


class TestOptions:
    def test_defaults(self):
        o = ExpOptions()
        assert o.n == 16 and o.mode == "full" and o.shift is None and o.parallel and o.threads == "auto"

    @pytest.mark.parametrize("shift", ["AUTO", float("inf"), float("nan"), True])
    def test_bad_shift(self, shift):
        with pytest.raises(BadSpec):
            ExpOptions(shift=shift)

    @pytest.mark.parametrize("threads", [0, -2, 1.5, True, "four"])
    def test_bad_threads(self, threads):
        with pytest.raises(BadSpec):
            ExpOptions(threads=threads)

    @pytest.mark.parametrize("n", [7, 0, 66, True])
    def test_bad_order(self, n):
        with pytest.raises(OrderOutOfRange):
            ExpOptions(n=n)

    def test_bad_mode(self):
        with pytest.raises(BadSpec):
            ExpOptions(mode="banana")


class TestResult:
    def test_t_para_invariant(self):
        with pytest.raises(InvariantViolation):
            ExpResult(np.eye(2), None, None, (1.0, 2.0), 1.0, 3.0)

    def test_bound_kind_pairing(self):
        with pytest.raises(InvariantViolation):
            ExpResult(np.eye(2), 0.5, None, (1.0,), 1.0, 1.0)


class TestBounds:
    def test_rho1_n4_hand_value(self):
        got = apriori_bound(SpectralBounds(-1.0, 0.0), 4)
        assert math.isclose(got, 24.0 / 65.0 - math.exp(-1.0), rel_tol=1e-12)

    def test_order_too_small(self):
        with pytest.raises(OrderTooSmall):
            apriori_bound(SpectralBounds(-1.0, 0.0), 2)

    def test_positive_interval(self):
        with pytest.raises(BadSpec):
            apriori_bound(SpectralBounds(-1.0, 0.5), 16)

    def test_approx_error_matches_high_precision(self):
        mp = pytest.importorskip("mpmath")
        mp.mp.dps = 50
        for n in (8, 16, 24):
            for x in (-1.0, -3.0, -9.0, -20.0, -40.0):
                en = sum(mp.mpf(-x) ** k / mp.factorial(k) for k in range(n + 1))
                want = float(1 / en - mp.exp(x))
                assert math.isclose(approx_error(n, x), want, rel_tol=1e-12)


class TestTypes:
    def test_hermitian_rejects_nonhermitian(self):
        with pytest.raises(InvariantViolation):
            HermitianMatrix(np.array([[0.0, 1.0], [0.0, 0.0]]))

    def test_entries_frozen(self):
        m = HermitianMatrix(np.eye(3))
        with pytest.raises(ValueError):
            m.entries[0, 0] = 2.0

    def test_gershgorin_structured_equals_dense(self):
        N = 30
        d, o = workloads.c2_matrix(N, scale=1.0)
        T = TridiagonalHermitian(d, o)
        D = HermitianMatrix(np.diag(d) + np.diag(o, 1) + np.diag(o, -1))
        assert gershgorin_bounds(T) == gershgorin_bounds(D)
        m = 5
        band = workloads.c5_band(m, scale=1.0)
        B = BandedHermitian(band)
        A = np.zeros((m * m, m * m))
        for r in range(m + 1):
            for j in range(m * m - r):
                A[j + r, j] = A[j, j + r] = band[r, j]
        g1, g2 = gershgorin_bounds(B), gershgorin_bounds(HermitianMatrix(A))
        assert math.isclose(g1.lo, g2.lo) and math.isclose(g1.hi, g2.hi)

    def test_tridiagonal_shape_checked(self):
        with pytest.raises(InvariantViolation):
            TridiagonalHermitian(np.zeros(4), np.zeros(4))


class TestErrors:
    def test_status_mapping(self):
        with pytest.raises(SingularSystem):
            raise_for_status(1, "x")
        with pytest.raises(BadSpec):
            raise_for_status(2, "x")
        with pytest.raises(PfexpmError):
            raise_for_status(3, "x")
        raise_for_status(0, "x")

    def test_mode_mismatch(self):
        A = HermitianMatrix(np.eye(3) * -1.0)
        with pytest.raises(BadSpec):
            matexp_full(A, ExpOptions(mode="action"))
        with pytest.raises(BadSpec):
            matexp_action(A, np.ones(3), ExpOptions(mode="full"))

    def test_positive_certified_spectrum_refused(self):
        A = HermitianMatrix(np.eye(3), bounds=SpectralBounds(1.0, 1.0, exact=True))
        with pytest.raises(BadSpec):
            matexp_full(A, ExpOptions(n=8))

    def test_shape_mismatch(self):
        A = HermitianMatrix(-np.eye(5))
        with pytest.raises(BadSpec):
            matexp_action(A, np.ones(4), ExpOptions(mode="action"))


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    A = HermitianMatrix(-np.eye(4))
    with pytest.raises(PfexpmError, match="no CUDA device"):
        matexp_action(A, np.ones(4), ExpOptions(mode="action"))


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    # the product path has no CPU fallback: without libpfx.so every entry raises
    from paper_2306_16778_b200 import _native

    monkeypatch.setattr(_native, "LIB_PATH", str(tmp_path / "absent" / "libpfx.so"))
    monkeypatch.setattr(_native, "_lib", None)
    with pytest.raises(PfexpmError, match="missing"):
        _native.lib()
    assert not _native.available()
    with pytest.raises(PfexpmError):
        matexp_action(HermitianMatrix(-np.eye(4)), np.ones(4), ExpOptions(mode="action"))
