"""Partial pivoting on the dense product path (include/pfx.h pfx_set_pivot_mode).

The reference factors with LAPACK zgesv / zgetrf, i.e. partial pivoting
(/root/reference/pkg/src/pfexpm/engine.py:200,203,208; linalg.py:92-103).  The default mode
here, "checked", runs the interchange-free kernels and verifies per column that partial
pivoting (izamax on the updated column) would have kept the diagonal pivot; otherwise the call
is redone with interchanges.  These tests drive both outcomes:

  * Hermitian NSD inputs (every BASELINE config): the check passes, no redo, and the result
    equals the unchecked interchange-free result bit for bit (same kernels);
  * Hermitian inputs with a weak diagonal (|a_ij| >> |a_ii + theta|): partial pivoting must
    exchange rows, the check fails, the call is redone with interchanges and matches the
    LAPACK restatement -- on the batched kernels (d <= 512, both the NB = 32 and the two-CTA
    NB = 16 variants) and on the blocked large path (d > 512);
  * "always" (getrf interchanges on every column) agrees with "checked" to rounding.
"""
import numpy as np
import pytest

from oracle import restate
from paper_2306_16778_b200 import _native, workloads
from paper_2306_16778_b200.roots import default_table

pytestmark = pytest.mark.gpu
TOL = 1e-10


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture
def pivot_mode():
    old = _native.get_pivot_mode()
    yield _native.set_pivot_mode
    _native.set_pivot_mode(old)


def weak_diagonal_hermitian(d, seed, scale=20.0):
    """Hermitian with zero diagonal and O(scale) off-diagonal entries: for every pole,
    |a_r0| >> |theta|, so partial pivoting exchanges rows at the first column already."""
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
    A = (G + G.conj().T) * (scale / np.sqrt(2 * d))
    np.fill_diagonal(A, 0.0)
    return A


def run(A, v, n, batch=False):
    t2, c2 = default_table(n).interleaved()
    return _native.expm_dense_host(A, v, t2, c2, 0.0)


def test_default_mode_is_checked():
    assert _native.get_pivot_mode() == "checked"


@pytest.mark.parametrize("d", [48, 200, 700])
def test_weak_diagonal_needs_pivoting(d, pivot_mode):
    A = weak_diagonal_hermitian(d, seed=d)
    v = workloads.unit_vector(d, 3, d)
    pivot_mode("checked")
    before = _native.pivot_fallbacks()
    got = run(A, v, 16)
    assert _native.pivot_fallbacks() == before + 1  # the check failed and the call was redone
    want = restate.run_tasks_dense(A, v, 16)
    assert rel(got, want) <= TOL, rel(got, want)
    pivot_mode("always")
    got_piv = run(A, v, 16)
    assert rel(got_piv, want) <= TOL


def test_weak_diagonal_batched_two_cta_variant(pivot_mode):
    # 16 matrices x 10 pairs = 160 systems > 148 SMs: the two-CTA NB = 16 kernel (C3's)
    d, b, n = 96, 16, 20
    As = np.stack([weak_diagonal_hermitian(d, seed=100 + i) for i in range(b)])
    As[::2] = np.stack([workloads.random_complex_hermitian(d, -30.0, 0.0, seed=7, trial=i)[0] for i in range(0, b, 2)])
    V = np.stack([workloads.unit_vector(d, 4, i) for i in range(b)]).astype(complex)
    pivot_mode("checked")
    before = _native.pivot_fallbacks()
    got = run(As, V[..., None], n)[..., 0]
    assert _native.pivot_fallbacks() == before + 1
    for i in range(b):
        want = restate.run_tasks_dense(As[i], V[i], n)
        assert rel(got[i], want) <= TOL, (i, rel(got[i], want))


def test_weak_diagonal_full_mode_large(pivot_mode):
    d = 576
    A = weak_diagonal_hermitian(d, seed=11, scale=20.0)
    pivot_mode("checked")
    before = _native.pivot_fallbacks()
    t2, c2 = default_table(12).interleaved()
    got = _native.expm_dense_host(A, None, t2, c2, 0.0)
    assert _native.pivot_fallbacks() == before + 1
    want = restate.run_tasks_dense(A, None, 12)
    assert rel(got, want) <= TOL


@pytest.mark.parametrize("cfg", ["C1", "C3head", "large"])
def test_hermitian_nsd_check_passes_bitwise(cfg, pivot_mode):
    """On the configs' inputs the checked LU keeps every pivot: no redo, and the output is
    bitwise the unchecked interchange-free output; 'always' agrees to rounding."""
    if cfg == "C1":
        A, v, _ = workloads.c1_inputs()
        n = 16
    elif cfg == "C3head":
        A = np.stack([workloads.c3_matrix(i) for i in range(20)])
        v = np.stack([workloads.c3_vector(i) for i in range(20)])[..., None]
        n = 20
    else:
        A, _, _ = workloads.random_complex_hermitian(640, -500.0, 0.0, seed=3)
        v = workloads.unit_vector(640, 3)
        n = 24
    pivot_mode("checked")
    before = _native.pivot_fallbacks()
    chk = run(A, v, n)
    assert _native.pivot_fallbacks() == before
    pivot_mode("none")
    nop = run(A, v, n)
    assert np.array_equal(chk, nop)
    pivot_mode("always")
    piv = run(A, v, n)
    assert rel(piv, chk) <= 1e-12


def test_bad_pivot_mode():
    from paper_2306_16778_b200 import BadSpec

    with pytest.raises(BadSpec):
        _native.set_pivot_mode("sometimes")
