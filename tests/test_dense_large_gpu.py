"""Large dense path (d > 512, blocked LU on DMMA; config C4 shape) vs the CPU reference restatement."""
import numpy as np
import pytest

from oracle import restate
from paper_2306_16778_b200 import ExpOptions, HermitianMatrix, matexp_action, matexp_full, workloads

pytestmark = pytest.mark.gpu
TOL = 1e-10


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("d", [513, 700, 1024])
def test_full_complex(d):
    A, lo, hi = workloads.random_complex_hermitian(d, -60.0, 0.0, seed=4, trial=d)
    got = matexp_full(HermitianMatrix(A), ExpOptions(n=24)).value
    want = restate.run_tasks_dense(A, None, 24, threads=8)
    assert got.dtype == np.complex128
    assert rel(got, want) <= TOL, rel(got, want)
    assert np.allclose(got, got.conj().T, atol=1e-12)


def test_full_real():
    d = 600
    A, _, _ = workloads.random_real_symmetric(d, -30.0, 0.0, seed=2)
    got = matexp_full(HermitianMatrix(A), ExpOptions(n=16)).value
    assert got.dtype == np.float64
    assert rel(got, restate.run_tasks_dense(A, None, 16, threads=8)) <= TOL


def test_action_complex_and_real():
    d = 800
    A, _, _ = workloads.random_complex_hermitian(d, -40.0, 0.0, seed=3)
    v = workloads.unit_vector(d, 3)
    got = matexp_action(HermitianMatrix(A), v, ExpOptions(n=20, mode="action")).value
    assert rel(got, restate.run_tasks_dense(A, v, 20)) <= TOL
    Ar, _, _ = workloads.random_real_symmetric(d, -40.0, 0.0, seed=3)
    V = np.random.default_rng(5).standard_normal((d, 4))
    got = matexp_action(HermitianMatrix(Ar), V, ExpOptions(n=20, mode="action")).value
    for j in range(4):
        assert rel(got[:, j], restate.run_tasks_dense(Ar, V[:, j], 20)) <= TOL


@pytest.mark.parametrize("d", [577, 777])
def test_full_real_symmetric_inverse(d):
    # real A: the inverse of A + theta I is complex symmetric, only its lower triangle is
    # computed and the combine mirrors it -> exp(A) comes out exactly symmetric
    A, _, _ = workloads.random_real_symmetric(d, -50.0, 0.0, seed=d)
    got = matexp_full(HermitianMatrix(A), ExpOptions(n=20)).value
    assert got.dtype == np.float64
    assert rel(got, restate.run_tasks_dense(A, None, 20, threads=8)) <= TOL
    assert np.array_equal(got, got.T)
