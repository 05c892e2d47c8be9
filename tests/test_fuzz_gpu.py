"""Seeded randomized parity sweep over every GPU path (sizes around the tile / panel / band
boundaries, 1-5 right-hand sides, real and complex data) against the CPU restatement."""
import numpy as np
import pytest

from oracle import restate
from paper_2306_16778_b200 import (BandedHermitian, ExpOptions, HermitianMatrix, TridiagonalHermitian,
                                   matexp_action, matexp_full, workloads)

pytestmark = pytest.mark.gpu
TOL = 1e-10


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


DENSE = [(d, nrhs, cplx) for d, nrhs, cplx in
         [(1, 1, False), (7, 3, True), (17, 5, False), (33, 4, True), (65, 2, False), (100, 1, True),
          (129, 3, False), (255, 5, True), (257, 1, False), (300, 4, True), (511, 2, False), (513, 3, True)]]


@pytest.mark.parametrize("d,nrhs,cplx", DENSE)
def test_dense_action(d, nrhs, cplx):
    rng = np.random.default_rng(1000 + d)
    if cplx:
        A, _, _ = workloads.random_complex_hermitian(d, -20.0, 0.0, seed=d)
        V = rng.standard_normal((d, nrhs)) + 1j * rng.standard_normal((d, nrhs))
    else:
        A, _, _ = workloads.random_real_symmetric(d, -20.0, 0.0, seed=d)
        V = rng.standard_normal((d, nrhs))
    got = matexp_action(HermitianMatrix(A), V, ExpOptions(n=20, mode="action")).value
    for j in range(nrhs):
        assert rel(got[:, j], restate.run_tasks_dense(A, V[:, j], 20)) <= TOL


@pytest.mark.parametrize("d", [3, 31, 96, 200, 520])
def test_dense_full(d):
    A, _, _ = workloads.random_real_symmetric(d, -15.0, 0.0, seed=7 * d)
    got = matexp_full(HermitianMatrix(A), ExpOptions(n=16)).value
    assert rel(got, restate.run_tasks_dense(A, None, 16, threads=8)) <= TOL


@pytest.mark.parametrize("N,nrhs", [(2, 1), (255, 2), (256, 17), (257, 16), (4095, 3), (20000, 33)])
def test_tridiag(N, nrhs):
    rng = np.random.default_rng(N + nrhs)
    d = -rng.uniform(0.5, 4.0, N)
    o = rng.uniform(-1.0, 1.0, max(N - 1, 0)) * 0.9
    V = rng.standard_normal((N, nrhs))
    got = matexp_action(TridiagonalHermitian(d, o), V, ExpOptions(n=24, mode="action")).value
    assert rel(got, restate.tridiag_action(d, o, V, 24)) <= TOL


@pytest.mark.parametrize("N,kb,nrhs", [(63, 1, 1), (64, 63, 2), (130, 64, 3), (700, 130, 8), (1000, 500, 4)])
def test_banded(N, kb, nrhs):
    rng = np.random.default_rng(N * 3 + kb)
    band = rng.uniform(-1, 1, (kb + 1, N)) * (0.5 / np.sqrt(kb + 1))
    band[0] = -rng.uniform(0.5, 3.0, N)
    V = rng.standard_normal((N, nrhs))
    got = matexp_action(BandedHermitian(band), V, ExpOptions(n=16, mode="action")).value
    assert rel(got, restate.banded_action(band, V, 16)) <= TOL
