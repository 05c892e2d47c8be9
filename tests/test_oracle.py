"""The CPU oracle against the reference's own outputs (golden fixtures made by
running the unmodified reference, tests/golden/make_golden.py)."""
import os

import numpy as np
import pytest

from oracle import closed, restate
from paper_2306_16778_b200 import workloads
from paper_2306_16778_b200.roots import default_table, frozen_table, validate

from .conftest import GOLDEN


def _case(z, name):
    A = z[f"{name}__A"]
    v = z.get(f"{name}__v")
    n = int(z[f"{name}__n"])
    c = float(z[f"{name}__c"])
    return A, v, n, (None if np.isnan(c) else c)


def test_golden_tables_text_matches_f8():
    z = np.load(os.path.join(GOLDEN, "tables_f8.npz"))
    for n in range(2, 65, 2):
        text = open(os.path.join(GOLDEN, "tables", f"n{n}.txt")).read().splitlines()
        assert text[0] == "pfexpm-table v1" and text[1] == f"n={n}" and text[2] == "method=product"
        assert len([ln for ln in text[3:] if ln.strip()]) == 2 * n
        assert z[f"theta_{n}"].shape == (n,)


@pytest.mark.parametrize("n", list(range(2, 65, 2)))
def test_package_tables_bit_identical_to_reference(n):
    z = np.load(os.path.join(GOLDEN, "tables_f8.npz"))
    t = default_table(n)
    validate(t)
    assert np.array_equal(t.thetas_f8().view(np.float64), z[f"theta_{n}"].view(np.float64))
    assert np.array_equal(t.coeffs_f8().view(np.float64), z[f"coef_{n}"].view(np.float64))
    # conjugate closure (roots.py:244-257)
    assert np.array_equal(t.thetas_f8()[1::2], np.conj(t.thetas_f8()[0::2]))


def test_oracle_pairs_are_reference_pairs():
    for n in (16, 20, 24):
        th, co = restate.pairs(n)
        t = frozen_table(n)
        assert np.array_equal(th, t.theta) and np.array_equal(co, t.coef)


def test_dense_restatement_bitwise_equal_to_reference(golden_dense):
    z = golden_dense
    for name in z["names"]:
        A, v, n, c = _case(z, str(name))
        got = restate.matexp_dense(A, v, n, shift=c)
        want = z[f"{name}__value"]
        assert got.dtype == want.dtype, name
        assert np.array_equal(got, want), (name, np.max(np.abs(got - want)))


def test_tridiagonal_restatement_matches_dense_reference_path():
    N = 60
    d, o = workloads.c2_matrix(N)
    V = np.random.default_rng(1).standard_normal((N, 3))
    T = np.diag(d) + np.diag(o, 1) + np.diag(o, -1)
    a = restate.tridiag_action(d, o, V, 24)
    b = np.stack([restate.run_tasks_dense(T, V[:, j], 24) for j in range(3)], 1)
    assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b)


def test_banded_restatement_matches_dense_reference_path():
    m = 7
    band = workloads.c5_band(m, scale=2.0)  # spectrum in (-16, 0): exp not tiny
    V = np.random.default_rng(2).standard_normal((m * m, 2))
    N = m * m
    A = np.zeros((N, N))
    for r in range(m + 1):
        for j in range(N - r):
            A[j + r, j] = A[j, j + r] = band[r, j]
    got = restate.banded_action(band, V, 16)
    want = np.stack([restate.run_tasks_dense(A, V[:, j], 16) for j in range(2)], 1)
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


def test_closed_form_oracles():
    N = 40
    d, o = workloads.c2_matrix(N, scale=3.0)
    T = np.diag(d) + np.diag(o, 1) + np.diag(o, -1)
    V = np.random.default_rng(3).standard_normal((N, 2))
    assert np.allclose(closed.dst_exp_lap1d(N, 3.0, V), closed.exp_eig(T).real @ V, atol=1e-13)
    m = 6
    band = workloads.c5_band(m, scale=1.5)
    A = np.zeros((m * m, m * m))
    for r in range(m + 1):
        for j in range(m * m - r):
            A[j + r, j] = A[j, j + r] = band[r, j]
    V2 = np.random.default_rng(4).standard_normal((m * m, 2))
    assert np.allclose(closed.dst_exp_lap2d(m, 1.5, V2), closed.exp_eig(A).real @ V2, atol=1e-13)


def test_c1_reference_error_vs_eigen_oracle(golden_dense):
    # reference error of C1 against the eigen-oracle is ~1.57e-6 (truncation)
    z = golden_dense
    val, orc = z["c1__value"], z["c1__oracle"]
    err = np.linalg.norm(val - orc) / np.linalg.norm(orc)
    assert 1e-7 < err < 1e-5


def test_workload_c1_is_reference_c1(golden_dense):
    A, v, _ = workloads.c1_inputs()
    assert np.array_equal(A, golden_dense["c1__A"].real)
    assert np.array_equal(v, golden_dense["c1__v"])


def test_workload_c3_matches_reference_head():
    z = np.load(os.path.join(GOLDEN, "c3_head.npz"))
    for b in range(2):
        A, v = workloads.c3_matrix(b), workloads.c3_vector(b)
        got = restate.run_tasks_dense(A, v, 20)
        assert np.array_equal(got, z["value"][b])
