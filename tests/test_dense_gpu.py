"""Dense path on the GPU vs the reference (golden outputs) and the CPU oracle.

Parity bar (BASELINE north_star): relative 2-norm / Frobenius error <= 1e-10 against the
CPU reference on the same inputs (P1), and error vs the eigen-oracle <= 10x the
reference's own (P2).  All calls go through the public API -> libpfx.so."""
import os

import numpy as np
import pytest

from oracle import restate
from paper_2306_16778_b200 import (
    ExpOptions,
    HermitianMatrix,
    SingularSystem,
    SpectralBounds,
    matexp_action,
    matexp_action_batched,
    matexp_full,
    matexp_shifted,
    shifted_inverse,
    shifted_solve,
    solve_residual_bound,
    workloads,
)
from paper_2306_16778_b200.roots import default_table

from .conftest import GOLDEN

pytestmark = pytest.mark.gpu
TOL = 1e-10


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _run_golden(z, name):
    A = z[f"{name}__A"]
    v = z.get(f"{name}__v")
    n = int(z[f"{name}__n"])
    mode = str(z[f"{name}__mode"])
    shift = str(z[f"{name}__shift"])
    H = HermitianMatrix(A)
    opts = ExpOptions(n=n, mode=mode, shift=None if shift == "none" else float(z[f"{name}__c"]))
    if opts.shift is not None:
        return matexp_shifted(H, opts, v=v)
    return matexp_action(H, v, opts) if mode == "action" else matexp_full(H, opts)


def test_all_golden_cases(golden_dense):
    z = golden_dense
    for name in z["names"]:
        name = str(name)
        res = _run_golden(z, name)
        want = z[f"{name}__value"]
        assert res.value.dtype == want.dtype, name
        assert res.value.shape == want.shape, name
        r = rel(res.value, want)
        assert r <= TOL, (name, r)
        # P2: no worse than 10x the reference's own distance to the eigen-oracle
        orc = z[f"{name}__oracle"]
        assert np.linalg.norm(res.value - orc) <= 10 * np.linalg.norm(want - orc) + 1e-13 * np.linalg.norm(orc), name


def test_c1_config(golden_dense):
    A, v, (lo, hi) = workloads.c1_inputs()
    H = HermitianMatrix(A, bounds=SpectralBounds(lo, hi, exact=True))
    with pytest.warns(Warning):
        res = matexp_action(H, v, ExpOptions(n=16, mode="action"))
    assert res.value.dtype == np.float64
    assert rel(res.value, golden_dense["c1__value"]) <= 1e-12
    assert len(res.per_term_times) == 8 and res.t_para == max(res.per_term_times)


def test_c3_head_vs_reference():
    z = np.load(os.path.join(GOLDEN, "c3_head.npz"))
    b = z["value"].shape[0]
    As = np.stack([workloads.c3_matrix(i) for i in range(b)])
    V = np.stack([workloads.c3_vector(i) for i in range(b)])
    got = matexp_action_batched(As, V, ExpOptions(n=20, mode="action"))
    for i in range(b):
        assert rel(got[i], z["value"][i]) <= TOL
        assert np.linalg.norm(got[i] - z["oracle"][i]) <= 10 * np.linalg.norm(z["value"][i] - z["oracle"][i])


@pytest.mark.parametrize("d", [1, 2, 7, 31, 32, 33, 64, 100, 130, 256, 300, 512])
def test_sizes_real_and_complex(d, rng):
    n = 16
    # spectra in [-8, 0]: exp(A)v is O(1), so the relative error measures the solves,
    # not the cancellation floor of the partial fractions on a vanishing result
    A, lo, hi = workloads.random_real_symmetric(d, -8.0, 0.0, seed=5, trial=d)
    v = workloads.unit_vector(d, 5, d)
    got = matexp_action(HermitianMatrix(A), v, ExpOptions(n=n, mode="action")).value
    want = restate.run_tasks_dense(A, v, n)
    assert rel(got, want) <= TOL
    Ac, _, _ = workloads.random_complex_hermitian(d, -8.0, 0.0, seed=6, trial=d)
    vc = rng.standard_normal(d) + 1j * rng.standard_normal(d)
    got = matexp_action(HermitianMatrix(Ac), vc, ExpOptions(n=n, mode="action")).value
    want = restate.run_tasks_dense(Ac, vc, n)
    assert rel(got, want) <= TOL


@pytest.mark.parametrize("d", [5, 40, 96])
def test_full_mode_real_and_complex(d):
    A, _, _ = workloads.random_real_symmetric(d, -10.0, 0.0, seed=7, trial=d)
    got = matexp_full(HermitianMatrix(A), ExpOptions(n=12)).value
    assert got.dtype == np.float64
    assert rel(got, restate.run_tasks_dense(A, None, 12)) <= TOL
    Ac, _, _ = workloads.random_complex_hermitian(d, -10.0, 0.0, seed=8, trial=d)
    got = matexp_full(HermitianMatrix(Ac), ExpOptions(n=12)).value
    want = restate.run_tasks_dense(Ac, None, 12)
    assert rel(got, want) <= TOL
    assert np.allclose(got, got.conj().T, atol=1e-13)


def test_multi_rhs_action():
    d, nrhs = 50, 5
    A, _, _ = workloads.random_complex_hermitian(d, -20.0, 0.0, seed=9)
    V = np.random.default_rng(3).standard_normal((d, nrhs))
    got = matexp_action(HermitianMatrix(A), V, ExpOptions(n=20, mode="action")).value
    for j in range(nrhs):
        assert rel(got[:, j], restate.run_tasks_dense(A, V[:, j], 20)) <= TOL


def test_zero_matrix_identity():
    d, n = 7, 8
    res = matexp_full(HermitianMatrix(np.zeros((d, d))), ExpOptions(n=n))
    assert np.max(np.abs(res.value - np.eye(d))) <= n * d * np.finfo(float).eps


def test_shifted_positive_spectrum():
    A, lo, hi = workloads.random_real_symmetric(40, 0.0, 5.0, seed=9)
    H = HermitianMatrix(A, bounds=SpectralBounds(lo, hi, exact=True))
    v = workloads.unit_vector(40, 10)
    res = matexp_shifted(H, ExpOptions(n=32, mode="action", shift="auto"), v=v)
    want = restate.matexp_dense(A, v, 32, shift=hi)
    assert rel(res.value, want) <= TOL
    assert res.c_applied == hi and res.bound_kind == "relative"


def test_determinism_bitwise():
    A, _, _ = workloads.random_complex_hermitian(64, -20.0, 0.0, seed=11)
    v = workloads.unit_vector(64, 12)
    r1 = matexp_action(HermitianMatrix(A), v, ExpOptions(n=16, mode="action")).value
    r2 = matexp_action(HermitianMatrix(A), v, ExpOptions(n=16, mode="action")).value
    assert np.array_equal(r1, r2)


def test_shifted_solve_residual_contract():
    # reference tests/test_linalg.py:82-117
    rng = np.random.default_rng(1016)
    thetas = default_table(16).thetas_f8()
    for _ in range(20):
        d = int(rng.integers(2, 201))
        A, _, _ = workloads.random_complex_hermitian(d, -50.0, 50.0, seed=int(rng.integers(0, 1000)))
        H = HermitianMatrix(A)
        v = rng.standard_normal(d) + 1j * rng.standard_normal(d)
        theta = thetas[int(rng.integers(0, 16))]
        y = shifted_solve(H, theta, v)
        M = A + theta * np.eye(d)
        assert np.linalg.norm(M @ y - v) <= solve_residual_bound(H, theta, y)


def test_shifted_inverse_and_singular():
    A = HermitianMatrix(np.zeros((2, 2)))
    assert np.allclose(shifted_inverse(A, 1j), -1j * np.eye(2), atol=1e-16)
    with pytest.raises(SingularSystem):
        shifted_solve(A, 0.0, np.ones(2))


@pytest.mark.parametrize("d,theta", [(513, 0.37), (700, -2.5 + 0.0j), (1024, 0.5 + 0.8j)])
def test_shifted_solve_large_pivoted(d, theta):
    # d > 512: blocked getrf/getrs with partial pivoting; real shifts make A + theta I
    # Hermitian indefinite, where interchanges are needed
    rng = np.random.default_rng(d)
    A, _, _ = workloads.random_complex_hermitian(d, -10.0, 10.0, seed=d)
    H = HermitianMatrix(A)
    V = rng.standard_normal((d, 3)) + 1j * rng.standard_normal((d, 3))
    Y = shifted_solve(H, theta, V)
    M = A + theta * np.eye(d)
    for j in range(3):
        assert np.linalg.norm(M @ Y[:, j] - V[:, j]) <= solve_residual_bound(H, theta, Y[:, j])
    want = np.linalg.solve(M, V)
    assert np.linalg.norm(Y - want) / np.linalg.norm(want) <= 1e-9


def test_shifted_solve_large_singular():
    d = 600
    A = HermitianMatrix(np.diag(np.r_[np.ones(d - 1), 0.0]))
    with pytest.raises(SingularSystem):
        shifted_solve(A, 0.0, np.ones(d))


@pytest.mark.parametrize("batch,d", [(300, 16), (700, 32)])
def test_host_batch_pipeline_matches_device(batch, d):
    """Host-memory batches of at least two chunks (five rounds of the resident CTAs each) are
    copied in by chunks and factored as each lands; every system is computed exactly as in
    the device-memory call, so the two agree bitwise."""
    import torch

    from paper_2306_16778_b200 import _native

    rng = np.random.default_rng(batch + d)
    A = np.stack([workloads.random_complex_hermitian(d, -30.0, 0.0, seed=s)[0] for s in range(batch)])
    V = rng.standard_normal((batch, d, 1))
    t2, c2 = default_table(20).interleaved()
    host = _native.expm_dense_host(A, V, t2, c2, 0.0)
    dev = torch.device("cuda:0")
    devr = _native.expm_dense_device(torch.from_numpy(A).to(dev), torch.from_numpy(V).to(dev), t2, c2, 0.0)
    assert np.array_equal(np.asarray(host).reshape(-1), devr.cpu().numpy().reshape(-1))
    want = restate.run_tasks_dense(A[-1], V[-1, :, 0], 20)
    got = np.asarray(host).reshape(batch, d)[-1]
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-10


_BLOCKED_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from oracle import restate
from paper_2306_16778_b200 import _native, workloads
from paper_2306_16778_b200.roots import default_table
worst = 0.0
for d, batch, nr, ca, cv in [(256, 32, 1, 1, 0), (256, 30, 3, 1, 1), (192, 40, 1, 0, 0), (320, 32, 2, 1, 0),
                              (512, 32, 4, 0, 1), (200, 36, 1, 1, 0)]:
    rng = np.random.default_rng(d * 100 + batch)
    mk = workloads.random_complex_hermitian if ca else workloads.random_real_symmetric
    As = np.stack([mk(d, -30.0, 0.0, seed=11, trial=i)[0] for i in range(batch)])
    V = rng.standard_normal((batch, d, nr)) + (1j * rng.standard_normal((batch, d, nr)) if cv else 0)
    t2, c2 = default_table(20).interleaved()
    _native.prof_enable(True); _native.prof_read()
    got = _native.expm_dense_host(As, V, t2, c2, 0.0)
    kern = _native.prof_read(); _native.prof_enable(False)
    assert "db_build" in kern and "bt_solve" in kern, kern
    for i in [0, batch // 2, batch - 1]:
        want = restate.run_tasks_dense(As[i], V[i], 20)
        worst = max(worst, float(np.linalg.norm(got[i] - want) / np.linalg.norm(want)))
print("WORST", worst)
"""


def test_blocked_batched_path_opt_in():
    """The opt-in batched blocked path (PFX_DENSE_BLOCKED=1, dense_blocked.cu) against the
    restatement in a subprocess (the switch is read once per process): complex and real A, real
    and complex right-hand sides, up to 4 columns, partial last 64-blocks (d = 200, 320)."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PFX_DENSE_BLOCKED="1")
    res = subprocess.run([sys.executable, "-c", _BLOCKED_SCRIPT, root], cwd=root, env=env, capture_output=True,
                         text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    worst = float(res.stdout.split("WORST")[-1])
    assert worst <= TOL, worst
