"""Tridiagonal path (config C2) on the GPU vs the CPU restatement (zgtsv per pair)."""
import numpy as np
import pytest

from oracle import closed, restate
from paper_2306_16778_b200 import ExpOptions, TridiagonalHermitian, matexp_action, matexp_shifted, workloads

pytestmark = pytest.mark.gpu
TOL = 1e-10


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("N", [1, 2, 3, 127, 128, 129, 1000, 4096, 10007])
@pytest.mark.parametrize("nrhs", [1, 16])
def test_sizes(N, nrhs):
    # small N: a C2-scaled matrix would put exp(A)V ~ e^-25, below the partial-fraction
    # cancellation floor, so those sizes use an O(1) spectrum
    d, o = workloads.c2_matrix(N, scale=25.0 if N > 100 else 1.0)
    rng = np.random.default_rng(N)
    d = d + rng.uniform(-5, 5, N) * (1.0 if N > 100 else 0.1)  # non-constant diagonal
    o = o * rng.uniform(0.5, 1.5, N - 1)
    V = rng.standard_normal((N, nrhs))
    got = matexp_action(TridiagonalHermitian(d, o), V, ExpOptions(n=24, mode="action")).value
    want = restate.tridiag_action(d, o, V, 24)
    assert got.shape == want.shape
    assert rel(got, want) <= TOL, rel(got, want)


@pytest.mark.parametrize("n", [2, 16, 40, 64])
def test_orders(n):
    N = 3000
    d, o = workloads.c2_matrix(N, scale=2.0)
    V = np.random.default_rng(5).standard_normal((N, 3))
    got = matexp_action(TridiagonalHermitian(d, o), V, ExpOptions(n=n, mode="action")).value
    # two binary64 evaluations of R_n agree to ~eps * sum|a_k| (cancellation of the
    # partial fractions: sum|a_k| = 2.5e3 at n=24, 3.9e8 at n=64)
    from paper_2306_16778_b200.roots import default_table

    floor = 2e-16 * 2 * np.sum(np.abs(default_table(n).coef))
    assert rel(got, restate.tridiag_action(d, o, V, n)) <= max(TOL, floor)


def test_ragged_rhs_tiles():
    N, nrhs = 2000, 37
    d, o = workloads.c2_matrix(N)
    V = np.random.default_rng(6).standard_normal((N, nrhs))
    got = matexp_action(TridiagonalHermitian(d, o), V, ExpOptions(n=24, mode="action")).value
    assert rel(got, restate.tridiag_action(d, o, V, 24)) <= TOL


def test_vector_rhs_and_shift():
    N = 5000
    d, o = workloads.c2_matrix(N, scale=1.0)
    d = d + 3.0  # spectrum in (-1, 3): needs the shift method
    v = np.random.default_rng(7).standard_normal(N)
    T = TridiagonalHermitian(d, o)
    res = matexp_shifted(T, ExpOptions(n=32, mode="action", shift="auto"), v=v)
    c = res.c_applied
    want = np.exp(c) * restate.tridiag_action(d - c, o, v, 32)
    assert res.value.shape == (N,)
    assert rel(res.value, want) <= TOL


def test_c2_full_size_properties():
    """C2 at its BASELINE size: P1 on a column subset vs zgtsv, P2 vs the DST oracle."""
    N, nrhs = workloads.C2["N"], workloads.C2["nrhs"]
    d, o = workloads.c2_matrix()
    V = workloads.c2_rhs()
    got = matexp_action(TridiagonalHermitian(d, o), V, ExpOptions(n=24, mode="action")).value
    cols = [0, 9]
    want = restate.tridiag_action(d, o, V, 24, cols=cols)
    assert rel(got[:, cols], want) <= TOL
    E = closed.dst_exp_lap1d(N, 25.0, V[:, cols])
    assert np.linalg.norm(got[:, cols] - E) <= 10 * np.linalg.norm(want - E)


def test_shift_many_groups_ragged_tiles():
    # host-mode pipelining: 8 row groups (N = 40 chunks), per-group e^c scaling, 2 RHS tiles
    N, nrhs = 10007, 21
    d, o = workloads.c2_matrix(N, scale=1.0)
    d = d + 2.0
    V = np.random.default_rng(11).standard_normal((N, nrhs))
    T = TridiagonalHermitian(d, o)
    res = matexp_shifted(T, ExpOptions(n=24, mode="action", shift="auto"), v=V)
    c = res.c_applied
    assert c != 0.0
    want = np.exp(c) * restate.tridiag_action(d - c, o, V, 24)
    assert rel(res.value, want) <= TOL


@pytest.mark.parametrize("N,nrhs,scale", [(4096, 4, 25.0), (1 << 16, 16, 25.0), (1 << 18, 16, 25.0),
                                          (1 << 16, 3, 0.05), (4096, 4, 1e3), (8192, 3, 1e4)])
def test_host_pipeline_matches_device(N, nrhs, scale):
    """Host-memory calls pipeline the copies by row groups with per-group carries (backward
    carries truncated at the next group, verified by tri_trunc_check, global fallback
    otherwise).  The first four cases (C2-like scales, and scale 0.05) take the truncated
    carries (PFX_TRI_REPORT=1 prints the verdict).  A large scale (|l'| -> 1 when the
    off-diagonal dwarfs every pole) makes tri_trunc_check reject the truncation, so the last two
    cases exercise the global fallback.  Rounding grows with the norm (the oracle differs from
    both paths by as much), so the tolerance scales with it.  Both must agree with the
    device-memory call, which scans the carries globally (and uses longer chunks), to
    rounding."""
    import torch

    from paper_2306_16778_b200 import _native
    from paper_2306_16778_b200.roots import default_table

    d, o = workloads.c2_matrix(N, scale=scale)
    V = np.random.default_rng([N, nrhs]).standard_normal((N, nrhs))
    t2, c2 = default_table(24).interleaved()
    host = _native.expm_tridiag_host(d, o, V, t2, c2, 0.0)
    dev = torch.device("cuda:0")
    devr = _native.expm_tridiag_device(*(torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (d, o, V)), t2,
                                       c2, 0.0).cpu().numpy()
    tol = 5e-14 * max(scale, 20.0)
    assert rel(host, devr) <= tol, rel(host, devr)
