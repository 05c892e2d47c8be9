"""Column split of the dense full mode (pfx_expm_dense_cols; leftover pole pairs
split by inverse columns across the ranks): the partial outputs of a partition of the columns
add up to the unsplit full-mode result (reference engine.py:207-213, one reduce)."""
import numpy as np
import pytest

from oracle import restate
from paper_2306_16778_b200 import _native, workloads
from paper_2306_16778_b200.roots import default_table
from paper_2306_16778_b200.sharding import colsplit_plan

pytestmark = pytest.mark.gpu
TOL = 1e-10


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _sum_over_ranks(A, n, world, host=False):
    import torch

    t2, c2 = default_table(n).interleaved()
    d = A.shape[0]
    dev = torch.device("cuda:0")
    Ad = torch.from_numpy(A).to(dev)
    total = np.zeros((d, d), dtype=A.dtype)
    for r in range(world):
        tasks = colsplit_plan(n // 2, d, r, world)
        idx = [k for k, _, _ in tasks]
        th = np.concatenate([t2[2 * k: 2 * k + 2] for k in idx])
        co = np.concatenate([c2[2 * k: 2 * k + 2] for k in idx])
        rg = [(a, b) for _, a, b in tasks]
        if host:
            total += _native.expm_dense_cols_host(A, th, co, rg)
        else:
            total += _native.expm_dense_cols_device(Ad, th, co, rg).cpu().numpy()
    return total


@pytest.mark.parametrize("d,n,world", [(640, 24, 8), (1024, 24, 5), (1100, 16, 3), (768, 20, 16)])
def test_complex_full_partition_sums_to_reference(d, n, world):
    A, _, _ = workloads.random_complex_hermitian(d, -60.0, 0.0, seed=7, trial=d)
    got = _sum_over_ranks(A, n, world)
    want = restate.run_tasks_dense(A, None, n, threads=8)
    assert rel(got, want) <= TOL, rel(got, want)
    assert np.allclose(got, got.conj().T, atol=1e-12)


def test_real_full_partition_and_host_mode():
    d, n = 704, 16
    A, _, _ = workloads.random_real_symmetric(d, -30.0, 0.0, seed=9)
    want = restate.run_tasks_dense(A, None, n, threads=8)
    got = _sum_over_ranks(A, n, 3)
    assert got.dtype == np.float64 and rel(got, want) <= TOL, rel(got, want)
    got_h = _sum_over_ranks(A, n, 3, host=True)
    assert rel(got_h, want) <= TOL


def test_accumulate_and_whole_ranges_match_unsplit_call():
    import torch

    d, n = 832, 24
    A, _, _ = workloads.random_complex_hermitian(d, -80.0, 0.0, seed=11)
    t2, c2 = default_table(n).interleaved()
    dev = torch.device("cuda:0")
    Ad = torch.from_numpy(A).to(dev)
    ref = _native.expm_dense_device(Ad, None, t2, c2, 0.0).cpu().numpy()
    whole = _native.expm_dense_cols_device(Ad, t2, c2, [(0, d)] * (n // 2)).cpu().numpy()
    assert rel(whole, ref) <= 1e-13, rel(whole, ref)
    # two calls, the second accumulating: pairs 0-5 whole, then pairs 6-11 in two column halves
    out = _native.expm_dense_cols_device(Ad, t2[:12], c2[:12], [(0, d)] * 6)
    _native.expm_dense_cols_device(Ad, t2[12:], c2[12:], [(0, 384)] * 6, out=out, accumulate=True)
    _native.expm_dense_cols_device(Ad, t2[12:], c2[12:], [(384, d)] * 6, out=out, accumulate=True)
    assert rel(out.cpu().numpy(), ref) <= 1e-13


def test_host_mode_accumulate():
    d, n = 640, 8
    A, _, _ = workloads.random_complex_hermitian(d, -20.0, 0.0, seed=17)
    t2, c2 = default_table(n).interleaved()
    ref = _native.expm_dense_host(A, None, t2, c2, 0.0)
    out = _native.expm_dense_cols_host(A, t2[:4], c2[:4], [(0, d)] * 2)
    _native.expm_dense_cols_host(A, t2[4:], c2[4:], [(0, 192), (0, 192)], out=out, accumulate=True)
    _native.expm_dense_cols_host(A, t2[4:], c2[4:], [(192, d), (192, d)], out=out, accumulate=True)
    assert rel(out, ref) <= 1e-13, rel(out, ref)


def test_shift_and_pivot_fallback():
    import torch

    d, n = 640, 16
    A, _, _ = workloads.random_complex_hermitian(d, -40.0, 0.0, seed=13)
    t2, c2 = default_table(n).interleaved()
    dev = torch.device("cuda:0")
    Ad = torch.from_numpy(A).to(dev)
    ref = _native.expm_dense_device(Ad, None, t2, c2, -3.0).cpu().numpy()
    parts = [(0, 256), (256, d)]
    got = sum(_native.expm_dense_cols_device(Ad, t2, c2, [p] * 8, -3.0).cpu().numpy() for p in parts)
    assert rel(got, ref) <= 1e-13
    # interchanges forced: the pivoted blocked LU solves the same column ranges
    _native.set_pivot_mode("always")
    try:
        got_p = sum(_native.expm_dense_cols_device(Ad, t2, c2, [p] * 8, -3.0).cpu().numpy() for p in parts)
    finally:
        _native.set_pivot_mode("checked")
    assert rel(got_p, ref) <= 1e-12


def test_bad_ranges_rejected():
    import torch

    from paper_2306_16778_b200.errors import BadSpec

    d = 640
    A, _, _ = workloads.random_complex_hermitian(d, -10.0, 0.0, seed=1)
    t2, c2 = default_table(4).interleaved()
    Ad = torch.from_numpy(A).to("cuda:0")
    for bad in ([(0, d), (32, d)], [(0, d), (64, 64)], [(0, d), (0, d + 1)]):
        with pytest.raises(BadSpec):
            _native.expm_dense_cols_device(Ad, t2, c2, bad)
    with pytest.raises(BadSpec):  # the small batched path has no column split
        _native.expm_dense_cols_device(Ad[:256, :256].contiguous(), t2, c2, [(0, 256)] * 2)
