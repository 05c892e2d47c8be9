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


_LOADER_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2306_16778_b200 import (BandedHermitian, ExpOptions, HermitianMatrix, matexp_action, matexp_full,
                                   workloads)
A, _, _ = workloads.random_complex_hermitian(1000, -80.0, 0.0, seed=21)
full = matexp_full(HermitianMatrix(A), ExpOptions(n=12)).value
band = workloads.c5_band_rect(96, 40, scale=300.0)
V = np.random.default_rng(4).standard_normal((96 * 40, 3))
act = matexp_action(BandedHermitian(band), V, ExpOptions(n=16, mode="action")).value
np.savez(sys.argv[2], full=full, act=act)
"""


def test_zgemm_tma_matches_cp_async(tmp_path):
    """The zgemm tiles are staged by TMA (cp.async.bulk.tensor into the padded layout) by
    default; PFX_ZGEMM_CPASYNC=1 stages them with cp.async.  Same arithmetic in the same order,
    so the large dense path (every 64x64 and 32x32 zgemm shape of the LU and substitutions) and
    the band path (the short-K 32-deep variant) give bitwise identical results."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for tag, extra in (("tma", {}), ("cpasync", {"PFX_ZGEMM_CPASYNC": "1"})):
        env = {k: v for k, v in os.environ.items() if k != "PFX_ZGEMM_CPASYNC"}
        env.update(extra)
        path = str(tmp_path / f"{tag}.npz")
        res = subprocess.run([sys.executable, "-c", _LOADER_SCRIPT, root, path], cwd=root, env=env,
                             capture_output=True, text=True, timeout=600)
        assert res.returncode == 0, res.stderr[-2000:]
        outs[tag] = np.load(path)
    assert np.array_equal(outs["tma"]["full"], outs["cpasync"]["full"])
    assert np.array_equal(outs["tma"]["act"], outs["cpasync"]["act"])
    A, _, _ = workloads.random_complex_hermitian(1000, -80.0, 0.0, seed=21)
    assert rel(outs["tma"]["full"], restate.run_tasks_dense(A, None, 12, threads=8)) <= TOL


@pytest.mark.parametrize("d,cplx", [(2304, True), (2112, False)])
def test_host_pipeline_large(d, cplx):
    # d >= 2048 through host memory: the copy-in overlaps the first panel group (column slab first,
    # then row chunks, the first group's update applied chunk by chunk) and the result leaves by
    # L-shaped frontiers during the backward substitution; bitwise the device-memory result
    import torch

    from paper_2306_16778_b200 import _native
    from paper_2306_16778_b200.roots import default_table

    if cplx:
        A, _, _ = workloads.random_complex_hermitian(d, -40.0, 0.0, seed=d)
    else:
        A, _, _ = workloads.random_real_symmetric(d, -40.0, 0.0, seed=d)
    t2, c2 = default_table(8).interleaved()
    host = _native.expm_dense_host(A, None, t2, c2, 0.0)
    dev = _native.expm_dense_device(torch.from_numpy(A).cuda(), None, t2, c2, 0.0).cpu().numpy()
    assert np.array_equal(host, dev)
    want = restate.run_tasks_dense(A, None, 8, threads=8)
    assert rel(host, want) <= TOL, rel(host, want)
