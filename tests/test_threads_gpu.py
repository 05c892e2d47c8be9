"""Concurrent calls from several host threads (include/pfx.h "Threading").

The reference documents concurrent shifted solves on one matrix as safe
(/root/reference/pkg/src/pfexpm/linalg.py:1-8 module docstring) and runs its pair tasks on a
thread pool (engine.py:217-224).  ctypes releases the GIL around every library call, so these
threads really do enter libpfx.so at the same time: host-mode calls share the device's staging
slots and device-mode calls its workspace, which the per-device call lock (and the
workspace-free event for stream-ordered device calls) must keep consistent.
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

from paper_2306_16778_b200 import (
    BandedHermitian,
    ExpOptions,
    HermitianMatrix,
    TridiagonalHermitian,
    _native,
    matexp_action,
    shifted_solve,
    workloads,
)
from paper_2306_16778_b200.roots import default_table

pytestmark = pytest.mark.gpu


def _cases():
    cases = []
    for i in range(12):
        d = [40, 130, 256, 600][i % 4]
        A, _, _ = workloads.random_complex_hermitian(d, -20.0, 0.0, seed=31, trial=i)
        V = np.random.default_rng(i).standard_normal((d, 3)) + 1j * np.random.default_rng(i + 99).standard_normal((d, 3))
        cases.append((HermitianMatrix(A), V, complex(-1.5 + 0.1 * i, 2.0 + 0.05 * i)))
    return cases


def test_concurrent_shifted_solve_and_action():
    cases = _cases()
    opts = ExpOptions(n=16, mode="action")

    def work(i):
        H, V, th = cases[i]
        return shifted_solve(H, th, V), matexp_action(H, V[:, 0], opts).value

    seq = [work(i) for i in range(len(cases))]
    with ThreadPoolExecutor(max_workers=6) as pool:
        for _ in range(3):
            par = list(pool.map(work, range(len(cases))))
            for (a0, b0), (a1, b1) in zip(seq, par):
                assert np.array_equal(a0, a1)
                assert np.array_equal(b0, b1)


def test_concurrent_structured_host_calls():
    m = 24
    band = workloads.c5_band(m, scale=2.0)
    d, o = workloads.c2_matrix(5000)
    Vb = np.random.default_rng(1).standard_normal((m * m, 2))
    Vt = np.random.default_rng(2).standard_normal((5000, 4))
    opts = ExpOptions(n=16, mode="action")

    def work(i):
        if i % 2:
            return matexp_action(BandedHermitian(band), Vb, opts).value
        return matexp_action(TridiagonalHermitian(d, o), Vt, opts).value

    seq = [work(i) for i in range(8)]
    with ThreadPoolExecutor(max_workers=4) as pool:
        par = list(pool.map(work, range(8)))
    for a, b in zip(seq, par):
        assert np.array_equal(a, b)


def test_concurrent_device_calls_on_separate_streams():
    """Stream-ordered device calls from two threads on two streams share the workspace; the
    workspace-free event orders them on the GPU."""
    dev = torch.device("cuda:0")
    t2, c2 = default_table(24).interleaved()
    N = 1 << 16
    d, o = workloads.c2_matrix(N)
    dd, od = torch.from_numpy(d).to(dev), torch.from_numpy(o).to(dev)
    Vs = [torch.from_numpy(np.random.default_rng(k).standard_normal((N, 16))).to(dev) for k in range(4)]
    ref = [_native.expm_tridiag_device(dd, od, V, t2, c2, 0.0).cpu().numpy() for V in Vs]
    torch.cuda.synchronize()

    def work(k):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            out = _native.expm_tridiag_device(dd, od, Vs[k], t2, c2, 0.0, stream=s)
        s.synchronize()
        return out.cpu().numpy()

    for _ in range(3):
        with ThreadPoolExecutor(max_workers=4) as pool:
            got = list(pool.map(work, range(4)))
        for a, b in zip(ref, got):
            assert np.array_equal(a, b)
