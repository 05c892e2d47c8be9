"""Banded path (config C5 shape) on the GPU vs the CPU restatement (zgbsv per pair)."""
import numpy as np
import pytest

from oracle import restate
from paper_2306_16778_b200 import BandedHermitian, ExpOptions, matexp_action, matexp_shifted, workloads

pytestmark = pytest.mark.gpu
TOL = 1e-10


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("m", [3, 8, 20, 70])
def test_lap2d_grid(m):
    # 2-D 5-point Laplacian on m x m (kb = m), spectrum kept O(1..20) so exp(A)V is not tiny
    band = workloads.c5_band(m, scale=2.0)
    V = np.random.default_rng(m).standard_normal((m * m, 3))
    got = matexp_action(BandedHermitian(band), V, ExpOptions(n=16, mode="action")).value
    want = restate.banded_action(band, V, 16)
    assert rel(got, want) <= TOL, rel(got, want)


@pytest.mark.parametrize("N,kb", [(1, 0), (5, 1), (100, 7), (300, 64), (1000, 65), (2000, 130)])
def test_random_bands(N, kb):
    rng = np.random.default_rng(N + kb)
    band = rng.uniform(-1, 1, (kb + 1, N)) * 0.5
    band[0] = -4.0 * (kb + 1) * rng.uniform(0.2, 1.0, N) / max(kb, 1)  # negative-ish diagonal
    V = rng.standard_normal((N, 2))
    got = matexp_action(BandedHermitian(band), V, ExpOptions(n=20, mode="action")).value
    want = restate.banded_action(band, V, 20)
    assert rel(got, want) <= TOL, rel(got, want)


def test_vector_and_shift():
    m = 12
    band = workloads.c5_band(m, scale=1.0)
    band = band.copy()
    band[0] += 5.0  # positive part of the spectrum -> shift method
    v = np.random.default_rng(1).standard_normal(m * m)
    res = matexp_shifted(BandedHermitian(band), ExpOptions(n=32, mode="action", shift="auto"), v=v)
    c = res.c_applied
    sh = band.copy()
    sh[0] -= c
    want = np.exp(c) * restate.banded_action(sh, v[:, None], 32)[:, 0]
    assert rel(res.value, want) <= TOL


def test_c5_shape_scaled_down_vs_dst():
    m = 40
    band = workloads.c5_band(m, scale=50.0 * (m + 1) ** 2 / 513.0**2)  # same spectral scaling as C5 per grid
    V = workloads.c5_rhs(m, 8)
    got = matexp_action(BandedHermitian(band), V, ExpOptions(n=16, mode="action")).value
    want = restate.banded_action(band, V, 16)
    assert rel(got, want) <= TOL


@pytest.mark.parametrize("N,kb,nrhs", [(1500, 600, 1), (1300, 100, 70), (777, 40, 9)])
def test_wide_band_many_rhs(N, kb, nrhs):
    # back substitution: > 16 inner chunks (kb > 512), > 64 right-hand sides (column chunks),
    # and ragged 8-column groups
    rng = np.random.default_rng(N * 7 + kb)
    band = rng.uniform(-1, 1, (kb + 1, N)) * (0.5 / np.sqrt(kb + 1))
    band[0] = -rng.uniform(0.5, 3.0, N)
    V = rng.standard_normal((N, nrhs))
    got = matexp_action(BandedHermitian(band), V, ExpOptions(n=16, mode="action")).value
    want = restate.banded_action(band, V, 16)
    assert rel(got, want) <= TOL, rel(got, want)


@pytest.mark.parametrize("nx,ny,nrhs", [(32, 24, 3), (48, 40, 1), (64, 20, 9), (100, 26, 2)])
def test_two_partition_spike_grids(nx, ny, nrhs):
    """Even N with halves >= 8 kb: the band solve runs as two partitions (SPIKE, the second
    reversed) coupled through their interface rows; the result must match zgbsv on the whole
    band, including grids whose interface region is rounded up to a 64-row block."""
    band = workloads.c5_band_rect(nx, ny, scale=3.0)
    V = np.random.default_rng(nx * 7 + ny).standard_normal((nx * ny, nrhs))
    got = matexp_action(BandedHermitian(band), V, ExpOptions(n=16, mode="action")).value
    want = restate.banded_action(band, V, 16)
    assert rel(got, want) <= TOL, rel(got, want)


def test_two_partition_spike_random_band():
    rng = np.random.default_rng(77)
    N, kb = 3000, 90
    band = rng.uniform(-1, 1, (kb + 1, N)) * (0.5 / np.sqrt(kb + 1))
    band[0] = -rng.uniform(0.5, 3.0, N)
    V = rng.standard_normal((N, 4))
    got = matexp_action(BandedHermitian(band), V, ExpOptions(n=20, mode="action")).value
    want = restate.banded_action(band, V, 20)
    assert rel(got, want) <= TOL, rel(got, want)


@pytest.mark.parametrize("N,kb,spike", [(2560, 256, "0"), (3840, 320, "0"), (6400, 256, "1"), (4096, 512, "0"),
                                        (1024, 448, "0")])
def test_left_looking_far_update(N, kb, spike, monkeypatch):
    # PFX_BD_LL=1 (opt-in), kb and N multiples of 64 with kb >= 256: the far trailing update runs left-looking (one
    # K <= kb - 128 product per L-shaped panel, trapezoidal band edge skipped per tile), with
    # and without the two-partition split; random bands, so every in-band entry is nonzero
    import subprocess
    import sys
    code = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from oracle import restate
from paper_2306_16778_b200 import BandedHermitian, ExpOptions, matexp_action
N, kb = int(sys.argv[2]), int(sys.argv[3])
rng = np.random.default_rng(N + kb)
band = rng.uniform(-1, 1, (kb + 1, N)) * 0.5
band[0] = -4.0 * (kb + 1) * rng.uniform(0.2, 1.0, N) / kb
V = rng.standard_normal((N, 3))
got = matexp_action(BandedHermitian(band), V, ExpOptions(n=12, mode="action")).value
want = restate.banded_action(band, V, 12)
print("REL", float(np.linalg.norm(got - want) / np.linalg.norm(want)))
"""
    import os
    env = dict(os.environ, PFX_BD_SPIKE=spike, PFX_BD_LL="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, "-c", code, root, str(N), str(kb)], env=env, capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    r = float([l for l in res.stdout.splitlines() if l.startswith("REL")][0].split()[1])
    assert r <= TOL, r
