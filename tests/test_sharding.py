"""Multi-process pole sharding (world_size 2, gloo, CPU): the sharded sum of per-rank
partials equals the unsharded ascending reduction (the host logic of bench.py --gpus N)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_16778_b200.sharding import pair_range, sharded_run, slice_poles


def test_pair_ranges_cover_in_order():
    for npairs in (1, 8, 10, 12):
        for world in (1, 2, 3, 4, 8):
            got = [pair_range(npairs, r, world) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == npairs
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            sizes = [h - l for l, h in got]
            assert max(sizes) - min(sizes) <= 1


def test_slice_poles():
    t = np.arange(24.0)
    c = -np.arange(24.0)
    ts, cs = slice_poles(t, c, 3, 5)
    assert np.array_equal(ts, t[6:10]) and np.array_equal(cs, c[6:10])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import restate
    from paper_2306_16778_b200 import workloads

    N = 300
    d, o = workloads.c2_matrix(N, scale=2.0)
    V = np.random.default_rng(0).standard_normal((N, 3))
    theta, coef = restate.pairs(24)

    def solve_pairs(lo, hi):
        # per-pair CPU solves standing in for the rank's GPU kernels (gloo test of the plumbing)
        import scipy.linalg.lapack as lapack

        acc = None
        for k in range(lo, hi):
            _, _, _, y, _ = lapack.zgtsv(o.astype(complex), d + theta[k], o.astype(complex), V.astype(complex))
            s = 2.0 * (coef[k] * y).real
            acc = s if acc is None else acc + s
        return torch.from_numpy(acc)

    res = sharded_run(solve_pairs, len(theta), (N, 3), torch.float64, "cpu")
    if rank == 0:
        np.save(out_path, res.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_two_ranks_match_unsharded(tmp_path, world):
    out = str(tmp_path / "res.npy")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    got = np.load(out)
    from oracle import restate
    from paper_2306_16778_b200 import workloads

    N = 300
    d, o = workloads.c2_matrix(N, scale=2.0)
    V = np.random.default_rng(0).standard_normal((N, 3))
    want = restate.tridiag_action(d, o, V, 24)
    assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)


def _engine_worker(rank, world, port, out_path):
    # ExpOptions(distributed=True) through the public API; the rank's GPU call is stood in for
    # by per-pair LAPACK solves over exactly the pole slice the engine hands to the native layer
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2306_16778_b200 import ExpOptions, HermitianMatrix, _native, matexp_full, workloads

    seen = []

    def fake_dense_host(a, V, theta2, coef2, shift_c, per_pair_ms=None, out=None):
        th = theta2[0::2] + 1j * theta2[1::2]
        co = coef2[0::2] + 1j * coef2[1::2]
        seen.append(len(th))
        acc = np.zeros(a.shape)
        for k in range(len(th)):
            X = np.linalg.solve(a - shift_c * np.eye(a.shape[0]) + th[k] * np.eye(a.shape[0]), np.eye(a.shape[0]))
            acc = acc + 2.0 * (co[k] * X).real
            if per_pair_ms is not None:
                per_pair_ms[k] = 1.0 + rank  # ms
        return acc

    _native.expm_dense_host = fake_dense_host
    A, _, _ = workloads.random_real_symmetric(12, -8.0, 0.0, seed=4)
    res = matexp_full(HermitianMatrix(A), ExpOptions(n=12, distributed=True))
    if rank == 0:
        np.save(out_path, res.value)
        np.save(out_path + ".t.npy", np.array(res.per_term_times + (res.t_para,)))
    assert seen == [3]  # 6 pairs over 2 ranks
    dist.barrier()
    dist.destroy_process_group()


def test_engine_distributed_pole_sharding(tmp_path):
    out = str(tmp_path / "eng.npy")
    mp.spawn(_engine_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    from oracle import restate
    from paper_2306_16778_b200 import workloads

    A, _, _ = workloads.random_real_symmetric(12, -8.0, 0.0, seed=4)
    want = restate.run_tasks_dense(A, None, 12)
    got = np.load(out)
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)
    t = np.load(out + ".t.npy")
    assert np.allclose(t[:6], [1e-3] * 3 + [2e-3] * 3) and t[6] == t[:6].max()
