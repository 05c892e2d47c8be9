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


def test_colsplit_plan_partitions_every_pair():
    from paper_2306_16778_b200.sharding import colsplit_plan

    for npairs, d in ((12, 4096), (10, 1024), (8, 640), (5, 2048)):
        for world in (1, 2, 3, 4, 5, 7, 8, 16):
            plans = [colsplit_plan(npairs, d, r, world) for r in range(world)]
            cover = {}
            for tasks in plans:
                assert [k for k, _, _ in tasks] == sorted(k for k, _, _ in tasks)  # ascending pairs
                for k, a, b in tasks:
                    assert 0 <= a < b <= d and a % 64 == 0
                    cover.setdefault(k, []).append((a, b))
            assert sorted(cover) == list(range(npairs))
            for k, iv in cover.items():
                iv.sort()
                assert iv[0][0] == 0 and iv[-1][1] == d
                assert all(x[1] == y[0] for x, y in zip(iv, iv[1:]))
            # whole pairs are dealt evenly; a rank factors at most one pair beyond them
            whole = [sum(1 for k, a, b in t if k < (npairs // world) * world) for t in plans]
            assert max(whole) == min(whole) == npairs // world
            assert all(len(t) <= npairs // world + 1 for t in plans)
    # 12 pairs on 8 ranks (C4): one whole pair + one cost-balanced part of a shared pair each
    p = [colsplit_plan(12, 4096, r, 8) for r in range(8)]
    assert p[0] == [(0, 0, 4096), (8, 0, 1664)] and p[1] == [(1, 0, 4096), (8, 1664, 4096)]


def _colsplit_worker(rank, world, port, out_path):
    # the column-split partials (P + P^H on this rank's columns of each leftover pair) meet in one
    # reduce; per-pair LAPACK solves stand in for the rank's pfx_expm_dense_cols call
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import restate
    from paper_2306_16778_b200 import workloads
    from paper_2306_16778_b200.sharding import colsplit_plan, reduce_partials

    d, n = 128, 6
    A, _, _ = workloads.random_complex_hermitian(d, -12.0, 0.0, seed=2)
    theta, coef = restate.pairs(n)
    acc = np.zeros((d, d), dtype=complex)
    for k, c0, c1 in colsplit_plan(n // 2, d, rank, world):
        E = np.eye(d)[:, c0:c1]
        P = np.zeros((d, d), dtype=complex)
        P[:, c0:c1] = coef[k] * np.linalg.solve(A + theta[k] * np.eye(d), E)
        acc += P + P.conj().T
    res = reduce_partials(torch.from_numpy(acc))
    if rank == 0:
        np.save(out_path, res.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_colsplit_two_ranks_match_unsharded(tmp_path):
    out = str(tmp_path / "cs.npy")
    mp.spawn(_colsplit_worker, args=(2, _free_port(), out), nprocs=2, join=True)  # 3 pairs on 2 ranks
    from oracle import restate
    from paper_2306_16778_b200 import workloads

    A, _, _ = workloads.random_complex_hermitian(128, -12.0, 0.0, seed=2)
    want = restate.run_tasks_dense(A, None, 6)
    got = np.load(out)
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


def _engine_colsplit_worker(rank, world, port, out_path):
    # ExpOptions(distributed=True), full mode, d > 512, 3 pairs on 2 ranks: the engine hands the
    # native layer this rank's colsplit_plan tasks; LAPACK solves stand in for the GPU call
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2306_16778_b200 import ExpOptions, HermitianMatrix, _native, matexp_full, workloads
    from paper_2306_16778_b200.sharding import colsplit_plan

    seen = []

    def fake_cols_host(a, theta2, coef2, col_ranges, shift_c=0.0, out=None, accumulate=False):
        th = theta2[0::2] + 1j * theta2[1::2]
        co = coef2[0::2] + 1j * coef2[1::2]
        d = a.shape[0]
        seen.append([tuple(r) for r in col_ranges])
        acc = np.zeros((d, d), dtype=complex)
        for k, (c0, c1) in enumerate(col_ranges):
            P = np.zeros((d, d), dtype=complex)
            P[:, c0:c1] = co[k] * np.linalg.solve(a + (th[k] - shift_c) * np.eye(d), np.eye(d)[:, c0:c1])
            acc += P + P.conj().T
        return acc

    _native.expm_dense_cols_host = fake_cols_host
    A, _, _ = workloads.random_complex_hermitian(576, -6.0, 0.0, seed=8)
    res = matexp_full(HermitianMatrix(A), ExpOptions(n=6, distributed=True))
    assert seen == [[(a, b) for _, a, b in colsplit_plan(3, 576, rank, world)]]
    if rank == 0:
        np.save(out_path, res.value)
        assert len(res.per_term_times) == 3 and min(res.per_term_times) > 0
    dist.barrier()
    dist.destroy_process_group()


def test_engine_distributed_colsplit_full_mode(tmp_path):
    out = str(tmp_path / "engcs.npy")
    mp.spawn(_engine_colsplit_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    from oracle import restate
    from paper_2306_16778_b200 import workloads

    A, _, _ = workloads.random_complex_hermitian(576, -6.0, 0.0, seed=8)
    want = restate.run_tasks_dense(A, None, 6)
    got = np.load(out)
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)
