"""Pole-pair sharding across GPUs: one process per GPU, each rank solves a
contiguous ascending block of the n/2 conjugate pole pairs, and the partial sums meet in a
single reduce over the process group (NCCL over NVLink on GPUs; gloo in CPU tests).

The pairs are independent (reference engine.py:194-215), so the only exchange of the
path is the final sum (engine.py:226-228).  Within a rank the pairs are summed in
ascending order by the kernels; across ranks the collective adds the rank partials, so
results are bitwise reproducible for a fixed rank count.
"""
from __future__ import annotations

import numpy as np


def pair_range(npairs: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous ascending block [lo, hi) of pole pairs owned by `rank` (balanced to +-1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank/world {rank}/{world}")
    return rank * npairs // world, (rank + 1) * npairs // world


def slice_poles(theta2: np.ndarray, coef2: np.ndarray, lo: int, hi: int):
    """Interleaved (re, im) pole/residue arrays restricted to pairs [lo, hi)."""
    return np.ascontiguousarray(theta2[2 * lo: 2 * hi]), np.ascontiguousarray(coef2[2 * lo: 2 * hi])


def _col_cost(u: float) -> float:
    """Cost of the inverse columns [0, u d) of one pair in units of d^3 (complex full mode):
    a column at c takes a forward substitution over the rows below it, (1 - c/d)^2, and a
    backward substitution over every row, 1."""
    return (1.0 - (1.0 - u) ** 3) / 3.0 + u


def colsplit_plan(npairs: int, d: int, rank: int, world: int, align: int = 64):
    """Pole sharding with the leftover pairs split by columns (dense full mode).

    Each rank takes npairs // world whole pairs (contiguous, ascending).  The ranks are then
    dealt over the npairs % world leftover pairs (the first world % rem of them get one rank
    more), and each leftover pair's inverse columns are cut into as many pieces of equal
    substitution cost as it has ranks (cut points rounded to `align`), so a rank factors at most
    one extra pair.  Returns this rank's [(pair, c0, c1), ...] in ascending pair order, whole
    pairs as (k, 0, d).  Every pair's ranges over all ranks partition [0, d) exactly."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank/world {rank}/{world}")
    base, rem = divmod(npairs, world)
    tasks = [(k, 0, d) for k in range(rank * base, (rank + 1) * base)]
    if rem == 0:
        return tasks
    total = _col_cost(1.0)

    def cut(frac: float) -> int:
        """Column below which `frac` of one pair's substitution cost lies."""
        if frac <= 0.0:
            return 0
        if frac >= 1.0:
            return d
        lo, hi = 0.0, 1.0
        for _ in range(60):
            mid = 0.5 * (lo + hi)
            if _col_cost(mid) < frac * total:
                lo = mid
            else:
                hi = mid
        return min(max(int(round(hi * d / align)) * align, 0), d)

    # ranks per leftover pair, then this rank's (pair, piece)
    g, extra = divmod(world, rem)
    first = world * base
    r = rank
    for p in range(rem):
        gp = g + (1 if p < extra else 0)
        if r < gp:
            c0, c1 = cut(r / gp), cut((r + 1) / gp)
            if r == gp - 1:
                c1 = d
            if c1 > c0:
                tasks.append((first + p, c0, c1))
            break
        r -= gp
    return tasks


def reduce_partials(local, group=None, dst: int = 0):
    """Sum the ranks' partial results onto `dst` with ONE collective (torch.distributed.reduce).

    `local` is a torch tensor (CUDA for NCCL, CPU for gloo); it is reduced in place.  A rank
    that owns no pairs must pass zeros of the same shape."""
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size(group) > 1:
        import torch

        # complex partials go through the collective as their (re, im) float64 view (same memory)
        buf = torch.view_as_real(local) if local.is_complex() else local
        dist.reduce(buf, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return local


def sharded_run(solve_pairs, npairs: int, shape, dtype, device, group=None):
    """Run `solve_pairs(lo, hi) -> tensor` on this rank's pairs and reduce to rank 0.

    Returns the full sum on rank 0 and this rank's (reduced-in-place) buffer elsewhere."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    lo, hi = pair_range(npairs, rank, world)
    if hi > lo:
        local = solve_pairs(lo, hi).to(device=device, dtype=dtype).contiguous()
    else:
        local = torch.zeros(shape, dtype=dtype, device=device)
    return reduce_partials(local, group=group)
