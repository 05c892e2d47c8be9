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


def reduce_partials(local, group=None, dst: int = 0):
    """Sum the ranks' partial results onto `dst` with ONE collective (torch.distributed.reduce).

    `local` is a torch tensor (CUDA for NCCL, CPU for gloo); it is reduced in place.  A rank
    that owns no pairs must pass zeros of the same shape."""
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.reduce(local, dst=dst, op=dist.ReduceOp.SUM, group=group)
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
