"""Worker for tests/test_tridiag_shard_gpu.py, run under torchrun with gloo: every rank
solves its rows of a tridiagonal exp(A)V through pfx_expm_tridiag_shard (all ranks share the
one visible GPU; their kernels never wait on one another, only the host-side all-gathers
synchronise), rank 0 assembles the rows and prints the parity against the unsharded device
call and the oracle as one JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2306_16778_b200 import _native, workloads  # noqa: E402
from paper_2306_16778_b200.roots import default_table  # noqa: E402


def main():
    N, nrhs, n = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    shift = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    if N >= 4096:
        d, o = workloads.c2_matrix(N)
    else:
        rng = np.random.default_rng(N + nrhs)
        d = -rng.uniform(0.5, 4.0, N)
        o = rng.uniform(-1.0, 1.0, max(N - 1, 0)) * 0.9
    V = np.random.default_rng([0, 0, 1]).standard_normal((N, nrhs))
    t2, c2 = default_table(n).interleaved()
    D, O, Vd = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (d, o, V))

    def allgather(mine):
        parts = [torch.empty(mine.size, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(mine))
        return torch.cat(parts).numpy()

    out = _native.expm_tridiag_shard(D, O, Vd, t2, c2, shift, rank, world, allgather)
    torch.cuda.synchronize()
    r0, r1 = _native.tridiag_shard_rows(N, nrhs, rank, world)
    rows = torch.zeros((N, nrhs), dtype=torch.float64)
    rows[r0:r1] = out[r0:r1].cpu()
    dist.reduce(rows, dst=0)  # disjoint row blocks: the sum assembles them
    spans = [None] * world
    dist.all_gather_object(spans, (r0, r1))
    if rank == 0:
        from oracle import restate

        got = rows.numpy()
        full = _native.expm_tridiag_device(D, O, Vd, t2, c2, shift).cpu().numpy()
        want = restate.tridiag_action(d - shift, o, V, n) * np.exp(shift)
        rel = lambda a, b: float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))  # noqa: E731
        print(json.dumps({"vs_unsharded": rel(got, full), "vs_oracle": rel(got, want), "spans": spans}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
