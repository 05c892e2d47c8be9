"""Worker for tests/test_engine_distributed_gpu.py, run under torchrun with gloo: every rank
calls the public matexp_full / matexp_action with ExpOptions(distributed=True) on the one visible
GPU (the ranks' kernels never wait on one another; only the host-side all-reduce synchronises).
Rank 0 prints the parity against the unsharded call and the CPU restatement as one JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2306_16778_b200 import ExpOptions, HermitianMatrix, matexp_action, matexp_full, workloads  # noqa: E402


def main():
    d, n, cplx = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    torch.cuda.set_device(0)
    if cplx:
        A, _, _ = workloads.random_complex_hermitian(d, -25.0, 0.0, seed=d)
    else:
        A, _, _ = workloads.random_real_symmetric(d, -25.0, 0.0, seed=d)
    H = HermitianMatrix(A)
    full = matexp_full(H, ExpOptions(n=n, distributed=True))
    v = workloads.unit_vector(d, 3)
    act = matexp_action(H, v, ExpOptions(n=n, mode="action", distributed=True))
    if rank == 0:
        from oracle import restate

        rel = lambda a, b: float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))  # noqa: E731
        one = matexp_full(H, ExpOptions(n=n)).value
        print(json.dumps({
            "full_vs_unsharded": rel(full.value, one),
            "full_vs_oracle": rel(full.value, restate.run_tasks_dense(A, None, n, threads=8)),
            "action_vs_oracle": rel(act.value, restate.run_tasks_dense(A, v, n)),
            "times": len(full.per_term_times), "t_para_ok": full.t_para == max(full.per_term_times),
            "dtype": str(full.value.dtype)}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
