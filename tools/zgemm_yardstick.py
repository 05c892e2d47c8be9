"""Off-path yardstick: cuBLAS ZGEMM (torch.matmul on complex128) on the C4 GEMM shapes, to
bound what the hand-written zgemm could reach.  Not used by the product."""
import torch

torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda")
for (m, n, k, b) in [(4096, 4096, 4096, 1), (3840, 3840, 256, 12), (3840, 3840, 128, 12), (512, 4096, 3584, 12),
                     (512, 4096, 1024, 12), (64, 4096, 448, 12), (512, 2048, 2048, 12)]:
    A = torch.randn(b, m, k, dtype=torch.complex128, device=dev)
    B = torch.randn(b, k, n, dtype=torch.complex128, device=dev)
    C = torch.empty(b, m, n, dtype=torch.complex128, device=dev)
    for _ in range(3):
        torch.matmul(A, B, out=C)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        torch.matmul(A, B, out=C)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"cuBLAS zgemm m={m} n={n} k={k} batch={b}: {ms:.3f} ms, {8.0 * m * n * k * b / ms / 1e9:.1f} TF/s (8mnk)")
