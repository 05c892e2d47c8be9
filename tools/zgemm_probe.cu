// Tight-loop timing of pfx::zgemm on the C4 GEMM shapes (batch 12): the two-panel LU
// trailing update, the super-block backward / forward outer GEMMs and the inner ones.
// Variants are selected by the library's environment switches (PFX_ZGEMM_4M, _W4, ...).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2306_16778_b200/csrc \
//        tools/zgemm_probe.cu paper_2306_16778_b200/csrc/*.cu paper_2306_16778_b200/csrc/poles.cpp -o /tmp/zgp
#include <cstdio>
#include <vector>
#include "zblas.cuh"
using namespace pfx;

int main() {
  const int d = 4096, nsys = 12;
  double2 *M, *X;
  cudaMalloc(&M, (size_t)nsys * d * d * sizeof(double2));
  cudaMalloc(&X, (size_t)nsys * d * d * sizeof(double2));
  cudaMemset(M, 0, (size_t)nsys * d * d * sizeof(double2));
  cudaMemset(X, 0, (size_t)nsys * d * d * sizeof(double2));
  ZMat Mz{M, d, (int64_t)d * d}, Xz{X, d, (int64_t)d * d};
  auto sub = [](ZMat A, int64_t i, int64_t j) { ZMat r = A; r.p = A.p + i * A.ld + j; return r; };
  struct Shape { const char* name; int m, n, k, off; ZMat A, B, C; };
  std::vector<Shape> shapes = {
      {"lu_trail_k256", 3840, 3840, 256, -1, sub(Mz, 256, 0), sub(Mz, 0, 256), sub(Mz, 256, 256)},
      {"lu_trail_k128", 3840, 3840, 128, -1, sub(Mz, 256, 128), sub(Mz, 128, 256), sub(Mz, 256, 256)},
      {"lu_trail_k128_small", 1024, 1024, 128, -1, sub(Mz, 3072, 2944), sub(Mz, 2944, 3072), sub(Mz, 3072, 3072)},
      {"bwd_outer", 512, 4096, 3584, -1, sub(Mz, 0, 512), sub(Xz, 512, 0), sub(Xz, 0, 0)},
      {"bwd_outer_short", 512, 4096, 1024, -1, sub(Mz, 2560, 3072), sub(Xz, 3072, 0), sub(Xz, 2560, 0)},
      {"bwd_inner", 64, 4096, 448, -1, sub(Mz, 0, 64), sub(Xz, 64, 0), sub(Xz, 0, 0)},
      {"fwd_outer", 512, 2048, 2048, 0, sub(Mz, 2048, 0), sub(Xz, 0, 0), sub(Xz, 2048, 0)},
      {"fwd_inner", 64, 1088, 64, 1024, sub(Mz, 1088, 1024), sub(Xz, 1024, 0), sub(Xz, 1088, 0)},
  };
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (auto& sh : shapes) {
    for (int w = 0; w < 2; ++w) zgemm(0, nsys, sh.m, sh.n, sh.k, -1.0, sh.A, sh.B, sh.C, true, sh.off);
    cudaDeviceSynchronize();
    const int reps = 10;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) zgemm(0, nsys, sh.m, sh.n, sh.k, -1.0, sh.A, sh.B, sh.C, true, sh.off);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    double nz = 0;
    for (int c = 0; c < sh.n; ++c) nz += sh.off >= 0 ? std::max(0, sh.k - std::max(0, c - sh.off)) : sh.k;
    const double fl = 8.0 * sh.m * nz * nsys;
    printf("%-20s m=%5d n=%5d k=%5d  %8.3f ms  %6.2f TF/s (8mnk)  %s\n", sh.name, sh.m, sh.n, sh.k, ms, fl / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
