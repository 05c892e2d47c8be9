// Tight-loop timing of the small block kernels at the C5 block-step shapes (nb = 64,
// batch 8).  Built against the library sources:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2306_16778_b200/csrc \
//        tools/zblas_probe.cu paper_2306_16778_b200/csrc/*.cu paper_2306_16778_b200/csrc/poles.cpp -o /tmp/zp
#include <cstdio>
#include <vector>
#include <random>
#include "zblas.cuh"
using namespace pfx;

// ---- ablation copies of zgetrf_diag_kernel (MODE 0 full, 1 no row updates, 2 barriers only)
template <int MODE>
__global__ void __launch_bounds__(256) lu_var(int nb, ZMat D, int* sing, long long* clk) {
  __shared__ double2 prow[2][128];
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31;
  const int row = tid >> 2, cg = tid & 3;
  prow[tid >> 7][tid & 127] = make_double2(0, 0);
  long long t0 = clock64();
  cplx a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int c = cg + 4 * i;
    if (row < nb && c < nb) a[i] = ld(D.at(b, row, c));
    else a[i] = mk(row == c ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  long long t1 = clock64();
#pragma unroll 1
  for (int q = 0; q < 16; ++q) {
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int j = 4 * q + jj;
      double2* pr = prow[jj & 1];
      if (row == j) {
        if (cg >= jj) st(&pr[cg + 4 * q], a[0]);
#pragma unroll
        for (int i = 1; i < 16; ++i) st(&pr[cg + 4 * (q + i)], a[i]);
      }
      __syncthreads();
      if (MODE == 2) continue;
      const int src = (lane & ~3) | jj;
      cplx aj;
      aj.re = __shfl_sync(0xffffffffu, a[0].re, src);
      aj.im = __shfl_sync(0xffffffffu, a[0].im, src);
      if (MODE == 3) aj = a[0];
      if (MODE >= 5) {
        // branch-free: rows <= j get a zero multiplier (their update is a no-op)
        const bool below = row > j;
        cplx l = cmul(aj, crcp_fast(ld(&pr[j])));
        const cplx lz = below ? l : mk(0, 0);
        const cplx a0 = cfms(a[0], lz, ld(&pr[cg + 4 * q]));
        if (MODE == 5) {
#pragma unroll
          for (int i = 1; i < 16; ++i) a[i] = cfms(a[i], lz, ld(&pr[cg + 4 * (q + i)]));
        }
        a[0] = (below && cg == jj) ? l : (cg > jj ? a0 : a[0]);
      } else if (row > j) {
        const cplx l = MODE == 4 ? cmul(aj, ld(&pr[j])) : cmul(aj, crcp_fast(ld(&pr[j])));
        cplx a0 = a[0];
        if (MODE == 0) {
          a0 = cfms(a[0], l, ld(&pr[cg + 4 * q]));
#pragma unroll
          for (int i = 1; i < 16; ++i) a[i] = cfms(a[i], l, ld(&pr[cg + 4 * (q + i)]));
        }
        a[0] = cg == jj ? l : (cg > jj ? a0 : a[0]);
      }
    }
    const int c = cg + 4 * q;
    if (row < nb && c < nb) *D.at(b, row, c) = make_double2(a[0].re, a[0].im);
#pragma unroll
    for (int i = 0; i < 15; ++i) a[i] = a[i + 1];
    a[15] = mk(0, 0);
  }
  long long t2 = clock64();
  if (tid == 0 && b == 0) { clk[0] = t1 - t0; clk[1] = t2 - t1; }
}


// MODE 0 with explicit 32-bit shared addressing
__global__ void __launch_bounds__(256) lu_sh(int nb, ZMat D, int* sing, long long* clk) {
  __shared__ __align__(16) double2 prow[2][128];
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31;
  const int row = tid >> 2, cg = tid & 3;
  prow[tid >> 7][tid & 127] = make_double2(0, 0);
  const unsigned base = (unsigned)__cvta_generic_to_shared(&prow[0][0]);
  long long t0 = clock64();
  cplx a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int c = cg + 4 * i;
    if (row < nb && c < nb) a[i] = ld(D.at(b, row, c));
    else a[i] = mk(row == c ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  long long t1 = clock64();
#pragma unroll 1
  for (int q = 0; q < 16; ++q) {
    const unsigned qb = base + (unsigned)(cg + 4 * q) * 16u;  // &pr[cg + 4q] in buffer 0
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int j = 4 * q + jj;
      const unsigned pb = qb + (jj & 1) * 128u * 16u;
      if (row == j) {
        if (cg >= jj) sts2(pb, a[0]);
#pragma unroll
        for (int i = 1; i < 16; ++i) sts2(pb + 64u * i, a[i]);
      }
      __syncthreads();
      const int src = (lane & ~3) | jj;
      cplx aj;
      aj.re = __shfl_sync(0xffffffffu, a[0].re, src);
      aj.im = __shfl_sync(0xffffffffu, a[0].im, src);
      if (row > j) {
        const cplx piv = lds2(base + (jj & 1) * 128u * 16u + (unsigned)j * 16u);
        const cplx l = cmul(aj, crcp_fast(piv));
        const cplx a0 = cfms(a[0], l, lds2(pb));
#pragma unroll
        for (int i = 1; i < 16; ++i) a[i] = cfms(a[i], l, lds2(pb + 64u * i));
        a[0] = cg == jj ? l : (cg > jj ? a0 : a[0]);
      }
    }
    const int c = cg + 4 * q;
    if (row < nb && c < nb) *D.at(b, row, c) = make_double2(a[0].re, a[0].im);
#pragma unroll
    for (int i = 0; i < 15; ++i) a[i] = a[i + 1];
    a[15] = mk(0, 0);
  }
  long long t2 = clock64();
  if (tid == 0 && b == 0) { clk[0] = t1 - t0; clk[1] = t2 - t1; }
}


// (a flag-synchronised variant of the diagonal LU -- one SMEM slot and ready flag per pivot
// row, no CTA barriers -- was bitwise identical but slower: 45 vs 36 us; removed)
int main() {
  const int batch = 8, nb = 64, n = 512;
  const size_t dsz = (size_t)batch * nb * nb;
  std::vector<double2> h(dsz);
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  for (int b = 0; b < batch; ++b)
    for (int i = 0; i < nb; ++i)
      for (int j = 0; j < nb; ++j) h[(size_t)b * nb * nb + i * nb + j] = make_double2(0.1 * nd(rng) + (i == j ? 4.0 : 0.0), i == j ? 1.0 : 0.0);
  double2 *D, *D0, *Li, *Ui, *B;
  int* sing;
  cudaMalloc(&D, dsz * 16);
  cudaMalloc(&D0, dsz * 16);
  cudaMalloc(&Li, dsz * 16);
  cudaMalloc(&Ui, dsz * 16);
  cudaMalloc(&B, (size_t)batch * nb * n * 16);
  cudaMalloc(&sing, 4);
  cudaMemcpy(D0, h.data(), dsz * 16, cudaMemcpyHostToDevice);
  cudaMemset(B, 0, (size_t)batch * nb * n * 16);
  ZMat Dm{D, nb, nb * nb}, Lm{Li, nb, nb * nb}, Um{Ui, nb, nb * nb}, Bm{B, n, (int64_t)nb * n}, Bt{B, nb, (int64_t)nb * n};
  cudaStream_t s = 0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto fn) {
    for (int i = 0; i < 5; ++i) fn();
    cudaEventRecord(e0, s);
    const int R = 200;
    for (int i = 0; i < R; ++i) fn();
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s %8.2f us/launch  (%s)\n", name, ms * 1000 / R, cudaGetErrorString(cudaGetLastError()));
  };
  timeit("memcpy D (64 KB x 8)", [&] { cudaMemcpyAsync(D, D0, dsz * 16, cudaMemcpyDeviceToDevice, s); });
  timeit("zgetrf_diag (+memcpy)", [&] {
    cudaMemcpyAsync(D, D0, dsz * 16, cudaMemcpyDeviceToDevice, s);
    zgetrf_diag(s, batch, nb, Dm, sing);
  });
  timeit("ztrtri_diag", [&] { ztrtri_diag(s, batch, nb, Dm, Lm, Um); });
  timeit("ztrmm left 64x512", [&] { ztrmm_inplace(s, batch, nb, n, Lm, Bm, false, false); });
  timeit("ztrmm right 512x64", [&] { ztrmm_inplace(s, batch, nb, n, Um, Bt, true, true); });
  {
    double2 *U, *X;
    cudaMalloc(&U, (size_t)batch * 64 * 640 * 16);
    cudaMalloc(&X, (size_t)batch * 640 * 8 * 16);
    cudaMemset(U, 0, (size_t)batch * 64 * 640 * 16);
    cudaMemset(X, 0, (size_t)batch * 640 * 8 * 16);
    ZMat Um2{U, 640, 64 * 640}, Xa{X + 64 * 8, 8, 640 * 8}, Xb{X, 8, 640 * 8};
    timeit("zgemm back 64x8x512", [&] { zgemm(s, batch, 64, 8, 512, -1.0, Um2, Xa, Xb); });
    ZMat L21{U, 64, 640 * 64}, Xc{X + 64 * 8, 8, 640 * 8};
    timeit("zgemm rhs 512x8x64", [&] { zgemm(s, batch, 512, 8, 64, -1.0, L21, Xb, Xc); });
    timeit("ztrmm rhs 64x8", [&] { ztrmm_inplace(s, batch, nb, 8, Um, Xb, false, true); });
    double2* Mbig;
    cudaMalloc(&Mbig, (size_t)batch * 640 * 1280 * 16);
    cudaMemset(Mbig, 0, (size_t)batch * 640 * 1280 * 16);
    ZMat A21{Mbig + 64 * 1279, 1279, 640 * 1280}, A12{Mbig + 64, 1279, 640 * 1280}, A22{Mbig + 64 * 1279 + 64, 1279, 640 * 1280};
    timeit("zgemm A22 512x512x64", [&] { zgemm(s, batch, 512, 512, 64, -1.0, A21, A12, A22); });
    int lo, hi;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStream_t sh, sl;
    cudaStreamCreateWithPriority(&sh, cudaStreamNonBlocking, hi);
    cudaStreamCreateWithPriority(&sl, cudaStreamNonBlocking, lo);
    cudaEvent_t f0, f1, j1, j2;
    cudaEventCreate(&f0); cudaEventCreate(&f1); cudaEventCreate(&j1); cudaEventCreate(&j2);
    timeit("LU || gemm (hi/lo streams)", [&] {
      cudaEventRecord(f0, s);
      cudaStreamWaitEvent(sh, f0, 0);
      cudaStreamWaitEvent(sl, f0, 0);
      zgemm(sl, batch, 512, 512, 64, -1.0, A21, A12, A22);
      zgetrf_diag(sh, batch, nb, Dm, sing);
      cudaEventRecord(j1, sh);
      cudaEventRecord(j2, sl);
      cudaStreamWaitEvent(s, j1, 0);
      cudaStreamWaitEvent(s, j2, 0);
    });
    timeit("LU+trtri || gemm", [&] {
      cudaEventRecord(f0, s);
      cudaStreamWaitEvent(sh, f0, 0);
      cudaStreamWaitEvent(sl, f0, 0);
      zgemm(sl, batch, 512, 512, 64, -1.0, A21, A12, A22);
      zgetrf_diag(sh, batch, nb, Dm, sing);
      ztrtri_diag(sh, batch, nb, Dm, Lm, Um);
      cudaEventRecord(j1, sh);
      cudaEventRecord(j2, sl);
      cudaStreamWaitEvent(s, j1, 0);
      cudaStreamWaitEvent(s, j2, 0);
    });
    timeit("LU alone (no memcpy)", [&] { zgetrf_diag(s, batch, nb, Dm, sing); });
  }
  {
    // C4 shapes (12 systems): LU trailing update, and the skinny block-row updates of the solves
    const int nb4 = 12, D4 = 4096;
    double2* Mb;
    cudaMalloc(&Mb, (size_t)nb4 * D4 * D4 * 16);
    cudaMemset(Mb, 0, (size_t)nb4 * D4 * D4 * 16);
    ZMat A4{Mb, D4, (int64_t)D4 * D4};
    auto sub4 = [&](int64_t i, int64_t j) { ZMat r = A4; r.p = Mb + i * D4 + j; return r; };
    auto gf = [&](const char* nm, int m, int n, int k, ZMat A, ZMat Bm, ZMat C) {
      for (int i = 0; i < 2; ++i) zgemm(s, nb4, m, n, k, -1.0, A, Bm, C);
      cudaEventRecord(e0, s);
      for (int i = 0; i < 5; ++i) zgemm(s, nb4, m, n, k, -1.0, A, Bm, C);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double t = ms / 5 * 1e-3, fl = 8.0 * m * n * (double)k * nb4;
      printf("%-34s %9.1f us  %6.1f TFLOP/s  (%.0f%% of 36.9)\n", nm, t * 1e6, fl / t / 1e12, fl / t / 1e12 / 36.9 * 100);
    };
    gf("C4 LU update 4032x4032x64", 4032, 4032, 64, sub4(64, 0), sub4(0, 64), sub4(64, 64));
    gf("C4 LU update 2048x2048x64", 2048, 2048, 64, sub4(64, 0), sub4(0, 64), sub4(64, 64));
    gf("C4 fwd 64x2048xK2048", 64, 2048, 2048, sub4(2048, 0), sub4(0, 0), sub4(2048, 0));
    gf("C4 bwd 64x4096xK2048", 64, 4096, 2048, sub4(0, 2048), sub4(2048, 0), sub4(0, 0));
    cudaFree(Mb);
  }
  timeit("zgetf2_panel 64x64 (old)", [&] {
    cudaMemcpyAsync(D, D0, dsz * 16, cudaMemcpyDeviceToDevice, s);
    zgetf2_panel(s, batch, nb, nb, Dm, nullptr, sing);
  });
  long long* clk;
  cudaMallocManaged(&clk, 16);
  timeit("lu_var<0> full", [&] { cudaMemcpyAsync(D, D0, dsz * 16, cudaMemcpyDeviceToDevice, s); lu_var<0><<<batch, 256, 0, s>>>(nb, Dm, sing, clk); });
  cudaDeviceSynchronize(); printf("   clk load %lld loop %lld\n", clk[0], clk[1]);
  timeit("lu_var<1> no update", [&] { cudaMemcpyAsync(D, D0, dsz * 16, cudaMemcpyDeviceToDevice, s); lu_var<1><<<batch, 256, 0, s>>>(nb, Dm, sing, clk); });
  cudaDeviceSynchronize(); printf("   clk load %lld loop %lld\n", clk[0], clk[1]);
  timeit("lu_var<3> no upd, no shfl", [&] { cudaMemcpyAsync(D, D0, dsz * 16, cudaMemcpyDeviceToDevice, s); lu_var<3><<<batch, 256, 0, s>>>(nb, Dm, sing, clk); });
  cudaDeviceSynchronize(); printf("   clk load %lld loop %lld\n", clk[0], clk[1]);
  timeit("lu_var<4> no upd, no rcp", [&] { cudaMemcpyAsync(D, D0, dsz * 16, cudaMemcpyDeviceToDevice, s); lu_var<4><<<batch, 256, 0, s>>>(nb, Dm, sing, clk); });
  cudaDeviceSynchronize(); printf("   clk load %lld loop %lld\n", clk[0], clk[1]);
  timeit("lu_var<5> full branch-free", [&] { cudaMemcpyAsync(D, D0, dsz * 16, cudaMemcpyDeviceToDevice, s); lu_var<5><<<batch, 256, 0, s>>>(nb, Dm, sing, clk); });
  cudaDeviceSynchronize(); printf("   clk load %lld loop %lld\n", clk[0], clk[1]);
  timeit("lu_var<6> no upd branch-free", [&] { cudaMemcpyAsync(D, D0, dsz * 16, cudaMemcpyDeviceToDevice, s); lu_var<6><<<batch, 256, 0, s>>>(nb, Dm, sing, clk); });
  cudaDeviceSynchronize(); printf("   clk load %lld loop %lld\n", clk[0], clk[1]);
  timeit("lu_sh explicit shared", [&] { cudaMemcpyAsync(D, D0, dsz * 16, cudaMemcpyDeviceToDevice, s); lu_sh<<<batch, 256, 0, s>>>(nb, Dm, sing, clk); });
  cudaDeviceSynchronize(); printf("   clk load %lld loop %lld\n", clk[0], clk[1]);
  timeit("lu_var<2> barriers", [&] { cudaMemcpyAsync(D, D0, dsz * 16, cudaMemcpyDeviceToDevice, s); lu_var<2><<<batch, 256, 0, s>>>(nb, Dm, sing, clk); });
  cudaDeviceSynchronize(); printf("   clk load %lld loop %lld\n", clk[0], clk[1]);
  return 0;
}
