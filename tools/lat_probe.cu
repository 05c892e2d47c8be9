// Dependent-chain latency probe (cycles per op) for the FP64 / shuffle / shared-memory ops the
// small-block kernels chain together.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(double* out, long long* cyc, double seed) {
  __shared__ double sh[64];
  double x = seed, y = seed * 0.5;
  if (threadIdx.x < 64) sh[threadIdx.x] = seed;
  __syncthreads();
  const int N = 1024;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = fma(x, 0.999999, 1e-9);
  t1 = clock64();
  cyc[0] = t1 - t0;
  // DMUL chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) y = y * 1.0000001;
  t1 = clock64();
  cyc[1] = t1 - t0;
  // rcp.approx.ftz.f64 chain
  double z = 1.5;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    double r;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(z));
    z = r;
  }
  t1 = clock64();
  cyc[2] = t1 - t0;
  // shfl chain (32-bit)
  int v = threadIdx.x;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) v = __shfl_sync(0xffffffffu, v, (v + 1) & 31);
  t1 = clock64();
  cyc[3] = t1 - t0;
  // LDS chain (dependent index)
  int idx = threadIdx.x & 63;
  double w = 0;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    w = sh[idx];
    idx = ((int)w + i) & 63;
  }
  t1 = clock64();
  cyc[4] = t1 - t0;
  // full fp64 divide
  double q = 3.0;
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N / 8; ++i) q = 1.0 / (q + 1.0);
  t1 = clock64();
  cyc[5] = (t1 - t0) * 8;
  // __syncthreads round trip (256 threads)
  t0 = clock64();
  for (int i = 0; i < N; ++i) __syncthreads();
  t1 = clock64();
  cyc[6] = t1 - t0;
  out[threadIdx.x] = x + y + z + v + w + q;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 256 * sizeof(double));
  cudaMallocManaged(&cyc, 8 * sizeof(long long));
  probe<<<1, 256>>>(out, cyc, 1.25);
  cudaDeviceSynchronize();
  probe<<<1, 256>>>(out, cyc, 1.25);
  cudaDeviceSynchronize();
  const char* names[] = {"DFMA", "DMUL", "rcp.approx.f64", "SHFL", "LDS(dep)", "fp64 div (1/x)", "bar.sync(256thr)"};
  for (int i = 0; i < 7; ++i) printf("%-18s %6.1f cycles\n", names[i], cyc[i] / 1024.0);
  return 0;
}
