// Shared device helpers for the pfx kernels (sm_100a).
//
// Complex values are interleaved binary64 pairs (double2 {re, im}) in HBM,
// exactly the numpy complex128 layout, so host buffers map 1:1.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/pfx.h"

namespace pfx {

// ---- status / error plumbing (host) -------------------------------------
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
#define PFX_CUDA_TRY(expr)                                                              \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      return ::pfx::fail(PFX_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

// Grow-only device scratch arena, one per (device, slot).  Slots let one call
// hold several live buffers.  Freed by pfx_release().
void* scratch(int slot, size_t bytes);
// a pinned host word per thread for the status readback (a pageable 4-byte copy is staged
// through a driver bounce buffer: tens of microseconds on the small configs)
int* pinned_word();
// wait for `stream`: spin on cudaStreamQuery for up to ~200 us (short calls return without
// the blocking-sync wake-up latency), then fall back to a blocking synchronise
int sync_stream(cudaStream_t stream);
// Row sharding of the tridiagonal path (pfx_expm_tridiag_shard): this process is `rank` of
// `nranks`; allgather(ctx, buf, count) fills buf[j*count, (j+1)*count) with rank j's block.
struct TriShard {
  int rank, nranks;
  int (*allgather)(void* ctx, double* buf, int64_t count);
  void* ctx;
};
int tri_partition(int64_t N, int64_t nrhs, int rank, int nranks, int* L, int* P, int64_t* c0, int64_t* c1);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when `bytes` exceeds what was set
// before for this kernel (the call itself costs host time on every launch otherwise)
// Kept per (kernel, device): the attribute is a per-device property.
int raise_smem_limit(const void* kernel, size_t bytes);
void release_scratch();
// SM count of the current device (cached per device)
int device_sms();
// Every C-ABI entry point holds its device's lock for the whole call: the arena slots,
// staging streams and status words of a device are shared by all calls on it, and every
// call returns synchronised, so one call at a time per device keeps them consistent when
// several host threads call concurrently.
constexpr int kMaxDevices = 16;
int current_device();
// dense pivoting policy (pfx_set_pivot_mode) and the count of checked factorisations that
// had to be redone with interchanges
int pivot_mode();
void note_pivot_fallback();
// status word bits the dense kernels raise (atomicOr): an exactly zero pivot, and a pivot
// that partial pivoting would have exchanged (checked mode)
constexpr int ST_SINGULAR = 1;
constexpr int ST_PIVOT = 2;

// Kernel timing (pfx_prof_enable / pfx_prof_read).  PFX_LAUNCH brackets a launch
// with events when profiling is on; otherwise it is just the launch.
// PFX_LAUNCH_F also records the launch's algorithmic flop count.
bool prof_on();
void prof_mark(const char* name, cudaStream_t stream, bool begin, double flops = 0.0);
// Phase tag (this thread): while a ProfTag is alive, profiled launches are recorded as
// "name@tag" (e.g. zgemm@lu, zgemm@fwd), so the kernel breakdown separates the phases.
void prof_set_tag(const char* tag);
const char* prof_get_tag();
struct ProfTag {
  const char* prev;
  explicit ProfTag(const char* tag) : prev(prof_get_tag()) { prof_set_tag(tag); }
  ~ProfTag() { prof_set_tag(prev); }
};
#define PFX_LAUNCH_F(name, stream, flops, ...)                          \
  do {                                                                  \
    if (::pfx::prof_on()) ::pfx::prof_mark(name, stream, true, flops);  \
    __VA_ARGS__;                                                        \
    if (::pfx::prof_on()) ::pfx::prof_mark(name, stream, false);        \
  } while (0)
#define PFX_LAUNCH(name, stream, ...) PFX_LAUNCH_F(name, stream, 0.0, __VA_ARGS__)

// ---- complex arithmetic (device) -----------------------------------------
struct cplx {
  double re, im;
};

__host__ __device__ __forceinline__ cplx mk(double r, double i) { return cplx{r, i}; }
__host__ __device__ __forceinline__ cplx cadd(cplx a, cplx b) { return cplx{a.re + b.re, a.im + b.im}; }
__host__ __device__ __forceinline__ cplx csub(cplx a, cplx b) { return cplx{a.re - b.re, a.im - b.im}; }
__host__ __device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return cplx{fma(a.re, b.re, -a.im * b.im), fma(a.re, b.im, a.im * b.re)};
}
// a * conj(b)
__host__ __device__ __forceinline__ cplx cmulc(cplx a, cplx b) {
  return cplx{fma(a.re, b.re, a.im * b.im), fma(a.im, b.re, -a.re * b.im)};
}
// c - a*b
__host__ __device__ __forceinline__ cplx cfms(cplx c, cplx a, cplx b) {
  return cplx{fma(-a.re, b.re, fma(a.im, b.im, c.re)), fma(-a.re, b.im, fma(-a.im, b.re, c.im))};
}
// c + a*b
__host__ __device__ __forceinline__ cplx cfma(cplx a, cplx b, cplx c) {
  return cplx{fma(a.re, b.re, fma(-a.im, b.im, c.re)), fma(a.re, b.im, fma(a.im, b.re, c.im))};
}
__host__ __device__ __forceinline__ cplx cconj(cplx a) { return cplx{a.re, -a.im}; }
__host__ __device__ __forceinline__ cplx cscale(cplx a, double s) { return cplx{a.re * s, a.im * s}; }
// 1/z with Smith-style scaling to avoid overflow/underflow of |z|^2
__host__ __device__ __forceinline__ cplx crcp(cplx z) {
  double ar = fabs(z.re), ai = fabs(z.im);
  if (ar >= ai) {
    double r = z.im / z.re;
    double den = 1.0 / fma(z.im, r, z.re);
    return cplx{den, -r * den};
  } else {
    double r = z.re / z.im;
    double den = 1.0 / fma(z.re, r, z.im);
    return cplx{r * den, -den};
  }
}
__host__ __device__ __forceinline__ cplx cdiv(cplx a, cplx b) { return cmul(a, crcp(b)); }

// Fast binary64 reciprocal of a positive normal x: MUFU seed + two Newton steps on the
// FMA pipe (<= 1 ulp).
__device__ __forceinline__ double frcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// 2^(1023 - E(m)) for positive normal m (E = biased exponent): scales m into [1, 2)
// with integer ops only (no frexp/ldexp on the XU pipe).
__device__ __forceinline__ double pow2_inv_scale(double m) {
  long long e = (__double_as_longlong(m) >> 52) & 0x7ff;
  return __longlong_as_double((2046LL - e) << 52);
}
// 1/z = conj(z)/|z|^2 with the fast reciprocal; falls back to the scaled form
// when |z|^2 leaves the comfortable exponent range.
__device__ __forceinline__ cplx crcp_fast(cplx z) {
  double n = fma(z.re, z.re, z.im * z.im);
  if (!(n > 1e-280 && n < 1e280)) return crcp(z);
  double r = frcp(n);
  return cplx{z.re * r, -z.im * r};
}
__device__ __forceinline__ cplx cdiv_fast(cplx a, cplx b) { return cmul(a, crcp_fast(b)); }
// 1/z without the range guard: only for values known to be well inside the normal range
// (rescaled continuants, shifted pivots with |z| >= Im(theta) > 0)
__device__ __forceinline__ cplx crcp_nc(cplx z) {
  const double r = frcp(fma(z.re, z.re, z.im * z.im));
  return cplx{z.re * r, -z.im * r};
}
__host__ __device__ __forceinline__ double cabs1(cplx a) { return fabs(a.re) + fabs(a.im); }

__device__ __forceinline__ cplx ld(const double2* p) {
  double2 v = *p;
  return cplx{v.x, v.y};
}
__device__ __forceinline__ void st(double2* p, cplx v) { *p = make_double2(v.re, v.im); }
// explicit shared-window accesses by 32-bit address (keeps the window-base computation
// out of latency-critical loops)
__device__ __forceinline__ cplx lds2(unsigned addr) {
  double x, y;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(addr));
  return cplx{x, y};
}
__device__ __forceinline__ void sts2(unsigned addr, cplx v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(v.re), "d"(v.im));
}

// ---- FP64 tensor core (DMMA) ---------------------------------------------
// D(8x8) += A(8x4, row) * B(4x8, col), binary64.  Fragment ownership for lane l,
// g = l>>2, t = l&3:  a = A[g][t], b = B[t][g], c0 = C[g][2t], c1 = C[g][2t+1].
// ptxas lowers this to one native DMMA.8x8x4 on sm_100a.
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Complex 8x8x4 tile product C += A*B on four real DMMAs.
//   Cr += Ar*Br - Ai*Bi,   Ci += Ar*Bi + Ai*Br
__device__ __forceinline__ void zmma884(double (&cr)[2], double (&ci)[2], double ar, double ai, double br,
                                        double bi) {
  dmma884(cr[0], cr[1], ar, br);
  dmma884(cr[0], cr[1], -ai, bi);
  dmma884(ci[0], ci[1], ar, bi);
  dmma884(ci[0], ci[1], ai, br);
}

// ---- async copies (LDGSTS) ---------------------------------------------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace pfx
