// Real symmetric tridiagonal shifted solves with fused residue combine (config C2).
//
// The reference is dense-only; this follows its per-pair task and
// combine (engine.py:194-201: M = T - cI + theta_k I, y = M^{-1} V, 2 Re(a_k y))
// and ascending pair reduction (engine.py:226-228) with a structure-aware solver.
//
// Method: twisted factorisation, no pivoting (safe: every pivot of T + theta I
// has |Im| >= Im theta, SURVEY finding 7).  For M = T + theta I with diagonal
// b_i and off-diagonal e_i:
//   forward  (LU) pivots u_i  = b_i - e_{i-1}^2 / u_{i-1},  l_i  = e_{i-1}/u_{i-1}
//   backward (UL) pivots u'_i = b_i - e_i^2 / u'_{i+1},     l'_i = e_i/u'_{i+1}
//   forward  RHS g_i  = f_i - l_i  g_{i-1}
//   backward RHS g'_i = f_i - l'_i g'_{i+1}
//   x_i = (g_i + g'_i - f_i) / gamma_i,   gamma_i = u_i + u'_i - b_i
// (add the eliminated row equations from above and below and subtract row i).
// Both sweeps are first-order streaming recurrences, so no per-row RHS state
// has to be stored between them, and the combine 2 Re(a x_i) splits into a
// forward and a backward part.
//
// Parallel structure (N = 2^20 rows, 12 shifts, 16 RHS for C2):
//   K_T1 tri_mobius_chunks   per (chunk, shift): 2x2 Moebius transfer of the pivot
//                            recurrence over the chunk, both directions.
//   K_T2 tri_mobius_scan     per (shift, direction): block scan of the transfers ->
//                            exact pivot carry-in of every chunk.
//   K_T3 tri_local           per chunk: pivots, l, l', w = 2a/gamma in shared memory;
//                            forward and backward RHS sweeps with zero RHS carry-in;
//                            combine summed over shifts into out; per-chunk carry
//                            summaries.
//   K_T4 tri_carry_scan      per (shift, rhs, direction): affine scan over chunks ->
//                            true RHS carry-ins G (from above), G' (from below).
//   K_T5 tri_correct         per chunk: out_i += sum_k 2 Re(w (Lambda_i G + Lambda'_i G')),
//                            Lambda = running product of -l (resp. -l') from the chunk edge.
#include <algorithm>

#include "pfx_common.cuh"

namespace pfx {

constexpr int TR_L = 128;     // rows per chunk
constexpr int TR_RT = 16;     // RHS per tile (threads per shift)
constexpr int TR_KG = 16;     // max shifts per pass
constexpr int TR_WIN = 8;     // rows per combine window
constexpr int TR_SCAN_T = 512;

struct TriArgs {
  const double* diag;
  const double* off;
  int64_t N;
  const double* V;
  int nrhs;
  double c;
  const double2* theta;
  const double2* coef;
  int npairs;
  int P;  // chunks
  double2* Tf;  // P x npairs x 4   forward transfers
  double2* Tb;  // P x npairs x 4   backward transfers
  double2* rho_in;   // P x npairs  forward pivot carry: 1/u_{s-1} (0 for chunk 0)
  double2* rhob_in;  // P x npairs  backward pivot carry: 1/u'_{e}  (0 for last chunk)
  double2* gF;  // P x npairs x nrhs   forward zero-carry RHS at the chunk's last row
  double2* gB;  // P x npairs x nrhs   backward zero-carry RHS at the chunk's first row
  double2* LF;  // P x npairs          prod(-l) over the chunk
  double2* LB;  // P x npairs          prod(-l') over the chunk
  double2* G;   // P x npairs x nrhs   true forward carry-in g_{s-1}
  double2* Gb;  // P x npairs x nrhs   true backward carry-in g'_{e}
  double* out;  // N x nrhs
};

__device__ __forceinline__ double off2(const double* off, int64_t N, int64_t i) {
  // e_i^2 for the coupling between rows i and i+1 (0 outside the matrix)
  if (i < 0 || i >= N - 1) return 0.0;
  double e = off[i];
  return e * e;
}

// 2x2 complex matrix as 4 cplx: [m0 m1; m2 m3]
struct M22 {
  cplx m0, m1, m2, m3;
};

__device__ __forceinline__ M22 mmul(const M22& a, const M22& b) {
  M22 r;
  r.m0 = cadd(cmul(a.m0, b.m0), cmul(a.m1, b.m2));
  r.m1 = cadd(cmul(a.m0, b.m1), cmul(a.m1, b.m3));
  r.m2 = cadd(cmul(a.m2, b.m0), cmul(a.m3, b.m2));
  r.m3 = cadd(cmul(a.m2, b.m1), cmul(a.m3, b.m3));
  return r;
}

// exact power-of-two rescale so the largest |component| is in [1, 2)
__device__ __forceinline__ void mnorm(M22& a) {
  double mx = fmax(fmax(fmax(cabs1(a.m0), cabs1(a.m1)), fmax(cabs1(a.m2), cabs1(a.m3))), 1e-300);
  int ex;
  frexp(mx, &ex);
  double s = ldexp(1.0, 1 - ex);
  a.m0 = cscale(a.m0, s);
  a.m1 = cscale(a.m1, s);
  a.m2 = cscale(a.m2, s);
  a.m3 = cscale(a.m3, s);
}

__device__ __forceinline__ M22 mident() { return M22{mk(1, 0), mk(0, 0), mk(0, 0), mk(1, 0)}; }

// ---------------------------------------------------------------------------
// K_T1: transfer matrices.  Forward: (u_i; 1) ~ [b_i, -e_{i-1}^2; 1, 0] (u_{i-1}; 1).
// Backward: (u'_i; 1) ~ [b_i, -e_i^2; 1, 0] (u'_{i+1}; 1).
__global__ void tri_mobius_chunks(TriArgs a) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)a.P * a.npairs * 2;
  if (tid >= total) return;
  const int dir = (int)(tid & 1);
  const int64_t ck = tid >> 1;
  const int k = (int)(ck % a.npairs);
  const int64_t cidx = ck / a.npairs;
  const int64_t s = cidx * TR_L, e = (s + TR_L < a.N ? s + TR_L : a.N);
  const cplx th = ld(&a.theta[k]);
  M22 T = mident();
  int cnt = 0;
  if (dir == 0) {
    for (int64_t i = s; i < e; ++i) {
      cplx b = mk(a.diag[i] - a.c + th.re, th.im);
      double e2 = off2(a.off, a.N, i - 1);
      M22 r;
      r.m0 = csub(cmul(b, T.m0), cscale(T.m2, e2));
      r.m1 = csub(cmul(b, T.m1), cscale(T.m3, e2));
      r.m2 = T.m0;
      r.m3 = T.m1;
      T = r;
      if (((++cnt) & 7) == 0) mnorm(T);
    }
  } else {
    for (int64_t i = e - 1; i >= s; --i) {
      cplx b = mk(a.diag[i] - a.c + th.re, th.im);
      double e2 = off2(a.off, a.N, i);
      M22 r;
      r.m0 = csub(cmul(b, T.m0), cscale(T.m2, e2));
      r.m1 = csub(cmul(b, T.m1), cscale(T.m3, e2));
      r.m2 = T.m0;
      r.m3 = T.m1;
      T = r;
      if (((++cnt) & 7) == 0) mnorm(T);
    }
  }
  mnorm(T);
  double2* dst = (dir == 0 ? a.Tf : a.Tb) + ck * 4;
  st(&dst[0], T.m0);
  st(&dst[1], T.m1);
  st(&dst[2], T.m2);
  st(&dst[3], T.m3);
}

// ---------------------------------------------------------------------------
// K_T2: per (shift, direction) block scan.  Chunk order is reversed for the
// backward direction.  Carry of chunk c = pivot reciprocal entering it:
// state vector v = (num; den) with u = num/den, rho = den/num; start (1; 0).
__global__ void __launch_bounds__(TR_SCAN_T) tri_mobius_scan(TriArgs a) {
  __shared__ M22 sm[TR_SCAN_T];
  const int k = blockIdx.x >> 1, dir = blockIdx.x & 1;
  const int P = a.P;
  const int per = (P + TR_SCAN_T - 1) / TR_SCAN_T;
  const int t = threadIdx.x;
  const double2* Tsrc = dir == 0 ? a.Tf : a.Tb;
  double2* dst = dir == 0 ? a.rho_in : a.rhob_in;
  // composite of this thread's range (in processing order)
  M22 acc = mident();
  for (int j = 0; j < per; ++j) {
    int q = t * per + j;
    if (q >= P) break;
    int c = dir == 0 ? q : P - 1 - q;
    const double2* src = Tsrc + ((int64_t)c * a.npairs + k) * 4;
    M22 T{ld(&src[0]), ld(&src[1]), ld(&src[2]), ld(&src[3])};
    acc = mmul(T, acc);
    mnorm(acc);
  }
  sm[t] = acc;
  __syncthreads();
  // Hillis-Steele inclusive scan: S_t = A_t * A_{t-1} * ... * A_0
  for (int off = 1; off < TR_SCAN_T; off <<= 1) {
    M22 mine = sm[t];
    M22 other = t >= off ? sm[t - off] : mident();
    __syncthreads();
    if (t >= off) {
      M22 r = mmul(mine, other);
      mnorm(r);
      sm[t] = r;
    }
    __syncthreads();
  }
  M22 pre = t > 0 ? sm[t - 1] : mident();
  // state entering this thread's range
  cplx vn = pre.m0, vd = pre.m2;  // pre * (1; 0)
  for (int j = 0; j < per; ++j) {
    int q = t * per + j;
    if (q >= P) break;
    int c = dir == 0 ? q : P - 1 - q;
    // rho = den / num
    cplx rho = (vn.re == 0.0 && vn.im == 0.0) ? mk(0, 0) : cdiv(vd, vn);
    if (q == 0) rho = mk(0, 0);
    st(&dst[(int64_t)c * a.npairs + k], rho);
    const double2* src = Tsrc + ((int64_t)c * a.npairs + k) * 4;
    M22 T{ld(&src[0]), ld(&src[1]), ld(&src[2]), ld(&src[3])};
    cplx nn = cadd(cmul(T.m0, vn), cmul(T.m1, vd));
    cplx nd = cadd(cmul(T.m2, vn), cmul(T.m3, vd));
    double mx = fmax(fmax(cabs1(nn), cabs1(nd)), 1e-300);
    int ex;
    frexp(mx, &ex);
    double s = ldexp(1.0, 1 - ex);
    vn = cscale(nn, s);
    vd = cscale(nd, s);
  }
}

// ---------------------------------------------------------------------------
// Shared-memory factor data of one chunk for a group of shifts.
struct TriSmem {
  double dg[TR_L];            // diag - c
  double of[TR_L + 1];        // of[i] = e_{s-1+i}  (coupling rows s-1+i, s+i), 0 outside
  double2 l[TR_KG][TR_L];     // forward multipliers
  double2 lb[TR_KG][TR_L];    // backward multipliers
  double2 w[TR_KG][TR_L];     // 2 a / gamma (or w*Lambda in the correction kernel)
  double2 wb[TR_KG][TR_L];    // correction kernel only: w*Lambda'
  double cbuf[TR_KG][TR_WIN][TR_RT];
  double F[TR_L][TR_RT];
  double2 lam[TR_KG][2];      // chunk products / carries
};

// Pivot chains for shift slot kk (thread-level, serial in rows), writing l / lb,
// and (want_lambda) the running products Lambda into w / wb.
__device__ void tri_chain(TriSmem& S, const TriArgs& a, int64_t c, int k, int kk, int dir, int rows,
                          bool want_lambda) {
  const cplx th = ld(&a.theta[k]);
  if (dir == 0) {
    cplx rho = ld(&a.rho_in[c * a.npairs + k]);
    cplx lam = mk(1, 0);
    for (int i = 0; i < rows; ++i) {
      cplx b = mk(S.dg[i] + th.re, th.im);
      double e = S.of[i];
      cplx l = cscale(rho, e);
      cplx u = csub(b, cscale(l, e));
      rho = crcp(u);
      S.l[kk][i] = make_double2(l.re, l.im);
      lam = cmul(lam, mk(-l.re, -l.im));
      if (want_lambda) S.w[kk][i] = make_double2(lam.re, lam.im);
    }
    S.lam[kk][0] = make_double2(lam.re, lam.im);
  } else {
    cplx rho = ld(&a.rhob_in[c * a.npairs + k]);
    cplx lam = mk(1, 0);
    for (int i = rows - 1; i >= 0; --i) {
      cplx b = mk(S.dg[i] + th.re, th.im);
      double e = S.of[i + 1];
      cplx l = cscale(rho, e);
      cplx u = csub(b, cscale(l, e));
      rho = crcp(u);
      S.lb[kk][i] = make_double2(l.re, l.im);
      lam = cmul(lam, mk(-l.re, -l.im));
      if (want_lambda) S.wb[kk][i] = make_double2(lam.re, lam.im);
    }
    S.lam[kk][1] = make_double2(lam.re, lam.im);
  }
}

__device__ void tri_load_chunk(TriSmem& S, const TriArgs& a, int64_t s, int rows) {
  for (int i = threadIdx.x; i < rows; i += blockDim.x) S.dg[i] = a.diag[s + i] - a.c;
  for (int i = threadIdx.x; i <= rows; i += blockDim.x) {
    int64_t gi = s - 1 + i;  // coupling (gi, gi+1)
    S.of[i] = (gi >= 0 && gi < a.N - 1) ? a.off[gi] : 0.0;
  }
}

// gamma / w for all (kk, i) of the chunk
__device__ void tri_weights(TriSmem& S, const TriArgs& a, int k0, int kg, int rows, double2 (*dst)[TR_L]) {
  for (int e = threadIdx.x; e < kg * rows; e += blockDim.x) {
    int kk = e / rows, i = e - kk * rows;
    const cplx th = ld(&a.theta[k0 + kk]);
    cplx b = mk(S.dg[i] + th.re, th.im);
    cplx l = ld(&S.l[kk][i]), lb = ld(&S.lb[kk][i]);
    // gamma = b - e_{i-1} l_i - e_i l'_i
    cplx gam = csub(csub(b, cscale(l, S.of[i])), cscale(lb, S.of[i + 1]));
    cplx co = ld(&a.coef[k0 + kk]);
    cplx w = cscale(cdiv(co, gam), 2.0);
    dst[kk][i] = make_double2(w.re, w.im);
  }
}

// K_T3 ------------------------------------------------------------------------
__global__ void __launch_bounds__(TR_RT* TR_KG) tri_local(TriArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TriSmem& S = *reinterpret_cast<TriSmem*>(smem_raw);
  const int64_t c = blockIdx.x;
  const int r0 = blockIdx.y * TR_RT;
  const int64_t s = c * TR_L;
  const int rows = (int)(TR_L < a.N - s ? TR_L : a.N - s);
  const int t = threadIdx.x;
  const int r = t % TR_RT;       // rhs lane
  const int kk = t / TR_RT;      // shift slot
  const int rg = r0 + r;
  const bool rv = rg < a.nrhs;
  tri_load_chunk(S, a, s, rows);
  for (int i = t; i < rows * TR_RT; i += blockDim.x) (&S.F[0][0])[i] = 0.0;
  __syncthreads();
  for (int k0 = 0; k0 < a.npairs; k0 += TR_KG) {
    const int kg = min(TR_KG, a.npairs - k0);
    // pivot chains: threads [0,kg) forward, [kg, 2kg) backward
    if (t < 2 * kg) tri_chain(S, a, c, k0 + (t % kg), t % kg, t / kg, rows, false);
    __syncthreads();
    tri_weights(S, a, k0, kg, rows, S.w);
    __syncthreads();
    const bool active = kk < kg;
    const int k = k0 + kk;
    // forward sweep: contributions 2 Re(w (g - f))
    cplx g = mk(0, 0);
    for (int i0 = 0; i0 < rows; i0 += TR_WIN) {
      const int wn = min(TR_WIN, rows - i0);
      if (active) {
        for (int j = 0; j < wn; ++j) {
          const int i = i0 + j;
          double f = rv ? a.V[(s + i) * a.nrhs + rg] : 0.0;
          cplx l = ld(&S.l[kk][i]);
          g = cplx{fma(-l.re, g.re, fma(l.im, g.im, f)), fma(-l.re, g.im, -l.im * g.re)};
          cplx w = ld(&S.w[kk][i]);
          S.cbuf[kk][j][r] = fma(w.re, g.re - f, -w.im * g.im);
        }
      }
      __syncthreads();
      for (int e = t; e < wn * TR_RT; e += blockDim.x) {
        int j = e / TR_RT, rr = e - j * TR_RT;
        double acc = S.F[i0 + j][rr];
        for (int q = 0; q < kg; ++q) acc += S.cbuf[q][j][rr];
        S.F[i0 + j][rr] = acc;
      }
      __syncthreads();
    }
    if (active && rv) st(&a.gF[(c * a.npairs + k) * a.nrhs + rg], g);
    // backward sweep: contributions 2 Re(w g')
    cplx gb = mk(0, 0);
    for (int i1 = rows; i1 > 0; i1 -= TR_WIN) {
      const int wn = min(TR_WIN, i1);
      const int i0 = i1 - wn;
      if (active) {
        for (int j = wn - 1; j >= 0; --j) {
          const int i = i0 + j;
          double f = rv ? a.V[(s + i) * a.nrhs + rg] : 0.0;
          cplx l = ld(&S.lb[kk][i]);
          gb = cplx{fma(-l.re, gb.re, fma(l.im, gb.im, f)), fma(-l.re, gb.im, -l.im * gb.re)};
          cplx w = ld(&S.w[kk][i]);
          S.cbuf[kk][j][r] = fma(w.re, gb.re, -w.im * gb.im);
        }
      }
      __syncthreads();
      for (int e = t; e < wn * TR_RT; e += blockDim.x) {
        int j = e / TR_RT, rr = e - j * TR_RT;
        double acc = S.F[i0 + j][rr];
        for (int q = 0; q < kg; ++q) acc += S.cbuf[q][j][rr];
        S.F[i0 + j][rr] = acc;
      }
      __syncthreads();
    }
    if (active && rv) st(&a.gB[(c * a.npairs + k) * a.nrhs + rg], gb);
    if (t < kg && blockIdx.y == 0) {
      a.LF[c * a.npairs + k0 + t] = S.lam[t][0];
      a.LB[c * a.npairs + k0 + t] = S.lam[t][1];
    }
    __syncthreads();
  }
  for (int e = t; e < rows * TR_RT; e += blockDim.x) {
    int i = e / TR_RT, rr = e - i * TR_RT;
    if (r0 + rr < a.nrhs) a.out[(s + i) * a.nrhs + r0 + rr] = S.F[i][rr];
  }
}

// K_T4 ------------------------------------------------------------------------
// One warp per (shift, rhs, direction).  Affine maps x -> A x + B composed over chunks.
__global__ void tri_carry_scan(TriArgs a) {
  const int warp_global = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  const int total = a.npairs * a.nrhs * 2;
  if (warp_global >= total) return;
  const int dir = warp_global & 1;
  const int kr = warp_global >> 1;
  const int k = kr / a.nrhs, rr = kr - k * a.nrhs;
  const int P = a.P;
  const int per = (P + 31) / 32;
  // lane composite
  cplx A = mk(1, 0), B = mk(0, 0);
  for (int j = 0; j < per; ++j) {
    int q = lane * per + j;
    if (q >= P) break;
    int cc = dir == 0 ? q : P - 1 - q;
    cplx Lc = ld(&(dir == 0 ? a.LF : a.LB)[(int64_t)cc * a.npairs + k]);
    cplx gc = ld(&(dir == 0 ? a.gF : a.gB)[((int64_t)cc * a.npairs + k) * a.nrhs + rr]);
    // new = Lc * (A x + B) + gc
    B = cadd(cmul(Lc, B), gc);
    A = cmul(Lc, A);
  }
  // inclusive warp scan (later lanes apply after earlier ones)
  for (int off = 1; off < 32; off <<= 1) {
    cplx pA, pB;
    pA.re = __shfl_up_sync(0xffffffffu, A.re, off);
    pA.im = __shfl_up_sync(0xffffffffu, A.im, off);
    pB.re = __shfl_up_sync(0xffffffffu, B.re, off);
    pB.im = __shfl_up_sync(0xffffffffu, B.im, off);
    if (lane >= off) {
      // mine o prev : x -> A (pA x + pB) + B
      B = cadd(cmul(A, pB), B);
      A = cmul(A, pA);
    }
  }
  cplx x;  // carry entering this lane's first chunk = exclusive prefix applied to 0
  x.re = __shfl_up_sync(0xffffffffu, B.re, 1);
  x.im = __shfl_up_sync(0xffffffffu, B.im, 1);
  if (lane == 0) x = mk(0, 0);
  for (int j = 0; j < per; ++j) {
    int q = lane * per + j;
    if (q >= P) break;
    int cc = dir == 0 ? q : P - 1 - q;
    st(&(dir == 0 ? a.G : a.Gb)[((int64_t)cc * a.npairs + k) * a.nrhs + rr], x);
    cplx Lc = ld(&(dir == 0 ? a.LF : a.LB)[(int64_t)cc * a.npairs + k]);
    cplx gc = ld(&(dir == 0 ? a.gF : a.gB)[((int64_t)cc * a.npairs + k) * a.nrhs + rr]);
    x = cadd(cmul(Lc, x), gc);
  }
}

// K_T5 ------------------------------------------------------------------------
__global__ void __launch_bounds__(TR_RT* TR_KG) tri_correct(TriArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TriSmem& S = *reinterpret_cast<TriSmem*>(smem_raw);
  const int64_t c = blockIdx.x;
  const int r0 = blockIdx.y * TR_RT;
  const int64_t s = c * TR_L;
  const int rows = (int)(TR_L < a.N - s ? TR_L : a.N - s);
  const int t = threadIdx.x;
  tri_load_chunk(S, a, s, rows);
  for (int i = t; i < rows * TR_RT; i += blockDim.x) (&S.F[0][0])[i] = 0.0;
  __syncthreads();
  for (int k0 = 0; k0 < a.npairs; k0 += TR_KG) {
    const int kg = min(TR_KG, a.npairs - k0);
    if (t < 2 * kg) tri_chain(S, a, c, k0 + (t % kg), t % kg, t / kg, rows, true);
    __syncthreads();
    // w (into cbuf-free storage): multiply Lambda in place by w
    for (int e = t; e < kg * rows; e += blockDim.x) {
      int kk = e / rows, i = e - kk * rows;
      const cplx th = ld(&a.theta[k0 + kk]);
      cplx b = mk(S.dg[i] + th.re, th.im);
      cplx l = ld(&S.l[kk][i]), lb = ld(&S.lb[kk][i]);
      cplx gam = csub(csub(b, cscale(l, S.of[i])), cscale(lb, S.of[i + 1]));
      cplx w = cscale(cdiv(ld(&a.coef[k0 + kk]), gam), 2.0);
      cplx wl = cmul(w, ld(&S.w[kk][i]));
      cplx wlb = cmul(w, ld(&S.wb[kk][i]));
      S.w[kk][i] = make_double2(wl.re, wl.im);
      S.wb[kk][i] = make_double2(wlb.re, wlb.im);
    }
    // carries of this chunk into l[][] scratch rows? use lam-free registers: stage in cbuf as doubles
    __syncthreads();
    for (int e = t; e < rows * TR_RT; e += blockDim.x) {
      int i = e / TR_RT, rr = e - i * TR_RT;
      int rg = r0 + rr;
      if (rg >= a.nrhs) continue;
      double acc = S.F[i][rr];
      for (int kk = 0; kk < kg; ++kk) {
        int k = k0 + kk;
        cplx G = ld(&a.G[(c * a.npairs + k) * a.nrhs + rg]);
        cplx Gb = ld(&a.Gb[(c * a.npairs + k) * a.nrhs + rg]);
        cplx wl = ld(&S.w[kk][i]), wlb = ld(&S.wb[kk][i]);
        acc = fma(wl.re, G.re, acc);
        acc = fma(-wl.im, G.im, acc);
        acc = fma(wlb.re, Gb.re, acc);
        acc = fma(-wlb.im, Gb.im, acc);
      }
      S.F[i][rr] = acc;
    }
    __syncthreads();
  }
  for (int e = t; e < rows * TR_RT; e += blockDim.x) {
    int i = e / TR_RT, rr = e - i * TR_RT;
    if (r0 + rr < a.nrhs) {
      size_t o = (s + i) * a.nrhs + r0 + rr;
      a.out[o] = a.out[o] + S.F[i][rr];
    }
  }
}

__global__ void scale_kernel(double* x, size_t n, double s) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    x[i] *= s;
}

int tridiag_run(const double* diag, const double* off, int64_t N, const double* V, int64_t nrhs, double shift_c,
                const double2* theta_d, const double2* coef_d, int npairs, double* out, cudaStream_t stream,
                float* launch_ms) {
  const int P = (int)ceil_div(N, TR_L);
  const size_t nP = (size_t)P * npairs;
  const size_t nPR = nP * nrhs;
  size_t bytes = (nP * 4 * 2 + nP * 4 + nPR * 4) * sizeof(double2);
  double2* ws = static_cast<double2*>(scratch(1, bytes));
  if (!ws) return fail(PFX_CUDA, "tridiagonal workspace allocation failed");
  TriArgs a;
  a.diag = diag;
  a.off = off;
  a.N = N;
  a.V = V;
  a.nrhs = (int)nrhs;
  a.c = shift_c;
  a.theta = theta_d;
  a.coef = coef_d;
  a.npairs = npairs;
  a.P = P;
  a.Tf = ws;
  a.Tb = a.Tf + nP * 4;
  a.rho_in = a.Tb + nP * 4;
  a.rhob_in = a.rho_in + nP;
  a.LF = a.rhob_in + nP;
  a.LB = a.LF + nP;
  a.gF = a.LB + nP;
  a.gB = a.gF + nPR;
  a.G = a.gB + nPR;
  a.Gb = a.G + nPR;
  a.out = out;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (launch_ms) {
    PFX_CUDA_TRY(cudaEventCreate(&e0));
    PFX_CUDA_TRY(cudaEventCreate(&e1));
    PFX_CUDA_TRY(cudaEventRecord(e0, stream));
  }
  {
    int64_t th = (int64_t)P * npairs * 2;
    PFX_LAUNCH("tri_mobius_chunks", stream, tri_mobius_chunks<<<(unsigned)ceil_div(th, 128), 128, 0, stream>>>(a));
    PFX_CUDA_TRY(cudaGetLastError());
    PFX_LAUNCH("tri_mobius_scan", stream, tri_mobius_scan<<<npairs * 2, TR_SCAN_T, 0, stream>>>(a));
    PFX_CUDA_TRY(cudaGetLastError());
  }
  const int smem = (int)sizeof(TriSmem);
  const int kg = std::min(npairs, TR_KG);
  dim3 grid((unsigned)P, (unsigned)ceil_div(nrhs, TR_RT));
  PFX_CUDA_TRY(cudaFuncSetAttribute(tri_local, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  PFX_LAUNCH("tri_local", stream, tri_local<<<grid, TR_RT * kg, smem, stream>>>(a));
  PFX_CUDA_TRY(cudaGetLastError());
  {
    int warps = npairs * (int)nrhs * 2;
    PFX_LAUNCH("tri_carry_scan", stream, tri_carry_scan<<<(unsigned)ceil_div(warps * 32, 256), 256, 0, stream>>>(a));
    PFX_CUDA_TRY(cudaGetLastError());
  }
  PFX_CUDA_TRY(cudaFuncSetAttribute(tri_correct, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  PFX_LAUNCH("tri_correct", stream, tri_correct<<<grid, TR_RT * kg, smem, stream>>>(a));
  PFX_CUDA_TRY(cudaGetLastError());
  if (shift_c != 0.0) {
    PFX_LAUNCH("scale_kernel", stream, scale_kernel<<<1184, 256, 0, stream>>>(out, (size_t)N * nrhs, exp(shift_c)));
    PFX_CUDA_TRY(cudaGetLastError());
  }
  if (launch_ms) {
    PFX_CUDA_TRY(cudaEventRecord(e1, stream));
    PFX_CUDA_TRY(cudaEventSynchronize(e1));
    PFX_CUDA_TRY(cudaEventElapsedTime(launch_ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  return PFX_OK;
}

}  // namespace pfx
