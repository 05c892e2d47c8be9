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
#include <complex>
#include <cstring>
#include <type_traits>
#include <vector>

#include "pfx_common.cuh"

namespace pfx {

constexpr int TR_L = 256;     // maximum rows per chunk (the chunk length a.L is chosen per call)
constexpr int TR_RT = 16;     // RHS per tile (threads per shift)
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
  int L;  // rows per chunk (multiple of 32, <= TR_L)
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
  double2* Lf;  // N x npairs  forward multipliers l_i
  double2* Lb;  // N x npairs  backward multipliers l'_i
  double2* Wt;  // N x npairs  twisted weights 2a/gamma_i
  int* contr;   // P          1 if every |l|, |l'| of the chunk is <= 1 (running products shrink)
  unsigned long long* vmax;  // nrhs  bit pattern of max_i |V[i, r]|
  double* out;  // N x nrhs
  // Row sharding (pfx_expm_tridiag_shard): this call owns chunks [c0, c1) of the P; the two
  // chunk scans then run in two passes, an aggregate pass (agg != 0: the range's composite
  // goes to magg / cagg) and a replay pass entering the range with the state the other
  // ranks' aggregates give (msin / csin; null = the start of the matrix).
  int64_t c0, c1;
  int agg;
  const double2* msin;  // npairs x 2 dirs x (vn, vd)      Moebius state entering the range
  double2* magg;        // npairs x 2 dirs x 4              transfer over the range
  const double2* csin;  // npairs x nrhs x 2 dirs           RHS carry entering the range
  double2* cagg;        // npairs x nrhs x 2 dirs x (A, B)  affine map over the range
  // Host-mode group pipeline (carry scans per row group): directions scanned (bit 0 forward,
  // bit 1 backward), carries stored only for chunks [w0, w1), and cin_prev = the forward
  // carry entering the range is continued from the previous chunk's (G, LF, gF)
  int dirmask;
  int64_t w0, w1;
  int cin_prev;
};

// chunk summaries are stored chunk-fastest so the carry scan (one block per pair, rhs and
// direction, walking the chunks) reads contiguous memory; the producers' stores scatter
__device__ __forceinline__ int64_t g_at(const TriArgs& a, int64_t c, int k, int r) {
  return ((int64_t)k * a.nrhs + r) * a.P + c;
}
__device__ __forceinline__ int64_t l_at(const TriArgs& a, int64_t c, int k) { return (int64_t)k * a.P + c; }

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
  double s = pow2_inv_scale(mx);
  a.m0 = cscale(a.m0, s);
  a.m1 = cscale(a.m1, s);
  a.m2 = cscale(a.m2, s);
  a.m3 = cscale(a.m3, s);
}

__device__ __forceinline__ M22 mident() { return M22{mk(1, 0), mk(0, 0), mk(0, 0), mk(1, 0)}; }

// ---------------------------------------------------------------------------
// K_T1: transfer matrices.  Forward: (u_i; 1) ~ [b_i, -e_{i-1}^2; 1, 0] (u_{i-1}; 1).
// Backward: (u'_i; 1) ~ [b_i, -e_i^2; 1, 0] (u'_{i+1}; 1).
constexpr int TR_SEG = 4;  // row segments per (chunk, shift) in tri_mobius_chunks

__device__ __forceinline__ M22 shfl_m22(const M22& m, int src) {
  M22 r;
  const cplx* in = &m.m0;
  cplx* o = &r.m0;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    o[t].re = __shfl_sync(0xffffffffu, in[t].re, src);
    o[t].im = __shfl_sync(0xffffffffu, in[t].im, src);
  }
  return r;
}

// One thread per (chunk, shift, 64-row segment); both directions from the same row loads:
// forward T <- M_i T (rows ascending), backward T' <- T' M'_i (rows ascending, i.e. the
// product M'_lo ... M'_hi that the descending recurrence applies).  The TR_SEG segment
// transfers of a (chunk, shift) sit in adjacent lanes and are combined by shuffles.
__global__ void __launch_bounds__(128) tri_mobius_chunks(TriArgs a) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t total = (a.c1 - a.c0) * a.npairs * TR_SEG;
  const bool live = tid < total;
  const int seg = (int)(tid & (TR_SEG - 1));
  const int64_t ck = live ? tid / TR_SEG + a.c0 * a.npairs : 0;
  const int k = (int)(ck % a.npairs);
  const int64_t cidx = ck / a.npairs;
  const int64_t s = cidx * a.L, e = (s + a.L < a.N ? s + a.L : a.N);
  const int SL = a.L / TR_SEG;
  const int64_t s0 = s + (int64_t)seg * SL;
  const int64_t rem = e - s0;
  const int rows = (!live || rem <= 0) ? 0 : (rem < SL ? (int)rem : SL);
  const cplx th = ld(&a.theta[k]);
  // Only the forward product is formed.  With the first row's coupling replaced by 1 it is
  // F' = [A, -C; D, -E] in the chunk's continuants (A: rows 1..n, C: 2..n, D: 1..n-1,
  // E: 2..n-1), and both transfers follow from it: F = F' diag(1, e_0^2) and
  // B = [A, -e_n^2 D; C, -e_n^2 E] (e_0, e_n: couplings into the chunk from above / below).
  // Every entry is a forward continuant, so nothing is lost by not running the backward
  // recurrence; the scan uses the transfers only up to a common scale.
  M22 F = mident();
  for (int i0 = 0; i0 < rows; i0 += 8) {
    double bre[8], e2[8];  // e2[u] = e_{i-1}^2 for row i = s0 + i0 + u (1 for the segment's first row)
#pragma unroll
    for (int u = 0; u < 8; ++u) bre[u] = (i0 + u < rows) ? a.diag[s0 + i0 + u] - a.c + th.re : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) e2[u] = (i0 + u == 0) ? 1.0 : (i0 + u < rows) ? off2(a.off, a.N, s0 + i0 + u - 1) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (i0 + u < rows) {
        const cplx b = mk(bre[u], th.im);
        // [b, -e_{i-1}^2; 1, 0] F
        const cplx f0 = csub(cmul(b, F.m0), cscale(F.m2, e2[u]));
        const cplx f1 = csub(cmul(b, F.m1), cscale(F.m3, e2[u]));
        F.m2 = F.m0;
        F.m3 = F.m1;
        F.m0 = f0;
        F.m1 = f1;
      }
    }
    mnorm(F);
  }
  // segments after the first carry their true coupling into the product
  if (seg > 0 && rows > 0) {
    const double es = off2(a.off, a.N, s0 - 1);
    F.m1 = cscale(F.m1, es);
    F.m3 = cscale(F.m3, es);
  }
  // combine segments: F' = F3 F2 F1 F'0
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int w = 1; w < TR_SEG; w <<= 1) {
    const M22 Fp = shfl_m22(F, lane + w < 32 ? lane + w : lane);
    if ((seg & (2 * w - 1)) == 0) {
      F = mmul(Fp, F);
      mnorm(F);
    }
  }
  if (live && seg == 0) {
    const double e0 = off2(a.off, a.N, s - 1), en = off2(a.off, a.N, e - 1);
    double2* df = a.Tf + ck * 4;
    double2* db = a.Tb + ck * 4;
    st(&df[0], F.m0);
    st(&df[1], cscale(F.m1, e0));
    st(&df[2], F.m2);
    st(&df[3], cscale(F.m3, e0));
    st(&db[0], F.m0);
    st(&db[1], cscale(F.m2, -en));
    st(&db[2], cscale(F.m1, -1.0));
    st(&db[3], cscale(F.m3, en));
  }
}

// ---------------------------------------------------------------------------
// K_T2: per (shift, direction) block scan.  Chunk order is reversed for the
// backward direction.  Carry of chunk c = pivot reciprocal entering it:
// state vector v = (num; den) with u = num/den, rho = den/num; start (1; 0).
__global__ void __launch_bounds__(TR_SCAN_T) tri_mobius_scan(TriArgs a) {
  // the thread composites, stored component-major: with 64-byte M22 records the scan's
  // 16-byte loads hit the same banks four lanes at a time (measured: ~20 us of bank-conflict
  // stalls per launch); here consecutive lanes read consecutive 16-byte words
  __shared__ cplx sm[4][TR_SCAN_T];
  auto sm_ld = [&](int i) { return M22{sm[0][i], sm[1][i], sm[2][i], sm[3][i]}; };
  auto sm_st = [&](int i, const M22& m) {
    sm[0][i] = m.m0;
    sm[1][i] = m.m1;
    sm[2][i] = m.m2;
    sm[3][i] = m.m3;
  };
  const int k = blockIdx.x >> 1, dir = blockIdx.x & 1;
  const int P = (int)(a.c1 - a.c0);  // chunks of this call's range
  const int per = (P + TR_SCAN_T - 1) / TR_SCAN_T;
  const int t = threadIdx.x;
  const double2* Tsrc = dir == 0 ? a.Tf : a.Tb;
  double2* dst = dir == 0 ? a.rho_in : a.rhob_in;
  auto chunk_of = [&](int q) { return dir == 0 ? a.c0 + q : a.c1 - 1 - q; };
  // composite of this thread's range (in processing order)
  M22 acc = mident();
  for (int j = 0; j < per; ++j) {
    int q = t * per + j;
    if (q >= P) break;
    const int64_t c = chunk_of(q);
    const double2* src = Tsrc + ((int64_t)c * a.npairs + k) * 4;
    M22 T{ld(&src[0]), ld(&src[1]), ld(&src[2]), ld(&src[3])};
    acc = mmul(T, acc);
    mnorm(acc);
  }
  sm_st(t, acc);
  __syncthreads();
  // Hillis-Steele inclusive scan: S_t = A_t * A_{t-1} * ... * A_0
  for (int off = 1; off < TR_SCAN_T; off <<= 1) {
    M22 mine = sm_ld(t);
    M22 other = t >= off ? sm_ld(t - off) : mident();
    __syncthreads();
    if (t >= off) {
      M22 r = mmul(mine, other);
      mnorm(r);
      sm_st(t, r);
    }
    __syncthreads();
  }
  if (a.agg) {  // aggregate pass: the range's transfer only
    if (t == TR_SCAN_T - 1) {
      double2* o = a.magg + (k * 2 + dir) * 4;
      st(&o[0], sm[0][t]);
      st(&o[1], sm[1][t]);
      st(&o[2], sm[2][t]);
      st(&o[3], sm[3][t]);
    }
    return;
  }
  M22 pre = t > 0 ? sm_ld(t - 1) : mident();
  // state entering this thread's range: pre * s0, s0 = (1; 0) at the start of the matrix
  const cplx s0n = a.msin ? ld(&a.msin[(k * 2 + dir) * 2]) : mk(1, 0);
  const cplx s0d = a.msin ? ld(&a.msin[(k * 2 + dir) * 2 + 1]) : mk(0, 0);
  cplx vn = cadd(cmul(pre.m0, s0n), cmul(pre.m1, s0d)), vd = cadd(cmul(pre.m2, s0n), cmul(pre.m3, s0d));
  for (int j = 0; j < per; ++j) {
    int q = t * per + j;
    if (q >= P) break;
    const int64_t c = chunk_of(q);
    // rho = den / num (0 entering the first chunk of the matrix: no coupling)
    cplx rho = (vn.re == 0.0 && vn.im == 0.0) ? mk(0, 0) : cdiv(vd, vn);
    st(&dst[(int64_t)c * a.npairs + k], rho);
    const double2* src = Tsrc + ((int64_t)c * a.npairs + k) * 4;
    M22 T{ld(&src[0]), ld(&src[1]), ld(&src[2]), ld(&src[3])};
    cplx nn = cadd(cmul(T.m0, vn), cmul(T.m1, vd));
    cplx nd = cadd(cmul(T.m2, vn), cmul(T.m3, vd));
    double mx = fmax(fmax(cabs1(nn), cabs1(nd)), 1e-300);
    double s = pow2_inv_scale(mx);
    vn = cscale(nn, s);
    vd = cscale(nd, s);
  }
}

// ---------------------------------------------------------------------------
// K_T3 tri_factor: one thread per (chunk, shift).  Pivot chains in continuant form
// (the only loop-carried dependency is the three-term recurrence; the ratio
// rho = p_{i-2}/p_{i-1} and everything after it is off the critical path):
//   backward: q_i = b_i q_{i+1} - e_i^2 q_{i+2},  l'_i = e_i q_{i+2}/q_{i+1}
//   forward:  p_i = b_i p_{i-1} - e_{i-1}^2 p_{i-2}, l_i = e_{i-1} p_{i-2}/p_{i-1}
//   gamma_i = b_i - e_{i-1} l_i - e_i l'_i,  w_i = 2 a / gamma_i
// Outputs (row-major [row][shift], so a row's shifts are contiguous for the sweeps):
//   Lf = l, Lb = l', Wt = w, and the chunk products LF = prod(-l), LB = prod(-l').
__device__ __forceinline__ void rescale2(cplx& x, cplx& y) {
  double mx = fmax(fmax(cabs1(x), cabs1(y)), 1e-300);
  double s = pow2_inv_scale(mx);
  x = cscale(x, s);
  y = cscale(y, s);
}

__global__ void __launch_bounds__(128) tri_factor(TriArgs a) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= (int64_t)a.P * a.npairs) return;
  const int k = (int)(tid % a.npairs);
  const int64_t c = tid / a.npairs;
  const int64_t s = c * a.L;
  const int rows = (int)(a.L < a.N - s ? a.L : a.N - s);
  const cplx th = ld(&a.theta[k]);
  const int np = a.npairs;
  auto offe = [&](int64_t gi) -> double { return (gi >= 0 && gi < a.N - 1) ? a.off[gi] : 0.0; };
  bool noncontr = false;
  // backward chain
  {
    cplx q1 = mk(1, 0), q2 = ld(&a.rhob_in[c * np + k]);
    cplx lam = mk(1, 0);
    double e = offe(s + rows - 1);
    for (int i = rows - 1; i >= 0; --i) {
      cplx rho = cmul(q2, crcp_fast(q1));
      cplx lv = cscale(rho, e);
      cplx b = mk(a.diag[s + i] - a.c + th.re, th.im);
      double e2 = e * e;
      cplx q0 = cplx{fma(b.re, q1.re, fma(-b.im, q1.im, -e2 * q2.re)), fma(b.re, q1.im, fma(b.im, q1.re, -e2 * q2.im))};
      st(&a.Lb[(s + i) * np + k], lv);
      if (fma(lv.re, lv.re, lv.im * lv.im) > 1.0) noncontr = true;
      lam = cmul(lam, mk(-lv.re, -lv.im));
      q2 = q1;
      q1 = q0;
      if ((i & 3) == 0) rescale2(q1, q2);
      e = offe(s + i - 1);
    }
    st(&a.LB[l_at(a, c, k)], lam);
  }
  // forward chain + twisted weights
  {
    const cplx co2 = cscale(ld(&a.coef[k]), 2.0);
    cplx p1 = mk(1, 0), p2 = ld(&a.rho_in[c * np + k]);
    cplx lam = mk(1, 0);
    double e0 = offe(s - 1);
    for (int i = 0; i < rows; ++i) {
      double e1 = offe(s + i);
      cplx rho = cmul(p2, crcp_fast(p1));
      cplx lv = cscale(rho, e0);
      cplx b = mk(a.diag[s + i] - a.c + th.re, th.im);
      double e2 = e0 * e0;
      cplx p0 = cplx{fma(b.re, p1.re, fma(-b.im, p1.im, -e2 * p2.re)), fma(b.re, p1.im, fma(b.im, p1.re, -e2 * p2.im))};
      cplx lbv = ld(&a.Lb[(s + i) * np + k]);
      cplx gam = csub(csub(b, cscale(lv, e0)), cscale(lbv, e1));
      cplx w = cdiv_fast(co2, gam);
      st(&a.Lf[(s + i) * np + k], lv);
      st(&a.Wt[(s + i) * np + k], w);
      if (fma(lv.re, lv.re, lv.im * lv.im) > 1.0) noncontr = true;
      lam = cmul(lam, mk(-lv.re, -lv.im));
      p2 = p1;
      p1 = p0;
      if ((i & 3) == 3) rescale2(p1, p2);
      e0 = e1;
    }
    st(&a.LF[l_at(a, c, k)], lam);
  }
  if (noncontr) atomicAnd(&a.contr[c], 0);
}

// K_T4 tri_sweep / K_T5 tri_fix share one streaming skeleton.  Thread layout: a
// half-warp = one (chunk, 16-RHS tile), lane r = one right-hand side; the
// recurrences of all shifts of that RHS run interleaved in registers (ILP =
// npairs) and are summed over shifts in ascending order (deterministic).  Each
// half-warp stages its chunk's factor data (l or l', w) and RHS rows through
// shared memory in TR_T-row tiles with cp.async double buffering, so the global
// loads of tile t+1 overlap the FP64 work of tile t.
//   MODE 0 (tri_sweep): forward sweep (writes F_i = sum_k Re(w (g - f))), then the
//     backward sweep of the same chunk adds sum_k Re(w g') (F read back while L2-hot);
//     zero RHS carry-in, chunk summaries gF/gB, running max |V[:, r]|.
//   MODE 1 (tri_fix): true carries through Lambda_i = prod_{j<=i}(-l_j) (forward, from
//     the chunk top) and Lambda'_i (backward, from the chunk bottom).  In a contractive
//     chunk (all |l|, |l'| <= 1) |Lambda| never grows, and |w| <= 2|a|/Im(theta) (the
//     pivots of T + theta I satisfy |gamma| >= Im(theta)), so once
//     sum_k (2|a_k|/Im theta_k) |Lambda_k| |G_k| <= 2^-53 max|V[:, r]| every remaining
//     row's correction is below one unit roundoff of max|V[:, r]| and the pass stops
//     (below the binary64 rounding of the 2n-term pole sum itself; full pass for
//     non-contractive chunks).
constexpr int TR_FIX_EXP = 53;     // fix-pass stop: remaining correction <= 2^-53 max|V|
constexpr int TR_T = 8;            // rows per staged tile
constexpr int TR_SW_WARPS = 4;     // warps per block

template <int KM>
struct TriStage {
  double2 l[2][TR_T][KM];
  double2 w[2][TR_T][KM];
  double f[2][TR_T][TR_RT];
};

// stage rows [r0, r0+cnt) (cnt <= TR_T) of L and Wt plus the RHS tile into buffer b
template <int KM>
__device__ __forceinline__ void stage_tile(TriStage<KM>& S, int b, const TriArgs& a, const double2* L, int64_t r0,
                                           int cnt, int rt0, int lane16, bool want_f) {
  const int np = a.npairs;
  const int nel = cnt * np;  // complex elements per array
  const double2* ls = L + r0 * np;
  const double2* ws = a.Wt + r0 * np;
  double2* ld_ = &S.l[b][0][0];
  double2* wd = &S.w[b][0][0];
  for (int e = lane16; e < nel; e += 16) {
    int rr = e / np, k = e - rr * np;
    cp_async16(&ld_[rr * KM + k], &ls[e]);
    cp_async16(&wd[rr * KM + k], &ws[e]);
  }
  const int rg = rt0 + lane16;
  if (want_f && rg < a.nrhs)
    for (int rr = 0; rr < cnt; ++rr) cp_async8(&S.f[b][rr][lane16], &a.V[(r0 + rr) * a.nrhs + rg]);
}

template <int KM, int MODE>
__global__ void __launch_bounds__(TR_SW_WARPS * 32) tri_pass(TriArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = lane >> 4, lane16 = lane & 15;
  const unsigned hmask = half ? 0xffff0000u : 0x0000ffffu;
  TriStage<KM>& S = reinterpret_cast<TriStage<KM>*>(smem_raw)[warp * 2 + half];
  const int ntile = (a.nrhs + TR_RT - 1) / TR_RT;
  const int64_t unit = (blockIdx.x * (int64_t)TR_SW_WARPS + warp) * 2 + half;  // (chunk, rhs tile)
  if (unit >= (int64_t)a.P * ntile) return;  // whole half-warps exit together
  const int64_t c = unit / ntile;
  const int rt0 = (int)(unit - c * ntile) * TR_RT;
  const int r = rt0 + lane16;
  const bool rv = r < a.nrhs;
  const int64_t s = c * a.L;
  const int rows = (int)(a.L < a.N - s ? a.L : a.N - s);
  const int np = a.npairs;
  const int ntl = (rows + TR_T - 1) / TR_T;
  double vmx = 0.0;
  double tau = 0.0;
  bool contr = false;
  double beta[KM];
  if (MODE == 1) {
    tau = rv ? ldexp(__longlong_as_double((long long)a.vmax[r]), -TR_FIX_EXP) : 1.0;
    contr = a.contr[c] != 0;
#pragma unroll
    for (int k = 0; k < KM; ++k) {
      if (k < np) {
        cplx th = ld(&a.theta[k]), co = ld(&a.coef[k]);
        beta[k] = 2.0 * (fabs(co.re) + fabs(co.im)) / th.im;
      } else {
        beta[k] = 0.0;
      }
    }
  }
  for (int dir = 0; dir < 2; ++dir) {
    const double2* L = dir == 0 ? a.Lf : a.Lb;
    cplx g[KM], G[KM];
#pragma unroll
    for (int k = 0; k < KM; ++k) {
      if (MODE == 0) {
        g[k] = mk(0, 0);
      } else {
        g[k] = mk(1, 0);  // Lambda
        const double2* Gs = dir == 0 ? a.G : a.Gb;
        G[k] = (k < np && rv) ? ld(&Gs[(c * np + k) * a.nrhs + r]) : mk(0, 0);
      }
    }
    auto tile_first = [&](int t) { return dir == 0 ? t * TR_T : max(rows - (t + 1) * TR_T, 0); };
    auto tile_cnt = [&](int t) {
      return dir == 0 ? min(TR_T, rows - t * TR_T) : rows - t * TR_T - max(rows - (t + 1) * TR_T, 0);
    };
    bool done = false;
    stage_tile<KM>(S, 0, a, L, s + tile_first(0), tile_cnt(0), rt0, lane16, MODE == 0);
    cp_async_commit();
    for (int t = 0; t < ntl; ++t) {
      const int b = t & 1;
      if (t + 1 < ntl) stage_tile<KM>(S, b ^ 1, a, L, s + tile_first(t + 1), tile_cnt(t + 1), rt0, lane16, MODE == 0);
      cp_async_commit();
      cp_async_wait<1>();
      __syncwarp(hmask);
      const int first = tile_first(t), cnt = tile_cnt(t);
      for (int jj = 0; jj < cnt; ++jj) {
        const int j = dir == 0 ? jj : cnt - 1 - jj;
        const int64_t row = s + first + j;
        double acc = 0.0;
        if (MODE == 1 || dir == 1) acc = rv ? a.out[row * a.nrhs + r] : 0.0;
        if (MODE == 0) {
          const double f = S.f[b][j][lane16];
          vmx = fmax(vmx, fabs(f));
#pragma unroll
          for (int k = 0; k < KM; ++k) {
            if (k < np) {
              const cplx l = ld(&S.l[b][j][k]);
              const cplx w = ld(&S.w[b][j][k]);
              g[k] = cplx{fma(-l.re, g[k].re, fma(l.im, g[k].im, f)), fma(-l.re, g[k].im, -l.im * g[k].re)};
              const double gre = dir == 0 ? g[k].re - f : g[k].re;
              acc = fma(w.re, gre, fma(-w.im, g[k].im, acc));
            }
          }
        } else {
          double bound = 0.0;
#pragma unroll
          for (int k = 0; k < KM; ++k) {
            if (k < np) {
              const cplx l = ld(&S.l[b][j][k]);
              const cplx w = ld(&S.w[b][j][k]);
              g[k] = cmul(g[k], mk(-l.re, -l.im));
              const cplx tt = cmul(g[k], G[k]);
              acc = fma(w.re, tt.re, fma(-w.im, tt.im, acc));
              bound = fma(beta[k] * cabs1(g[k]), cabs1(G[k]), bound);
            }
          }
          if (contr && bound <= tau) done = true;
        }
        if (rv) a.out[row * a.nrhs + r] = acc;
      }
      __syncwarp(hmask);
      if (MODE == 1 && !__any_sync(hmask, !done)) {
        cp_async_wait<0>();
        break;
      }
    }
    if (MODE == 0 && rv) {
      double2* dst = dir == 0 ? a.gF : a.gB;
#pragma unroll
      for (int k = 0; k < KM; ++k)
        if (k < np) st(&dst[g_at(a, c, k, r)], g[k]);
    }
    cp_async_wait<0>();
    __syncwarp(hmask);
  }
  if (MODE == 0 && rv) atomicMax(&a.vmax[r], (unsigned long long)__double_as_longlong(vmx));
}

#include "tridiag_ls.cuh"

// K_T4 ------------------------------------------------------------------------
// One 256-thread block per (shift, rhs, direction).  Affine maps x -> A x + B composed
// over chunks: each thread composes a contiguous range (loads batched), block scan of the
// thread composites through shared memory, then each thread replays its range.
constexpr int CS_T = 256;
// carry entering the scanned range: the exchanged one (row sharding), the previous chunk's
// carried through its summary (host-mode group pipeline, forward), else zero (matrix edge)
__device__ __forceinline__ cplx carry_in(const TriArgs& a, int k, int rr, int dir) {
  if (a.csin) return ld(&a.csin[(k * a.nrhs + rr) * 2 + dir]);
  if (a.cin_prev && dir == 0 && a.c0 > 0) {
    const int64_t c = a.c0 - 1;
    return cadd(cmul(ld(&a.LF[l_at(a, c, k)]), ld(&a.G[(c * a.npairs + k) * a.nrhs + rr])), ld(&a.gF[g_at(a, c, k, rr)]));
  }
  return mk(0, 0);
}

__global__ void __launch_bounds__(CS_T) tri_carry_scan(TriArgs a) {
  __shared__ cplx sA[CS_T], sB[CS_T];
  const int bid = blockIdx.x;
  const int dir = bid & 1;
  if (!((a.dirmask >> dir) & 1)) return;
  const int kr = bid >> 1;
  const int k = kr / a.nrhs, rr = kr - k * a.nrhs;
  const int P = (int)(a.c1 - a.c0);  // chunks of this call's range
  const int t = threadIdx.x;
  const int per = (P + CS_T - 1) / CS_T;
  const double2* Ls = dir == 0 ? a.LF : a.LB;
  const double2* gs = dir == 0 ? a.gF : a.gB;
  auto chunk_of = [&](int q) { return dir == 0 ? a.c0 + q : a.c1 - 1 - q; };
  cplx A = mk(1, 0), B = mk(0, 0);
  for (int j0 = 0; j0 < per; j0 += 8) {
    cplx Lc[8], gc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int q = t * per + j0 + u;
      if (j0 + u < per && q < P) {
        const int cc = chunk_of(q);
        Lc[u] = ld(&Ls[l_at(a, cc, k)]);
        gc[u] = ld(&gs[g_at(a, cc, k, rr)]);
      } else {
        Lc[u] = mk(1, 0);
        gc[u] = mk(0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      B = cadd(cmul(Lc[u], B), gc[u]);
      A = cmul(Lc[u], A);
    }
  }
  sA[t] = A;
  sB[t] = B;
  __syncthreads();
  for (int off = 1; off < CS_T; off <<= 1) {
    cplx pA = t >= off ? sA[t - off] : mk(1, 0), pB = t >= off ? sB[t - off] : mk(0, 0);
    __syncthreads();
    if (t >= off) {
      B = cadd(cmul(A, pB), B);
      A = cmul(A, pA);
      sA[t] = A;
      sB[t] = B;
    }
    __syncthreads();
  }
  if (a.agg) {  // aggregate pass: the range's affine map only
    if (t == CS_T - 1) {
      st(&a.cagg[((k * a.nrhs + rr) * 2 + dir) * 2], A);
      st(&a.cagg[((k * a.nrhs + rr) * 2 + dir) * 2 + 1], B);
    }
    return;
  }
  const cplx x0 = carry_in(a, k, rr, dir);
  cplx x = t > 0 ? cadd(cmul(sA[t - 1], x0), sB[t - 1]) : x0;
  double2* dst = dir == 0 ? a.G : a.Gb;
  for (int j0 = 0; j0 < per; j0 += 8) {
    cplx Lc[8], gc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int q = t * per + j0 + u;
      if (j0 + u < per && q < P) {
        const int cc = chunk_of(q);
        Lc[u] = ld(&Ls[l_at(a, cc, k)]);
        gc[u] = ld(&gs[g_at(a, cc, k, rr)]);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int q = t * per + j0 + u;
      if (j0 + u < per && q < P) {
        const int64_t cq = chunk_of(q);
        if (cq >= a.w0 && cq < a.w1) st(&dst[(cq * a.npairs + k) * a.nrhs + rr], x);
        x = cadd(cmul(Lc[u], x), gc[u]);
      }
    }
  }
}

// Same scan with the block's whole column staged in shared memory by one round of coalesced
// cp.async (chunk-fastest summaries: L and g of this (pair, rhs) are two contiguous runs of P
// complex); used when 2 P complex fit (P <= CS_SMEM_P).
constexpr int CS_SMEM_P = 6144;
__global__ void __launch_bounds__(CS_T) tri_carry_scan_smem(TriArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // one pad slot per 16 chunks: thread t walks chunks 16t.., so unpadded its lanes would sit
  // 256 B apart in one bank group; padded (272 B) they spread over all banks
  auto sx = [](int cc) { return cc + (cc >> 4); };
  const int P = (int)(a.c1 - a.c0);  // chunks of this call's range (local index = chunk - c0)
  const int PP = P + (P >> 4) + 1;
  double2* sL = reinterpret_cast<double2*>(smem_raw);  // PP
  double2* sg = sL + PP;                               // PP
  __shared__ cplx sA[CS_T], sB[CS_T];
  const int bid = blockIdx.x;
  const int dir = bid & 1;
  if (!((a.dirmask >> dir) & 1)) return;
  const int kr = bid >> 1;
  const int k = kr / a.nrhs, rr = kr - k * a.nrhs;
  const int t = threadIdx.x;
  const double2* Ls = (dir == 0 ? a.LF : a.LB) + l_at(a, a.c0, k);
  const double2* gs = (dir == 0 ? a.gF : a.gB) + g_at(a, a.c0, k, rr);
  for (int e = t; e < P; e += CS_T) {
    cp_async16(&sL[sx(e)], &Ls[e]);
    cp_async16(&sg[sx(e)], &gs[e]);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  const int per = (P + CS_T - 1) / CS_T;
  auto chunk_of = [&](int q) { return dir == 0 ? q : P - 1 - q; };  // local
  cplx A = mk(1, 0), B = mk(0, 0);
  for (int j = 0; j < per; ++j) {
    const int q = t * per + j;
    if (q >= P) break;
    const int cc = sx(chunk_of(q));
    const cplx L = ld(&sL[cc]);
    B = cadd(cmul(L, B), ld(&sg[cc]));
    A = cmul(L, A);
  }
  sA[t] = A;
  sB[t] = B;
  __syncthreads();
  for (int off = 1; off < CS_T; off <<= 1) {
    cplx pA = t >= off ? sA[t - off] : mk(1, 0), pB = t >= off ? sB[t - off] : mk(0, 0);
    __syncthreads();
    if (t >= off) {
      B = cadd(cmul(A, pB), B);
      A = cmul(A, pA);
      sA[t] = A;
      sB[t] = B;
    }
    __syncthreads();
  }
  if (a.agg) {  // aggregate pass: the range's affine map only
    if (t == CS_T - 1) {
      st(&a.cagg[((k * a.nrhs + rr) * 2 + dir) * 2], A);
      st(&a.cagg[((k * a.nrhs + rr) * 2 + dir) * 2 + 1], B);
    }
    return;
  }
  const cplx x0 = carry_in(a, k, rr, dir);
  cplx x = t > 0 ? cadd(cmul(sA[t - 1], x0), sB[t - 1]) : x0;
  double2* dst = dir == 0 ? a.G : a.Gb;
  for (int j = 0; j < per; ++j) {
    const int q = t * per + j;
    if (q >= P) break;
    const int cc = chunk_of(q);
    if (a.c0 + cc >= a.w0 && a.c0 + cc < a.w1) st(&dst[((a.c0 + cc) * a.npairs + k) * a.nrhs + rr], x);
    x = cadd(cmul(ld(&sL[sx(cc)]), x), ld(&sg[sx(cc)]));
  }
}

// Host-mode group pipeline: group g's backward carries were scanned from the end of group g+1
// with zero entering (truncation).  The neglected term is (prod over group g+1 of L') times the
// true carry entering there, |carry| <= N max|V| when every chunk is contractive (|l'| <= 1),
// and it reaches the output through |z| <= beta_k: it stays below one unit roundoff of max|V|
// when N sum_k beta_k max_k prod_{c in g+1} |LB_k(c)| <= 2^-53.  Otherwise (or for any
// non-contractive chunk) *flag is set and the caller redoes the carries globally.
__global__ void tri_trunc_check(TriArgs a, int ng, int* flag) {
  // one warp per (truncated group, pair): log2 of the product, summed over the group's chunks
  const int np = a.npairs;
  const int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (w < (ng - 1) * np) {
    const int g = w / np + 1, k = w - (w / np) * np;  // group g (>= 1) was truncated away
    const int64_t lo = (int64_t)a.P * g / ng, hi = (int64_t)a.P * (g + 1) / ng;
    double lg = 0.0;
    for (int64_t c = lo + lane; c < hi; c += 32) {
      const cplx l = ld(&a.LB[l_at(a, c, k)]);
      lg += 0.5 * log2(fma(l.re, l.re, l.im * l.im));  // -inf for an exact zero: fine
    }
    for (int off = 16; off > 0; off >>= 1) lg += __shfl_xor_sync(0xffffffffu, lg, off);
    double bsum = 0.0;
    for (int q = 0; q < np; ++q) {
      const cplx th = ld(&a.theta[q]), co = ld(&a.coef[q]);
      bsum += 2.0 * cabs1(co) / th.im;
    }
    if (lane == 0 && !(lg + log2((double)a.N * bsum) <= -53.0)) atomicExch(flag, 1);
  } else if (w == (ng - 1) * np) {
    for (int64_t c = lane; c < a.P; c += 32)
      if (!a.contr[c]) atomicExch(flag, 1);
  }
}

static int carry_scan(const TriArgs& a, int npairs, int64_t nrhs, cudaStream_t stream) {
  const unsigned blocks = (unsigned)(npairs * nrhs * 2);
  const int64_t np_ = a.c1 - a.c0;
  if (np_ <= CS_SMEM_P) {
    const int smem = 2 * (int)(np_ + (np_ >> 4) + 1) * (int)sizeof(double2);
    const int mx = 2 * (CS_SMEM_P + (CS_SMEM_P >> 4) + 1) * (int)sizeof(double2);
    if (int rc = raise_smem_limit(reinterpret_cast<const void*>(tri_carry_scan_smem), mx)) return rc;
    PFX_LAUNCH("tri_carry_scan", stream, tri_carry_scan_smem<<<blocks, CS_T, smem, stream>>>(a));
  } else {
    PFX_LAUNCH("tri_carry_scan", stream, tri_carry_scan<<<blocks, CS_T, 0, stream>>>(a));
  }
  PFX_CUDA_TRY(cudaGetLastError());
  return PFX_OK;
}

__global__ void scale_kernel(double* x, size_t n, double s) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    x[i] *= s;
}

template <int KM>
static int launch_stream(const TriArgs& a, cudaStream_t stream, int which) {
  const int ntile = (a.nrhs + TR_RT - 1) / TR_RT;
  const int64_t units = (int64_t)a.P * ntile;
  const unsigned blocks = (unsigned)ceil_div(units, TR_SW_WARPS * 2);
  const int smem = (int)(sizeof(TriStage<KM>) * TR_SW_WARPS * 2);
  const int th = TR_SW_WARPS * 32;
  if (which == 0) {
    if (int rc = raise_smem_limit(reinterpret_cast<const void*>(tri_pass<KM, 0>), smem)) return rc;
    PFX_LAUNCH("tri_sweep", stream, (tri_pass<KM, 0><<<blocks, th, smem, stream>>>(a)));
  } else {
    if (int rc = raise_smem_limit(reinterpret_cast<const void*>(tri_pass<KM, 1>), smem)) return rc;
    PFX_LAUNCH("tri_fix", stream, (tri_pass<KM, 1><<<blocks, th, smem, stream>>>(a)));
  }
  return PFX_OK;
}

static int sweeps(const TriArgs& a, cudaStream_t stream, int which) {
  if (a.npairs <= 8) return launch_stream<8>(a, stream, which);
  if (a.npairs <= 12) return launch_stream<12>(a, stream, which);
  if (a.npairs <= 16) return launch_stream<16>(a, stream, which);
  return launch_stream<32>(a, stream, which);
}

__global__ void scale_rows(double* x, int64_t n, double s) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    x[e] *= s;
}

namespace {
#ifndef PFX_TR_GROUPS
#define PFX_TR_GROUPS 16  // row groups of the host pipeline (tools/ab_c2_host.sh)
#endif
constexpr int TR_GROUPS = PFX_TR_GROUPS;
struct TriPipe {
  cudaStream_t in = nullptr, outs = nullptr;
  cudaStream_t cs[TR_GROUPS] = {};  // per-group fix streams: earlier groups first (D2H order)
  cudaStream_t sw[TR_GROUPS] = {};  // per-group sweep streams: later groups first (their rows land last)
  cudaEvent_t ev[4 * TR_GROUPS + 2] = {};
  cudaEvent_t kick = nullptr;  // timing-enabled (see the group loop)
};
int tri_pipe(TriPipe& T) {
  static TriPipe gs[kMaxDevices];  // streams and events belong to the device they were made on
  const int dev = current_device();
  if (dev < 0 || dev >= kMaxDevices) return fail(PFX_CUDA, "device index out of range");
  TriPipe& g = gs[dev];
  if (!g.in) {
    PFX_CUDA_TRY(cudaStreamCreateWithFlags(&g.in, cudaStreamNonBlocking));
    PFX_CUDA_TRY(cudaStreamCreateWithFlags(&g.outs, cudaStreamNonBlocking));
    // sweeps: the last-arriving rows are on the critical path -> later groups higher
    // priority; fixes: earlier groups go back over PCIe first -> earlier groups higher
    int lo = 0, hi = 0;
    PFX_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    for (int i = 0; i < TR_GROUPS; ++i) {
      const int pr = hi + (int)((int64_t)(lo - hi) * i / TR_GROUPS);
      PFX_CUDA_TRY(cudaStreamCreateWithPriority(&g.cs[i], cudaStreamNonBlocking, pr));
      PFX_CUDA_TRY(cudaStreamCreateWithPriority(&g.sw[TR_GROUPS - 1 - i], cudaStreamNonBlocking, pr));
    }
    for (auto& e : g.ev) PFX_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    PFX_CUDA_TRY(cudaEventCreate(&g.kick));
  }
  T = g;
  return PFX_OK;
}
}  // namespace

// V_host / out_host (optional, host mode with npairs <= 16): V is copied into the device
// buffer V in row groups on a copy stream, each group's sweep starts as soon as its rows
// have landed, and each group's result goes back as soon as its edge fix is done, so the
// PCIe transfers hide the compute (out is final only after the global carry scan, so the
// H2D and D2H phases themselves cannot overlap).
// Chunk partition: the sweep keeps 32 (chunk, 16-RHS tile) units resident per SM, so the
// chunks are sized to fill every SM in one wave (C2: 224 rows -> 4682 units on 148 SMs, where
// 256 rows left 20 SMs idle), within [32, TR_L] rows and a multiple of 32.  Row-sharded calls
// size them for one rank's share of the rows; rank r owns chunks [P r / R, P (r + 1) / R).
int tri_partition(int64_t N, int64_t nrhs, int rank, int nranks, int* L_, int* P_, int64_t* c0, int64_t* c1) {
  const int64_t slots = (int64_t)device_sms() * 2 * LS_WARPS * 4;
  const int64_t per = ceil_div(ceil_div(N, nranks) * ceil_div(nrhs, 16), slots);
  const int L = (int)std::min<int64_t>(TR_L, std::max<int64_t>(nranks > 1 ? 32 : 64, ceil_div(per, 32) * 32));
  const int P = (int)ceil_div(N, L);
  *L_ = L;
  *P_ = P;
  *c0 = (int64_t)P * rank / nranks;
  *c1 = (int64_t)P * (rank + 1) / nranks;
  return PFX_OK;
}

namespace {
// host-side composition of the ranks' aggregates (row sharding)
using zc = std::complex<double>;
inline zc zl(const double* p) { return zc(p[0], p[1]); }
}  // namespace

int tridiag_run(const double* diag, const double* off, int64_t N, const double* V, int64_t nrhs, double shift_c,
                const double2* theta_d, const double2* coef_d, int npairs, double* out, cudaStream_t stream,
                float* launch_ms, const double* V_host, double* out_host, const TriShard* sh) {
  const int rank = sh ? sh->rank : 0, nranks = sh ? sh->nranks : 1;
  int L = 0, P = 0;
  int64_t c0 = 0, c1 = 0;
  if (int rc = tri_partition(N, nrhs, rank, nranks, &L, &P, &c0, &c1)) return rc;
  if (V_host && npairs <= 16) {
    // host-memory pipeline: each row group is swept as its rows land, a partial wave whose
    // duration is one unit's latency (proportional to the chunk length); the compute hides
    // behind the copies, so short chunks (more, faster units per group) shorten the tail
    static const int hl = getenv("PFX_TRI_HOST_L") ? atoi(getenv("PFX_TRI_HOST_L")) : 96;
    L = std::max(32, std::min(TR_L, hl / 32 * 32));
    P = (int)ceil_div(N, L);
    c0 = 0;
    c1 = P;
  }
  const size_t nP = (size_t)P * npairs;
  const size_t nPR = nP * nrhs;
  const size_t nN = (size_t)N * npairs;
  const size_t nNf = npairs <= 16 ? 0 : nN;  // factor arrays only on the npairs > 16 path
  // + row-sharding exchange buffers: Moebius aggregates (4 per pair and direction) and entry
  // states (2), RHS-carry aggregates (2 per pair, rhs and direction) and entry carries (1)
  const size_t nX = (size_t)npairs * 2 * 6 + (size_t)npairs * nrhs * 2 * 3;
  size_t bytes = (nP * 4 * 2 + nP * 4 + nPR * 4 + nNf * 3 + nX) * sizeof(double2) + (size_t)P * sizeof(int) +
                 (TR_GROUPS + 1) * (size_t)nrhs * sizeof(unsigned long long) + 64;
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
  a.L = L;
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
  a.Lf = a.Gb + nPR;
  a.Lb = a.Lf + nNf;
  a.Wt = a.Lb + nNf;
  a.c0 = c0;
  a.c1 = c1;
  a.agg = 0;
  a.msin = nullptr;
  a.csin = nullptr;
  a.magg = a.Wt + nNf;
  double2* msin_d = a.magg + (size_t)npairs * 2 * 4;
  a.cagg = msin_d + (size_t)npairs * 2 * 2;
  double2* csin_d = a.cagg + (size_t)npairs * nrhs * 2 * 2;
  a.contr = reinterpret_cast<int*>(csin_d + (size_t)npairs * nrhs * 2);
  a.vmax = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(a.contr) + ((P * sizeof(int) + 15) & ~size_t(15)));
  a.out = out;
  PFX_CUDA_TRY(cudaMemsetAsync(a.contr, 0x01, (size_t)P * sizeof(int), stream));
  // max|V| per rhs: one slice per host-pipeline row group (+ the whole matrix), then a flag word
  int* trunc_flag = reinterpret_cast<int*>(a.vmax + (TR_GROUPS + 1) * (size_t)nrhs);
  PFX_CUDA_TRY(cudaMemsetAsync(a.vmax, 0, (TR_GROUPS + 1) * (size_t)nrhs * sizeof(unsigned long long) + sizeof(int),
                               stream));
  a.dirmask = 3;
  a.w0 = 0;
  a.w1 = P;
  a.cin_prev = 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (launch_ms) {
    PFX_CUDA_TRY(cudaEventCreate(&e0));
    PFX_CUDA_TRY(cudaEventCreate(&e1));
    PFX_CUDA_TRY(cudaEventRecord(e0, stream));
  }
  // all-gather of this rank's `cnt` doubles (host) through the caller's callback
  std::vector<double> xbuf;
  auto exchange = [&](const double2* dev_src, int64_t cnt, const double* extra, int64_t nextra) -> int {
    xbuf.assign((size_t)nranks * (cnt + nextra), 0.0);
    double* mine = xbuf.data() + (size_t)rank * (cnt + nextra);
    PFX_CUDA_TRY(cudaMemcpyAsync(mine, dev_src, (size_t)cnt * sizeof(double), cudaMemcpyDeviceToHost, stream));
    PFX_CUDA_TRY(cudaStreamSynchronize(stream));
    for (int64_t i = 0; i < nextra; ++i) mine[cnt + i] = extra[i];
    if (sh->allgather(sh->ctx, xbuf.data(), cnt + nextra) != 0) return fail(PFX_CUDA, "row-shard all-gather failed");
    return PFX_OK;
  };
  {
    int64_t th = (c1 - c0) * npairs * TR_SEG;
    if (th > 0) {
      PFX_LAUNCH("tri_mobius_chunks", stream, tri_mobius_chunks<<<(unsigned)ceil_div(th, 128), 128, 0, stream>>>(a));
      PFX_CUDA_TRY(cudaGetLastError());
    }
    if (nranks > 1) {
      // pivot carries across ranks: aggregate transfer of every rank's chunks, then the
      // state entering this rank's range (forward: ranks below, backward: ranks above)
      a.agg = 1;
      PFX_LAUNCH("tri_mobius_scan", stream, tri_mobius_scan<<<npairs * 2, TR_SCAN_T, 0, stream>>>(a));
      PFX_CUDA_TRY(cudaGetLastError());
      const int64_t cnt = (int64_t)npairs * 2 * 4 * 2;
      if (int rc = exchange(a.magg, cnt, nullptr, 0)) return rc;
      std::vector<double> s0((size_t)npairs * 2 * 2 * 2);
      for (int k = 0; k < npairs; ++k)
        for (int dir = 0; dir < 2; ++dir) {
          zc vn(1, 0), vd(0, 0);
          for (int j = dir == 0 ? 0 : nranks - 1; dir == 0 ? j < rank : j > rank; j += dir == 0 ? 1 : -1) {
            const double* m = xbuf.data() + (size_t)j * cnt + (size_t)(k * 2 + dir) * 8;
            const zc nn = zl(m) * vn + zl(m + 2) * vd, nd = zl(m + 4) * vn + zl(m + 6) * vd;
            const double mx = std::max({std::abs(nn.real()), std::abs(nn.imag()), std::abs(nd.real()),
                                        std::abs(nd.imag()), 1e-300});
            const double sc = std::ldexp(1.0, -std::ilogb(mx));
            vn = nn * sc;
            vd = nd * sc;
          }
          double* o = s0.data() + (size_t)(k * 2 + dir) * 4;
          o[0] = vn.real(), o[1] = vn.imag(), o[2] = vd.real(), o[3] = vd.imag();
        }
      PFX_CUDA_TRY(cudaMemcpyAsync(msin_d, s0.data(), s0.size() * sizeof(double), cudaMemcpyHostToDevice, stream));
      a.agg = 0;
      a.msin = msin_d;
    }
    PFX_LAUNCH("tri_mobius_scan", stream, tri_mobius_scan<<<npairs * 2, TR_SCAN_T, 0, stream>>>(a));
    PFX_CUDA_TRY(cudaGetLastError());
  }
  const bool ls = npairs <= 16;
  const bool pipe = V_host != nullptr;
  if (pipe && !ls) return fail(PFX_BADARG, "tridiag_run: host pipelining needs npairs <= 16");
  if (nranks > 1 && (pipe || !ls)) return fail(PFX_BADARG, "tridiag_run: row sharding needs device memory and npairs <= 16");
  // RHS carries across ranks (row sharding): aggregate affine maps + max|V| of every rank,
  // then the carries entering this rank's range and the global max|V| (fix-pass stop rule)
  auto carry_exchange = [&]() -> int {
    a.agg = 1;
    if (int rc = carry_scan(a, npairs, nrhs, stream)) return rc;
    std::vector<unsigned long long> vm((size_t)nrhs);
    PFX_CUDA_TRY(cudaMemcpyAsync(vm.data(), a.vmax, (size_t)nrhs * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                 stream));
    PFX_CUDA_TRY(cudaStreamSynchronize(stream));
    std::vector<double> vmd((size_t)nrhs);
    for (int64_t r = 0; r < nrhs; ++r) std::memcpy(&vmd[r], &vm[r], sizeof(double));
    const int64_t cnt = (int64_t)npairs * nrhs * 2 * 2 * 2;
    if (int rc = exchange(a.cagg, cnt, vmd.data(), nrhs)) return rc;
    const int64_t stride = cnt + nrhs;
    std::vector<double> x0((size_t)npairs * nrhs * 2 * 2);
    for (int64_t kr = 0; kr < (int64_t)npairs * nrhs; ++kr)
      for (int dir = 0; dir < 2; ++dir) {
        zc x(0, 0);
        for (int j = dir == 0 ? 0 : nranks - 1; dir == 0 ? j < rank : j > rank; j += dir == 0 ? 1 : -1) {
          const double* m = xbuf.data() + (size_t)j * stride + (size_t)(kr * 2 + dir) * 4;
          x = zl(m) * x + zl(m + 2);
        }
        x0[(size_t)(kr * 2 + dir) * 2] = x.real();
        x0[(size_t)(kr * 2 + dir) * 2 + 1] = x.imag();
      }
    for (int64_t r = 0; r < nrhs; ++r) {
      double m = 0.0;
      for (int j = 0; j < nranks; ++j) m = std::max(m, xbuf[(size_t)j * stride + cnt + r]);
      std::memcpy(&vm[r], &m, sizeof(double));
    }
    PFX_CUDA_TRY(cudaMemcpyAsync(csin_d, x0.data(), x0.size() * sizeof(double), cudaMemcpyHostToDevice, stream));
    PFX_CUDA_TRY(cudaMemcpyAsync(a.vmax, vm.data(), (size_t)nrhs * sizeof(unsigned long long), cudaMemcpyHostToDevice,
                                 stream));
    // the host vectors die with this scope: the copies must land first
    PFX_CUDA_TRY(cudaStreamSynchronize(stream));
    a.agg = 0;
    a.csin = csin_d;
    return PFX_OK;
  };
  LsArgs lsa{};
  if (ls) {
    // checkpoints live in arena slot 2 (L2-resident: 2 x P x 32 x 16 x 32 B); the fix data
    // (z per row and pair, both directions, plus the per-block bounds) in slot 7
    const size_t ckn = (size_t)P * LS_NBLK * 16;
    LsCk* ckbuf = static_cast<LsCk*>(scratch(2, 2 * ckn * sizeof(LsCk)));
    char* zbuf = static_cast<char*>(scratch(7, 2 * nN * sizeof(double2) + 2 * ckn * sizeof(double)));
    if (!ckbuf || !zbuf) return fail(PFX_CUDA, "tridiagonal checkpoint allocation failed");
    lsa.ckb = ckbuf;
    lsa.ckf = ckbuf + ckn;
    lsa.zf = reinterpret_cast<double2*>(zbuf);
    lsa.zb = lsa.zf + nN;
    lsa.lamf = reinterpret_cast<double*>(lsa.zb + nN);
    lsa.lamb = lsa.lamf + ckn;
    const int ntile = (int)ceil_div(nrhs, 16);
    const int smem = (int)(sizeof(LsSmem) * LS_WARPS * 2);
    const int smem_fix = (int)(sizeof(FzBuf) * 2 * LS_WARPS * 2);
    // phase B runs KM (>= npairs) pair slots: exact small widths keep a pole-sharded rank's
    // work closer to its share of the pairs
    using K = decltype(&tri_ls<16>);
    const K k0 = npairs <= 2    ? tri_ls<2>
                 : npairs <= 4  ? tri_ls<4>
                 : npairs <= 6  ? tri_ls<6>
                 : npairs <= 8  ? tri_ls<8>
                 : npairs <= 12 ? tri_ls<12>
                                : tri_ls<16>;
    const K k1 = npairs <= 2    ? tri_fixz<2>
                 : npairs <= 4  ? tri_fixz<4>
                 : npairs <= 6  ? tri_fixz<6>
                 : npairs <= 8  ? tri_fixz<8>
                 : npairs <= 12 ? tri_fixz<12>
                                : tri_fixz<16>;
    if (int rc = raise_smem_limit(reinterpret_cast<const void*>(k0), smem)) return rc;
    if (int rc = raise_smem_limit(reinterpret_cast<const void*>(k1), smem_fix)) return rc;
    // row groups: whole chunks, one launch each (a single group in device mode)
    const int ng = pipe ? (int)std::min<int64_t>(TR_GROUPS, P) : 1;
    auto grp = [&](int g, int64_t& c0, int64_t& c1) {
      c0 = (int64_t)P * g / ng;
      c1 = (int64_t)P * (g + 1) / ng;
    };
    auto launch_ls = [&](bool fix, int64_t c0, int64_t c1, cudaStream_t st, const TriArgs* aa = nullptr) -> int {
      const TriArgs& ta = aa ? *aa : a;
      LsArgs la = lsa;
      la.unit0 = c0 * ntile;
      la.unit1 = c1 * ntile;
      const unsigned blocks = (unsigned)ceil_div(la.unit1 - la.unit0, LS_WARPS * 2);
      if (blocks == 0) return PFX_OK;
      if (fix)
        PFX_LAUNCH("tri_fix", st, (k1<<<blocks, LS_WARPS * 32, smem_fix, st>>>(ta, la)));
      else
        PFX_LAUNCH("tri_sweep", st, (k0<<<blocks, LS_WARPS * 32, smem, st>>>(ta, la)));
      PFX_CUDA_TRY(cudaGetLastError());
      return PFX_OK;
    };
    if (!pipe) {
      if (int rc = launch_ls(false, c0, c1, stream)) return rc;
      if (nranks > 1)
        if (int rc = carry_exchange()) return rc;
      if (int rc = carry_scan(a, npairs, nrhs, stream)) return rc;
      if (int rc = launch_ls(true, c0, c1, stream)) return rc;
    } else {
      // events: [0, G) V group landed, [G, 2G) sweep done, [2G, 3G) result ready,
      // 4G: fork point, 4G + 1: all copies back
      TriPipe TP;
      if (int rc = tri_pipe(TP)) return rc;
      cudaEvent_t* ev = TP.ev;
      const int G = TR_GROUPS;
      static const bool tl = getenv("PFX_TRI_TIMELINE") != nullptr;
      static cudaEvent_t tev[5 * TR_GROUPS + 2];
      static bool tev_init = false;
      if (tl && !tev_init) {
        for (auto& e : tev) cudaEventCreate(&e);
        tev_init = true;
      }
      if (tl) cudaEventRecord(tev[5 * G], stream);
      // the copy-in starts at once: the staging buffers are idle on entry (every host-mode
      // call ends synchronised) and V does not feed the Moebius kernels
      PFX_CUDA_TRY(cudaEventRecord(ev[4 * G], stream));  // Moebius scan done
      for (int g = 0; g < ng; ++g) {
        int64_t c0, c1;
        grp(g, c0, c1);
        const int64_t r0 = c0 * L, r1 = std::min<int64_t>(c1 * L, N);
        PFX_CUDA_TRY(cudaMemcpyAsync(const_cast<double*>(V) + r0 * nrhs, V_host + r0 * nrhs,
                                     (size_t)(r1 - r0) * nrhs * sizeof(double), cudaMemcpyHostToDevice, TP.in));
        PFX_CUDA_TRY(cudaEventRecord(ev[g], TP.in));
        if (tl) cudaEventRecord(tev[g], TP.in);
      }
      auto sweep_group = [&](int g) -> int {
        int64_t c0, c1;
        grp(g, c0, c1);
        PFX_CUDA_TRY(cudaStreamWaitEvent(TP.sw[g], ev[4 * G], 0));  // after the Moebius scan
        PFX_CUDA_TRY(cudaStreamWaitEvent(TP.sw[g], ev[g], 0));
        TriArgs ag = a;
        ag.vmax = a.vmax + (size_t)g * nrhs;  // this group's max|V| (its fix's stop rule)
        if (int rc = launch_ls(false, c0, c1, TP.sw[g], &ag)) return rc;
        PFX_CUDA_TRY(cudaEventRecord(ev[G + g], TP.sw[g]));
        if (tl) cudaEventRecord(tev[G + g], TP.sw[g]);
        return PFX_OK;
      };
      // Carries per group instead of one global scan, so group g's fix and copy-back start
      // once group g + 1 is swept and overlap the copy-in of the later groups:
      //   forward: chained group to group on the main stream (each scan continues from the
      //     previous group's last chunk);
      //   backward: group g's carries are scanned from the end of group g + 1 with zero
      //     entering there.  The neglected term is below one unit roundoff of max|V| when the
      //     decay over group g + 1 is strong enough (tri_trunc_check, after every sweep; the
      //     call falls back to the global scans otherwise).
      // Each group's fix stops at one unit roundoff of its own rows' max|V| (stricter than the
      // whole matrix's).
      auto finish_group = [&](int g) -> int {
        int64_t c0, c1, n0, n1;
        grp(g, c0, c1);
        grp(std::min(g + 1, ng - 1), n0, n1);
        const int64_t r0 = c0 * L, r1 = std::min<int64_t>(c1 * L, N);
        TriArgs ag = a;
        ag.vmax = a.vmax + (size_t)g * nrhs;
        ag.c0 = c0;
        ag.c1 = c1;
        ag.w0 = c0;
        ag.w1 = c1;
        ag.dirmask = 1;
        ag.cin_prev = 1;
        PFX_CUDA_TRY(cudaStreamWaitEvent(stream, ev[G + g], 0));
        if (int rc = carry_scan(ag, npairs, nrhs, stream)) return rc;
        PFX_CUDA_TRY(cudaEventRecord(ev[3 * G + g], stream));
        // A timing-enabled event recorded on the main stream makes the driver submit its
        // queued work at once; without it the forward-carry chain (and the fixes and
        // copy-backs behind it) started late (C2 host call 5.31 -> 4.32 ms; a timing-disabled
        // event does not have the effect)
        PFX_CUDA_TRY(cudaEventRecord(TP.kick, stream));
        ag.c1 = n1;
        ag.dirmask = 2;
        ag.cin_prev = 0;
        PFX_CUDA_TRY(cudaStreamWaitEvent(TP.cs[g], ev[G + g], 0));
        PFX_CUDA_TRY(cudaStreamWaitEvent(TP.cs[g], ev[G + std::min(g + 1, ng - 1)], 0));
        if (int rc = carry_scan(ag, npairs, nrhs, TP.cs[g])) return rc;
        PFX_CUDA_TRY(cudaStreamWaitEvent(TP.cs[g], ev[3 * G + g], 0));
        ag.c1 = c1;
        if (int rc = launch_ls(true, c0, c1, TP.cs[g], &ag)) return rc;
        if (shift_c != 0.0) {
          PFX_LAUNCH("scale_kernel", TP.cs[g],
                     scale_rows<<<296, 256, 0, TP.cs[g]>>>(out + r0 * nrhs, (r1 - r0) * nrhs, exp(shift_c)));
          PFX_CUDA_TRY(cudaGetLastError());
        }
        PFX_CUDA_TRY(cudaEventRecord(ev[2 * G + g], TP.cs[g]));
        if (tl) cudaEventRecord(tev[2 * G + g], TP.cs[g]);
        PFX_CUDA_TRY(cudaStreamWaitEvent(TP.outs, ev[2 * G + g], 0));
        PFX_CUDA_TRY(cudaMemcpyAsync(out_host + r0 * nrhs, out + r0 * nrhs, (size_t)(r1 - r0) * nrhs * sizeof(double),
                                     cudaMemcpyDeviceToHost, TP.outs));
        if (tl) cudaEventRecord(tev[3 * G + g], TP.outs);
        return PFX_OK;
      };
      // enqueue order: a group's carries, fix and copy-back right after the next group's sweep
      // (the host reaches the first fix after two sweeps, not after all of them)
      if (tl) cudaEventRecord(tev[5 * G + 1], stream);
      for (int g = 0; g < ng; ++g) {
        if (int rc = sweep_group(g)) return rc;
        if (g > 0)
          if (int rc = finish_group(g - 1)) return rc;
      }
      if (int rc = finish_group(ng - 1)) return rc;
      if (tl) {
        cudaDeviceSynchronize();
        auto at = [&](int i) {
          float ms = 0;
          cudaEventElapsedTime(&ms, tev[5 * G], tev[i]);
          return ms;
        };
        fprintf(stderr, "[tri timeline ms] in:");
        for (int g = 0; g < ng; ++g) fprintf(stderr, " %.2f", at(g));
        fprintf(stderr, " | sweep:");
        for (int g = 0; g < ng; ++g) fprintf(stderr, " %.2f", at(G + g));
        fprintf(stderr, " | scan %.2f | fix:", at(5 * G + 1));
        for (int g = 0; g < ng; ++g) fprintf(stderr, " %.2f", at(2 * G + g));
        fprintf(stderr, " | out:");
        for (int g = 0; g < ng; ++g) fprintf(stderr, " %.2f", at(3 * G + g));
        fprintf(stderr, "\n");
      }
      // the main stream has waited for every sweep (forward chain): check the truncation while
      // the last groups are fixed and copied back
      PFX_LAUNCH("tri_trunc_check", stream,
                 tri_trunc_check<<<(unsigned)ceil_div((int64_t)(ng - 1) * npairs + 1, 8), 256, 0, stream>>>(a, ng,
                                                                                                       trunc_flag));
      PFX_CUDA_TRY(cudaGetLastError());
      PFX_CUDA_TRY(cudaEventRecord(ev[4 * G + 1], TP.outs));
      PFX_CUDA_TRY(cudaStreamWaitEvent(stream, ev[4 * G + 1], 0));
      int* hflag = pinned_word();
      if (!hflag) return fail(PFX_CUDA, "pinned status word allocation failed");
      PFX_CUDA_TRY(cudaMemcpyAsync(hflag, trunc_flag, sizeof(int), cudaMemcpyDeviceToHost, stream));
      if (int rc = sync_stream(stream)) return rc;
      static const bool rep = getenv("PFX_TRI_REPORT") != nullptr;
      if (rep) fprintf(stderr, "[tri host pipeline] truncation %s\n", *hflag ? "rejected: global fallback" : "accepted");
      if (*hflag) {
        // weak decay across a row group: redo the carries globally (V is on the device)
        TriArgs af = a;
        af.vmax = a.vmax + (size_t)TR_GROUPS * nrhs;
        if (int rc = launch_ls(false, 0, P, stream, &af)) return rc;
        if (int rc = carry_scan(af, npairs, nrhs, stream)) return rc;
        if (int rc = launch_ls(true, 0, P, stream, &af)) return rc;
        if (shift_c != 0.0) {
          PFX_LAUNCH("scale_kernel", stream,
                     scale_kernel<<<1184, 256, 0, stream>>>(out, (size_t)N * nrhs, exp(shift_c)));
          PFX_CUDA_TRY(cudaGetLastError());
        }
        PFX_CUDA_TRY(cudaMemcpyAsync(out_host, out, (size_t)N * nrhs * sizeof(double), cudaMemcpyDeviceToHost, stream));
      }
      shift_c = 0.0;  // applied per group above (or in the fallback)
    }
  } else {
    PFX_LAUNCH("tri_factor", stream, tri_factor<<<(unsigned)ceil_div((int64_t)P * npairs, 128), 128, 0, stream>>>(a));
    PFX_CUDA_TRY(cudaGetLastError());
    if (int rc = sweeps(a, stream, 0)) return rc;
    PFX_CUDA_TRY(cudaGetLastError());
    if (int rc = carry_scan(a, npairs, nrhs, stream)) return rc;
    if (int rc = sweeps(a, stream, 1)) return rc;
    PFX_CUDA_TRY(cudaGetLastError());
  }
  if (shift_c != 0.0) {
    const int64_t r0 = c0 * L, r1 = std::min<int64_t>(c1 * L, N);
    PFX_LAUNCH("scale_kernel", stream,
               scale_kernel<<<1184, 256, 0, stream>>>(out + r0 * nrhs, (size_t)(r1 - r0) * nrhs, exp(shift_c)));
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
