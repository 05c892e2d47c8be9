// Batched dense shifted solves with fused residue combine (configs C1, C3; small full-mode cases).
//
// Replaces the per-pair task of reference engine._run_tasks
// (/root/reference/pkg/src/pfexpm/engine.py:194-215):
//   K0  M = A - cI + theta_k I            fused into the load (engine.py:197, 299-301)
//   K1/K2 LU with partial pivoting         getrf semantics   (engine.py:200,203,208)
//   K3  Y = M^{-1} V,  Yc = M^{-H} V        getrs 'N' / 'C'   (engine.py:204-205)
//   K5  residue combine into a per-system slot                (engine.py:201,206,210-213)
//   K6  ascending-pair reduction + e^c scale (separate tiny kernel; engine.py:226-228,303-304)
//
// One persistent CTA per SM walks the (matrix, pair) systems.  Each system is
// factored in an L2-resident workspace slot with a blocked right-looking LU:
// the panel (up to d x NB complex) lives in shared memory, row interchanges are
// applied to the rest of the slot, U12 strips are solved in shared memory and
// the trailing update A22 -= L21 U12 runs on the FP64 tensor cores (DMMA
// m8n8k4, four real MMAs per complex 8x8x4 step) straight from the panel/strip
// in shared memory into accumulator fragments loaded from and stored back to
// the slot.
#include <cstdlib>

#include <vector>

#include "pfx_common.cuh"

namespace pfx {

constexpr int DB_THREADS = 256;
constexpr int DB_WARPS = DB_THREADS / 32;
constexpr int DB_SW = 64;  // strip width of the trailing update

struct DenseBatchArgs {
  const double* A;
  int a_complex;
  int d;
  int batch;
  const double* V;
  int v_complex;
  int ncols;  // RHS columns (action) or d (full)
  int full;
  int real_path;
  int solve_only;  // pfx_shifted_solve: stage = Y (complex), no combine
  double shift_c;
  const double2* theta;  // device, npairs
  const double2* coef;   // device, npairs
  int npairs;
  int aug;        // RHS columns carried through the LU (W is d x (d + aug)); 0 = separate solves
  double2* W;     // slots x d*d
  double2* Xa;    // slots x d*aug  carried right-hand sides
  int* ipiv;      // slots x d
  double2* Y;     // slots x d*ncols   (solution Y, or X in full mode)
  double2* Yc;    // slots x d*ncols   (complex action: M^{-H} V)
  double* stage;  // systems x d*ncols (x2 if complex)
  int* status;
  unsigned long long* dbg;  // optional: per-phase clock totals (PFX_DENSE_PHASES env)
};

__device__ __forceinline__ void block_argmax(double val, int idx, double* sv, int* si, double& best, int& bidx) {
  // max |.|_1, ties -> smallest index (izamax semantics)
  for (int off = 16; off > 0; off >>= 1) {
    double ov = __shfl_down_sync(0xffffffffu, val, off);
    int oi = __shfl_down_sync(0xffffffffu, idx, off);
    if (ov > val || (ov == val && oi < idx)) {
      val = ov;
      idx = oi;
    }
  }
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sv[warp] = val;
    si[warp] = idx;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    val = threadIdx.x < DB_WARPS ? sv[threadIdx.x] : -1.0;
    idx = threadIdx.x < DB_WARPS ? si[threadIdx.x] : 0x7fffffff;
    for (int off = 16; off > 0; off >>= 1) {
      double ov = __shfl_down_sync(0xffffffffu, val, off);
      int oi = __shfl_down_sync(0xffffffffu, idx, off);
      if (ov > val || (ov == val && oi < idx)) {
        val = ov;
        idx = oi;
      }
    }
    if (threadIdx.x == 0) {
      sv[0] = val;
      si[0] = idx;
    }
  }
  __syncthreads();
  best = sv[0];
  bidx = si[0];
  __syncthreads();
}

// ---------------------------------------------------------------------------
// LU of the d x d row-major slot W (in place), pivots into ipiv (0-based, global rows).
// Returns nonzero (in *sing) if an exactly zero pivot was met (factorization continues,
// as LAPACK does, and the caller reports PFX_SINGULAR).
// PIV = false: no interchanges (exp path: A Hermitian and Im(theta) > 0, so every pivot of
// A + theta I has |Im| >= Im(theta) > 0, SURVEY finding 7); one barrier per panel column.
// Xa (d x na, row-major): right-hand sides carried through the factorisation (row
// interchanges + per-panel forward elimination turn them into L^{-1} P v).  The panel head of
// the carried columns is broadcast through the strip buffer S (idle between the interchanges
// and the strips; >= 32 x 33 complex >= NB x 4).
// The trailing update uses the 3M complex product (three DMMAs per step) over NCH column
// chunks of the strip (fewer live accumulators per chunk for the register-capped variant).
template <int NB, bool PIV, int NCH>
__device__ void lu_blocked(double2* __restrict__ W, int* __restrict__ ipiv, int d, double2* __restrict__ Xa, int na,
                           double2* P, double2* S, double* red_v, int* red_i, int* s_piv, int* sing,
                           unsigned long long* dbg) {
  const size_t ldw = (size_t)d;
  long long tph = 0;
  constexpr int PS = NB + 1;        // padded panel row stride (double2)
  constexpr int SS = DB_SW + 1;     // padded strip row stride
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;

  for (int p = 0; p < d; p += NB) {
    const int jb = min(NB, d - p);
    const int m = d - p;
    // ---- load panel rows p..d-1, cols p..p+jb-1
    for (int e = tid; e < m * jb; e += DB_THREADS) {
      int r = e / jb, c = e - r * jb;
      P[r * PS + c] = W[(size_t)(p + r) * ldw + p + c];
    }
    __syncthreads();
    if (dbg && tid == 0) tph = clock64();
    // ---- unblocked getf2 on the panel, two barriers per column:
    //   A: per-warp argmax candidates are published; every thread reduces the 8 of them
    //   B: pivot row and displaced row are staged in prow/trow; then each thread eliminates
    //      its own rows (the interchange folded in) and tracks the next column's argmax.
    if (!PIV) {
      const int tpr = m <= DB_THREADS / 4 ? 4 : (m <= DB_THREADS / 2 ? 2 : 1);  // threads per row
      const int cq = tid % tpr;
      for (int jj = 0; jj < jb; ++jj) {
        __syncthreads();  // panel row jj is final
        const cplx pv = ld(&P[jj * PS + jj]);
        if (tid == 0) {
          s_piv[jj] = jj;
          ipiv[p + jj] = p + jj;
          if (pv.re == 0.0 && pv.im == 0.0) atomicOr(sing, ST_SINGULAR);
        }
        const cplx rp = (pv.re == 0.0 && pv.im == 0.0) ? mk(0.0, 0.0) : crcp_fast(pv);
        const double pabs = fabs(pv.re) + fabs(pv.im);
        // short panels: 2 or 4 threads share a row (interleaved groups of four columns), so the
        // dependent load -> update -> store rounds per column step shrink with the panel
        // (uniform trip count: every lane reaches the __syncwarp that orders the sharers' reads
        // of the column entry before the multiplier overwrites it)
        for (int rb = jj + 1; rb < m; rb += DB_THREADS / tpr) {
          const int r = rb + tid / tpr;
          const bool live = r < m;
          double2* row = &P[(live ? r : jj) * PS];
          const cplx xj = ld(&row[jj]);
          // partial-pivoting check (izamax on the updated column): row r would displace jj
          if (live && cq == 0 && fabs(xj.re) + fabs(xj.im) > pabs) atomicOr(sing, ST_PIVOT);
          const cplx l = cmul(xj, rp);
          const double2* prow_j = &P[jj * PS];
          // four columns per round: all loads first (this row is never the pivot row, but
          // the compiler cannot prove it), then the updates and stores
          for (int c = jj + 1 + 4 * cq; live && c < jb; c += 4 * tpr) {
            cplx x[4], y[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              x[u] = c + u < jb ? ld(&row[c + u]) : mk(0.0, 0.0);
              y[u] = c + u < jb ? ld(&prow_j[c + u]) : mk(0.0, 0.0);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (c + u < jb) st(&row[c + u], cfms(x[u], l, y[u]));
          }
          if (tpr > 1) __syncwarp();
          if (live && cq == 0) st(&row[jj], l);
        }
      }
    }
    double2* prow = S;           // strip buffer is idle during the panel
    double2* trow = S + 64;
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int r = tid; r < m && PIV; r += DB_THREADS) {
      double2 x = P[r * PS];
      double v = fabs(x.x) + fabs(x.y);
      if (v > bv) {
        bv = v;
        bi = r;
      }
    }
    for (int jj = 0; jj < jb && PIV; ++jj) {
      for (int off = 16; off > 0; off >>= 1) {
        double ov = __shfl_down_sync(0xffffffffu, bv, off);
        int oi = __shfl_down_sync(0xffffffffu, bi, off);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (lane == 0) {
        red_v[warp + 8 * (jj & 1)] = bv;
        red_i[warp + 8 * (jj & 1)] = bi;
      }
      __syncthreads();  // A
      double best = red_v[8 * (jj & 1)];
      int piv = red_i[8 * (jj & 1)];
      for (int w = 1; w < DB_WARPS; ++w) {
        double v = red_v[w + 8 * (jj & 1)];
        int i = red_i[w + 8 * (jj & 1)];
        if (v > best || (v == best && i < piv)) {
          best = v;
          piv = i;
        }
      }
      if (tid == 0) {
        s_piv[jj] = piv;
        ipiv[p + jj] = p + piv;
        if (best == 0.0) atomicOr(sing, ST_SINGULAR);
      }
      for (int c = tid; c < jb; c += DB_THREADS) {
        prow[c] = P[piv * PS + c];
        trow[c] = P[jj * PS + c];
      }
      __syncthreads();  // B
      const cplx pv = ld(&prow[jj]);
      const cplx rp = (pv.re == 0.0 && pv.im == 0.0) ? mk(0.0, 0.0) : crcp(pv);
      for (int c = tid; c < jb; c += DB_THREADS) P[jj * PS + c] = prow[c];
      bv = -1.0;
      bi = 0x7fffffff;
      for (int r = jj + 1 + tid; r < m; r += DB_THREADS) {
        const double2* src = (r == piv) ? trow : &P[r * PS];
        double2* dst = &P[r * PS];
        if (r == piv)
          for (int c = 0; c < jj; ++c) dst[c] = trow[c];  // the displaced row's multipliers move too
        const cplx l = cmul(ld(&src[jj]), rp);
        for (int c = jj + 1; c < jb; ++c) {
          const cplx v = cfms(ld(&src[c]), l, ld(&prow[c]));
          st(&dst[c], v);
          if (c == jj + 1) {
            const double av = fabs(v.re) + fabs(v.im);
            if (av > bv || (av == bv && r < bi)) {
              bv = av;
              bi = r;
            }
          }
        }
        st(&dst[jj], l);
      }
    }
    __syncthreads();
    if (dbg && tid == 0) {
      atomicAdd(&dbg[2], (unsigned long long)(clock64() - tph));
      tph = clock64();
    }
    // ---- write panel back
    for (int e = tid; e < m * jb; e += DB_THREADS) {
      int r = e / jb, c = e - r * jb;
      W[(size_t)(p + r) * ldw + p + c] = P[r * PS + c];
    }
    // ---- row interchanges on the columns outside the panel (in order, per column)
    for (int c = tid; c < d - jb + na && PIV; c += DB_THREADS) {
      const bool carried = c >= d - jb;  // columns of Xa
      const int col = carried ? c - (d - jb) : (c < p ? c : c + jb);
      double2* base = carried ? Xa : W;
      const size_t ld = carried ? (size_t)na : ldw;
      for (int jj = 0; jj < jb; ++jj) {
        int pr = s_piv[jj];
        if (pr != jj) {
          size_t a = (size_t)(p + jj) * ld + col, b = (size_t)(p + pr) * ld + col;
          double2 x = base[a];
          base[a] = base[b];
          base[b] = x;
        }
      }
    }
    __syncthreads();
    if (dbg && tid == 0) {
      atomicAdd(&dbg[3], (unsigned long long)(clock64() - tph));
      tph = clock64();
    }
    // ---- strips of the trailing columns: U12 = L11^{-1} A12, A22 -= L21 U12
    // ---- L11^{-1} (unit lower) over the panel's top block (the panel is already back in W,
    // and only L21 below it is read from here on): warp per column, lane = row, forward
    // substitution by shuffles.  The strips then apply it on DMMA instead of a dependent
    // triangular solve.
    {
      constexpr int CPW = NB / DB_WARPS;  // columns per warp
      cplx inv[CPW];
#pragma unroll
      for (int u = 0; u < CPW; ++u) {
        const int c = warp + u * DB_WARPS;
        cplx x = mk(lane == c ? 1.0 : 0.0, 0.0);
        for (int k = c; k < jb; ++k) {
          cplx xk;
          xk.re = __shfl_sync(0xffffffffu, x.re, k);
          xk.im = __shfl_sync(0xffffffffu, x.im, k);
          if (lane > k && lane < jb) x = cfms(x, ld(&P[lane * PS + k]), xk);
        }
        inv[u] = x;
      }
      __syncthreads();  // every read of L11 is done
#pragma unroll
      for (int u = 0; u < CPW; ++u) {
        const int c = warp + u * DB_WARPS;
        if (lane < jb && c < jb) st(&P[lane * PS + c], inv[u]);
      }
      __syncthreads();
    }
    // ---- carried right-hand sides: head = L11^{-1} head (warp per column; the result also
    // goes to shared memory), then tail -= L21 head (thread per row and column)
    if (na > 0) {
      double2* xs = S;
      for (int c = warp; c < na; c += DB_WARPS) {
        const cplx h = lane < jb ? ld(&Xa[(size_t)(p + lane) * na + c]) : mk(0.0, 0.0);
        cplx x = mk(0.0, 0.0);
        for (int k = 0; k < jb; ++k) {
          cplx hk;
          hk.re = __shfl_sync(0xffffffffu, h.re, k);
          hk.im = __shfl_sync(0xffffffffu, h.im, k);
          if (lane >= k && lane < jb) x = cfma(ld(&P[lane * PS + k]), hk, x);
        }
        if (lane < jb) {
          st(&Xa[(size_t)(p + lane) * na + c], x);
          st(&xs[c * NB + lane], x);
        }
      }
      __syncthreads();  // (also orders the xs reads before the first strip reuses S)
      for (int e = tid; e < (m - jb) * na; e += DB_THREADS) {
        const int r = e / na + jb, c = e - (r - jb) * na;
        cplx y = ld(&Xa[(size_t)(p + r) * na + c]);
#pragma unroll 4
        for (int k = 0; k < jb; ++k) y = cfms(y, ld(&P[r * PS + k]), ld(&xs[c * NB + k]));
        st(&Xa[(size_t)(p + r) * na + c], y);
      }
      __syncthreads();
    }
    for (int q = p + jb; q < d; q += DB_SW) {
      const int sw = min(DB_SW, d - q);
      for (int e = tid; e < jb * sw; e += DB_THREADS) {
        int r = e / sw, c = e - r * sw;
        S[r * SS + c] = W[(size_t)(p + r) * ldw + q + c];
      }
      __syncthreads();
      // U12 = L11^{-1} A12 on DMMA: output 8x8 tiles (NB/8 row tiles x sw/8 column tiles)
      // spread over the warps; results held in registers until every read of S is done
      {
        constexpr int MT = NB / 8;
        constexpr int TPW = (MT * (DB_SW / 8) + DB_WARPS - 1) / DB_WARPS;  // tiles per warp
        const int ntl = MT * ((sw + 7) >> 3);
        double cr[TPW][2], ci[TPW][2];
#pragma unroll
        for (int u = 0; u < TPW; ++u) {
          cr[u][0] = cr[u][1] = ci[u][0] = ci[u][1] = 0.0;
          const int tl = warp + u * DB_WARPS;
          if (tl < ntl) {
            const int mt = tl % MT, nt = tl / MT;
            for (int k0 = 0; k0 < jb; k0 += 4) {
              const int kk = k0 + t;
              double2 x = make_double2(0, 0), y = make_double2(0, 0);
              if (kk < jb) {
                x = P[(mt * 8 + g) * PS + kk];
                if (nt * 8 + g < sw) y = S[kk * SS + nt * 8 + g];
              }
              zmma884(cr[u], ci[u], x.x, x.y, y.x, y.y);
            }
          }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < TPW; ++u) {
          const int tl = warp + u * DB_WARPS;
          if (tl < ntl) {
            const int mt = tl % MT, nt = tl / MT;
            const int r = mt * 8 + g;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int c = nt * 8 + 2 * t + h;
              if (r < jb && c < sw) S[r * SS + c] = make_double2(cr[u][h], ci[u][h]);
            }
          }
        }
      }
      __syncthreads();
      for (int e = tid; e < jb * sw; e += DB_THREADS) {
        int r = e / sw, c = e - r * sw;
        W[(size_t)(p + r) * ldw + q + c] = S[r * SS + c];
      }
      if (dbg && tid == 0) {
        atomicAdd(&dbg[4], (unsigned long long)(clock64() - tph));
        tph = clock64();
      }
      // DMMA trailing update of rows p+jb..d-1, cols q..q+sw-1
      const int mrows = m - jb;
      const int rtiles = (mrows + 7) >> 3;
      const int ctiles = (sw + 7) >> 3;
      // 3M complex product (three DMMAs per complex 8x8x4 step): T1 = sum Lr Ur,
      // T2 = sum Li Ui, T3 = sum (Lr + Li)(Ur + Ui); C -= (T1 - T2, T3 - T1 - T2).  The strip's
      // column tiles go in NCH chunks (fewer live accumulators) and each chunk's C values are
      // fetched before its k loop, so the loads overlap the DMMAs.
      constexpr int CH = DB_SW / 8 / NCH;  // column tiles per chunk
      for (int rt = warp; rt < rtiles; rt += DB_WARPS) {
        const int grow = p + jb + rt * 8 + g;  // C row owned by this lane
        const int prow = jb + rt * 8 + g;      // panel row of the A fragment
#pragma unroll 1
        for (int hf = 0; hf < NCH; ++hf) {
          const int cb = hf * CH;
          if (cb >= ctiles) break;
          double t1[CH][2], t2[CH][2], t3[CH][2];
          double2 cv[CH][2];
#pragma unroll
          for (int u = 0; u < CH; ++u) {
            t1[u][0] = t1[u][1] = t2[u][0] = t2[u][1] = t3[u][0] = t3[u][1] = 0.0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int c0 = (cb + u) * 8 + 2 * t + h;
              cv[u][h] = (cb + u < ctiles && grow < d && c0 < sw) ? W[(size_t)grow * ldw + q + c0] : make_double2(0, 0);
            }
          }
          for (int k0 = 0; k0 < jb; k0 += 4) {
            double ar = 0.0, ai = 0.0;
            if (prow < m && k0 + t < jb) {
              double2 x = P[prow * PS + k0 + t];
              ar = x.x;
              ai = x.y;
            }
            const double as = ar + ai;
#pragma unroll
            for (int u = 0; u < CH; ++u) {
              if (cb + u < ctiles) {
                double br = 0.0, bi = 0.0;
                int col = (cb + u) * 8 + g;
                if (k0 + t < jb && col < sw) {
                  double2 y = S[(k0 + t) * SS + col];
                  br = y.x;
                  bi = y.y;
                }
                dmma884(t1[u][0], t1[u][1], ar, br);
                dmma884(t2[u][0], t2[u][1], ai, bi);
                dmma884(t3[u][0], t3[u][1], as, br + bi);
              }
            }
          }
#pragma unroll
          for (int u = 0; u < CH; ++u) {
            if (cb + u < ctiles && grow < d) {
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int c0 = (cb + u) * 8 + 2 * t + h;
                if (c0 < sw) {
                  double2 x = cv[u][h];
                  x.x -= t1[u][h] - t2[u][h];
                  x.y -= t3[u][h] - t1[u][h] - t2[u][h];
                  W[(size_t)grow * ldw + q + c0] = x;
                }
              }
            }
          }
        }
      }
      __syncthreads();
      if (dbg && tid == 0) {
        atomicAdd(&dbg[5], (unsigned long long)(clock64() - tph));
        tph = clock64();
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Interchange-free LU (exp path) with a delayed, two-panel trailing update (NB = 16 panels):
// the trailing matrix is streamed through L2 once per 32 columns instead of once per 16,
// which halves the dominant L2/DRAM traffic of the factorisation and doubles the DMMA work
// per C tile.  Per 32-column step at p (panels a = [p, p+16), b = [p+16, p+32)):
//   1. panel a: getf2 in shared memory, written back; L11a and Lba (its rows 16..31) are
//      copied into T; Ia = L11a^{-1} over T's top-left block; carried RHS updated.
//   2. look-ahead: panel b's columns get panel a's update only (a 16-column strip, K = 16).
//   3. panel b: getf2, written back; Ib = L11b^{-1}; carried RHS updated.
//      T becomes the full inverse of the 32 x 32 unit lower block:
//      [Ia 0; -Ib Lba Ia  Ib].
//   4. 32-column strips right of the step: U12 = T A12 (one product, K = 32), then
//      A22 -= [L21a L21b] U12 on DMMA (3M product, K = 32, A fragments from the slot).
// T: 32 x TST complex, S: 32 x TSS complex.  Same results as lu_blocked<16, false> up to rounding order.
// Strides chosen for conflict-free DMMA fragment loads: a quarter-warp reads rows t (0..3) and
// columns g (0..1) of an A operand (row stride = 4 mod 8 in 16-byte words) or rows t, columns g
// of a B operand stored k-major (row stride = 2 mod 8); with 33 both patterns were 2-way
// conflicted.
constexpr int TST = 36;  // T (A operand of the strip products)
constexpr int TSS = 34;  // S (B operand of the strip and trailing products)
#ifndef PFX_DP_CH
#define PFX_DP_CH 1  // column tiles per chunk of the two-panel update in the two-CTA variant
#endif
constexpr int DP_SW = 32;  // strip width of the two-panel update

// this warp's 8 x 8 complex tile (rt, ct) of C = A (rows x K, stride lda) * S (K x sw rows
// brow0.., stride ldb); rows >= arows and k >= K read as zero
__device__ __forceinline__ void dp_tile(const double2* A, size_t lda, int arows, int K, const double2* Sb, int ldb, int sw,
                                        int rt, int ct, int kbeg, double (&cr)[2], double (&ci)[2]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  cr[0] = cr[1] = ci[0] = ci[1] = 0.0;
  const int r = rt * 8 + g, col = ct * 8 + g;
  for (int k0 = kbeg; k0 < K; k0 += 4) {
    const int kk = k0 + t;
    double2 x = make_double2(0, 0), y = make_double2(0, 0);
    if (kk < K) {
      if (r < arows) x = A[(size_t)r * lda + kk];
      if (col < sw) y = Sb[kk * ldb + col];
    }
    zmma884(cr, ci, x.x, x.y, y.x, y.y);
  }
}

// unit lower inverse of the jb x jb block at T + off*(TST+1) (in place), warp per column
__device__ __forceinline__ void dp_inv16(double2* T, int off, int jb) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* B = T + off * (TST + 1);
  cplx inv[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int c = warp + u * DB_WARPS;
    cplx x = mk(lane == c ? 1.0 : 0.0, 0.0);
    for (int k = c; k < jb; ++k) {
      cplx xk;
      xk.re = __shfl_sync(0xffffffffu, x.re, k);
      xk.im = __shfl_sync(0xffffffffu, x.im, k);
      if (lane > k && lane < jb) x = cfms(x, ld(&B[lane * TST + k]), xk);
    }
    inv[u] = x;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int c = warp + u * DB_WARPS;
    if (lane < jb && c < jb) st(&B[lane * TST + c], lane >= c ? inv[u] : mk(0.0, 0.0));
  }
  __syncthreads();
}

template <int CH>
__device__ void lu_nopiv_dp(double2* __restrict__ W, int* __restrict__ ipiv, int d, double2* __restrict__ Xa, int na,
                            double2* P, double2* S, double2* T, int* s_piv, int* sing, unsigned long long* dbg) {
  constexpr int NB = 16;
  constexpr int PS = NB + 1;
  const size_t ldw = (size_t)d;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  long long tph = 0;

  // panel [p, p+jb) x rows [p, d): load, getf2 without interchanges, write back; L11 (and,
  // for panel a, the next 16 rows of L21) into T at toff; L11^{-1} over it; carried RHS.
  auto panel = [&](int p, int jb, int toff, bool keep_below) {
    const int m = d - p;
    for (int e = tid; e < m * jb; e += DB_THREADS) {
      const int r = e / jb, c = e - r * jb;
      P[r * PS + c] = W[(size_t)(p + r) * ldw + p + c];
    }
    __syncthreads();
    if (dbg && tid == 0) tph = clock64();
    const int tpr = m <= DB_THREADS / 4 ? 4 : (m <= DB_THREADS / 2 ? 2 : 1);  // threads per row
    const int cq = tid % tpr;
    for (int jj = 0; jj < jb; ++jj) {
      __syncthreads();  // panel row jj is final
      const cplx pv = ld(&P[jj * PS + jj]);
      if (tid == 0) {
        s_piv[jj] = jj;
        ipiv[p + jj] = p + jj;
        if (pv.re == 0.0 && pv.im == 0.0) atomicOr(sing, ST_SINGULAR);
      }
      const cplx rp = (pv.re == 0.0 && pv.im == 0.0) ? mk(0.0, 0.0) : crcp_fast(pv);
      const double pabs = fabs(pv.re) + fabs(pv.im);
      // short panels: 2 or 4 threads share a row (interleaved groups of four columns); uniform
      // trip count, so every lane reaches the __syncwarp before the multiplier is stored
      for (int rb = jj + 1; rb < m; rb += DB_THREADS / tpr) {
        const int r = rb + tid / tpr;
        const bool live = r < m;
        double2* row = &P[(live ? r : jj) * PS];
        const cplx xj = ld(&row[jj]);
        // partial-pivoting check (izamax on the updated column): row r would displace jj
        if (live && cq == 0 && fabs(xj.re) + fabs(xj.im) > pabs) atomicOr(sing, ST_PIVOT);
        const cplx l = cmul(xj, rp);
        const double2* prow_j = &P[jj * PS];
        for (int c = jj + 1 + 4 * cq; live && c < jb; c += 4 * tpr) {
          cplx x[4], y[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            x[u] = c + u < jb ? ld(&row[c + u]) : mk(0.0, 0.0);
            y[u] = c + u < jb ? ld(&prow_j[c + u]) : mk(0.0, 0.0);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (c + u < jb) st(&row[c + u], cfms(x[u], l, y[u]));
        }
        if (tpr > 1) __syncwarp();
        if (live && cq == 0) st(&row[jj], l);
      }
    }
    __syncthreads();
    if (dbg && tid == 0) {
      atomicAdd(&dbg[2], (unsigned long long)(clock64() - tph));
      tph = clock64();
    }
    for (int e = tid; e < m * jb; e += DB_THREADS) {
      const int r = e / jb, c = e - r * jb;
      W[(size_t)(p + r) * ldw + p + c] = P[r * PS + c];
    }
    // L11 (rows 0..jb) and, for panel a, the L21 rows jb..2 NB (Lba) into T
    const int tr = keep_below ? min(2 * NB, m) : jb;
    for (int e = tid; e < tr * NB; e += DB_THREADS) {
      const int r = e / NB, c = e - r * NB;
      T[(toff + r) * TST + toff + c] = c < jb ? P[r * PS + c] : make_double2(0, 0);
    }
    __syncthreads();
    dp_inv16(T, toff, jb);
    // carried right-hand sides: head = L11^{-1} head, tail -= L21 head
    if (na > 0) {
      double2* xs = S;
      const double2* I = T + toff * (TST + 1);
      for (int c = warp; c < na; c += DB_WARPS) {
        const cplx h = lane < jb ? ld(&Xa[(size_t)(p + lane) * na + c]) : mk(0.0, 0.0);
        cplx x = mk(0.0, 0.0);
        for (int k = 0; k < jb; ++k) {
          cplx hk;
          hk.re = __shfl_sync(0xffffffffu, h.re, k);
          hk.im = __shfl_sync(0xffffffffu, h.im, k);
          if (lane >= k && lane < jb) x = cfma(ld(&I[lane * TST + k]), hk, x);
        }
        if (lane < jb) {
          st(&Xa[(size_t)(p + lane) * na + c], x);
          st(&xs[c * NB + lane], x);
        }
      }
      __syncthreads();
      for (int e = tid; e < (m - jb) * na; e += DB_THREADS) {
        const int r = e / na + jb, c = e - (r - jb) * na;
        cplx y = ld(&Xa[(size_t)(p + r) * na + c]);
#pragma unroll 4
        for (int k = 0; k < jb; ++k) y = cfms(y, ld(&P[r * PS + k]), ld(&xs[c * NB + k]));
        st(&Xa[(size_t)(p + r) * na + c], y);
      }
      __syncthreads();
    }
  };

  // trailing update of rows [r0, d) x cols [q, q + sw): C -= L (slot columns [p, p + K)) * S
  // (K x sw at S, stride TSS), 3M product on DMMA; CH column tiles per chunk
  auto trailing = [&](int p, int K, int r0, int q, int sw) {
    const int rtiles = (d - r0 + 7) >> 3;
    const int ctiles = (sw + 7) >> 3;
    for (int rt = warp; rt < rtiles; rt += DB_WARPS) {
      const int grow = r0 + rt * 8 + g;
      // A fragments of this row tile for the whole K (<= 32): loaded once, reused by every chunk
      double ar[2 * NB / 4], ai[2 * NB / 4];
#pragma unroll
      for (int s4 = 0; s4 < 2 * NB / 4; ++s4) {
        const int kk = s4 * 4 + t;
        double2 x = make_double2(0, 0);
        if (grow < d && kk < K) x = W[(size_t)grow * ldw + p + kk];
        ar[s4] = x.x;
        ai[s4] = x.y;
      }
#pragma unroll 1
      for (int cb = 0; cb < ctiles; cb += CH) {
        double t1[CH][2], t2[CH][2], t3[CH][2];
        double2 cv[CH][2];
#pragma unroll
        for (int u = 0; u < CH; ++u) {
          t1[u][0] = t1[u][1] = t2[u][0] = t2[u][1] = t3[u][0] = t3[u][1] = 0.0;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c0 = (cb + u) * 8 + 2 * t + h;
            cv[u][h] = (grow < d && c0 < sw) ? W[(size_t)grow * ldw + q + c0] : make_double2(0, 0);
          }
        }
#pragma unroll
        for (int s4 = 0; s4 < 2 * NB / 4; ++s4) {
          if (s4 * 4 < K) {
            const int kk = s4 * 4 + t;
            const double as = ar[s4] + ai[s4];
#pragma unroll
            for (int u = 0; u < CH; ++u) {
              const int col = (cb + u) * 8 + g;
              double2 y = make_double2(0, 0);
              if (kk < K && col < sw) y = S[kk * TSS + col];
              dmma884(t1[u][0], t1[u][1], ar[s4], y.x);
              dmma884(t2[u][0], t2[u][1], ai[s4], y.y);
              dmma884(t3[u][0], t3[u][1], as, y.x + y.y);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < CH; ++u) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c0 = (cb + u) * 8 + 2 * t + h;
            if (grow < d && c0 < sw) {
              double2 x = cv[u][h];
              x.x -= t1[u][h] - t2[u][h];
              x.y -= t3[u][h] - t1[u][h] - t2[u][h];
              W[(size_t)grow * ldw + q + c0] = x;
            }
          }
        }
      }
    }
  };

  // strip rows [p, p + K) x cols [q, q + sw) of the slot -> S; U12 = T(K x K, lower) S in
  // place (written back to the slot); then the trailing update below it
  auto strip = [&](int p, int K, int q, int sw) {
    for (int e = tid; e < K * sw; e += DB_THREADS) {
      const int r = e / sw, c = e - r * sw;
      S[r * TSS + c] = W[(size_t)(p + r) * ldw + q + c];
    }
    __syncthreads();
    // K x sw output: (K/8) x (sw/8) tiles, at most 16 over 8 warps; T is lower triangular,
    // so row tile rt only needs k < 8 (rt + 1)
    const int mtl = (K + 7) >> 3, ntl = (sw + 7) >> 3;
    double cr[2][2], ci[2][2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int tl = warp + u * DB_WARPS;
      if (tl < mtl * ntl) {
        const int rt = tl % mtl, ct = tl / mtl;
        dp_tile(T, TST, K, min(K, 8 * (rt + 1)), S, TSS, sw, rt, ct, 0, cr[u], ci[u]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int tl = warp + u * DB_WARPS;
      if (tl < mtl * ntl) {
        const int rt = tl % mtl, ct = tl / mtl;
        const int r = rt * 8 + g;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = ct * 8 + 2 * t + h;
          if (r < K && c < sw) S[r * TSS + c] = make_double2(cr[u][h], ci[u][h]);
        }
      }
    }
    __syncthreads();
    for (int e = tid; e < K * sw; e += DB_THREADS) {
      const int r = e / sw, c = e - r * sw;
      W[(size_t)(p + r) * ldw + q + c] = S[r * TSS + c];
    }
    if (dbg && tid == 0) {
      atomicAdd(&dbg[4], (unsigned long long)(clock64() - tph));
      tph = clock64();
    }
    trailing(p, K, p + K, q, sw);
    __syncthreads();
    if (dbg && tid == 0) {
      atomicAdd(&dbg[5], (unsigned long long)(clock64() - tph));
      tph = clock64();
    }
  };

  for (int p = 0; p < d; p += 2 * NB) {
    const int ja = min(NB, d - p);
    const int jb = min(NB, d - p - ja);  // 0: panel a is the last
    for (int e = tid; e < 2 * NB * TST; e += DB_THREADS) T[e] = make_double2(0, 0);
    __syncthreads();
    panel(p, ja, 0, jb > 0);
    if (jb == 0) {
      // last (partial) step: the columns right of panel a are none
      break;
    }
    // look-ahead: panel b's columns with panel a's update (T's top-left block holds Ia)
    strip(p, ja, p + ja, jb);
    panel(p + ja, jb, NB, false);
    // T's bottom-left block: -Ib Lba Ia (two 16 x 16 x 16 products, four warps)
    {
      double2* L = T + NB * TST;  // Lba
      double cr[2], ci[2];
      const int rt = warp & 1, ct = (warp >> 1) & 1;
      if (warp < 4) dp_tile(L, TST, jb, ja, T, TST, ja, rt, ct, 0, cr, ci);  // Lba Ia (Ia at T)
      __syncthreads();
      if (warp < 4) {
#pragma unroll
        for (int h = 0; h < 2; ++h) L[(rt * 8 + g) * TST + ct * 8 + 2 * t + h] = make_double2(cr[h], ci[h]);
      }
      __syncthreads();
      // -Ib (Lba Ia): B operand = rows of L -> through dp_tile with Sb = L
      if (warp < 4) dp_tile(T + NB * (TST + 1), TST, jb, jb, L, TST, ja, rt, ct, 0, cr, ci);
      __syncthreads();
      if (warp < 4) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = rt * 8 + g, c = ct * 8 + 2 * t + h;
          L[r * TST + c] = (r < jb && c < ja) ? make_double2(-cr[h], -ci[h]) : make_double2(0, 0);
        }
      }
      __syncthreads();
    }
    const int K = ja + jb;
    for (int q = p + K; q < d; q += DP_SW) strip(p, K, q, min(DP_SW, d - q));
  }
}

// ---------------------------------------------------------------------------
// Triangular solves on one RHS column z (shared memory, length d) against the LU in W.
// kind 0: L  (unit lower, forward)      z <- L^{-1} z
// kind 1: U  (upper, backward)          z <- U^{-1} z
// kind 2: U^H (lower, forward, conj)    z <- U^{-H} z
// kind 3: L^H (unit upper, backward)    z <- L^{-H} z
// Blocked by 32 rows: the contribution of already-solved blocks is a GEMV with
// coalesced reads of W, the 32x32 diagonal block is solved by warp 0 in registers.
__device__ void trsv_blocked(const double2* __restrict__ W, int d, size_t ldw, int kind, double2* z, double2* part,
                             double2* diag, const double2* rdiag) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool forward = (kind == 0 || kind == 2);
  const int nblk = (d + 31) >> 5;
  for (int bb = 0; bb < nblk; ++bb) {
    const int blk = forward ? bb : nblk - 1 - bb;
    const int i0 = blk * 32;
    const int bs = min(32, d - i0);
    // previously solved index range
    const int j0 = forward ? 0 : i0 + bs;
    const int j1 = forward ? i0 : d;
    // GEMV: part[i] = sum_j op(W)[i][j] z[j]
    if (kind <= 1) {
      // rows of W are contiguous: warp w handles rows i0+w, i0+w+8, i0+w+16, i0+w+24 together
      // (four independent L2 loads per column step, two column steps per round); lanes stride j
      constexpr int RW = 32 / DB_WARPS;  // rows per warp
      cplx acc[RW];
#pragma unroll
      for (int u = 0; u < RW; ++u) acc[u] = mk(0.0, 0.0);
      for (int j = j0 + lane; j < j1; j += 64) {
        const bool j2 = j + 32 < j1;
        const cplx z0 = ld(&z[j]), z1 = j2 ? ld(&z[j + 32]) : mk(0.0, 0.0);
        cplx w0[RW], w1[RW];
#pragma unroll
        for (int u = 0; u < RW; ++u) {
          const int ii = warp + u * DB_WARPS;
          const double2* row = W + (size_t)(i0 + ii) * ldw;
          w0[u] = ii < bs ? ld(&row[j]) : mk(0.0, 0.0);
          w1[u] = (ii < bs && j2) ? ld(&row[j + 32]) : mk(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < RW; ++u) acc[u] = cfma(w1[u], z1, cfma(w0[u], z0, acc[u]));
      }
#pragma unroll
      for (int u = 0; u < RW; ++u) {
        for (int off = 16; off > 0; off >>= 1) {
          acc[u].re += __shfl_down_sync(0xffffffffu, acc[u].re, off);
          acc[u].im += __shfl_down_sync(0xffffffffu, acc[u].im, off);
        }
        const int ii = warp + u * DB_WARPS;
        if (lane == 0 && ii < bs) st(&part[ii], acc[u]);
      }
    } else {
      // op(W)[i][j] = conj(W[j][i]): lanes along i (contiguous in row j), warps stride j
      cplx acc = mk(0.0, 0.0);
      if (lane < bs)
        for (int j = j0 + warp; j < j1; j += DB_WARPS) acc = cadd(acc, cmulc(ld(&z[j]), ld(&W[(size_t)j * ldw + i0 + lane])));
      // reduce over warps through shared memory (diag scratch as buffer)
      st(&diag[warp * 32 + lane], acc);
      __syncthreads();
      if (warp == 0) {
        cplx s = mk(0.0, 0.0);
        for (int w = 0; w < DB_WARPS; ++w) s = cadd(s, ld(&diag[w * 32 + lane]));
        if (lane < bs) st(&part[lane], s);
      }
    }
    __syncthreads();
    // load the diagonal block (op applied) into shared memory: diag[r*33 + c] = op(W)[i0+r][i0+c]
    for (int e = tid; e < bs * bs; e += DB_THREADS) {
      int r = e / bs, c = e - r * bs;
      cplx v = (kind <= 1) ? ld(&W[(size_t)(i0 + r) * ldw + i0 + c]) : cconj(ld(&W[(size_t)(i0 + c) * ldw + i0 + r]));
      st(&diag[r * 33 + c], v);
    }
    __syncthreads();
    if (warp == 0) {
      cplx x = (lane < bs) ? csub(ld(&z[i0 + lane]), ld(&part[lane])) : mk(0.0, 0.0);
      const bool unit = (kind == 0 || kind == 3);
      if (forward) {
        for (int k = 0; k < bs; ++k) {
          cplx xk;
          xk.re = __shfl_sync(0xffffffffu, x.re, k);
          xk.im = __shfl_sync(0xffffffffu, x.im, k);
          if (!unit) {
            const cplx rd = ld(&rdiag[i0 + k]);
            xk = cmul(xk, kind == 2 ? cconj(rd) : rd);
            if (lane == k) x = xk;
          }
          if (lane > k && lane < bs) x = cfms(x, ld(&diag[lane * 33 + k]), xk);
        }
      } else {
        for (int k = bs - 1; k >= 0; --k) {
          cplx xk;
          xk.re = __shfl_sync(0xffffffffu, x.re, k);
          xk.im = __shfl_sync(0xffffffffu, x.im, k);
          if (!unit) {
            const cplx rd = ld(&rdiag[i0 + k]);
            xk = cmul(xk, kind == 2 ? cconj(rd) : rd);
            if (lane == k) x = xk;
          }
          if (lane < k) x = cfms(x, ld(&diag[lane * 33 + k]), xk);
        }
      }
      if (lane < bs) st(&z[i0 + lane], x);
    }
    __syncthreads();
  }
}

// NB = panel width; MINB = resident CTAs per SM the register budget is sized for.
//   <32, 1>: few systems (latency mode, e.g. C1);  <16, 2>: many systems with d <= 256
//   (two CTAs per SM overlap one system's panel with another's DMMA update, e.g. C3);
//   <16, 1>: 256 < d <= 512.
template <int NB, int MINB, bool PIV>
__global__ void __launch_bounds__(DB_THREADS, MINB) dense_batched_kernel(DenseBatchArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int d = a.d;
  double2* P = reinterpret_cast<double2*>(smem_raw);                // d x (NB+1)
  double2* S = P + (size_t)d * (NB + 1);                            // NB x (SW+1), aliased by diag
  double2* diag = S;                                                // 32 x 33 (solves only)
  const size_t sreg = (size_t)NB * (DB_SW + 1) > 32 * TSS ? (size_t)NB * (DB_SW + 1) : 32 * TSS;
  double2* T = S + sreg;                                            // 32 x TST (two-panel LU)
  double2* part = T + 32 * TST;                                     // 32
  double* red_v = reinterpret_cast<double*>(part + 32);             // 32
  int* red_i = reinterpret_cast<int*>(red_v + 32);                  // 32
  int* s_piv = red_i + 32;                                          // NB
  int* s_sing = s_piv + NB;                                         // 1
  int* s_perm = s_sing + 4;                                         // d  (row permutation)
  // solve-phase vectors live in the panel buffer (idle after the factorisation)
  double2* z = P;                                                   // d
  double2* zc = z + d;                                              // d
  double2* rdiag = zc + d;                                          // d  (1 / U_ii)

  const int tid = threadIdx.x;
  const int slot = blockIdx.x;
  const size_t ldw = (size_t)d;
  double2* W = a.W + (size_t)slot * d * ldw;
  double2* Xa = a.Xa + (size_t)slot * d * a.aug;
  int* ipiv = a.ipiv + (size_t)slot * d;
  const int nsys = a.batch * a.npairs;
  const size_t dd = (size_t)d * d;
  const int nc = a.ncols;

  for (int sys = blockIdx.x; sys < nsys; sys += gridDim.x) {
    const int b = sys / a.npairs, k = sys - b * a.npairs;
    const cplx th = ld(&a.theta[k]);
    const cplx co = ld(&a.coef[k]);
    long long t_sys0 = clock64();
    if (tid == 0) *s_sing = 0;
    // ---- K0: M = A_b - cI + theta I into the slot
    // rows of A into the slot (row stride ldw); warp per row, lanes along the row, four rows
    // per round so each lane keeps several independent loads in flight
    {
      const int warp = tid >> 5, lane = tid & 31;
      for (int i0 = warp * 4; i0 < d; i0 += DB_WARPS * 4) {
        if (a.a_complex) {
          const double2* Ab = reinterpret_cast<const double2*>(a.A) + (size_t)b * dd;
          for (int c = lane; c < d; c += 32) {
            double2 x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = i0 + u < d ? Ab[(size_t)(i0 + u) * d + c] : make_double2(0, 0);
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (i0 + u < d) W[(size_t)(i0 + u) * ldw + c] = x[u];
          }
        } else {
          const double* Ab = a.A + (size_t)b * dd;
          for (int c = lane; c < d; c += 32) {
            double x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = i0 + u < d ? Ab[(size_t)(i0 + u) * d + c] : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (i0 + u < d) W[(size_t)(i0 + u) * ldw + c] = make_double2(x[u], 0.0);
          }
        }
      }
      // right-hand sides carried through the factorisation
      for (int e = tid; e < d * a.aug; e += DB_THREADS) {
        const int i = e / a.aug, c = e - i * a.aug;
        const size_t vi = ((size_t)b * d + i) * nc + c;
        Xa[(size_t)i * a.aug + c] =
            a.v_complex ? reinterpret_cast<const double2*>(a.V)[vi] : make_double2(a.V[vi], 0.0);
      }
    }
    __syncthreads();
    for (int i = tid; i < d; i += DB_THREADS) {
      double2 x = W[(size_t)i * ldw + i];
      x.x = (x.x - a.shift_c) + th.re;
      x.y = x.y + th.im;
      W[(size_t)i * ldw + i] = x;
    }
    __syncthreads();
    if (a.dbg && tid == 0) atomicAdd(&a.dbg[7], (unsigned long long)(clock64() - t_sys0));
    // ---- K1/K2: LU with partial pivoting
    long long t_lu0 = clock64();
    if constexpr (NB == 16 && !PIV)
      lu_nopiv_dp<MINB == 1 ? 4 : PFX_DP_CH>(W, ipiv, d, Xa, a.aug, P, S, T, s_piv, s_sing, a.dbg);
    else
      lu_blocked<NB, PIV, MINB == 1 ? 2 : 4>(W, ipiv, d, Xa, a.aug, P, S, red_v, red_i, s_piv, s_sing, a.dbg);
    __syncthreads();
    if (a.dbg && tid == 0) atomicAdd(&a.dbg[0], (unsigned long long)(clock64() - t_lu0));
    long long t_sv0 = clock64();
    // row permutation of P M = L U (swaps applied in order to the identity) and 1/U_ii
    for (int i = tid; i < d; i += DB_THREADS) {
      s_perm[i] = ipiv[i];
      const cplx u = ld(&W[(size_t)i * ldw + i]);
      st(&rdiag[i], (u.re == 0.0 && u.im == 0.0) ? mk(0.0, 0.0) : crcp(u));
    }
    __syncthreads();
    __syncthreads();
    if (tid == 0 && PIV) {
      // s_perm holds ipiv; apply the swaps in order to the identity, in shared memory
      int* piv = s_perm;
      // walk backwards-compatible: build perm in rdiag-free scratch (the S strip buffer)
      int* perm = reinterpret_cast<int*>(S);
      for (int i = 0; i < d; ++i) perm[i] = i;
      for (int i = 0; i < d; ++i) {
        const int pr = piv[i];
        if (pr != i) {
          const int t = perm[i];
          perm[i] = perm[pr];
          perm[pr] = t;
        }
      }
    }
    __syncthreads();
    for (int i = tid; i < d; i += DB_THREADS) s_perm[i] = PIV ? reinterpret_cast<int*>(S)[i] : i;
    __syncthreads();
    if (tid == 0 && *s_sing) atomicOr(a.status, *s_sing);
    // ---- K3: solves, one RHS column at a time through shared memory
    double2* Yg = a.Y + (size_t)slot * d * nc;
    double2* Ycg = a.Yc ? a.Yc + (size_t)slot * d * nc : nullptr;
    const bool want_conj = (!a.full) && (!a.real_path) && (!a.solve_only);
    for (int c = 0; c < nc; ++c) {
      // load RHS column (identity column in full mode)
      auto rhs = [&](int i) -> double2 {
        if (a.full) return make_double2(i == c ? 1.0 : 0.0, 0.0);
        if (a.v_complex) return reinterpret_cast<const double2*>(a.V)[((size_t)b * d + i) * nc + c];
        return make_double2(a.V[((size_t)b * d + i) * nc + c], 0.0);
      };
      // Y = U^{-1} L^{-1} P V : P applied as a gather through the permutation; a carried
      // column already holds L^{-1} P v
      const bool carried = c < a.aug;
      for (int i = tid; i < d; i += DB_THREADS) {
        z[i] = carried ? Xa[(size_t)i * a.aug + c] : rhs(s_perm[i]);
        zc[i] = rhs(i);
      }
      __syncthreads();
      if (!carried) trsv_blocked(W, d, ldw, 0, z, part, diag, rdiag);
      trsv_blocked(W, d, ldw, 1, z, part, diag, rdiag);
      for (int i = tid; i < d; i += DB_THREADS) Yg[(size_t)i * nc + c] = z[i];
      if (want_conj) {
        // Yc = M^{-H} V = P^T L^{-H} U^{-H} V
        trsv_blocked(W, d, ldw, 2, zc, part, diag, rdiag);
        trsv_blocked(W, d, ldw, 3, zc, part, diag, rdiag);
        // P^T applied as a scatter through the permutation
        for (int i = tid; i < d; i += DB_THREADS) Ycg[(size_t)s_perm[i] * nc + c] = zc[i];
      }
      __syncthreads();
    }
    __syncthreads();
    if (a.dbg && tid == 0) atomicAdd(&a.dbg[1], (unsigned long long)(clock64() - t_sv0));
    // ---- K5: residue combine into this system's slot of the stage buffer
    const size_t ne = (size_t)d * nc;
    if (a.solve_only) {
      double2* out = reinterpret_cast<double2*>(a.stage) + (size_t)sys * ne;
      for (size_t e = tid; e < ne; e += DB_THREADS) out[e] = Yg[e];
    } else if (a.real_path) {
      double* out = a.stage + (size_t)sys * ne;
      for (size_t e = tid; e < ne; e += DB_THREADS) {
        cplx y = ld(&Yg[e]);
        out[e] = 2.0 * fma(co.re, y.re, -co.im * y.im);
      }
    } else if (!a.full) {
      double2* out = reinterpret_cast<double2*>(a.stage) + (size_t)sys * ne;
      for (size_t e = tid; e < ne; e += DB_THREADS) {
        cplx v = cadd(cmul(co, ld(&Yg[e])), cmul(cconj(co), ld(&Ycg[e])));
        st(&out[e], v);
      }
    } else {
      double2* out = reinterpret_cast<double2*>(a.stage) + (size_t)sys * ne;
      for (size_t e = tid; e < ne; e += DB_THREADS) {
        int i = (int)(e / d), j = (int)(e - (size_t)i * d);
        cplx x = cmul(co, ld(&Yg[e]));
        cplx y = cconj(cmul(co, ld(&Yg[(size_t)j * d + i])));
        st(&out[e], cadd(x, y));
      }
    }
    __syncthreads();
    if (a.dbg && tid == 0) atomicAdd(&a.dbg[6], (unsigned long long)(clock64() - t_sys0));
  }
}

// K6: out[b] = e^c * sum_k stage[b*npairs + k]  (ascending k, bitwise deterministic)
__global__ void reduce_pairs_kernel(const double* __restrict__ stage, double* __restrict__ out, int batch,
                                    int npairs, size_t per_sys, double scale) {
  size_t total = (size_t)batch * per_sys;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    size_t b = e / per_sys, r = e - b * per_sys;
    const double* base = stage + b * npairs * per_sys + r;
    double acc = base[0];
    for (int k = 1; k < npairs; ++k) acc = acc + base[(size_t)k * per_sys];
    out[e] = scale == 1.0 ? acc : scale * acc;
  }
}

static size_t dense_smem_bytes(int d, int nb) {
  size_t sreg = (size_t)nb * (DB_SW + 1) > 32 * TSS ? (size_t)nb * (DB_SW + 1) : 32 * TSS;
  // panel (z, zc, 1/U_ii alias it in the solves) + strip + T (32 x 33) + part
  size_t c2 = (size_t)d * (nb + 1) + sreg + 32 * TST + 32;
  return c2 * sizeof(double2) + 32 * sizeof(double) + (32 + nb + 4) * sizeof(int) + ((d + 3) & ~3) * sizeof(int) + 64;
}

int dense_batched_supported(int64_t d) { return d >= 1 && d <= 512; }

// resident CTAs (= concurrently factored systems) of dense_batched_run for nsys systems of size d
int dense_batched_slots(int d, int64_t nsys) {
  const int sms = device_sms();
  const bool many = nsys > sms;
  return (d <= 256 && many) ? 2 * sms : sms;
}

// Launch the batched path.  All pointers are device pointers.
int dense_batched_run(const double* A, int a_complex, int d, int batch, const double* V, int v_complex, int ncols,
                      int full, int real_path, int solve_only, double shift_c, const double2* theta_d, const double2* coef_d,
                      int npairs, double* out, cudaStream_t stream, float* launch_ms, int pivot) {
  const int sms = device_sms();
  const int dev_sms = sms;
  const bool many = (int64_t)batch * npairs > dev_sms;
  const int nb = (d <= 256 && !many) ? 32 : 16;
  const int minb = (d <= 256 && many) ? 2 : 1;
  const size_t smem = dense_smem_bytes(d, nb);
  const int nsys = batch * npairs;
  const int slots = nsys < minb * sms ? nsys : minb * sms;
  const size_t per_sys = (size_t)d * ncols;
  // action mode with a few right-hand sides: carry them through the LU (forward solve free)
  const int aug = (!full && ncols <= 4) ? ncols : 0;

  const size_t stage_elems = (size_t)nsys * per_sys * (real_path ? 1 : 2);
  char* ws = static_cast<char*>(scratch(1, (size_t)slots * ((size_t)d * (d + aug) + 2 * per_sys) * sizeof(double2) +
                                               (size_t)slots * d * sizeof(int) + sizeof(int) + 256));
  if (!ws) return fail(PFX_CUDA, "dense workspace allocation failed");
  double* stage = static_cast<double*>(scratch(2, stage_elems * sizeof(double)));
  if (!stage) return fail(PFX_CUDA, "dense stage allocation failed");
  DenseBatchArgs args;
  args.A = A;
  args.a_complex = a_complex;
  args.d = d;
  args.batch = batch;
  args.V = V;
  args.v_complex = v_complex;
  args.ncols = ncols;
  args.full = full;
  args.real_path = real_path;
  args.solve_only = solve_only;
  args.shift_c = shift_c;
  args.theta = theta_d;
  args.coef = coef_d;
  args.npairs = npairs;
  args.aug = aug;
  args.W = reinterpret_cast<double2*>(ws);
  args.Xa = args.W + (size_t)slots * d * d;
  args.Y = args.Xa + (size_t)slots * d * aug;
  args.Yc = args.Y + (size_t)slots * per_sys;
  args.ipiv = reinterpret_cast<int*>(args.Yc + (size_t)slots * per_sys);
  args.status = args.ipiv + (size_t)slots * d;
  args.stage = stage;
  args.dbg = nullptr;
  static unsigned long long* dbg_devs[kMaxDevices] = {};
  if (getenv("PFX_DENSE_PHASES")) {
    unsigned long long*& dbg_dev = dbg_devs[current_device() & (kMaxDevices - 1)];
    if (!dbg_dev) PFX_CUDA_TRY(cudaMalloc(&dbg_dev, 8 * sizeof(unsigned long long)));
    PFX_CUDA_TRY(cudaMemsetAsync(dbg_dev, 0, 8 * sizeof(unsigned long long), stream));
    args.dbg = dbg_dev;
  }
  PFX_CUDA_TRY(cudaMemsetAsync(args.status, 0, sizeof(int), stream));

  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (launch_ms) {
    PFX_CUDA_TRY(cudaEventCreate(&e0));
    PFX_CUDA_TRY(cudaEventCreate(&e1));
    PFX_CUDA_TRY(cudaEventRecord(e0, stream));
  }
  auto kern = pivot == 1 ? (nb == 32 ? dense_batched_kernel<32, 1, true>
                                : (minb == 2 ? dense_batched_kernel<16, 2, true> : dense_batched_kernel<16, 1, true>))
                    : (nb == 32 ? dense_batched_kernel<32, 1, false>
                                : (minb == 2 ? dense_batched_kernel<16, 2, false> : dense_batched_kernel<16, 1, false>));
  if (int rc = raise_smem_limit(reinterpret_cast<const void*>(kern), smem)) return rc;
  {
    // the variant in the profile name: NB, resident CTAs per SM, interchanges
    ProfTag tag(pivot == 1 ? (nb == 32 ? "nb32piv" : (minb == 2 ? "nb16x2piv" : "nb16piv"))
                           : (nb == 32 ? "nb32" : (minb == 2 ? "nb16x2" : "nb16")));
    PFX_LAUNCH("dense_batched_kernel", stream, kern<<<slots, DB_THREADS, smem, stream>>>(args));
  }
  PFX_CUDA_TRY(cudaGetLastError());
  const size_t per_out = per_sys * (real_path ? 1 : 2);
  const double scale = shift_c == 0.0 ? 1.0 : exp(shift_c);
  int rb = (int)std::min<size_t>(ceil_div((size_t)batch * per_out, 256), (size_t)sms * 8);
  PFX_LAUNCH("reduce_pairs_kernel", stream, reduce_pairs_kernel<<<rb, 256, 0, stream>>>(stage, out, batch, npairs, per_out, scale));
  PFX_CUDA_TRY(cudaGetLastError());
  if (launch_ms) {
    PFX_CUDA_TRY(cudaEventRecord(e1, stream));
    PFX_CUDA_TRY(cudaEventSynchronize(e1));
    PFX_CUDA_TRY(cudaEventElapsedTime(launch_ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  int* hst = pinned_word();
  if (!hst) return fail(PFX_CUDA, "pinned status word allocation failed");
  PFX_CUDA_TRY(cudaMemcpyAsync(hst, args.status, sizeof(int), cudaMemcpyDeviceToHost, stream));
  if (int rc_ = sync_stream(stream)) return rc_;
  const int st = *hst;
  if (pivot == 2 && (st & ST_PIVOT)) {
    // checked mode: some column's diagonal pivot is not the one partial pivoting picks ->
    // redo the whole call with interchanges
    note_pivot_fallback();
    return dense_batched_run(A, a_complex, d, batch, V, v_complex, ncols, full, real_path, solve_only, shift_c,
                             theta_d, coef_d, npairs, out, stream, launch_ms, 1);
  }
  if (args.dbg) {
    unsigned long long h[8];
    PFX_CUDA_TRY(cudaMemcpy(h, args.dbg, sizeof(h), cudaMemcpyDeviceToHost));
    fprintf(stderr,
            "[pfx dense phases, Mcycles summed over CTAs] system=%.1f build=%.1f lu=%.1f solves=%.1f panel=%.1f "
            "swaps=%.1f trsm=%.1f gemm=%.1f\n",
            h[6] / 1e6, h[7] / 1e6, h[0] / 1e6, h[1] / 1e6, h[2] / 1e6, h[3] / 1e6, h[4] / 1e6, h[5] / 1e6);
  }
  if (st & ST_SINGULAR) return fail(PFX_SINGULAR, "exactly zero pivot in a shifted factorization");
  return PFX_OK;
}

}  // namespace pfx
