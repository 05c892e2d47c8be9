// On-chip ("lane = pole pair") variant of the tridiagonal sweeps, used when npairs <= 16.
// Included by tridiag.cu after TriArgs / the Moebius kernels.
//
// One half-warp = one (chunk of a.L <= TR_L rows, 16-RHS tile).  Lane k owns pole pair k: it
// runs pair k's pivot chains itself and the recurrences of all 16 right-hand sides
// (ILP 16).  The per-row sum over pairs goes through a shared-memory transpose and is
// added in ascending k (deterministic, the reference's order).  No factor data leaves
// the chip: the backward pivots the forward pass needs (and the forward pivots the
// backward pass needs) are recomputed per LS_B-row block from continuant checkpoints
// (two complex numbers per block and pair, L2-resident).
//   P1  backward continuant over the chunk, checkpoints at block boundaries
//   P2  per block, top-down: recompute l' (from P1 checkpoints) -> forward chain, gamma,
//       w = 2a/gamma -> forward RHS sweep, F_i = sum_k Re(w (g - f)) -> out
//   P3  per block, bottom-up: recompute l (from P2 checkpoints) -> backward chain, gamma,
//       w -> backward RHS sweep, out_i += sum_k Re(w g')
//   summaries gF/gB, LF/LB, contractivity flag, max|V| -> the same carry scan.  P2/P3 also
//   store z = w Lambda per (row, pair) (Lambda = running product of -l, resp. -l', from the
//   chunk edge) and the per-block bounds beta |Lambda|, so the edge fix (tri_fixz) is a
//   streaming pass out_i += sum_k Re(z_f G + z_b G') with no chain recomputation.
#pragma once
// (included inside namespace pfx)

constexpr int LS_B = 8;       // rows per recompute block
constexpr int LS_WARPS = 4;   // warps per block (8 units)
constexpr int LS_NBLK = TR_L / LS_B;

struct LsBuf {
  double f[LS_B][16];   // RHS rows of the block
  double dg[LS_B];      // diag
  double of[LS_B + 2];  // of[j] = e_{row0 - 1 + j} (j <= LS_B), 0 outside the matrix
};

struct LsSmem {
  double2 fw[LS_B][2][16];  // per row: [0][pair] l or l', [1][pair] w (pair-fastest: a
                            // phase-A store of 16 lanes is one conflict-free 256-byte row);
                            // [0] holds the recomputed opposite-direction multiplier until
                            // the lane overwrites it
  LsBuf buf[2];             // cp.async double buffer of the staged rows
  double lamabs[16];        // |Lambda_k| after the block (fix pass stop test)
};

struct LsCk {
  double2 a, b;  // continuant state (x_{i}, x_{i +- 1}) entering a block
};

__device__ __forceinline__ double ls_off(const TriArgs& a, int64_t gi) {
  return (gi >= 0 && gi < a.N - 1) ? a.off[gi] : 0.0;
}

// Issue cp.async copies of diag/off/RHS rows [r0, r0+cnt) of this unit's tile into B.
// Couplings outside the matrix and missing RHS columns are written as zeros directly.
__device__ __forceinline__ void ls_stage_async(LsBuf& B, const TriArgs& a, int64_t r0, int cnt, int rt0, int lane16,
                                               bool want_f) {
  if (lane16 < cnt) cp_async8(&B.dg[lane16], &a.diag[r0 + lane16]);
  if (lane16 <= cnt) {
    const int64_t gi = r0 - 1 + lane16;
    if (gi >= 0 && gi < a.N - 1)
      cp_async8(&B.of[lane16], &a.off[gi]);
    else
      B.of[lane16] = 0.0;
  }
  if (want_f) {
    const int rg = rt0 + lane16;
#pragma unroll
    for (int j = 0; j < LS_B; ++j) {
      if (j < cnt) {
        if (rg < a.nrhs)
          cp_async8(&B.f[j][lane16], &a.V[(r0 + j) * a.nrhs + rg]);
        else
          B.f[j][lane16] = 0.0;
      }
    }
  }
}

// one backward continuant step at local row j of the staged block: returns l'_i and
// advances (q1, q2) <- (q0, q1).  Rescale schedule is tied to the global row index.
__device__ __forceinline__ cplx ls_bstep(const LsBuf& S, double cshift, int j, int64_t row, cplx th, cplx& q1,
                                         cplx& q2) {
  const double e = S.of[j + 1];
  const cplx rho = cmul(q2, crcp_nc(q1));  // q1: rescaled continuant, |q1| >= Im(theta) |q2|
  const cplx lv = cscale(rho, e);
  const cplx b = mk(S.dg[j] - cshift + th.re, th.im);
  const double e2 = e * e;
  const cplx q0 = cplx{fma(b.re, q1.re, fma(-b.im, q1.im, -e2 * q2.re)), fma(b.re, q1.im, fma(b.im, q1.re, -e2 * q2.im))};
  q2 = q1;
  q1 = q0;
  if ((row & 7) == 0) rescale2(q1, q2);  // growth over 8 rows stays far inside binary64
  return lv;
}

__device__ __forceinline__ cplx ls_fstep(const LsBuf& S, double cshift, int j, int64_t row, cplx th, cplx& p1,
                                         cplx& p2) {
  const double e0 = S.of[j];
  const cplx rho = cmul(p2, crcp_nc(p1));
  const cplx lv = cscale(rho, e0);
  const cplx b = mk(S.dg[j] - cshift + th.re, th.im);
  const double e2 = e0 * e0;
  const cplx p0 = cplx{fma(b.re, p1.re, fma(-b.im, p1.im, -e2 * p2.re)), fma(b.re, p1.im, fma(b.im, p1.re, -e2 * p2.im))};
  p2 = p1;
  p1 = p0;
  if ((row & 7) == 7) rescale2(p1, p2);
  return lv;
}

struct LsArgs {
  LsCk* ckb;  // P x LS_NBLK x 16
  LsCk* ckf;  // P x LS_NBLK x 16
  double2* zf;    // N x npairs  w_i Lambda_i, Lambda_i = prod_{s <= j <= i} (-l_j)   (chunk top s)
  double2* zb;    // N x npairs  w_i Lambda'_i, Lambda'_i = prod_{i <= j <= e} (-l'_j) (chunk bottom e)
  double* lamf;   // P x LS_NBLK x 16  beta_k |Lambda_k| after each block (forward)
  double* lamb;   // P x LS_NBLK x 16  beta_k |Lambda'_k| after each block (backward)
  int64_t unit0, unit1;  // units [unit0, unit1) of this launch (row-group pipelining)
};

// The sweep (zero RHS carry-in).
// Phase A of a block: lane k = pole pair k computes its chain -> (l, w) in shared memory,
// and z = w Lambda plus the block-end bound beta |Lambda| to global memory for the fix.
// Phase B of a block: lane r = right-hand side r sweeps all pairs from broadcast loads and
// sums over pairs in registers (ascending k).
template <int KM>
__global__ void __launch_bounds__(LS_WARPS * 32, 4) tri_ls(TriArgs a, LsArgs ck) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = lane >> 4, k = lane & 15;  // k: pair in phase A, rhs in phase B
  const unsigned hmask = half ? 0xffff0000u : 0x0000ffffu;
  LsSmem& S = reinterpret_cast<LsSmem*>(smem_raw)[warp * 2 + half];
  const int ntile = (a.nrhs + 15) / 16;
  const int64_t unit = ck.unit0 + (blockIdx.x * (int64_t)LS_WARPS + warp) * 2 + half;
  if (unit >= ck.unit1) return;
  const int64_t c = unit / ntile;
  const int rt0 = (int)(unit - c * ntile) * 16;
  const int np = a.npairs;
  const bool act = k < np;                 // lane is a live pair in phase A
  const bool wz = act && rt0 == 0;         // z and the bounds are per (row, pair): one tile stores them
  const int rg = rt0 + k;                  // rhs of this lane in phase B
  const bool rv = rg < a.nrhs;
  const int64_t s = c * a.L;
  const int rows = (int)(a.L < a.N - s ? a.L : a.N - s);
  const int nblk = (rows + LS_B - 1) / LS_B;
  const double csh = a.c;
  const cplx th = act ? ld(&a.theta[k]) : mk(0, 1);
  const cplx co2 = act ? cscale(ld(&a.coef[k]), 2.0) : mk(0, 0);
  const double beta = act ? (fabs(co2.re) + fabs(co2.im)) / th.im : 0.0;
  LsCk* ckb = ck.ckb + (c * LS_NBLK) * 16;
  LsCk* ckf = ck.ckf + (c * LS_NBLK) * 16;
  bool noncontr = false;
  double vmx = 0.0;
  if (!act) {  // padded pair slots (k >= np) stay zero: phase B adds exact zeros for them
#pragma unroll
    for (int j = 0; j < LS_B; ++j) S.fw[j][0][k] = S.fw[j][1][k] = make_double2(0, 0);
  }
  auto blk_r0 = [&](int b) { return s + (int64_t)b * LS_B; };
  auto blk_cnt = [&](int b) { return min(LS_B, rows - b * LS_B); };

  // ---- P1: backward continuant, checkpoints entering each block from below
  {
    cplx q1 = mk(1, 0), q2 = act ? ld(&a.rhob_in[c * np + k]) : mk(0, 0);
    ls_stage_async(S.buf[0], a, blk_r0(nblk - 1), blk_cnt(nblk - 1), rt0, k, false);
    cp_async_commit();
    for (int bb = 0; bb < nblk; ++bb) {
      const int b = nblk - 1 - bb;
      const int cur = bb & 1;
      if (bb + 1 < nblk) ls_stage_async(S.buf[cur ^ 1], a, blk_r0(b - 1), blk_cnt(b - 1), rt0, k, false);
      cp_async_commit();
      cp_async_wait<1>();
      __syncwarp(hmask);
      const int64_t r0 = blk_r0(b);
      const int cnt = blk_cnt(b);
      if (act) {
        ckb[b * 16 + k] = LsCk{make_double2(q1.re, q1.im), make_double2(q2.re, q2.im)};
#pragma unroll
        for (int jj = 0; jj < LS_B; ++jj) {
          const int j = LS_B - 1 - jj;
          if (j < cnt) (void)ls_bstep(S.buf[cur], csh, j, r0 + j, th, q1, q2);
        }
      }
      __syncwarp(hmask);
    }
    cp_async_wait<0>();
  }

  for (int dir = 0; dir < 2; ++dir) {
    cplx g[KM];
#pragma unroll
    for (int q = 0; q < KM; ++q) g[q] = mk(0, 0);
    cplx x1 = mk(1, 0);
    cplx x2 = act ? ld(dir == 0 ? &a.rho_in[c * np + k] : &a.rhob_in[c * np + k]) : mk(0, 0);
    cplx lam = mk(1, 0);
    double2* const zo = (dir == 0 ? ck.zf : ck.zb) + k;
    double* const lo = (dir == 0 ? ck.lamf : ck.lamb) + (c * LS_NBLK) * 16 + k;
    auto blk_of = [&](int bb) { return dir == 0 ? bb : nblk - 1 - bb; };
    __syncwarp(hmask);
    ls_stage_async(S.buf[0], a, blk_r0(blk_of(0)), blk_cnt(blk_of(0)), rt0, k, true);
    cp_async_commit();
    LsCk ck_next = act ? (dir == 0 ? ckb[blk_of(0) * 16 + k] : ckf[blk_of(0) * 16 + k]) : LsCk{};
    for (int bb = 0; bb < nblk; ++bb) {
      const int b = blk_of(bb);
      const int cur = bb & 1;
      const LsCk ckv = ck_next;
      if (bb + 1 < nblk) {
        ls_stage_async(S.buf[cur ^ 1], a, blk_r0(blk_of(bb + 1)), blk_cnt(blk_of(bb + 1)), rt0, k, true);
        if (act) ck_next = dir == 0 ? ckb[blk_of(bb + 1) * 16 + k] : ckf[blk_of(bb + 1) * 16 + k];
      }
      cp_async_commit();
      cp_async_wait<1>();
      __syncwarp(hmask);
      const LsBuf& B = S.buf[cur];
      const int64_t r0 = blk_r0(b);
      const int cnt = blk_cnt(b);
      // ---- phase A (lane = pair)
#if defined(PFX_TRI_EXP) && PFX_TRI_EXP == 2
      if (act && bb == 0) {  // timing ablation: chains of the first block only
#else
      if (act) {
#endif
        if (dir == 0) {
          cplx q1 = mk(ckv.a.x, ckv.a.y), q2 = mk(ckv.b.x, ckv.b.y);
#pragma unroll
          for (int jj = 0; jj < LS_B; ++jj) {
            const int j = LS_B - 1 - jj;
            if (j < cnt) {
              cplx lv = ls_bstep(B, csh, j, r0 + j, th, q1, q2);
              S.fw[j][0][k] = make_double2(lv.re, lv.im);
              if (fma(lv.re, lv.re, lv.im * lv.im) > 1.0) noncontr = true;
            }
          }
          ckf[b * 16 + k] = LsCk{make_double2(x1.re, x1.im), make_double2(x2.re, x2.im)};
#pragma unroll
          for (int j = 0; j < LS_B; ++j) {
            if (j < cnt) {
              const cplx lv = ls_fstep(B, csh, j, r0 + j, th, x1, x2);
              const cplx lbv = ld(&S.fw[j][0][k]);
              const cplx bd = mk(B.dg[j] - csh + th.re, th.im);
              const cplx gam = csub(csub(bd, cscale(lv, B.of[j])), cscale(lbv, B.of[j + 1]));
              const cplx w = cmul(co2, crcp_nc(gam));  // |gamma| >= Im(theta)
              lam = cmul(lam, mk(-lv.re, -lv.im));
              if (fma(lv.re, lv.re, lv.im * lv.im) > 1.0) noncontr = true;
              S.fw[j][0][k] = make_double2(lv.re, lv.im);
              S.fw[j][1][k] = make_double2(w.re, w.im);
              if (wz) st(&zo[(r0 + j) * np], cmul(w, lam));
            }
          }
        } else {
          cplx p1 = mk(ckv.a.x, ckv.a.y), p2 = mk(ckv.b.x, ckv.b.y);
#pragma unroll
          for (int j = 0; j < LS_B; ++j) {
            if (j < cnt) {
              cplx lv = ls_fstep(B, csh, j, r0 + j, th, p1, p2);
              S.fw[j][0][k] = make_double2(lv.re, lv.im);
            }
          }
#pragma unroll
          for (int jj = 0; jj < LS_B; ++jj) {
            const int j = LS_B - 1 - jj;
            if (j < cnt) {
              const cplx lbv = ls_bstep(B, csh, j, r0 + j, th, x1, x2);
              const cplx lv = ld(&S.fw[j][0][k]);
              const cplx bd = mk(B.dg[j] - csh + th.re, th.im);
              const cplx gam = csub(csub(bd, cscale(lv, B.of[j])), cscale(lbv, B.of[j + 1]));
              const cplx w = cmul(co2, crcp_nc(gam));  // |gamma| >= Im(theta)
              lam = cmul(lam, mk(-lbv.re, -lbv.im));
              S.fw[j][0][k] = make_double2(lbv.re, lbv.im);
              S.fw[j][1][k] = make_double2(w.re, w.im);
              if (wz) st(&zo[(r0 + j) * np], cmul(w, lam));
            }
          }
        }
        if (wz) lo[b * 16] = beta * cabs1(lam);
      }
      __syncwarp(hmask);
      // ---- phase B (lane = rhs).  Per row: independent per-pair terms, then a fixed
      // pairwise tree over pairs (deterministic); rows unrolled for ILP.
      double* const obase = a.out + r0 * a.nrhs + rg;
#if defined(PFX_TRI_EXP) && PFX_TRI_EXP == 1
      const int cnt_b = bb < 0 ? cnt : 0;  // timing ablation: no RHS sweep
#else
      const int cnt_b = cnt;
#endif
#pragma unroll
      for (int jj = 0; jj < LS_B; ++jj) {
        if (jj < cnt_b) {
          const int j = dir == 0 ? jj : cnt - 1 - jj;
          // sum over pairs: two interleaved FMA chains (even / odd pairs), fixed order
          double acc0 = 0.0, acc1 = 0.0;
          const double f = B.f[j][k];
          if (dir == 0) vmx = fmax(vmx, fabs(f));
#pragma unroll
          for (int q = 0; q < KM; ++q) {
            const double2 l2 = S.fw[j][0][q], w2 = S.fw[j][1][q];
            g[q] = cplx{fma(-l2.x, g[q].re, fma(l2.y, g[q].im, f)), fma(-l2.x, g[q].im, -l2.y * g[q].re)};
            const double gre = dir == 0 ? g[q].re - f : g[q].re;
            double& acc = (q & 1) ? acc1 : acc0;
            acc = fma(w2.x, gre, acc);
            acc = fma(-w2.y, g[q].im, acc);
          }
          const double acc = acc0 + acc1;
          if (rv) {
            double* o = obase + j * a.nrhs;
            if (dir == 0)
              *o = acc;
            else
              *o = *o + acc;
          }
        }
      }
      __syncwarp(hmask);
    }
    cp_async_wait<0>();
    __syncwarp(hmask);
    if (rv) {
#pragma unroll
      for (int q = 0; q < KM; ++q)
        if (q < np) st(&(dir == 0 ? a.gF : a.gB)[g_at(a, c, q, rg)], g[q]);
    }
    if (act && rt0 == 0) st(&(dir == 0 ? a.LF : a.LB)[l_at(a, c, k)], lam);
  }
  if (noncontr) atomicAnd(&a.contr[c], 0);
  if (rv) atomicMax(&a.vmax[rg], (unsigned long long)__double_as_longlong(vmx));
}

// Edge fix with the true carries G (from above) and G' (from below), from the sweep's
// stored z:   out_i += sum_k Re(zf_{k,i} G_k) + Re(zb_{k,i} G'_k).
// In a contractive chunk (every |l|, |l'| <= 1) |Lambda| never grows and |w| <= 2|a|/Im(theta)
// (|gamma| >= Im(theta)), so after the first block whose end bound
// sum_k beta_k |Lambda_k| |G_k| is <= 2^-53 max|V[:, r]| every later row's correction is below
// one unit roundoff of max|V[:, r]| (below the binary64 rounding of the pole sum itself):
// the forward terms cover blocks [0, endF), the backward terms [begB, nblk), and only their
// union is visited (all blocks in a non-contractive chunk).
// Layout: a half-warp = one (chunk, 16-RHS tile), lane = right-hand side; the z rows of a
// block are staged by cp.async (double buffered) and read back as broadcasts.
#ifndef PFX_FIXZ_MINB
#define PFX_FIXZ_MINB 4  // resident CTAs per SM the fix kernel's registers are sized for
#endif
struct FzBuf {
  double2 z[LS_B][16];  // [row][pair] of one direction
};

template <int KM>
__global__ void __launch_bounds__(LS_WARPS * 32, PFX_FIXZ_MINB) tri_fixz(TriArgs a, LsArgs ck) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = lane >> 4, k = lane & 15;
  const unsigned hmask = half ? 0xffff0000u : 0x0000ffffu;
  FzBuf* const Z = reinterpret_cast<FzBuf*>(smem_raw) + (warp * 2 + half) * 2;
  const int ntile = (a.nrhs + 15) / 16;
  const int64_t unit = ck.unit0 + (blockIdx.x * (int64_t)LS_WARPS + warp) * 2 + half;
  if (unit >= ck.unit1) return;
  const int64_t c = unit / ntile;
  const int rt0 = (int)(unit - c * ntile) * 16;
  const int np = a.npairs;
  const int rg = rt0 + k;
  const bool rv = rg < a.nrhs;
  const int64_t s = c * a.L;
  const int rows = (int)(a.L < a.N - s ? a.L : a.N - s);
  const int nblk = (rows + LS_B - 1) / LS_B;
  // padded pair slots read as zeros
#pragma unroll
  for (int t = 0; t < 2; ++t)
    for (int e = k; e < LS_B * 16; e += 16)
      if ((e & 15) >= np) (&Z[t].z[0][0])[e] = make_double2(0, 0);
  const bool contr = a.contr[c] != 0;
  const double tau = rv ? ldexp(__longlong_as_double((long long)a.vmax[rg]), -TR_FIX_EXP) : 0.0;
  // the two directions one after the other (only one set of carries live at a time): the
  // forward terms over blocks [0, endF), then the backward terms over [begB, nblk)
  for (int dir = 0; dir < 2; ++dir) {
    cplx g[KM];
    const double2* Gs = dir == 0 ? a.G : a.Gb;
#pragma unroll
    for (int q = 0; q < KM; ++q) g[q] = (q < np && rv) ? ld(&Gs[(c * np + q) * a.nrhs + rg]) : mk(0, 0);
    int need = nblk;  // blocks from this direction's edge that can carry a correction
    if (contr) {
      const double* lb = (dir == 0 ? ck.lamf : ck.lamb) + (c * LS_NBLK) * 16;
      int e = nblk;
      for (int bb = 0; bb < nblk; ++bb) {
        double y = 0.0;
#pragma unroll
        for (int q = 0; q < KM; ++q) y = fma(lb[(dir == 0 ? bb : nblk - 1 - bb) * 16 + q], cabs1(g[q]), y);
        if (y <= tau) {
          e = bb + 1;
          break;
        }
      }
      for (int off = 8; off > 0; off >>= 1) e = max(e, __shfl_xor_sync(hmask, e, off));
      need = e;
    }
    const int b0 = dir == 0 ? 0 : nblk - need, b1 = dir == 0 ? need : nblk;
    const double2* zs = dir == 0 ? ck.zf : ck.zb;
    auto stage = [&](FzBuf& D, int b) {
      const int64_t r0 = s + (int64_t)b * LS_B;
      const int n = min(LS_B, rows - b * LS_B) * np;
      for (int e = k; e < n; e += 16) {
        const int j = e / np;
        cp_async16(&D.z[j][e - j * np], &zs[r0 * np + e]);
      }
    };
    __syncwarp(hmask);
    int cur = 0;
    if (b0 < b1) stage(Z[0], b0);
    cp_async_commit();
    for (int b = b0; b < b1; ++b) {
      if (b + 1 < b1) stage(Z[cur ^ 1], b + 1);
      cp_async_commit();
      const int64_t r0 = s + (int64_t)b * LS_B;
      const int cnt = min(LS_B, rows - b * LS_B);
      double ov[LS_B];
      double* const obase = a.out + r0 * a.nrhs + rg;
#pragma unroll
      for (int j = 0; j < LS_B; ++j) ov[j] = (rv && j < cnt) ? obase[j * a.nrhs] : 0.0;
      cp_async_wait<1>();
      __syncwarp(hmask);
      const FzBuf& D = Z[cur];
#pragma unroll
      for (int j = 0; j < LS_B; ++j) {
        double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
        for (int q = 0; q < KM; ++q) {
          const double2 z = D.z[j][q];
          acc0 = fma(z.x, g[q].re, acc0);
          acc1 = fma(-z.y, g[q].im, acc1);
        }
        ov[j] += acc0 + acc1;
      }
#pragma unroll
      for (int j = 0; j < LS_B; ++j)
        if (rv && j < cnt) obase[j * a.nrhs] = ov[j];
      __syncwarp(hmask);
      cur ^= 1;
    }
    cp_async_wait<0>();
    __syncwarp(hmask);
  }
}
