// Real symmetric banded shifted solves with fused residue combine (config C5).
//
// The reference is dense-only; this follows its per-pair task and combine
// (engine.py:194-201: M = A - cI + theta_k I, y = M^{-1} V, 2 Re(a_k y)) and the ascending
// reduction (engine.py:226-228) with a band LU.
//
// Storage: every pole pair gets its own row-band copy of M_k: row i holds columns
// i-kb-nb .. i+kb+nb (Wd = 2kb+2nb+1 complex entries, the nb extra diagonals on each side
// stay zero).  Element (i, j) lives at base + i*Wd + (j - i + kb + nb) = p + i*(Wd-1) + j
// with p = base + kb + nb, i.e. the band IS a dense row-major matrix with ld = Wd - 1 for
// every access inside |i - j| <= kb + nb.  The zero padding lets the L21/U12 panels of a
// block step (which reach nb diagonals past the band) be read as plain rectangles.
//
// Factorisation (no pivoting, safe by SURVEY finding 7; the band then never fills in),
// all pole pairs batched in every launch, nb = 64, for each block step j0:
//   L11 U11 = M11                         zgetrf_diag (diagonal 64x64 block in SMEM)
//   L11^{-1}, U11^{-1}                     ztrtri_diag (one warp per column; U11^{-1} is kept
//                                          per block row for the back substitution)
//   U12 = L11^{-1} M12, L21 = M21 U11^{-1}  ztrmm (in-place DMMA products, kb-wide panels)
//   M22 -= L21 U12                         zgemm on DMMA (kb x kb x 64)
//   y1 = L11^{-1} y1, y2 -= L21 y1          forward elimination of the RHS alongside
// then block back substitution y1 = U11^{-1}(y1 - U12 y2), and the combine kernel.  Applying
// the explicit inverses keeps every block-step kernel on DMMA with one barrier-free pass
// instead of a 64-step dependent triangular solve (the latency bound of the TRSM version).
#include "zblas.cuh"

namespace pfx {

constexpr int BD_NB = 64;

// grid (row groups, systems): each warp writes whole rows of the padded row band (no index
// division: the band is ~40 GB for C5, so this is a pure HBM write stream).
// Partitioned solve (nparts = 2, SPIKE): system s = part * npairs + k holds the rows of
// partition `part` (Np = N / 2 rows each), the second partition REVERSED (local row i <->
// global row N - 1 - i), so both factorisations run top-down in one batch and each
// partition's interface rows are its last ones.  Couplings across the partition boundary are
// left out here (bd_spike_*).  Global rows [g0, g1) of every system are built.
__device__ __forceinline__ double band_at(const double* band, int64_t N, int kb, int64_t gi, int64_t gj) {
  const int64_t d = gj - gi;
  const int64_t ad = d < 0 ? -d : d;
  if (ad > kb || gi < 0 || gj < 0 || gi >= N || gj >= N) return 0.0;
  return band[ad * N + (gi < gj ? gi : gj)];
}

__global__ void bd_build(const double* band, int64_t N, int kb, int Wd, const double* V, int nrhs, double shift_c,
                         const double2* theta, ZMat M, ZMat X, int64_t g0, int64_t g1, int npairs, int nparts,
                         int64_t Np) {
  const int s = blockIdx.y;
  const int part = s / npairs, k = s - part * npairs;
  const cplx th = ld(&theta[k]);
  double2* base = M.p - (kb + BD_NB) + s * M.stride;  // row-band base of system s
  // local rows of this system whose global row lies in [g0, g1)
  int64_t i0, i1;
  if (part == 0) {
    i0 = g0 < Np ? g0 : Np;
    i1 = g1 < Np ? g1 : Np;
  } else {
    const int64_t a = (N - g1) > 0 ? N - g1 : 0, b = N - g0;  // local = N - 1 - global
    i0 = a;
    i1 = b < Np ? b : Np;
  }
  if (i1 <= i0) return;
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = i0 + wid; i < i1; i += nw) {
    double2* rowp = base + i * Wd;
    const int64_t gi = part ? N - 1 - i : i;
    for (int e = lane; e < Wd; e += 32) {
      const int off = e - (kb + BD_NB);  // local j - i
      const int64_t j = i + off;
      double v = 0.0;
      if (j >= 0 && j < Np) v = band_at(band, N, kb, gi, part ? N - 1 - j : j);
      double2 z = make_double2(v, 0.0);
      if (off == 0) {
        z.x = (v - shift_c) + th.re;
        z.y = th.im;
      }
      rowp[e] = z;
    }
  }
  for (int64_t e = i0 * nrhs + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < i1 * nrhs;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / nrhs, c = e - i * nrhs;
    const int64_t gi = part ? N - 1 - i : i;
    X.p[s * X.stride + e] = make_double2(V[gi * nrhs + c], 0.0);
  }
}

// The factorisation + solves touch only the workspace, so the ~8 launches per 64-row
// block step are captured once into a CUDA graph per (shape, workspace) and replayed:
// the per-launch host overhead was the bound of this path (N/64 = 4096 block steps).
// Block back substitution y1 = U11^{-1} (y1 - U12 y2) for one 64-row block, all systems:
// bd_back_partial splits the kb-long inner dimension into 32-wide chunks (one CTA per chunk
// and system: P[q] = U12[:, chunk q] y2[chunk q]), bd_back_finish sums the chunks in
// ascending order (deterministic), subtracts, and applies the stored U11^{-1}.
constexpr int BK_C = 32;

// Fused residue combine (engine.py:201,226-228): out[rows of block j] = e^c sum_k 2 Re(a_k X_k)
// in ascending pair order.  It rides along in the back substitution: the partial-product
// launch of block j - 1 carries one extra CTA that combines block j, whose rows every pair
// finished in the previous launch (L2-hot), so the combine adds no step to the serial chain
// and no pass re-reads the n/2 solutions; block 0 is combined by one last small launch.
// The parameters live in device memory (the back substitution is replayed from a captured
// graph; `out` and the residues change per call).
struct BdCombine {
  const double2* coef;
  double scale;
  double* out;
  int npairs, nparts;  // systems = nparts x npairs (partition 1 reversed)
  int64_t Np, N;       // rows per system, global rows
};

__device__ void bd_combine_rows(const ZMat& X, int64_t j0, int jb, int nr, const BdCombine* cmb) {
  const double2* coef = cmb->coef;
  const double sc = cmb->scale;
  const int npairs = cmb->npairs;
  for (int part = 0; part < cmb->nparts; ++part)
    for (int e = threadIdx.x; e < jb * nr; e += blockDim.x) {
      const int64_t li = j0 + e / nr, c = e % nr;
      const int64_t i = li * nr + c;  // element of the system's Np x nr block
      double acc = 0.0;
      for (int k = 0; k < npairs; ++k) {
        const cplx a = ld(&coef[k]);
        const double2 x = X.p[(part * npairs + k) * X.stride + i];
        const double sk = 2.0 * fma(a.re, x.x, -a.im * x.y);
        acc = k == 0 ? sk : acc + sk;
      }
      const int64_t gi = part ? cmb->N - 1 - li : li;
      cmb->out[gi * nr + c] = sc == 1.0 ? acc : sc * acc;
    }
}

__global__ void bd_combine_block(ZMat X, int64_t j0, int jb, int nr, const BdCombine* cmb) {
  bd_combine_rows(X, j0, jb, nr, cmb);
}

// grid (nq + 1, npairs): CTA x = nq (pair 0 only) is the ride-along combine of the block
// below (rows [cj0, cj0 + cjb), final for every pair).
__global__ void __launch_bounds__(256) bd_back_partial(ZMat M, ZMat X, int64_t j0, int jb, int rest, int nr,
                                                       double2* P, int nq, const BdCombine* cmb, int64_t cj0,
                                                       int cjb) {
  __shared__ __align__(16) double2 us[64][BK_C + 1];
  __shared__ __align__(16) double2 xs[BK_C][9];
  const int q = blockIdx.x, b = blockIdx.y;
  if (q == nq) {
    if (b == 0) bd_combine_rows(X, cj0, cjb, nr, cmb);
    return;
  }
  const int tid = threadIdx.x;
  const int t0 = q * BK_C, tn = min(BK_C, rest - t0);
  const int64_t col0 = j0 + jb + t0;
  for (int e = tid; e < 64 * BK_C; e += 256) {
    const int r = e >> 5, t = e & 31;
    if (r < jb && t < tn) cp_async16(&us[r][t], M.at(b, j0 + r, col0 + t));
    else us[r][t] = make_double2(0, 0);
  }
  cp_async_commit();
  const int r = tid >> 2, cg = tid & 3;
  for (int c0 = 0; c0 < nr; c0 += 8) {
    const int nc = min(8, nr - c0);
    __syncthreads();
    for (int e = tid; e < BK_C * 8; e += 256) {
      const int t = e >> 3, c = e & 7;
      xs[t][c] = (t < tn && c < nc) ? *X.at(b, col0 + t, c0 + c) : make_double2(0, 0);
    }
    cp_async_wait<0>();
    __syncthreads();
    cplx a0 = mk(0, 0), a1 = mk(0, 0), b0 = mk(0, 0), b1 = mk(0, 0);
#pragma unroll 8
    for (int t = 0; t < BK_C; t += 2) {
      const cplx u = ld(&us[r][t]), v = ld(&us[r][t + 1]);
      a0 = cfma(u, ld(&xs[t][cg]), a0);
      a1 = cfma(u, ld(&xs[t][cg + 4]), a1);
      b0 = cfma(v, ld(&xs[t + 1][cg]), b0);
      b1 = cfma(v, ld(&xs[t + 1][cg + 4]), b1);
    }
    if (r < jb) {
      double2* pq = P + (((int64_t)b * nq + q) * 64 + r) * nr + c0;
      if (cg < nc) pq[cg] = make_double2(a0.re + b0.re, a0.im + b0.im);
      if (cg + 4 < nc) pq[cg + 4] = make_double2(a1.re + b1.re, a1.im + b1.im);
    }
  }
}

__global__ void __launch_bounds__(256) bd_back_finish(ZMat X, ZMat Ui, int64_t j0, int jb, int nr, int nq,
                                                      const double2* P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* us = reinterpret_cast<double2*>(smem_raw);  // 64 x 65 (upper triangle of U11^{-1})
  double2* ts = us + 64 * 65;                          // 64 x ncl (this CTA's column chunk)
  const int b = blockIdx.x;
  const int cc = blockIdx.y * 64, ncl = min(64, nr - cc);
  const int tid = threadIdx.x;
  for (int e = tid; e < 64 * 64; e += 256) {
    const int r = e >> 6, c = e & 63;
    if (r < jb && c < jb && c >= r) cp_async16(&us[r * 65 + c], Ui.at(b, r, c));
  }
  cp_async_commit();
  for (int e = tid; e < jb * ncl; e += 256) {
    const int r = e / ncl, c = e - r * ncl;
    cplx v = ld(X.at(b, j0 + r, cc + c));
    const double2* pe = P + ((int64_t)b * nq * 64 + r) * nr + cc + c;
    const int64_t qs = (int64_t)64 * nr;
    int q = 0;
    for (; q + 4 <= nq; q += 4) {  // four independent loads per round, subtracted in order
      const cplx p0 = ld(pe + q * qs), p1 = ld(pe + (q + 1) * qs), p2 = ld(pe + (q + 2) * qs), p3 = ld(pe + (q + 3) * qs);
      v = csub(csub(csub(csub(v, p0), p1), p2), p3);
    }
    for (; q < nq; ++q) v = csub(v, ld(pe + q * qs));
    ts[r * ncl + c] = make_double2(v.re, v.im);
  }
  cp_async_wait<0>();
  __syncthreads();
  for (int e = tid; e < jb * ncl; e += 256) {
    const int r = e / ncl, c = e - r * ncl;
    cplx a0 = mk(0, 0), a1 = mk(0, 0);
    int k = r;
    for (; k + 2 <= jb; k += 2) {
      a0 = cfma(ld(&us[r * 65 + k]), ld(&ts[k * ncl + c]), a0);
      a1 = cfma(ld(&us[r * 65 + k + 1]), ld(&ts[(k + 1) * ncl + c]), a1);
    }
    if (k < jb) a0 = cfma(ld(&us[r * 65 + k]), ld(&ts[k * ncl + c]), a0);
    *X.at(b, j0 + r, cc + c) = make_double2(a0.re + a1.re, a0.im + a1.im);
  }
}

// ---------------------------------------------------------------------------
// Two-partition SPIKE interface (nparts = 2).  With M0 (rows [0, Np)) and the reversed M1
// (rows [Np, N) read backwards) factored side by side, the bottom KB rows of each system are the
// interface (KB >= kb, rounded so the region starts on a 64-row block).  E0 (KB x KB) couples
// partition 0's interface rows to partition 1's interface unknowns (its local order), and
// E1 = E0^T the other way (A symmetric).  With y = L^{-1} f from the forward elimination:
//   V_p = U_bb^{-1} L_bb^{-1} E_p,  g_p = U_bb^{-1} y_bb        (bottom-block products only:
//        a right-hand side zero above the interface stays zero under L^{-1}, and the bottom
//        rows of U^{-1} z involve only z's bottom rows)
//   [I V0; V1 I] [a; b] = [g0; g1]  ->  (I - V0 V1) a = g0 - V0 g1,  b = g1 - V1 a
//   y0_bb -= L0_bb^{-1} (E0 b),  y1_bb -= L1_bb^{-1} (E1 a)           (the coupling moved to
//        the right-hand side; only the interface rows of y change)
// then the ordinary back substitution of both partitions gives the exact solution: the
// chain of dependent block steps is half as long (N / 2 / 64 instead of N / 64).
struct BdSpike {
  int KB = 0;               // interface rows per system
  int64_t R0 = 0;           // first interface row (local), a multiple of 64
  ZMat W{nullptr, 0, 0};    // nsys x KB x (KB + nr): [coupling | y_bb] -> [V | g]
  ZMat E{nullptr, 0, 0};    // KB x KB (E0), batch stride 0
  ZMat Et{nullptr, 0, 0};   // KB x KB (E0^T), batch stride 0
  ZMat S{nullptr, 0, 0};    // npairs x KB x KB
  ZMat AB{nullptr, 0, 0};   // nsys x KB x nr: interface unknowns a (part 0), b (part 1)
  ZMat T{nullptr, 0, 0};    // nsys x KB x nr: corrections
  ZMat LiS{nullptr, 0, 0}, UiS{nullptr, 0, 0};  // npairs x (KB / 64) x 64 x 64
  const double* band = nullptr;
  int64_t N = 0;
  int kb = 0;
};

__global__ void bd_spike_coupling(const double* band, int64_t N, int kb, int64_t Np, int KB, ZMat E, ZMat Et) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)KB * KB;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / KB), t = (int)(e - (e / KB) * KB);
    const int64_t g0 = Np - KB + r;           // partition 0 interface row r (global)
    const int64_t g1 = N - 1 - (Np - KB + t);  // partition 1 interface row t (global)
    const double v = band_at(band, N, kb, g0, g1);
    E.p[(int64_t)r * E.ld + t] = make_double2(v, 0.0);
    Et.p[(int64_t)t * Et.ld + r] = make_double2(v, 0.0);
  }
}

// W[s] = [E_s | y_s(interface rows)]
__global__ void bd_spike_setup(ZMat W, ZMat E, ZMat Et, ZMat X, int64_t R0, int KB, int nr, int npairs) {
  const int s = blockIdx.y;
  const ZMat& C = s < npairs ? E : Et;
  const int w = KB + nr;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)KB * w;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / w), c = (int)(e - (e / w) * w);
    W.p[s * W.stride + (int64_t)r * W.ld + c] = c < KB ? C.p[(int64_t)r * C.ld + c] : *X.at(s, R0 + r, c - KB);
  }
}

// S[k] = I;  AB[k] = g0 (R, the right-hand side of S a = g0 - V0 g1);  AB[npairs + k] = g1
__global__ void bd_spike_init(ZMat S, ZMat AB, ZMat W, int KB, int nr, int npairs) {
  const int k = blockIdx.y;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)KB * KB;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / KB), c = (int)(e - (e / KB) * KB);
    S.p[k * S.stride + e] = make_double2(r == c ? 1.0 : 0.0, 0.0);
  }
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)KB * nr;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / nr), c = (int)(e - (e / nr) * nr);
    AB.p[k * AB.stride + e] = W.p[k * W.stride + (int64_t)r * W.ld + KB + c];
    AB.p[(npairs + k) * AB.stride + e] = W.p[(npairs + k) * W.stride + (int64_t)r * W.ld + KB + c];
  }
}

// X[s](interface rows) -= T[s]
__global__ void bd_spike_correct(ZMat X, ZMat T, int64_t R0, int KB, int nr) {
  const int s = blockIdx.y;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)KB * nr;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / nr), c = (int)(e - (e / nr) * nr);
    double2* x = X.at(s, R0 + r, c);
    const double2 t = T.p[s * T.stride + e];
    *x = make_double2(x->x - t.x, x->y - t.y);
  }
}

int lu_solve_nopiv(cudaStream_t s, int nsys, int d, ZMat M, ZMat X, ZMat Li, ZMat Ui, int ncols, int* sing,
                   bool identity_rhs, bool sym_lower, bool check_pivots, const ZCombine* cmb);

// B = L_bb^{-1} B (lower = true) or U_bb^{-1} B, over the interface rows [R0, R0 + KB) of every
// system's band factors; B: KB x ncols dense per system.  Blocked by the band LU's own 64-row
// blocks and their stored diagonal inverses.
static int bd_region_solve(cudaStream_t st, int nsys, ZMat M, ZMat Li, ZMat Ui, int64_t R0, int KB, ZMat B, int ncols,
                           bool lower) {
  const int nb = BD_NB;
  const int nbk = (KB + nb - 1) / nb;  // the last block may be partial (Np not a multiple of 64)
  auto sub = [](ZMat A, int64_t i, int64_t j) {
    ZMat r = A;
    r.p = A.p + i * A.ld + j;
    return r;
  };
  auto blk = [&](ZMat T, int64_t j0) {
    ZMat r = T;
    r.p = T.p + (j0 / nb) * nb * nb;
    return r;
  };
  int rc;
  for (int q = 0; q < nbk; ++q) {
    const int p = lower ? q : nbk - 1 - q;
    const int64_t j0 = R0 + (int64_t)p * nb;
    const int jb = std::min(nb, KB - p * nb);
    if (lower) {
      if (p > 0 && (rc = zgemm(st, nsys, jb, ncols, p * nb, -1.0, sub(M, j0, R0), sub(B, 0, 0), sub(B, p * nb, 0))))
        return rc;
      if ((rc = ztrmm_inplace(st, nsys, jb, ncols, blk(Li, j0), sub(B, p * nb, 0), false, false))) return rc;
    } else {
      const int below = KB - p * nb - jb;
      if (below > 0 && (rc = zgemm(st, nsys, jb, ncols, below, -1.0, sub(M, j0, j0 + jb), sub(B, p * nb + jb, 0),
                                   sub(B, p * nb, 0))))
        return rc;
      if ((rc = ztrmm_inplace(st, nsys, jb, ncols, blk(Ui, j0), sub(B, p * nb, 0), false, true))) return rc;
    }
  }
  return PFX_OK;
}

static int bd_spike_interface(cudaStream_t st, const BdSpike& sp, ZMat M, ZMat X, ZMat Li, ZMat Ui, int64_t Np,
                              int nr, int npairs, int* sing) {
  const int KB = sp.KB, nsys = 2 * npairs;
  int rc;
  ZMat Wv = sp.W;  // V columns [0, KB) of W
  ZMat Wg = sp.W;  // g columns [KB, KB + nr)
  Wg.p = sp.W.p + KB;
  PFX_LAUNCH("bd_spike", st, bd_spike_coupling<<<296, 256, 0, st>>>(sp.band, sp.N, sp.kb, Np, KB, sp.E, sp.Et));
  PFX_CUDA_TRY(cudaGetLastError());
  PFX_LAUNCH("bd_spike", st, bd_spike_setup<<<dim3(64, nsys), 256, 0, st>>>(sp.W, sp.E, sp.Et, X, sp.R0, KB, nr, npairs));
  PFX_CUDA_TRY(cudaGetLastError());
  // V = U_bb^{-1} L_bb^{-1} E (coupling columns), g = U_bb^{-1} y_bb (right-hand-side columns)
  if ((rc = bd_region_solve(st, nsys, M, Li, Ui, sp.R0, KB, Wv, KB, true))) return rc;
  if ((rc = bd_region_solve(st, nsys, M, Li, Ui, sp.R0, KB, Wv, KB + nr, false))) return rc;
  PFX_LAUNCH("bd_spike", st, bd_spike_init<<<dim3(64, npairs), 256, 0, st>>>(sp.S, sp.AB, sp.W, KB, nr, npairs));
  PFX_CUDA_TRY(cudaGetLastError());
  ZMat V0 = Wv, V1 = Wv, g1 = Wg;
  V1.p = Wv.p + npairs * Wv.stride;
  g1.p = Wg.p + npairs * Wg.stride;
  ZMat A0 = sp.AB, A1 = sp.AB;  // a (part 0), b (part 1) slots
  A1.p = sp.AB.p + npairs * sp.AB.stride;
  // S = I - V0 V1,  a-slot = g0 - V0 g1,  a = S^{-1} (a-slot)
  if ((rc = zgemm(st, npairs, KB, KB, KB, -1.0, V0, V1, sp.S))) return rc;
  if ((rc = zgemm(st, npairs, KB, nr, KB, -1.0, V0, g1, A0))) return rc;
  if ((rc = lu_solve_nopiv(st, npairs, KB, sp.S, A0, sp.LiS, sp.UiS, nr, sing, false, false, false, nullptr))) return rc;
  // b = g1 - V1 a
  if ((rc = zgemm(st, npairs, KB, nr, KB, -1.0, V1, A0, A1))) return rc;
  // corrections T0 = L0_bb^{-1} (E0 b), T1 = L1_bb^{-1} (E1 a), applied to the interface rows of y
  ZMat T0 = sp.T, T1 = sp.T;
  T1.p = sp.T.p + npairs * sp.T.stride;
  if ((rc = zgemm(st, npairs, KB, nr, KB, 1.0, sp.E, A1, T0, false))) return rc;
  if ((rc = zgemm(st, npairs, KB, nr, KB, 1.0, sp.Et, A0, T1, false))) return rc;
  if ((rc = bd_region_solve(st, nsys, M, Li, Ui, sp.R0, KB, sp.T, nr, true))) return rc;
  PFX_LAUNCH("bd_spike", st, bd_spike_correct<<<dim3(8, nsys), 256, 0, st>>>(X, sp.T, sp.R0, KB, nr));
  PFX_CUDA_TRY(cudaGetLastError());
  return PFX_OK;
}

// Three streams inside one captured graph: the critical chain (diagonal LU -> inverses ->
// L21 -> A22 update -> next LU) stays on `main`; U12 = L11^{-1} M12 runs beside L21 on
// `s1`; the right-hand-side elimination (y1 = L11^{-1} y1, y2 -= L21 y1) trails on `s2`,
// where it overlaps the next block steps (its inputs, L11^{-1} per block and the L21
// columns, are never written again).
struct BdStreams {
  cudaStream_t s1 = nullptr, s2 = nullptr, s3 = nullptr, s4 = nullptr, s5 = nullptr;
  cudaEvent_t ev[10] = {};
};
static int bd_streams(BdStreams& S) {
  static BdStreams gs[kMaxDevices];
  const int dev = current_device();
  if (dev < 0 || dev >= kMaxDevices) return fail(PFX_CUDA, "device index out of range");
  BdStreams& g = gs[dev];
  if (!g.s1) {
    // the critical chain must win the SM slots whenever a trailing-update CTA retires:
    // s1 (panel beside the critical chain) high priority, s2 / s3 (trailing work) low
    int lo = 0, hi = 0;
    PFX_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    PFX_CUDA_TRY(cudaStreamCreateWithPriority(&g.s1, cudaStreamNonBlocking, hi));
    PFX_CUDA_TRY(cudaStreamCreateWithPriority(&g.s4, cudaStreamNonBlocking, hi));
    PFX_CUDA_TRY(cudaStreamCreateWithPriority(&g.s5, cudaStreamNonBlocking, hi));
    PFX_CUDA_TRY(cudaStreamCreateWithPriority(&g.s2, cudaStreamNonBlocking, lo));
    PFX_CUDA_TRY(cudaStreamCreateWithPriority(&g.s3, cudaStreamNonBlocking, lo));
    for (auto& e : g.ev) PFX_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  S = g;
  return PFX_OK;
}

// N, npairs: rows per system and systems in the batch (SPIKE: Np and 2 npairs; sp the interface)
static int bd_factor_solve(cudaStream_t stream, ZMat M, ZMat X, ZMat Li, ZMat Ui, double2* P, int64_t N, int kb,
                           int nr, int npairs, int* sing, const BdCombine* cmb, const BdSpike* sp) {
  const int nb = BD_NB;
  auto sub = [](ZMat A, int64_t i, int64_t j) {
    ZMat r = A;
    r.p = A.p + i * A.ld + j;
    return r;
  };
  auto blk = [&](ZMat T, int64_t j0) {
    ZMat r = T;
    r.p = T.p + (j0 / nb) * nb * nb;
    return r;
  };
  BdStreams S;
  int rc;
  if ((rc = bd_streams(S))) return rc;
  // a profiled pass (pfx_prof_enable; direct launches, no graph) keeps every launch on the one
  // stream: its per-launch event times are then the kernels' own durations, not shares of
  // overlapped time
  if (prof_on()) S.s1 = S.s2 = S.s3 = S.s4 = S.s5 = stream;
  // PFX_BD_SKIP (timing experiments only, results are wrong): bit 0 back substitution,
  // bit 1 rhs chain, bit 2 trailing update, bit 3 diagonal LU + inverses, bit 4 panel products
  static const int skip = [] {
    const char* e = getenv("PFX_BD_SKIP");
    return e ? atoi(e) : 0;
  }();
  cudaEvent_t evT = S.ev[0], evU = S.ev[1], evL = S.ev[2], evR = S.ev[3], evP = S.ev[4], evB = S.ev[5];
  cudaEvent_t evS = S.ev[6], evA = S.ev[7], evT2 = S.ev[8];
  // PFX_BD_LL=1 (opt-in): left-looking far update instead of t2 (see below).  Measured on C5:
  // 278.7 ms against 255.8 -- the two long-K launches per step have few, long CTAs (at most
  // 384 + 320 of 32 x 32, K up to 384) and the same one-step deadline as t2, so they hold the
  // chain back more than their smaller traffic gains; with 64 x 64 tiles 304 ms.
  static const bool ll_on = [] {
    const char* e = getenv("PFX_BD_LL");
    return e && atoi(e) != 0;
  }();
  const bool ll = ll_on && kb % nb == 0 && kb >= 4 * nb && N % nb == 0;
  bool pending_t2 = false;  // a t2 (far trailing update) is queued on s3
  bool pending_s = false;  // strips of the previous step queued on s4
  // s2 / s3 start after everything already queued on main (the build kernel)
  PFX_CUDA_TRY(cudaEventRecord(evT, stream));
  PFX_CUDA_TRY(cudaStreamWaitEvent(S.s2, evT, 0));
  PFX_CUDA_TRY(cudaStreamWaitEvent(S.s3, evT, 0));
  bool pending_b = false;  // a trailing update of the previous step is queued on s3
  for (int64_t j0 = 0; j0 < N; j0 += nb) {
    const int jb = (int)std::min<int64_t>(nb, N - j0);
    const int rest = (int)std::min<int64_t>(kb, N - j0 - jb);  // rows/cols coupled below/right
    if (!(skip & 8) && (rc = zgetrf_diag(stream, npairs, jb, sub(M, j0, j0), sing))) return rc;
    if (!(skip & 8) && (rc = ztrtri_diag(stream, npairs, jb, sub(M, j0, j0), blk(Li, j0), blk(Ui, j0)))) return rc;
    // this block's panels are the previous step's strips (s4)
    if (pending_s) PFX_CUDA_TRY(cudaStreamWaitEvent(stream, evS, 0));
    if (rest > 0 && !(skip & 16)) {
      PFX_CUDA_TRY(cudaEventRecord(evT, stream));
      PFX_CUDA_TRY(cudaStreamWaitEvent(S.s1, evT, 0));
      if ((rc = ztrmm_inplace(S.s1, npairs, jb, rest, blk(Li, j0), sub(M, j0, j0 + jb), false, false))) return rc;
      PFX_CUDA_TRY(cudaEventRecord(evU, S.s1));
      if ((rc = ztrmm_inplace(stream, npairs, jb, rest, blk(Ui, j0), sub(M, j0 + jb, j0), true, true))) return rc;
    }
    PFX_CUDA_TRY(cudaEventRecord(evL, stream));
    PFX_CUDA_TRY(cudaStreamWaitEvent(S.s2, evL, 0));
    if (!(skip & 2) && (rc = ztrmm_inplace(S.s2, npairs, jb, nr, blk(Li, j0), sub(X, j0, 0), false, false))) return rc;
    if (rest > 0 && !(skip & 2) && (rc = zgemm(S.s2, npairs, rest, nr, jb, -1.0, sub(M, j0 + jb, j0), sub(X, j0, 0),
                                sub(X, j0 + jb, 0))))
      return rc;
    if (rest > 0) {
      // Depth-two look-ahead.  Step j's update A -= L[:, j] U[j, :] of the coupled region
      // [j + 1, j + 1 + kb)^2 is split by how soon it is needed:
      //   main  the next diagonal block (ra x ra), before the next LU;
      //   s4    the rest of the next row / column strips (the next panel products read them);
      //   s5    t1: the row / column strips of block j + 2 (needed by the NEXT step's diagonal
      //         update and strips) -- waits for t2 of the previous step, which covered them;
      //   s3    t2: everything from block j + 3 on, needed only two steps later.
      // So the critical chain waits for a 64-wide L-shaped strip, not for the whole trailing
      // update (which, with 2 x npairs systems per launch under SPIKE, outlasted the chain).
      const int ra = std::min(nb, rest);
      PFX_CUDA_TRY(cudaStreamWaitEvent(stream, evU, 0));
      if (pending_b) PFX_CUDA_TRY(cudaStreamWaitEvent(stream, evB, 0));  // t1 of the previous step
      PFX_CUDA_TRY(cudaEventRecord(evP, stream));  // panels of this step are final
      if ((rc = zgemm(stream, npairs, ra, ra, jb, -1.0, sub(M, j0 + jb, j0), sub(M, j0, j0 + jb),
                      sub(M, j0 + jb, j0 + jb))))
        return rc;
      pending_s = false;
      pending_b = false;
      if (rest > ra) {
        PFX_CUDA_TRY(cudaStreamWaitEvent(S.s4, evP, 0));
        if ((rc = zgemm(S.s4, npairs, ra, rest - ra, jb, -1.0, sub(M, j0 + jb, j0), sub(M, j0, j0 + jb + ra),
                        sub(M, j0 + jb, j0 + jb + ra))))
          return rc;
        if ((rc = zgemm(S.s4, npairs, rest - ra, ra, jb, -1.0, sub(M, j0 + jb + ra, j0), sub(M, j0, j0 + jb),
                        sub(M, j0 + jb + ra, j0 + jb))))
          return rc;
        PFX_CUDA_TRY(cudaEventRecord(evS, S.s4));
        pending_s = true;
        if (!(skip & 4)) {
          const int64_t k0 = j0 + jb + ra;     // first row / column of block j + 2
          const int r2 = rest - ra;            // coupled rows / cols from block j + 2 on
          const int rb = std::min(nb, r2);     // block j + 2
          // t1: block j + 2's row strip (rb x r2) and column strip ((r2 - rb) x rb)
          PFX_CUDA_TRY(cudaEventRecord(evA, stream));
          PFX_CUDA_TRY(cudaStreamWaitEvent(S.s5, evA, 0));
          if (pending_t2) PFX_CUDA_TRY(cudaStreamWaitEvent(S.s5, evT2, 0));
          if ((rc = zgemm(S.s5, npairs, rb, r2, jb, -1.0, sub(M, k0, j0), sub(M, j0, k0), sub(M, k0, k0)))) return rc;
          if (r2 > rb && (rc = zgemm(S.s5, npairs, r2 - rb, rb, jb, -1.0, sub(M, k0 + rb, j0), sub(M, j0, k0),
                                     sub(M, k0 + rb, k0))))
            return rc;
          PFX_CUDA_TRY(cudaEventRecord(evB, S.s5));
          pending_b = true;
          // Left-looking far update (PFX_BD_LL=1; kb and N multiples of 64): instead of t2 -- every block of
          // the window taking panel j's K = 64 contribution now, eight read-modify-write passes
          // per block -- the L-shaped panel of block c = j + 3 takes, in ONE product per arm, all
          // the contributions still missing from it: those of the panels three or more steps
          // back, c - 8 .. c - 3 = j - 5 .. j (the two nearest panels stay right-looking: the
          // strips and t1).  K up to 384 instead of 64: a sixth of the traffic on the window
          // blocks.  The operands' band edge is a trapezoid (U[i][s] = 0 for s - i > kb,
          // L[r][i] = 0 for r - i > kb): zgemm skips the out-of-band K range per tile.
          if (ll) {
            const int64_t c0 = k0 + rb;  // first row / column of block j + 3
            if (c0 < N) {
              PFX_CUDA_TRY(cudaStreamWaitEvent(S.s3, evA, 0));
              const int64_t pend = j0 + jb;  // panels [p, pend) are final
              // row arm: blocks (c, c .. c + 5)
              const int64_t p0 = std::max<int64_t>(0, c0 - kb);
              const int mr = (int)std::min<int64_t>(nb, N - c0);
              const int ncr = (int)std::min<int64_t>(kb - 2 * nb, N - c0);
              if ((rc = zgemm(S.s3, npairs, mr, ncr, (int)(pend - p0), -1.0, sub(M, c0, p0), sub(M, p0, c0),
                              sub(M, c0, c0), true, (int)(kb - (c0 - p0)), nullptr, -2)))
                return rc;
              // column arm: blocks (c + 1 .. c + 5, c)
              const int64_t r1 = c0 + nb;
              if (r1 < N) {
                const int64_t p1 = std::max<int64_t>(0, r1 - kb);
                const int mc = (int)std::min<int64_t>(kb - 3 * nb, N - r1);
                if (pend > p1 && (rc = zgemm(S.s3, npairs, mc, mr, (int)(pend - p1), -1.0, sub(M, r1, p1),
                                             sub(M, p1, c0), sub(M, r1, c0), true, -1, nullptr,
                                             (int)(kb - (r1 - p1)))))
                  return rc;
              }
              PFX_CUDA_TRY(cudaEventRecord(evT2, S.s3));
              pending_t2 = true;
            }
          } else if (r2 > rb) {
            PFX_CUDA_TRY(cudaStreamWaitEvent(S.s3, evA, 0));
            if ((rc = zgemm(S.s3, npairs, r2 - rb, r2 - rb, jb, -1.0, sub(M, k0 + rb, j0), sub(M, j0, k0 + rb),
                            sub(M, k0 + rb, k0 + rb))))
              return rc;
            PFX_CUDA_TRY(cudaEventRecord(evT2, S.s3));
            pending_t2 = true;
          }
        }
      }
    }
  }
  if (pending_s) PFX_CUDA_TRY(cudaStreamWaitEvent(stream, evS, 0));
  if (pending_b) PFX_CUDA_TRY(cudaStreamWaitEvent(stream, evB, 0));
  if (pending_t2) PFX_CUDA_TRY(cudaStreamWaitEvent(stream, evT2, 0));
  PFX_CUDA_TRY(cudaEventRecord(evR, S.s2));
  PFX_CUDA_TRY(cudaStreamWaitEvent(stream, evR, 0));
  PFX_CUDA_TRY(cudaEventRecord(S.ev[9], S.s3));  // s3 joins even when nothing was queued on it
  PFX_CUDA_TRY(cudaStreamWaitEvent(stream, S.ev[9], 0));
  if (sp && (rc = bd_spike_interface(stream, *sp, M, X, Li, Ui, N, nr, npairs / 2, sing))) return rc;
  const int64_t nblk = (N + nb - 1) / nb;
  for (int64_t pb = nblk - 1; pb >= 0 && !(skip & 1); --pb) {
    const int64_t j0 = pb * nb;
    const int jb = (int)std::min<int64_t>(nb, N - j0);
    const int rest = (int)std::min<int64_t>(kb, N - j0 - jb);
    const int nq = (int)ceil_div(rest, BK_C);
    if (nq > 0) {
      // + one CTA combining block pb + 1 (finished by the previous launch)
      dim3 g((unsigned)nq + 1, (unsigned)npairs);
      const int64_t cj0 = j0 + nb;
      const int cjb = (int)std::min<int64_t>(nb, N - cj0);
      PFX_LAUNCH_F("bd_back_partial", stream, 8.0 * jb * rest * (double)nr * npairs,
                   bd_back_partial<<<g, 256, 0, stream>>>(M, X, j0, jb, rest, nr, P, nq, cmb, cj0, cjb));
      PFX_CUDA_TRY(cudaGetLastError());
    }
    const int fsm = (64 * 65 + 64 * std::min(nr, 64)) * (int)sizeof(double2);
    if (int rc = raise_smem_limit(reinterpret_cast<const void*>(bd_back_finish), fsm)) return rc;
    dim3 gf((unsigned)npairs, (unsigned)ceil_div(nr, 64));
    PFX_LAUNCH_F("bd_back_finish", stream, 4.0 * jb * jb * (double)nr * npairs,
                 bd_back_finish<<<gf, 256, fsm, stream>>>(X, blk(Ui, j0), j0, jb, nr, nq, P));
    PFX_CUDA_TRY(cudaGetLastError());
  }
  if (!(skip & 1)) {
    // block 0 (the last one the back substitution finishes)
    PFX_LAUNCH("bd_combine_block", stream,
               bd_combine_block<<<1, 256, 0, stream>>>(X, 0, (int)std::min<int64_t>(nb, N), nr, cmb));
    PFX_CUDA_TRY(cudaGetLastError());
  }
  return PFX_OK;
}

namespace {
struct BdGraph {
  cudaGraphExec_t exec = nullptr;
  void* ws = nullptr;
  int64_t N = 0;
  int kb = 0, nr = 0, np = 0;
  const double* band = nullptr;
};
BdGraph g_bd_graph[kMaxDevices];  // per device: a graph is bound to the device it was captured on
}  // namespace

// band_host / V_host (host mode): the band (diagonal-major, (kb+1) x N) and V are copied in by
// row chunks on a copy stream, and each chunk's rows are built as soon as the band columns they
// read (i0 - kb .. i1) have landed, so the 1 GB copy-in overlaps the build.
int banded_run(const double* band, int64_t N, int64_t kb64, const double* V, int64_t nrhs, double shift_c,
               const double2* theta_d, const double2* coef_d, int npairs, double* out, cudaStream_t stream,
               float* per_pair_ms, const double* band_host, const double* V_host) {
  const int kb = (int)kb64;
  const int nb = BD_NB;
  const int Wd = 2 * kb + 2 * nb + 1;
  ZgemmShortK short_k(true);  // the block steps' K = 64 updates run on the 32 x 32 tiles
  // Two-partition SPIKE (BdSpike) when the halves are long against the band: the serial chain of
  // block steps halves.  PFX_BD_SPIKE=0 keeps the single-partition factorisation.
  static const bool spike_on = [] {
    const char* e = getenv("PFX_BD_SPIKE");
    return !(e && atoi(e) == 0);
  }();
  const int64_t Nh = N / 2;
  const int KB = kb > 0 ? (int)(Nh - ((Nh - kb) / nb) * nb) : 0;  // interface rows, from a block start
  const bool spike = spike_on && kb > 0 && N % 2 == 0 && Nh >= 8 * (int64_t)kb && Nh >= 4 * nb && KB <= 1024 &&
                     (Nh - KB) % nb == 0;
  const int nparts = spike ? 2 : 1;
  const int64_t Np = spike ? Nh : N;  // rows per system
  const int nsys = nparts * npairs;
  const size_t mbytes = (size_t)nsys * Np * Wd * sizeof(double2);
  const size_t xbytes = (size_t)nsys * Np * nrhs * sizeof(double2);
  const int64_t nblk = (Np + nb - 1) / nb;
  const size_t libytes = (size_t)nsys * nblk * nb * nb * sizeof(double2);
  const size_t uibytes = (size_t)nsys * nblk * nb * nb * sizeof(double2);
  const size_t pbytes = (size_t)nsys * ceil_div(kb, BK_C) * nb * nrhs * sizeof(double2);
  // SPIKE interface buffers
  const size_t wbytes = spike ? (size_t)nsys * KB * (KB + nrhs) * sizeof(double2) : 0;
  const size_t ebytes = spike ? (size_t)2 * KB * KB * sizeof(double2) : 0;
  const size_t sbytes = spike ? (size_t)npairs * KB * KB * sizeof(double2) : 0;
  const size_t abbytes = spike ? (size_t)2 * nsys * KB * nrhs * sizeof(double2) : 0;
  const int kbb = (KB + nb - 1) / nb;  // 64-row blocks of the interface
  const size_t lsbytes = spike ? (size_t)2 * npairs * kbb * nb * nb * sizeof(double2) : 0;
  const size_t base_bytes = mbytes + xbytes + libytes + uibytes + pbytes + 256 + 64;
  char* ws = static_cast<char*>(scratch(1, base_bytes + wbytes + ebytes + sbytes + abbytes + lsbytes + 256));
  if (!ws) return fail(PFX_CUDA, "banded workspace allocation failed (needs " + std::to_string((mbytes + xbytes) >> 20) + " MiB)");
  ZMat M{reinterpret_cast<double2*>(ws) + kb + nb, Wd - 1, (int64_t)Np * Wd};
  ZMat X{reinterpret_cast<double2*>(ws + mbytes), nrhs, Np * nrhs};
  ZMat Li{reinterpret_cast<double2*>(ws + mbytes + xbytes), nb, nblk * nb * nb};
  ZMat Ui{reinterpret_cast<double2*>(ws + mbytes + xbytes + libytes), nb, nblk * nb * nb};
  double2* P = reinterpret_cast<double2*>(ws + mbytes + xbytes + libytes + uibytes);
  int* sing = reinterpret_cast<int*>(ws + mbytes + xbytes + libytes + uibytes + pbytes);
  PFX_CUDA_TRY(cudaMemsetAsync(sing, 0, sizeof(int), stream));
  BdSpike sp;
  if (spike) {
    double2* q = reinterpret_cast<double2*>(ws + base_bytes);
    sp.KB = KB;
    sp.R0 = Np - KB;
    sp.W = ZMat{q, KB + nrhs, (int64_t)KB * (KB + nrhs)};
    q += (size_t)nsys * KB * (KB + nrhs);
    sp.E = ZMat{q, KB, 0};
    q += (size_t)KB * KB;
    sp.Et = ZMat{q, KB, 0};
    q += (size_t)KB * KB;
    sp.S = ZMat{q, KB, (int64_t)KB * KB};
    q += (size_t)npairs * KB * KB;
    sp.AB = ZMat{q, nrhs, (int64_t)KB * nrhs};
    q += (size_t)nsys * KB * nrhs;
    sp.T = ZMat{q, nrhs, (int64_t)KB * nrhs};
    q += (size_t)nsys * KB * nrhs;
    sp.LiS = ZMat{q, nb, (int64_t)kbb * nb * nb};
    q += (size_t)npairs * kbb * nb * nb;
    sp.UiS = ZMat{q, nb, (int64_t)kbb * nb * nb};
    sp.band = band;
    sp.N = N;
    sp.kb = kb;
  }
  // combine parameters (device copy read by the graph-captured back substitution)
  BdCombine* cmb_d = reinterpret_cast<BdCombine*>(ws + mbytes + xbytes + libytes + uibytes + pbytes + 256);
  {
    static_assert(sizeof(BdCombine) <= 64, "combine parameters fit their slot");
    const BdCombine h{coef_d, shift_c == 0.0 ? 1.0 : exp(shift_c), out, npairs, nparts, Np, N};
    // pageable source: the runtime stages it before returning, so a stack value is safe
    PFX_CUDA_TRY(cudaMemcpyAsync(cmb_d, &h, sizeof(h), cudaMemcpyHostToDevice, stream));
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (per_pair_ms) {
    PFX_CUDA_TRY(cudaEventCreate(&e0));
    PFX_CUDA_TRY(cudaEventCreate(&e1));
    PFX_CUDA_TRY(cudaEventRecord(e0, stream));
  }
  dim3 bg((unsigned)(nsys > 8 ? 592 : 1184), nsys);
  if (!band_host) {
    PFX_LAUNCH("bd_build", stream,
               bd_build<<<bg, 256, 0, stream>>>(band, N, kb, Wd, V, (int)nrhs, shift_c, theta_d, M, X, 0, N, npairs,
                                                nparts, Np));
    PFX_CUDA_TRY(cudaGetLastError());
  } else {
    constexpr int NCH = 8;
    struct CopyIn {
      cudaStream_t cin = nullptr;
      cudaEvent_t evs[NCH + 1];
    };
    static CopyIn cis[kMaxDevices];
    const int dev = current_device();
    if (dev < 0 || dev >= kMaxDevices) return fail(PFX_CUDA, "device index out of range");
    cudaStream_t& cin = cis[dev].cin;
    cudaEvent_t* evs = cis[dev].evs;
    if (!cin) {
      PFX_CUDA_TRY(cudaStreamCreateWithFlags(&cin, cudaStreamNonBlocking));
      for (int i = 0; i <= NCH; ++i) PFX_CUDA_TRY(cudaEventCreateWithFlags(&evs[i], cudaEventDisableTiming));
    }
    // the staging buffers are idle on entry (host-mode calls end synchronised)
    PFX_CUDA_TRY(cudaEventRecord(evs[NCH], stream));
    PFX_CUDA_TRY(cudaStreamWaitEvent(cin, evs[NCH], 0));
    double* bandd = const_cast<double*>(band);
    double* Vd = const_cast<double*>(V);
    int64_t done = 0;  // band columns [0, done) copied
    for (int c = 0; c < NCH; ++c) {
      const int64_t i0 = N * c / NCH, i1 = N * (c + 1) / NCH;
      if (i1 > done) {
        PFX_CUDA_TRY(cudaMemcpy2DAsync(bandd + done, (size_t)N * sizeof(double), band_host + done,
                                       (size_t)N * sizeof(double), (size_t)(i1 - done) * sizeof(double),
                                       (size_t)kb + 1, cudaMemcpyHostToDevice, cin));
        done = i1;
      }
      PFX_CUDA_TRY(cudaMemcpyAsync(Vd + i0 * nrhs, V_host + i0 * nrhs, (size_t)(i1 - i0) * nrhs * sizeof(double),
                                   cudaMemcpyHostToDevice, cin));
      PFX_CUDA_TRY(cudaEventRecord(evs[c], cin));
      PFX_CUDA_TRY(cudaStreamWaitEvent(stream, evs[c], 0));
      PFX_LAUNCH("bd_build", stream,
                 bd_build<<<bg, 256, 0, stream>>>(band, N, kb, Wd, V, (int)nrhs, shift_c, theta_d, M, X, i0, i1, npairs,
                                                  nparts, Np));
      PFX_CUDA_TRY(cudaGetLastError());
    }
  }
  if (prof_on()) {
    // profiling wants per-kernel events: run the launches directly
    if (int rc = bd_factor_solve(stream, M, X, Li, Ui, P, Np, kb, (int)nrhs, nsys, sing, cmb_d, spike ? &sp : nullptr))
      return rc;
  } else {
    const int gdev = current_device();
    if (gdev < 0 || gdev >= kMaxDevices) return fail(PFX_CUDA, "device index out of range");
    BdGraph& G = g_bd_graph[gdev];
    if (!G.exec || G.ws != ws || G.N != N || G.kb != kb || G.nr != (int)nrhs || G.np != npairs || G.band != band) {
      if (G.exec) {
        cudaGraphExecDestroy(G.exec);
        G.exec = nullptr;
      }
      BdStreams S;  // create the side streams before capturing
      if (int rc = bd_streams(S)) return rc;
      cudaStream_t cs;  // capture origin = the critical chain: highest priority
      int lo = 0, hi = 0;
      PFX_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      PFX_CUDA_TRY(cudaStreamCreateWithPriority(&cs, cudaStreamNonBlocking, hi));
      cudaGraph_t graph;
      PFX_CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      int rc = bd_factor_solve(cs, M, X, Li, Ui, P, Np, kb, (int)nrhs, nsys, sing, cmb_d, spike ? &sp : nullptr);
      cudaError_t ce = cudaStreamEndCapture(cs, &graph);
      if (rc) return rc;
      if (ce != cudaSuccess) return fail(PFX_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
      // kernel nodes keep the priority of the stream they were captured from
      PFX_CUDA_TRY(cudaGraphInstantiateWithFlags(&G.exec, graph, cudaGraphInstantiateFlagUseNodePriority));
      cudaGraphDestroy(graph);
      cudaStreamDestroy(cs);
      G.ws = ws;
      G.N = N;
      G.kb = kb;
      G.nr = (int)nrhs;
      G.np = npairs;
      G.band = band;  // the SPIKE coupling kernel reads the band
    }
    PFX_CUDA_TRY(cudaGraphLaunch(G.exec, stream));
  }
  // (the residue combine ran fused into the back substitution: bd_back_finish)
  int* hsg = pinned_word();
  if (!hsg) return fail(PFX_CUDA, "pinned status word allocation failed");
  PFX_CUDA_TRY(cudaMemcpyAsync(hsg, sing, sizeof(int), cudaMemcpyDeviceToHost, stream));
  if (per_pair_ms) PFX_CUDA_TRY(cudaEventRecord(e1, stream));
  if (int rc_ = sync_stream(stream)) return rc_;
  if (per_pair_ms) {
    float ms = 0.0f;
    PFX_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    for (int k = 0; k < npairs; ++k) per_pair_ms[k] = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  if (*hsg & ST_SINGULAR) return fail(PFX_SINGULAR, "exactly zero pivot in a shifted band factorization");
  return PFX_OK;
}

}  // namespace pfx
