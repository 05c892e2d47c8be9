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

// grid (row groups, pairs): each warp writes whole rows of the padded row band (no index
// division: the band is ~40 GB for C5, so this is a pure HBM write stream)
__global__ void bd_build(const double* band, int64_t N, int kb, int Wd, const double* V, int nrhs, double shift_c,
                         const double2* theta, ZMat M, ZMat X, int64_t i0, int64_t i1) {  // rows [i0, i1)
  const int k = blockIdx.y;
  const cplx th = ld(&theta[k]);
  double2* base = M.p - (kb + BD_NB) + k * M.stride;  // row-band base of pair k
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = i0 + wid; i < i1; i += nw) {
    double2* rowp = base + i * Wd;
    for (int e = lane; e < Wd; e += 32) {
      const int off = e - (kb + BD_NB);  // j - i
      const int64_t j = i + off;
      const int ao = off < 0 ? -off : off;
      double v = 0.0;
      if (ao <= kb && j >= 0 && j < N) v = ao == 0 ? band[i] : band[(int64_t)ao * N + (off < 0 ? j : i)];
      double2 z = make_double2(v, 0.0);
      if (off == 0) {
        z.x = (v - shift_c) + th.re;
        z.y = th.im;
      }
      rowp[e] = z;
    }
  }
  for (int64_t e = i0 * nrhs + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < i1 * nrhs;
       e += (int64_t)gridDim.x * blockDim.x)
    X.p[k * X.stride + e] = make_double2(V[e], 0.0);
}


// The factorisation + solves touch only the workspace, so the ~8 launches per 64-row
// block step are captured once into a CUDA graph per (shape, workspace) and replayed:
// the per-launch host overhead was the bound of this path (N/64 = 4096 block steps).
// Block back substitution y1 = U11^{-1} (y1 - U12 y2) for one 64-row block, all pairs:
// bd_back_partial splits the kb-long inner dimension into 32-wide chunks (one CTA per chunk
// and pair: P[q] = U12[:, chunk q] y2[chunk q]), bd_back_finish sums the chunks in
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
};

__device__ void bd_combine_rows(const ZMat& X, int64_t j0, int jb, int nr, int npairs, const BdCombine* cmb) {
  const double2* coef = cmb->coef;
  const double sc = cmb->scale;
  for (int e = threadIdx.x; e < jb * nr; e += blockDim.x) {
    const int64_t i = (j0 + e / nr) * nr + e % nr;  // element of the N x nr block
    double acc = 0.0;
    for (int k = 0; k < npairs; ++k) {
      const cplx a = ld(&coef[k]);
      const double2 x = X.p[k * X.stride + i];
      const double sk = 2.0 * fma(a.re, x.x, -a.im * x.y);
      acc = k == 0 ? sk : acc + sk;
    }
    cmb->out[i] = sc == 1.0 ? acc : sc * acc;
  }
}

__global__ void bd_combine_block(ZMat X, int64_t j0, int jb, int nr, int npairs, const BdCombine* cmb) {
  bd_combine_rows(X, j0, jb, nr, npairs, cmb);
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
    if (b == 0) bd_combine_rows(X, cj0, cjb, nr, gridDim.y, cmb);
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

// Three streams inside one captured graph: the critical chain (diagonal LU -> inverses ->
// L21 -> A22 update -> next LU) stays on `main`; U12 = L11^{-1} M12 runs beside L21 on
// `s1`; the right-hand-side elimination (y1 = L11^{-1} y1, y2 -= L21 y1) trails on `s2`,
// where it overlaps the next block steps (its inputs, L11^{-1} per block and the L21
// columns, are never written again).
struct BdStreams {
  cudaStream_t s1 = nullptr, s2 = nullptr, s3 = nullptr, s4 = nullptr;
  cudaEvent_t ev[8] = {};
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
    PFX_CUDA_TRY(cudaStreamCreateWithPriority(&g.s2, cudaStreamNonBlocking, lo));
    PFX_CUDA_TRY(cudaStreamCreateWithPriority(&g.s3, cudaStreamNonBlocking, lo));
    for (auto& e : g.ev) PFX_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  S = g;
  return PFX_OK;
}

static int bd_factor_solve(cudaStream_t stream, ZMat M, ZMat X, ZMat Li, ZMat Ui, double2* P, int64_t N, int kb,
                           int nr, int npairs, int* sing, const BdCombine* cmb) {
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
  // PFX_BD_SKIP (timing experiments only, results are wrong): bit 0 back substitution,
  // bit 1 rhs chain, bit 2 trailing update, bit 3 diagonal LU + inverses, bit 4 panel products
  static const int skip = [] {
    const char* e = getenv("PFX_BD_SKIP");
    return e ? atoi(e) : 0;
  }();
  cudaEvent_t evT = S.ev[0], evU = S.ev[1], evL = S.ev[2], evR = S.ev[3], evP = S.ev[4], evB = S.ev[5];
  cudaEvent_t evS = S.ev[6], evA = S.ev[7];
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
      // look-ahead: only the next diagonal block (ra x ra) is updated on main before the next
      // LU; the rest of the next row / column strips (needed by the next panel products)
      // go to s4, and the trailing (rest - ra)^2 part to s3, both overlapping the next LU /
      // inverses.  Everything here lies inside the previous step's trailing region, so main
      // waits for it (evB) first.
      const int ra = std::min(nb, rest);
      PFX_CUDA_TRY(cudaStreamWaitEvent(stream, evU, 0));
      if (pending_b) PFX_CUDA_TRY(cudaStreamWaitEvent(stream, evB, 0));
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
          // the trailing update becomes ready together with the next block's LU (both after
          // the diagonal-block update), so the higher-priority LU is dispatched first
          PFX_CUDA_TRY(cudaEventRecord(evA, stream));
          PFX_CUDA_TRY(cudaStreamWaitEvent(S.s3, evA, 0));
          if ((rc = zgemm(S.s3, npairs, rest - ra, rest - ra, jb, -1.0, sub(M, j0 + jb + ra, j0),
                          sub(M, j0, j0 + jb + ra), sub(M, j0 + jb + ra, j0 + jb + ra))))
            return rc;
          PFX_CUDA_TRY(cudaEventRecord(evB, S.s3));
          pending_b = true;
        }
      }
    }
  }
  if (pending_s) PFX_CUDA_TRY(cudaStreamWaitEvent(stream, evS, 0));
  if (pending_b) PFX_CUDA_TRY(cudaStreamWaitEvent(stream, evB, 0));
  PFX_CUDA_TRY(cudaEventRecord(evR, S.s2));
  PFX_CUDA_TRY(cudaStreamWaitEvent(stream, evR, 0));
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
               bd_combine_block<<<1, 256, 0, stream>>>(X, 0, (int)std::min<int64_t>(nb, N), nr, npairs, cmb));
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
  const size_t mbytes = (size_t)npairs * N * Wd * sizeof(double2);
  const size_t xbytes = (size_t)npairs * N * nrhs * sizeof(double2);
  const int64_t nblk = (N + nb - 1) / nb;
  const size_t libytes = (size_t)npairs * nblk * nb * nb * sizeof(double2);
  const size_t uibytes = (size_t)npairs * nblk * nb * nb * sizeof(double2);
  const size_t pbytes = (size_t)npairs * ceil_div(kb, BK_C) * nb * nrhs * sizeof(double2);
  char* ws = static_cast<char*>(scratch(1, mbytes + xbytes + libytes + uibytes + pbytes + 256 + 64));
  if (!ws) return fail(PFX_CUDA, "banded workspace allocation failed (needs " + std::to_string((mbytes + xbytes) >> 20) + " MiB)");
  ZMat M{reinterpret_cast<double2*>(ws) + kb + nb, Wd - 1, (int64_t)N * Wd};
  ZMat X{reinterpret_cast<double2*>(ws + mbytes), nrhs, N * nrhs};
  ZMat Li{reinterpret_cast<double2*>(ws + mbytes + xbytes), nb, nblk * nb * nb};
  ZMat Ui{reinterpret_cast<double2*>(ws + mbytes + xbytes + libytes), nb, nblk * nb * nb};
  double2* P = reinterpret_cast<double2*>(ws + mbytes + xbytes + libytes + uibytes);
  int* sing = reinterpret_cast<int*>(ws + mbytes + xbytes + libytes + uibytes + pbytes);
  PFX_CUDA_TRY(cudaMemsetAsync(sing, 0, sizeof(int), stream));
  // combine parameters (device copy read by the graph-captured back substitution)
  BdCombine* cmb_d = reinterpret_cast<BdCombine*>(ws + mbytes + xbytes + libytes + uibytes + pbytes + 256);
  {
    static_assert(sizeof(BdCombine) <= 64, "combine parameters fit their slot");
    const BdCombine h{coef_d, shift_c == 0.0 ? 1.0 : exp(shift_c), out};
    // pageable source: the runtime stages it before returning, so a stack value is safe
    PFX_CUDA_TRY(cudaMemcpyAsync(cmb_d, &h, sizeof(h), cudaMemcpyHostToDevice, stream));
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (per_pair_ms) {
    PFX_CUDA_TRY(cudaEventCreate(&e0));
    PFX_CUDA_TRY(cudaEventCreate(&e1));
    PFX_CUDA_TRY(cudaEventRecord(e0, stream));
  }
  dim3 bg(1184, npairs);
  if (!band_host) {
    PFX_LAUNCH("bd_build", stream,
               bd_build<<<bg, 256, 0, stream>>>(band, N, kb, Wd, V, (int)nrhs, shift_c, theta_d, M, X, 0, N));
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
                 bd_build<<<bg, 256, 0, stream>>>(band, N, kb, Wd, V, (int)nrhs, shift_c, theta_d, M, X, i0, i1));
      PFX_CUDA_TRY(cudaGetLastError());
    }
  }
  if (prof_on()) {
    // profiling wants per-kernel events: run the launches directly
    if (int rc = bd_factor_solve(stream, M, X, Li, Ui, P, N, kb, (int)nrhs, npairs, sing, cmb_d)) return rc;
  } else {
    const int gdev = current_device();
    if (gdev < 0 || gdev >= kMaxDevices) return fail(PFX_CUDA, "device index out of range");
    BdGraph& G = g_bd_graph[gdev];
    if (!G.exec || G.ws != ws || G.N != N || G.kb != kb || G.nr != (int)nrhs || G.np != npairs) {
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
      int rc = bd_factor_solve(cs, M, X, Li, Ui, P, N, kb, (int)nrhs, npairs, sing, cmb_d);
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
