// Batched blocked path for MANY small dense systems in action mode (config C3: 512 matrices x
// 10 pole pairs = 5,120 systems of d = 256, one right-hand side).
//
// Replaces, for those shapes, the persistent one-CTA-per-system kernel of dense_batched.cu:
// the systems are factored together by the block toolkit (zblas.cu), every launch batched over
// all of them, so the LU runs as DMMA GEMMs on the 64 x 64 four-warp tiles instead of inside
// one SM's shared memory.  Reference (engine.py:194-206, complex action):
//   M_k = A_b - cI + theta_k I,   [M | V] -> [U | L^{-1} V]       lu_factor_nopiv, the RHS carried
//                                                                  as extra columns of M
//   y  = U^{-1} (L^{-1} V)                                          bt_solve mode 0
//   yc = M^{-H} V = L^{-H} U^{-H} V                                 bt_solve modes 1, 2 (the
//        conjugate-transpose solves on the same LU, lu_solve(trans=2) of engine.py:205)
//   out_b = e^c sum_k a_k y + conj(a_k) yc   (real path: 2 Re(a_k y))   db_combine, k ascending
// Pivoting: the LU is interchange-free and checked against partial pivoting (pfx_set_pivot_mode);
// a failed check redoes the call on the pivoting kernels of dense_batched.cu.
#include "zblas.cuh"

namespace pfx {

int lu_factor_nopiv(cudaStream_t s, int nsys, int d, int naug, ZMat M, ZMat Li, ZMat Ui, int* sing,
                    bool check_pivots);
int dense_batched_run(const double* A, int a_complex, int d, int batch, const double* V, int v_complex, int ncols,
                      int full, int real_path, int solve_only, double shift_c, const double2* theta_d,
                      const double2* coef_d, int npairs, double* out, cudaStream_t stream, float* launch_ms,
                      int pivot);

constexpr int DB2_NB = 64;
constexpr int BT_NR = 4;  // right-hand sides handled by the solve kernel

// [M | V] for system s = b * npairs + k: M = A_b - cI + theta_k I (d x d), V_b (d x nr)
__global__ void db_build(const double* A, int a_complex, int d, const double* V, int v_complex, int nr,
                         double shift_c, const double2* theta, int npairs, ZMat M) {
  const int s = blockIdx.y;
  const int b = s / npairs, k = s - b * npairs;
  const cplx th = ld(&theta[k]);
  const int w = d + nr;
  const int64_t dd = (int64_t)d * d;
  double2* Ms = M.p + s * M.stride;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)d * w;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / w), j = (int)(e - (e / w) * w);
    double2 v;
    if (j < d) {
      const int64_t ai = (int64_t)b * dd + (int64_t)i * d + j;
      v = a_complex ? reinterpret_cast<const double2*>(A)[ai] : make_double2(A[ai], 0.0);
      if (i == j) {
        v.x = (v.x - shift_c) + th.re;
        v.y = v.y + th.im;
      }
    } else {
      const int64_t vi = ((int64_t)b * d + i) * nr + (j - d);
      v = v_complex ? reinterpret_cast<const double2*>(V)[vi] : make_double2(V[vi], 0.0);
    }
    Ms[(int64_t)i * M.ld + j] = v;
  }
}

// Block triangular solves on one system per CTA (256 threads), the unknowns in shared memory.
//   mode 0  x = U^{-1} x,  x = columns d.. of M (in place): rows of U read along the row
//   mode 1  z = U^{-H} v   (v = the system's V_b):             columns of U read along rows
//   mode 2  x = L^{-H} z   (z in Z, in place):                 columns of L read along rows
// Diagonal blocks through the stored inverses (Ui = U_pp^{-1}, Li = L_pp^{-1}; for the
// conjugate transposes their conjugate transposes).
__global__ void __launch_bounds__(256) bt_solve(int mode, int d, int nr, ZMat M, ZMat Li, ZMat Ui, ZMat Z,
                                                const double* V, int v_complex, int npairs) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* xs = reinterpret_cast<double2*>(smem_raw);  // d x BT_NR
  double2* part = xs + (size_t)d * BT_NR;              // 4 x 64 x BT_NR partial sums, then t
  const int s = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double2* Ms = M.p + s * M.stride;
  const double2* Lis = Li.p + s * Li.stride;
  const double2* Uis = Ui.p + s * Ui.stride;
  const int nblk = (d + DB2_NB - 1) / DB2_NB;
  // load the right-hand sides
  for (int e = tid; e < d * BT_NR; e += 256) {
    const int i = e / BT_NR, c = e - (e / BT_NR) * BT_NR;
    double2 v = make_double2(0, 0);
    if (c < nr) {
      if (mode == 0) {
        v = Ms[(int64_t)i * M.ld + d + c];
      } else if (mode == 1) {
        const int b = s / npairs;
        const int64_t vi = ((int64_t)b * d + i) * nr + c;
        v = v_complex ? reinterpret_cast<const double2*>(V)[vi] : make_double2(V[vi], 0.0);
      } else {
        v = Z.p[s * Z.stride + (int64_t)i * nr + c];
      }
    }
    xs[e] = v;
  }
  __syncthreads();
  for (int q = 0; q < nblk; ++q) {
    const int p = mode == 1 ? q : nblk - 1 - q;
    const int j0 = p * DB2_NB, jb = min(DB2_NB, d - j0);
    // ---- t = x_p - (coupling to the finished blocks) x_done
    if (mode == 0) {
      // rows of U: warp per row, lanes along the row
      for (int i = warp; i < jb; i += 8) {
        cplx acc[BT_NR];
#pragma unroll
        for (int c = 0; c < BT_NR; ++c) acc[c] = mk(0, 0);
        const double2* urow = Ms + (int64_t)(j0 + i) * M.ld;
        for (int j = j0 + jb + lane; j < d; j += 32) {
          const cplx u = ld(&urow[j]);
#pragma unroll
          for (int c = 0; c < BT_NR; ++c) acc[c] = cfma(u, ld(&xs[j * BT_NR + c]), acc[c]);
        }
#pragma unroll
        for (int c = 0; c < BT_NR; ++c) {
          for (int o = 16; o > 0; o >>= 1) {
            acc[c].re += __shfl_xor_sync(0xffffffffu, acc[c].re, o);
            acc[c].im += __shfl_xor_sync(0xffffffffu, acc[c].im, o);
          }
        }
        if (lane < BT_NR) {
          const cplx x = ld(&xs[(j0 + i) * BT_NR + lane]);
          cplx a = acc[0];
#pragma unroll
          for (int c = 1; c < BT_NR; ++c)
            if (lane == c) a = acc[c];
          st(&part[i * BT_NR + lane], csub(x, a));
        }
      }
    } else {
      // columns of U (mode 1: rows j < j0) or L (mode 2: rows j >= j0 + jb), read along rows:
      // thread (i = output, slice sl) walks its quarter of the rows, conj-transposed products
      const int i = tid & 63, sl = tid >> 6;
      const int r0 = mode == 1 ? 0 : j0 + jb, r1 = mode == 1 ? j0 : d;
      const int len = r1 - r0, per = (len + 3) / 4;
      const int a0 = r0 + sl * per, a1 = min(r1, a0 + per);
      cplx acc[BT_NR];
#pragma unroll
      for (int c = 0; c < BT_NR; ++c) acc[c] = mk(0, 0);
      if (i < jb)
        for (int j = a0; j < a1; ++j) {
          const cplx u = cconj(ld(&Ms[(int64_t)j * M.ld + j0 + i]));
#pragma unroll
          for (int c = 0; c < BT_NR; ++c) acc[c] = cfma(u, ld(&xs[j * BT_NR + c]), acc[c]);
        }
#pragma unroll
      for (int c = 0; c < BT_NR; ++c) st(&part[(sl * 64 + i) * BT_NR + c], acc[c]);
      __syncthreads();
      if (sl == 0 && i < jb) {
#pragma unroll
        for (int c = 0; c < BT_NR; ++c) {
          cplx a = ld(&part[i * BT_NR + c]);
          for (int q2 = 1; q2 < 4; ++q2) a = cadd(a, ld(&part[(q2 * 64 + i) * BT_NR + c]));
          st(&part[i * BT_NR + c], csub(ld(&xs[(j0 + i) * BT_NR + c]), a));
        }
      }
    }
    __syncthreads();
    // ---- x_p = T t  (T = Ui, Ui^H or Li^H: 64 x 64 block p)
    {
      const int i = tid & 63, sl = tid >> 6;
      const double2* T = (mode == 2 ? Lis : Uis) + (int64_t)p * DB2_NB * DB2_NB;
      cplx acc[BT_NR];
#pragma unroll
      for (int c = 0; c < BT_NR; ++c) acc[c] = mk(0, 0);
      if (i < jb)
        for (int j = sl * 16; j < min(jb, sl * 16 + 16); ++j) {
          cplx tv;
          if (mode == 0) tv = j >= i ? ld(&T[i * DB2_NB + j]) : mk(0, 0);         // Ui[i][j], upper
          else if (mode == 1) tv = j <= i ? cconj(ld(&T[j * DB2_NB + i])) : mk(0, 0);  // Ui^H, lower
          else tv = j >= i ? cconj(ld(&T[j * DB2_NB + i])) : mk(0, 0);            // Li^H, upper
#pragma unroll
          for (int c = 0; c < BT_NR; ++c) acc[c] = cfma(tv, ld(&part[j * BT_NR + c]), acc[c]);
        }
      __syncthreads();  // every read of t done
      double2* red = part + 64 * BT_NR;  // partials of this product (the t rows stay intact above)
#pragma unroll
      for (int c = 0; c < BT_NR; ++c) st(&red[(sl * 64 + i) * BT_NR + c], acc[c]);
      __syncthreads();
      if (sl == 0 && i < jb) {
#pragma unroll
        for (int c = 0; c < BT_NR; ++c) {
          cplx a = ld(&red[i * BT_NR + c]);
          for (int q2 = 1; q2 < 4; ++q2) a = cadd(a, ld(&red[(q2 * 64 + i) * BT_NR + c]));
          st(&xs[(j0 + i) * BT_NR + c], a);
        }
      }
      __syncthreads();
    }
  }
  // write back: mode 0 into M's right-hand-side columns, modes 1 / 2 into Z
  for (int e = tid; e < d * nr; e += 256) {
    const int i = e / nr, c = e - (e / nr) * nr;
    const double2 v = xs[i * BT_NR + c];
    if (mode == 0) const_cast<double2*>(Ms)[(int64_t)i * M.ld + d + c] = v;
    else Z.p[s * Z.stride + e] = v;
  }
}

// out_b = e^c sum_k S_k, k ascending (engine.py:201,206,225-228)
__global__ void db_combine(ZMat M, ZMat Z, int d, int nr, int batch, int npairs, const double2* coef, int real_path,
                           double scale, double* out) {
  const int64_t per = (int64_t)d * nr;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)batch * per;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(e / per);
    const int64_t r = e - (int64_t)b * per;
    const int i = (int)(r / nr), c = (int)(r - (r / nr) * nr);
    if (real_path) {
      double acc = 0.0;
      for (int k = 0; k < npairs; ++k) {
        const cplx a = ld(&coef[k]);
        const cplx y = ld(M.at(b * npairs + k, i, d + c));
        const double sk = 2.0 * fma(a.re, y.re, -a.im * y.im);
        acc = k == 0 ? sk : acc + sk;
      }
      out[e] = scale == 1.0 ? acc : scale * acc;
    } else {
      cplx acc = mk(0, 0);
      for (int k = 0; k < npairs; ++k) {
        const int s = b * npairs + k;
        const cplx a = ld(&coef[k]);
        const cplx sk = cadd(cmul(a, ld(M.at(s, i, d + c))), cmul(cconj(a), ld(&Z.p[s * Z.stride + r])));
        acc = k == 0 ? sk : cadd(acc, sk);
      }
      if (scale != 1.0) acc = cscale(acc, scale);
      reinterpret_cast<double2*>(out)[e] = make_double2(acc.re, acc.im);
    }
  }
}

// Opt-in (PFX_DENSE_BLOCKED=1): measured on C3 (5,120 systems of d = 256) at 26.5 ms against
// 19.0 ms for the one-CTA-per-system kernel -- the LU GEMMs take 6.2 ms, but the 64 x 64 panel
// kernels at this count (diagonal LU 3.9 ms, triangular inverses 6.0 ms, panel products 5.4 ms)
// cost more than the fused kernel's whole factorisation.  Kept, tested, for A/B work.
int dense_blocked_eligible(int64_t d, int64_t batch, int npairs, int full, int64_t ncols) {
  static const int force = [] {
    const char* e = getenv("PFX_DENSE_BLOCKED");
    return e ? atoi(e) : 0;
  }();
  if (full || ncols < 1 || ncols > BT_NR || d < 64 || d > 512) return 0;
  return force > 0;
}

int dense_blocked_run(const double* A, int a_complex, int d, int batch, const double* V, int v_complex, int nr,
                      int real_path, double shift_c, const double2* theta_d, const double2* coef_d, int npairs,
                      double* out, cudaStream_t stream, float* launch_ms, int pivot) {
  const int nb = DB2_NB;
  const int nsys = batch * npairs;
  const int w = d + nr;
  const int nblk = (d + nb - 1) / nb;
  const size_t mbytes = (size_t)nsys * d * w * sizeof(double2);
  const size_t tbytes = (size_t)nsys * nblk * nb * nb * sizeof(double2);
  const size_t zbytes = real_path ? 0 : (size_t)nsys * d * nr * sizeof(double2);
  char* ws = static_cast<char*>(scratch(1, mbytes + 2 * tbytes + zbytes + 256));
  if (!ws) return fail(PFX_CUDA, "blocked dense workspace allocation failed");
  ZMat M{reinterpret_cast<double2*>(ws), w, (int64_t)d * w};
  ZMat Li{reinterpret_cast<double2*>(ws + mbytes), nb, (int64_t)nblk * nb * nb};
  ZMat Ui{reinterpret_cast<double2*>(ws + mbytes + tbytes), nb, (int64_t)nblk * nb * nb};
  ZMat Z{reinterpret_cast<double2*>(ws + mbytes + 2 * tbytes), nr, (int64_t)d * nr};
  int* sing = reinterpret_cast<int*>(ws + mbytes + 2 * tbytes + zbytes);
  PFX_CUDA_TRY(cudaMemsetAsync(sing, 0, sizeof(int), stream));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (launch_ms) {
    PFX_CUDA_TRY(cudaEventCreate(&e0));
    PFX_CUDA_TRY(cudaEventCreate(&e1));
    PFX_CUDA_TRY(cudaEventRecord(e0, stream));
  }
  PFX_LAUNCH("db_build", stream,
             db_build<<<dim3(8, nsys), 256, 0, stream>>>(A, a_complex, d, V, v_complex, nr, shift_c, theta_d, npairs, M));
  PFX_CUDA_TRY(cudaGetLastError());
  int rc = lu_factor_nopiv(stream, nsys, d, nr, M, Li, Ui, sing, pivot == 2);
  if (rc) return rc;
  int* hsg = pinned_word();
  if (!hsg) return fail(PFX_CUDA, "pinned status word allocation failed");
  if (pivot == 2) {
    PFX_CUDA_TRY(cudaMemcpyAsync(hsg, sing, sizeof(int), cudaMemcpyDeviceToHost, stream));
    if (int rc_ = sync_stream(stream)) return rc_;
    if (*hsg & ST_PIVOT) {
      // a column partial pivoting would have exchanged: redo on the pivoting kernels
      note_pivot_fallback();
      if (launch_ms) {
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
      }
      return dense_batched_run(A, a_complex, d, batch, V, v_complex, nr, 0, real_path, 0, shift_c, theta_d, coef_d,
                               npairs, out, stream, launch_ms, 1);
    }
  }
  const int smem = (d * BT_NR + 2 * 4 * 64 * BT_NR) * (int)sizeof(double2);
  if ((rc = raise_smem_limit(reinterpret_cast<const void*>(bt_solve), smem))) return rc;
  PFX_LAUNCH("bt_solve", stream, bt_solve<<<nsys, 256, smem, stream>>>(0, d, nr, M, Li, Ui, Z, V, v_complex, npairs));
  PFX_CUDA_TRY(cudaGetLastError());
  if (!real_path) {
    PFX_LAUNCH("bt_solve", stream, bt_solve<<<nsys, 256, smem, stream>>>(1, d, nr, M, Li, Ui, Z, V, v_complex, npairs));
    PFX_CUDA_TRY(cudaGetLastError());
    PFX_LAUNCH("bt_solve", stream, bt_solve<<<nsys, 256, smem, stream>>>(2, d, nr, M, Li, Ui, Z, V, v_complex, npairs));
    PFX_CUDA_TRY(cudaGetLastError());
  }
  const double scale = shift_c == 0.0 ? 1.0 : exp(shift_c);
  PFX_LAUNCH("db_combine", stream,
             db_combine<<<1184, 256, 0, stream>>>(M, Z, d, nr, batch, npairs, coef_d, real_path, scale, out));
  PFX_CUDA_TRY(cudaGetLastError());
  PFX_CUDA_TRY(cudaMemcpyAsync(hsg, sing, sizeof(int), cudaMemcpyDeviceToHost, stream));
  if (launch_ms) PFX_CUDA_TRY(cudaEventRecord(e1, stream));
  if (int rc_ = sync_stream(stream)) return rc_;
  if (launch_ms) {
    PFX_CUDA_TRY(cudaEventElapsedTime(launch_ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  if (*hsg & ST_SINGULAR) return fail(PFX_SINGULAR, "exactly zero pivot in a shifted factorization");
  return PFX_OK;
}

}  // namespace pfx
