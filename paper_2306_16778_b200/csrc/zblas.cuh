// Batched complex128 building blocks for blocked LU on sm_100a (used by the large dense
// path, config C4, and the banded path, config C5).
//
// All matrices are row-major complex128 (double2), addressed as base + i*ld + j, with a
// per-batch stride.  A banded matrix stored by rows with its diagonals padded by zeros
// is a dense row-major matrix with ld = (row length - 1), so the same kernels run on
// the band window (banded.cu).
#pragma once
#include "pfx_common.cuh"

namespace pfx {

struct ZMat {
  double2* p;
  int64_t ld;
  int64_t stride;  // batch stride (elements)
  __host__ __device__ double2* at(int b, int64_t i, int64_t j) const { return p + b * stride + i * ld + j; }
};

// Fused residue combine (K5/K6 of the dense path, engine.py:199-213,225-228), riding along in the
// substitution's next GEMM launch: when the backward substitution has finished block row r0
// (rows [r0, r0 + nb) of every system's X_k are final), the next zgemm launch carries one extra
// z-slice of CTAs that sums the systems in ascending k for the entries that block row decides
// and writes them to `out` -- in parallel with that GEMM's tiles, reading rows just written
// (L2-hot), so no separate pass over the n/2 solutions and no step on the serial chain.
//   mode 1  complex full:   out = sum_k a_k X_k + (a_k X_k)^H  (Hermitian; the block row's
//           entries right of its diagonal and their mirror images, X_k[strip, block] rows
//           being final already: every (i, j) is written by block row min(i, j))
//   mode 2  real full, X_k complex symmetric stored as its lower triangle:
//           out = sum_k 2 Re(a_k X_k)  (entries left of the diagonal and their mirrors)
//   mode 3  real action:    out = sum_k 2 Re(a_k Y_k)
//   mode 4  complex action: out = sum_k a_k Y_k + conj(a_k) Yc_k  (Yc_k = system npairs + k)
struct ZCombine {
  int mode = 0;          // 0: no combine
  int npairs = 0;
  const double2* coef = nullptr;
  double scale = 1.0;    // e^c of the shift method
  double* out = nullptr; // d x ncols, real (modes 2, 3) or complex (1, 4), row-major
  int64_t ldo = 0;       // row stride of out (elements)
  ZMat X{nullptr, 0, 0}; // the systems' solutions, rows relative to row0
  int64_t row0 = 0;      // first row of the finished block row (= its column for the diagonal)
  int nb = 0;            // rows in the block row
  int ncols = 0;         // columns of out / X
};
// Launch a combine on its own (the last block row, which no later GEMM follows).
int zcombine(cudaStream_t s, const ZCombine& cm);

// C[b] += alpha * A[b] (m x k) * B[b] (k x n) (accumulate = true) or C[b] = alpha * A B.
// DMMA m8n8k4, 64x64x16 tiles.
// b_lower_off >= 0: B (k x n) is lower triangular with that row offset, B[r][c] = 0 for
// r + b_lower_off < c; each column tile skips the zero rows (the forward substitution of the
// identity right-hand side).  -1: B dense.
// ride (optional): a residue combine carried by this launch (one extra z-slice of CTAs).
int zgemm(cudaStream_t s, int batch, int m, int n, int k, double alpha, ZMat A, ZMat B, ZMat C,
          bool accumulate = true, int b_lower_off = -1, const ZCombine* ride = nullptr, int a_upper_off = -1);
// a_upper_off >= 0: A (m x k) is upper trapezoidal with that offset, A[r][c] = 0 for
// c + a_upper_off < r; each row tile skips the zero columns (the band edge in a left-looking
// update).  a_upper_off = -2: no structure in A, but -- like a_upper_off >= 0 -- the operands live
// in band storage, so the skipped K range (also b_lower_off's) is rounded to whole 64-blocks.

// While alive on this thread, K <= 64 zgemm launches prefer the 32 x 32 tiles even on large
// grids (the banded path's K = 64 trailing updates; see zgemm()).
class ZgemmShortK {
 public:
  explicit ZgemmShortK(bool on);
  ~ZgemmShortK();
  ZgemmShortK(const ZgemmShortK&) = delete;
  ZgemmShortK& operator=(const ZgemmShortK&) = delete;

 private:
  bool prev_;
};

// No-pivot LU of the nb x nb diagonal block D (nb <= 64) in registers, in place.  Raises
// ST_SINGULAR in *sing on an exactly zero pivot and ST_PIVOT where partial pivoting inside the
// block would have exchanged rows (the rows below the block are checked by ztrmm_inplace).
int zgetrf_diag(cudaStream_t s, int batch, int nb, ZMat D, int* sing);
// Triangular inverses of a factored diagonal block: Li = L^{-1} (unit lower), Ui = U^{-1}.
int ztrtri_diag(cudaStream_t s, int batch, int nb, ZMat D, ZMat Li, ZMat Ui);
// In place: B = Tinv * B (left, B nb x n) or B = B * Tinv (right, B n x nb), Tinv nb x nb
// (nb <= 64) triangular (upper or lower), on DMMA; one CTA per 32-wide strip of B.

// pivot_flag (right products only): B = L21 = A21 U11^{-1} of a no-pivot LU step whose
// diagonal block (factored in place) is Dg; every entry is checked against partial pivoting
// (|l u_cc|_1 > |u_cc|_1 means row interchanges were due) and ST_PIVOT is or-ed into *pivot_flag.
int ztrmm_inplace(cudaStream_t s, int batch, int nb, int n, ZMat Tinv, ZMat B, bool right, bool upper,
                  ZMat Dg = ZMat{nullptr, 0, 0}, int* pivot_flag = nullptr);

// Unblocked LU of the m x nb panel at P (in place).  ipiv (optional, batch x nb, 0-based
// rows relative to the panel) -> partial pivoting with row swaps inside the panel only.
// sing: device int set to 1 on an exactly zero pivot.
int zgetf2_panel(cudaStream_t s, int batch, int m, int nb, ZMat P, int* ipiv, int* sing);

// Apply the panel's interchanges (rows r0+j <-> r0+ipiv[j], j = 0..nb-1, in order) to
// columns [c0, c1) of A (skipping nothing; caller passes the column ranges).
int zlaswp(cudaStream_t s, int batch, int nb, ZMat A, int64_t r0, int64_t c0, int64_t c1, const int* ipiv, int dir);

// B = L^{-1} B, L = unit lower nb x nb at Lm (strictly lower part used), B nb x n.
int ztrsm_llnu(cudaStream_t s, int batch, int nb, int n, ZMat Lm, ZMat B);
// B = U^{-1} B, U = upper (non-unit) nb x nb, B nb x n.
int ztrsm_lunn(cudaStream_t s, int batch, int nb, int n, ZMat Um, ZMat B);

}  // namespace pfx
