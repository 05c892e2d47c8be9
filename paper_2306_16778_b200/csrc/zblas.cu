// Batched complex128 block toolkit for sm_100a (see zblas.cuh): GEMM, diagonal-block LU and
// triangular inverses, in-place triangular products, and the pivoting panel / row
// interchange / TRSM kernels of the general shifted solve.
//
// zgemm: 64x64 (8 warps, 32x16 per warp) or 32x32 (4 warps) output tile per CTA, K staged
// 16 complex at a time through shared memory with cp.async double buffering.  A complex
// 8x8x4 step is three real DMMA.8x8x4 (3M: T1 = Ar Br, T2 = Ai Bi, T3 = (Ar+Ai)(Br+Bi);
// Cr = T1 - T2, Ci = T3 - T1 - T2), or four with PFX_ZGEMM_4M=1.  Shared-memory rows are
// padded (GAS, TN + 2) so both fragment loads spread over all 32 banks (4 wavefronts per
// 512-byte warp request, the minimum).
#include "zblas.cuh"

#include <cuda.h>  // CUtensorMap (the encoder is fetched from the driver at run time, no -lcuda)

namespace pfx {

// K staged KS complex at a time (16 by default; 32 for the small-grid, K <= 64 launches of the
// band LU's critical chain, where the number of load round trips sets the latency).
// Row strides (in 16-byte words) for conflict-free DMMA fragment loads: a quarter-warp reads
// A at rows g (0..1) x columns t (0..3) -> stride 4 mod 8; B at rows t x columns g -> stride
// 2 mod 8 (KS + 1 and TN + 1 were 2-way conflicted: ncu counted half the wavefronts as excess)
// NS-stage cp.async ring (double buffering)
template <int TM, int TN, int KS, int NS = 2>
struct GemmSmem {
  double2 A[NS][TM][KS + 4];
  double2 B[NS][KS][TN + 2];
};
template <int TM, int NW>
__host__ __device__ constexpr int gemm_stages() { return 2; }  // 3 stages on the 4-warp layout: no gain on long K, -14% on K = 128 (tools/zgemm_probe.cu)

// ---------------------------------------------------------------------------
// TMA staging of the zgemm tiles (cp.async.bulk.tensor, completion on an mbarrier).  The row
// padding of GemmSmem (A rows KS + 4, B rows TN + 2 complex) is produced by widening the box:
// the A box is KS + 4 complex wide and the B box TN + 2, so the copy lands in exactly the
// padded, bank-conflict-free layout the fragment loads expect (the extra columns are never
// read; columns past the matrix edge are zero-filled like every out-of-range element).
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
  static const EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return (EncodeTiledFn) nullptr;
    }
    return (EncodeTiledFn)f;
  }();
  return fn;
}

// Tensor map of a batch of rows x cols complex matrices (row stride ld, batch stride `stride`,
// elements) as float64 [batch][rows][2 cols]; box = box_rows x box_cols complex.  False when
// the driver has no encoder or the layout is not expressible (the caller then stages with
// cp.async).
static bool zmat_tensor_map(CUtensorMap* map, const ZMat& M, int rows, int cols, int batch, int box_rows,
                            int box_cols) {
  const EncodeTiledFn enc = encode_tiled();
  if (!enc || batch < 1 || rows < 1 || cols < 1) return false;
  if (batch > 1 && M.stride <= 0) return false;  // broadcast operand
  if ((reinterpret_cast<uintptr_t>(M.p) & 15) != 0) return false;
  const int64_t bstride = batch > 1 ? M.stride : M.ld * rows;
  const cuuint64_t dims[3] = {2 * (cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)batch};
  const cuuint64_t strides[2] = {(cuuint64_t)M.ld * 16, (cuuint64_t)bstride * 16};
  const cuuint32_t box[3] = {2 * (cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)M.p, dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, bool valid) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}

// ---------------------------------------------------------------------------
// Residue combine riding along in a later launch (see ZCombine in zblas.cuh).  All loads of
// the solutions bypass L1 (other CTAs of earlier launches wrote them).
__device__ __forceinline__ cplx ldcg(const double2* p) {
  const double2 v = __ldcg(p);
  return cplx{v.x, v.y};
}

// Mode 1 (complex full, Hermitian) for the block row's columns [c0, c1): the mirrored reads
// X_k[c, r0 + r] and the mirrored writes out[c, r0 + r] go through shared memory (sm: >= 64 x 65
// double2) so that every global access runs along a row; each thread keeps its elements' sums
// in registers across the systems.
__device__ void combine_hermitian(const ZCombine& cm, int c0, int c1, double2* sm) {
  constexpr int MAXE = (64 * 64) / 128;  // >= 128 threads per CTA
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t r0 = cm.row0;
  const int nb = cm.nb, w = c1 - c0;
  const int SP = nb + 1;  // sm[c * SP + r]
  const ZMat& X = cm.X;
  cplx acc[MAXE];
#pragma unroll
  for (int i = 0; i < MAXE; ++i) acc[i] = mk(0, 0);
  for (int k = 0; k < cm.npairs; ++k) {
    __syncthreads();
    // X_k[c0 + cc, r0 + r], coalesced along r; eight loads in flight per thread
    for (int e0 = tid; e0 < w * nb; e0 += 8 * nt) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * nt;
        const int cc = e / nb, r = e - cc * nb;
        v[u] = e < w * nb ? __ldcg(X.at(k, c0 + cc - r0, r0 + r)) : make_double2(0, 0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * nt;
        const int cc = e / nb, r = e - cc * nb;
        if (e < w * nb) sm[cc * SP + r] = v[u];
      }
    }
    __syncthreads();
    const cplx a = ld(&cm.coef[k]);
#pragma unroll
    for (int i = 0; i < MAXE; ++i) {
      const int e = tid + nt * i;
      if (e < nb * w) {
        const int r = e / w, c = e - r * w;  // coalesced along c
        const cplx x = ldcg(X.at(k, r, c0 + c));
        const cplx y = ld(&sm[c * SP + r]);
        const cplx sk = cadd(cmul(a, x), cconj(cmul(a, y)));
        acc[i] = k == 0 ? sk : cadd(acc[i], sk);
      }
    }
  }
  __syncthreads();
  double2* out = reinterpret_cast<double2*>(cm.out);
#pragma unroll
  for (int i = 0; i < MAXE; ++i) {
    const int e = tid + nt * i;
    if (e < nb * w) {
      const int r = e / w, c = e - r * w;
      cplx v = acc[i];
      if (cm.scale != 1.0) v = cscale(v, cm.scale);
      out[(r0 + r) * cm.ldo + c0 + c] = make_double2(v.re, v.im);
      sm[c * SP + r] = make_double2(v.re, -v.im);  // the mirror image, written row-wise below
    }
  }
  __syncthreads();
  for (int e = tid; e < w * nb; e += nt) {
    const int cc = e / nb, r = e - cc * nb;
    if (c0 + cc != r0 + r) out[(int64_t)(c0 + cc) * cm.ldo + r0 + r] = sm[cc * SP + r];
  }
}

// Modes 2-4 for the block row's columns [c0, c1) (no transposed reads).
__device__ void combine_plain(const ZCombine& cm, int c0, int c1) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t r0 = cm.row0;
  const int nb = cm.nb, w = c1 - c0;
  const double sc = cm.scale;
  const ZMat& X = cm.X;
  for (int e = tid; e < nb * w; e += nt) {
    const int r = e / w, c = c0 + (e - r * w);
    const int64_t gr = r0 + r;
    if (cm.mode == 4) {
      cplx acc = mk(0, 0);
      for (int k = 0; k < cm.npairs; ++k) {
        const cplx a = ld(&cm.coef[k]);
        const cplx sk = cadd(cmul(a, ldcg(X.at(k, r, c))), cmul(cconj(a), ldcg(X.at(cm.npairs + k, r, c))));
        acc = k == 0 ? sk : cadd(acc, sk);
      }
      if (sc != 1.0) acc = cscale(acc, sc);
      reinterpret_cast<double2*>(cm.out)[gr * cm.ldo + c] = make_double2(acc.re, acc.im);
      continue;
    }
    if (cm.mode == 2 && c > gr) continue;  // lower triangle (the diagonal block's upper half mirrors)
    double acc = 0.0;
    for (int k = 0; k < cm.npairs; ++k) {
      const cplx a = ld(&cm.coef[k]);
      const cplx x = ldcg(X.at(k, r, c));
      const double sk = 2.0 * fma(a.re, x.re, -a.im * x.im);
      acc = k == 0 ? sk : acc + sk;
    }
    if (sc != 1.0) acc *= sc;
    cm.out[gr * cm.ldo + c] = acc;
    if (cm.mode == 2 && c != gr) cm.out[(int64_t)c * cm.ldo + gr] = acc;
  }
}

// The column groups one finished block row decides: mode 1 its diagonal block (one group: the
// mirrored reads cross its own rows) and the 32-wide strips right of it; mode 2 the diagonal
// block and the strips left of it; modes 3/4 every column.  Group g -> [c0, c1).
__device__ __forceinline__ int combine_groups(const ZCombine& cm) {
  const int64_t r0 = cm.row0;
  if (cm.mode == 1) return 1 + (int)((cm.ncols - (r0 + cm.nb) + 31) / 32);
  if (cm.mode == 2) return 1 + (int)((r0 + 31) / 32);
  return (cm.ncols + 31) / 32;
}
__device__ __forceinline__ void combine_group_cols(const ZCombine& cm, int g, int& c0, int& c1) {
  const int r0 = (int)cm.row0;
  if (cm.mode == 3 || cm.mode == 4) {
    c0 = g * 32;
    c1 = min(cm.ncols, c0 + 32);
  } else if (g == 0) {
    c0 = r0;
    c1 = r0 + cm.nb;
  } else if (cm.mode == 1) {
    c0 = r0 + cm.nb + (g - 1) * 32;
    c1 = min(cm.ncols, c0 + 32);
  } else {
    c0 = (g - 1) * 32;
    c1 = min(r0, c0 + 32);
  }
}

// Every CTA of the carrying slice takes groups cta, cta + nctas, ...
__device__ void ride_combine(const ZCombine& cm, int cta, int nctas, double2* sm) {
  const int ng = combine_groups(cm);
  for (int g = cta; g < ng; g += nctas) {
    int c0, c1;
    combine_group_cols(cm, g, c0, c1);
    if (c1 <= c0) continue;
    if (cm.mode == 1) combine_hermitian(cm, c0, c1, sm);
    else combine_plain(cm, c0, c1);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) zcombine_kernel(ZCombine cm) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ride_combine(cm, blockIdx.x, gridDim.x, reinterpret_cast<double2*>(smem_raw));
}

int zcombine(cudaStream_t s, const ZCombine& cm) {
  if (cm.mode == 0) return PFX_OK;
  const int smem = 64 * 65 * (int)sizeof(double2);
  if (int rc = raise_smem_limit(reinterpret_cast<const void*>(zcombine_kernel), smem)) return rc;
  PFX_LAUNCH("zcombine", s, zcombine_kernel<<<148, 256, smem, s>>>(cm));
  PFX_CUDA_TRY(cudaGetLastError());
  return PFX_OK;
}

// TM x TN output tile, NW warps in a 2 x (NW/2) grid, each warp FM x FN DMMA 8x8 tiles.
// 64x64/8 warps for large problems; 32x32/4 warps when the 64-tile grid would leave SMs
// idle (one 64x64x64 complex tile is ~16K DMMA cycles of a single SM).
// M3: the 3M complex product -- three real DMMAs per complex 8x8x4 step instead of four:
// T1 = sum Ar Br, T2 = sum Ai Bi, T3 = sum (Ar + Ai)(Br + Bi), then Cr = T1 - T2 and
// Ci = T3 - T1 - T2 (normwise-stable; the imaginary part's error is bounded by eps |A||B|
// instead of componentwise).
// Two CTAs per SM for the 64x64 tile (<= 128 registers): one CTA's epilogue and K-stage loads
// overlap the other's DMMA stream (at 156 registers a single CTA per SM ran 15% slower).
// TMA: tiles staged by the tensor-memory accelerator (one elected thread issues both boxes of a
// stage, every thread waits on the stage's mbarrier) instead of 16-byte cp.async by all threads.
template <int TM, int TN, int NW, bool M3 = false, int GK = 16, bool TMA = false>
__global__ void __launch_bounds__(NW * 32, (TM == 64 && NW == 4) || NW == 8 ? 2 : 1)
    zgemm_kernel(int m, int n, int k, double alpha, ZMat A, ZMat B, ZMat C, int accumulate, int b_lower_off,
                 ZCombine ride, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 int a_upper_off) {
  constexpr int NT = NW * 32;
  if constexpr (TM == 64 && NW == 4) {  // only this layout carries a combine (register budget)
    // the carried residue combine is slice z = 0: dispatched first, it runs beside the tiles
    if (ride.mode != 0 && blockIdx.z == 0) {
      extern __shared__ __align__(16) unsigned char smem_raw[];
      ride_combine(ride, blockIdx.y * gridDim.x + blockIdx.x, gridDim.x * gridDim.y,
                   reinterpret_cast<double2*>(smem_raw));
      return;
    }
  }
  constexpr int WN = NW / 2;
  constexpr int FM = TM / 2 / 8, FN = TN / WN / 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int NS = gemm_stages<TM, NW>();
  GemmSmem<TM, TN, GK, NS>& S = *reinterpret_cast<GemmSmem<TM, TN, GK, NS>*>(smem_raw);
  const int b = blockIdx.z - ((TM == 64 && NW == 4 && ride.mode != 0) ? 1 : 0);
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;  // warp tile rows [wm*TM/2, +TM/2), cols [wn*FN*8, +FN*8)
  const double2* Ab = A.p + b * A.stride;
  const double2* Bb = B.p + b * B.stride;
  double cr[FM][FN][2], ci[FM][FN][2];
  double t3[M3 ? FM : 1][M3 ? FN : 1][2];  // M3: cr = T1, ci = T2, t3 = T3
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) {
      cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;
      if (M3) t3[M3 ? i : 0][M3 ? j : 0][0] = t3[M3 ? i : 0][M3 ? j : 0][1] = 0.0;
    }

  const int ktiles = (k + GK - 1) / GK;
  // b_lower_off >= 0: B is lower triangular with offset (B[r][c] = 0 for r + off < c), so
  // this column tile's products start at row n0 - off of B; a tile entirely right of the
  // triangle adds nothing
  // a_upper_off >= 0: A is upper trapezoidal with offset (A[r][c] = 0 for c + off < r: the band's
  // edge in a left-looking update), so this row tile's products start at column m0 - off of A.
  // a_upper_off != -1 (band storage, where out-of-band entries alias other rows beyond the 64
  // padded diagonals): the start is rounded down to a 64-row block, never to a finer K stage.
  int ks = 0;
  if (b_lower_off >= 0) ks = max(ks, n0 - b_lower_off);
  if (a_upper_off >= 0) ks = max(ks, m0 - a_upper_off);
  if (a_upper_off != -1) ks &= ~63;
  const int kt0 = ks / GK;
  if ((b_lower_off >= 0 || a_upper_off >= 0) && accumulate && kt0 >= ktiles) return;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + sizeof(GemmSmem<TM, TN, GK, NS>));
  if constexpr (TMA) {
    if (tid == 0) {
#pragma unroll
      for (int st = 0; st < NS; ++st) mbar_init(&bars[st], 1);
      mbar_fence_init();
    }
    __syncthreads();
  }
  auto load = [&](int buf, int kt) {
    const int k0 = kt * GK;
    if constexpr (TMA) {
      if (tid == 0) {
        constexpr unsigned bytes = (unsigned)sizeof(S.A[0]) + (unsigned)sizeof(S.B[0]);
        mbar_expect_tx(&bars[buf], bytes);
        tma_load_3d(&S.A[buf][0][0], &tmA, 2 * k0, m0, b, &bars[buf]);
        tma_load_3d(&S.B[buf][0][0], &tmB, 2 * n0, k0, b, &bars[buf]);
      }
      return;
    }
#pragma unroll
    for (int u = 0; u < (TM * GK) / NT; ++u) {
      int e = tid + u * NT;
      int r = e / GK, c = e % GK;
      bool v = (m0 + r < m) && (k0 + c < k);
      const double2* src = v ? Ab + (int64_t)(m0 + r) * A.ld + k0 + c : Ab;
      cp_async16_zfill(&S.A[buf][r][c], src, v);
    }
#pragma unroll
    for (int u = 0; u < (GK * TN) / NT; ++u) {
      int e = tid + u * NT;
      int r = e / TN, c = e % TN;
      bool v = (k0 + r < k) && (n0 + c < n);
      const double2* src = v ? Bb + (int64_t)(k0 + r) * B.ld + n0 + c : Bb;
      cp_async16_zfill(&S.B[buf][r][c], src, v);
    }
  };
#pragma unroll
  for (int st = 0; st < NS - 1; ++st) {
    if (kt0 + st < ktiles) load(st, kt0 + st);
    if constexpr (!TMA) cp_async_commit();
  }
  for (int kt = kt0; kt < ktiles; ++kt) {
    const int buf = (kt - kt0) % NS;
    if (kt + NS - 1 < ktiles) load((kt - kt0 + NS - 1) % NS, kt + NS - 1);
    if constexpr (TMA) {
      mbar_wait(&bars[buf], (unsigned)((kt - kt0) / NS) & 1u);
    } else {
      cp_async_commit();
      cp_async_wait<NS - 1>();
      __syncthreads();
    }
#pragma unroll
    for (int kk = 0; kk < GK; kk += 4) {
      double ar[FM], ai[FM], br[FN], bi[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i) {
        double2 x = S.A[buf][wm * (TM / 2) + i * 8 + g][kk + t];
        ar[i] = x.x;  // alpha is applied once, in the epilogue
        ai[i] = x.y;
      }
#pragma unroll
      for (int j = 0; j < FN; ++j) {
        double2 y = S.B[buf][kk + t][wn * FN * 8 + j * 8 + g];
        br[j] = y.x;
        bi[j] = y.y;
      }
      if (M3) {
        double as[FM], bs[FN];
#pragma unroll
        for (int i = 0; i < FM; ++i) as[i] = ar[i] + ai[i];
#pragma unroll
        for (int j = 0; j < FN; ++j) bs[j] = br[j] + bi[j];
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j) {
            dmma884(cr[i][j][0], cr[i][j][1], ar[i], br[j]);
            dmma884(ci[i][j][0], ci[i][j][1], ai[i], bi[j]);
            dmma884(t3[M3 ? i : 0][M3 ? j : 0][0], t3[M3 ? i : 0][M3 ? j : 0][1], as[i], bs[j]);
          }
      } else {
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j) zmma884(cr[i][j], ci[i][j], ar[i], ai[i], br[j], bi[j]);
      }
    }
    __syncthreads();
  }
  if (M3) {
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double t1 = cr[i][j][h], t2 = ci[i][j][h];
          cr[i][j][h] = t1 - t2;
          ci[i][j][h] = t3[M3 ? i : 0][M3 ? j : 0][h] - t1 - t2;
        }
  }
  // epilogue C = C + alpha * acc: every C load of the thread is issued before the first add
  // (one round trip to L2/HBM per thread instead of one per element)
  // (two fragment rows per round keeps the loaded values within the register budget)
  double2* Cb = C.p + b * C.stride;
  constexpr int EH = FM >= 2 ? 2 : 1;
#pragma unroll
  for (int i0 = 0; i0 < FM; i0 += EH) {
    double2 cv[EH][FN][2];
#pragma unroll
    for (int u = 0; u < EH; ++u) {
      const int row = m0 + wm * (TM / 2) + (i0 + u) * 8 + g;
#pragma unroll
      for (int j = 0; j < FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = n0 + wn * FN * 8 + j * 8 + 2 * t + h;
          cv[u][j][h] = (accumulate && row < m && col < n) ? __ldcg(Cb + (int64_t)row * C.ld + col)
                                                           : make_double2(0.0, 0.0);
        }
    }
#pragma unroll
    for (int u = 0; u < EH; ++u) {
      const int i = i0 + u;
      const int row = m0 + wm * (TM / 2) + i * 8 + g;
      if (row >= m) continue;
#pragma unroll
      for (int j = 0; j < FN; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = n0 + wn * FN * 8 + j * 8 + 2 * t + h;
          if (col < n) {
            double2 v = cv[u][j][h];
            v.x = fma(alpha, cr[i][j][h], v.x);
            v.y = fma(alpha, ci[i][j][h], v.y);
            Cb[(int64_t)row * C.ld + col] = v;
          }
        }
      }
    }
  }
}

// PFX_ZGEMM_CPASYNC=1 stages the tiles with cp.async (the round-1 loader) for A/B checks.
static bool zgemm_use_tma() {
  static const bool on = getenv("PFX_ZGEMM_CPASYNC") == nullptr;
  return on;
}

template <int TM, int TN, int NW, bool M3, int KS = 16>
static int zgemm_launch(cudaStream_t s, int batch, int m, int n, int k, double alpha, ZMat A, ZMat B, ZMat C,
                        bool accumulate, int b_lower_off, const ZCombine* ride, int a_upper_off) {
  constexpr int NS = gemm_stages<TM, NW>();
  CUtensorMap tmA, tmB;
  memset(&tmA, 0, sizeof(tmA));
  memset(&tmB, 0, sizeof(tmB));
  const bool tma = zgemm_use_tma() && zmat_tensor_map(&tmA, A, m, k, batch, TM, KS + 4) &&
                   zmat_tensor_map(&tmB, B, k, n, batch, KS, TN + 2);
  auto kfn = tma ? zgemm_kernel<TM, TN, NW, M3, KS, true> : zgemm_kernel<TM, TN, NW, M3, KS, false>;
  const int smem = (int)sizeof(GemmSmem<TM, TN, KS, NS>) + (tma ? NS * 8 : 0);
  if (int rc = raise_smem_limit(reinterpret_cast<const void*>(kfn), smem)) return rc;
  ZCombine rd;
  if (ride) rd = *ride;
  // the combine's shared-memory staging (64 x 65) must fit the GEMM's allocation
  static_assert(sizeof(GemmSmem<TM, TN, KS, gemm_stages<TM, NW>()>) >= 64 * 65 * sizeof(double2) || TM < 64,
                "combine staging fits");
  constexpr bool carries = TM == 64 && NW == 4;
  dim3 grid((unsigned)ceil_div(n, TN), (unsigned)ceil_div(m, TM), (unsigned)batch + (ride && carries ? 1 : 0));
  if (ride && !carries) {  // other layouts: the combine goes on its own launch
    if (int rc = zcombine(s, rd)) return rc;
    rd = ZCombine();
  }
  // algorithmic flops: 8 per complex multiply-add actually required (b_lower: the products
  // with the zero triangle of B are not counted)
  double fl = 8.0 * (double)m * n * k * batch;
  if (b_lower_off >= 0) {
    double nz = 0.0;  // nonzero rows of B summed over its columns
    for (int c = 0; c < n; ++c) nz += (double)std::max(0, k - std::max(0, c - b_lower_off));
    fl = 8.0 * (double)m * batch * nz;
  }
  if (a_upper_off >= 0) {
    double nz = 0.0;  // nonzero columns of A summed over its rows
    for (int r = 0; r < m; ++r) nz += (double)std::max(0, k - std::max(0, r - a_upper_off));
    fl = 8.0 * (double)n * batch * nz;
  }
  PFX_LAUNCH_F("zgemm", s, fl,
               (kfn<<<grid, NW * 32, smem, s>>>(m, n, k, alpha, A, B, C, accumulate ? 1 : 0, b_lower_off, rd,
                                                 tmA, tmB, a_upper_off)));
  PFX_CUDA_TRY(cudaGetLastError());
  return PFX_OK;
}

static thread_local bool g_zgemm_short_k = false;

ZgemmShortK::ZgemmShortK(bool on) : prev_(g_zgemm_short_k) { g_zgemm_short_k = on; }
ZgemmShortK::~ZgemmShortK() { g_zgemm_short_k = prev_; }

int zgemm(cudaStream_t s, int batch, int m, int n, int k, double alpha, ZMat A, ZMat B, ZMat C, bool accumulate,
          int b_lower_off, const ZCombine* ride, int a_upper_off) {
  if (m <= 0 || n <= 0 || k <= 0 || batch <= 0) return ride ? zcombine(s, *ride) : PFX_OK;
  const int sms = device_sms();
  static const bool m3 = getenv("PFX_ZGEMM_4M") == nullptr;  // 3M by default; 4M for A/B checks
  const int64_t tiles64 = ceil_div(m, 64) * ceil_div(n, 64) * (int64_t)batch;
  static const bool ks32 = getenv("PFX_ZGEMM_KS16") == nullptr;
  // Short-K preference (ZgemmShortK, set by the banded path; PFX_ZGEMM_SHORTK32=1/0 forces it
  // on / off everywhere): every K <= 64 launch on the 32 x 32 tiles -- four CTAs per SM instead
  // of two 64 x 64 ones, more prologue / epilogue overlap per unit of DMMA work.  C5 258.5 ->
  // 255.1 ms; on C4's narrow K = 64 launches it costs 0.3 ms, so the dense path leaves it off.
  static const int shortk_env = [] {
    const char* e = getenv("PFX_ZGEMM_SHORTK32");
    return e ? (atoi(e) != 0 ? 1 : 0) : -1;
  }();
  const bool shortk32 = shortk_env >= 0 ? shortk_env == 1 : g_zgemm_short_k;
  if (tiles64 < 2 * sms || (shortk32 && k <= 64)) {
    if (k <= 64 && ks32)  // short K: two 32-deep stages instead of four 16-deep ones
      return m3 ? zgemm_launch<32, 32, 4, true, 32>(s, batch, m, n, k, alpha, A, B, C, accumulate, b_lower_off, ride, a_upper_off)
                : zgemm_launch<32, 32, 4, false, 32>(s, batch, m, n, k, alpha, A, B, C, accumulate, b_lower_off, ride, a_upper_off);
    return m3 ? zgemm_launch<32, 32, 4, true>(s, batch, m, n, k, alpha, A, B, C, accumulate, b_lower_off, ride, a_upper_off)
              : zgemm_launch<32, 32, 4, false>(s, batch, m, n, k, alpha, A, B, C, accumulate, b_lower_off, ride, a_upper_off);
  }
  // 64x64 tiles on 4 warps of 32x32 (248 registers, two CTAs per SM): per 4-deep K step a
  // warp issues 8 fragment loads and 8 operand sums for 48 DMMAs (3M), where the 8-warp
  // 32x16 layout issued 6 + 6 for 24; 5-8% faster on every C4 shape (tools/zgemm_probe.cu).
  // PFX_ZGEMM_W8=1 keeps the 8-warp layout for A/B checks.
  static const bool w8 = getenv("PFX_ZGEMM_W8") != nullptr;
  if (m3 && !w8) return zgemm_launch<64, 64, 4, true>(s, batch, m, n, k, alpha, A, B, C, accumulate, b_lower_off, ride, a_upper_off);
  return m3 ? zgemm_launch<64, 64, 8, true>(s, batch, m, n, k, alpha, A, B, C, accumulate, b_lower_off, ride, a_upper_off)
            : zgemm_launch<64, 64, 8, false>(s, batch, m, n, k, alpha, A, B, C, accumulate, b_lower_off, ride, a_upper_off);
}

// ---------------------------------------------------------------------------
// Unblocked LU of an m x nb panel, one CTA per batch element, panel in global memory
// (L2-resident).  With ipiv: partial pivoting inside the panel (max |re|+|im|, first
// index on ties).  nb <= 64.
constexpr int P_THREADS = 256;

__global__ void __launch_bounds__(P_THREADS) zgetf2_kernel(int m, int nb, ZMat P, int* ipiv, int* sing) {
  __shared__ double sv[P_THREADS / 32];
  __shared__ int si[P_THREADS / 32];
  __shared__ double2 prow[64];
  __shared__ int s_piv;
  const int b = blockIdx.x;
  double2* A = P.p + b * P.stride;
  const int64_t lda = P.ld;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int j = 0; j < nb && j < m; ++j) {
    int piv = j;
    if (ipiv) {
      double bv = -1.0;
      int bi = 0x7fffffff;
      for (int r = j + tid; r < m; r += P_THREADS) {
        double2 x = A[(int64_t)r * lda + j];
        double v = fabs(x.x) + fabs(x.y);
        if (v > bv) {
          bv = v;
          bi = r;
        }
      }
      for (int off = 16; off > 0; off >>= 1) {
        double ov = __shfl_down_sync(0xffffffffu, bv, off);
        int oi = __shfl_down_sync(0xffffffffu, bi, off);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (lane == 0) {
        sv[warp] = bv;
        si[warp] = bi;
      }
      __syncthreads();
      if (tid == 0) {
        double best = sv[0];
        int bidx = si[0];
        for (int w = 1; w < P_THREADS / 32; ++w)
          if (sv[w] > best || (sv[w] == best && si[w] < bidx)) {
            best = sv[w];
            bidx = si[w];
          }
        s_piv = bidx;
        ipiv[b * nb + j] = bidx;
      }
      __syncthreads();
      piv = s_piv;
      if (piv != j)
        for (int c = tid; c < nb; c += P_THREADS) {
          double2 x = A[(int64_t)j * lda + c];
          A[(int64_t)j * lda + c] = A[(int64_t)piv * lda + c];
          A[(int64_t)piv * lda + c] = x;
        }
      __syncthreads();
    }
    for (int c = tid; c < nb; c += P_THREADS) prow[c] = A[(int64_t)j * lda + c];
    __syncthreads();
    cplx pv = ld(&prow[j]);
    if (pv.re == 0.0 && pv.im == 0.0) {
      if (tid == 0) atomicOr(sing, ST_SINGULAR);
      continue;
    }
    cplx rp = crcp(pv);
    // rows below: scale column j, rank-1 update of columns j+1..nb-1
    const int cols = nb - j - 1;
    for (int r = j + 1 + tid; r < m; r += P_THREADS) {
      double2* row = A + (int64_t)r * lda;
      cplx l = cmul(ld(&row[j]), rp);
      st(&row[j], l);
      for (int c = 0; c < cols; ++c) st(&row[j + 1 + c], cfms(ld(&row[j + 1 + c]), l, ld(&prow[j + 1 + c])));
    }
    __syncthreads();
  }
}

// Shared-memory variant for panels that fit on chip (m*nb <= 4096 complex, e.g. the
// 64x64 diagonal blocks of the no-pivot LUs): one CTA per batch element, the panel
// is loaded once, factored with one __syncthreads per column, written back once.
constexpr int PS_MAXEL = 64 * 65;
__global__ void __launch_bounds__(P_THREADS) zgetf2_smem_kernel(int m, int nb, ZMat P, int* ipiv, int* sing) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* Ps = reinterpret_cast<double2*>(smem_raw);
  __shared__ double sv[P_THREADS / 32];
  __shared__ int si[P_THREADS / 32];
  __shared__ int s_piv;
  const int b = blockIdx.x;
  double2* A = P.p + b * P.stride;
  const int64_t lda = P.ld;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ps = nb + 1;
  for (int e = tid; e < m * nb; e += P_THREADS) {
    int r = e / nb, c = e - r * nb;
    Ps[r * ps + c] = A[(int64_t)r * lda + c];
  }
  __syncthreads();
  for (int j = 0; j < nb && j < m; ++j) {
    if (ipiv) {
      double bv = -1.0;
      int bi = 0x7fffffff;
      for (int r = j + tid; r < m; r += P_THREADS) {
        double2 x = Ps[r * ps + j];
        double v = fabs(x.x) + fabs(x.y);
        if (v > bv) {
          bv = v;
          bi = r;
        }
      }
      for (int off = 16; off > 0; off >>= 1) {
        double ov = __shfl_down_sync(0xffffffffu, bv, off);
        int oi = __shfl_down_sync(0xffffffffu, bi, off);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (lane == 0) {
        sv[warp] = bv;
        si[warp] = bi;
      }
      __syncthreads();
      if (tid == 0) {
        double best = sv[0];
        int bidx = si[0];
        for (int w = 1; w < P_THREADS / 32; ++w)
          if (sv[w] > best || (sv[w] == best && si[w] < bidx)) {
            best = sv[w];
            bidx = si[w];
          }
        s_piv = bidx;
        ipiv[b * nb + j] = bidx;
      }
      __syncthreads();
      const int piv = s_piv;
      if (piv != j)
        for (int c = tid; c < nb; c += P_THREADS) {
          double2 x = Ps[j * ps + c];
          Ps[j * ps + c] = Ps[piv * ps + c];
          Ps[piv * ps + c] = x;
        }
      __syncthreads();
    }
    const cplx pv = ld(&Ps[j * ps + j]);
    if (pv.re == 0.0 && pv.im == 0.0) {
      if (tid == 0) atomicOr(sing, ST_SINGULAR);
      __syncthreads();
      continue;
    }
    const cplx rp = crcp_fast(pv);
    // warp w owns rows j+1+w, j+1+w+8, ...: each lane scales its row's multiplier once and
    // updates columns j+1.. of that row; rows are independent, one barrier per column
    const int cols = nb - j - 1;
    for (int r = j + 1 + warp; r < m; r += P_THREADS / 32) {
      const cplx l = cmul(ld(&Ps[r * ps + j]), rp);
      for (int c = lane; c < cols; c += 32)
        st(&Ps[r * ps + j + 1 + c], cfms(ld(&Ps[r * ps + j + 1 + c]), l, ld(&Ps[j * ps + j + 1 + c])));
      __syncwarp();
      if (lane == 0) st(&Ps[r * ps + j], l);
    }
    __syncthreads();
  }
  for (int e = tid; e < m * nb; e += P_THREADS) {
    int r = e / nb, c = e - r * nb;
    A[(int64_t)r * lda + c] = Ps[r * ps + c];
  }
}

int zgetf2_panel(cudaStream_t s, int batch, int m, int nb, ZMat P, int* ipiv, int* sing) {
  if (nb > 64) return fail(PFX_BADARG, "zgetf2_panel: nb > 64");
  if ((int64_t)m * (nb + 1) <= PS_MAXEL) {
    const int smem = (int)((int64_t)m * (nb + 1) * sizeof(double2));
    if (int rc = raise_smem_limit(reinterpret_cast<const void*>(zgetf2_smem_kernel), PS_MAXEL * 16 + 64)) return rc;
    PFX_LAUNCH_F("zgetf2", s, 8.0 / 3.0 * nb * nb * (double)m * batch,
                 zgetf2_smem_kernel<<<batch, P_THREADS, smem, s>>>(m, nb, P, ipiv, sing));
    PFX_CUDA_TRY(cudaGetLastError());
    return PFX_OK;
  }
  PFX_LAUNCH("zgetf2", s, zgetf2_kernel<<<batch, P_THREADS, 0, s>>>(m, nb, P, ipiv, sing));
  PFX_CUDA_TRY(cudaGetLastError());
  return PFX_OK;
}

// ---------------------------------------------------------------------------
// Row interchanges: for each column c in [c0, c1) (one thread per column), apply
// swaps j = 0..nb-1 (dir = +1) or nb-1..0 (dir = -1) of rows r0+j <-> r0+ipiv[j].
__global__ void zlaswp_kernel(int nb, ZMat A, int64_t r0, int64_t c0, int64_t c1, const int* ipiv, int dir) {
  const int b = blockIdx.y;
  const int64_t c = c0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= c1) return;
  double2* Ab = A.p + b * A.stride;
  const int* ip = ipiv + b * nb;
  for (int jj = 0; jj < nb; ++jj) {
    int j = dir > 0 ? jj : nb - 1 - jj;
    int p = ip[j];
    if (p != j) {
      double2* x = Ab + (r0 + j) * A.ld + c;
      double2* y = Ab + (r0 + p) * A.ld + c;
      double2 tmp = *x;
      *x = *y;
      *y = tmp;
    }
  }
}

int zlaswp(cudaStream_t s, int batch, int nb, ZMat A, int64_t r0, int64_t c0, int64_t c1, const int* ipiv, int dir) {
  if (c1 <= c0) return PFX_OK;
  dim3 grid((unsigned)ceil_div(c1 - c0, 128), (unsigned)batch);
  PFX_LAUNCH("zlaswp", s, zlaswp_kernel<<<grid, 128, 0, s>>>(nb, A, r0, c0, c1, ipiv, dir));
  PFX_CUDA_TRY(cudaGetLastError());
  return PFX_OK;
}

// ---------------------------------------------------------------------------
// Left triangular solves on an nb x n block: each CTA owns a strip of 32 columns
// (one lane per column), the triangle in shared memory.  MODE 0: unit lower
// (forward), MODE 1: upper non-unit (backward).
constexpr int T_COLS = 32;
constexpr int T_THREADS = 256;  // 8 warps: warp w handles rows w, w+8, ... of the update

template <int MODE>
__global__ void __launch_bounds__(T_THREADS) ztrsm_left_kernel(int nb, int n, ZMat T, ZMat B) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* Ts = reinterpret_cast<double2*>(smem_raw);  // nb x (nb+1)
  double2* Bs = Ts + nb * (nb + 1);                    // nb x (T_COLS+1)
  const int b = blockIdx.y;
  const int c0 = blockIdx.x * T_COLS;
  const int tid = threadIdx.x;
  const double2* Tb = T.p + b * T.stride;
  double2* Bb = B.p + b * B.stride;
  for (int e = tid; e < nb * nb; e += T_THREADS) {
    int r = e / nb, c = e % nb;
    Ts[r * (nb + 1) + c] = Tb[(int64_t)r * T.ld + c];
  }
  for (int e = tid; e < nb * T_COLS; e += T_THREADS) {
    int r = e / T_COLS, c = e % T_COLS;
    Bs[r * (T_COLS + 1) + c] = (c0 + c < n) ? Bb[(int64_t)r * B.ld + c0 + c] : make_double2(0, 0);
  }
  __syncthreads();
  // warp w owns columns 4w..4w+3 of the strip; lane = (column-in-group, row slice):
  // lanes 8c..8c+7 share column 4w+c and split the rows 8 ways; only __syncwarp inside
  const int warp = tid >> 5, lane = tid & 31;
  const int col = warp * 4 + (lane >> 3), rs = lane & 7;
  if (MODE == 0) {
    for (int kk = 0; kk < nb; ++kk) {
      const cplx x = ld(&Bs[kk * (T_COLS + 1) + col]);
      for (int r = kk + 1 + rs; r < nb; r += 8)
        st(&Bs[r * (T_COLS + 1) + col], cfms(ld(&Bs[r * (T_COLS + 1) + col]), ld(&Ts[r * (nb + 1) + kk]), x));
      __syncwarp();
    }
  } else {
    for (int kk = nb - 1; kk >= 0; --kk) {
      const cplx x = cmul(ld(&Bs[kk * (T_COLS + 1) + col]), crcp_fast(ld(&Ts[kk * (nb + 1) + kk])));
      __syncwarp();
      if (rs == 0) st(&Bs[kk * (T_COLS + 1) + col], x);
      for (int r = rs; r < kk; r += 8)
        st(&Bs[r * (T_COLS + 1) + col], cfms(ld(&Bs[r * (T_COLS + 1) + col]), ld(&Ts[r * (nb + 1) + kk]), x));
      __syncwarp();
    }
  }
  __syncthreads();
  for (int e = tid; e < nb * T_COLS; e += T_THREADS) {
    int r = e / T_COLS, c = e % T_COLS;
    if (c0 + c < n) Bb[(int64_t)r * B.ld + c0 + c] = Bs[r * (T_COLS + 1) + c];
  }
}

static int trsm_smem(int nb) { return (int)((size_t)nb * (nb + 1) + (size_t)nb * (T_COLS + 1)) * (int)sizeof(double2); }
static const int kTrsmSmemMax = (64 * 65 + 64 * 33) * (int)sizeof(double2);
static int trsm_attrs() {
  if (int rc = raise_smem_limit(reinterpret_cast<const void*>(ztrsm_left_kernel<0>), kTrsmSmemMax)) return rc;
  return raise_smem_limit(reinterpret_cast<const void*>(ztrsm_left_kernel<1>), kTrsmSmemMax);
}

int ztrsm_llnu(cudaStream_t s, int batch, int nb, int n, ZMat Lm, ZMat B) {
  if (n <= 0) return PFX_OK;
  const int smem = trsm_smem(nb);
  if (int rc = trsm_attrs()) return rc;
  dim3 grid((unsigned)ceil_div(n, T_COLS), (unsigned)batch);
  PFX_LAUNCH("ztrsm", s, ztrsm_left_kernel<0><<<grid, T_THREADS, smem, s>>>(nb, n, Lm, B));
  PFX_CUDA_TRY(cudaGetLastError());
  return PFX_OK;
}

int ztrsm_lunn(cudaStream_t s, int batch, int nb, int n, ZMat Um, ZMat B) {
  if (n <= 0) return PFX_OK;
  const int smem = trsm_smem(nb);
  if (int rc = trsm_attrs()) return rc;
  dim3 grid((unsigned)ceil_div(n, T_COLS), (unsigned)batch);
  PFX_LAUNCH("ztrsm", s, ztrsm_left_kernel<1><<<grid, T_THREADS, smem, s>>>(nb, n, Um, B));
  PFX_CUDA_TRY(cudaGetLastError());
  return PFX_OK;
}

// ---------------------------------------------------------------------------
// Diagonal-block LU (nb <= 64, no pivoting), one CTA (256 threads) per batch member,
// factors written back in place.
constexpr int DI_MAX = 64;
constexpr int DI_S = DI_MAX + 1;

// Two columns per barrier: rows j and j+1 are published together (both final with respect to
// the columns before j), every thread forms the 2 x 2 pivot block's factors itself
// (l10 = a_{j+1,j} / u_jj, u'_11 = a_{j+1,j+1} - l10 u_{j,j+1}), and the rows below apply the
// rank-2 update a_rc -= m1 u_jc + l2 a_{j+1,c} with l1 = a_rj / u_jj, l2 = (a_{r,j+1} - l1 u_{j,j+1}) / u'_11,
// m1 = l1 - l2 l10 (the same factors as two rank-1 steps; rounding differs).  Half the
// barriers and pivot reciprocals on the critical chain of the diagonal LU.
template <int NL>
__device__ __forceinline__ void lu_diag_phase2(int q0, cplx (&a)[16], int nb, ZMat D, int b, int row, int cg,
                                               int lane, unsigned base, int* sing) {
  constexpr unsigned ROW = 2 * DI_MAX * 16;  // bytes per published row (64 past the block, zero)
  constexpr unsigned BUF = 2 * ROW;          // rows j and j+1
#pragma unroll 1
  for (int q = q0; q < q0 + 4; ++q) {
    const unsigned qb = base + (unsigned)(cg + 4 * q) * 16u;  // &row0[cg + 4q]
#pragma unroll
    for (int jj = 0; jj < 4; jj += 2) {
      const int j = 4 * q + jj;
      const unsigned p0 = qb + ((jj >> 1) & 1) * BUF, p1 = p0 + ROW;  // this lane's column in rows j / j+1
      const unsigned r0b = base + ((jj >> 1) & 1) * BUF, r1b = r0b + ROW;
      if (row == j || row == j + 1) {
        // entries left of j in a[0] are finished multipliers: publish only c >= j
        const unsigned pb = row == j ? p0 : p1;
        if (cg >= jj) sts2(pb, a[0]);
#pragma unroll
        for (int i = 1; i < NL; ++i) sts2(pb + 64u * i, a[i]);
      }
      __syncthreads();
      const cplx u00 = lds2(r0b + (unsigned)j * 16u), u01 = lds2(r0b + (unsigned)(j + 1) * 16u);
      const cplx a10 = lds2(r1b + (unsigned)j * 16u), a11 = lds2(r1b + (unsigned)(j + 1) * 16u);
      const cplx r00 = crcp_fast(u00);
      const cplx l10 = cmul(a10, r00);
      const cplx u11 = cfms(a11, l10, u01);
      if (row == j && cg == jj && u00.re == 0.0 && u00.im == 0.0) atomicOr(sing, ST_SINGULAR);
      if (row == j + 1 && cg == jj + 1 && u11.re == 0.0 && u11.im == 0.0) atomicOr(sing, ST_SINGULAR);
      // partial-pivoting check (izamax, first index on ties): column j's updated entries
      // below the diagonal (a10 for row j+1, a_rj below) against u00; column j+1's against u11
      const double pa0 = cabs1(u00), pa1 = cabs1(u11);
      if (row == j + 1 && cg == 0 && cabs1(a10) > pa0) atomicOr(sing, ST_PIVOT);
      // a_rj, a_{r,j+1} from the row's lanes holding columns j, j+1 (whole warp: no divergence)
      const int src = (lane & ~3) | jj;
      cplx aj, aj1;
      aj.re = __shfl_sync(0xffffffffu, a[0].re, src);
      aj.im = __shfl_sync(0xffffffffu, a[0].im, src);
      aj1.re = __shfl_sync(0xffffffffu, a[0].re, src + 1);
      aj1.im = __shfl_sync(0xffffffffu, a[0].im, src + 1);
      if (row > j + 1) {
        const cplx l1 = cmul(aj, r00);
        const cplx a1 = cfms(aj1, l1, u01);
        if (cg == 0 && row < nb && (cabs1(aj) > pa0 || cabs1(a1) > pa1)) atomicOr(sing, ST_PIVOT);
        const cplx l2 = cmul(a1, crcp_fast(u11));
        const cplx m1 = cfms(l1, l2, l10);
        const cplx x0 = cfms(cfms(a[0], m1, lds2(p0)), l2, lds2(p1));
#pragma unroll
        for (int i = 1; i < NL; ++i) a[i] = cfms(cfms(a[i], m1, lds2(p0 + 64u * i)), l2, lds2(p1 + 64u * i));
        a[0] = cg == jj ? l1 : (cg == jj + 1 ? l2 : (cg > jj + 1 ? x0 : a[0]));
      } else if (row == j + 1) {
        // row j+1: its multiplier l10 in column j, the eliminated U row from column j+1 on
        const cplx x0 = cfms(a[0], l10, lds2(p0));
#pragma unroll
        for (int i = 1; i < NL; ++i) a[i] = cfms(a[i], l10, lds2(p0 + 64u * i));
        a[0] = cg == jj ? l10 : (cg > jj ? x0 : a[0]);
      }
    }
    const int c = cg + 4 * q;
    if (row < nb && c < nb) *D.at(b, row, c) = make_double2(a[0].re, a[0].im);
#pragma unroll
    for (int i = 0; i < NL - 1; ++i) a[i] = a[i + 1];
    a[NL - 1] = mk(0, 0);
  }
}

__global__ void __launch_bounds__(256) zgetrf_diag2_kernel(int nb, ZMat D, int* sing) {
  // two double-buffered pairs of pivot rows, each running 64 entries past the block, kept zero
  __shared__ __align__(16) double2 prow[2][2][2 * DI_MAX];
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31;
  const int row = tid >> 2, cg = tid & 3;
  (&prow[0][0][0])[tid] = make_double2(0, 0);
  (&prow[0][0][0])[tid + 256] = make_double2(0, 0);
  const unsigned base = (unsigned)__cvta_generic_to_shared(&prow[0][0][0]);
  cplx a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int c = cg + 4 * i;
    if (row < nb && c < nb) a[i] = ld(D.at(b, row, c));
    else a[i] = mk(row == c ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  lu_diag_phase2<16>(0, a, nb, D, b, row, cg, lane, base, sing);
  lu_diag_phase2<12>(4, a, nb, D, b, row, cg, lane, base, sing);
  lu_diag_phase2<8>(8, a, nb, D, b, row, cg, lane, base, sing);
  lu_diag_phase2<4>(12, a, nb, D, b, row, cg, lane, base, sing);
}

// Register-resident: thread (row = tid / 4, phase = tid % 4) holds A[row][phase + 4(q + i)],
// i < 16 - q, where q is the current 4-column block: after every 4 columns the finished
// register a[0] is stored and the window rotates, so every register index stays static
// while the code stays a small loop (a fully unrolled 64-column body overflows the
// instruction cache).  Step j: row j publishes itself to shared memory (double-buffered:
// one barrier per column), every lower row takes its multiplier's numerator from the
// owning lane by shuffle and updates its entries right of j.  nb < 64 pads with I.
// One phase of four 4-column blocks with NL live registers (the window holds columns
// phase + 4 (q + i), i < NL; NL >= 16 - q for every q of the phase, the excess are zeros).
template <int NL>
__device__ __forceinline__ void lu_diag_phase(int q0, cplx (&a)[16], int nb, ZMat D, int b, int row, int cg,
                                              int lane, unsigned base, int* sing) {
  constexpr unsigned BUF = 2 * DI_MAX * 16;  // bytes per pivot-row buffer
#pragma unroll 1
  for (int q = q0; q < q0 + 4; ++q) {
    const unsigned qb = base + (unsigned)(cg + 4 * q) * 16u;  // &prow[0][cg + 4q]
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int j = 4 * q + jj;
      const unsigned pb = qb + (jj & 1) * BUF;
      if (row == j) {
        // entries left of j in the first register are stale multipliers: publish only c >= j
        if (cg >= jj) sts2(pb, a[0]);
#pragma unroll
        for (int i = 1; i < NL; ++i) sts2(pb + 64u * i, a[i]);
        if (cg == jj && a[0].re == 0.0 && a[0].im == 0.0) atomicOr(sing, ST_SINGULAR);
      }
      __syncthreads();
      const int src = (lane & ~3) | jj;
      cplx aj;
      aj.re = __shfl_sync(0xffffffffu, a[0].re, src);
      aj.im = __shfl_sync(0xffffffffu, a[0].im, src);
      if (row > j) {
        const cplx pv = lds2(base + (jj & 1) * BUF + (unsigned)j * 16u);
        if (cg == 0 && row < nb && cabs1(aj) > cabs1(pv)) atomicOr(sing, ST_PIVOT);  // partial-pivoting check
        const cplx l = cmul(aj, crcp_fast(pv));
        const cplx a0 = cfms(a[0], l, lds2(pb));
#pragma unroll
        for (int i = 1; i < NL; ++i) a[i] = cfms(a[i], l, lds2(pb + 64u * i));
        a[0] = cg == jj ? l : (cg > jj ? a0 : a[0]);
      }
    }
    const int c = cg + 4 * q;
    if (row < nb && c < nb) *D.at(b, row, c) = make_double2(a[0].re, a[0].im);
#pragma unroll
    for (int i = 0; i < NL - 1; ++i) a[i] = a[i + 1];
    a[NL - 1] = mk(0, 0);
  }
}

// Register-resident: thread (row = tid / 4, phase = tid % 4) holds A[row][phase + 4(q + i)]
// where q is the current 4-column block: after every 4 columns the finished register a[0]
// is stored and the window rotates, so register indices stay static.  The column loop runs
// in four phases whose live width (16, 12, 8, 4 registers) tracks the shrinking trailing
// matrix, so dead registers are not updated.  Step j: row j publishes itself to shared
// memory (double-buffered: one barrier per column), every lower row takes its multiplier's
// numerator from the owning lane by shuffle and updates its entries right of j.
// nb < 64 pads with the identity.
__global__ void __launch_bounds__(256) zgetrf_diag_kernel(int nb, ZMat D, int* sing) {
  // the pivot row buffer runs 64 entries past the block, kept zero: updates of registers
  // past the live window read those zeros
  __shared__ __align__(16) double2 prow[2][2 * DI_MAX];
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31;
  const int row = tid >> 2, cg = tid & 3;
  prow[tid >> 7][tid & 127] = make_double2(0, 0);
  const unsigned base = (unsigned)__cvta_generic_to_shared(&prow[0][0]);
  cplx a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int c = cg + 4 * i;
    if (row < nb && c < nb) a[i] = ld(D.at(b, row, c));
    else a[i] = mk(row == c ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  lu_diag_phase<16>(0, a, nb, D, b, row, cg, lane, base, sing);
  lu_diag_phase<12>(4, a, nb, D, b, row, cg, lane, base, sing);
  lu_diag_phase<8>(8, a, nb, D, b, row, cg, lane, base, sing);
  lu_diag_phase<4>(12, a, nb, D, b, row, cg, lane, base, sing);
}

// Triangular inverses of the factored block: grid (nb/8 column groups, 2 triangles, batch);
// warp w of a CTA owns one column of L^{-1} (blockIdx.y = 0) or U^{-1} (= 1), lanes hold
// rows lane and lane + 32, and the substitution broadcasts the finished entry by shuffle.
__global__ void __launch_bounds__(256) ztrtri_diag_kernel(int nb, ZMat D, ZMat Li, ZMat Ui) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* A = reinterpret_cast<double2*>(smem_raw);
  double2* rdiag = A + DI_MAX * DI_S;
  const int b = blockIdx.z;
  const bool upper = blockIdx.y != 0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // the zero / identity padding (rows, columns >= nb) makes every update unconditional
  for (int e = tid; e < DI_MAX * DI_MAX; e += 256) {
    const int r = e >> 6, c = e & 63;
    const bool keep = upper ? c >= r : c < r;
    if (keep && r < nb && c < nb) cp_async16(&A[r * DI_S + c], D.at(b, r, c));
    else A[r * DI_S + c] = make_double2(r == c && r >= nb ? 1.0 : 0.0, 0.0);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  if (upper && tid < DI_MAX) {
    const cplx r = crcp(ld(&A[tid * DI_S + tid]));
    rdiag[tid] = make_double2(r.re, r.im);
  }
  __syncthreads();
  const int c = blockIdx.x * 8 + warp;
  if (c >= nb) return;
  const int r0 = lane, r1 = lane + 32;
  cplx x0 = mk(r0 == c ? 1.0 : 0.0, 0.0), x1 = mk(r1 == c ? 1.0 : 0.0, 0.0);
  if (!upper) {
    // X = L^{-1} e_c (unit diagonal; A holds L strictly below, zeros elsewhere): rows
    // at or above k see L[r][k] = 0, so the update needs no row test
    for (int k = c; k < nb - 1; ++k) {
      const cplx src = k < 32 ? x0 : x1;
      const cplx l0 = ld(&A[r0 * DI_S + k]), l1 = ld(&A[r1 * DI_S + k]);
      cplx xk;
      xk.re = __shfl_sync(0xffffffffu, src.re, k & 31);
      xk.im = __shfl_sync(0xffffffffu, src.im, k & 31);
      x0 = cfms(x0, l0, xk);
      x1 = cfms(x1, l1, xk);
    }
    if (r0 < nb) *Li.at(b, r0, c) = make_double2(x0.re, x0.im);
    if (r1 < nb) *Li.at(b, r1, c) = make_double2(x1.re, x1.im);
  } else {
    // X = U^{-1} e_c: step k finalises row k (scale by 1/U_kk) and eliminates it from the
    // rows above (U[r][k] = 0 for r >= k in A's padded copy except the diagonal)
    for (int k = c; k >= 0; --k) {
      const cplx src = k < 32 ? x0 : x1;
      const cplx rd = ld(&rdiag[k]);
      const cplx u0 = r0 < k ? ld(&A[r0 * DI_S + k]) : mk(0, 0);
      const cplx u1 = r1 < k ? ld(&A[r1 * DI_S + k]) : mk(0, 0);
      cplx xk;
      xk.re = __shfl_sync(0xffffffffu, src.re, k & 31);
      xk.im = __shfl_sync(0xffffffffu, src.im, k & 31);
      xk = cmul(xk, rd);
      x0 = r0 == k ? xk : cfms(x0, u0, xk);
      x1 = r1 == k ? xk : cfms(x1, u1, xk);
    }
    if (r0 < nb) *Ui.at(b, r0, c) = make_double2(x0.re, x0.im);
    if (r1 < nb) *Ui.at(b, r1, c) = make_double2(x1.re, x1.im);
  }
}

int zgetrf_diag(cudaStream_t s, int batch, int nb, ZMat D, int* sing) {
  static const bool getrf2 = getenv("PFX_GETRF1") == nullptr;  // PFX_GETRF1=1: one column per barrier
  if (nb > DI_MAX) return fail(PFX_BADARG, "zgetrf_diag: nb > 64");
  PFX_LAUNCH_F("zgetrf_diag", s, 8.0 / 3.0 * nb * nb * (double)nb * batch,
               (getrf2 ? zgetrf_diag2_kernel<<<batch, 256, 0, s>>>(nb, D, sing)
                       : zgetrf_diag_kernel<<<batch, 256, 0, s>>>(nb, D, sing)));
  PFX_CUDA_TRY(cudaGetLastError());
  return PFX_OK;
}

int ztrtri_diag(cudaStream_t s, int batch, int nb, ZMat D, ZMat Li, ZMat Ui) {
  if (nb > DI_MAX) return fail(PFX_BADARG, "ztrtri_diag: nb > 64");
  const int smem = (DI_MAX * DI_S + DI_MAX) * (int)sizeof(double2);
  if (int rc = raise_smem_limit(reinterpret_cast<const void*>(ztrtri_diag_kernel), smem)) return rc;
  dim3 grid((unsigned)ceil_div(nb, 8), 2, (unsigned)batch);
  PFX_LAUNCH_F("ztrtri_diag", s, 8.0 / 3.0 * nb * nb * (double)nb * batch,
               ztrtri_diag_kernel<<<grid, 256, smem, s>>>(nb, D, Li, Ui));
  PFX_CUDA_TRY(cudaGetLastError());
  return PFX_OK;
}

// In-place product with a small triangular inverse T (nb <= 64): left B(nb x n) = T B, or
// right B(n x nb) = B T.  One CTA per 32-wide strip of B: T and the strip are staged in
// shared memory by cp.async, the product runs on DMMA m8n8k4 with the k range cut to T's
// nonzero triangle, and the strip is written back over itself.
constexpr int TM_T = 64;
constexpr int TM_W = 32;

// Persistent over the strips of one system: grid (CTAs per system, batch); each CTA loads T
// once and walks strips blockIdx.x, blockIdx.x + gridDim.x, ..., the next strip's cp.async
// load in flight while the current one is multiplied (two strip buffers).
template <bool RIGHT>
__global__ void __launch_bounds__(256) ztrmm_kernel(int nb, int n, ZMat T, ZMat B, int upper, ZMat Dg, int* flag) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // row strides (16-byte words) for conflict-free DMMA fragment loads: an A-operand array
  // (read at rows g x columns tt of a quarter-warp) 4 mod 8, a B-operand array (rows tt x
  // columns g) 2 mod 8.  T is the A operand on the left and the B operand on the right.
  constexpr int TSS_ = RIGHT ? TM_T + 2 : TM_T + 4;  // Ts
  constexpr int BSL = TM_W + 2;                      // Bs, left: [k][col] (B operand)
  constexpr int BSR = TM_T + 4;                      // Bs, right: [row][k] (A operand)
  constexpr int BSZ = (TM_T * BSL > TM_W * BSR) ? TM_T * BSL : TM_W * BSR;
  double2* Ts = reinterpret_cast<double2*>(smem_raw);  // 64 x TSS_
  double2* Bs0 = Ts + TM_T * (TM_T + 4);               // left: [k 64][col BSL]; right: [row TM_W][k BSR]
  const int b = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tt = lane & 3;
  const int nstrips = (n + TM_W - 1) / TM_W;
  for (int e = tid; e < TM_T * TM_T; e += 256) {
    const int r = e >> 6, c = e & 63;
    if (r < nb && c < nb) cp_async16(&Ts[r * TSS_ + c], T.at(b, r, c));
    else Ts[r * TSS_ + c] = make_double2(0, 0);
  }
  auto load_strip = [&](int st, double2* Bs) {
    const int t0 = st * TM_W;
    for (int e = tid; e < TM_T * TM_W; e += 256) {
      if (!RIGHT) {  // Bs[k][col] = B[k][t0 + col]
        const int r = e / TM_W, c = e - r * TM_W;
        if (r < nb && t0 + c < n) cp_async16(&Bs[r * BSL + c], B.at(b, r, t0 + c));
        else Bs[r * BSL + c] = make_double2(0, 0);
      } else {  // Bs[row][k] = B[t0 + row][k]
        const int r = e >> 6, c = e & 63;
        if (t0 + r < n && c < nb) cp_async16(&Bs[r * BSR + c], B.at(b, t0 + r, c));
        else Bs[r * BSR + c] = make_double2(0, 0);
      }
    }
  };
  if ((int)blockIdx.x < nstrips) load_strip(blockIdx.x, Bs0);
  cp_async_commit();
  // left: R (64 x 32) = T Bs, warp = 8-row slab, 4 column fragments
  // right: R (32 x 64) = Bs T, warp = (8-row slab wm = warp >> 1, 32-column half wn = warp & 1)
  const int wm = RIGHT ? (warp >> 1) : warp;
  const int wn = RIGHT ? (warp & 1) : 0;
  int klo = 0, khi = TM_T;
  if (!RIGHT) {
    if (upper) klo = wm * 8;          // T upper: T[r][k] = 0 for k < r
    else khi = wm * 8 + 8;            // T lower: T[r][k] = 0 for k > r
  } else {
    if (upper) khi = wn * 32 + 32;    // T upper: T[k][c] = 0 for k > c
    else klo = wn * 32;               // T lower: T[k][c] = 0 for k < c
  }
  int it = 0;
  for (int st = blockIdx.x; st < nstrips; st += gridDim.x, ++it) {
    double2* Bs = Bs0 + (it & 1) * BSZ;
    const int nxt = st + gridDim.x;
    if (nxt < nstrips) load_strip(nxt, Bs0 + ((it + 1) & 1) * BSZ);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const int t0 = st * TM_W;
    // 3M complex product: T1 = sum Xr Yr, T2 = sum Xi Yi, T3 = sum (Xr + Xi)(Yr + Yi)
    double t1[4][2], t2[4][2], t3[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j) t1[j][0] = t1[j][1] = t2[j][0] = t2[j][1] = t3[j][0] = t3[j][1] = 0.0;
    for (int k0 = klo; k0 < khi; k0 += 4) {
      double2 x;
      if (!RIGHT) x = Ts[(wm * 8 + g) * TSS_ + k0 + tt];
      else x = Bs[(wm * 8 + g) * BSR + k0 + tt];
      const double xs = x.x + x.y;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double2 y = RIGHT ? Ts[(k0 + tt) * TSS_ + wn * 32 + j * 8 + g] : Bs[(k0 + tt) * BSL + j * 8 + g];
        dmma884(t1[j][0], t1[j][1], x.x, y.x);
        dmma884(t2[j][0], t2[j][1], x.y, y.y);
        dmma884(t3[j][0], t3[j][1], xs, y.x + y.y);
      }
    }
    const int r = wm * 8 + g;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = wn * 32 + j * 8 + 2 * tt + h;
        const double2 v = make_double2(t1[j][h] - t2[j][h], t3[j][h] - t1[j][h] - t2[j][h]);
        if (!RIGHT) {
          if (r < nb && t0 + c < n) *B.at(b, r, t0 + c) = v;
        } else {
          if (t0 + r < n && c < nb) {
            *B.at(b, t0 + r, c) = v;
            if (flag) {
              // L21 = A21 U11^{-1}: the updated column entry l u_cc of a row below the block
              // must not exceed the pivot u_cc (partial-pivoting check, izamax order)
              const cplx u = ld(Dg.at(b, c, c));
              if (cabs1(cmul(mk(v.x, v.y), u)) > cabs1(u)) atomicOr(flag, ST_PIVOT);
            }
          }
        }
      }
    __syncthreads();  // this strip buffer is refilled two iterations on
  }
}

int ztrmm_inplace(cudaStream_t s, int batch, int nb, int n, ZMat Tinv, ZMat B, bool right, bool upper, ZMat Dg,
                  int* pivot_flag) {
  if (n <= 0) return PFX_OK;
  if (nb > TM_T) return fail(PFX_BADARG, "ztrmm_inplace: nb > 64");
  // T + two strip buffers (64 x 34 left / 32 x 68 right)
  const int smem = (TM_T * (TM_T + 4) + 2 * TM_T * (TM_W + 2)) * (int)sizeof(double2);
  static_assert(TM_T * (TM_W + 2) >= TM_W * (TM_T + 4), "strip buffer size");
  if (int rc = raise_smem_limit(reinterpret_cast<const void*>(ztrmm_kernel<false>), smem)) return rc;
  if (int rc = raise_smem_limit(reinterpret_cast<const void*>(ztrmm_kernel<true>), smem)) return rc;
  // about one CTA per SM in all (two strip buffers + T: 139 KB of shared memory per CTA)
  const int nstrips = (int)ceil_div(n, TM_W);
  // latency-critical small launches (all strips fit about two CTAs per SM) keep one strip per
  // CTA; large ones go persistent, one CTA per SM in all
  const int sms = device_sms();
  const int per_sys = (int64_t)nstrips * batch <= 2 * sms ? nstrips : std::max(1, std::min(nstrips, sms / batch));
  dim3 grid((unsigned)per_sys, (unsigned)batch);
  const double fl = 4.0 * nb * nb * (double)n * batch;  // triangular: half the square product
  if (right)
    PFX_LAUNCH_F("ztrmm", s, fl,
                 ztrmm_kernel<true><<<grid, 256, smem, s>>>(nb, n, Tinv, B, upper ? 1 : 0, Dg, pivot_flag));
  else
    PFX_LAUNCH_F("ztrmm", s, fl,
                 ztrmm_kernel<false><<<grid, 256, smem, s>>>(nb, n, Tinv, B, upper ? 1 : 0, Dg, nullptr));
  PFX_CUDA_TRY(cudaGetLastError());
  return PFX_OK;
}

}  // namespace pfx
