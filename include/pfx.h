/*
 * pfx.h — C ABI of the B200-native partial-fraction exp(A)V engine.
 *
 * The reference (arXiv 2306.16778, package `pfexpm`) has no FFI: its hot path
 * is the private Python function
 *     engine._run_tasks(A, v, opts) -> (acc, per_task_times, t_total)
 *     /root/reference/pkg/src/pfexpm/engine.py:178-230
 * called from engine._matexp (engine.py:241) and engine.matexp_shifted
 * (engine.py:302).  Each entry point below replaces the body of that function
 * for one matrix structure; the package's public API (matexp_full /
 * matexp_action / matexp_shifted, engine.py:254-320) stays Python and calls
 * these through ctypes (paper_2306_16778_b200/_native.py).
 *
 * Semantics shared by every pfx_expm_* call (engine.py:180-229):
 *   out = exp(c) * sum_{k=0}^{npairs-1} S_k      (k ascending)
 *   S_k = 2 Re(a_k Y_k)                 real path  (A real and V real or absent)
 *   S_k = a_k Y_k + conj(a_k) Yc_k      complex action path, Yc_k = (A - cI + theta_k I)^{-H} V
 *   S_k = a_k X_k + (a_k X_k)^H         complex full path,   X_k = (A - cI + theta_k I)^{-1}
 *   Y_k = (A - cI + theta_k I)^{-1} V
 * theta_k, a_k = the n/2 pair representatives of default_table(n)
 * (roots.py:222-226), passed interleaved [re0, im0, re1, im1, ...] in HOST memory.
 * c (shift_c) is 0.0 for the unshifted path; matexp_shifted passes its c
 * (engine.py:299-304 build A - cI and scale by e^c; here both are fused).
 *
 * Memory: `mem` = PFX_MEM_DEVICE -> A, V, out are device pointers on the
 * current CUDA device and `stream` is the cudaStream_t to run on (NULL = legacy
 * default stream); PFX_MEM_HOST -> they are host pointers (pinned or pageable),
 * the library stages them through its device arena and the call returns after
 * the result is back in host memory.  All arrays are C-contiguous (row-major);
 * complex arrays are interleaved binary64 pairs (numpy complex128 layout).
 *
 * Errors: every call returns a status; pfx_last_error() describes the last
 * failure of the calling thread.  Status -> Python exception mapping
 * (errors.py:4-61): PFX_SINGULAR -> SingularSystem, PFX_BADARG -> BadSpec,
 * PFX_CUDA -> PfexpmError.  Inputs are never modified.
 *
 * per_pair_ms (optional, host, npairs floats): device time attributed to each
 * pair, feeding ExpResult.per_term_times (engine.py:102-122).  Pairs that run
 * concurrently inside one launch all report that launch's duration, so
 * max(per_pair_ms) is the simulated-parallel time t_para of the paper.
 */
#ifndef PFX_H
#define PFX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PFX_OK 0
#define PFX_SINGULAR 1
#define PFX_BADARG 2
#define PFX_CUDA 3

#define PFX_MEM_DEVICE 0
#define PFX_MEM_HOST 1

#define PFX_PIVOT_CHECKED 0
#define PFX_PIVOT_ALWAYS 1
#define PFX_PIVOT_NONE 2

/* Library version (major*10000 + minor*100 + patch). */
int pfx_version(void);

/* Message of the last failed call on this thread ("" if none). */
const char* pfx_last_error(void);

/* Free the device arenas and cached pole tables held by the library on the current device. */
int pfx_release(void);

/*
 * Pivoting policy of the dense path (pfx_expm_dense; process-wide, default
 * PFX_PIVOT_CHECKED; see pfx_expm_dense).  pfx_pivot_fallbacks() counts the dense calls
 * whose checked interchange-free factorisation was redone with interchanges.
 */
int pfx_set_pivot_mode(int mode);
int pfx_get_pivot_mode(void);
long long pfx_pivot_fallbacks(void);

/*
 * Threading: one call at a time per device.  Every entry point holds its device's lock
 * for the whole call (the device workspace is shared by all calls on that device);
 * device-memory calls are ordered after the previous call's use of the workspace on the
 * GPU as well (an event the next call's stream waits on), so host threads may call
 * concurrently, on any streams and devices.
 */

/*
 * Pole/residue table of R_n(z) = 1/exp_n(-z): n even in [2, 64].
 * Writes the n/2 representatives theta_k (Im > 0, ascending Re) and residues
 * a_k, interleaved, into theta2[n] and coef2[n] (host arrays of n doubles).
 * Bit-identical to reference roots.default_table(n).thetas_f8()[0::2] /
 * coeffs_f8()[0::2] (roots.py:143-226, 315-318): double-double Newton on
 * exp_n, product-formula residues, conjugate pairing, sorted by (Re, Im).
 */
int pfx_pole_table(int n, double* theta2, double* coef2);

/*
 * Dense Hermitian path — replaces engine._run_tasks for HermitianMatrix
 * (engine.py:194-213; K0 shift formation, K1/K2/K3 solves, K4 inverse,
 * K5 combine, K6 ordered reduction).
 *   A    batch x d x d, real (a_complex = 0) or complex Hermitian.
 *   V    batch x d x nrhs, real or complex; nrhs == 0 selects full mode
 *        (V = I, out is batch x d x d).
 *   out  batch x d x (nrhs or d); complex iff out_complex.  out_complex must
 *        equal !(real path) as defined above (engine.py:185), else PFX_BADARG.
 * Factorisation: LU with partial pivoting, as the reference's LAPACK zgesv / zgetrf
 * (engine.py:200,203,208), under the pivoting policy of pfx_set_pivot_mode:
 *   PFX_PIVOT_CHECKED (default): the factorisation runs without row interchanges and
 *     checks, for every column, that partial pivoting (izamax: max |re|+|im| of the
 *     updated column, first index on ties) would have kept the diagonal pivot; if any
 *     column fails the check, the call is redone with interchanges.  The result is
 *     therefore always a partial-pivoting LU.  For Hermitian A the check essentially never
 *     fails (every pivot of A + theta I has |Im| >= Im theta > 0, SURVEY finding 7, and
 *     the diagonal dominates), so the interchange-free kernels run at full speed.
 *   PFX_PIVOT_ALWAYS: getrf-style interchanges on every column (PFX_DENSE_PIVOT=1 in the
 *     environment forces this too).
 *   PFX_PIVOT_NONE: interchange-free, unchecked (opt-in).
 * (d <= 512: batched SMEM-panel LU; d > 512: blocked LU on DMMA.)  For real A in full
 * mode and d > 512 the inverse is taken as complex symmetric (lower triangle computed,
 * mirrored in the combine).  An exactly zero pivot returns PFX_SINGULAR.
 */
int pfx_expm_dense(int mem, const double* A, int a_complex, int64_t d, int64_t batch, const double* V,
                   int v_complex, int64_t nrhs, double shift_c, const double* theta2, const double* coef2,
                   int npairs, double* out, int out_complex, float* per_pair_ms, void* stream);

/*
 * Column split of the dense full mode for d > 512 (multi-GPU balance: "pole-shard
 * the factorisations, then split each pair's inverse/solve columns across GPUs").  Pair k
 * contributes only the columns [col_ranges[2k], col_ranges[2k+1]) of its inverse X_k
 * (host array of 2*npairs values; each start a multiple of 64):
 *   complex A:  out (+)= e^c sum_k (P_k + P_k^H),  P_k = a_k X_k restricted to its columns
 *   real A:     out (+)= e^c sum_k 2 Re(P_k)
 * so the outputs of calls whose ranges partition [0, d) for every pair add up to
 * pfx_expm_dense's full-mode result (one NCCL reduce across the ranks, as for pole sharding).
 * Every pair is factored whole (one batched LU); its forward substitution starts at its first
 * column (rows above it of L^{-1}E are zero) and only its columns are solved.  accumulate != 0
 * adds to `out` instead of overwriting it.  Replaces the same reference lines as
 * pfx_expm_dense's full mode (engine.py:207-213).
 */
int pfx_expm_dense_cols(int mem, const double* A, int a_complex, int64_t d, double shift_c, const double* theta2,
                        const double* coef2, int npairs, const int64_t* col_ranges, double* out, int out_complex,
                        int accumulate, void* stream);

/*
 * Real symmetric tridiagonal path.
 *   diag (N), off (N-1): T[i][i] = diag[i], T[i+1][i] = T[i][i+1] = off[i].
 *   V, out: N x nrhs real.  Real path only (2 Re(a_k Y_k)).
 * No pivoting: with T real symmetric and Im theta_k > 0 every pivot of
 * T - cI + theta_k I has |Im| >= Im theta_k (SURVEY finding 7).
 */
int pfx_expm_tridiag(int mem, const double* diag, const double* off, int64_t N, const double* V, int64_t nrhs,
                     double shift_c, const double* theta2, const double* coef2, int npairs, double* out,
                     float* per_pair_ms, void* stream);

/*
 * Row-sharded tridiagonal path: multi-GPU domain decomposition of the call above
 * (one process per GPU; device memory on the caller's stream).  The chunk rows are
 * split into nranks contiguous blocks; pfx_tridiag_shard_rows gives this rank's rows
 * [r0, r1).  diag, off, V are the full arrays (only the rank's rows and the couplings
 * at its edges are read); out (N x nrhs) receives rows [r0, r1) only, each final (no
 * reduction: the pole sum is complete per row).  The two chunk scans that cross rank
 * edges (pivot carries, right-hand-side carries) each exchange one small aggregate
 * per rank, through allgather(ctx, buf, count): buf holds nranks x count doubles,
 * this rank's block at buf + rank * count filled by the library, the callback fills
 * the others (a torch.distributed all-gather on the Python side) and returns 0.
 * Same results as pfx_expm_tridiag up to the rounding of a different chunking.
 * npairs <= 16.
 */
typedef int (*pfx_allgather_fn)(void* ctx, double* buf, int64_t count);
int pfx_tridiag_shard_rows(int64_t N, int64_t nrhs, int rank, int nranks, int64_t* r0, int64_t* r1);
int pfx_expm_tridiag_shard(const double* diag, const double* off, int64_t N, const double* V, int64_t nrhs,
                           double shift_c, const double* theta2, const double* coef2, int npairs, double* out,
                           int rank, int nranks, pfx_allgather_fn allgather, void* ctx, void* stream);
/*
 * Real symmetric banded path.
 *   band (kb+1) x N, lower symmetric band storage: band[r][j] = A[j+r][j].
 *   V, out: N x nrhs real.  No pivoting (same argument as above).
 */
int pfx_expm_banded(int mem, const double* band, int64_t N, int64_t kb, const double* V, int64_t nrhs,
                    double shift_c, const double* theta2, const double* coef2, int npairs, double* out,
                    float* per_pair_ms, void* stream);

/*
 * Single-shift solve (reference linalg.shifted_solve, linalg.py:92-103):
 * Y = (A + theta I)^{-1} V for one dense Hermitian A, partial pivoting (any d:
 * d <= 512 the batched SMEM-panel kernel, d > 512 blocked getrf/getrs on DMMA).
 * theta may be real.  V, Y: d x nrhs complex.  Device or host memory as `mem`.
 */
int pfx_shifted_solve(int mem, const double* A, int a_complex, int64_t d, double theta_re, double theta_im,
                      const double* V, int64_t nrhs, double* Y, void* stream);

/*
 * Kernel timing (used by bench.py to time the dominant kernel live, on the
 * stream the kernels run on).  When enabled, every kernel launch of the
 * library is bracketed by CUDA events on its stream.  pfx_prof_read()
 * synchronises those events and writes one line per kernel name,
 * "name launches total_ms total_flops\n" (flops = algorithmic count of the
 * launches that declare one, else 0), into buf (NUL-terminated, truncated to buflen),
 * then clears the record.  Returns the number of bytes needed.
 */
int pfx_prof_enable(int on);
int pfx_prof_read(char* buf, int buflen);

#ifdef __cplusplus
}
#endif

#endif /* PFX_H */
