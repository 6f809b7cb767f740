/*
 * srlu.h — C ABI of the B200 (sm_100a) sparse randomized LU library
 * (libsrlu.so).  Plain pointers and sizes only; every device buffer is
 * owned by the caller (e.g. the torch caching allocator), every call is
 * asynchronous on the caller's stream, nothing allocates, no C++ exception
 * crosses the boundary.  Return 0 (SRLU_OK) or a negative SRLU_ERR_*;
 * srlu_last_error() returns a thread-local message for the last failure.
 *
 * Reference interfaces replaced (paths relative to
 * /root/reference/pkg/src/sparselu/):
 *   srlu_seed_key / srlu_draw_sem / srlu_draw_fast_transform
 *        <- sketch.py:42-43 (_rng), :103-114 (build_sem),
 *           :214-235 (build_fast_transform), :269-278 (build_composite)
 *   srlu_sem_plan             <- the accumulation order of _fast.pyx:44-90
 *                                (bucket-grouped, ascending source index)
 *   srlu_sketch_right_dense   <- sketch.py:362-368 apply_sketch_right =
 *                                _fast.pyx:44-54 sem_gather_dense +
 *                                sketch.py:322-335 _fast_adjoint_right +
 *                                _fast.pyx:23-41 fwht_rows (fused)
 *   srlu_sketch_right_csr     <- same with _fast.pyx:57-68 sem_gather_csc
 *   srlu_sem_gather_dense     <- _kernels.sem_gather_dense (_fast.pyx:44-54)
 *   srlu_fwht_rows            <- _kernels.fwht_rows (_fast.pyx:23-41)
 *   srlu_sketch_left_dense    <- matrix.py:201-207 permute_rows +
 *                                sketch.py:371-378 apply_sketch_left =
 *                                _fast.pyx:71-78 sem_scatter_dense +
 *                                sketch.py:338-349 _fast_mul_left (fused;
 *                                P·A is never materialised)
 *   srlu_sketch_left_csr      <- same with _fast.pyx:81-90 sem_scatter_csc
 *   srlu_lu_rowpiv            <- factor.py:49-77 lu_row_pivot
 *   srlu_lu_colpiv            <- factor.py:80-109 lu_col_pivot
 */
#ifndef SRLU_H
#define SRLU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *srlu_stream_t; /* == cudaStream_t */

#define SRLU_OK 0
#define SRLU_ERR_ARG (-1)
#define SRLU_ERR_CUDA (-2)
#define SRLU_ERR_UNSUPPORTED (-3)
#define SRLU_ERR_WORKSPACE (-4)

/* element type codes of the input matrix A (arithmetic is always fp64) */
#define SRLU_F32 0
#define SRLU_F64 1

const char *srlu_last_error(void);
int srlu_version(void);

/* ---- seed-derived draws (K0) ------------------------------------------ */

/* numpy SeedSequence(seed).generate_state(2, uint64): the Philox key. Host. */
int srlu_seed_key(uint64_t seed, uint64_t key[2]);

/* build_fast_transform(k, l, "hadamard", seed) on the HOST (pad <= 2^20
 * sequential Fisher-Yates swaps): phase[l] = +-1, sample_idx[k], *pad. */
int srlu_draw_fast_transform(uint64_t seed, int64_t k, int64_t l, double *phase,
                             int64_t *sample_idx, int64_t *pad);

/* build_composite(k, l, n, seed) (sketch.py:269-278) in ONE call: the
 * transform stage (seed + 2**32) drawn on the host into `staging` (pinned,
 * srlu_build_composite_staging bytes; the caller must not reuse it before the
 * uploads on `stream` completed) and uploaded to phase[l] / sample_idx[k]
 * (int32); the sparse stage drawn on the device (row_of[n], sign[n]) and its
 * accumulation plan (sorted[n], bucket_ptr[l+1]) as srlu_sem_plan.
 * *pad (host) = the transform's power-of-two length. */
size_t srlu_build_composite_workspace(int64_t n, int64_t l);
size_t srlu_build_composite_staging(int64_t k, int64_t l);
int srlu_build_composite(uint64_t seed, int64_t k, int64_t l, int64_t n, int32_t *row_of,
                         double *sign, int32_t *sorted, int32_t *bucket_ptr, double *phase,
                         int32_t *sample_idx, int64_t *pad, void *staging, size_t staging_bytes,
                         void *ws, size_t ws_bytes, srlu_stream_t stream);

/* build_composite plus, when sched != NULL, the scheduled K1's gather
 * schedule for an A of element type dtype (srlu_k1_schedule), in one call. */
int srlu_build_composite_k1(uint64_t seed, int64_t k, int64_t l, int64_t n, int32_t *row_of,
                            double *sign, int32_t *sorted, int32_t *bucket_ptr, double *phase,
                            int32_t *sample_idx, int64_t *pad, void *staging, size_t staging_bytes,
                            void *ws, size_t ws_bytes, int dtype, void *sched, size_t sched_bytes,
                            srlu_stream_t stream);

/* build_composite_k1 followed, on the same stream and in the same call, by
 * *nonfinite = 0 and the stage-1 sketch Y = A . Omega^* of a dense A
 * (srlu_sketch_right_dense_sched when sched != NULL, else
 * srlu_sketch_right_dense): randlu.py:252-253 (build_composite, then
 * apply_sketch_right) as one host entry.  mult = scale / sqrt(pad) with
 * scale = sqrt(pad / k) (sketch.py:330). */
int srlu_composite_sketch_right_dense(uint64_t seed, int64_t k, int64_t l, int64_t n,
                                      int32_t *row_of, double *sign, int32_t *sorted,
                                      int32_t *bucket_ptr, double *phase, int32_t *sample_idx,
                                      int64_t *pad, void *staging, size_t staging_bytes, void *ws,
                                      size_t ws_bytes, void *sched, size_t sched_bytes,
                                      const void *a, int dtype, int64_t m, int64_t lda,
                                      double mult, double *y, int64_t ldy, int *nonfinite,
                                      srlu_stream_t stream);

/* build_sem(l, n, seed) on the DEVICE: row_of[n] in [0,l), sign[n] = +-1.
 * Bit-exact with numpy Generator(Philox(seed)).integers (Lemire). */
size_t srlu_draw_sem_workspace(int64_t n, int64_t l);
int srlu_draw_sem(uint64_t seed, int64_t l, int64_t n, int32_t *row_of, double *sign,
                  void *ws, size_t ws_bytes, srlu_stream_t stream);

/* ---- sparse-embedding plan -------------------------------------------- */

/* Stable bucket sort of the n sources by row_of: sorted[bucket_ptr[t] ..
 * bucket_ptr[t+1]) lists, ascending, the sources j with row_of[j] == t;
 * the sign is folded into bit 31 (set = -1). */
size_t srlu_sem_plan_workspace(int64_t n, int64_t l);
int srlu_sem_plan(const int32_t *row_of, const double *sign, int64_t n, int64_t l,
                  int32_t *sorted, int32_t *bucket_ptr, void *ws, size_t ws_bytes,
                  srlu_stream_t stream);

/* ---- stage 1: Y = A · Omega1^*  (K1) ----------------------------------- */

/* A: m x n row-major (lda >= n), dtype SRLU_F32/F64.  Y: m x k1 row-major
 * fp64.  mult1 = scale/sqrt(pad1).  *nonfinite |= 1 if any Y entry (hence
 * any A entry) is not finite. */
int srlu_sketch_right_dense(const void *a, int dtype, int64_t m, int64_t n, int64_t lda,
                            const int32_t *sorted1, const int32_t *bucket_ptr1, int64_t l1,
                            const double *phase1, const int32_t *idx1, int64_t k1,
                            int64_t pad1, double mult1, double *y, int64_t ldy,
                            int *nonfinite, srlu_stream_t stream);

/* Scheduled K1 (same result, bit for bit; replaces the same reference lines
 * as srlu_sketch_right_dense).  srlu_k1_schedule_bytes returns 0 when the
 * shape is outside the scheduled kernel's range (rows of more than four
 * 32 KB chunks, l1 > 3584, pad1 outside [32, 8192]); the caller then uses
 * srlu_sketch_right_dense.  srlu_k1_schedule builds, from the plan of
 * srlu_sem_plan, the per-warp gather schedule (bank-conflict-free 16-bit
 * codes) into `sched`; it depends only on the sketch, n and dtype and can
 * be reused for every A with that shape.  A must be 16-byte aligned with a
 * 16-byte row pitch. */
size_t srlu_k1_schedule_bytes(int64_t n, int64_t l1, int64_t pad1, int dtype);
/* the scheduled kernel's geometry for a shape (diagnostics): info = {rows
 * per block, bucket slots per lane, chunk columns, chunks, stages, code
 * bytes that fit in shared memory, shared memory bytes, max lanes per bank};
 * SRLU_ERR_UNSUPPORTED (info zeroed) when the shape is not scheduled. */
int srlu_k1_config(int64_t n, int64_t l1, int64_t pad1, int dtype, int64_t info[8]);
int srlu_k1_schedule(const int32_t *sorted1, const int32_t *bucket_ptr1, int64_t n, int64_t l1,
                     int64_t pad1, int dtype, void *sched, size_t sched_bytes,
                     srlu_stream_t stream);
int srlu_sketch_right_dense_sched(const void *a, int dtype, int64_t m, int64_t n, int64_t lda,
                                  const void *sched, size_t sched_bytes, int64_t l1,
                                  const double *phase1, const int32_t *idx1, int64_t k1,
                                  int64_t pad1, double mult1, double *y, int64_t ldy,
                                  int *nonfinite, srlu_stream_t stream);

/* A in CSR: indptr[m+1] (int64), indices (int32, ascending per row),
 * values (dtype).  row_of1/sign1: the raw draws. */
int srlu_sketch_right_csr(const int64_t *indptr, const int32_t *indices, const void *vals,
                          int dtype, int64_t m, int64_t n, const int32_t *row_of1,
                          const double *sign1, int64_t l1, const double *phase1,
                          const int32_t *idx1, int64_t k1, int64_t pad1, double mult1,
                          double *y, int64_t ldy, int *nonfinite, srlu_stream_t stream);

/* plugin seam: out (m x l row-major fp64) = A · S^T (no transform) */
int srlu_sem_gather_dense(const void *a, int dtype, int64_t m, int64_t n, int64_t lda,
                          const int32_t *sorted, const int32_t *bucket_ptr, int64_t l,
                          double *out, int64_t ldo, srlu_stream_t stream);

/* plugin seam: in-place unnormalised Walsh-Hadamard of each row of x
 * (m x n row-major fp64, n a power of two, ldx >= n) */
int srlu_fwht_rows(double *x, int64_t m, int64_t n, int64_t ldx, srlu_stream_t stream);

/* ---- stage 2: Omega2 · (P A)  (K3) ------------------------------------- */

/* Member table for the left sketch of P·A restricted to the local row
 * shard [row0, row0+rows): for every PA index q (grouped by bucket via
 * sorted2/bucket_ptr2), member_row[e] = perm[q]-row0 if that row is local,
 * else -1; member_sign[e] = +-1.  perm == NULL means P = identity. */
int srlu_sem_members(const int32_t *sorted2, int64_t m, const int64_t *perm, int64_t row0,
                     int64_t rows, int32_t *member_row, double *member_sign,
                     srlu_stream_t stream);

/* out (n x k2 row-major, ldo >= k2) = (Omega2 · P A)^T over the local rows.
 * S (l2 x n fp64) is caller scratch: srlu_sketch_left_workspace bytes. */
size_t srlu_sketch_left_workspace(int64_t n, int64_t l2, int64_t pad2);
int srlu_sketch_left_dense(const void *a, int dtype, int64_t rows, int64_t n, int64_t lda,
                           const int32_t *member_row, const double *member_sign,
                           const int32_t *bucket_ptr2, int64_t l2, const double *phase2,
                           const int32_t *idx2, int64_t k2, int64_t pad2, double mult2,
                           double *out, int64_t ldo, void *ws, size_t ws_bytes,
                           srlu_stream_t stream);

/* plugin seam: out (l x n row-major fp64, ldo >= n) = S · (P A) over the
 * members (no transform); rows with member_row < 0 are skipped. */
int srlu_sem_scatter_dense(const void *a, int dtype, int64_t rows, int64_t n, int64_t lda,
                           const int32_t *member_row, const double *member_sign,
                           const int32_t *bucket_ptr, int64_t l, double *out, int64_t ldo,
                           srlu_stream_t stream);

/* plugin seam, sparse variants, O(nnz), one thread per row / column walking
 * its entries in ascending index (the reference's sequential sums):
 *   srlu_sem_gather_csr  <- _fast.pyx:57-68 sem_gather_csc, on the CSR form
 *     of the same matrix (rows x n, entries ascending in j per row):
 *     out[i, row_of[j]] += sign[j] * a[i, j], out rows x l row-major fp64;
 *   srlu_sem_scatter_csc <- _fast.pyx:81-90 sem_scatter_csc on the CSC
 *     arrays (entries ascending in i per column):
 *     out[row_of[i], j] += sign[i] * a[i, j], out l x cols row-major fp64. */
int srlu_sem_gather_csr(const int64_t *indptr, const int32_t *indices, const void *vals,
                        int dtype, int64_t rows, const int32_t *row_of, const double *sign,
                        double *out, int64_t ldo, srlu_stream_t stream);
int srlu_sem_scatter_csc(const int64_t *indptr, const int32_t *indices, const void *vals,
                         int dtype, int64_t cols, const int32_t *row_of, const double *sign,
                         double *out, int64_t ldo, srlu_stream_t stream);

/* CSR variant; inv_perm[row] = PA index of local row (row0 offset applied
 * by the caller), row_of2/sign2 indexed by PA index.  Any column length
 * (columns beyond one CTA's 8192-entry sort are folded in bucket ranges and
 * ascending-q chunks); *flags |= 2 is kept for an internal inconsistency
 * only. */
size_t srlu_sketch_left_csr_workspace(int64_t rows, int64_t n, int64_t nnz, int64_t l2,
                                      int64_t pad2);
int srlu_sketch_left_csr(const int64_t *indptr, const int32_t *indices, const void *vals,
                         int dtype, int64_t rows, int64_t n, int64_t nnz,
                         const int32_t *inv_perm, const int32_t *row_of2, const double *sign2,
                         int64_t l2, const double *phase2, const int32_t *idx2, int64_t k2,
                         int64_t pad2, double mult2, double *out, int64_t ldo, void *ws,
                         size_t ws_bytes, int *flags, srlu_stream_t stream);

/* ---- pivoted LU of the sketches (K2, K5) ------------------------------- */

/* Workspace for a persistent LU over M entities of k values. */
size_t srlu_lu_workspace(int64_t M, int64_t k);

/* Row-pivoted LU of Y (m x k row-major, overwritten as scratch):
 * perm[m] (position -> row), L (m x k row-major, position order, unit
 * lower-trapezoidal), U (k x k row-major, may be NULL). */
int srlu_lu_rowpiv(double *y, int64_t m, int64_t k, int64_t ldy, int64_t *perm, double *L,
                   int64_t ldl, double *U, int64_t ldu, int reserve_sms, void *ws,
                   size_t ws_bytes, srlu_stream_t stream);

/* Both LUs are one cooperative persistent kernel, one CTA per SM;
 * `reserve_sms` SMs are left out of the grid so a kernel already running on
 * another stream (the rank test, srlu_qr_rank) does not hold the launch
 * back.  0 = use every SM. */

/* Column-pivoted LU of core (k x n) given as its transpose ct (n x k
 * row-major, overwritten): q[n], Lt (k x k row-major unit lower),
 * UT (n x k row-major) = U^T, i.e. U (k x n) in column-major storage. */
int srlu_lu_colpiv(double *ct, int64_t n, int64_t k, int64_t ldc, int64_t *q, double *Lt,
                   int64_t ldlt, double *UT, int64_t ldut, int reserve_sms, void *ws,
                   size_t ws_bytes, srlu_stream_t stream);

/* ---- small dense tail (K4) --------------------------------------------- */

/* left_pseudo_inverse (factor.py:112-130) of M (k2 x k1) given as mT = M^T
 * (k1 x k2 row-major), in one CTA: Householder QR, rank test, and
 * pinvT = (R^-1 Q^T)^T (k2 x k1 row-major); the rank test is
 * srlu_qr_rank (stats[4]: sigma_max estimate, sigma_min estimate, cond,
 * singular flag = 1.0 when sigma_min <= 1e-10 sigma_max, factor.py:124).
 * `stats` is unused here (kept for ABI stability).  When M does not fit one
 * CTA (srlu_qr_pinv_smem_bytes(k1, k2) > 220 KiB or k1 > 256) the QR runs
 * on one thread-block cluster of up to 16 CTAs (k1 <= 576; M's columns
 * spread over the CTAs' shared memory, reflectors pushed through DSMEM). */
size_t srlu_qr_pinv_smem_bytes(int64_t k1, int64_t k2);
size_t srlu_qr_pinv_workspace(int64_t k1, int64_t k2);
int srlu_qr_pinv(const double *mT, int64_t k1, int64_t k2, int64_t ldm, double *pinvT,
                 int64_t ldp, double *stats, void *ws, size_t ws_bytes, srlu_stream_t stream);

/* the rank test on the R left in the srlu_qr_pinv workspace `ws` (run it
 * after srlu_qr_pinv on the same stream; it can overlap later work on
 * other streams: only the host's final decision needs stats). */
int srlu_qr_rank(const void *ws, int64_t k1, int64_t k2, double *stats, srlu_stream_t stream);

/* srlu_qr_rank plus certified bounds, once pinvT (srlu_qr_pinv's output) is
 * ready: stats[8] = {sigma_max estimate, sigma_min estimate, cond estimate,
 * flag, ||R||_F, ||pinv||_F, ||R||_F ||pinv||_F, 0}.  The estimates bracket
 * the extreme singular values from the inside and ||R||_F, 1/||R^-1||_F =
 * 1/||pinv||_F from the outside, so flag = 1 (singular: sigma_min <= 1e-10
 * sigma_max, factor.py:123-124) and flag = 0 (not) are certain; flag = 2:
 * the bounds straddle the threshold — call srlu_rank_exact. */
int srlu_qr_rank_certified(const void *ws, int64_t k1, int64_t k2, const double *pinvT,
                           int64_t ldp, double *stats, srlu_stream_t stream);

/* the reference's decision on the singular values themselves (factor.py:
 * 122-128 numpy.linalg.svd of R): one-sided Jacobi on the R left in the
 * srlu_qr_pinv workspace qr_ws; stats[4] = {sigma_max, sigma_min, cond,
 * singular flag}.  ws: srlu_rank_exact_workspace(k1) bytes. */
size_t srlu_rank_exact_workspace(int64_t k1);
int srlu_rank_exact(const void *qr_ws, int64_t k1, int64_t k2, void *ws, size_t ws_bytes,
                    double *stats, srlu_stream_t stream);

/* the same rank test on an upper-triangular R (k x k, k <= 576, device),
 * given row-major (R, ldr) and transposed (RT = R^T row-major, ldt) */
int srlu_rank_estimate(const double *R, int64_t k, int64_t ldr, const double *RT, int64_t ldt,
                       double *stats, srlu_stream_t stream);

/* ---- FP64 tensor-core GEMMs (DMMA) and the approximation error (K7) ---- */

/* C (M x N) = A (M x K) · B (K x N), row-major fp64 on the FP64 tensor cores
 * (matrix.py:219-230 matmul for randlu.py:267 core = pinv·(Omega2 P A) and
 * randlu.py:272 L = L1·L~).  srlu_dgemm_ex flags: SRLU_GEMM_B_LOWER — B is
 * lower triangular (B[j][c] == 0 for j < c, like L~), the zero blocks are
 * skipped. */
#define SRLU_GEMM_B_LOWER 1
int srlu_dgemm(const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
               int64_t ldc, int64_t M, int64_t N, int64_t K, srlu_stream_t stream);
int srlu_dgemm_ex(const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                  int64_t ldc, int64_t M, int64_t N, int64_t K, int flags,
                  srlu_stream_t stream);

/* approximation_error (randlu.py:279-302): *sq (device) = ||L U - P A Q||_F^2
 * for L (m x k row-major, positions), U given as UT (n x k row-major, U^T),
 * perm[m] / q[n] the row / column permutations, A dense (m x n, lda) or
 * CSR (indptr int64[m+1], indices int32 ascending per row, values).  Fixed
 * summation order: deterministic.  Workspace: srlu_lu_error_workspace. */
size_t srlu_lu_error_workspace(int64_t m, int64_t n, int64_t k);
int srlu_lu_error_dense(const double *L, int64_t ldl, const double *UT, int64_t ldut,
                        const int64_t *perm, const int64_t *q, const void *a, int dtype,
                        int64_t m, int64_t n, int64_t lda, int64_t k, double *sq, void *ws,
                        size_t ws_bytes, srlu_stream_t stream);
int srlu_lu_error_csr(const double *L, int64_t ldl, const double *UT, int64_t ldut,
                      const int64_t *perm, const int64_t *q, const int64_t *indptr,
                      const int32_t *indices, const void *vals, int dtype, int64_t m, int64_t n,
                      int64_t k, double *sq, void *ws, size_t ws_bytes, srlu_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SRLU_H */
