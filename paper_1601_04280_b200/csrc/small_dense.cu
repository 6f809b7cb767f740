// K4 — the small dense tail of the pipeline (reference: factor.py:112-130
// left_pseudo_inverse, randlu.py:266-267 and :272 matmul).
//
//  * srlu_qr_pinv: Householder QR of M = Omega2·L1 (k2 x k1) in ONE CTA with
//    M resident in shared memory (LAPACK dgeqr2/dlarfg conventions), the
//    rank test, and pinv^T = (R^-1 Q^T)^T.  Replaces numpy.linalg.qr +
//    numpy.linalg.svd + scipy solve_triangular.
//  * rank test: the reference compares the extreme singular values of R
//    (sv[-1] <= 1e-10 sv[0]).  Here: sigma_max >= max(|R_jj|, ||R x||) from
//    8 power iterations, sigma_min <= min(|R_jj|, ||(R^T R)^-1 x||^-1/2)
//    from 8 inverse iterations — estimates that bracket the true values from
//    the inside and agree with the SVD decision except when cond(R) sits
//    within the estimators' slack of 1e10.
//  * srlu_rank_estimate: the same test on an R in global memory (used when
//    M does not fit one CTA; the QR then comes from cuSOLVER).
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"
#include "tma.cuh"

#ifdef SRLU_QR_TRACE
__device__ long long g_qr_trace[256][6];
#define QR_T(c, i) \
    do { if ((threadIdx.x % 8) == 0) g_qr_trace[c][i] = clock64(); } while (0)
#else
#define QR_T(c, i) do { } while (0)
#endif

namespace srlu {

// qr_cluster.cu
int qr_cluster_launch(const double *mT, int64_t k1, int64_t k2, int64_t ldm, double *qa,
                      double *qtau, double *rrow, cudaStream_t st);
size_t jacobi_workspace(int64_t k);
int jacobi_launch(const double *rrow, int64_t k, void *ws, double *stats, cudaStream_t st);

constexpr double kRankRtol = 1e-10;  // factor.py:22

__device__ inline double block_sum(double v, double *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
    const int nw = blockDim.x >> 5;
    for (int w = 0; w < nw; ++w) s += red[w];
    return s;
}

__device__ inline double block_max(double v, double *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = red[0];
    const int nw = blockDim.x >> 5;
    for (int w = 1; w < nw; ++w) s = fmax(s, red[w]);
    return s;
}

__device__ inline double block_min(double v, double *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off; off >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, off));
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = red[0];
    const int nw = blockDim.x >> 5;
    for (int w = 1; w < nw; ++w) s = fmin(s, red[w]);
    return s;
}

// Rank test on an upper-triangular R given twice: Rr (row-major, row r
// contiguous) and Rc (column-major, column c contiguous).  stats[0] =
// sigma_max estimate, [1] = sigma_min estimate, [2] = cond, [3] = singular.
//  * sigma_max >= max(|R_jj|, ||R x||) over 6 power iterations (whole CTA);
//  * sigma_min <= min(|R_jj|, ||(R^T R)^-1 x||^-1/2) over 3 inverse
//    iterations.  The two triangular solves run on warp 0 in axpy form with
//    the vector distributed over the lanes' registers (lane l owns entries
//    j == l mod 32) and the next row/column prefetched, so each of the k
//    sequential steps costs one shuffle broadcast + k/32 FMAs.
constexpr int kRankMaxPerLane = 18;  // k <= 576
constexpr int kTailMaxPer = 8;       // register-resident pinv columns: k2 <= 256

// warp 0: 3 inverse iterations, vectors distributed over lane registers
// (lane l owns entries j == l mod 32, PER per lane), next row prefetched.
template <int PER>
__device__ double inverse_iteration(const double *__restrict__ Rr, int64_t ldr,
                                    const double *__restrict__ Rc, int64_t ldc, int k,
                                    double est, double inv_sqrt_k) {
    const int lane = threadIdx.x & 31;
    double v[PER], rd[PER], w[PER], nx[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int j = i * 32 + lane;
        v[i] = j < k ? ((j & 1) ? -inv_sqrt_k : inv_sqrt_k) : 0.0;
        rd[i] = j < k ? 1.0 / Rr[(int64_t)j * ldr + j] : 0.0;
        w[i] = 0.0;
    }
    for (int it = 0; it < 3; ++it) {
        // R^T w = v (forward, axpy form on rows of R)
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int c = i * 32 + lane;
            nx[i] = c < k ? Rr[c] : 0.0;  // row 0
        }
        for (int r = 0; r < k; ++r) {
            double cur[PER];
#pragma unroll
            for (int i = 0; i < PER; ++i) cur[i] = nx[i];
            if (r + 1 < k) {
                const double *nrow = Rr + (int64_t)(r + 1) * ldr;
#pragma unroll
                for (int i = 0; i < PER; ++i) {
                    const int c = i * 32 + lane;
                    nx[i] = c < k ? nrow[c] : 0.0;
                }
            }
            const int ro = r & 31, ri = r >> 5;
            double vr = 0.0, rdr = 0.0;
#pragma unroll
            for (int i = 0; i < PER; ++i)
                if (i == ri) { vr = v[i]; rdr = rd[i]; }
            const double wr = __shfl_sync(0xffffffffu, vr * rdr, ro);
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const int c = i * 32 + lane;
                if (c > r) v[i] = __fma_rn(-cur[i], wr, v[i]);
                if (i == ri && lane == ro) w[i] = wr;
            }
        }
        // R z = w (backward, axpy form on columns of R = rows of Rc)
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int r = i * 32 + lane;
            nx[i] = r < k ? Rc[(int64_t)(k - 1) * ldc + r] : 0.0;
        }
        for (int c = k - 1; c >= 0; --c) {
            double cur[PER];
#pragma unroll
            for (int i = 0; i < PER; ++i) cur[i] = nx[i];
            if (c > 0) {
                const double *ncol = Rc + (int64_t)(c - 1) * ldc;
#pragma unroll
                for (int i = 0; i < PER; ++i) {
                    const int r = i * 32 + lane;
                    nx[i] = r < c - 1 ? ncol[r] : 0.0;
                }
            }
            const int co = c & 31, ci = c >> 5;
            double wc = 0.0, rdc = 0.0;
#pragma unroll
            for (int i = 0; i < PER; ++i)
                if (i == ci) { wc = w[i]; rdc = rd[i]; }
            const double zc = __shfl_sync(0xffffffffu, wc * rdc, co);
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const int r = i * 32 + lane;
                if (r < c) w[i] = __fma_rn(-cur[i], zc, w[i]);
                if (i == ci && lane == co) v[i] = zc;
            }
        }
        double zz = 0.0;
#pragma unroll
        for (int i = 0; i < PER; ++i) zz = __fma_rn(v[i], v[i], zz);
#pragma unroll
        for (int off = 16; off; off >>= 1) zz += __shfl_xor_sync(0xffffffffu, zz, off);
        if (!(zz > 0.0) || !isfinite(zz)) return 0.0;
        est = fmin(est, 1.0 / sqrt(sqrt(zz)));
        const double inv = 1.0 / sqrt(zz);
#pragma unroll
        for (int i = 0; i < PER; ++i) v[i] *= inv;
    }
    return est;
}

__device__ void rank_estimate(const double *__restrict__ Rr, int64_t ldr,
                              const double *__restrict__ Rc, int64_t ldc, int k, double *x,
                              double *y, double *red, double *stats,
                              const double *__restrict__ pinvT = nullptr, int64_t ldp = 0,
                              int k2 = 0) {
    const int tid = threadIdx.x;
    double dmax = 0.0, dmin = INFINITY;
    for (int j = tid; j < k; j += blockDim.x) {
        const double d = fabs(Rr[(int64_t)j * ldr + j]);
        dmax = fmax(dmax, d);
        dmin = fmin(dmin, d);
    }
    dmax = block_max(dmax, red);
    dmin = block_min(dmin, red);
    double smax = dmax, smin = dmin;
    const double inv_sqrt_k = 1.0 / sqrt((double)k);
    for (int j = tid; j < k; j += blockDim.x) x[j] = inv_sqrt_k;
    __syncthreads();
    for (int it = 0; it < 6 && dmax > 0.0; ++it) {
        double ss = 0.0;
        for (int r = tid; r < k; r += blockDim.x) {  // y = R x (row r of R)
            const double *row = Rr + (int64_t)r * ldr;
            double s0 = 0.0, s1 = 0.0;
            int c = r;
            for (; c + 1 < k; c += 2) {
                s0 += row[c] * x[c];
                s1 += row[c + 1] * x[c + 1];
            }
            if (c < k) s0 += row[c] * x[c];
            y[r] = s0 + s1;
            ss += (s0 + s1) * (s0 + s1);
        }
        ss = block_sum(ss, red);
        smax = fmax(smax, sqrt(ss));
        double zz = 0.0;
        for (int c = tid; c < k; c += blockDim.x) {  // x = R^T y (column c of R)
            const double *col = Rc + (int64_t)c * ldc;
            double s0 = 0.0, s1 = 0.0;
            int r = 0;
            for (; r + 1 <= c; r += 2) {
                s0 += col[r] * y[r];
                s1 += col[r + 1] * y[r + 1];
            }
            if (r <= c) s0 += col[r] * y[r];
            x[c] = s0 + s1;
            zz += (s0 + s1) * (s0 + s1);
        }
        zz = block_sum(zz, red);
        const double inv = zz > 0.0 ? 1.0 / sqrt(zz) : 0.0;
        for (int c = tid; c < k; c += blockDim.x) x[c] *= inv;
        __syncthreads();
    }
    if (dmin > 0.0 && tid < 32) {
        if (k <= 128) smin = inverse_iteration<4>(Rr, ldr, Rc, ldc, k, smin, inv_sqrt_k);
        else if (k <= 256) smin = inverse_iteration<8>(Rr, ldr, Rc, ldc, k, smin, inv_sqrt_k);
        else smin = inverse_iteration<kRankMaxPerLane>(Rr, ldr, Rc, ldc, k, smin, inv_sqrt_k);
    } else if (!(dmin > 0.0)) {
        smin = 0.0;
    }
    // certified bounds (pinvT given): sigma_max <= ||R||_F and sigma_min >=
    // 1/||R^-1||_F = 1/||pinv||_F (pinv = R^-1 Q^T, Q orthonormal columns)
    double fr = 0.0, fp = 0.0;
    if (pinvT != nullptr) {
        for (int64_t i = tid; i < (int64_t)k * k; i += blockDim.x) {
            const int r = (int)(i / k), c = (int)(i % k);
            if (c >= r) {
                const double v = Rr[(int64_t)r * ldr + c];
                fr = __fma_rn(v, v, fr);
            }
        }
        for (int64_t i = tid; i < (int64_t)k2 * k; i += blockDim.x) {
            const double v = pinvT[(i / k) * ldp + i % k];
            fp = __fma_rn(v, v, fp);
        }
        fr = block_sum(fr, red);
        fp = block_sum(fp, red);
    }
    if (tid == 0) {
        stats[0] = smax;
        stats[1] = smin;
        stats[2] = smin > 0.0 ? smax / smin : INFINITY;
        // estimates bracket from the inside: smin_true <= smin, smax_true >= smax
        const bool sing = smax == 0.0 || smin <= kRankRtol * smax;
        stats[3] = sing ? 1.0 : 0.0;
        if (pinvT != nullptr) {
            const double hi = sqrt(fr) * sqrt(fp);  // >= the true condition number
            stats[4] = sqrt(fr);
            stats[5] = sqrt(fp);
            stats[6] = hi;
            stats[7] = 0.0;
            // certain when the outside bound already clears the threshold
            // (1e-4 margin: pinv's own rounding at cond <= 1e10), else
            // flag 2 = undecided: the host runs the exact singular values
            if (!sing && !(isfinite(hi) && hi * (1.0 + 1e-4) < 1.0 / kRankRtol)) stats[3] = 2.0;
        }
    }
}

// Phase 1 (one CTA): Householder QR of M in shared memory (LAPACK dgeqr2 /
// dlarfg conventions); the packed reflectors/R (column-major, stride ld),
// tau and R row-major (for the rank test) go to global memory.
// Dataflow, no CTA-wide barrier in the sweep: a group of TPC threads owns
// column c.  It waits for reflectors 0..c-1 in order (one mbarrier per
// reflector, completed by the TPC threads of the group that formed it),
// applies each to its column, and — with the sub-diagonal norm accumulated
// inside the last update — forms reflector c (dlarfg) and arrives on its
// mbarrier.  The critical path per reflector is therefore one column
// update + one dlarfg; every other column catches up off that path.
// Reflectors stay unscaled during the sweep (the 1/(alpha-beta) factor is
// folded into the dot and the update) and are scaled once at the end.
template <int TPC>
__device__ inline double group_sum(double v) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned mask = (TPC == 32 ? 0xffffffffu : ((1u << TPC) - 1u) << (lane & ~(TPC - 1)));
#pragma unroll
    for (int off = 1; off < TPC; off <<= 1) v += __shfl_xor_sync(mask, v, off);
    return v;
}

// dlarfg on a column whose alpha = col[j] and sub-diagonal sum of squares
// `part` are known; writes tau, scal = 1/(alpha-beta) and beta into col[j].
__device__ inline void dlarfg(double *col, int j, double part, double *tau_out,
                              double *scal_out) {
    const double alpha = col[j];
    double t = 0.0, scal = 0.0;
    if (part > 0.0) {
        const double beta = -copysign(sqrt(__fma_rn(alpha, alpha, part)), alpha);
        t = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
        col[j] = beta;
    }
    *tau_out = t;
    *scal_out = scal;
}

template <int TPC>
__global__ void __launch_bounds__(1024, 1) qr_kernel(const double *__restrict__ mT, int k1,
                                                     int k2, int64_t ldm,
                                                     double *__restrict__ qa,
                                                     double *__restrict__ qtau,
                                                     double *__restrict__ rrow) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int ld = k2 | 1;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw);           // k1 mbarriers
    double *s_tau = reinterpret_cast<double *>(smem_raw) + k1;        // k1
    double *s_scal = s_tau + k1;                                      // k1
    double *A = s_scal + k1;  // column c: A[c*ld + r] = M[r][c]
    const int tid = threadIdx.x;
    const int c = tid / TPC, q = tid % TPC;
    const unsigned gmask = (TPC == 32 ? 0xffffffffu
                                      : ((1u << TPC) - 1u) << ((tid & 31) & ~(TPC - 1)));

    {  // stage M (loads batched 8 deep: the copy is L2-latency bound)
        const int n = k1 * k2;
        for (int i0 = tid; i0 < n; i0 += 8 * blockDim.x) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * blockDim.x;
                v[u] = i < n ? mT[(int64_t)(i / k2) * ldm + i % k2] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * blockDim.x;
                if (i < n) A[(i / k2) * ld + i % k2] = v[u];
            }
        }
    }
    for (int i = tid; i < k1; i += blockDim.x) mbar_init(bar + i, TPC);
    __syncthreads();

    if (c < k1) {
        double *colc = A + (size_t)c * ld;
        double part0 = 0.0, part1 = 0.0;
        if (c == 0)
            for (int r = 1 + q; r < k2; r += TPC) part0 = __fma_rn(colc[r], colc[r], part0);
        for (int j = 0; j < c; ++j) {
            mbar_wait(bar + j, 0);
            const double tj = s_tau[j], scal = s_scal[j];
            const bool last = j == c - 1;
            if (last) QR_T(c, 0);
            if (tj == 0.0) {
                if (last)
                    for (int r = c + 1 + q; r < k2; r += TPC) part0 = __fma_rn(colc[r], colc[r], part0);
                continue;
            }
            const double *colj = A + (size_t)j * ld;
            // w = v^T A[:,c] with v_j = 1, v_r = scal * colj[r]
            double w0 = 0.0, w1 = 0.0, w2 = 0.0, w3 = 0.0;
            int r = j + 1 + q;
            for (; r + 3 * TPC < k2; r += 4 * TPC) {
                const double a0 = colj[r], a1 = colj[r + TPC], a2 = colj[r + 2 * TPC],
                             a3 = colj[r + 3 * TPC];
                const double b0 = colc[r], b1 = colc[r + TPC], b2 = colc[r + 2 * TPC],
                             b3 = colc[r + 3 * TPC];
                w0 = __fma_rn(a0, b0, w0);
                w1 = __fma_rn(a1, b1, w1);
                w2 = __fma_rn(a2, b2, w2);
                w3 = __fma_rn(a3, b3, w3);
            }
            for (; r < k2; r += TPC) w0 = __fma_rn(colj[r], colc[r], w0);
            const double dot = group_sum<TPC>((w0 + w1) + (w2 + w3));
            if (last) QR_T(c, 1);
            const double f = tj * __fma_rn(scal, dot, colc[j]);
            const double fs = f * scal;
            __syncwarp(gmask);  // every lane has read colc[j]
            if (q == 0) colc[j] -= f;
            r = j + 1 + q;
            for (; r + 3 * TPC < k2; r += 4 * TPC) {
                const double a0 = colj[r], a1 = colj[r + TPC], a2 = colj[r + 2 * TPC],
                             a3 = colj[r + 3 * TPC];
                const double b0 = colc[r], b1 = colc[r + TPC], b2 = colc[r + 2 * TPC],
                             b3 = colc[r + 3 * TPC];
                const double n0 = __fma_rn(-fs, a0, b0), n1 = __fma_rn(-fs, a1, b1),
                             n2 = __fma_rn(-fs, a2, b2), n3 = __fma_rn(-fs, a3, b3);
                colc[r] = n0;
                colc[r + TPC] = n1;
                colc[r + 2 * TPC] = n2;
                colc[r + 3 * TPC] = n3;
                if (last) {
                    part0 = __fma_rn(n0, r == c ? 0.0 : n0, part0);
                    part1 = __fma_rn(n1, n1, part1);
                    part0 = __fma_rn(n2, n2, part0);
                    part1 = __fma_rn(n3, n3, part1);
                }
            }
            for (; r < k2; r += TPC) {
                const double nv = __fma_rn(-fs, colj[r], colc[r]);
                colc[r] = nv;
                if (last) part0 = __fma_rn(nv, r == c ? 0.0 : nv, part0);
            }
        }
        // reflector c
        QR_T(c, 2);
        const double part = group_sum<TPC>(part0 + part1);
        QR_T(c, 3);
        if (q == 0) dlarfg(colc, c, part, s_tau + c, s_scal + c);
        QR_T(c, 4);
        mbar_arrive(bar + c);
    }
    __syncthreads();
    for (int i = tid; i < k1; i += blockDim.x) qtau[i] = s_tau[i];
    // scale the stored reflectors: v_r = scal_j * u_r below the diagonal
    for (int i = tid; i < k1 * ld; i += blockDim.x) {
        const int cc = i / ld, r = i % ld;
        double v = A[i];
        if (r > cc && r < k2 && s_tau[cc] != 0.0) v *= s_scal[cc];
        qa[i] = v;
    }
    for (int i = tid; i < k1 * k1; i += blockDim.x) {  // R row-major (for the rank test)
        const int r = i / k1, cc = i % k1;
        rrow[i] = r <= cc ? A[cc * ld + r] : 0.0;
    }
}

// Phase 2 (many CTAs): every warp forms one column c of
// pinv^T = (R^-1 Q^T)^T: z = Q^T e_c (the k1 reflectors in order), then the
// back substitution R x = z[:k1].  The packed reflectors/R are staged in
// each CTA's shared memory and z lives in the lanes' registers (lane l owns
// rows r == l mod 32, PER per lane), so the 2·k1 sequential steps cost a
// warp reduction or a shuffle broadcast each, never a global round trip.
template <int PER>
__global__ void __launch_bounds__(256) qr_tail_kernel(const double *__restrict__ qa,
                                                      const double *__restrict__ qtau, int k1,
                                                      int k2, double *__restrict__ pinvT,
                                                      int64_t ldp) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int ld = k2 | 1;
    double *V = reinterpret_cast<double *>(smem_raw);  // k1 x ld, as qa
    double *tau = V + (size_t)k1 * ld;                  // qtau follows qa in the workspace
    __shared__ uint64_t tbar;
    (void)qtau;
    if (threadIdx.x == 0) {
        mbar_init(&tbar, 1);
        fence_mbar_init();
        // one bulk copy of reflectors + tau (rounded up to 16 B; the
        // workspace has slack after tau)
        const unsigned bytes = (unsigned)((sizeof(double) * ((size_t)k1 * ld + k1) + 15) & ~15ull);
        mbar_arrive_expect_tx(&tbar, bytes);
        bulk_g2s(V, qa, bytes, &tbar);
    }
    __syncthreads();
    mbar_wait(&tbar, 0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c = blockIdx.x * (blockDim.x >> 5) + warp;
    if (c >= k2) return;
    double z[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) z[i] = (i * 32 + lane == c) ? 1.0 : 0.0;
    for (int j = 0; j < k1; ++j) {
        const double tj = tau[j];
        if (tj == 0.0) continue;
        const double *vj = V + (size_t)j * ld;
        double w = 0.0;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int r = i * 32 + lane;
            const double v = r == j ? 1.0 : (r > j && r < k2 ? vj[r] : 0.0);
            w = __fma_rn(v, z[i], w);
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) w += __shfl_xor_sync(0xffffffffu, w, off);
        const double f = tj * w;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int r = i * 32 + lane;
            const double v = r == j ? 1.0 : (r > j && r < k2 ? vj[r] : 0.0);
            z[i] = __fma_rn(-f, v, z[i]);
        }
    }
    // back substitution on the first k1 entries: R x = z
    for (int r = k1 - 1; r >= 0; --r) {
        const double *rc = V + (size_t)r * ld;  // column r of R (rows < r)
        const int ro = r & 31, ri = r >> 5;
        double zr = 0.0;
#pragma unroll
        for (int i = 0; i < PER; ++i)
            if (i == ri) zr = z[i];
        const double xr = __shfl_sync(0xffffffffu, zr, ro) / rc[r];
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int q = i * 32 + lane;
            if (q < r) z[i] = __fma_rn(-rc[q], xr, z[i]);
            if (i == ri && lane == ro) z[i] = xr;
        }
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int q = i * 32 + lane;
        if (q < k1) pinvT[(int64_t)c * ldp + q] = z[i];
    }
}

// the same for any k2 (z in shared memory): used when k2 > 32 * kTailMaxPer
__global__ void __launch_bounds__(256) qr_tail_any_kernel(const double *__restrict__ qa,
                                                          const double *__restrict__ qtau,
                                                          int k1, int k2,
                                                          double *__restrict__ pinvT,
                                                          int64_t ldp) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int ld = k2 | 1;
    const int k2p = (k2 + 1) & ~1;
    double *sm = reinterpret_cast<double *>(smem_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c = blockIdx.x * (blockDim.x >> 5) + warp;
    if (c >= k2) return;
    double *z = sm + (size_t)warp * k2p;
    for (int r = lane; r < k2; r += 32) z[r] = (r == c) ? 1.0 : 0.0;
    __syncwarp();
    for (int j = 0; j < k1; ++j) {
        const double tj = qtau[j];
        if (tj == 0.0) continue;
        const double *colj = qa + (size_t)j * ld;
        double w = lane == 0 ? z[j] : 0.0;
        for (int r = j + 1 + lane; r < k2; r += 32) w += colj[r] * z[r];
#pragma unroll
        for (int off = 16; off; off >>= 1) w += __shfl_xor_sync(0xffffffffu, w, off);
        const double f = tj * w;
        __syncwarp();
        if (lane == 0) z[j] -= f;
        for (int r = j + 1 + lane; r < k2; r += 32) z[r] -= f * colj[r];
        __syncwarp();
    }
    for (int i = k1 - 1; i >= 0; --i) {
        const double zi = z[i] / qa[(size_t)i * ld + i];
        __syncwarp();
        for (int r = lane; r < i; r += 32) z[r] -= qa[(size_t)i * ld + r] * zi;
        if (lane == 0) z[i] = zi;
        __syncwarp();
    }
    for (int i = lane; i < k1; i += 32) pinvT[(int64_t)c * ldp + i] = z[i];
}

__global__ void __launch_bounds__(256, 1) rank_estimate_kernel(const double *__restrict__ R,
                                                                      int k, int64_t ldr,
                                                                      const double *__restrict__ RT,
                                                                      int64_t ldt,
                                                                      double *__restrict__ stats,
                                                                      const double *__restrict__ pinvT,
                                                                      int64_t ldp, int k2) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *xv = reinterpret_cast<double *>(smem_raw);
    double *yv = xv + k;
    double *red = yv + k;
    rank_estimate(R, ldr, RT, ldt, k, xv, yv, red, stats, pinvT, ldp, k2);
}


static size_t qr_pinv_smem(int64_t k1, int64_t k2) {
    const int64_t ld = k2 | 1;
    return sizeof(double) * (size_t)(k1 * ld + 3 * k1) + 64;
}

}  // namespace srlu

using namespace srlu;

extern "C" size_t srlu_qr_pinv_smem_bytes(int64_t k1, int64_t k2) { return qr_pinv_smem(k1, k2); }

// Lookahead variant (k1 * TPC + 32 <= 1024): warp 0 runs the critical
// chain alone — for column c it applies reflector c-1 and forms reflector c
// (32 lanes on one column, warp-level sums) — while the group of TPC
// threads that owns column c applies reflectors 0..c-2 in the background
// and then hands the column to warp 0 (mbarrier rdy[c]).  In qr_kernel the
// critical column's group shares its warp with three other columns'
// groups (divergent paths issue one at a time) and its scheduler with
// every spinning waiter; here the chain has a warp of its own and the
// background waits suspend.  Same reflector conventions as qr_kernel.
template <int TPC>
__global__ void __launch_bounds__(1024, 1) qr_la_kernel(const double *__restrict__ mT, int k1,
                                                        int k2, int64_t ldm,
                                                        double *__restrict__ qa,
                                                        double *__restrict__ qtau,
                                                        double *__restrict__ rrow, int depth) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int ld = k2 | 1;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw);           // k1: reflector formed
    double *s_tau = reinterpret_cast<double *>(smem_raw) + k1;        // k1
    double *s_scal = s_tau + k1;                                      // k1
    double *A = s_scal + k1;                                          // column c: A[c*ld + r]
    uint64_t *rdy = reinterpret_cast<uint64_t *>(A + (size_t)k1 * ld);  // k1: background done
    const int tid = threadIdx.x;
    {
        const int n = k1 * k2;
        for (int i0 = tid; i0 < n; i0 += 8 * blockDim.x) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * blockDim.x;
                v[u] = i < n ? mT[(int64_t)(i / k2) * ldm + i % k2] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * blockDim.x;
                if (i < n) A[(i / k2) * ld + i % k2] = v[u];
            }
        }
    }
    for (int i = tid; i < k1; i += blockDim.x) {
        mbar_init(bar + i, 32);
        mbar_init(rdy + i, TPC);
    }
    __syncthreads();

    if (tid < 32) {
        // ---- the critical chain ----
        const int lane = tid;
        for (int c = 0; c < k1; ++c) {
            double *colc = A + (size_t)c * ld;
            double p0 = 0.0, p1 = 0.0;
            if (c > 0) mbar_wait(rdy + c, 0);
            // reflectors c-depth .. c-2 (the background applied the earlier ones)
            for (int j = max(0, c - depth); j + 1 < c; ++j) {
                const double tq = s_tau[j];
                if (tq == 0.0) continue;
                const double scal = s_scal[j];
                const double *colj = A + (size_t)j * ld;
                double w0 = 0.0, w1 = 0.0;
                int r = j + 1 + lane;
                for (; r + 32 < k2; r += 64) {
                    w0 = __fma_rn(colj[r], colc[r], w0);
                    w1 = __fma_rn(colj[r + 32], colc[r + 32], w1);
                }
                if (r < k2) w0 = __fma_rn(colj[r], colc[r], w0);
                const double dot = group_sum<32>(w0 + w1);
                const double f = tq * __fma_rn(scal, dot, colc[j]);
                const double fs = f * scal;
                __syncwarp();
                if (lane == 0) colc[j] -= f;
                for (r = j + 1 + lane; r < k2; r += 32) colc[r] = __fma_rn(-fs, colj[r], colc[r]);
                __syncwarp();
            }
            const double tj = c > 0 ? s_tau[c - 1] : 0.0;
            if (c > 0 && tj != 0.0) {
                const int j = c - 1;
                const double scal = s_scal[j];
                const double *colj = A + (size_t)j * ld;
                double w0 = 0.0, w1 = 0.0;
                int r = j + 1 + lane;
                for (; r + 32 < k2; r += 64) {
                    w0 = __fma_rn(colj[r], colc[r], w0);
                    w1 = __fma_rn(colj[r + 32], colc[r + 32], w1);
                }
                if (r < k2) w0 = __fma_rn(colj[r], colc[r], w0);
                const double dot = group_sum<32>(w0 + w1);
                const double f = tj * __fma_rn(scal, dot, colc[j]);
                const double fs = f * scal;
                __syncwarp();  // every lane has read colc[j]
                if (lane == 0) colc[j] -= f;
                for (r = j + 1 + lane; r < k2; r += 32) {
                    const double nv = __fma_rn(-fs, colj[r], colc[r]);
                    colc[r] = nv;
                    if (r > c) {
                        if (r & 32) p1 = __fma_rn(nv, nv, p1);
                        else p0 = __fma_rn(nv, nv, p0);
                    }
                }
            } else {
                for (int r = c + 1 + lane; r < k2; r += 32) p0 = __fma_rn(colc[r], colc[r], p0);
            }
            const double part = group_sum<32>(p0 + p1);
            __syncwarp();
            if (lane == 0) dlarfg(colc, c, part, s_tau + c, s_scal + c);
            __syncwarp();
            mbar_arrive(bar + c);
        }
    } else {
        // ---- background: column c gets reflectors 0..c-2 ----
        const int g = (tid - 32) / TPC, q = (tid - 32) % TPC;
        const unsigned gmask = (TPC == 32 ? 0xffffffffu
                                          : ((1u << TPC) - 1u) << ((tid & 31) & ~(TPC - 1)));
        const int c = g;
        if (c < k1) {
            double *colc = A + (size_t)c * ld;
            for (int j = 0; j < c - depth; ++j) {
                mbar_wait_suspend(bar + j, 0);
                const double tj = s_tau[j];
                if (tj == 0.0) continue;
                const double scal = s_scal[j];
                const double *colj = A + (size_t)j * ld;
                double w0 = 0.0, w1 = 0.0, w2 = 0.0, w3 = 0.0;
                int r = j + 1 + q;
                for (; r + 3 * TPC < k2; r += 4 * TPC) {
                    w0 = __fma_rn(colj[r], colc[r], w0);
                    w1 = __fma_rn(colj[r + TPC], colc[r + TPC], w1);
                    w2 = __fma_rn(colj[r + 2 * TPC], colc[r + 2 * TPC], w2);
                    w3 = __fma_rn(colj[r + 3 * TPC], colc[r + 3 * TPC], w3);
                }
                for (; r < k2; r += TPC) w0 = __fma_rn(colj[r], colc[r], w0);
                const double dot = group_sum<TPC>((w0 + w1) + (w2 + w3));
                const double f = tj * __fma_rn(scal, dot, colc[j]);
                const double fs = f * scal;
                __syncwarp(gmask);
                if (q == 0) colc[j] -= f;
                for (r = j + 1 + q; r < k2; r += TPC) colc[r] = __fma_rn(-fs, colj[r], colc[r]);
            }
            mbar_arrive(rdy + c);
        }
    }
    __syncthreads();
    for (int i = tid; i < k1; i += blockDim.x) qtau[i] = s_tau[i];
    for (int i = tid; i < k1 * ld; i += blockDim.x) {
        const int cc = i / ld, r = i % ld;
        double v = A[i];
        if (r > cc && r < k2 && s_tau[cc] != 0.0) v *= s_scal[cc];
        qa[i] = v;
    }
    for (int i = tid; i < k1 * k1; i += blockDim.x) {
        const int r = i / k1, cc = i % k1;
        rrow[i] = r <= cc ? A[cc * ld + r] : 0.0;
    }
}

// Register-resident variant (k2 <= 8 * RPT, k1 <= 128): the 8 threads of
// column c's group keep its rows q, q + 8, ... in registers for the whole
// sweep; shared memory only carries each reflector once it is formed (the
// groups of a warp read the same reflector words: broadcast), so the
// trailing columns no longer stream their own data through shared memory
// and the critical chain (apply reflector c-1, form reflector c) competes
// for far fewer shared-memory cycles.  Same dataflow and dlarfg
// conventions as qr_kernel (not the same summation order: the QR is
// compared with LAPACK's to tolerance anyway).
template <int RPT>
__device__ __forceinline__ double pick_reg(const double (&v)[RPT], int idx) {
    double x = 0.0;
#pragma unroll
    for (int i = 0; i < RPT; ++i) x = (i == idx) ? v[i] : x;
    return x;
}

template <int RPT>
__global__ void __launch_bounds__(1024, 1) qr_reg_kernel(const double *__restrict__ mT, int k1,
                                                         int k2, int64_t ldm,
                                                         double *__restrict__ qa,
                                                         double *__restrict__ qtau,
                                                         double *__restrict__ rrow) {
    constexpr int TPC = 8;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int ld = k2 | 1;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw);           // k1 mbarriers
    double *s_tau = reinterpret_cast<double *>(smem_raw) + k1;        // k1
    double *s_scal = s_tau + k1;                                      // k1
    double *A = s_scal + k1;  // column c: A[c*ld + r] (reflectors, then the result)
    const int tid = threadIdx.x;
    const int c = tid / TPC, q = tid % TPC;
    const unsigned gmask = ((1u << TPC) - 1u) << ((tid & 31) & ~(TPC - 1));
    for (int i = tid; i < k1; i += blockDim.x) mbar_init(bar + i, TPC);
    double v[RPT];
    if (c < k1) {
        const double *src = mT + (int64_t)c * ldm;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int r = q + TPC * i;
            v[i] = r < k2 ? __ldg(src + r) : 0.0;
        }
    }
    __syncthreads();
    if (c < k1) {
        // element of row rr: lane rr % TPC of the group, register rr / TPC
#define QR_ROW_VAL(out, rr) \
    out = __shfl_sync(gmask, pick_reg<RPT>(v, (rr) / TPC), (tid & 31 & ~(TPC - 1)) + (rr) % TPC)
        for (int j = 0; j < c; ++j) {
            mbar_wait(bar + j, 0);
            const double tj = s_tau[j];
            if (tj == 0.0) continue;
            const double scal = s_scal[j];
            const double *colj = A + (size_t)j * ld;
            double w0 = 0.0, w1 = 0.0;
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const int r = q + TPC * i;
                if (r > j && r < k2) {
                    if (i & 1) w1 = __fma_rn(colj[r], v[i], w1);
                    else w0 = __fma_rn(colj[r], v[i], w0);
                }
            }
            const double dot = group_sum<TPC>(w0 + w1);
            double vj;
            QR_ROW_VAL(vj, j);
            const double f = tj * __fma_rn(scal, dot, vj);
            const double fs = f * scal;
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const int r = q + TPC * i;
                if (r == j) v[i] -= f;
                else if (r > j && r < k2) v[i] = __fma_rn(-fs, colj[r], v[i]);
            }
        }
        // reflector c from rows > c, alpha = row c
        double p0 = 0.0, p1 = 0.0;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int r = q + TPC * i;
            if (r > c && r < k2) {
                if (i & 1) p1 = __fma_rn(v[i], v[i], p1);
                else p0 = __fma_rn(v[i], v[i], p0);
            }
        }
        const double part = group_sum<TPC>(p0 + p1);
        double alpha;
        QR_ROW_VAL(alpha, c);
#undef QR_ROW_VAL
        double t = 0.0, scal = 0.0, beta = alpha;
        if (part > 0.0) {
            beta = -copysign(sqrt(__fma_rn(alpha, alpha, part)), alpha);
            t = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        }
        double *colc = A + (size_t)c * ld;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int r = q + TPC * i;
            if (r == c) v[i] = beta;
            if (r < k2) colc[r] = v[i];  // rows < c: R (final); > c: the reflector
        }
        if (q == 0) {
            s_tau[c] = t;
            s_scal[c] = scal;
        }
        mbar_arrive(bar + c);
    }
    __syncthreads();
    for (int i = tid; i < k1; i += blockDim.x) qtau[i] = s_tau[i];
    for (int i = tid; i < k1 * ld; i += blockDim.x) {
        const int cc = i / ld, r = i % ld;
        double x = A[i];
        if (r > cc && r < k2 && s_tau[cc] != 0.0) x *= s_scal[cc];
        qa[i] = x;
    }
    for (int i = tid; i < k1 * k1; i += blockDim.x) {
        const int r = i / k1, cc = i % k1;
        rrow[i] = r <= cc ? A[cc * ld + r] : 0.0;
    }
}

extern "C" size_t srlu_qr_pinv_workspace(int64_t k1, int64_t k2) {
    return sizeof(double) * (size_t)(k1 * (k2 | 1) + k1 + k1 * k1) + 256;
}

extern "C" int srlu_qr_pinv(const double *mT, int64_t k1, int64_t k2, int64_t ldm, double *pinvT,
                            int64_t ldp, double *stats, void *ws, size_t ws_bytes,
                            srlu_stream_t stream) {
    SRLU_REQUIRE(k1 >= 1 && k2 >= k1 && ldm >= k2 && ldp >= k1, SRLU_ERR_ARG,
                 "left_pseudo_inverse: need rows >= cols, got %lld x %lld", (long long)k2,
                 (long long)k1);
    SRLU_REQUIRE(ws_bytes >= srlu_qr_pinv_workspace(k1, k2), SRLU_ERR_WORKSPACE,
                 "qr_pinv: workspace too small");
    size_t smem = qr_pinv_smem(k1, k2);
    cudaStream_t s = (cudaStream_t)stream;
    double *qa = (double *)ws;
    double *qtau = qa + (size_t)k1 * (k2 | 1);
    double *rrow = qtau + k1;
    const char *qv = getenv("SRLU_QR");  // testing knob: smem | reg | cluster
    if (smem > 220 * 1024 || k1 > 256 || (qv && !strcmp(qv, "cluster"))) {
        // M does not fit one CTA: the cluster QR (qr_cluster.cu)
        SRLU_REQUIRE(k1 <= 32 * kRankMaxPerLane, SRLU_ERR_UNSUPPORTED, "qr_pinv: k1 > %d",
                     32 * kRankMaxPerLane);
        const int rc0 = qr_cluster_launch(mT, k1, k2, ldm, qa, qtau, rrow, s);
        if (rc0 != SRLU_OK) return rc0;
    } else {  // one group of 8 (k1 <= 128) or 4 threads per column; register-resident
       // columns when they fit 16 registers per thread
        void (*qr)(const double *, int, int, int64_t, double *, double *, double *) =
            k1 <= 128 ? qr_kernel<8> : qr_kernel<4>;
        if (k1 <= 128 && k2 <= 128 && qv && !strcmp(qv, "reg")) qr = qr_reg_kernel<16>;
        else if (k1 * 8 + 32 <= 1024 && !(qv && !strcmp(qv, "smem"))) {
            qr = nullptr;  // qr_la_kernel<8>
            smem += sizeof(uint64_t) * (size_t)k1;
        }
        SRLU_REQUIRE(k1 <= 256, SRLU_ERR_UNSUPPORTED, "qr_pinv: k1 > 256");
        if (qr == nullptr)
            SRLU_CUDA(cudaFuncSetAttribute(qr_la_kernel<8>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        else
            SRLU_CUDA(cudaFuncSetAttribute(qr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        if (qr == nullptr) {
            const char *dv = getenv("SRLU_QR_DEPTH");  // testing knob
            const int depth = dv ? atoi(dv) : 1;  // measured: 1 < 2 < 3 < 4 (tools/time_qr.py)
            SRLU_REQUIRE(depth >= 1, SRLU_ERR_ARG, "qr_pinv: SRLU_QR_DEPTH must be >= 1");
            qr_la_kernel<8><<<1, 1024, smem, s>>>(mT, (int)k1, (int)k2, ldm, qa, qtau, rrow, depth);
        } else {
            qr<<<1, 1024, smem, s>>>(mT, (int)k1, (int)k2, ldm, qa, qtau, rrow);
        }
    }
    SRLU_CHECK_LAUNCH("qr_kernel");
    const unsigned tail_grid = (unsigned)ceil_div(k2, 8);
    const size_t smem_v = sizeof(double) * (size_t)(k1 * (k2 | 1) + k1) + 64;  // +16 B round-up
    auto tail = [&](auto kern) -> int {
        SRLU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem_v));
        kern<<<tail_grid, 256, smem_v, s>>>(qa, qtau, (int)k1, (int)k2, pinvT, ldp);
        return SRLU_OK;
    };
    int rc;
    if (smem_v > 220 * 1024) rc = SRLU_ERR_UNSUPPORTED;  // reflectors do not fit: any-k2 tail
    else if (k2 <= 32) rc = tail(qr_tail_kernel<1>);
    else if (k2 <= 64) rc = tail(qr_tail_kernel<2>);
    else if (k2 <= 128) rc = tail(qr_tail_kernel<4>);
    else if (k2 <= 192) rc = tail(qr_tail_kernel<6>);
    else if (k2 <= 32 * kTailMaxPer) rc = tail(qr_tail_kernel<kTailMaxPer>);
    else rc = SRLU_ERR_UNSUPPORTED;
    if (rc == SRLU_ERR_UNSUPPORTED) {
        const size_t smem2 = sizeof(double) * (size_t)(8 * ((k2 + 1) & ~1) + 64);
        SRLU_REQUIRE(smem2 <= 200 * 1024, SRLU_ERR_UNSUPPORTED, "qr_pinv: k2 too large");
        SRLU_CUDA(cudaFuncSetAttribute(qr_tail_any_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
        qr_tail_any_kernel<<<tail_grid, 256, smem2, s>>>(qa, qtau, (int)k1, (int)k2, pinvT, ldp);
        rc = SRLU_OK;
    }
    if (rc != SRLU_OK) return rc;
    SRLU_CHECK_LAUNCH("qr_tail_kernel");
    return SRLU_OK;
}

extern "C" int srlu_rank_estimate(const double *R, int64_t k, int64_t ldr, const double *RT,
                                  int64_t ldt, double *stats, srlu_stream_t stream) {
    SRLU_REQUIRE(k >= 1 && ldr >= k && ldt >= k, SRLU_ERR_ARG, "rank_estimate: bad sizes");
    SRLU_REQUIRE(k <= 32 * kRankMaxPerLane, SRLU_ERR_UNSUPPORTED, "rank_estimate: k > 576");
    size_t smem = sizeof(double) * (size_t)(2 * k + 64);
    SRLU_REQUIRE(smem <= 200 * 1024, SRLU_ERR_UNSUPPORTED, "rank_estimate: k too large");
    SRLU_CUDA(cudaFuncSetAttribute(rank_estimate_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // max shared carveout: the rank test overlaps the column-pivot LU, whose
    // ~200 KB CTAs must still land on the SM this CTA occupies
    SRLU_CUDA(cudaFuncSetAttribute(rank_estimate_kernel,
                                   cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    rank_estimate_kernel<<<1, 256, smem, (cudaStream_t)stream>>>(R, (int)k, ldr, RT, ldt,
                                                                         stats, nullptr, 0, 0);
    SRLU_CHECK_LAUNCH("rank_estimate_kernel");
    return SRLU_OK;
}


extern "C" int srlu_qr_rank(const void *ws, int64_t k1, int64_t k2, double *stats,
                            srlu_stream_t stream) {
    SRLU_REQUIRE(k1 >= 1 && k2 >= k1 && k1 <= 32 * kRankMaxPerLane, SRLU_ERR_ARG,
                 "qr_rank: bad sizes");
    const double *qa = (const double *)ws;
    const double *rrow = qa + (size_t)k1 * (k2 | 1) + k1;
    size_t smem = sizeof(double) * (size_t)(2 * k1 + 64);
    SRLU_CUDA(cudaFuncSetAttribute(rank_estimate_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // max shared carveout: the rank test overlaps the column-pivot LU, whose
    // ~200 KB CTAs must still land on the SM this CTA occupies
    SRLU_CUDA(cudaFuncSetAttribute(rank_estimate_kernel,
                                   cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    // R row-major = rrow, R column-major = the packed QR (column stride k2|1)
    rank_estimate_kernel<<<1, 256, smem, (cudaStream_t)stream>>>(rrow, (int)k1, k1, qa,
                                                                 (int64_t)(k2 | 1), stats,
                                                                 nullptr, 0, 0);
    SRLU_CHECK_LAUNCH("rank_estimate_kernel");
    return SRLU_OK;
}

extern "C" int srlu_qr_rank_certified(const void *ws, int64_t k1, int64_t k2, const double *pinvT,
                                      int64_t ldp, double *stats, srlu_stream_t stream) {
    SRLU_REQUIRE(k1 >= 1 && k2 >= k1 && k1 <= 32 * kRankMaxPerLane && ldp >= k1 && pinvT,
                 SRLU_ERR_ARG, "qr_rank: bad sizes");
    const double *qa = (const double *)ws;
    const double *rrow = qa + (size_t)k1 * (k2 | 1) + k1;
    size_t smem = sizeof(double) * (size_t)(2 * k1 + 64);
    SRLU_CUDA(cudaFuncSetAttribute(rank_estimate_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SRLU_CUDA(cudaFuncSetAttribute(rank_estimate_kernel,
                                   cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    rank_estimate_kernel<<<1, 256, smem, (cudaStream_t)stream>>>(rrow, (int)k1, k1, qa,
                                                                 (int64_t)(k2 | 1), stats,
                                                                 pinvT, ldp, (int)k2);
    SRLU_CHECK_LAUNCH("rank_estimate_kernel");
    return SRLU_OK;
}

extern "C" size_t srlu_rank_exact_workspace(int64_t k1) { return jacobi_workspace(k1); }

extern "C" int srlu_rank_exact(const void *qr_ws, int64_t k1, int64_t k2, void *ws,
                               size_t ws_bytes, double *stats, srlu_stream_t stream) {
    SRLU_REQUIRE(k1 >= 1 && k2 >= k1, SRLU_ERR_ARG, "rank_exact: bad sizes");
    SRLU_REQUIRE(ws && ws_bytes >= jacobi_workspace(k1), SRLU_ERR_WORKSPACE,
                 "rank_exact: workspace too small");
    const double *rrow = (const double *)qr_ws + (size_t)k1 * (k2 | 1) + k1;
    int rc = jacobi_launch(rrow, k1, ws, stats, (cudaStream_t)stream);
    if (rc) return rc;
    SRLU_CHECK_LAUNCH("jacobi_sv_kernel");
    return SRLU_OK;
}
