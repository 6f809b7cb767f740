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
//  * srlu_dgemm: C = A·B row-major fp64 SIMT-FMA GEMM for the skinny core
//    and L products (cuBLAS picks a 32x32 DMMA tile that reached <3 TFLOP/s
//    on the 16384x118x110 shape).
#include <math.h>

#include "common.cuh"

namespace srlu {

constexpr int kQrThreads = 512;
constexpr int kQrWarps = kQrThreads / 32;
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
                              double *y, double *red, double *stats) {
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
    if (tid == 0) {
        stats[0] = smax;
        stats[1] = smin;
        stats[2] = smin > 0.0 ? smax / smin : INFINITY;
        stats[3] = (smax == 0.0 || smin <= kRankRtol * smax) ? 1.0 : 0.0;
    }
}

// Phase 1 (one CTA): Householder QR of M in shared memory; the packed
// reflectors/R (column-major, stride ld) and tau go to global memory.
// Reflector j is formed by warp 0 (norm + dlarfg); applying it to the
// trailing columns is one thread per column (dot + axpy over the column).
__global__ void __launch_bounds__(kQrThreads, 1) qr_kernel(const double *__restrict__ mT, int k1,
                                                           int k2, int64_t ldm,
                                                           double *__restrict__ qa,
                                                           double *__restrict__ qtau,
                                                           double *__restrict__ rrow) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int ld = k2 | 1;
    double *A = reinterpret_cast<double *>(smem_raw);  // column c: A[c*ld + r] = M[r][c]
    __shared__ double s_tau, s_scal;
    const int tid = threadIdx.x, lane = tid & 31;

    for (int i = tid; i < k1 * k2; i += blockDim.x) {
        const int c = i / k2, r = i % k2;
        A[c * ld + r] = mT[(int64_t)c * ldm + r];
    }
    __syncthreads();
    for (int j = 0; j < k1; ++j) {
        double *colj = A + j * ld;
        if (tid < 32) {  // dlarfg on column j (warp 0)
            double part = 0.0;
            for (int r = j + 1 + lane; r < k2; r += 32) part += colj[r] * colj[r];
#pragma unroll
            for (int off = 16; off; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
            if (lane == 0) {
                const double alpha = colj[j];
                double t = 0.0, scal = 0.0;
                if (part > 0.0) {
                    const double beta = -copysign(hypot(alpha, sqrt(part)), alpha);
                    t = (beta - alpha) / beta;
                    scal = 1.0 / (alpha - beta);
                    colj[j] = beta;
                }
                s_tau = t;
                s_scal = scal;
                qtau[j] = t;
            }
        }
        __syncthreads();
        const double tj = s_tau, scal = s_scal;
        if (tj != 0.0) {
            // 4 threads per trailing column c: w = v^T A[:,c] (v_j = 1,
            // v_r = scal*colj[r]), quad-shuffle reduction, then the update
            const int q = tid & 3;
            for (int c = j + 1 + (tid >> 2); c < k1; c += blockDim.x >> 2) {
                double *colc = A + c * ld;
                double w0 = q == 0 ? colc[j] : 0.0, w1 = 0.0;
                int r = j + 1 + q;
                for (; r + 4 < k2; r += 8) {
                    w0 = __fma_rn(colj[r] * scal, colc[r], w0);
                    w1 = __fma_rn(colj[r + 4] * scal, colc[r + 4], w1);
                }
                for (; r < k2; r += 4) w0 = __fma_rn(colj[r] * scal, colc[r], w0);
                double w = w0 + w1;
                const unsigned qmask = 0xFu << ((threadIdx.x & 31) & ~3);  // the quad
                w += __shfl_xor_sync(qmask, w, 1);
                w += __shfl_xor_sync(qmask, w, 2);
                const double f = tj * w;
                if (q == 0) colc[j] -= f;
                for (int rr = j + 1 + q; rr < k2; rr += 4) colc[rr] = __fma_rn(-f, colj[rr] * scal, colc[rr]);
            }
        }
        __syncthreads();
        if (tj != 0.0)
            for (int r = j + 1 + tid; r < k2; r += blockDim.x) colj[r] *= scal;
        __syncthreads();
    }
    for (int i = tid; i < k1 * ld; i += blockDim.x) qa[i] = A[i];
    for (int i = tid; i < k1 * k1; i += blockDim.x) {  // R row-major (for the rank test)
        const int r = i / k1, c = i % k1;
        rrow[i] = r <= c ? A[c * ld + r] : 0.0;
    }
}

// Phase 2 (many CTAs): CTA 0 runs the rank test on R; every warp of the
// other CTAs forms one column of pinv^T = (R^-1 Q^T)^T from the reflectors.
__global__ void __launch_bounds__(256) qr_tail_kernel(const double *__restrict__ qa,
                                                      const double *__restrict__ qtau, int k1,
                                                      int k2, double *__restrict__ pinvT,
                                                      int64_t ldp, double *__restrict__ stats,
                                                      const double *__restrict__ rrow) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int ld = k2 | 1;
    const int k2p = (k2 + 1) & ~1;
    double *sm = reinterpret_cast<double *>(smem_raw);
    (void)stats;
    (void)rrow;
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
                                                                      double *__restrict__ stats) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *xv = reinterpret_cast<double *>(smem_raw);
    double *yv = xv + k;
    double *red = yv + k;
    rank_estimate(R, ldr, RT, ldt, k, xv, yv, red, stats);
}

// ---------------------------------------------------------------------------
// C (M x N) = A (M x K) . B (K x N), row-major fp64, FMA.

constexpr int kGemmBM = 64, kGemmBN = 64, kGemmBK = 16;

__global__ void __launch_bounds__(256) dgemm_kernel(const double *__restrict__ A, int64_t lda,
                                                    const double *__restrict__ B, int64_t ldb,
                                                    double *__restrict__ C, int64_t ldc,
                                                    int64_t M, int N, int K) {
    __shared__ double As[kGemmBK][kGemmBM + 2];
    __shared__ double Bs[kGemmBK][kGemmBN + 2];
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;
    const int64_t m0 = (int64_t)blockIdx.x * kGemmBM;
    const int n0 = blockIdx.y * kGemmBN;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int k0 = 0; k0 < K; k0 += kGemmBK) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int e = tid + i * 256;  // 0..1023
            const int am = e / kGemmBK, ak = e % kGemmBK;
            const int64_t gm = m0 + am;
            const int gk = k0 + ak;
            As[ak][am] = (gm < M && gk < K) ? A[gm * lda + gk] : 0.0;
            const int bk = e / kGemmBN, bn = e % kGemmBN;
            const int gk2 = k0 + bk, gn = n0 + bn;
            Bs[bk][bn] = (gk2 < K && gn < N) ? B[(int64_t)gk2 * ldb + gn] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kGemmBK; ++kk) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __fma_rn(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t gm = m0 + ty * 4 + i;
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gn = n0 + tx + 16 * j;
            if (gn < N) C[gm * ldc + gn] = acc[i][j];
        }
    }
}

static size_t qr_pinv_smem(int64_t k1, int64_t k2) {
    const int64_t ld = k2 | 1;
    return sizeof(double) * (size_t)(k1 * ld) + 64;
}

}  // namespace srlu

using namespace srlu;

extern "C" size_t srlu_qr_pinv_smem_bytes(int64_t k1, int64_t k2) { return qr_pinv_smem(k1, k2); }

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
    SRLU_REQUIRE(smem <= 220 * 1024, SRLU_ERR_UNSUPPORTED,
                 "qr_pinv: %lld x %lld does not fit one CTA's shared memory", (long long)k2,
                 (long long)k1);
    cudaStream_t s = (cudaStream_t)stream;
    double *qa = (double *)ws;
    double *qtau = qa + (size_t)k1 * (k2 | 1);
    double *rrow = qtau + k1;
    SRLU_CUDA(cudaFuncSetAttribute(qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    qr_kernel<<<1, kQrThreads, smem, s>>>(mT, (int)k1, (int)k2, ldm, qa, qtau, rrow);
    SRLU_CHECK_LAUNCH("qr_kernel");
    const int k2p = (int)((k2 + 1) & ~1);
    size_t smem2 = sizeof(double) * (size_t)(8 * k2p + 64);
    size_t smem_rank = sizeof(double) * (size_t)(3 * k2p + 64);
    if (smem_rank > smem2) smem2 = smem_rank;
    SRLU_CUDA(cudaFuncSetAttribute(qr_tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem2));
    qr_tail_kernel<<<(unsigned)ceil_div(k2, 8), 256, smem2, s>>>(qa, qtau, (int)k1, (int)k2,
                                                                       pinvT, ldp, stats, rrow);
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
                                                                         stats);
    SRLU_CHECK_LAUNCH("rank_estimate_kernel");
    return SRLU_OK;
}

extern "C" int srlu_dgemm(const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                          int64_t ldc, int64_t M, int64_t N, int64_t K, srlu_stream_t stream) {
    SRLU_REQUIRE(M >= 0 && N >= 0 && K >= 0 && N < (1 << 30) && K < (1 << 30), SRLU_ERR_ARG,
                 "dgemm: bad sizes");
    if (M == 0 || N == 0) return SRLU_OK;
    dim3 grid((unsigned)ceil_div(M, kGemmBM), (unsigned)ceil_div(N, kGemmBN));
    dgemm_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(A, lda, B, ldb, C, ldc, M, (int)N, (int)K);
    SRLU_CHECK_LAUNCH("dgemm_kernel");
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
                                                                 (int64_t)(k2 | 1), stats);
    SRLU_CHECK_LAUNCH("rank_estimate_kernel");
    return SRLU_OK;
}
