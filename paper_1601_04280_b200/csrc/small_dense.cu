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

// R accessor: upper triangle R(r, c), r <= c
struct RSmem {  // column-major with stride ld (the QR workspace)
    const double *a;
    int ld;
    __device__ double operator()(int r, int c) const { return a[c * ld + r]; }
};
struct RGlobalRowMajor {
    const double *a;
    int64_t ld;
    __device__ double operator()(int r, int c) const { return a[(int64_t)r * ld + c]; }
};

// stats[0] = sigma_max estimate, [1] = sigma_min estimate, [2] = cond, [3] = singular flag
template <typename RA>
__device__ void rank_estimate(RA R, int k, double *x, double *y, double *rinv, double *red,
                              double *stats) {
    const int tid = threadIdx.x;
    double dmax = 0.0, dmin = INFINITY;
    for (int j = tid; j < k; j += blockDim.x) {
        double d = fabs(R(j, j));
        dmax = fmax(dmax, d);
        dmin = fmin(dmin, d);
    }
    dmax = block_max(dmax, red);
    dmin = block_min(dmin, red);
    double smax = dmax, smin = dmin;
    const double inv_sqrt_k = 1.0 / sqrt((double)k);
    // power iteration: sigma_max >= ||R x|| for unit x
    for (int j = tid; j < k; j += blockDim.x) x[j] = inv_sqrt_k;
    __syncthreads();
    for (int it = 0; it < 6 && dmax > 0.0; ++it) {
        double ss = 0.0;
        for (int r = tid; r < k; r += blockDim.x) {
            double s = 0.0;
            for (int c = r; c < k; ++c) s += R(r, c) * x[c];
            y[r] = s;
            ss += s * s;
        }
        ss = block_sum(ss, red);
        smax = fmax(smax, sqrt(ss));
        double zz = 0.0;
        for (int c = tid; c < k; c += blockDim.x) {
            double s = 0.0;
            for (int r = 0; r <= c; ++r) s += R(r, c) * y[r];
            x[c] = s;  // y is complete (synced by block_sum)
            zz += s * s;
        }
        zz = block_sum(zz, red);
        const double inv = zz > 0.0 ? 1.0 / sqrt(zz) : 0.0;
        for (int c = tid; c < k; c += blockDim.x) x[c] *= inv;
        __syncthreads();
    }
    // inverse iteration: sigma_min <= ||(R^T R)^-1 x||^(-1/2) for unit x;
    // the triangular solves run on warp 0 only (syncwarp per step)
    if (dmin > 0.0) {
        if (tid < 32) {
            const int lane = tid;
            for (int j = lane; j < k; j += 32) {
                x[j] = ((j & 1) ? -inv_sqrt_k : inv_sqrt_k);
                rinv[j] = 1.0 / R(j, j);
            }
            __syncwarp();
            double est = smin;
            for (int it = 0; it < 4; ++it) {
                // R^T y = x (forward, axpy form): y_r = x_r / R_rr; x_c -= R_rc y_r
                for (int r = 0; r < k; ++r) {
                    const double yr = x[r] * rinv[r];
                    for (int c = r + 1 + lane; c < k; c += 32) x[c] -= R(r, c) * yr;
                    if (lane == 0) y[r] = yr;
                    __syncwarp();
                }
                // R z = y (backward, axpy form): z_c = y_c / R_cc; y_r -= R_rc z_c
                for (int c = k - 1; c >= 0; --c) {
                    const double zc = y[c] * rinv[c];
                    for (int r = lane; r < c; r += 32) y[r] -= R(r, c) * zc;
                    if (lane == 0) x[c] = zc;
                    __syncwarp();
                }
                double zz = 0.0;
                for (int c = lane; c < k; c += 32) zz += x[c] * x[c];
#pragma unroll
                for (int off = 16; off; off >>= 1) zz += __shfl_xor_sync(0xffffffffu, zz, off);
                if (!(zz > 0.0) || !isfinite(zz)) {
                    est = 0.0;
                    break;
                }
                est = fmin(est, 1.0 / sqrt(sqrt(zz)));
                const double inv = 1.0 / sqrt(zz);
                for (int c = lane; c < k; c += 32) x[c] *= inv;
                __syncwarp();
            }
            smin = est;
        }
    } else {
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
                                                           double *__restrict__ qtau) {
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
            // thread per trailing column c: w = v^T A[:,c] (v_j = 1, v_r = scal*colj[r])
            for (int c = j + 1 + tid; c < k1; c += blockDim.x) {
                double *colc = A + c * ld;
                double w0 = colc[j], w1 = 0.0, w2 = 0.0, w3 = 0.0;
                int r = j + 1;
                for (; r + 3 < k2; r += 4) {
                    w0 += (colj[r] * scal) * colc[r];
                    w1 += (colj[r + 1] * scal) * colc[r + 1];
                    w2 += (colj[r + 2] * scal) * colc[r + 2];
                    w3 += (colj[r + 3] * scal) * colc[r + 3];
                }
                for (; r < k2; ++r) w0 += (colj[r] * scal) * colc[r];
                const double f = tj * ((w0 + w1) + (w2 + w3));
                colc[j] -= f;
                for (int rr = j + 1; rr < k2; ++rr) colc[rr] -= f * (colj[rr] * scal);
            }
        }
        __syncthreads();
        if (tj != 0.0)
            for (int r = j + 1 + tid; r < k2; r += blockDim.x) colj[r] *= scal;
        __syncthreads();
    }
    for (int i = tid; i < k1 * ld; i += blockDim.x) qa[i] = A[i];
}

// Phase 2 (many CTAs): CTA 0 runs the rank test on R; every warp of the
// other CTAs forms one column of pinv^T = (R^-1 Q^T)^T from the reflectors.
__global__ void __launch_bounds__(256) qr_tail_kernel(const double *__restrict__ qa,
                                                      const double *__restrict__ qtau, int k1,
                                                      int k2, double *__restrict__ pinvT,
                                                      int64_t ldp, double *__restrict__ stats) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int ld = k2 | 1;
    const int k2p = (k2 + 1) & ~1;
    double *sm = reinterpret_cast<double *>(smem_raw);
    if (blockIdx.x == 0) {
        rank_estimate(RSmem{qa, ld}, k1, sm, sm + k2p, sm + 2 * k2p, sm + 3 * k2p, stats);
        return;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c = (blockIdx.x - 1) * (blockDim.x >> 5) + warp;
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

__global__ void __launch_bounds__(kQrThreads, 1) rank_estimate_kernel(const double *__restrict__ R,
                                                                      int k, int64_t ldr,
                                                                      double *__restrict__ stats) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *xv = reinterpret_cast<double *>(smem_raw);
    double *yv = xv + k;
    double *rv = yv + k;
    double *red = rv + k;
    rank_estimate(RGlobalRowMajor{R, ldr}, k, xv, yv, rv, red, stats);
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
    return sizeof(double) * (size_t)(k1 * (k2 | 1) + k1) + 256;
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
    SRLU_CUDA(cudaFuncSetAttribute(qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    qr_kernel<<<1, kQrThreads, smem, s>>>(mT, (int)k1, (int)k2, ldm, qa, qtau);
    SRLU_CHECK_LAUNCH("qr_kernel");
    const int k2p = (int)((k2 + 1) & ~1);
    size_t smem2 = sizeof(double) * (size_t)(8 * k2p + 64);
    size_t smem_rank = sizeof(double) * (size_t)(4 * k2p + 64);
    if (smem_rank > smem2) smem2 = smem_rank;
    SRLU_CUDA(cudaFuncSetAttribute(qr_tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem2));
    qr_tail_kernel<<<(unsigned)(1 + ceil_div(k2, 8)), 256, smem2, s>>>(qa, qtau, (int)k1, (int)k2,
                                                                       pinvT, ldp, stats);
    SRLU_CHECK_LAUNCH("qr_tail_kernel");
    return SRLU_OK;
}

extern "C" int srlu_rank_estimate(const double *R, int64_t k, int64_t ldr, double *stats,
                                  srlu_stream_t stream) {
    SRLU_REQUIRE(k >= 1 && ldr >= k, SRLU_ERR_ARG, "rank_estimate: bad sizes");
    size_t smem = sizeof(double) * (size_t)(3 * k + 64);
    SRLU_REQUIRE(smem <= 200 * 1024, SRLU_ERR_UNSUPPORTED, "rank_estimate: k too large");
    SRLU_CUDA(cudaFuncSetAttribute(rank_estimate_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    rank_estimate_kernel<<<1, kQrThreads, smem, (cudaStream_t)stream>>>(R, (int)k, ldr, stats);
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
