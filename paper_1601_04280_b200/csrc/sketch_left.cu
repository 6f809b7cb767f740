// K3 — stage-2 projection  Omega2 · (P A)  (reference: matrix.py:201-207
// permute_rows + sketch.py:371-378 apply_sketch_left = _fast.pyx:71-78
// sem_scatter_dense + sketch.py:338-349 _fast_mul_left).
//
// P·A is never materialised.  K3a: one CTA per (bucket t, column tile)
// streams, in ascending PA index q, the member rows perm[q] of bucket t
// (srlu_sem_members) straight from A and accumulates the signed rows in
// registers -> S[t, cols] (exactly the reference's (bucket, column) order).
// Every row of A is read exactly once.  K3b: one CTA per column group
// applies +-phase, the radix-2 FWHT down the bucket axis (pad2) and the
// k2-row subsample, writing (Omega2 P A)^T (n x k2).  Only the l2 x n
// bucket matrix S (about 6% of A's bytes at the BASELINE configs) makes a
// round trip, mostly through L2.
#include <stdlib.h>

#include "async_copy.cuh"
#include "fwht.cuh"
#include "fwht_warp.cuh"

namespace srlu {

template <typename T, int V, int NT>
__global__ void __launch_bounds__(NT) k3a_dense_kernel(const T *__restrict__ a, int64_t rows,
                                                       int64_t n, int64_t lda,
                                                       const int32_t *__restrict__ member_row,
                                                       const double *__restrict__ member_sign,
                                                       const int32_t *__restrict__ bptr,
                                                       double *__restrict__ S, int64_t lds) {
    const int t = blockIdx.x;
    const int64_t c0 = ((int64_t)blockIdx.y * NT + threadIdx.x) * V;
    if (c0 >= n) return;
    const bool full = c0 + V <= n;
    double acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = 0.0;
    const int beg = bptr[t], end = bptr[t + 1];
    constexpr int U = 4;
    int e = beg;
    for (; e + U <= end; e += U) {
        int r[U];
        double sg[U];
        T x[U][V];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            r[u] = __ldg(member_row + e + u);
            sg[u] = __ldg(member_sign + e + u);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (r[u] >= 0) {
                const T *src = a + (int64_t)r[u] * lda + c0;
                if constexpr (V == 1) {
                    x[u][0] = __ldcs(src);
                } else if (full) {
                    if constexpr (sizeof(T) * V == 16) {
                        if constexpr (sizeof(T) == 4) {
                            float4 q = __ldcs(reinterpret_cast<const float4 *>(src));
                            x[u][0] = q.x; x[u][1] = q.y; x[u][2] = q.z; x[u][3] = q.w;
                        } else {
                            double2 q = __ldcs(reinterpret_cast<const double2 *>(src));
                            x[u][0] = q.x; x[u][1] = q.y;
                        }
                    }
                } else {
#pragma unroll
                    for (int v = 0; v < V; ++v) x[u][v] = c0 + v < n ? src[v] : T(0);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (r[u] >= 0) {
                const bool neg = sg[u] < 0.0;
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    double d = (double)x[u][v];
                    acc[v] = __dadd_rn(acc[v], neg ? -d : d);
                }
            }
        }
    }
    for (; e < end; ++e) {
        const int r = member_row[e];
        if (r < 0) continue;
        const bool neg = member_sign[e] < 0.0;
        const T *src = a + (int64_t)r * lda + c0;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            if (c0 + v < n) {
                double d = (double)src[v];
                acc[v] = __dadd_rn(acc[v], neg ? -d : d);
            }
        }
    }
    double *dst = S + (int64_t)t * lds + c0;
#pragma unroll
    for (int v = 0; v < V; ++v)
        if (c0 + v < n) dst[v] = acc[v];
}

// one CTA per CB columns: x[t][c] = phase[t]*S[t][c]; FWHT over t; sample
__global__ void k3b_kernel(const double *__restrict__ S, int64_t n, int l, int pad, int CB,
                           const double *__restrict__ phase, const int32_t *__restrict__ idx,
                           int k, double mult, double *__restrict__ out, int64_t ldo) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *xs = reinterpret_cast<double *>(smem_raw);
    const int64_t c0 = (int64_t)blockIdx.x * CB;
    const int nc = (int)((n - c0) < CB ? (n - c0) : CB);
    for (int w = threadIdx.x; w < pad * CB; w += blockDim.x) {
        int t = w / CB, c = w % CB;
        double v = 0.0;
        if (t < l && c < nc) {
            v = S[(int64_t)t * n + c0 + c];
            if (phase[t] < 0.0) v = -v;
        }
        xs[w] = v;
    }
    __syncthreads();
    fwht_smem_cols(xs, pad, CB, CB);
    for (int w = threadIdx.x; w < nc * k; w += blockDim.x) {
        int c = w / k, kk = w % k;
        out[(c0 + c) * ldo + kk] = __dmul_rn(xs[idx[kk] * CB + c], mult);
    }
}

// K3b v2: one warp per column; the column's bucket vector (pad2 doubles,
// swizzled, row stride pad2+1 to spread banks on the transposing store)
// is transformed in registers per 1024-block; cross-block stages are
// output-pruned.  32 <= pad2 <= 8192.
__global__ void __launch_bounds__(512) k3b_v2_kernel(const double *__restrict__ S, int64_t n,
                                                     int l, int pad, int CB,
                                                     const double *__restrict__ phase,
                                                     const int32_t *__restrict__ idx, int k,
                                                     double mult, double *__restrict__ out,
                                                     int64_t ldo) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *xs = reinterpret_cast<double *>(smem_raw);
    // only the bsize-blocks that hold buckets are stored (the rest stay zero
    // through the in-block stages; the pruned combine treats them as zeros)
    const int bsize = pad < 1024 ? pad : 1024;
    const int nb = pad / bsize;  // <= 8 for pad2 <= 8192
    const int nzb = (l + bsize - 1) / bsize;
    const int xlen = nzb * bsize;
    const int ldx = xlen + 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t c0 = (int64_t)blockIdx.x * CB;
    const int nc = (int)((n - c0) < CB ? (n - c0) : CB);
    // U loads in flight per thread (the tile is read once from HBM; one at
    // a time left each CTA waiting ~pad*CB/blockDim round trips)
    constexpr int U = 8;
    const int total = xlen * CB;
    for (int w0 = threadIdx.x; w0 < total; w0 += U * blockDim.x) {
        double v[U];
        bool neg[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int w = w0 + u * blockDim.x;
            const int t = w / CB, c = w % CB;
            const bool ld = w < total && t < l && c < nc;
            v[u] = ld ? S[(int64_t)t * n + c0 + c] : 0.0;
            neg[u] = ld && phase[t] < 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int w = w0 + u * blockDim.x;
            if (w < total) {
                const int t = w / CB, c = w % CB;
                xs[c * ldx + fwht_sw(t)] = neg[u] ? -v[u] : v[u];
            }
        }
    }
    __syncthreads();
    for (int item = warp; item < nc * nzb; item += nw) {
        const int c = item / nzb, b = item % nzb;
        fwht_block_warp_dyn(xs + c * ldx + b * bsize, bsize, lane);
    }
    __syncthreads();
    for (int w = threadIdx.x; w < nc * k; w += blockDim.x) {
        const int c = w / k, kk = w % k;
        out[(c0 + c) * ldo + kk] =
            __dmul_rn(fwht_combine_blocks(xs + c * ldx, bsize, nb, idx[kk], nzb), mult);
    }
}

// K3b v3: one CTA per 32 columns.  The tile x[t][c] (row stride 34) stays
// in shared memory; the FWHT down t runs in register passes of up to four
// stages: a warp item holds, for its 32 columns (lanes), the 16 values
// t = base + j*h0 of one butterfly group, so loads/stores are conflict-free
// and no transpose is needed.  The tile arrives by cp.async (all in flight);
// the first pass applies
// +-phase; the output pass reads the k sampled rows and writes Y^T rows.
// CB columns per CTA (16 or 32); row stride CB+2 doubles (16-byte rows for
// cp.async, conflict-free row accesses).  A warp holds 32/CB items at once.
template <int CB>
struct K3bGeo {
    static constexpr int LD = CB + 2;
    static constexpr int SUB = 32 / CB;
};

template <int CB, int E>
__device__ __forceinline__ void k3b_pass(double *xs, int l, int pad, int lh0,
                                         const uint32_t *sgn, bool first) {
    constexpr int LD = K3bGeo<CB>::LD, SUB = K3bGeo<CB>::SUB;
    constexpr int LE = E == 16 ? 4 : (E == 8 ? 3 : (E == 4 ? 2 : 1));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int col = lane % CB, sub = lane / CB;
    const int items = pad >> LE;
    const int h0 = 1 << lh0;
    for (int it0 = warp * SUB; it0 < items; it0 += nw * SUB) {
        const int it = it0 + sub;
        const int base = (it & (h0 - 1)) + ((it >> lh0) << (LE + lh0));
        double v[E];
#pragma unroll
        for (int j = 0; j < E; ++j) {
            const int t = base + (j << lh0);
            // first pass: rows t >= l were never loaded (zero) and carry the
            // +-phase sign; later passes read the in-place results
            double x = (!first || t < l) ? xs[t * LD + col] : 0.0;
            if (first) x = __hiloint2double(__double2hiint(x) ^ (int)sgn[t], __double2loint(x));
            v[j] = x;
        }
#pragma unroll
        for (int hh = 1; hh < E; hh <<= 1) {
#pragma unroll
            for (int j = 0; j < E; ++j) {
                if ((j & hh) == 0) {
                    const double a = v[j], b = v[j + hh];
                    v[j] = __dadd_rn(a, b);
                    v[j + hh] = __dsub_rn(a, b);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < E; ++j) xs[(base + j * h0) * LD + col] = v[j];
    }
}

template <int CB>
__global__ void __launch_bounds__(256) k3b_v3_kernel(const double *__restrict__ S, int64_t n,
                                                     int l, int pad,
                                                     const double *__restrict__ phase,
                                                     const int32_t *__restrict__ idx, int k,
                                                     double mult, double *__restrict__ out,
                                                     int64_t ldo) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *xs = reinterpret_cast<double *>(smem_raw);
    constexpr int LD = K3bGeo<CB>::LD, Q = CB / 2;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t c0 = (int64_t)blockIdx.x * CB;
    const int nc = (int)((n - c0) < CB ? (n - c0) : CB);
    // the l x CB tile of S, all in flight at once (cp.async, 16 B per copy;
    // columns past n zero-filled)
    for (int w = threadIdx.x; w < l * Q; w += blockDim.x) {
        const int t = w / Q, q = (w % Q) * 2;
        // 16-byte copies need an even row pitch (S + t*n + c0 + q aligned)
        const bool ok = (n & 1) == 0 && q + 1 < nc;
        if (ok) {
            cp_async_16(xs + t * LD + q, S + (int64_t)t * n + c0 + q, true);
        } else {
            xs[t * LD + q] = q < nc ? S[(int64_t)t * n + c0 + q] : 0.0;
            xs[t * LD + q + 1] = q + 1 < nc ? S[(int64_t)t * n + c0 + q + 1] : 0.0;
        }
    }
    // sign bits of the phase (bit 31 of the high word), zero past l
    uint32_t *sgn = reinterpret_cast<uint32_t *>(xs + (size_t)pad * LD);
    for (int t = threadIdx.x; t < pad; t += blockDim.x)
        sgn[t] = (t < l && phase[t] < 0.0) ? 0x80000000u : 0u;
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    bool first = true;
    for (int lh0 = 0; (1 << lh0) < pad;) {
        const int e = (pad >> lh0) >= 16 ? 16 : (pad >> lh0);
        switch (e) {
            case 16: k3b_pass<CB, 16>(xs, l, pad, lh0, sgn, first); lh0 += 4; break;
            case 8: k3b_pass<CB, 8>(xs, l, pad, lh0, sgn, first); lh0 += 3; break;
            case 4: k3b_pass<CB, 4>(xs, l, pad, lh0, sgn, first); lh0 += 2; break;
            default: k3b_pass<CB, 2>(xs, l, pad, lh0, sgn, first); lh0 += 1; break;
        }
        first = false;
        __syncthreads();
    }
    // sample and scale: warp per column, lanes over the k outputs
    for (int c = warp; c < nc; c += nw)
        for (int kk = lane; kk < k; kk += 32)
            out[(c0 + c) * ldo + kk] = __dmul_rn(xs[idx[kk] * LD + c], mult);
}

template <typename T>
static int launch_k3a(const T *a, int64_t rows, int64_t n, int64_t lda, const int32_t *member_row,
                      const double *member_sign, const int32_t *bptr, int64_t l2, double *S,
                      int64_t lds, cudaStream_t stream) {
    constexpr int NT = 128;
    constexpr int V = 16 / sizeof(T);
    bool vec_ok = ((uintptr_t)a % 16 == 0) && (lda % V == 0);
    if (vec_ok) {
        dim3 grid((unsigned)l2, (unsigned)ceil_div(n, NT * V));
        k3a_dense_kernel<T, V, NT><<<grid, NT, 0, stream>>>(a, rows, n, lda, member_row,
                                                            member_sign, bptr, S, lds);
    } else {
        dim3 grid((unsigned)l2, (unsigned)ceil_div(n, NT));
        k3a_dense_kernel<T, 1, NT><<<grid, NT, 0, stream>>>(a, rows, n, lda, member_row,
                                                            member_sign, bptr, S, lds);
    }
    SRLU_CHECK_LAUNCH("k3a_dense_kernel");
    return SRLU_OK;
}

int launch_k3b(const double *S, int64_t n, int64_t l2, int64_t pad2, const double *phase2,
               const int32_t *idx2, int64_t k2, double mult2, double *out, int64_t ldo,
               cudaStream_t stream) {
    // v3: 16 columns per CTA when three CTAs then fit an SM, else 32
    const int v3cb = getenv("SRLU_K3B_CB") ? atoi(getenv("SRLU_K3B_CB")) : 0;
    if (pad2 >= 32 && getenv("SRLU_K3B_V2") == nullptr &&
        ((v3cb != 32 && pad2 * 18 * 8 <= 75 * 1024) || pad2 * 34 * 8 <= 196 * 1024)) {
        const bool cb16 = v3cb != 32 && pad2 * 18 * 8 <= 75 * 1024;
        const size_t smem = (size_t)pad2 * (cb16 ? 18 : 34) * 8 + (size_t)pad2 * 4;
        auto kern = cb16 ? k3b_v3_kernel<16> : k3b_v3_kernel<32>;
        SRLU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<(unsigned)ceil_div(n, cb16 ? 16 : 32), 256, smem, stream>>>(
            S, n, (int)l2, (int)pad2, phase2, idx2, (int)k2, mult2, out, ldo);
        SRLU_CHECK_LAUNCH("k3b_v3_kernel");
        return SRLU_OK;
    }
    if (pad2 >= 32 && pad2 <= 8192) {
        int CB = (int)(16384 / pad2);  // ~128 KB of smem
        if (const char *e = getenv("SRLU_K3B_V2CB")) CB = atoi(e);  // testing knob
        if (CB < 1) CB = 1;
        if (CB > 64) CB = 64;
        const int64_t bs2 = pad2 < 1024 ? pad2 : 1024;
        size_t smem = (size_t)(ceil_div(l2, bs2) * bs2 + 1) * CB * 8;
        SRLU_CUDA(cudaFuncSetAttribute(k3b_v2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
        k3b_v2_kernel<<<(unsigned)ceil_div(n, CB), 512, smem, stream>>>(
            S, n, (int)l2, (int)pad2, CB, phase2, idx2, (int)k2, mult2, out, ldo);
        SRLU_CHECK_LAUNCH("k3b_v2_kernel");
        return SRLU_OK;
    }
    int CB = (int)(8192 / pad2);
    if (CB < 1) CB = 1;
    if (CB > 64) CB = 64;
    size_t smem = (size_t)pad2 * CB * 8;
    SRLU_REQUIRE(smem <= 200 * 1024, SRLU_ERR_UNSUPPORTED, "sketch_left: pad2=%lld too large",
                 (long long)pad2);
    SRLU_CUDA(cudaFuncSetAttribute(k3b_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    k3b_kernel<<<(unsigned)ceil_div(n, CB), 256, smem, stream>>>(S, n, (int)l2, (int)pad2, CB,
                                                                 phase2, idx2, (int)k2, mult2,
                                                                 out, ldo);
    SRLU_CHECK_LAUNCH("k3b_kernel");
    return SRLU_OK;
}

}  // namespace srlu

using namespace srlu;

extern "C" size_t srlu_sketch_left_workspace(int64_t n, int64_t l2, int64_t pad2) {
    (void)pad2;
    return sizeof(double) * (size_t)(n * l2) + 256;
}

extern "C" int srlu_sketch_left_dense(const void *a, int dtype, int64_t rows, int64_t n,
                                      int64_t lda, const int32_t *member_row,
                                      const double *member_sign, const int32_t *bptr2, int64_t l2,
                                      const double *phase2, const int32_t *idx2, int64_t k2,
                                      int64_t pad2, double mult2, double *out, int64_t ldo,
                                      void *ws, size_t ws_bytes, srlu_stream_t stream) {
    SRLU_REQUIRE(rows >= 0 && n >= 1 && lda >= n && l2 >= 1 && k2 >= 1 && k2 <= pad2 &&
                     pad2 >= l2 && (pad2 & (pad2 - 1)) == 0 && ldo >= k2,
                 SRLU_ERR_ARG, "sketch_left_dense: bad sizes");
    SRLU_REQUIRE(l2 < 65536, SRLU_ERR_UNSUPPORTED, "sketch_left_dense: l2 >= 65536");
    SRLU_REQUIRE(ws_bytes >= srlu_sketch_left_workspace(n, l2, pad2), SRLU_ERR_WORKSPACE,
                 "sketch_left_dense: workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    double *S = (double *)ws;
    int rc;
    if (dtype == SRLU_F32)
        rc = launch_k3a<float>((const float *)a, rows, n, lda, member_row, member_sign, bptr2, l2,
                               S, n, s);
    else if (dtype == SRLU_F64)
        rc = launch_k3a<double>((const double *)a, rows, n, lda, member_row, member_sign, bptr2,
                                l2, S, n, s);
    else {
        set_error("sketch_left_dense: unknown dtype %d", dtype);
        return SRLU_ERR_ARG;
    }
    if (rc) return rc;
    return launch_k3b(S, n, l2, pad2, phase2, idx2, k2, mult2, out, ldo, s);
}

extern "C" int srlu_sem_scatter_dense(const void *a, int dtype, int64_t rows, int64_t n,
                                      int64_t lda, const int32_t *member_row,
                                      const double *member_sign, const int32_t *bptr, int64_t l,
                                      double *out, int64_t ldo, srlu_stream_t stream) {
    SRLU_REQUIRE(rows >= 0 && n >= 1 && lda >= n && l >= 1 && ldo >= n, SRLU_ERR_ARG,
                 "sem_scatter_dense: bad sizes");
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == SRLU_F32)
        return launch_k3a<float>((const float *)a, rows, n, lda, member_row, member_sign, bptr, l,
                                 out, ldo, s);
    if (dtype == SRLU_F64)
        return launch_k3a<double>((const double *)a, rows, n, lda, member_row, member_sign, bptr,
                                  l, out, ldo, s);
    set_error("sem_scatter_dense: unknown dtype %d", dtype);
    return SRLU_ERR_ARG;
}
