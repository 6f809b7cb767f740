// K1 — stage-1 sketch  Y = A · Omega1^*  (reference: sketch.py:362-368
// apply_sketch_right = _fast.pyx:44-54 sem_gather_dense (or :57-68 csc)
// + sketch.py:322-335 _fast_adjoint_right + _fast.pyx:23-41 fwht_rows).
//
// Dense: one CTA owns R rows of A (row-major) and streams them once in
// column chunks through a 2-stage cp.async pipeline.  Each thread owns a
// fixed set of buckets t (registers acc[R][BPT]) and walks each bucket's
// ascending source list (srlu_sem_plan) chunk by chunk, so every (row,
// bucket) sum is accumulated in exactly the reference's order (ascending
// column j) -> bit-identical B0.  Epilogue per row: +-phase, radix-2 FWHT
// (stages h = 1, 2, 4, ...) in shared memory, gather the k1 sampled
// coordinates, scale, write Y; B0 never touches HBM.
//
// CSR: one warp per row; the row's nonzeros (ascending column) are added
// into a shared-memory bucket row 32 at a time; lanes that hit the same
// bucket in one chunk are serialised in lane (= column) order, which again
// reproduces the reference's ascending-j order.
#include <limits.h>
#include <stdlib.h>

#include "async_copy.cuh"
#include "fwht.cuh"
#include "fwht_warp.cuh"
#include "tma.cuh"

namespace srlu {

template <typename T, int R>
struct K1Shape {
    static constexpr int C = 32768 / (R * (int)sizeof(T));  // columns per chunk
    static constexpr int TILE_BYTES = 2 * R * C * (int)sizeof(T);
};

template <typename T, int NT, int BPT, int R, bool FUSED>
__global__ void __launch_bounds__(NT) k1_dense_kernel(
    const T *__restrict__ a, int64_t m, int64_t n, int64_t lda, const int32_t *__restrict__ sorted,
    const int32_t *__restrict__ bptr, int l, const double *__restrict__ phase,
    const int32_t *__restrict__ idx, int k, int pad, double mult, double *__restrict__ y,
    int64_t ldy, int *nonfinite, bool vec_ok) {
    constexpr int C = K1Shape<T, R>::C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *tiles = reinterpret_cast<T *>(smem_raw);
    double *x = reinterpret_cast<double *>(smem_raw);
    const int tid = threadIdx.x;
    const int64_t row0 = (int64_t)blockIdx.x * R;

    int cur[BPT], end[BPT], code[BPT];
    double acc[R][BPT];
#pragma unroll
    for (int b = 0; b < BPT; ++b) {
        int t = tid + b * NT;
        cur[b] = t < l ? bptr[t] : 0;
        end[b] = t < l ? bptr[t + 1] : 0;
        code[b] = cur[b] < end[b] ? sorted[cur[b]] : INT_MAX;
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r][b] = 0.0;
    }

    const int64_t nchunks = ceil_div(n, C);
    load_tile_async<T, R, C, NT>(tiles, a, m, n, lda, row0, 0, vec_ok);
    cp_async_commit();
    for (int64_t ch = 0; ch < nchunks; ++ch) {
        if (ch + 1 < nchunks) {
            load_tile_async<T, R, C, NT>(tiles + ((ch + 1) & 1) * R * C, a, m, n, lda, row0,
                                         (ch + 1) * C, vec_ok);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const T *tl = tiles + (ch & 1) * R * C;
        const int c0 = (int)(ch * C);
        const int c1 = c0 + C;
#pragma unroll
        for (int b = 0; b < BPT; ++b) {
            int cd = code[b];
            while ((cd & 0x7FFFFFFF) < c1) {
                const int cc = (cd & 0x7FFFFFFF) - c0;
                const bool neg = cd < 0;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    double v = (double)tl[r * C + cc];
                    acc[r][b] = __dadd_rn(acc[r][b], neg ? -v : v);
                }
                ++cur[b];
                cd = cur[b] < end[b] ? __ldg(sorted + cur[b]) : INT_MAX;
            }
            code[b] = cd;
        }
        __syncthreads();
    }

    if constexpr (FUSED) {
        bool bad = false;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t row = row0 + r;
            if (row0 + r >= m) break;  // uniform across the CTA
#pragma unroll
            for (int b = 0; b < BPT; ++b) {
                int t = tid + b * NT;
                if (t < l) x[t] = phase[t] < 0.0 ? -acc[r][b] : acc[r][b];
            }
            for (int t = l + tid; t < pad; t += NT) x[t] = 0.0;
            __syncthreads();
            fwht_smem_cta(x, pad);
            for (int kk = tid; kk < k; kk += NT) {
                double v = __dmul_rn(x[idx[kk]], mult);
                y[row * ldy + kk] = v;
                bad |= !isfinite(v);
            }
            __syncthreads();
        }
        if (bad) atomicOr(nonfinite, 1);
    } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t row = row0 + r;
            if (row >= m) break;
#pragma unroll
            for (int b = 0; b < BPT; ++b) {
                int t = tid + b * NT;
                if (t < l) y[row * ldy + t] = acc[r][b];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// K1 v2 (aligned shapes, 32 <= pad1 <= 8192): 3-stage TMA bulk-copy
// pipeline of R x C row segments (one elected thread issues R
// cp.async.bulk per chunk, mbarrier completion), register-resident warp
// FWHT per 1024-block, output-pruned cross-block stages.

constexpr int kK1Stages = 2;

template <typename T, int R>
struct K1v2Shape {
    static constexpr int C = 65536 / (R * (int)sizeof(T));  // 64 KB per stage
};

template <typename T, int NT, int BPT, int R>
__global__ void __launch_bounds__(NT) k1v2_kernel(
    const T *__restrict__ a, int64_t m, int64_t n, int64_t lda, const int32_t *__restrict__ sorted,
    const int32_t *__restrict__ bptr, int l, const double *__restrict__ phase,
    const int32_t *__restrict__ idx, int k, int pad, double mult, double *__restrict__ y,
    int64_t ldy, int *nonfinite) {
    constexpr int C = K1v2Shape<T, R>::C;
    constexpr int NW = NT / 32;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full[kK1Stages];
    T *tiles = reinterpret_cast<T *>(smem_raw);
    double *xs = reinterpret_cast<double *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t row0 = (int64_t)blockIdx.x * R;
    const int nrows = (int)min((int64_t)R, m - row0);
    const int64_t nchunks = ceil_div(n, C);

    if (tid == 0) {
        for (int s = 0; s < kK1Stages; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int stage, int64_t ch) {
        const int64_t c0 = ch * C;
        const int cols = (int)min((int64_t)C, n - c0);
        const unsigned bytes = (unsigned)(cols * sizeof(T));
        mbar_arrive_expect_tx(&full[stage], bytes * nrows);
        for (int r = 0; r < nrows; ++r)
            bulk_g2s(tiles + ((size_t)stage * R + r) * C, a + (row0 + r) * lda + c0, bytes,
                     &full[stage]);
    };
    if (tid == 0)
        for (int s = 0; s < kK1Stages && s < nchunks; ++s) issue(s, s);

    // code[b]: the slot's current source; nxt[b]: the one after it, loaded one
    // step ahead so that the walk's loop condition never waits on a load
    int cur[BPT], end[BPT], code[BPT], nxt[BPT];
    double acc[R][BPT];
#pragma unroll
    for (int b = 0; b < BPT; ++b) {
        const int t = tid + b * NT;
        cur[b] = t < l ? bptr[t] : 0;
        end[b] = t < l ? bptr[t + 1] : 0;
        code[b] = cur[b] < end[b] ? sorted[cur[b]] : INT_MAX;
        nxt[b] = cur[b] + 1 < end[b] ? sorted[cur[b] + 1] : INT_MAX;
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r][b] = 0.0;
    }

    for (int64_t ch = 0; ch < nchunks; ++ch) {
        const int stage = (int)(ch % kK1Stages);
        mbar_wait(&full[stage], (unsigned)((ch / kK1Stages) & 1));
        const T *tl = tiles + (size_t)stage * R * C;
        const int c0 = (int)(ch * C);
        const int c1 = c0 + C;
#pragma unroll
        for (int b = 0; b < BPT; ++b) {
            int cd = code[b], nx = nxt[b];
            while ((cd & 0x7FFFFFFF) < c1) {
                const int nn = cur[b] + 2 < end[b] ? __ldg(sorted + cur[b] + 2) : INT_MAX;
                const int cc = (cd & 0x7FFFFFFF) - c0;
                const bool neg = cd < 0;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const double v = (double)tl[r * C + cc];
                    acc[r][b] = neg ? __dsub_rn(acc[r][b], v) : __dadd_rn(acc[r][b], v);
                }
                ++cur[b];
                cd = nx;
                nx = nn;
            }
            code[b] = cd;
            nxt[b] = nx;
        }
        __syncthreads();
        if (tid == 0 && ch + kK1Stages < nchunks) {
            fence_proxy_async_smem();
            issue(stage, ch + kK1Stages);
        }
    }

    // ---- epilogue: +-phase, FWHT per row, sample, scale ------------------
    // (all chunks consumed: every bulk copy has landed and been read)
#pragma unroll
    for (int r = 0; r < R; ++r) {
        double *row = xs + (size_t)r * pad;
#pragma unroll
        for (int b = 0; b < BPT; ++b) {
            const int t = tid + b * NT;
            if (t < l) row[fwht_sw(t)] = phase[t] < 0.0 ? -acc[r][b] : acc[r][b];
        }
        for (int t = l + tid; t < pad; t += NT) row[fwht_sw(t)] = 0.0;
    }
    __syncthreads();
    const int bsize = pad < 512 ? pad : 512;  // 16 values per lane in registers
    const int nb = pad / bsize;
    const int nzb = (l + bsize - 1) / bsize;  // blocks holding nonzeros
    for (int item = warp; item < nrows * nzb; item += NW) {
        const int r = item / nzb, b = item % nzb;
        fwht_block_warp_dyn512(xs + (size_t)r * pad + (size_t)b * bsize, bsize, lane);
    }
    __syncthreads();
    bool bad = false;
    for (int w = tid; w < nrows * k; w += NT) {
        const int r = w / k, kk = w % k;
        const double v =
            __dmul_rn(fwht_combine_blocks(xs + (size_t)r * pad, bsize, nb, idx[kk]), mult);
        y[(row0 + r) * ldy + kk] = v;
        bad |= !isfinite(v);
    }
    if (bad) atomicOr(nonfinite, 1);
}

// ---------------------------------------------------------------------------
// K1 v3: persistent (grid = #SMs); each CTA walks its row blocks (R rows)
// and their 1-D chunks as ONE item stream through a kK1Stages-deep TMA
// bulk-copy ring, so the loads of the next row block are in flight while
// the current block's FWHT epilogue runs (separate epilogue buffer).

template <typename T, int NT, int BPT, int R>
__global__ void __launch_bounds__(NT, 1) k1v3_kernel(
    const T *__restrict__ a, int64_t m, int64_t n, int64_t lda, const int32_t *__restrict__ sorted,
    const int32_t *__restrict__ bptr, int l, const double *__restrict__ phase,
    const int32_t *__restrict__ idx, int k, int pad, double mult, double *__restrict__ y,
    int64_t ldy, int *nonfinite, int C) {
    constexpr int NW = NT / 32;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full[kK1Stages];
    T *tiles = reinterpret_cast<T *>(smem_raw);
    double *xs = reinterpret_cast<double *>(smem_raw + (size_t)kK1Stages * R * C * sizeof(T));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t nrb = ceil_div(m, R);
    const int64_t nchunks = ceil_div(n, C);
    const int64_t my_rb = nrb > blockIdx.x ? ceil_div(nrb - blockIdx.x, gridDim.x) : 0;
    const int64_t nitems = my_rb * nchunks;

    if (tid == 0) {
        for (int st = 0; st < kK1Stages; ++st) mbar_init(&full[st], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int64_t it) {
        const int stage = (int)(it % kK1Stages);
        const int64_t rb = blockIdx.x + (it / nchunks) * gridDim.x;
        const int64_t ch = it % nchunks;
        const int64_t row0 = rb * R;
        const int nrows = (int)min((int64_t)R, m - row0);
        const int64_t c0 = ch * C;
        const int cols = (int)min((int64_t)C, n - c0);
        const unsigned bytes = (unsigned)(cols * sizeof(T));
        mbar_arrive_expect_tx(&full[stage], bytes * nrows);
        for (int r = 0; r < nrows; ++r)
            bulk_g2s(tiles + ((size_t)stage * R + r) * C, a + (row0 + r) * lda + c0, bytes,
                     &full[stage]);
    };
    if (tid == 0)
        for (int64_t it = 0; it < kK1Stages && it < nitems; ++it) issue(it);

    int cur[BPT], end[BPT], code[BPT];
    double acc[R][BPT];
    bool bad = false;
    for (int64_t it = 0; it < nitems; ++it) {
        const int stage = (int)(it % kK1Stages);
        const int64_t ch = it % nchunks;
        const int64_t rb = blockIdx.x + (it / nchunks) * gridDim.x;
        if (ch == 0) {
#pragma unroll
            for (int b = 0; b < BPT; ++b) {
                const int t = tid + b * NT;
                cur[b] = t < l ? bptr[t] : 0;
                end[b] = t < l ? bptr[t + 1] : 0;
                code[b] = cur[b] < end[b] ? __ldg(sorted + cur[b]) : INT_MAX;
#pragma unroll
                for (int r = 0; r < R; ++r) acc[r][b] = 0.0;
            }
        }
        mbar_wait(&full[stage], (unsigned)((it / kK1Stages) & 1));
        const T *tl = tiles + (size_t)stage * R * C;
        const int c0 = (int)(ch * C);
        const int c1 = c0 + C;
#pragma unroll
        for (int b = 0; b < BPT; ++b) {
            int cd = code[b];
            while ((cd & 0x7FFFFFFF) < c1) {
                const int cc = (cd & 0x7FFFFFFF) - c0;
                const bool neg = cd < 0;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const double v = (double)tl[r * C + cc];
                    acc[r][b] = neg ? __dsub_rn(acc[r][b], v) : __dadd_rn(acc[r][b], v);
                }
                ++cur[b];
                cd = cur[b] < end[b] ? __ldg(sorted + cur[b]) : INT_MAX;
            }
            code[b] = cd;
        }
        __syncthreads();  // stage consumed by everyone
        if (tid == 0 && it + kK1Stages < nitems) {
            fence_proxy_async_smem();
            issue(it + kK1Stages);
        }
        if (ch == nchunks - 1) {
            // epilogue for row block rb: +-phase, FWHT, sample, scale
            const int64_t row0 = rb * R;
            const int nrows = (int)min((int64_t)R, m - row0);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                double *row = xs + (size_t)r * pad;
#pragma unroll
                for (int b = 0; b < BPT; ++b) {
                    const int t = tid + b * NT;
                    if (t < l) row[fwht_sw(t)] = phase[t] < 0.0 ? -acc[r][b] : acc[r][b];
                }
                for (int t = l + tid; t < pad; t += NT) row[fwht_sw(t)] = 0.0;
            }
            __syncthreads();
            const int bsize = pad < 512 ? pad : 512;
            const int nb = pad / bsize;
            const int nzb = (l + bsize - 1) / bsize;
            for (int item = warp; item < nrows * nzb; item += NW) {
                const int r = item / nzb, b = item % nzb;
                fwht_block_warp_dyn512(xs + (size_t)r * pad + (size_t)b * bsize, bsize, lane);
            }
            __syncthreads();
            for (int w = tid; w < nrows * k; w += NT) {
                const int r = w / k, kk = w % k;
                const double v =
                    __dmul_rn(fwht_combine_blocks(xs + (size_t)r * pad, bsize, nb, idx[kk]), mult);
                y[(row0 + r) * ldy + kk] = v;
                bad |= !isfinite(v);
            }
            __syncthreads();  // xs reused by the next block
        }
    }
    if (bad) atomicOr(nonfinite, 1);
}

template <typename T, int NT, int BPT, int R>
static int launch_k1v3(const T *a, int64_t m, int64_t n, int64_t lda, const int32_t *sorted,
                       const int32_t *bptr, int l, const double *phase, const int32_t *idx, int k,
                       int pad, double mult, double *y, int64_t ldy, int *nonfinite,
                       cudaStream_t stream) {
    const size_t xs_bytes = (size_t)R * pad * sizeof(double);
    const size_t budget = 200 * 1024;
    size_t stage = 64 * 1024;
    if (kK1Stages * stage + xs_bytes > budget) stage = (budget - xs_bytes) / kK1Stages;
    int C = (int)(stage / (R * sizeof(T)));
    C &= ~127;  // multiple of 128 elements (16-byte bulk copies)
    if ((int64_t)C > n) C = (int)((n + 3) & ~3LL);
    if (C < 128) C = 128;
    const size_t smem = (size_t)kK1Stages * R * C * sizeof(T) + xs_bytes;
    auto kern = k1v3_kernel<T, NT, BPT, R>;
    SRLU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t nrb = ceil_div(m, R);
    const unsigned grid = (unsigned)(nrb < sms ? nrb : sms);
    kern<<<grid, NT, smem, stream>>>(a, m, n, lda, sorted, bptr, l, phase, idx, k, pad, mult, y,
                                     ldy, nonfinite, C);
    SRLU_CHECK_LAUNCH("k1v3_kernel");
    return SRLU_OK;
}

template <typename T, int NT, int BPT, int R>
static int launch_k1v2(const T *a, int64_t m, int64_t n, int64_t lda, const int32_t *sorted,
                       const int32_t *bptr, int l, const double *phase, const int32_t *idx, int k,
                       int pad, double mult, double *y, int64_t ldy, int *nonfinite,
                       cudaStream_t stream) {
    constexpr int C = K1v2Shape<T, R>::C;
    size_t smem = (size_t)kK1Stages * R * C * sizeof(T);
    size_t ep = (size_t)R * pad * sizeof(double);
    if (ep > smem) smem = ep;
    auto kern = k1v2_kernel<T, NT, BPT, R>;
    SRLU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)ceil_div(m, R), NT, smem, stream>>>(a, m, n, lda, sorted, bptr, l, phase, idx,
                                                        k, pad, mult, y, ldy, nonfinite);
    SRLU_CHECK_LAUNCH("k1v2_kernel");
    return SRLU_OK;
}

template <typename T>
static int dispatch_k1v2(const T *a, int64_t m, int64_t n, int64_t lda, const int32_t *sorted,
                         const int32_t *bptr, int64_t l, const double *phase, const int32_t *idx,
                         int64_t k, int64_t pad, double mult, double *y, int64_t ldy,
                         int *nonfinite, cudaStream_t s) {
    int L = (int)l, K = (int)k, P = (int)pad;
    // persistent grid, TMA ring, 512 threads (128 registers: no spills)
    if (getenv("SRLU_K1_V3") != nullptr) {  // experimental persistent variant (slower today)
        if (l <= 512)
            return launch_k1v3<T, 512, 1, (sizeof(T) == 4 ? 4 : 2)>(
                a, m, n, lda, sorted, bptr, L, phase, idx, K, P, mult, y, ldy, nonfinite, s);
        if (l <= 1024)
            return launch_k1v3<T, 512, 2, (sizeof(T) == 4 ? 4 : 2)>(
                a, m, n, lda, sorted, bptr, L, phase, idx, K, P, mult, y, ldy, nonfinite, s);
        if (l <= 2048)
            return launch_k1v3<T, 512, 4, 2>(a, m, n, lda, sorted, bptr, L, phase, idx, K, P,
                                             mult, y, ldy, nonfinite, s);
        if (l <= 4096)
            return launch_k1v3<T, 512, 8, 2>(a, m, n, lda, sorted, bptr, L, phase, idx, K, P,
                                             mult, y, ldy, nonfinite, s);
        return launch_k1v3<T, 512, 16, 1>(a, m, n, lda, sorted, bptr, L, phase, idx, K, P, mult,
                                          y, ldy, nonfinite, s);
    }
    if (l <= 1024)
        return launch_k1v2<T, 1024, 1, (sizeof(T) == 4 ? 4 : 2)>(a, m, n, lda, sorted, bptr, L,
                                                                   phase, idx, K, P, mult, y, ldy,
                                                                   nonfinite, s);
    if (l <= 2048)
        return launch_k1v2<T, 1024, 2, 2>(a, m, n, lda, sorted, bptr, L, phase, idx, K, P, mult,
                                          y, ldy, nonfinite, s);
    if (l <= 4096)
        return launch_k1v2<T, 1024, 4, 2>(a, m, n, lda, sorted, bptr, L, phase, idx, K, P, mult,
                                          y, ldy, nonfinite, s);
    if (l <= 5120)  // BASELINE config 5 (l1 = 4400): 5 slots per thread, fewer registers
        return launch_k1v2<T, 1024, 5, 2>(a, m, n, lda, sorted, bptr, L, phase, idx, K, P, mult,
                                          y, ldy, nonfinite, s);
    return launch_k1v2<T, 1024, 8, 2>(a, m, n, lda, sorted, bptr, L, phase, idx, K, P, mult, y,
                                      ldy, nonfinite, s);
}

template <typename T, int NT, int BPT, int R, bool FUSED>
static int launch_k1_dense(const T *a, int64_t m, int64_t n, int64_t lda, const int32_t *sorted,
                           const int32_t *bptr, int l, const double *phase, const int32_t *idx,
                           int k, int pad, double mult, double *y, int64_t ldy, int *nonfinite,
                           cudaStream_t stream) {
    constexpr int V = 16 / sizeof(T);
    bool vec_ok = ((uintptr_t)a % 16 == 0) && (lda % V == 0);
    size_t smem = K1Shape<T, R>::TILE_BYTES;
    if (FUSED) smem = smem > (size_t)pad * 8 ? smem : (size_t)pad * 8;
    auto kern = k1_dense_kernel<T, NT, BPT, R, FUSED>;
    SRLU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    unsigned grid = (unsigned)ceil_div(m, R);
    kern<<<grid, NT, smem, stream>>>(a, m, n, lda, sorted, bptr, l, phase, idx, k, pad, mult, y,
                                     ldy, nonfinite, vec_ok);
    SRLU_CHECK_LAUNCH("k1_dense_kernel");
    return SRLU_OK;
}

template <typename T, bool FUSED>
static int dispatch_k1_dense(const T *a, int64_t m, int64_t n, int64_t lda, const int32_t *sorted,
                             const int32_t *bptr, int64_t l, const double *phase,
                             const int32_t *idx, int64_t k, int64_t pad, double mult, double *y,
                             int64_t ldy, int *nonfinite, cudaStream_t s) {
    int L = (int)l, K = (int)k, P = (int)pad;
    if (l <= 256)
        return launch_k1_dense<T, 256, 1, 8, FUSED>(a, m, n, lda, sorted, bptr, L, phase, idx, K,
                                                    P, mult, y, ldy, nonfinite, s);
    if (l <= 512)
        return launch_k1_dense<T, 256, 2, 8, FUSED>(a, m, n, lda, sorted, bptr, L, phase, idx, K,
                                                    P, mult, y, ldy, nonfinite, s);
    if (l <= 1024)
        return launch_k1_dense<T, 256, 4, 8, FUSED>(a, m, n, lda, sorted, bptr, L, phase, idx, K,
                                                    P, mult, y, ldy, nonfinite, s);
    if (l <= 2048)
        return launch_k1_dense<T, 256, 8, 4, FUSED>(a, m, n, lda, sorted, bptr, L, phase, idx, K,
                                                    P, mult, y, ldy, nonfinite, s);
    if (l <= 4096)
        return launch_k1_dense<T, 512, 8, 4, FUSED>(a, m, n, lda, sorted, bptr, L, phase, idx, K,
                                                    P, mult, y, ldy, nonfinite, s);
    if (l <= 8192)
        return launch_k1_dense<T, 512, 16, 2, FUSED>(a, m, n, lda, sorted, bptr, L, phase, idx, K,
                                                     P, mult, y, ldy, nonfinite, s);
    set_error("sketch_right: l1=%lld > 8192 is not supported", (long long)l);
    return SRLU_ERR_UNSUPPORTED;
}

// ---------------------------------------------------------------------------
// CSR

template <typename T, int WPB>
__global__ void __launch_bounds__(WPB * 32, 3) k1_csr_kernel(
    const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
    const T *__restrict__ vals, int64_t m, const int32_t *__restrict__ row_of,
    const double *__restrict__ sign, int l, const double *__restrict__ phase,
    const int32_t *__restrict__ idx, int k, int pad, double mult, double *__restrict__ y,
    int64_t ldy, int *nonfinite) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *x = reinterpret_cast<double *>(smem_raw) + (size_t)warp * pad;
    // +-phase folded into each entry's sign (phase[t] * sum = sum of
    // phase[t] * terms exactly: negation commutes with rounding)
    __shared__ unsigned phbits[8192 / 32];
    for (int w = threadIdx.x; w < (pad + 31) / 32; w += blockDim.x) {
        unsigned bits = 0;
        for (int i = 0; i < 32; ++i) {
            const int t = w * 32 + i;
            if (t < l && phase[t] < 0.0) bits |= 1u << i;
        }
        phbits[w] = bits;
    }
    __syncthreads();
    // register FWHT (512-point blocks, swizzled) when pad >= 32
    const bool reg = pad >= 32;
    auto P = [&](int t) { return reg ? fwht_sw(t) : t; };
    const int bsize = pad < 512 ? pad : 512;
    const int nb = pad / bsize;
    const int nzb = (l + bsize - 1) / bsize;
    bool bad = false;
    for (int64_t row = (int64_t)blockIdx.x * WPB + warp; row < m; row += (int64_t)gridDim.x * WPB) {
        for (int t = lane; t < pad; t += 32) x[t] = 0.0;
        __syncwarp();
        const int64_t p0 = indptr[row], p1 = indptr[row + 1];
        for (int64_t pb = p0; pb < p1; pb += 32) {
            const int64_t p = pb + lane;
            const bool valid = p < p1;
            int t = 0;
            double val = 0.0;
            if (valid) {
                int j = indices[p];
                double v = (double)vals[p];
                t = row_of[j];
                val = (sign[j] < 0.0) != (((phbits[t >> 5] >> (t & 31)) & 1u) != 0) ? -v : v;
            }
            const unsigned active = __ballot_sync(0xffffffffu, valid);
            unsigned peers = 0;
            if (valid) peers = __match_any_sync(active, t);
            const bool uniq = valid && peers == (1u << lane);
            if (uniq) x[P(t)] = __dadd_rn(x[P(t)], val);
            unsigned conflict = __ballot_sync(0xffffffffu, valid && !uniq);
            while (conflict) {  // same bucket twice in this chunk: ascending column order
                const int src = __ffs(conflict) - 1;
                if (lane == src) x[P(t)] = __dadd_rn(x[P(t)], val);
                __syncwarp();
                conflict &= conflict - 1;
            }
            __syncwarp();
        }
        if (reg) {
            for (int b = 0; b < nzb; ++b) fwht_block_warp_dyn512(x + b * bsize, bsize, lane);
        } else {
            fwht_smem_warp(x, pad, lane);
        }
        for (int kk = lane; kk < k; kk += 32) {
            const double fv = reg ? fwht_combine_blocks(x, bsize, nb, idx[kk]) : x[idx[kk]];
            const double v = __dmul_rn(fv, mult);
            y[row * ldy + kk] = v;
            bad |= !isfinite(v);
        }
        __syncwarp();
    }
    if (bad) atomicOr(nonfinite, 1);
}

template <typename T>
static int launch_k1_csr(const int64_t *indptr, const int32_t *indices, const T *vals, int64_t m,
                         const int32_t *row_of, const double *sign, int64_t l,
                         const double *phase, const int32_t *idx, int64_t k, int64_t pad,
                         double mult, double *y, int64_t ldy, int *nonfinite,
                         cudaStream_t stream) {
    constexpr int WPB = 8;
    size_t smem = (size_t)WPB * pad * 8;
    SRLU_REQUIRE(smem <= 200 * 1024, SRLU_ERR_UNSUPPORTED, "sketch_right_csr: pad1=%lld too large",
                 (long long)pad);
    auto kern = k1_csr_kernel<T, WPB>;
    SRLU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int64_t grid = ceil_div(m, WPB);
    if (grid > 148 * 64) grid = 148 * 64;
    kern<<<(unsigned)grid, WPB * 32, smem, stream>>>(indptr, indices, vals, m, row_of, sign,
                                                     (int)l, phase, idx, (int)k, (int)pad, mult,
                                                     y, ldy, nonfinite);
    SRLU_CHECK_LAUNCH("k1_csr_kernel");
    return SRLU_OK;
}

// ---------------------------------------------------------------------------
// plugin seam: fwht_rows

__global__ void fwht_rows_kernel(double *x, int64_t m, int n, int64_t ldx) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *s = reinterpret_cast<double *>(smem_raw);
    for (int64_t row = blockIdx.x; row < m; row += gridDim.x) {
        for (int j = threadIdx.x; j < n; j += blockDim.x) s[j] = x[row * ldx + j];
        __syncthreads();
        fwht_smem_cta(s, n);
        for (int j = threadIdx.x; j < n; j += blockDim.x) x[row * ldx + j] = s[j];
        __syncthreads();
    }
}

}  // namespace srlu

using namespace srlu;

static bool pow2(int64_t v) { return v >= 1 && (v & (v - 1)) == 0; }

extern "C" int srlu_sketch_right_dense(const void *a, int dtype, int64_t m, int64_t n, int64_t lda,
                                       const int32_t *sorted1, const int32_t *bptr1, int64_t l1,
                                       const double *phase1, const int32_t *idx1, int64_t k1,
                                       int64_t pad1, double mult1, double *y, int64_t ldy,
                                       int *nonfinite, srlu_stream_t stream) {
    SRLU_REQUIRE(m >= 1 && n >= 1 && lda >= n && l1 >= 1 && l1 <= n && k1 >= 1 && k1 <= pad1 &&
                     pow2(pad1) && pad1 >= l1 && ldy >= k1,
                 SRLU_ERR_ARG, "sketch_right_dense: bad sizes");
    SRLU_REQUIRE(n < (1LL << 31) - 1, SRLU_ERR_UNSUPPORTED, "sketch_right_dense: n >= 2^31");
    cudaStream_t s = (cudaStream_t)stream;
    const size_t es = dtype == SRLU_F32 ? 4 : 8;
    const bool tma_ok = ((uintptr_t)a % 16 == 0) && ((lda * es) % 16 == 0) && ((n * es) % 16 == 0) &&
                        pad1 >= 32 && pad1 <= 8192 && l1 <= 8192 && getenv("SRLU_K1_V1") == nullptr;
    if (tma_ok && dtype == SRLU_F32)
        return dispatch_k1v2<float>((const float *)a, m, n, lda, sorted1, bptr1, l1, phase1, idx1,
                                    k1, pad1, mult1, y, ldy, nonfinite, s);
    if (tma_ok && dtype == SRLU_F64)
        return dispatch_k1v2<double>((const double *)a, m, n, lda, sorted1, bptr1, l1, phase1,
                                     idx1, k1, pad1, mult1, y, ldy, nonfinite, s);
    if (dtype == SRLU_F32)
        return dispatch_k1_dense<float, true>((const float *)a, m, n, lda, sorted1, bptr1, l1,
                                              phase1, idx1, k1, pad1, mult1, y, ldy, nonfinite, s);
    if (dtype == SRLU_F64)
        return dispatch_k1_dense<double, true>((const double *)a, m, n, lda, sorted1, bptr1, l1,
                                               phase1, idx1, k1, pad1, mult1, y, ldy, nonfinite, s);
    set_error("sketch_right_dense: unknown dtype %d", dtype);
    return SRLU_ERR_ARG;
}

extern "C" int srlu_sem_gather_dense(const void *a, int dtype, int64_t m, int64_t n, int64_t lda,
                                     const int32_t *sorted, const int32_t *bptr, int64_t l,
                                     double *out, int64_t ldo, srlu_stream_t stream) {
    SRLU_REQUIRE(m >= 1 && n >= 1 && lda >= n && l >= 1 && l <= n && ldo >= l, SRLU_ERR_ARG,
                 "sem_gather_dense: bad sizes");
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == SRLU_F32)
        return dispatch_k1_dense<float, false>((const float *)a, m, n, lda, sorted, bptr, l,
                                               nullptr, nullptr, 1, 1, 1.0, out, ldo, nullptr, s);
    if (dtype == SRLU_F64)
        return dispatch_k1_dense<double, false>((const double *)a, m, n, lda, sorted, bptr, l,
                                                nullptr, nullptr, 1, 1, 1.0, out, ldo, nullptr, s);
    set_error("sem_gather_dense: unknown dtype %d", dtype);
    return SRLU_ERR_ARG;
}

extern "C" int srlu_sketch_right_csr(const int64_t *indptr, const int32_t *indices,
                                     const void *vals, int dtype, int64_t m, int64_t n,
                                     const int32_t *row_of1, const double *sign1, int64_t l1,
                                     const double *phase1, const int32_t *idx1, int64_t k1,
                                     int64_t pad1, double mult1, double *y, int64_t ldy,
                                     int *nonfinite, srlu_stream_t stream) {
    SRLU_REQUIRE(m >= 1 && n >= 1 && l1 >= 1 && l1 <= n && k1 >= 1 && k1 <= pad1 &&
                     pow2(pad1) && pad1 >= l1 && ldy >= k1,
                 SRLU_ERR_ARG, "sketch_right_csr: bad sizes");
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == SRLU_F32)
        return launch_k1_csr<float>(indptr, indices, (const float *)vals, m, row_of1, sign1, l1,
                                    phase1, idx1, k1, pad1, mult1, y, ldy, nonfinite, s);
    if (dtype == SRLU_F64)
        return launch_k1_csr<double>(indptr, indices, (const double *)vals, m, row_of1, sign1, l1,
                                     phase1, idx1, k1, pad1, mult1, y, ldy, nonfinite, s);
    set_error("sketch_right_csr: unknown dtype %d", dtype);
    return SRLU_ERR_ARG;
}

extern "C" int srlu_fwht_rows(double *x, int64_t m, int64_t n, int64_t ldx, srlu_stream_t stream) {
    SRLU_REQUIRE(m >= 1 && pow2(n) && ldx >= n, SRLU_ERR_ARG,
                 "fwht_rows: need a power-of-two width");
    SRLU_REQUIRE(n <= 16384, SRLU_ERR_UNSUPPORTED, "fwht_rows: width > 16384");
    size_t smem = (size_t)n * 8;
    SRLU_CUDA(cudaFuncSetAttribute(fwht_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    int64_t grid = m < 148 * 8 ? m : 148 * 8;
    fwht_rows_kernel<<<(unsigned)grid, 256, smem, (cudaStream_t)stream>>>(x, m, (int)n, ldx);
    SRLU_CHECK_LAUNCH("fwht_rows_kernel");
    return SRLU_OK;
}
