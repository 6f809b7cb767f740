// Sparse-embedding plan: stable bucket sort of the sources of a sparse sign
// embedding.  The reference accumulates every (row, bucket) sum of
// sem_gather (_fast.pyx:44-54) and every (bucket, column) sum of
// sem_scatter (_fast.pyx:71-78) in ascending source index; the sorted
// member lists produced here let the K1/K3 kernels replay exactly that
// order without atomics (bit-exact sums).
#include "common.cuh"

namespace srlu {

constexpr int kPlanBlock = 256;  // sources per counting block (one warp each)

__global__ void plan_hist_kernel(const int32_t *row_of, int64_t n, int l, int *counts) {
    extern __shared__ int hist[];
    for (int t = threadIdx.x; t < l; t += blockDim.x) hist[t] = 0;
    __syncthreads();
    int64_t b0 = (int64_t)blockIdx.x * kPlanBlock;
    int64_t b1 = min(n, b0 + kPlanBlock);
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) atomicAdd(&hist[row_of[i]], 1);
    __syncthreads();
    for (int t = threadIdx.x; t < l; t += blockDim.x)
        counts[(int64_t)t * gridDim.x + blockIdx.x] = hist[t];
}

// one CTA per bucket: exclusive scan of its per-block counts; bucket totals
__global__ void plan_scan_blocks_kernel(int *counts, int nblk, int l, int *total) {
    __shared__ int warp_sums[32];
    __shared__ int carry;
    const int t = blockIdx.x;
    int *row = counts + (int64_t)t * nblk;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int b0 = 0; b0 < nblk; b0 += blockDim.x) {
        const int b = b0 + threadIdx.x;
        const int v = b < nblk ? row[b] : 0;
        int incl = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            int o = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += o;
        }
        if (lane == 31) warp_sums[warp] = incl;
        __syncthreads();
        int wbase = 0;
        for (int w = 0; w < warp; ++w) wbase += warp_sums[w];
        int tile_total = 0;
        for (int w = 0; w < nw; ++w) tile_total += warp_sums[w];
        const int c = carry;
        if (b < nblk) row[b] = c + wbase + incl - v;
        __syncthreads();
        if (threadIdx.x == 0) carry = c + tile_total;
        __syncthreads();
    }
    if (threadIdx.x == 0) total[t] = carry;
}

// single CTA: bucket_ptr = exclusive scan of totals (per-thread run, then a
// warp-shuffle block scan of the 1024 partial sums)
__global__ void __launch_bounds__(1024) plan_scan_buckets_kernel(const int *total, int l,
                                                                 int32_t *bucket_ptr) {
    __shared__ int wsum[32];
    const int nt = blockDim.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int per = (l + nt - 1) / nt;
    const int lo = threadIdx.x * per, hi = min(l, lo + per);
    int s = 0;
    for (int t = lo; t < hi; ++t) s += total[t];
    int incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int w = lane < (nt >> 5) ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += v;
        }
        wsum[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    int run = incl - s + (warp ? wsum[warp - 1] : 0);
    if (threadIdx.x == nt - 1) bucket_ptr[l] = run + s;
    for (int t = lo; t < hi; ++t) {
        bucket_ptr[t] = run;
        run += total[t];
    }
}

// one warp per block: ranks in ascending source order via match_any
__global__ void plan_scatter_kernel(const int32_t *row_of, const double *sign, int64_t n, int l,
                                    const int *counts, const int32_t *bucket_ptr,
                                    int32_t *sorted) {
    extern __shared__ int cursor[];
    int lane = threadIdx.x;
    for (int t = lane; t < l; t += 32)
        cursor[t] = bucket_ptr[t] + counts[(int64_t)t * gridDim.x + blockIdx.x];
    __syncwarp();
    int64_t b0 = (int64_t)blockIdx.x * kPlanBlock;
    int64_t b1 = min(n, b0 + kPlanBlock);
    unsigned lt_mask = (1u << lane) - 1u;
    // all of the block's draws in flight at once (kPlanBlock / 32 per lane)
    constexpr int NC = kPlanBlock / 32;
    int tv[NC];
    bool neg[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
        const int64_t i = b0 + q * 32 + lane;
        tv[q] = i < b1 ? row_of[i] : 0;
        neg[q] = i < b1 ? sign[i] < 0.0 : false;
    }
#pragma unroll
    for (int q = 0; q < NC; ++q) {
        int64_t i = b0 + q * 32 + lane;
        bool valid = i < b1;
        unsigned active = __ballot_sync(0xffffffffu, valid);
        if (valid) {
            int t = tv[q];
            unsigned peers = __match_any_sync(active, t);
            int rank = __popc(peers & lt_mask);
            int base = cursor[t];
            __syncwarp(active);
            int32_t code = (int32_t)i | (neg[q] ? (int32_t)0x80000000 : 0);
            sorted[base + rank] = code;
            if (rank == 0) cursor[t] = base + __popc(peers);
        }
        __syncwarp();
    }
}

__global__ void members_kernel(const int32_t *sorted2, int64_t m, const int64_t *perm,
                               int64_t row0, int64_t rows, int32_t *member_row,
                               double *member_sign) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    int32_t code = sorted2[e];
    int64_t q = code & 0x7FFFFFFF;
    int64_t row = perm ? perm[q] : q;
    row -= row0;
    member_row[e] = (row >= 0 && row < rows) ? (int32_t)row : -1;
    member_sign[e] = code < 0 ? -1.0 : 1.0;
}

}  // namespace srlu

using namespace srlu;

extern "C" size_t srlu_sem_plan_workspace(int64_t n, int64_t l) {
    int64_t nblk = ceil_div(n, kPlanBlock);
    return sizeof(int) * (size_t)(nblk * l + l) + 256;
}

extern "C" int srlu_sem_plan(const int32_t *row_of, const double *sign, int64_t n, int64_t l,
                             int32_t *sorted, int32_t *bucket_ptr, void *ws, size_t ws_bytes,
                             srlu_stream_t stream_) {
    cudaStream_t stream = (cudaStream_t)stream_;
    SRLU_REQUIRE(n >= 1 && l >= 1 && l <= n, SRLU_ERR_ARG, "sem_plan: bad sizes n=%lld l=%lld",
                 (long long)n, (long long)l);
    SRLU_REQUIRE(n < (1LL << 31) && l <= 50000, SRLU_ERR_UNSUPPORTED,
                 "sem_plan: n must be < 2^31 and l <= 50000");
    SRLU_REQUIRE(ws_bytes >= srlu_sem_plan_workspace(n, l), SRLU_ERR_WORKSPACE,
                 "sem_plan: workspace too small");
    int nblk = (int)ceil_div(n, kPlanBlock);
    int *counts = (int *)ws;
    int *total = counts + (int64_t)nblk * l;
    size_t smem = sizeof(int) * (size_t)l;
    if (smem > 48 * 1024) {
        SRLU_CUDA(cudaFuncSetAttribute(plan_hist_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        SRLU_CUDA(cudaFuncSetAttribute(plan_scatter_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    plan_hist_kernel<<<nblk, 256, smem, stream>>>(row_of, n, (int)l, counts);
    SRLU_CHECK_LAUNCH("plan_hist_kernel");
    plan_scan_blocks_kernel<<<(unsigned)l, 256, 0, stream>>>(counts, nblk, (int)l, total);
    SRLU_CHECK_LAUNCH("plan_scan_blocks_kernel");
    plan_scan_buckets_kernel<<<1, 1024, 0, stream>>>(total, (int)l, bucket_ptr);
    SRLU_CHECK_LAUNCH("plan_scan_buckets_kernel");
    plan_scatter_kernel<<<nblk, 32, smem, stream>>>(row_of, sign, n, (int)l, counts, bucket_ptr,
                                                    sorted);
    SRLU_CHECK_LAUNCH("plan_scatter_kernel");
    return SRLU_OK;
}

extern "C" int srlu_sem_members(const int32_t *sorted2, int64_t m, const int64_t *perm,
                                int64_t row0, int64_t rows, int32_t *member_row,
                                double *member_sign, srlu_stream_t stream_) {
    cudaStream_t stream = (cudaStream_t)stream_;
    SRLU_REQUIRE(m >= 1, SRLU_ERR_ARG, "sem_members: m must be positive");
    members_kernel<<<(unsigned)ceil_div(m, 256), 256, 0, stream>>>(sorted2, m, perm, row0, rows,
                                                                   member_row, member_sign);
    SRLU_CHECK_LAUNCH("members_kernel");
    return SRLU_OK;
}
