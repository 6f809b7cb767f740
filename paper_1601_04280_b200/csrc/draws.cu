// K0 — seed-derived sketch draws, bit-exact with the reference's numpy
// Generator(Philox(seed)) (sketch.py:42-43, :103-114, :214-235).
//
//  * srlu_seed_key: numpy SeedSequence entropy pool -> 2 x uint64 key (host).
//  * srlu_draw_sem: n bucket draws via Lemire's bounded multiply with
//    rejection, then n sign draws, on the device.  Rejections make the
//    stream position of draw i data dependent: kernel 1 finds the (rare)
//    rejected positions, kernel 2 sorts them, kernel 3 maps draw i to its
//    position by skipping them.
//  * srlu_draw_fast_transform: +-1 phases then Fisher-Yates of arange(pad)
//    (numpy Generator.permutation) on the host — pad sequential swaps.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"

namespace srlu {

static const uint32_t kInitA = 0x43B0D7E5u, kMultA = 0x931E8875u;
static const uint32_t kInitB = 0x8B51F9DDu, kMultB = 0x58F38DEDu;
static const uint32_t kMixL = 0xCA01F9DDu, kMixR = 0x4973F715u;

static void seed_sequence_key(uint64_t seed, uint64_t key[2]) {
    uint32_t ent[2];
    int nent = 0;
    if (seed == 0) {
        ent[nent++] = 0;
    } else {
        while (seed) {
            ent[nent++] = (uint32_t)seed;
            seed >>= 32;
        }
    }
    uint32_t hc = kInitA;
    auto hashmix = [&](uint32_t v) {
        v ^= hc;
        hc *= kMultA;
        v *= hc;
        v ^= v >> 16;
        return v;
    };
    auto mix = [](uint32_t x, uint32_t y) {
        uint32_t r = kMixL * x - kMixR * y;
        r ^= r >> 16;
        return r;
    };
    uint32_t pool[4];
    for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < nent ? ent[i] : 0u);
    for (int s = 0; s < 4; ++s)
        for (int d = 0; d < 4; ++d)
            if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
    uint32_t hb = kInitB, w[4];
    for (int i = 0; i < 4; ++i) {
        uint32_t v = pool[i];
        v ^= hb;
        hb *= kMultB;
        v *= hb;
        v ^= v >> 16;
        w[i] = v;
    }
    key[0] = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
    key[1] = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
}

// sequential host consumer of the uint32 stream
struct HostStream {
    uint64_t k0, k1, pos = 0, blk = ~0ULL;
    uint64_t buf[4];
    uint32_t next() {
        uint64_t b = pos / 8;
        if (b != blk) {
            philox4x64_10(b + 1, k0, k1, buf);
            blk = b;
        }
        uint64_t w = buf[(pos % 8) / 2];
        uint32_t r = (pos & 1) ? (uint32_t)(w >> 32) : (uint32_t)w;
        ++pos;
        return r;
    }
};

// stream slack scanned beyond n: 1024 + 8x the expected rejection count
static int64_t reject_cap(int64_t n, int64_t l) {
    double e = (double)(n + 1024) * (double)l / 4294967296.0;
    return 1024 + 8 * (int64_t)ceil(e);
}

// kernel 1: rejected positions of integers(0, l) in [0, n + kMaxRejects)
__global__ void find_rejects_kernel(uint64_t k0, uint64_t k1, uint32_t l, uint32_t thresh,
                                    int64_t npos, uint32_t *rej, uint32_t *nrej, uint32_t cap) {
    int64_t blk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (blk * 8 >= npos) return;
    uint64_t o[4];
    philox4x64_10((uint64_t)blk + 1, k0, k1, o);
#pragma unroll
    for (int h = 0; h < 8; ++h) {
        int64_t q = blk * 8 + h;
        if (q >= npos) break;
        uint32_t w = (h & 1) ? (uint32_t)(o[h / 2] >> 32) : (uint32_t)o[h / 2];
        uint64_t mm = (uint64_t)w * l;
        uint32_t lo = (uint32_t)mm;
        if (lo < l && lo < thresh) {
            uint32_t slot = atomicAdd(nrej, 1u);
            if (slot < cap) rej[slot] = (uint32_t)q;
        }
    }
}

// kernel 2: sort the rejection list (tiny) and compute the sign-stream start
__global__ void sort_rejects_kernel(uint32_t *rej, const uint32_t *nrej, int64_t n, int has_draws,
                                    int64_t *sign_start, int *overflow, uint32_t cap) {
    uint32_t c = *nrej;
    if (c >= cap) {  // not reachable in practice (Poisson tail); flagged
        *overflow = 1;
        c = cap;
    }
    for (uint32_t i = 1; i < c; ++i) {
        uint32_t v = rej[i];
        int j = (int)i - 1;
        while (j >= 0 && rej[j] > v) {
            rej[j + 1] = rej[j];
            --j;
        }
        rej[j + 1] = v;
    }
    if (!has_draws) {
        *sign_start = 0;
        return;
    }
    // position of draw n-1, then +1
    uint64_t q = (uint64_t)(n - 1);
    for (uint32_t i = 0; i < c; ++i) {
        if (rej[i] <= q) ++q;
        else break;
    }
    *sign_start = (int64_t)q + 1;
}

// kernel 3: draw i -> bucket, sign
__global__ void draw_sem_kernel(uint64_t k0, uint64_t k1, uint32_t l, int64_t n,
                                const uint32_t *rej, const uint32_t *nrej,
                                const int64_t *sign_start, int32_t *row_of, double *sign,
                                uint32_t cap) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (l > 1) {
        uint32_t c = min(*nrej, cap);
        uint64_t q = (uint64_t)i;
        for (uint32_t r = 0; r < c; ++r) {
            if (rej[r] <= q) ++q;
            else break;
        }
        uint32_t w = philox_u32_at(k0, k1, q);
        row_of[i] = (int32_t)(((uint64_t)w * l) >> 32);
    } else {
        row_of[i] = 0;  // integers(0, 1) consumes no draws
    }
    uint32_t s = philox_u32_at(k0, k1, (uint64_t)(*sign_start + i));
    sign[i] = (s >> 31) ? 1.0 : -1.0;  // integers(0,2): (w*2)>>32 = top bit
}

}  // namespace srlu

using namespace srlu;

extern "C" int srlu_seed_key(uint64_t seed, uint64_t key[2]) {
    SRLU_REQUIRE(key != nullptr, SRLU_ERR_ARG, "srlu_seed_key: null key");
    seed_sequence_key(seed, key);
    return SRLU_OK;
}

extern "C" int srlu_draw_fast_transform(uint64_t seed, int64_t k, int64_t l, double *phase,
                                        int64_t *sample_idx, int64_t *pad_out) {
    SRLU_REQUIRE(l >= 1, SRLU_ERR_ARG, "build_fast_transform: need l >= 1, got %lld",
                 (long long)l);
    int64_t pad = 1;
    while (pad < l) pad <<= 1;
    SRLU_REQUIRE(k >= 1 && k <= pad, SRLU_ERR_ARG,
                 "build_fast_transform: need 1 <= k <= %lld, got k=%lld", (long long)pad,
                 (long long)k);
    SRLU_REQUIRE(pad <= (1 << 24), SRLU_ERR_UNSUPPORTED, "build_fast_transform: pad too large");
    uint64_t key[2];
    seed_sequence_key(seed, key);
    HostStream s{key[0], key[1]};
    for (int64_t i = 0; i < l; ++i) phase[i] = (s.next() >> 31) ? 1.0 : -1.0;
    int64_t *a = (int64_t *)malloc(sizeof(int64_t) * pad);
    SRLU_REQUIRE(a != nullptr, SRLU_ERR_ARG, "build_fast_transform: out of host memory");
    for (int64_t i = 0; i < pad; ++i) a[i] = i;
    for (int64_t i = pad - 1; i > 0; --i) {
        uint64_t mask = (uint64_t)i;
        mask |= mask >> 1;
        mask |= mask >> 2;
        mask |= mask >> 4;
        mask |= mask >> 8;
        mask |= mask >> 16;
        mask |= mask >> 32;
        uint64_t v;
        while ((v = (s.next() & mask)) > (uint64_t)i) {
        }
        int64_t t = a[i];
        a[i] = a[v];
        a[v] = t;
    }
    memcpy(sample_idx, a, sizeof(int64_t) * k);
    free(a);
    *pad_out = pad;
    return SRLU_OK;
}

extern "C" size_t srlu_draw_sem_workspace(int64_t n, int64_t l) {
    return sizeof(uint32_t) * (size_t)(reject_cap(n, l) + 16) + 64;
}

extern "C" int srlu_draw_sem(uint64_t seed, int64_t l, int64_t n, int32_t *row_of, double *sign,
                             void *ws, size_t ws_bytes, srlu_stream_t stream_) {
    cudaStream_t stream = (cudaStream_t)stream_;
    SRLU_REQUIRE(l >= 1 && l <= n, SRLU_ERR_ARG, "build_sem: need 1 <= k <= n, got k=%lld, n=%lld",
                 (long long)l, (long long)n);
    int64_t cap64 = reject_cap(n, l);
    SRLU_REQUIRE(l < (1LL << 31) && n + cap64 < (1LL << 32), SRLU_ERR_UNSUPPORTED,
                 "build_sem: sizes beyond 32-bit stream positions");
    SRLU_REQUIRE(ws_bytes >= srlu_draw_sem_workspace(n, l), SRLU_ERR_WORKSPACE,
                 "draw_sem: workspace too small");
    uint32_t cap = (uint32_t)cap64;
    uint64_t key[2];
    seed_sequence_key(seed, key);
    char *w = (char *)ws;
    uint32_t *rej = (uint32_t *)w;
    uint32_t *nrej = rej + cap;
    int *overflow = (int *)(nrej + 1);
    int64_t *sign_start = (int64_t *)(((uintptr_t)(nrej + 4) + 7) & ~(uintptr_t)7);
    SRLU_CUDA(cudaMemsetAsync(nrej, 0, 4 * sizeof(uint32_t), stream));
    uint32_t ul = (uint32_t)l;
    if (l > 1) {
        uint32_t thresh = (uint32_t)((0x100000000ULL - ul) % ul);
        int64_t npos = n + cap64;
        int64_t nblk = ceil_div(npos, 8);
        find_rejects_kernel<<<(unsigned)ceil_div(nblk, 256), 256, 0, stream>>>(
            key[0], key[1], ul, thresh, npos, rej, nrej, cap);
        SRLU_CHECK_LAUNCH("find_rejects_kernel");
    }
    sort_rejects_kernel<<<1, 1, 0, stream>>>(rej, nrej, n, l > 1, sign_start, overflow, cap);
    SRLU_CHECK_LAUNCH("sort_rejects_kernel");
    draw_sem_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, stream>>>(key[0], key[1], ul, n, rej,
                                                                    nrej, sign_start, row_of, sign,
                                                                    cap);
    SRLU_CHECK_LAUNCH("draw_sem_kernel");
    return SRLU_OK;
}

// ---------------------------------------------------------------------------
// build_composite (sketch.py:269-278) in one call: the transform stage's
// draws on the host (sequential Fisher-Yates, as numpy) into the caller's
// pinned staging buffer and uploaded on `stream`, then the sparse stage's
// device draws and its accumulation plan — one host entry instead of the
// dozen allocations / copies / launches of the separate calls.

static size_t align256(size_t n) { return (n + 255) & ~(size_t)255; }

extern "C" size_t srlu_build_composite_workspace(int64_t n, int64_t l) {
    return align256(srlu_draw_sem_workspace(n, l)) + align256(srlu_sem_plan_workspace(n, l));
}

extern "C" size_t srlu_build_composite_staging(int64_t k, int64_t l) {
    return sizeof(double) * (size_t)l + sizeof(int64_t) * (size_t)k + sizeof(int32_t) * (size_t)k + 64;
}

// device half: sparse-stage draws and the accumulation plan
static int composite_device(uint64_t seed, int64_t l, int64_t n, int32_t *row_of, double *sign,
                            int32_t *sorted, int32_t *bucket_ptr, void *ws, size_t ws_bytes,
                            srlu_stream_t stream) {
    SRLU_REQUIRE(ws_bytes >= srlu_build_composite_workspace(n, l), SRLU_ERR_WORKSPACE,
                 "build_composite: workspace too small");
    char *w = (char *)ws;
    const size_t ws_sem = align256(srlu_draw_sem_workspace(n, l));
    int rc = srlu_draw_sem(seed, l, n, row_of, sign, w, ws_sem, stream);
    if (rc != SRLU_OK) return rc;
    return srlu_sem_plan(row_of, sign, n, l, sorted, bucket_ptr, w + ws_sem, ws_bytes - ws_sem,
                         stream);
}

// host half: the transform stage (seed + 2**32, sketch.py:36, :276) drawn
// sequentially like numpy into the pinned staging buffer, uploaded in one
// copy.  Staging layout: phase[l] f64 | idx32[k] | idx64[k]; when phase and
// sample_idx are adjacent on the device (sample_idx == phase + l) both go up
// in a single copy.
static int composite_host(uint64_t seed, int64_t k, int64_t l, double *phase, int32_t *sample_idx,
                          int64_t *pad, void *staging, size_t staging_bytes, srlu_stream_t stream) {
    SRLU_REQUIRE(staging_bytes >= srlu_build_composite_staging(k, l), SRLU_ERR_WORKSPACE,
                 "build_composite: staging too small");
    cudaStream_t s = (cudaStream_t)stream;
    double *ph = (double *)staging;
    int32_t *idx32 = (int32_t *)(ph + l);
    int64_t *idx64 = (int64_t *)(((uintptr_t)(idx32 + k) + 7) & ~(uintptr_t)7);
    int rc = srlu_draw_fast_transform(seed + (1ULL << 32), k, l, ph, idx64, pad);
    if (rc != SRLU_OK) return rc;
    for (int64_t i = 0; i < k; ++i) idx32[i] = (int32_t)idx64[i];
    if ((void *)sample_idx == (void *)(phase + l)) {
        SRLU_CUDA(cudaMemcpyAsync(phase, ph, sizeof(double) * (size_t)l + sizeof(int32_t) * (size_t)k,
                                  cudaMemcpyHostToDevice, s));
    } else {
        SRLU_CUDA(cudaMemcpyAsync(phase, ph, sizeof(double) * (size_t)l, cudaMemcpyHostToDevice, s));
        SRLU_CUDA(cudaMemcpyAsync(sample_idx, idx32, sizeof(int32_t) * (size_t)k,
                                  cudaMemcpyHostToDevice, s));
    }
    return SRLU_OK;
}

extern "C" int srlu_build_composite(uint64_t seed, int64_t k, int64_t l, int64_t n, int32_t *row_of,
                                    double *sign, int32_t *sorted, int32_t *bucket_ptr,
                                    double *phase, int32_t *sample_idx, int64_t *pad,
                                    void *staging, size_t staging_bytes, void *ws, size_t ws_bytes,
                                    srlu_stream_t stream) {
    // device work first (the GPU starts while the host draws the transform)
    int rc = composite_device(seed, l, n, row_of, sign, sorted, bucket_ptr, ws, ws_bytes, stream);
    if (rc != SRLU_OK) return rc;
    return composite_host(seed, k, l, phase, sample_idx, pad, staging, staging_bytes, stream);
}

extern "C" size_t srlu_k1_schedule_bytes(int64_t n, int64_t l1, int64_t pad1, int dtype);
extern "C" int srlu_k1_schedule(const int32_t *sorted1, const int32_t *bucket_ptr1, int64_t n,
                                int64_t l1, int64_t pad1, int dtype, void *sched,
                                size_t sched_bytes, srlu_stream_t stream);

extern "C" int srlu_build_composite_k1(uint64_t seed, int64_t k, int64_t l, int64_t n,
                                       int32_t *row_of, double *sign, int32_t *sorted,
                                       int32_t *bucket_ptr, double *phase, int32_t *sample_idx,
                                       int64_t *pad, void *staging, size_t staging_bytes, void *ws,
                                       size_t ws_bytes, int dtype, void *sched, size_t sched_bytes,
                                       srlu_stream_t stream) {
    // device draws, plan and the K1 schedule (which needs only the plan) are
    // all enqueued before the host draws the transform stage
    int rc = composite_device(seed, l, n, row_of, sign, sorted, bucket_ptr, ws, ws_bytes, stream);
    if (rc != SRLU_OK) return rc;
    if (sched != nullptr) {
        int64_t pad1 = 1;
        while (pad1 < l) pad1 <<= 1;
        rc = srlu_k1_schedule(sorted, bucket_ptr, n, l, pad1, dtype, sched, sched_bytes, stream);
        if (rc != SRLU_OK) return rc;
    }
    return composite_host(seed, k, l, phase, sample_idx, pad, staging, staging_bytes, stream);
}

extern "C" int srlu_sketch_right_dense_sched(const void *a, int dtype, int64_t m, int64_t n,
                                             int64_t lda, const void *sched, size_t sched_bytes,
                                             int64_t l1, const double *phase1, const int32_t *idx1,
                                             int64_t k1, int64_t pad1, double mult1, double *y,
                                             int64_t ldy, int *nonfinite, srlu_stream_t stream);
extern "C" int srlu_sketch_right_dense(const void *a, int dtype, int64_t m, int64_t n, int64_t lda,
                                       const int32_t *sorted1, const int32_t *bucket_ptr1,
                                       int64_t l1, const double *phase1, const int32_t *idx1,
                                       int64_t k1, int64_t pad1, double mult1, double *y,
                                       int64_t ldy, int *nonfinite, srlu_stream_t stream);

// Stage 1 of an attempt (randlu.py:252 build_composite + :253 apply_sketch_right)
// in one host entry: the composite draws, plan and K1 schedule, the
// non-finite flag reset and the K1 launch are enqueued back to back, so the
// sketch kernel does not wait on the caller's bookkeeping between them.
extern "C" int srlu_composite_sketch_right_dense(
    uint64_t seed, int64_t k, int64_t l, int64_t n, int32_t *row_of, double *sign,
    int32_t *sorted, int32_t *bucket_ptr, double *phase, int32_t *sample_idx, int64_t *pad,
    void *staging, size_t staging_bytes, void *ws, size_t ws_bytes, void *sched,
    size_t sched_bytes, const void *a, int dtype, int64_t m, int64_t lda, double mult, double *y,
    int64_t ldy, int *nonfinite, srlu_stream_t stream) {
    SRLU_REQUIRE(a != nullptr && y != nullptr && nonfinite != nullptr, SRLU_ERR_ARG,
                 "composite_sketch_right_dense: null A, Y or flag");
    int rc = srlu_build_composite_k1(seed, k, l, n, row_of, sign, sorted, bucket_ptr, phase,
                                     sample_idx, pad, staging, staging_bytes, ws, ws_bytes, dtype,
                                     sched, sched_bytes, stream);
    if (rc != SRLU_OK) return rc;
    SRLU_CUDA(cudaMemsetAsync(nonfinite, 0, sizeof(int), (cudaStream_t)stream));
    if (sched != nullptr)
        return srlu_sketch_right_dense_sched(a, dtype, m, n, lda, sched, sched_bytes, l, phase,
                                             sample_idx, k, *pad, mult, y, ldy, nonfinite, stream);
    return srlu_sketch_right_dense(a, dtype, m, n, lda, sorted, bucket_ptr, l, phase, sample_idx, k,
                                   *pad, mult, y, ldy, nonfinite, stream);
}
