// Shared device helpers for the sm_100a sparse-randomized-LU kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/srlu.h"

namespace srlu {

// Per-thread last error (set by the C-ABI wrappers, read by srlu_last_error).
void set_error(const char *fmt, ...);

#define SRLU_CHECK_LAUNCH(what)                                                  \
    do {                                                                         \
        cudaError_t e_ = cudaGetLastError();                                     \
        if (e_ != cudaSuccess) {                                                 \
            ::srlu::set_error("%s: %s", what, cudaGetErrorString(e_));           \
            return SRLU_ERR_CUDA;                                                \
        }                                                                        \
    } while (0)

#define SRLU_CUDA(call)                                                          \
    do {                                                                         \
        cudaError_t e_ = (call);                                                 \
        if (e_ != cudaSuccess) {                                                 \
            ::srlu::set_error("%s: %s", #call, cudaGetErrorString(e_));          \
            return SRLU_ERR_CUDA;                                                \
        }                                                                        \
    } while (0)

#define SRLU_REQUIRE(cond, code, ...)                                            \
    do {                                                                         \
        if (!(cond)) {                                                           \
            ::srlu::set_error(__VA_ARGS__);                                      \
            return code;                                                         \
        }                                                                        \
    } while (0)

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------------------
// Philox4x64-10 (Random123), numpy's Philox bit generator: block b (1-based
// counter [b,0,0,0]) yields 4 uint64; the uint32 stream takes the low then
// the high half of each.  Reference: sketch.py:42-43 (_rng).

__host__ __device__ inline void philox4x64_10(uint64_t c0, uint64_t key0, uint64_t key1,
                                              uint64_t out[4]) {
    uint64_t x0 = c0, x1 = 0, x2 = 0, x3 = 0;
    uint64_t k0 = key0, k1 = key1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B97F4A7C15ULL;
            k1 += 0xBB67AE8584CAA73BULL;
        }
        const uint64_t m0 = 0xD2E7470EE14C6C93ULL, m1 = 0xCA5A826395121157ULL;
#ifdef __CUDA_ARCH__
        uint64_t hi0 = __umul64hi(m0, x0), lo0 = m0 * x0;
        uint64_t hi1 = __umul64hi(m1, x2), lo1 = m1 * x2;
#else
        unsigned __int128 p0 = (unsigned __int128)m0 * x0;
        unsigned __int128 p1 = (unsigned __int128)m1 * x2;
        uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
        uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
#endif
        uint64_t n0 = hi1 ^ x1 ^ k0, n1 = lo1, n2 = hi0 ^ x3 ^ k1, n3 = lo0;
        x0 = n0; x1 = n1; x2 = n2; x3 = n3;
    }
    out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

// uint32 at stream position q
__host__ __device__ inline uint32_t philox_u32_at(uint64_t key0, uint64_t key1, uint64_t q) {
    uint64_t o[4];
    philox4x64_10(q / 8 + 1, key0, key1, o);
    uint64_t w = o[(q % 8) / 2];
    return (q & 1) ? (uint32_t)(w >> 32) : (uint32_t)w;
}

// ---------------------------------------------------------------------------
// Grid-wide barrier for persistent (cooperatively launched) kernels.  The
// counter is monotonically increasing; `target` = (#barriers so far) * grid.

__device__ inline void grid_arrive_wait(unsigned int *counter, unsigned int target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(counter, 1u);
        unsigned int v;
        while (true) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
            if ((int)(v - target) >= 0) break;
            __nanosleep(32);
        }
    }
    __syncthreads();
}

// The same barrier in two halves: arrive (all of the CTA's prior global
// writes are published), then — after independent work — wait.
__device__ inline void grid_arrive(unsigned int *counter) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(counter, 1u);
    }
}

__device__ inline void grid_wait(unsigned int *counter, unsigned int target) {
    if (threadIdx.x == 0) {
        unsigned int v;
        while (true) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
            if ((int)(v - target) >= 0) break;
            __nanosleep(32);
        }
    }
    __syncthreads();
}

__device__ inline double ld_cg(const double *p) { return __ldcg(p); }

// a / b correctly rounded (bit-identical to the IEEE division) from the
// correctly rounded reciprocal y = __drcp_rn(b), shared by many dividends:
// q0 = RN(a y), r = a - b q0 exact (FMA), q = RN(q0 + r y) (Markstein's
// correction).  Outside the range where the theorem's no-underflow /
// no-overflow conditions hold (and for zeros, inf, NaN) it takes the real
// division.  Checked bit for bit against a / b on 1e10 random, hard-rounding
// and edge-case pairs (tools/check_div.cu).
__device__ __forceinline__ double div_by_recip(double a, double b, double y) {
    const double fb = fabs(b), fa = fabs(a);
    if (!(fb >= 0x1p-1000 && fb <= 0x1p+1000 && fa >= 0x1p-960 && fa <= 0x1p+1000)) return a / b;
    const double q0 = __dmul_rn(a, y);
    const double fq = fabs(q0);
    if (!(fq >= 0x1p-960 && fq <= 0x1p+1000)) return a / b;
    const double r = __fma_rn(-b, q0, a);
    return __fma_rn(r, y, q0);
}

template <typename T> struct ValueTraits;
template <> struct ValueTraits<float> { static constexpr int code = SRLU_F32; };
template <> struct ValueTraits<double> { static constexpr int code = SRLU_F64; };

}  // namespace srlu
