// cp.async (LDGSTS) helpers: global -> shared copies with zero fill.
#pragma once
#include "common.cuh"

namespace srlu {

__device__ inline void cp_async_16(void *smem, const void *gmem, bool valid) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(sz)
                 : "memory");
}

template <int BYTES>
__device__ inline void cp_async_small(void *smem, const void *gmem, bool valid) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    int sz = valid ? BYTES : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(s), "l"(gmem), "n"(BYTES),
                 "r"(sz)
                 : "memory");
}

__device__ inline void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

template <int N>
__device__ inline void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Stage rows [row0, row0+R) x cols [c0, c0+C) of a row-major matrix into
// tile[R][C] (zero-filled outside the matrix).
template <typename T, int R, int C, int NT>
__device__ inline void load_tile_async(T *tile, const T *a, int64_t m, int64_t n, int64_t lda,
                                       int64_t row0, int64_t c0, bool vec_ok) {
    constexpr int V = 16 / sizeof(T);
    static_assert(C % V == 0, "chunk must be a multiple of the vector width");
    if (vec_ok) {
        for (int idx = threadIdx.x; idx < R * (C / V); idx += NT) {
            int r = idx / (C / V), cv = idx % (C / V);
            int64_t row = row0 + r, col = c0 + (int64_t)cv * V;
            T *dst = tile + r * C + cv * V;
            const T *src = a + row * lda + col;
            if (row < m && col + V <= n) {
                cp_async_16(dst, src, true);
            } else if (row < m && col < n) {
#pragma unroll
                for (int e = 0; e < V; ++e)
                    cp_async_small<sizeof(T)>(dst + e, col + e < n ? src + e : a, col + e < n);
            } else {
                cp_async_16(dst, a, false);
            }
        }
    } else {
        for (int idx = threadIdx.x; idx < R * C; idx += NT) {
            int r = idx / C, c = idx % C;
            int64_t row = row0 + r, col = c0 + c;
            bool ok = row < m && col < n;
            cp_async_small<sizeof(T)>(tile + idx, ok ? a + row * lda + col : a, ok);
        }
    }
}

}  // namespace srlu
