// Microbenchmarks behind the TMEM-accumulator stage-1 sketch kernel (K1T):
//  (A) read-modify-write of fp64 accumulators kept in tensor memory
//      (tcgen05.ld.32x32b.x2 -> DADD -> tcgen05.st.32x32b.x2, lanes = rows),
//      cycles per warp step per SM for 8..32 warps, serialised waits or
//      four independent slots per wait;
//  (B) LDG.32 -> STS.32 streaming of a row-major fp32 matrix into a padded
//      (odd pitch) shared-memory tile by NL loader warps per SM: GB/s.
// Build (on the GPU box, tools/bin/ never ships):
//   nvcc -cudart shared -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/bench_tmem.cu -o /tmp/bench_tmem
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void tm_ld2(unsigned taddr, unsigned &lo, unsigned &hi) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
                 : "=r"(lo), "=r"(hi) : "r"(taddr) : "memory");
}
__device__ __forceinline__ void tm_st2(unsigned taddr, unsigned lo, unsigned hi) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};"
                 :: "r"(taddr), "r"(lo), "r"(hi) : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// MODE 0: one slot per wait pair; MODE 1: four independent slots per wait pair;
// MODE 2: like 0 but no wait::st (is a later ld of the same slot ordered? checked by the sum)
template <int MODE>
__global__ void __launch_bounds__(1024, 1) rmw_kernel(int iters, long long *cycles, double *out) {
    __shared__ unsigned tbase;
    const int warp = threadIdx.x / 32, nw = blockDim.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned q = warp & 3, grp = warp >> 2, ngrp = (nw + 3) / 4;
    const unsigned ncol = 512 / ngrp & ~1u;           // columns of this warp
    const unsigned base = tbase + ((q * 32u) << 16) + grp * ncol;
    const unsigned nslot = ncol / 2;
    for (unsigned s = 0; s < nslot; ++s) tm_st2(base + 2 * s, 0u, 0u);
    tm_wait_st();
    __syncthreads();
    const double inc = 1.0 + threadIdx.x;
    long long t0 = clock64();
    unsigned h = 12345u + warp;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 1) {
            unsigned s0 = (h >> 3) % (nslot / 4) * 4;
            unsigned lo[4], hi[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) tm_ld2(base + 2 * (s0 + u), lo[u], hi[u]);
            tm_wait_ld();
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                double v = __hiloint2double(hi[u], lo[u]);
                v = __dadd_rn(v, inc);
                tm_st2(base + 2 * (s0 + u), __double2loint(v), __double2hiint(v));
            }
            tm_wait_st();
        } else {
            unsigned s0 = (h >> 3) % nslot;
            unsigned lo, hi;
            tm_ld2(base + 2 * s0, lo, hi);
            tm_wait_ld();
            double v = __hiloint2double(hi, lo);
            v = __dadd_rn(v, inc);
            tm_st2(base + 2 * s0, __double2loint(v), __double2hiint(v));
            if (MODE == 0) tm_wait_st();
        }
        h = h * 1664525u + 1013904223u;
    }
    tm_wait_st();
    long long t1 = clock64();
    double sum = 0;
    for (unsigned s = 0; s < nslot; ++s) {
        unsigned lo, hi;
        tm_ld2(base + 2 * s, lo, hi);
        tm_wait_ld();
        sum += __hiloint2double(hi, lo);
    }
    if (threadIdx.x % 32 == 0 && blockIdx.x == 0) cycles[warp] = t1 - t0;
    // every step adds inc once (MODE 1: four times)
    const double expect = inc * (double)iters * (MODE == 1 ? 4 : 1);
    if (sum != expect) out[0] = sum;   // flag a lost update
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
}

// (B) loader: each loader warp copies 32-column pieces of RB rows into a tile
// with pitch C+1 words, U loads in flight per thread.
template <int U>
__global__ void __launch_bounds__(1024, 1) load_kernel(const float *a, long long m, int n, int rb, int c,
                                                       float *sink) {
    extern __shared__ float tile[];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
    const int pitch = c + 1;
    const int pieces_per_row = c / 32;               // 32-column pieces per row of a chunk
    const int nchunk = n / c;
    const long long nblk = m / rb;
    float acc = 0.f;
    for (long long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        for (int ch = 0; ch < nchunk; ++ch) {
            float *st = tile + (size_t)((ch & 1) * rb) * pitch;
            const float *src = a + blk * rb * (long long)n + (long long)ch * c;
            const int npieces = rb * pieces_per_row;
            for (int p0 = warp * U; p0 < npieces; p0 += nw * U) {
                float v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int p = p0 + u, r = p / pieces_per_row, cc = (p % pieces_per_row) * 32 + lane;
                    v[u] = p < npieces ? __ldcs(src + (long long)r * n + cc) : 0.f;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int p = p0 + u, r = p / pieces_per_row, cc = (p % pieces_per_row) * 32 + lane;
                    if (p < npieces) st[r * pitch + cc] = v[u];
                }
            }
        }
    }
    __syncthreads();
    acc = tile[threadIdx.x];
    if (acc == 123.456f) sink[0] = acc;
}

int main() {
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    long long *cyc;
    double *out;
    cudaMalloc(&cyc, 32 * 8);
    cudaMalloc(&out, 8);
    cudaMemset(out, 0, 8);
    const int iters = 20000;
    for (int mode = 0; mode < 3; ++mode)
        for (int nw : {8, 16, 24, 32}) {
            long long h[32];
            for (int rep = 0; rep < 2; ++rep) {
                if (mode == 0) rmw_kernel<0><<<148, nw * 32>>>(iters, cyc, out);
                if (mode == 1) rmw_kernel<1><<<148, nw * 32>>>(iters, cyc, out);
                if (mode == 2) rmw_kernel<2><<<148, nw * 32>>>(iters, cyc, out);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("rmw mode %d nw %d: %s\n", mode, nw, cudaGetErrorString(e)); return 1; }
            }
            cudaMemcpy(h, cyc, nw * 8, cudaMemcpyDeviceToHost);
            double o;
            cudaMemcpy(&o, out, 8, cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int w = 0; w < nw; ++w) mx = h[w] > mx ? h[w] : mx;
            const double steps = (double)iters * nw * (mode == 1 ? 4 : 1);
            printf("RMW mode %d warps %2d: %.1f cycles per warp-iteration, %.2f cycles per slot-RMW per SM, lost-update flag %g\n",
                   mode, nw, (double)mx / iters, (double)mx / steps, o);
            cudaMemset(out, 0, 8);
        }
    // (B)
    const long long m = 16384;
    const int n = 16384;
    float *a, *sink;
    cudaMalloc(&a, m * n * 4);
    cudaMalloc(&sink, 4);
    cudaMemset(a, 0, m * n * 4);
    for (int rb : {32}) for (int c : {256, 512}) for (int nl : {8, 12, 16, 32}) {
        const size_t smem = (size_t)2 * rb * (c + 1) * 4;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int uu : {8, 16, 32}) {
            float best = 1e9;
            for (int rep = 0; rep < 4; ++rep) {
                cudaEventRecord(e0);
                if (uu == 8) {
                    cudaFuncSetAttribute(load_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    load_kernel<8><<<148, nl * 32, smem>>>(a, m, n, rb, c, sink);
                } else if (uu == 16) {
                    cudaFuncSetAttribute(load_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    load_kernel<16><<<148, nl * 32, smem>>>(a, m, n, rb, c, sink);
                } else {
                    cudaFuncSetAttribute(load_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    load_kernel<32><<<148, nl * 32, smem>>>(a, m, n, rb, c, sink);
                }
                cudaEventRecord(e1);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("load: %s\n", cudaGetErrorString(e)); return 1; }
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
            }
            printf("LOAD rb %d c %d loader warps %2d U %2d: %.3f ms  %.0f GB/s\n", rb, c, nl, uu, best,
                   (double)m * n * 4 / best * 1e-6);
        }
    }
    return 0;
}
