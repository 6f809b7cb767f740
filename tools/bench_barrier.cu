// Microbenchmark: cost of one grid-wide barrier (+ candidate exchange) for a
// persistent cooperative kernel with one CTA per SM.  Used to pick the
// barrier used by lu.cu.  Build: nvcc -cudart shared -gencode arch=compute_100a,code=sm_100a -O3
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <int V>
__global__ void barrier_kernel(unsigned *counter, unsigned *flags, unsigned long long *cand,
                               double *rows, int rounds, unsigned long long *out) {
    const int G = gridDim.x;
    unsigned target = 0;
    long long t0 = clock64();
    __shared__ double u[128];
    for (int r = 0; r < rounds; ++r) {
        if (V >= 4) {  // publish a candidate (key + 110-double row)
            if (threadIdx.x < 110) rows[((size_t)(r & 1) * G + blockIdx.x) * 128 + threadIdx.x] = r + threadIdx.x;
            if (threadIdx.x == 0) cand[(r & 1) * G + blockIdx.x] = (unsigned long long)r * 1000 + blockIdx.x;
        }
        __syncthreads();
        target += G;
        if (threadIdx.x == 0) {
            if (V == 1) {
                __threadfence();
                atomicAdd(counter, 1u);
                while ((int)(ld_acquire(counter) - target) < 0) {}
            } else if (V == 2 || V == 4) {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
                while ((int)(ld_acquire(counter) - target) < 0) {}
            } else {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
                while ((int)(ld_relaxed(counter) - target) < 0) {}
            }
        }
        __syncthreads();
        if (V >= 4 && threadIdx.x < 32) {  // warp 0: read all candidates, pick max, read its row
            unsigned long long best = 0;
            int bc = 0;
            for (int c = threadIdx.x; c < G; c += 32) {
                unsigned long long v = __ldcg(cand + (r & 1) * G + c);
                if (v > best) { best = v; bc = c; }
            }
            for (int off = 16; off; off >>= 1) {
                unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, off);
                int oc = __shfl_xor_sync(0xffffffffu, bc, off);
                if (ob > best) { best = ob; bc = oc; }
            }
            for (int x = threadIdx.x; x < 110; x += 32) u[x] = __ldcg(rows + ((size_t)(r & 1) * G + bc) * 128 + x);
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
}

template <int V>
void run(int G, int rounds) {
    unsigned *counter, *flags;
    unsigned long long *cand, *out;
    double *rows;
    cudaMalloc(&counter, 4);
    cudaMalloc(&flags, 4 * 1024);
    cudaMalloc(&cand, 8 * 2 * 1024);
    cudaMalloc(&rows, 8 * 2 * 1024 * 128);
    cudaMalloc(&out, 8);
    cudaMemset(counter, 0, 4);
    void *args[] = {&counter, &flags, &cand, &rows, &rounds, &out};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void *)barrier_kernel<V>, G, 256, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long cyc;
    cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
    printf("variant %d grid %d: %.3f us/round (%.0f cycles/round) err=%s\n", V, G, ms * 1e3 / rounds,
           (double)cyc / rounds, cudaGetErrorString(cudaGetLastError()));
    cudaFree(counter); cudaFree(flags); cudaFree(cand); cudaFree(rows); cudaFree(out);
}

int main() {
    int G = 148, R = 2000;
    run<1>(G, R); run<2>(G, R); run<3>(G, R); run<4>(G, R); run<5>(G, R);
    run<3>(74, R); run<5>(74, R); run<3>(16, R); run<5>(16, R);
    return 0;
}
