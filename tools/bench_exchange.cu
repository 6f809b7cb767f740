// Microbenchmark of one LU pivot exchange round (the per-step critical path
// of lu.cu): publish {key, 110-double row}, grid barrier, every CTA reduces
// the G keys and reads the winner row.  Variants of the fences / polling.
#include <cstdio>
#include <cstdint>

struct Cand { unsigned long long absbits; unsigned pos; int entity; };

template <int R>
__global__ void xchg12_kernel(unsigned *counter, Cand *cand, double *rows, int rounds, int k,
                              unsigned long long *out, double *sink) {
    const int G = gridDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned target = 0;
    __shared__ double u[2][640];
    long long t0 = clock64();
    unsigned long long seed = blockIdx.x * 2654435761ull;
    const int my = blockIdx.x % R;
    for (int r = 0; r < rounds; ++r) {
        const int slot = r & 1;
        if (warp == 0) {
            for (int rep = 0; rep < R; ++rep) {
                double *crow = rows + (((size_t)rep * 2 + slot) * G + blockIdx.x) * k;
                for (int x = lane; x < k; x += 32) crow[x] = (double)(r + x);
            }
            if (lane < R) {
                seed = seed * 6364136223846793005ull + 1442695040888963407ull;
                Cand c; c.absbits = (seed >> 12) + r; c.pos = blockIdx.x; c.entity = blockIdx.x;
                cand[((size_t)lane * 2 + slot) * G + blockIdx.x] = c;
            }
            __syncwarp();
            if (lane == 0) {
                target += G;
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
                unsigned v;
                do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory"); }
                while ((int)(v - target) < 0);
            }
            __syncwarp();
            unsigned long long ga = 0; unsigned gp = 0xffffffffu; int gc = 0;
            for (int c = lane; c < G; c += 32) {
                const Cand *cp = cand + ((size_t)my * 2 + slot) * G + c;
                unsigned long long a = __ldcg(&cp->absbits); unsigned pp = __ldcg(&cp->pos);
                if (a > ga || (a == ga && pp < gp)) { ga = a; gp = pp; gc = c; }
            }
            for (int off = 16; off; off >>= 1) {
                unsigned long long oa = __shfl_xor_sync(0xffffffffu, ga, off);
                unsigned op = __shfl_xor_sync(0xffffffffu, gp, off);
                int oc = __shfl_xor_sync(0xffffffffu, gc, off);
                if (oa > ga || (oa == ga && op < gp)) { ga = oa; gp = op; gc = oc; }
            }
            const double *wrow = rows + (((size_t)my * 2 + slot) * G + gc) * k;
            for (int x = lane; x < k; x += 32) u[slot][x] = __ldcg(wrow + x);
        }
        __syncthreads();
        if (threadIdx.x == 0) u[slot][0] += 1.0;
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) sink[blockIdx.x] = u[0][0];
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
}

template <int R>
void run12(int G, int rounds, int k) {
    unsigned *counter; Cand *cand; double *rows, *sink; unsigned long long *out;
    cudaMalloc(&counter, 4); cudaMalloc(&cand, sizeof(Cand) * 2 * G * R);
    cudaMalloc(&rows, 8 * 2 * (size_t)G * k * R); cudaMalloc(&out, 8); cudaMalloc(&sink, 8 * G);
    cudaMemset(counter, 0, 4);
    void *args[] = {&counter, &cand, &rows, &rounds, &k, &out, &sink};
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void *)xchg12_kernel<R>, G, 256, args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long cyc; cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
    printf("variant 12 R=%d G=%d k=%d: %.3f us/round (%.0f cyc) %s\n", R, G, k, ms * 1e3 / rounds,
           (double)cyc / rounds, cudaGetErrorString(cudaGetLastError()));
    cudaFree(counter); cudaFree(cand); cudaFree(rows); cudaFree(out); cudaFree(sink);
}

template <int V>
__global__ void xchg_kernel(unsigned *counter, Cand *cand, double *rows, int rounds, int k,
                            unsigned long long *out, double *sink) {
    const int G = gridDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned target = 0;
    __shared__ double u[2][640];
    long long t0 = clock64();
    unsigned long long seed = blockIdx.x * 2654435761ull;
    for (int r = 0; r < rounds; ++r) {
        const int slot = r & 1;
        if (warp == 0) {
            double *crow = rows + ((size_t)slot * G + blockIdx.x) * k;
            if (V != 4 && V < 8) for (int x = lane; x < k; x += 32) crow[x] = (double)(r + x);
            if (lane == 0 && V != 8) {
                seed = seed * 6364136223846793005ull + 1442695040888963407ull;
                Cand c; c.absbits = seed >> 12; c.pos = blockIdx.x; c.entity = blockIdx.x;
                cand[slot * G + blockIdx.x] = c;
            }
            __syncwarp();
            if (lane == 0) {
                target += G;
                if (V == 0 || V == 1) {
                    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
                } else {
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
                }
                unsigned v;
                if (V == 0) {
                    do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory"); }
                    while ((int)(v - target) < 0);
                } else {
                    do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory"); }
                    while ((int)(v - target) < 0);
                }
            }
            __syncwarp();
            unsigned long long ga = 0; unsigned gp = 0xffffffffu; int gc = 0;
            for (int c = lane; c < G && V != 8 && V != 9; c += 32) {
                const Cand *cp = cand + slot * G + c;
                unsigned long long a; unsigned pp;
                if (V == 3) {
                    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(a) : "l"(&cp->absbits));
                    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(pp) : "l"(&cp->pos));
                } else if (V == 7) {
                    a = __ldcg(&cp->absbits); pp = c;
                } else {
                    a = __ldcg(&cp->absbits); pp = __ldcg(&cp->pos);
                }
                if (V == 5) { a = 0; pp = 0; }
                if (a > ga || (a == ga && pp < gp)) { ga = a; gp = pp; gc = c; }
            }
            for (int off = 16; off; off >>= 1) {
                unsigned long long oa = __shfl_xor_sync(0xffffffffu, ga, off);
                unsigned op = __shfl_xor_sync(0xffffffffu, gp, off);
                int oc = __shfl_xor_sync(0xffffffffu, gc, off);
                if (oa > ga || (oa == ga && op < gp)) { ga = oa; gp = op; gc = oc; }
            }
            const double *wrow = rows + ((size_t)slot * G + gc) * k;
            if (V != 6 && V < 8) for (int x = lane; x < k; x += 32) u[slot][x] = __ldcg(wrow + x);
        }
        __syncthreads();
        if (threadIdx.x == 0) sink[blockIdx.x] += u[slot][3];
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
}

// V11: no counter; each CTA publishes {hi: absbits | parity<<63, lo: seq<<32 | pos}
// after a release fence; readers poll the G records until all carry seq.
__global__ void xchg11_kernel(unsigned long long *keys, double *rows, int rounds, int k,
                              unsigned long long *out, double *sink) {
    const int G = gridDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ double u[2][640];
    long long t0 = clock64();
    unsigned long long seed = blockIdx.x * 2654435761ull + 1;
    for (int r = 0; r < rounds; ++r) {
        const int slot = r & 1;
        const unsigned long long par = (unsigned long long)((r >> 1) & 1) << 63;
        if (warp == 0) {
            double *crow = rows + ((size_t)slot * G + blockIdx.x) * (k + 1);
            for (int x = lane; x < k; x += 32) crow[x] = (double)(r + x);
            __syncwarp();
            if (lane == 0) {
                seed = seed * 6364136223846793005ull + 1442695040888963407ull;
                unsigned long long hi = (seed >> 12) | par;
                unsigned long long lo = ((unsigned long long)(unsigned)r << 32) | blockIdx.x;
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(keys + 2 * (slot * G + blockIdx.x)), "l"(hi), "l"(lo) : "memory");
            }
            unsigned long long ga = 0; unsigned gp = 0xffffffffu; int gc = 0;
            for (int c0 = 0; c0 < G; c0 += 32) {
                const int c = c0 + lane;
                unsigned long long hi = 0, lo = 0;
                if (c < G) {
                    bool ok;
                    do {
                        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(hi), "=l"(lo) : "l"(keys + 2 * (slot * G + c)) : "memory");
                        ok = (unsigned)(lo >> 32) == (unsigned)r && (hi & (1ull << 63)) == par;
                    } while (!ok);
                    unsigned long long a = hi & ~(1ull << 63); unsigned pp = (unsigned)lo;
                    if (a > ga || (a == ga && pp < gp)) { ga = a; gp = pp; gc = c; }
                }
            }
            for (int off = 16; off; off >>= 1) {
                unsigned long long oa = __shfl_xor_sync(0xffffffffu, ga, off);
                unsigned op = __shfl_xor_sync(0xffffffffu, gp, off);
                int oc = __shfl_xor_sync(0xffffffffu, gc, off);
                if (oa > ga || (oa == ga && op < gp)) { ga = oa; gp = op; gc = oc; }
            }
            const double *wrow = rows + ((size_t)slot * G + gc) * (k + 1);
            for (int x = lane; x < k; x += 32) u[slot][x] = __ldcg(wrow + x);
        }
        __syncthreads();
        if (threadIdx.x == 0) u[slot][0] += 1.0;
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) sink[blockIdx.x] = u[0][0];
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
}

void run11(int G, int rounds, int k) {
    unsigned long long *keys, *out; double *rows, *sink;
    cudaMalloc(&keys, 16 * 2 * G); cudaMemset(keys, 0xff, 16 * 2 * G);
    cudaMalloc(&rows, 8 * 2 * (size_t)G * (k + 1)); cudaMalloc(&out, 8); cudaMalloc(&sink, 8 * G);
    void *args[] = {&keys, &rows, &rounds, &k, &out, &sink};
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void *)xchg11_kernel, G, 256, args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long cyc; cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
    printf("variant 11 G=%d k=%d: %.3f us/round (%.0f cyc) %s\n", G, k, ms * 1e3 / rounds,
           (double)cyc / rounds, cudaGetErrorString(cudaGetLastError()));
    cudaFree(keys); cudaFree(rows); cudaFree(out); cudaFree(sink);
}

template <int V>
void run(int G, int rounds, int k) {
    unsigned *counter; Cand *cand; double *rows, *sink; unsigned long long *out;
    cudaMalloc(&counter, 4); cudaMalloc(&cand, sizeof(Cand) * 2 * G);
    cudaMalloc(&rows, 8 * 2 * (size_t)G * k); cudaMalloc(&out, 8); cudaMalloc(&sink, 8 * G);
    cudaMemset(counter, 0, 4);
    void *args[] = {&counter, &cand, &rows, &rounds, &k, &out, &sink};
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void *)xchg_kernel<V>, G, 256, args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long cyc; cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
    printf("variant %d G=%d k=%d: %.3f us/round (%.0f cyc) %s\n", V, G, k, ms * 1e3 / rounds,
           (double)cyc / rounds, cudaGetErrorString(cudaGetLastError()));
    cudaFree(counter); cudaFree(cand); cudaFree(rows); cudaFree(out); cudaFree(sink);
}

int main() {
    run<1>(148, 2000, 110); run12<1>(148, 2000, 110); run12<4>(148, 2000, 110); run12<8>(148, 2000, 110);
    run12<16>(148, 2000, 110); run12<8>(148, 2000, 550);
    return 0;
}
