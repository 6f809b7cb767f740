// FP64 vector-pipe throughput on this GPU: DADD, DMUL and DFMA chains with 8
// independent accumulators per thread, all SMs.  Prints G ops/s and
// warp-instructions per clock per SM (at the measured SM clock).
// Build: nvcc -cudart shared -gencode arch=compute_100a,code=sm_100a -O3 tools/bench_fp64.cu -o tools/bin/bench_fp64
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(double *out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) x[i] = __dadd_rn(x[i], a);
            if (OP == 1) x[i] = __dmul_rn(x[i], b);
            if (OP == 2) x[i] = __fma_rn(x[i], b, a);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double *out;
    cudaMalloc(&out, 8);
    const int iters = 4096, threads = 512, blocks = sms * 4;
    const char *names[3] = {"DADD", "DMUL", "DFMA"};
    for (int op = 0; op < 3; ++op) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (op == 0) k<0><<<blocks, threads>>>(out, iters, 1e-9, 1.0000001);
            if (op == 1) k<1><<<blocks, threads>>>(out, iters, 1e-9, 1.0000001);
            if (op == 2) k<2><<<blocks, threads>>>(out, iters, 1e-9, 1.0000001);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = (double)blocks * threads * iters * 8;
        const double per_clk_sm = ops / 32.0 / (ms * 1e-3) / (clk * 1e3) / sms;
        printf("%s: %.1f G ops/s (%.2f warp-instr/clk/SM at the %d MHz base attribute clock)\n",
               names[op], ops / (ms * 1e-3) / 1e9, per_clk_sm, clk / 1000);
    }
    return 0;
}
