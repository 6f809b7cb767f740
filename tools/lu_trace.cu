// Phase timing of the LU kernels (rank 0, thread 0 clock64 sums).
// Usage: tools/lu_trace m k [col]
// Build: nvcc -cudart shared -DSRLU_LU_TRACE -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false \
//   -std=c++17 tools/lu_trace.cu paper_1601_04280_b200/csrc/abi.cu -o tools/bin/lu_trace
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1601_04280_b200/csrc/lu.cu"

int main(int argc, char **argv) {
    const int64_t m = argc > 1 ? atol(argv[1]) : 16384, k = argc > 2 ? atol(argv[2]) : 110;
    std::vector<double> h((size_t)m * k);
    srand(1);
    for (auto &v : h) v = (double)rand() / RAND_MAX - 0.5;
    double *y, *y0, *L, *U;
    int64_t *perm;
    void *ws;
    cudaMalloc(&y, h.size() * 8);
    cudaMalloc(&y0, h.size() * 8);
    cudaMalloc(&L, h.size() * 8);
    cudaMalloc(&U, (size_t)k * k * 8);
    cudaMalloc(&perm, m * 8);
    size_t wsb = srlu_lu_workspace(m, k);
    cudaMalloc(&ws, wsb);
    cudaMemcpy(y0, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    long long zero[8] = {0};
    for (int it = 0; it < 4; ++it) {
        cudaMemcpy(y, y0, h.size() * 8, cudaMemcpyDeviceToDevice);
        cudaMemcpyToSymbol(g_lu_trace, zero, sizeof(zero));
        cudaEventRecord(e0);
        const bool col = argc > 3 && argv[3][0] == 'c';  // col mode: m entities = columns
        int rc = col ? srlu_lu_colpiv(y, m, k, k, perm, U, k, L, k, 0, ws, wsb, 0)
                     : srlu_lu_rowpiv(y, m, k, k, perm, L, k, U, k, 0, ws, wsb, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        long long t[8];
        cudaMemcpyFromSymbol(t, g_lu_trace, sizeof(t));
        printf("rc=%d %.1f us | t0 %lld t1 %lld t2 %lld t3 %lld t4 %lld t5 %lld t6 %lld t7 %lld"
               " (cycles, rank 0)  %s\n", rc, ms * 1e3, t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7],
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
