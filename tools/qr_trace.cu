// Per-reflector clock64 trace of qr_kernel (critical chain timing).
// Build: nvcc -cudart shared -DSRLU_QR_TRACE -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false \
//   -std=c++17 -I paper_1601_04280_b200/csrc tools/qr_trace.cu paper_1601_04280_b200/csrc/abi.cu -o tools/bin/qr_trace
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "small_dense.cu"

int main() {
    const int k1 = 110, k2 = 118;
    std::vector<double> h((size_t)k1 * k2);
    srand(1);
    for (auto &v : h) v = (double)rand() / RAND_MAX - 0.5;
    double *mT, *pinvT, *stats;
    void *ws;
    cudaMalloc(&mT, h.size() * 8);
    cudaMalloc(&pinvT, (size_t)k2 * k1 * 8);
    cudaMalloc(&stats, 64);
    size_t wsb = srlu_qr_pinv_workspace(k1, k2);
    cudaMalloc(&ws, wsb);
    cudaMemcpy(mT, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int it = 0; it < 3; ++it) srlu_qr_pinv(mT, k1, k2, k2, pinvT, k1, stats, ws, wsb, 0);
    cudaEventRecord(e0);
    srlu_qr_pinv(mT, k1, k2, k2, pinvT, k1, stats, ws, wsb, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long t[256][6];
    cudaMemcpyFromSymbol(t, g_qr_trace, sizeof(t));
    printf("qr_pinv %.1f us  err=%s\n", ms * 1e3, cudaGetErrorString(cudaGetLastError()));
    long long sum[5] = {0};
    for (int c = 2; c < k1; ++c) {
        long long d[5] = {t[c][0] - t[c - 1][4], t[c][1] - t[c][0], t[c][2] - t[c][1],
                          t[c][3] - t[c][2], t[c][4] - t[c][3]};
        for (int i = 0; i < 5; ++i) sum[i] += d[i];
        if (c < 8 || c % 20 == 0)
            printf("c=%3d wait %5lld dot %5lld axpy %5lld norm %5lld dlarfg %5lld\n", c, d[0], d[1],
                   d[2], d[3], d[4]);
    }
    printf("avg   wait %5lld dot %5lld axpy %5lld norm %5lld dlarfg %5lld  (cycles)\n",
           sum[0] / (k1 - 2), sum[1] / (k1 - 2), sum[2] / (k1 - 2), sum[3] / (k1 - 2),
           sum[4] / (k1 - 2));
    return 0;
}
