// Exhaustive-style check: q = fma(fma(-b, RN(a*y), a), y, RN(a*y)) with
// y = __drcp_rn(b) equals a / b bit for bit, over random and adversarial
// (a, b) in the range the LU uses (|a| <= |b|, finite, normal).
// nvcc -cudart shared -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false tools/check_div.cu -o tools/bin/check_div
#include <cstdio>
#include <cstdint>

__device__ unsigned long long g_bad, g_tested;
__device__ double g_ex[4];

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
    return x;
}

__device__ __forceinline__ double div_recip(double a, double b, double y) {
    const double fb = fabs(b), fa = fabs(a);
    if (!(fb >= 0x1p-1000 && fb <= 0x1p+1000 && fa >= 0x1p-960 && fa <= 0x1p+1000)) return a / b;
    const double q0 = __dmul_rn(a, y);
    const double fq = fabs(q0);
    if (!(fq >= 0x1p-960 && fq <= 0x1p+1000)) return a / b;
    const double r = __fma_rn(-b, q0, a);
    return __fma_rn(r, y, q0);
}

__global__ void kern(uint64_t seed, int per_thread, int mode) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    unsigned long long bad = 0;
    for (int i = 0; i < per_thread; ++i) {
        uint64_t h1 = mix(seed ^ (tid * 0x9E3779B97F4A7C15ULL + i));
        uint64_t h2 = mix(h1 + 0x632BE59BD9B4E019ULL);
        double a, b;
        if (mode == 0) {  // random mantissas, exponents spread over +-60
            b = __longlong_as_double((int64_t)((h1 & 0x000FFFFFFFFFFFFFULL) | ((uint64_t)(1023 + (int)((h1 >> 52) % 121) - 60) << 52)));
            a = __longlong_as_double((int64_t)((h2 & 0x000FFFFFFFFFFFFFULL) | ((uint64_t)(1023 + (int)((h2 >> 52) % 121) - 60) << 52)));
        } else if (mode == 1) {  // mantissas near 1 / near 2 (hard rounding cases)
            uint64_t mb = (h1 & 1) ? (h1 >> 20) & 0xFFF : 0x000FFFFFFFFFFFFFULL - ((h1 >> 20) & 0xFFF);
            uint64_t ma = (h2 & 1) ? (h2 >> 20) & 0xFFFFF : 0x000FFFFFFFFFFFFFULL - ((h2 >> 20) & 0xFFFFF);
            b = __longlong_as_double((int64_t)(mb | (1023ULL << 52)));
            a = __longlong_as_double((int64_t)(ma | ((uint64_t)(1023 - (h2 >> 60)) << 52)));
        } else if (mode == 3) {  // zeros, denormals, extremes, inf/nan mixed in
            const uint64_t sel = h1 % 8;
            b = __longlong_as_double((int64_t)((h1 >> 3) & 0x7FFFFFFFFFFFFFFFULL));
            a = __longlong_as_double((int64_t)((h2 >> 1) & 0x7FFFFFFFFFFFFFFFULL));
            if (sel == 0) a = 0.0;
            if (sel == 1) a = -0.0;
            if (sel == 2) a = __longlong_as_double((int64_t)(h2 & 0x000FFFFFFFFFFFFFULL));  // denormal
            if (sel == 3) b = __longlong_as_double((int64_t)((h1 & 0x000FFFFFFFFFFFFFULL) | (1ULL << 52)));
            if (b == 0.0) b = 3.0;
        } else {  // small integers and their ratios
            b = (double)((int64_t)(h1 % 2001) - 1000);
            a = (double)((int64_t)(h2 % 2001) - 1000);
            if (b == 0.0) b = 7.0;
        }
        if (h2 & 2) a = -a;
        const double y = __drcp_rn(b);
        const double q = div_recip(a, b, y);
        const double t = a / b;
        if (__double_as_longlong(q) != __double_as_longlong(t) && !(q != q && t != t)) {
            if (bad == 0) { g_ex[0] = a; g_ex[1] = b; g_ex[2] = q; g_ex[3] = t; }
            ++bad;
        }
    }
    atomicAdd(&g_bad, bad);
    atomicAdd(&g_tested, (unsigned long long)per_thread);
}

int main() {
    for (int mode = 0; mode < 4; ++mode) {
        unsigned long long z = 0;
        cudaMemcpyToSymbol(g_bad, &z, 8);
        cudaMemcpyToSymbol(g_tested, &z, 8);
        for (int rep = 0; rep < 4; ++rep) kern<<<148 * 8, 256>>>(1234567ULL + rep * 77 + mode * 1000003ULL, 2048, mode);
        cudaDeviceSynchronize();
        unsigned long long bad, tested;
        double ex[4];
        cudaMemcpyFromSymbol(&bad, g_bad, 8);
        cudaMemcpyFromSymbol(&tested, g_tested, 8);
        cudaMemcpyFromSymbol(ex, g_ex, sizeof(ex));
        printf("mode %d: tested %llu  mismatches %llu  %s", mode, tested, bad, cudaGetErrorString(cudaGetLastError()));
        if (bad) printf("  e.g. a=%.17g b=%.17g recip=%.17g div=%.17g", ex[0], ex[1], ex[2], ex[3]);
        printf("\n");
    }
    return 0;
}
