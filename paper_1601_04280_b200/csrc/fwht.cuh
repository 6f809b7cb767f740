// Walsh-Hadamard butterflies with the reference's exact network:
// stages h = 1, 2, 4, ... ; butterfly (a+b, a-b) on (j, j+h)
// (_fast.pyx:23-41).  Any thread assignment gives bit-identical results
// because every output is produced by the same tree of fp64 add/sub.
#pragma once
#include "common.cuh"

namespace srlu {

// CTA-cooperative in-place FWHT of x[0..pad) in shared memory.
__device__ inline void fwht_smem_cta(double *x, int pad) {
    int half = pad >> 1;
    for (int h = 1; h < pad; h <<= 1) {
        for (int p = threadIdx.x; p < half; p += blockDim.x) {
            int j = ((p / h) * (h << 1)) + (p % h);
            double a = x[j], b = x[j + h];
            x[j] = __dadd_rn(a, b);
            x[j + h] = __dsub_rn(a, b);
        }
        __syncthreads();
    }
}

// Warp-cooperative in-place FWHT of x[0..pad) in shared memory.
__device__ inline void fwht_smem_warp(double *x, int pad, int lane) {
    int half = pad >> 1;
    for (int h = 1; h < pad; h <<= 1) {
        for (int p = lane; p < half; p += 32) {
            int j = ((p / h) * (h << 1)) + (p % h);
            double a = x[j], b = x[j + h];
            x[j] = __dadd_rn(a, b);
            x[j + h] = __dsub_rn(a, b);
        }
        __syncwarp();
    }
}

// CTA-cooperative FWHT down the columns of a (pad x ncol) smem tile with
// row stride `ld` (x[t*ld + c]); one independent transform per column.
__device__ inline void fwht_smem_cols(double *x, int pad, int ncol, int ld) {
    int half = pad >> 1;
    int work = half * ncol;
    for (int h = 1; h < pad; h <<= 1) {
        for (int w = threadIdx.x; w < work; w += blockDim.x) {
            int c = w % ncol, p = w / ncol;
            int j = ((p / h) * (h << 1)) + (p % h);
            double a = x[j * ld + c], b = x[(j + h) * ld + c];
            x[j * ld + c] = __dadd_rn(a, b);
            x[(j + h) * ld + c] = __dsub_rn(a, b);
        }
        __syncthreads();
    }
}

}  // namespace srlu
