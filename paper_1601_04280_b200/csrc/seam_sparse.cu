// Sparse variants of the reference's kernel seam (_kernels/__init__.py:9-31),
// O(nnz) and bit-identical to the compiled reference lane:
//   srlu_sem_gather_csr  <- _fast.pyx:57-68 sem_gather_csc
//       out[i, row_of[j]] += sign[j] * a[i, j]   (every (i, t) cell in ascending j)
//   srlu_sem_scatter_csc <- _fast.pyx:81-90 sem_scatter_csc
//       out[row_of[i], j] += sign[i] * a[i, j]   (every (t, j) cell in ascending i)
// One thread walks one row (gather, entries ascending in j) or one column
// (scatter, entries ascending in i): the reference's sequential sums.  These
// are seam utilities; the pipeline's hot paths are K1-CSR and K3-CSR.
#include "common.cuh"

namespace srlu {

template <typename T>
__global__ void sem_gather_csr_kernel(const int64_t *__restrict__ indptr,
                                      const int32_t *__restrict__ indices,
                                      const T *__restrict__ vals, int64_t rows,
                                      const int32_t *__restrict__ row_of,
                                      const double *__restrict__ sign, double *__restrict__ out,
                                      int64_t ldo) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    double *dst = out + i * ldo;
    for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
        const int j = indices[p];
        const int t = row_of[j];
        dst[t] = __dadd_rn(dst[t], __dmul_rn(sign[j], (double)vals[p]));
    }
}

template <typename T>
__global__ void sem_scatter_csc_kernel(const int64_t *__restrict__ indptr,
                                       const int32_t *__restrict__ indices,
                                       const T *__restrict__ vals, int64_t cols,
                                       const int32_t *__restrict__ row_of,
                                       const double *__restrict__ sign, double *__restrict__ out,
                                       int64_t ldo) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= cols) return;
    for (int64_t p = indptr[j]; p < indptr[j + 1]; ++p) {
        const int i = indices[p];
        double *dst = out + (int64_t)row_of[i] * ldo + j;
        *dst = __dadd_rn(*dst, __dmul_rn(sign[i], (double)vals[p]));
    }
}

}  // namespace srlu

using namespace srlu;

extern "C" int srlu_sem_gather_csr(const int64_t *indptr, const int32_t *indices, const void *vals,
                                   int dtype, int64_t rows, const int32_t *row_of,
                                   const double *sign, double *out, int64_t ldo,
                                   srlu_stream_t stream) {
    SRLU_REQUIRE(rows >= 0 && ldo >= 1, SRLU_ERR_ARG, "sem_gather_csr: bad sizes");
    if (rows == 0) return SRLU_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const unsigned grid = (unsigned)ceil_div(rows, 128);
    if (dtype == SRLU_F32)
        sem_gather_csr_kernel<float><<<grid, 128, 0, s>>>(indptr, indices, (const float *)vals,
                                                         rows, row_of, sign, out, ldo);
    else if (dtype == SRLU_F64)
        sem_gather_csr_kernel<double><<<grid, 128, 0, s>>>(indptr, indices, (const double *)vals,
                                                          rows, row_of, sign, out, ldo);
    else {
        set_error("sem_gather_csr: unknown dtype %d", dtype);
        return SRLU_ERR_ARG;
    }
    SRLU_CHECK_LAUNCH("sem_gather_csr_kernel");
    return SRLU_OK;
}

extern "C" int srlu_sem_scatter_csc(const int64_t *indptr, const int32_t *indices,
                                    const void *vals, int dtype, int64_t cols,
                                    const int32_t *row_of, const double *sign, double *out,
                                    int64_t ldo, srlu_stream_t stream) {
    SRLU_REQUIRE(cols >= 0 && ldo >= cols, SRLU_ERR_ARG, "sem_scatter_csc: bad sizes");
    if (cols == 0) return SRLU_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const unsigned grid = (unsigned)ceil_div(cols, 128);
    if (dtype == SRLU_F32)
        sem_scatter_csc_kernel<float><<<grid, 128, 0, s>>>(indptr, indices, (const float *)vals,
                                                          cols, row_of, sign, out, ldo);
    else if (dtype == SRLU_F64)
        sem_scatter_csc_kernel<double><<<grid, 128, 0, s>>>(indptr, indices, (const double *)vals,
                                                           cols, row_of, sign, out, ldo);
    else {
        set_error("sem_scatter_csc: unknown dtype %d", dtype);
        return SRLU_ERR_ARG;
    }
    SRLU_CHECK_LAUNCH("sem_scatter_csc_kernel");
    return SRLU_OK;
}
