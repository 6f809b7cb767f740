/* ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into the product path.
 *
 * Plain-C restatement of the reference's compiled hot kernels
 * (/root/reference/pkg/src/sparselu/_kernels/_fast.pyx), real float64
 * lane only, with the SAME loop nests and therefore the same floating
 * point accumulation order:
 *
 *   oracle_fwht_rows        <- _fast.pyx:23-41   (stages h = 1, 2, 4, ...)
 *   oracle_sem_gather_dense <- _fast.pyx:44-54   (j outer ascending, i inner)
 *   oracle_sem_gather_csc   <- _fast.pyx:57-68   (j outer, nnz of col j)
 *   oracle_sem_scatter_dense<- _fast.pyx:71-78   (j outer, i ascending)
 *   oracle_sem_scatter_csc  <- _fast.pyx:81-90
 *
 * Dense operands are column-major (Fortran) with leading dimension ld,
 * exactly like the reference's value_t[::1, :] memoryviews; x of
 * fwht_rows is C-contiguous.  Built by oracle/Makefile into
 * oracle/_build/liboracle.so and called through ctypes by oracle/randlu.py.
 */
#include <stdint.h>

void oracle_fwht_rows(double *x, int64_t m, int64_t n) {
    for (int64_t i = 0; i < m; ++i) {
        double *row = x + i * n;
        for (int64_t h = 1; h < n; h *= 2) {
            for (int64_t start = 0; start < n; start += 2 * h) {
                for (int64_t j = start; j < start + h; ++j) {
                    double a = row[j], b = row[j + h];
                    row[j] = a + b;
                    row[j + h] = a - b;
                }
            }
        }
    }
}

/* out[:, row_of[j]] += sign[j] * a[:, j] */
void oracle_sem_gather_dense(const double *a, int64_t m, int64_t n, int64_t lda,
                             const int64_t *row_of, const double *sign,
                             double *out, int64_t ldo) {
    for (int64_t j = 0; j < n; ++j) {
        int64_t t = row_of[j];
        double s = sign[j];
        const double *col = a + j * lda;
        double *dst = out + t * ldo;
        for (int64_t i = 0; i < m; ++i) dst[i] = dst[i] + s * col[i];
    }
}

void oracle_sem_gather_csc(const double *data, const int64_t *indices,
                           const int64_t *indptr, int64_t n,
                           const int64_t *row_of, const double *sign,
                           double *out, int64_t ldo) {
    for (int64_t j = 0; j < n; ++j) {
        int64_t t = row_of[j];
        double s = sign[j];
        for (int64_t p = indptr[j]; p < indptr[j + 1]; ++p) {
            double *d = out + indices[p] + t * ldo;
            *d = *d + s * data[p];
        }
    }
}

/* out[row_of[i], :] += sign[i] * a[i, :] */
void oracle_sem_scatter_dense(const double *a, int64_t m, int64_t n, int64_t lda,
                              const int64_t *row_of, const double *sign,
                              double *out, int64_t ldo) {
    for (int64_t j = 0; j < n; ++j) {
        const double *col = a + j * lda;
        double *dst = out + j * ldo;
        for (int64_t i = 0; i < m; ++i)
            dst[row_of[i]] = dst[row_of[i]] + sign[i] * col[i];
    }
}

void oracle_sem_scatter_csc(const double *data, const int64_t *indices,
                            const int64_t *indptr, int64_t n,
                            const int64_t *row_of, const double *sign,
                            double *out, int64_t ldo) {
    for (int64_t j = 0; j < n; ++j) {
        double *dst = out + j * ldo;
        for (int64_t p = indptr[j]; p < indptr[j + 1]; ++p) {
            int64_t i = indices[p];
            dst[row_of[i]] = dst[row_of[i]] + sign[i] * data[p];
        }
    }
}
