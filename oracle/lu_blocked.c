/* ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into the product path.
 *
 * Blocked, multithreaded restatement of the reference's pivoted LUs for the
 * full-size parity checks (configs 3-5, where the numpy loops of
 * oracle/randlu.py take minutes):
 *
 *   mode 0: lu_row_pivot (/root/reference/pkg/src/sparselu/factor.py:49-77)
 *           on w = Y (M x k, row-major: one row per entity);
 *   mode 1: lu_col_pivot (factor.py:80-109) on W = core^T (M = n x k,
 *           row-major: row r of W is column r of core).
 *
 * Bit-exactness argument: the reference updates every trailing element
 * w[r][c] once per step j < min(r, c) as w - (l * u) (numpy outer, then
 * subtract: one rounded product, one rounded difference; -ffp-contract=off
 * keeps them separate here), in ascending j.  The blocked order applies the
 * panel's steps to the panel columns immediately (the pivot search needs
 * them) and defers the trailing columns to one pass per panel that applies
 * the same products in the same ascending j per element; the division of
 * the multipliers happens on the same values.  So every element sees the
 * identical operation sequence.  Pivot search: first index of the maximum
 * |value| (numpy argmax); rows are partitioned in ascending contiguous
 * chunks and candidates combined in chunk order with a strict '>'.
 *
 * Checked bit for bit against oracle/randlu.py's numpy restatement (itself
 * pinned to the reference's golden vectors) in tests/test_oracle.py.
 */
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#else  /* serial fallback (a compiler without libgomp) */
static int omp_get_max_threads(void) { return 1; }
static int omp_get_thread_num(void) { return 0; }
static int omp_get_num_threads(void) { return 1; }
#endif
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MAXT 1024

void oracle_lu_blocked(double *w, int64_t M, int64_t k, int mode, double thresh,
                       int64_t *perm, int nthreads, int64_t panel) {
    if (panel <= 0) panel = 32;
    int nt = nthreads > 0 ? nthreads : omp_get_max_threads();
    if (nt > MAXT) nt = MAXT;
    for (int64_t i = 0; i < M; ++i) perm[i] = i;
    double cand_v[MAXT];
    int64_t cand_i[MAXT];
    unsigned char *flag = (unsigned char *)calloc((size_t)k + 1, 1);
    double *piv = (double *)calloc((size_t)k + 1, sizeof(double));
    double *tmp = (double *)malloc(sizeof(double) * (size_t)(k + 1));

#pragma omp parallel num_threads(nt)
    {
        const int t = omp_get_thread_num(), T = omp_get_num_threads();
        const int64_t rb = M * t / T, re = M * (t + 1) / T;
        for (int64_t p0 = 0; p0 < k; p0 += panel) {
            const int64_t p1 = p0 + panel < k ? p0 + panel : k;
            for (int64_t i = p0; i < p1; ++i) {
                double best = -1.0;
                int64_t bi = -1;
                for (int64_t r = rb > i ? rb : i; r < re; ++r) {
                    const double v = fabs(w[r * k + i]);
                    if (v > best) {
                        best = v;
                        bi = r;
                    }
                }
                cand_v[t] = best;
                cand_i[t] = bi;
#pragma omp barrier
#pragma omp single
                {
                    double bv = -1.0;
                    int64_t p = i;
                    for (int u = 0; u < T; ++u)
                        if (cand_i[u] >= 0 && cand_v[u] > bv) {
                            bv = cand_v[u];
                            p = cand_i[u];
                        }
                    if (p != i) {
                        memcpy(tmp, w + i * k, sizeof(double) * (size_t)k);
                        memcpy(w + i * k, w + p * k, sizeof(double) * (size_t)k);
                        memcpy(w + p * k, tmp, sizeof(double) * (size_t)k);
                        const int64_t q = perm[i];
                        perm[i] = perm[p];
                        perm[p] = q;
                    }
                    const double pv = w[i * k + i];
                    piv[i] = pv;
                    flag[i] = fabs(pv) > thresh;
                    if (mode == 1) {  /* w[i+1:, i] /= piv (or = 0): row i of W, panel part */
                        double *wi = w + i * k;
                        for (int64_t c = i + 1; c < p1; ++c) wi[c] = flag[i] ? wi[c] / pv : 0.0;
                    }
                }  /* implicit barrier */
                const double pv = piv[i];
                const double *wi = w + i * k;
                for (int64_t r = rb > i + 1 ? rb : i + 1; r < re; ++r) {
                    double *wr = w + r * k;
                    if (mode == 0) {
                        if (flag[i]) {
                            const double l = wr[i] / pv;
                            wr[i] = l;
                            for (int64_t c = i + 1; c < p1; ++c) wr[c] = wr[c] - l * wi[c];
                        } else {
                            wr[i] = 0.0;
                        }
                    } else if (flag[i]) {
                        const double f = wr[i];
                        for (int64_t c = i + 1; c < p1; ++c) wr[c] = wr[c] - wi[c] * f;
                    }
                }
            }
            if (p1 < k) {
#pragma omp barrier
#pragma omp single
                {
                    /* pivot rows of the panel, in order: steps j < i of the panel */
                    for (int64_t i = p0; i < p1; ++i) {
                        double *wi = w + i * k;
                        for (int64_t j = p0; j < i; ++j) {
                            if (!flag[j]) continue;
                            const double *wj = w + j * k;
                            const double f = wi[j];
                            if (mode == 0)
                                for (int64_t c = p1; c < k; ++c) wi[c] = wi[c] - f * wj[c];
                            else
                                for (int64_t c = p1; c < k; ++c) wi[c] = wi[c] - wj[c] * f;
                        }
                        if (mode == 1)
                            for (int64_t c = p1; c < k; ++c)
                                wi[c] = flag[i] ? wi[c] / piv[i] : 0.0;
                    }
                }  /* implicit barrier */
                for (int64_t r = rb > p1 ? rb : p1; r < re; ++r) {
                    double *wr = w + r * k;
                    for (int64_t j = p0; j < p1; ++j) {
                        if (!flag[j]) continue;
                        const double *wj = w + j * k;
                        const double f = wr[j];
                        if (mode == 0)
                            for (int64_t c = p1; c < k; ++c) wr[c] = wr[c] - f * wj[c];
                        else
                            for (int64_t c = p1; c < k; ++c) wr[c] = wr[c] - wj[c] * f;
                    }
                }
#pragma omp barrier
            }
        }
    }
    free(flag);
    free(piv);
    free(tmp);
}

/* ---- row-chunked stage-1 sketch: Y rows = apply_sketch_right of A rows ----
 * sketch.py:362-368 = sem_gather (_fast.pyx:44-54: per output (i, t) the
 * sum runs over source columns j ascending, dst = dst + s*a) then
 * _fast_adjoint_right (sketch.py:322-335: * phase, zero pad, fwht_rows
 * stages h = 1, 2, 4, ... (_fast.pyx:23-41), x[:, sample] * mult).  Each row
 * of Y depends only on the same row of A, so row blocks are independent. */
static void fwht_one(double *x, int64_t n) {
    for (int64_t h = 1; h < n; h *= 2)
        for (int64_t s = 0; s < n; s += 2 * h)
            for (int64_t j = s; j < s + h; ++j) {
                const double a = x[j], b = x[j + h];
                x[j] = a + b;
                x[j + h] = a - b;
            }
}

static void finish_row(double *x, const double *phase, int64_t l, int64_t pad,
                       const int64_t *sample, int64_t k, double mult, double *out,
                       int64_t stride) {
    for (int64_t t = 0; t < l; ++t) x[t] = x[t] * phase[t];
    fwht_one(x, pad);
    for (int64_t c = 0; c < k; ++c) out[c * stride] = x[sample[c]] * mult;
}

void oracle_sketch_right_dense_rows(const void *a, int dtype, int64_t rows, int64_t n,
                                    int64_t lda, const int64_t *row_of, const double *sign,
                                    const double *phase, int64_t l, int64_t pad,
                                    const int64_t *sample, int64_t k, double mult, double *y,
                                    int64_t ldy, int nthreads) {
    int nt = nthreads > 0 ? nthreads : omp_get_max_threads();
#pragma omp parallel num_threads(nt)
    {
        double *x = (double *)malloc(sizeof(double) * (size_t)pad);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < rows; ++i) {
            memset(x, 0, sizeof(double) * (size_t)pad);
            if (dtype == 0) {
                const float *ar = (const float *)a + i * lda;
                for (int64_t j = 0; j < n; ++j)
                    x[row_of[j]] = x[row_of[j]] + sign[j] * (double)ar[j];
            } else {
                const double *ar = (const double *)a + i * lda;
                for (int64_t j = 0; j < n; ++j) x[row_of[j]] = x[row_of[j]] + sign[j] * ar[j];
            }
            finish_row(x, phase, l, pad, sample, k, mult, y + i * ldy, 1);
        }
        free(x);
    }
}

/* CSR rows (indices ascending within a row = sem_gather_csc's j order) */
void oracle_sketch_right_csr_rows(const int64_t *indptr, const int32_t *indices,
                                  const void *vals, int dtype, int64_t rows,
                                  const int64_t *row_of, const double *sign, const double *phase,
                                  int64_t l, int64_t pad, const int64_t *sample, int64_t k,
                                  double mult, double *y, int64_t ldy, int nthreads) {
    int nt = nthreads > 0 ? nthreads : omp_get_max_threads();
#pragma omp parallel num_threads(nt)
    {
        double *x = (double *)malloc(sizeof(double) * (size_t)pad);
#pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < rows; ++i) {
            memset(x, 0, sizeof(double) * (size_t)pad);
            for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
                const int64_t j = indices[p];
                const double v = dtype == 0 ? (double)((const float *)vals)[p]
                                            : ((const double *)vals)[p];
                x[row_of[j]] = x[row_of[j]] + sign[j] * v;
            }
            finish_row(x, phase, l, pad, sample, k, mult, y + i * ldy, 1);
        }
        free(x);
    }
}

/* ---- column-blocked stage-2 sketch of P·A: out (nb x k2 row-major) ----
 * apply_sketch_left (sketch.py:371-378) of the columns of P·A held in a
 * row-major host block a (m x nb, lda): _sem_mul_left = sem_scatter_dense
 * (_fast.pyx:71-78: per (t, column) the sum runs over PA rows i ascending,
 * dst = dst + s*a), then _fast_mul_left (sketch.py:338-349) per column.
 * perm: row i of P·A = row perm[i] of A.  Columns are independent; each
 * thread takes blocks of CB columns and sweeps the rows once. */
#define CB 32
void oracle_sketch_left_dense_cols(const void *a, int dtype, int64_t m, int64_t nb, int64_t lda,
                                   const int64_t *perm, const int64_t *row_of,
                                   const double *sign, const double *phase, int64_t l,
                                   int64_t pad, const int64_t *sample, int64_t k, double mult,
                                   double *out, int64_t ldo, int nthreads) {
    int nt = nthreads > 0 ? nthreads : omp_get_max_threads();
#pragma omp parallel num_threads(nt)
    {
        double *acc = (double *)malloc(sizeof(double) * (size_t)pad * CB);
        double *x = (double *)malloc(sizeof(double) * (size_t)pad);
#pragma omp for schedule(dynamic, 1)
        for (int64_t c0 = 0; c0 < nb; c0 += CB) {
            const int64_t cw = nb - c0 < CB ? nb - c0 : CB;
            memset(acc, 0, sizeof(double) * (size_t)pad * CB);
            for (int64_t i = 0; i < m; ++i) {
                double *dst = acc + row_of[i] * CB;
                const double s = sign[i];
                if (dtype == 0) {
                    const float *ar = (const float *)a + perm[i] * lda + c0;
                    for (int64_t c = 0; c < cw; ++c) dst[c] = dst[c] + s * (double)ar[c];
                } else {
                    const double *ar = (const double *)a + perm[i] * lda + c0;
                    for (int64_t c = 0; c < cw; ++c) dst[c] = dst[c] + s * ar[c];
                }
            }
            for (int64_t c = 0; c < cw; ++c) {
                memset(x, 0, sizeof(double) * (size_t)pad);
                for (int64_t t = 0; t < l; ++t) x[t] = acc[t * CB + c];
                finish_row(x, phase, l, pad, sample, k, mult, out + (c0 + c) * ldo, 1);
            }
        }
        free(acc);
        free(x);
    }
}
