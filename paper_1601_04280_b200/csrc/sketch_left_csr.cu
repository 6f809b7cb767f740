// K3-CSR — stage-2 projection of a CSR matrix: Omega2 · (P A)
// (reference: matrix.py:201-207 permute_rows of the CSC array +
//  _fast.pyx:81-90 sem_scatter_csc + sketch.py:338-349 _fast_mul_left).
//
// The reference sums, for every (bucket t, column j), the signed entries
// of P·A in ascending PA-row index q.  CSR rows of A are scattered into
// per-column segments (counting sort by column; slot order inside a
// column is arbitrary), each entry carrying the key (t = h2(q), q).  One
// CTA per column then sorts its segment by key in shared memory (bitonic),
// folds each bucket's run in ascending q (bit-identical sums), applies
// +-phase, the radix-2 FWHT over pad2 and the k2-row subsample, and writes
// row j of (Omega2 P A)^T.  P·A is never formed.  Columns longer than one
// CTA's sort capacity are processed in bucket ranges (any length).
#include "fwht.cuh"
#include "fwht_warp.cuh"

namespace srlu {

constexpr int kCsrColCap = 8192;  // entries of one column sorted in smem

__global__ void csr_col_count_kernel(const int32_t *__restrict__ indices, int64_t nnz,
                                     int *__restrict__ cnt) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
         p += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + indices[p], 1);
}

// single CTA exclusive scan (int counts -> int64 pointers): per-thread
// chunk sums, a two-level warp-shuffle scan of the 1024 partials, then each
// thread writes its chunk (4-wide independent loads)
__global__ void __launch_bounds__(1024) csr_col_scan_kernel(const int *__restrict__ cnt, int64_t n,
                                                            int64_t *__restrict__ colptr,
                                                            int *__restrict__ maxcnt) {
    __shared__ int64_t wsum[32];
    __shared__ int wmax[32];
    const int nt = blockDim.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t per = (n + nt - 1) / nt;
    const int64_t lo = threadIdx.x * per, hi = min(n, lo + per);
    int64_t sum = 0;
    int mx = 0;
    for (int64_t j = lo; j < hi; ++j) {
        const int c = __ldg(cnt + j);
        sum += c;
        mx = max(mx, c);
    }
    int64_t incl = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
    }
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (lane == 31) wsum[warp] = incl;
    if (lane == 0) wmax[warp] = mx;
    __syncthreads();
    if (warp == 0) {
        const int nw = nt >> 5;
        int64_t v = lane < nw ? wsum[lane] : 0;
        int m2 = lane < nw ? wmax[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, v, d);
            if (lane >= d) v += y;
        }
        m2 = __reduce_max_sync(0xffffffffu, m2);
        wsum[lane] = v;  // inclusive warp totals
        if (lane == 31) {
            colptr[n] = v;
            *maxcnt = m2;
        }
    }
    __syncthreads();
    int64_t run = (warp > 0 ? wsum[warp - 1] : 0) + incl - sum;
    for (int64_t j = lo; j < hi; ++j) {
        colptr[j] = run;
        run += __ldg(cnt + j);
    }
}


// Three-launch exclusive scan of the column counts (int -> int64 pointers)
// for large n: tile sums and maxima (one CTA per 1024 counts), a single-CTA
// scan of the tile sums, then each tile's local scan.  (The one-CTA scan
// above takes 117 us at n = 65536.)
constexpr int kScanTile = 1024;

__device__ __forceinline__ int64_t block_excl_scan_256(int64_t v, int64_t *total, int64_t *wsum) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t incl = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int64_t base = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        const int64_t x = wsum[w];
        if (w < warp) base += x;
        tot += x;
    }
    __syncthreads();
    *total = tot;
    return base + incl - v;
}

__global__ void __launch_bounds__(256) csr_scan_tiles_kernel(const int *__restrict__ cnt,
                                                             int64_t n,
                                                             int64_t *__restrict__ tsum,
                                                             int *__restrict__ maxcnt) {
    __shared__ int64_t wsum[8];
    const int64_t j0 = (int64_t)blockIdx.x * kScanTile + threadIdx.x * 4;
    int64_t s = 0;
    int mx = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
        if (j0 + u < n) {
            const int c = cnt[j0 + u];
            s += c;
            mx = max(mx, c);
        }
    int64_t tot;
    block_excl_scan_256(s, &tot, wsum);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if ((threadIdx.x & 31) == 0 && mx > 0) atomicMax(maxcnt, mx);
    if (threadIdx.x == 0) tsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(256) csr_scan_tsum_kernel(int64_t *__restrict__ tsum, int ntiles,
                                                            int64_t *__restrict__ colptr_n) {
    __shared__ int64_t wsum[8];
    int64_t carry = 0;
    for (int t0 = 0; t0 < ntiles; t0 += 256) {
        const int t = t0 + threadIdx.x;
        const int64_t v = t < ntiles ? tsum[t] : 0;
        int64_t tot;
        const int64_t ex = block_excl_scan_256(v, &tot, wsum);
        if (t < ntiles) tsum[t] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) *colptr_n = carry;
}

__global__ void __launch_bounds__(256) csr_scan_apply_kernel(const int *__restrict__ cnt,
                                                             int64_t n,
                                                             const int64_t *__restrict__ tsum,
                                                             int64_t *__restrict__ colptr,
                                                             int *__restrict__ cursor) {
    __shared__ int64_t wsum[8];
    const int64_t j0 = (int64_t)blockIdx.x * kScanTile + threadIdx.x * 4;
    int c[4];
    int64_t s = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        c[u] = j0 + u < n ? cnt[j0 + u] : 0;
        s += c[u];
    }
    int64_t tot;
    int64_t run = tsum[blockIdx.x] + block_excl_scan_256(s, &tot, wsum);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        if (j0 + u < n) {
            colptr[j0 + u] = run;
            // absolute fill cursor (nnz < 2^32): the fill kernel needs no colptr gather
            if (cursor != nullptr) cursor[j0 + u] = (int)(unsigned)run;
        }
        run += c[u];
    }
}

// Entry codec.  16 bytes: {(t << 32) | q, double bits of +-v}.  8 bytes
// (fp32 values whose key (t, q) fits 32 bits — BASELINE config 4): one u64
// ((t << qb | q) << 32 | float bits of +-v); +-v is exact in fp32 and is
// widened at the fold, like the reference's upcast.  The mode is decided on
// the device from the largest position q (mode[0] = qb + 1, or 0 = 16 bytes).
__global__ void csr_mode_kernel(const int32_t *__restrict__ inv_perm, int64_t rows, int l,
                                int is_f32, int *mode) {
    int mx = 0;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
         r += (int64_t)gridDim.x * blockDim.x)
        mx = max(mx, inv_perm[r]);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if ((threadIdx.x & 31) == 0) atomicMax(mode + 1, mx);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(mode + 2, 1) == (int)gridDim.x - 1) {
        __threadfence();
        const int qmax = atomicAdd(mode + 1, 0);
        const int qb = qmax > 0 ? 32 - __clz(qmax) : 1;
        const int tb = l > 1 ? 32 - __clz(l - 1) : 1;
        mode[0] = (is_f32 && qb + tb <= 32) ? qb + 1 : 0;
    }
}

__device__ __forceinline__ void ent_read(const void *ent, int64_t i, int mode, unsigned &t,
                                         int &q, double &v) {
    if (mode) {
        const unsigned long long w = reinterpret_cast<const unsigned long long *>(ent)[i];
        const unsigned key = (unsigned)(w >> 32);
        const int qb = mode - 1;
        t = key >> qb;
        q = (int)(key & ((1u << qb) - 1u));
        v = (double)__uint_as_float((unsigned)w);
    } else {
        const ulonglong2 e = reinterpret_cast<const ulonglong2 *>(ent)[i];
        t = (unsigned)(e.x >> 32);
        q = (int)(unsigned)e.x;
        v = __longlong_as_double((long long)e.y);
    }
}

template <typename T>
__global__ void csr_fill_kernel(const int64_t *__restrict__ indptr,
                                const int32_t *__restrict__ indices, const T *__restrict__ vals,
                                int64_t rows, const int32_t *__restrict__ inv_perm,
                                const int32_t *__restrict__ row_of2,
                                const double *__restrict__ sign2,
                                const int64_t *__restrict__ colptr, int *__restrict__ fill,
                                int abs_cursor,
                                void *__restrict__ ent, const int *__restrict__ modep) {
    const int lane = threadIdx.x & 31;
    const int mode = sizeof(T) == 4 ? *modep : 0;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
    constexpr int U = 4;  // 32-entry chunks of one row in flight together
    // 32 rows per warp pass: lane i fetches row rb+i's metadata, then the
    // warp walks the rows in turn, U chunks of each row's loads in flight
    for (int64_t rb = warp * 32; rb < rows; rb += nwarp * 32) {
        const int64_t rr = rb + lane;
        int64_t mp0 = 0, mp1 = 0;
        unsigned long long mkey = 0;
        unsigned mkey8 = 0;
        bool mneg = false;
        if (rr < rows) {
            const int q = inv_perm[rr];
            const int t = row_of2[q];
            mkey = ((unsigned long long)(unsigned)t << 32) | (unsigned)q;
            mkey8 = mode ? ((unsigned)t << (mode - 1)) | (unsigned)q : 0u;
            mneg = sign2[q] < 0.0;
            mp0 = indptr[rr];
            mp1 = indptr[rr + 1];
        }
        const int nr = (int)min((int64_t)32, rows - rb);
        for (int i = 0; i < nr; ++i) {
            const int64_t p0 = __shfl_sync(0xffffffffu, mp0, i);
            const int64_t p1 = __shfl_sync(0xffffffffu, mp1, i);
            const unsigned long long key = __shfl_sync(0xffffffffu, mkey, i);
            const unsigned key8 = __shfl_sync(0xffffffffu, mkey8, i);
            const bool neg = __shfl_sync(0xffffffffu, (int)mneg, i) != 0;
            for (int64_t pb = p0; pb < p1; pb += 32 * U) {
                int j[U];
                T v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t p = pb + u * 32 + lane;
                    j[u] = p < p1 ? indices[p] : -1;
                    v[u] = p < p1 ? vals[p] : T(0);
                }
                int64_t slot[U];
#pragma unroll
                for (int u = 0; u < U; ++u)
                    slot[u] = j[u] < 0 ? 0
                              : abs_cursor ? (int64_t)(unsigned)atomicAdd(fill + j[u], 1)
                                           : colptr[j[u]] + atomicAdd(fill + j[u], 1);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (j[u] < 0) continue;
                    if (mode) {
                        const float f = (float)v[u];
                        reinterpret_cast<unsigned long long *>(ent)[slot[u]] =
                            ((unsigned long long)key8 << 32) | __float_as_uint(neg ? -f : f);
                    } else {
                        const double d = (double)v[u];
                        reinterpret_cast<ulonglong2 *>(ent)[slot[u]] = make_ulonglong2(
                            key, (unsigned long long)__double_as_longlong(neg ? -d : d));
                    }
                }
            }
        }
    }
}


// ---------------------------------------------------------------------------
// Banded column count (no global atomics).  The rows are cut into B bands of
// consecutive rows, one CTA each, which counts the band's entries per column
// in shared memory (16-bit counters, two per word: a band has fewer than
// 65536 rows) and writes them as tab16[band][column]; a scan over the bands
// gives the column totals (config 4: 0.09 ms against 0.48 ms for one global
// atomic per entry).  The banded FILL below (entry placed at colptr[j] +
// off32[band][j] + a shared-memory cursor) is kept as an opt-in experiment
// (SRLU_CSR_BANDFILL=1): it needs no global atomics but writes bands x
// columns short pieces at once (310 MB of partly filled sectors in flight,
// far beyond L2), and measured 3.3 ms against 1.3 ms for the atomic fill,
// whose time-ordered slots keep one open sector per column (2 MB).

constexpr int kBandThreads = 1024;

__global__ void __launch_bounds__(kBandThreads) csr_band_count_kernel(
    const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices, int64_t rows,
    int64_t rows_per_band, int64_t n, uint16_t *__restrict__ tab16) {
    extern __shared__ __align__(16) unsigned cnt2[];   // (n + 1) / 2 packed pairs
    const int64_t nw = (n + 1) / 2;
    for (int64_t t = threadIdx.x; t < nw; t += kBandThreads) cnt2[t] = 0u;
    __syncthreads();
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_band;
    const int64_t r1 = min(rows, r0 + rows_per_band);
    if (r0 < r1) {
        const int64_t p0 = indptr[r0], p1 = indptr[r1];
        // four independent index loads in flight per thread
        for (int64_t pb = p0 + threadIdx.x; pb < p1; pb += 4 * kBandThreads) {
            int j[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t p = pb + (int64_t)u * kBandThreads;
                j[u] = p < p1 ? __ldg(indices + p) : -1;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (j[u] >= 0) atomicAdd(&cnt2[j[u] >> 1], (j[u] & 1) ? 0x10000u : 1u);
        }
    }
    __syncthreads();
    unsigned *dst = reinterpret_cast<unsigned *>(tab16 + (int64_t)blockIdx.x * (2 * nw));
    for (int64_t t = threadIdx.x; t < nw; t += kBandThreads) dst[t] = cnt2[t];
}

// one thread per column: exclusive scan over the bands, column total
__global__ void csr_band_scan_kernel(const uint16_t *__restrict__ tab16, int nbands, int64_t n,
                                     int64_t ldt, unsigned *__restrict__ off32,
                                     int *__restrict__ cnt) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    unsigned run = 0;
    for (int b = 0; b < nbands; ++b) {
        const unsigned c = tab16[(int64_t)b * ldt + j];
        off32[(int64_t)b * ldt + j] = run;
        run += c;
    }
    cnt[j] = (int)run;
}

template <typename T>
__global__ void __launch_bounds__(kBandThreads) csr_band_fill_kernel(
    const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
    const T *__restrict__ vals, int64_t rows, int64_t rows_per_band, int64_t n,
    const int32_t *__restrict__ inv_perm, const int32_t *__restrict__ row_of2,
    const double *__restrict__ sign2, const int64_t *__restrict__ colptr,
    const unsigned *__restrict__ off32, int64_t ldt, void *__restrict__ ent,
    const int *__restrict__ modep) {
    extern __shared__ __align__(16) unsigned cur2[];   // packed 16-bit cursors
    const int64_t nw = (n + 1) / 2;
    for (int64_t t = threadIdx.x; t < nw; t += kBandThreads) cur2[t] = 0u;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int mode = sizeof(T) == 4 ? *modep : 0;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_band;
    const int64_t r1 = min(rows, r0 + rows_per_band);
    const unsigned *off = off32 + (int64_t)blockIdx.x * ldt;
    constexpr int U = 4;
    for (int64_t rb = r0 + warp * 32; rb < r1; rb += (kBandThreads / 32) * 32) {
        const int64_t rr = rb + lane;
        int64_t mp0 = 0, mp1 = 0;
        unsigned long long mkey = 0;
        unsigned mkey8 = 0;
        bool mneg = false;
        if (rr < r1) {
            const int q = inv_perm[rr];
            const int t = row_of2[q];
            mkey = ((unsigned long long)(unsigned)t << 32) | (unsigned)q;
            mkey8 = mode ? ((unsigned)t << (mode - 1)) | (unsigned)q : 0u;
            mneg = sign2[q] < 0.0;
            mp0 = indptr[rr];
            mp1 = indptr[rr + 1];
        }
        const int nr = (int)min((int64_t)32, r1 - rb);
        for (int i = 0; i < nr; ++i) {
            const int64_t p0 = __shfl_sync(0xffffffffu, mp0, i);
            const int64_t p1 = __shfl_sync(0xffffffffu, mp1, i);
            const unsigned long long key = __shfl_sync(0xffffffffu, mkey, i);
            const unsigned key8 = __shfl_sync(0xffffffffu, mkey8, i);
            const bool neg = __shfl_sync(0xffffffffu, (int)mneg, i) != 0;
            for (int64_t pb = p0; pb < p1; pb += 32 * U) {
                int j[U];
                T v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t p = pb + u * 32 + lane;
                    j[u] = p < p1 ? __ldg(indices + p) : -1;
                    v[u] = p < p1 ? __ldg(vals + p) : T(0);
                }
                int64_t slot[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (j[u] < 0) { slot[u] = 0; continue; }
                    const unsigned old = atomicAdd(&cur2[j[u] >> 1], (j[u] & 1) ? 0x10000u : 1u);
                    const unsigned mine = (j[u] & 1) ? old >> 16 : old & 0xffffu;
                    slot[u] = __ldg(colptr + j[u]) + __ldg(off + j[u]) + mine;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (j[u] < 0) continue;
                    if (mode) {
                        const float f = (float)v[u];
                        reinterpret_cast<unsigned long long *>(ent)[slot[u]] =
                            ((unsigned long long)key8 << 32) | __float_as_uint(neg ? -f : f);
                    } else {
                        const double d = (double)v[u];
                        reinterpret_cast<ulonglong2 *>(ent)[slot[u]] = make_ulonglong2(
                            key, (unsigned long long)__double_as_longlong(neg ? -d : d));
                    }
                }
            }
        }
    }
}

// bands of the banded column sort for this shape: 0 = use the atomic path
static int csr_bands(int64_t rows, int64_t n) {
    const char *e = getenv("SRLU_CSR_BANDS");
    int want = e && *e ? atoi(e) : 148;
    if (want <= 0 || rows <= 0) return 0;
    if (((n + 1) / 2) * 4 > 200 * 1024) return 0;          // counters must fit shared memory
    int64_t b = want;
    while (ceil_div(rows, b) > 65535) b *= 2;              // 16-bit per-band counts
    if (b > rows) b = rows;
    if (b * ((n + 1) / 2 * 2) * 6 > (int64_t)1 << 30) return 0;   // tables beyond 1 GiB
    return (int)b;
}

// One CTA per column (grid-stride); handles columns with more than lo
// entries.  A column of at most CAP entries is sorted by key (t, q) in
// shared memory (bitonic) and each bucket's run folded in ascending q.  A
// longer column is split by bucket ranges: its bucket histogram (shared
// memory) is cut into ranges of at most CAP entries, and for each range the
// CTA re-reads the column's segment, keeps the entries of that range, sorts
// and folds them.  A single bucket with more than CAP entries (a column
// denser than CAP x l2) is folded in ascending-q chunks of at most CAP
// (each chunk's upper q bound found by bisection over q), the running sum
// carried from chunk to chunk — the reference's one sequential sum.  Any
// column length, the same per-bucket sums.
template <int CAP>
__device__ void csr_sort_fold(unsigned long long *sk, double *sv, int cnt) {
    int n2 = 1;
    while (n2 < cnt) n2 <<= 1;
    for (int i = cnt + threadIdx.x; i < n2; i += blockDim.x) {
        sk[i] = ~0ULL;
        sv[i] = 0.0;
    }
    __syncthreads();
    for (int kk = 2; kk <= n2; kk <<= 1) {
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
            for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                const int ixj = i ^ jj;
                if (ixj > i) {
                    const bool up = (i & kk) == 0;
                    const unsigned long long a = sk[i], b = sk[ixj];
                    if ((a > b) == up) {
                        sk[i] = b;
                        sk[ixj] = a;
                        const double tv = sv[i];
                        sv[i] = sv[ixj];
                        sv[ixj] = tv;
                    }
                }
            }
            __syncthreads();
        }
    }
}

template <int CAP>
__global__ void __launch_bounds__(256) csr_col_project_kernel(
    const int64_t *__restrict__ colptr, const void *__restrict__ ent, const int *__restrict__ modep,
    int64_t n, int l, int pad, const double *__restrict__ phase, const int32_t *__restrict__ idx,
    int k, double mult, double *__restrict__ out, int64_t ldo, int *flags, int lo,
    const int *__restrict__ maxcnt) {
    const int mode = *modep;
    if (maxcnt != nullptr && *maxcnt <= lo) return;  // no column for this launch
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *x = reinterpret_cast<double *>(smem_raw);                          // pad
    unsigned long long *sk = reinterpret_cast<unsigned long long *>(x + pad);  // CAP
    double *sv = reinterpret_cast<double *>(sk + CAP);                         // CAP
    int *hist = reinterpret_cast<int *>(sv + CAP);                             // l + 1
    __shared__ int s_nr, s_fill, s_cnt;
    __shared__ int s_rb[257];      // range boundaries (a batch of up to 256 ranges)
    __shared__ unsigned char s_big[256];
    __shared__ double s_acc;
    const bool reg = pad >= 32;
    const int bsize = pad < 512 ? pad : 512;
    const int nb = pad / bsize;
    const int nzb = (l + bsize - 1) / bsize;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
        const int64_t p0 = colptr[j];
        const int64_t cnt64 = colptr[j + 1] - p0;
        if (cnt64 <= lo) continue;  // handled by the smaller-capacity launch (uniform)
        for (int t = threadIdx.x; t < pad; t += blockDim.x) x[t] = 0.0;
        const bool longcol = cnt64 > CAP;
        if (longcol)
            for (int t = threadIdx.x; t <= l; t += blockDim.x) hist[t] = 0;
        __syncthreads();
        if (longcol) {
            for (int64_t i = threadIdx.x; i < cnt64; i += blockDim.x) {
                unsigned t;
                int q;
                double v;
                ent_read(ent, p0 + i, mode, t, q, v);
                atomicAdd(hist + t, 1);
            }
            __syncthreads();
        }
        int tstart = 0;  // first bucket not yet folded
        while (tstart < l) {
            if (threadIdx.x == 0) {
                int nr = 0, t = tstart;
                if (!longcol) {
                    s_rb[0] = 0;
                    s_rb[1] = l;
                    s_big[0] = 0;
                    nr = 1;
                } else {
                    s_rb[0] = t;
                    while (t < l && nr < 256) {
                        int acc = 0;
                        const int t0 = t;
                        while (t < l && acc + hist[t] <= CAP) acc += hist[t++];
                        s_big[nr] = 0;
                        if (t == t0) {  // bucket t alone exceeds CAP
                            s_big[nr] = 1;
                            ++t;
                        }
                        s_rb[++nr] = t;
                    }
                }
                s_nr = nr;
            }
            __syncthreads();
            const int nr = s_nr;
            for (int r = 0; r < nr; ++r) {
                const unsigned t0 = (unsigned)s_rb[r], t1 = (unsigned)s_rb[r + 1];
                if (!s_big[r]) {
                    if (threadIdx.x == 0) s_fill = 0;
                    __syncthreads();
                    // gather the range's entries (all of them for a short column)
                    for (int64_t i = threadIdx.x; i < cnt64; i += blockDim.x) {
                        unsigned t;
                        int q;
                        double v;
                        ent_read(ent, p0 + i, mode, t, q, v);
                        if (t >= t0 && t < t1) {
                            const int e = longcol ? atomicAdd(&s_fill, 1) : (int)i;
                            sk[e] = ((unsigned long long)t << 32) | (unsigned)q;
                            sv[e] = v;
                        }
                    }
                    __syncthreads();
                    const int cnt = longcol ? s_fill : (int)cnt64;
                    csr_sort_fold<CAP>(sk, sv, cnt);
                    // fold each bucket's run in ascending q (reference order)
                    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
                        const unsigned t = (unsigned)(sk[i] >> 32);
                        if (i > 0 && (unsigned)(sk[i - 1] >> 32) == t) continue;
                        double acc = 0.0;
                        for (int e = i; e < cnt && (unsigned)(sk[e] >> 32) == t; ++e)
                            acc = __dadd_rn(acc, sv[e]);
                        x[reg ? fwht_sw((int)t) : (int)t] = phase[t] < 0.0 ? -acc : acc;
                    }
                    __syncthreads();
                    continue;
                }
                // one oversized bucket t0: ascending-q chunks of <= CAP entries
                int remaining = hist[t0];
                long long qlast = -1;
                if (threadIdx.x == 0) s_acc = 0.0;
                while (remaining > 0) {
                    long long qhi = 0x7fffffffLL;
                    if (remaining > CAP) {  // largest qhi with count(qlast < q <= qhi) <= CAP
                        long long a = qlast, b = 0x7fffffffLL;
                        while (b - a > 1) {
                            const long long mid = a + (b - a) / 2;
                            if (threadIdx.x == 0) s_cnt = 0;
                            __syncthreads();
                            int c = 0;
                            for (int64_t i = threadIdx.x; i < cnt64; i += blockDim.x) {
                                unsigned t;
                                int q;
                                double v;
                                ent_read(ent, p0 + i, mode, t, q, v);
                                c += (t == t0 && q > qlast && q <= mid);
                            }
                            atomicAdd(&s_cnt, c);
                            __syncthreads();
                            if (s_cnt <= CAP) a = mid; else b = mid;
                            __syncthreads();
                        }
                        qhi = a;
                    }
                    if (threadIdx.x == 0) s_fill = 0;
                    __syncthreads();
                    for (int64_t i = threadIdx.x; i < cnt64; i += blockDim.x) {
                        unsigned t;
                        int q;
                        double v;
                        ent_read(ent, p0 + i, mode, t, q, v);
                        if (t == t0 && q > qlast && q <= qhi) {
                            const int e = atomicAdd(&s_fill, 1);
                            sk[e] = ((unsigned long long)t << 32) | (unsigned)q;
                            sv[e] = v;
                        }
                    }
                    __syncthreads();
                    const int cnt = s_fill;
                    csr_sort_fold<CAP>(sk, sv, cnt);
                    if (threadIdx.x == 0) {
                        double acc = s_acc;
                        for (int e = 0; e < cnt; ++e) acc = __dadd_rn(acc, sv[e]);
                        s_acc = acc;
                    }
                    __syncthreads();
                    remaining -= cnt;
                    qlast = qhi;
                    if (cnt == 0) {  // cannot happen (the bucket has entries above qlast)
                        if (flags != nullptr && threadIdx.x == 0) atomicOr(flags, 2);
                        break;
                    }
                }
                if (threadIdx.x == 0)
                    x[reg ? fwht_sw((int)t0) : (int)t0] = phase[t0] < 0.0 ? -s_acc : s_acc;
                __syncthreads();
            }
            tstart = s_rb[nr];
            __syncthreads();
        }
        if (reg) {
            for (int b = warp; b < nzb; b += blockDim.x >> 5)
                fwht_block_warp_dyn512(x + b * bsize, bsize, lane);
            __syncthreads();
        } else {
            fwht_smem_cta(x, pad);
        }
        for (int kk = threadIdx.x; kk < k; kk += blockDim.x) {
            const double fv = reg ? fwht_combine_blocks(x, bsize, nb, idx[kk]) : x[idx[kk]];
            out[j * ldo + kk] = __dmul_rn(fv, mult);
        }
        __syncthreads();
    }
}

// One CTA per column (grid-stride) for columns with at most CAP entries
// (the common case: ~nnz/n entries per column).  The segment is ordered by
// a counting sort on the bucket t in shared memory (histogram + block scan +
// scatter); the few entries of one bucket (~nnz/(n*l) on average) are then
// put in ascending q by the thread that folds that bucket (insertion sort),
// so every bucket sum is the reference's sequential sum in PA-row order.
template <int CAP, int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) csr_col_bucket_kernel(
    const int64_t *__restrict__ colptr, const void *__restrict__ ent, const int *__restrict__ modep,
    int64_t n, int l, int pad, const double *__restrict__ phase, const int32_t *__restrict__ idx,
    int k, double mult, double *__restrict__ out, int64_t ldo) {
    constexpr int PER = CAP / NT;
    const int mode = *modep;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *x = reinterpret_cast<double *>(smem_raw);   // pad
    double *sv = x + pad;                               // CAP
    int *sq = reinterpret_cast<int *>(sv + CAP);         // CAP
    int *base = sq + CAP;                               // l + 1
    __shared__ int wsum[NT / 32];
    const bool reg = pad >= 32;
    const int bsize = pad < 512 ? pad : 512;
    const int nb = pad / bsize;
    const int nzb = (l + bsize - 1) / bsize;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int chunk = (l + NT - 1) / NT;
    for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
        const int64_t p0 = colptr[j];
        const int cnt = (int)(colptr[j + 1] - p0);
        if (cnt > CAP) continue;  // uniform: the bitonic launch takes it
        for (int t = threadIdx.x; t <= l; t += NT) base[t] = 0;
        __syncthreads();
        unsigned et[PER];
        int eq[PER];
        double evv[PER];
        int off[PER];
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const int e = threadIdx.x + r * NT;
            off[r] = -1;
            et[r] = 0;
            eq[r] = 0;
            evv[r] = 0.0;
            if (e < cnt) ent_read(ent, p0 + e, mode, et[r], eq[r], evv[r]);
        }
#pragma unroll
        for (int r = 0; r < PER; ++r)
            if (threadIdx.x + r * NT < cnt) off[r] = atomicAdd(base + (int)et[r], 1);
        __syncthreads();
        // exclusive scan of the l bucket counts (chunk per thread)
        const int c0 = threadIdx.x * chunk;
        int s = 0;
        for (int c = 0; c < chunk; ++c)
            if (c0 + c < l) s += base[c0 + c];
        int incl = s;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += y;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        int wpre = 0;
        for (int w = 0; w < warp; ++w) wpre += wsum[w];
        int run = wpre + incl - s;
        for (int c = 0; c < chunk; ++c)
            if (c0 + c < l) {
                const int v = base[c0 + c];
                base[c0 + c] = run;
                run += v;
            }
        if (threadIdx.x == NT - 1) base[l] = cnt;
        __syncthreads();
#pragma unroll
        for (int r = 0; r < PER; ++r)
            if (off[r] >= 0) {
                const int pos = base[(int)et[r]] + off[r];
                sq[pos] = eq[r];
                sv[pos] = evv[r];
            }
        __syncthreads();
        for (int t = threadIdx.x; t < pad; t += NT) {
            double acc = 0.0;
            if (t < l) {
                const int b0 = base[t], b1 = base[t + 1];
                for (int a = b0 + 1; a < b1; ++a) {  // insertion sort by q (tiny runs)
                    const int qa = sq[a];
                    const double va = sv[a];
                    int b = a - 1;
                    while (b >= b0 && sq[b] > qa) {
                        sq[b + 1] = sq[b];
                        sv[b + 1] = sv[b];
                        --b;
                    }
                    sq[b + 1] = qa;
                    sv[b + 1] = va;
                }
                for (int a = b0; a < b1; ++a) acc = __dadd_rn(acc, sv[a]);
                if (phase[t] < 0.0) acc = -acc;
            }
            x[reg ? fwht_sw(t) : t] = acc;
        }
        __syncthreads();
        if (reg) {
            for (int b = warp; b < nzb; b += NT >> 5) fwht_block_warp_dyn512(x + b * bsize, bsize, lane);
            __syncthreads();
        } else {
            fwht_smem_cta(x, pad);
        }
        for (int kk = threadIdx.x; kk < k; kk += NT) {
            const double fv = reg ? fwht_combine_blocks(x, bsize, nb, idx[kk]) : x[idx[kk]];
            out[j * ldo + kk] = __dmul_rn(fv, mult);
        }
        __syncthreads();
    }
}

struct CsrWs {
    int *cnt, *fill, *maxcnt, *mode;
    int64_t *colptr;
    void *ent;
    uint16_t *tab16;   // banded sort: [bands][ldt] counts
    unsigned *off32;   //              [bands][ldt] offsets inside the column
    int64_t *tsum;     // tile sums of the column-count scan
};

static size_t csr_ws_layout(int64_t rows, int64_t n, int64_t nnz, char *base, CsrWs *w) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) & ~(size_t)255;
        return base ? base + o : nullptr;
    };
    char *p;
    p = take(sizeof(int) * n);             if (w) w->cnt = (int *)p;
    p = take(sizeof(int) * n);             if (w) w->fill = (int *)p;
    p = take(sizeof(int) * 4);             if (w) w->maxcnt = (int *)p;
    p = take(sizeof(int) * 4);             if (w) w->mode = (int *)p;
    p = take(sizeof(int64_t) * (n + 1));   if (w) w->colptr = (int64_t *)p;
    p = take(sizeof(ulonglong2) * (nnz > 0 ? nnz : 1)); if (w) w->ent = (void *)p;
    const int64_t nb = csr_bands(rows, n), ldt = (n + 1) / 2 * 2;
    p = take(sizeof(uint16_t) * (nb ? nb * ldt : 1)); if (w) w->tab16 = (uint16_t *)p;
    p = take(sizeof(unsigned) * (nb ? nb * ldt : 1)); if (w) w->off32 = (unsigned *)p;
    p = take(sizeof(int64_t) * (ceil_div(n, (int64_t)1024) + 1)); if (w) w->tsum = (int64_t *)p;
    return off;
}

template <typename T>
static int run_csr_left(const int64_t *indptr, const int32_t *indices, const T *vals, int64_t rows,
                        int64_t n, int64_t nnz, const int32_t *inv_perm, const int32_t *row_of2,
                        const double *sign2, int64_t l2, const double *phase2,
                        const int32_t *idx2, int64_t k2, int64_t pad2, double mult2,
                        double *out, int64_t ldo, void *ws, int *flags, cudaStream_t s) {
    CsrWs w;
    csr_ws_layout(rows, n, nnz, (char *)ws, &w);
    const int nbands = csr_bands(rows, n);
    const int64_t ldt = (n + 1) / 2 * 2, rows_per_band = nbands ? ceil_div(rows, (int64_t)nbands) : 0;
    const size_t band_smem = (size_t)((n + 1) / 2) * 4;
    SRLU_CUDA(cudaMemsetAsync(w.cnt, 0, sizeof(int) * n, s));
    SRLU_CUDA(cudaMemsetAsync(w.fill, 0, sizeof(int) * n, s));
    // cursors start at the column's first slot (one scattered access per entry less)
    const int abs_cursor = n >= 8 * kScanTile && nnz < (1LL << 32) - 1 ? 1 : 0;
    SRLU_CUDA(cudaMemsetAsync(w.mode, 0, sizeof(int) * 4, s));
    if (rows > 0) {
        int64_t blocks = ceil_div(rows, 256);
        if (blocks > 148 * 4) blocks = 148 * 4;
        csr_mode_kernel<<<(unsigned)blocks, 256, 0, s>>>(inv_perm, rows, (int)l2,
                                                         sizeof(T) == 4 && !getenv("SRLU_CSR_E16"),
                                                         w.mode);
        SRLU_CHECK_LAUNCH("csr_mode_kernel");
    }
    if (nbands) {
        SRLU_CUDA(cudaFuncSetAttribute(csr_band_count_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)band_smem));
        csr_band_count_kernel<<<nbands, kBandThreads, band_smem, s>>>(indptr, indices, rows,
                                                                     rows_per_band, n, w.tab16);
        SRLU_CHECK_LAUNCH("csr_band_count_kernel");
        csr_band_scan_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(w.tab16, nbands, n, ldt,
                                                                       w.off32, w.cnt);
        SRLU_CHECK_LAUNCH("csr_band_scan_kernel");
    } else if (nnz > 0) {
        csr_col_count_kernel<<<148 * 8, 256, 0, s>>>(indices, nnz, w.cnt);
        SRLU_CHECK_LAUNCH("csr_col_count_kernel");
    }
    if (n >= 8 * kScanTile) {
        const int ntiles = (int)ceil_div(n, (int64_t)kScanTile);
        SRLU_CUDA(cudaMemsetAsync(w.maxcnt, 0, sizeof(int), s));
        csr_scan_tiles_kernel<<<ntiles, 256, 0, s>>>(w.cnt, n, w.tsum, w.maxcnt);
        csr_scan_tsum_kernel<<<1, 256, 0, s>>>(w.tsum, ntiles, w.colptr + n);
        csr_scan_apply_kernel<<<ntiles, 256, 0, s>>>(w.cnt, n, w.tsum, w.colptr,
                                                     abs_cursor ? w.fill : nullptr);
        SRLU_CHECK_LAUNCH("csr_scan_apply_kernel");
    } else {
        csr_col_scan_kernel<<<1, 1024, 0, s>>>(w.cnt, n, w.colptr, w.maxcnt);
        SRLU_CHECK_LAUNCH("csr_col_scan_kernel");
    }
    if (nbands && getenv("SRLU_CSR_BANDFILL") != nullptr) {
        SRLU_CUDA(cudaFuncSetAttribute(csr_band_fill_kernel<T>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)band_smem));
        csr_band_fill_kernel<T><<<nbands, kBandThreads, band_smem, s>>>(
            indptr, indices, vals, rows, rows_per_band, n, inv_perm, row_of2, sign2, w.colptr,
            w.off32, ldt, w.ent, w.mode);
        SRLU_CHECK_LAUNCH("csr_band_fill_kernel");
    } else if (rows > 0) {
        int64_t blocks = ceil_div(rows * 32, 256);
        if (blocks > 148 * 16) blocks = 148 * 16;
        csr_fill_kernel<T><<<(unsigned)blocks, 256, 0, s>>>(indptr, indices, vals, rows, inv_perm,
                                                           row_of2, sign2, w.colptr, w.fill, abs_cursor,
                                                           w.ent, w.mode);
        SRLU_CHECK_LAUNCH("csr_fill_kernel");
    }
    // columns with <= 2048 entries: bucket counting sort (high occupancy);
    // longer ones in a bitonic launch (bucket ranges of <= 8192 entries)
    const int64_t grid = n < 148 * 16 ? n : 148 * 16;
    {
        constexpr int CAP = 2048;
        size_t smem = sizeof(double) * pad2 + (sizeof(double) + sizeof(int)) * CAP +
                      sizeof(int) * (l2 + 1);
        SRLU_REQUIRE(smem <= 220 * 1024, SRLU_ERR_UNSUPPORTED, "sketch_left_csr: pad2 too large");
        const char *ntenv = getenv("SRLU_CSR_NT");  // testing knob: 512
        if (ntenv && atoi(ntenv) == 512) {
            SRLU_CUDA(cudaFuncSetAttribute(csr_col_bucket_kernel<CAP, 512>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            csr_col_bucket_kernel<CAP, 512><<<(unsigned)grid, 512, smem, s>>>(
                w.colptr, w.ent, w.mode, n, (int)l2, (int)pad2, phase2, idx2, (int)k2, mult2, out,
                ldo);
        } else {
            SRLU_CUDA(cudaFuncSetAttribute(csr_col_bucket_kernel<CAP, 256>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            csr_col_bucket_kernel<CAP, 256><<<(unsigned)grid, 256, smem, s>>>(
                w.colptr, w.ent, w.mode, n, (int)l2, (int)pad2, phase2, idx2, (int)k2, mult2, out,
                ldo);
        }
        SRLU_CHECK_LAUNCH("csr_col_bucket_kernel");
    }
    {
        size_t smem = sizeof(double) * pad2 + (sizeof(unsigned long long) + sizeof(double)) * kCsrColCap +
                      sizeof(int) * (l2 + 1);
        SRLU_REQUIRE(smem <= 220 * 1024, SRLU_ERR_UNSUPPORTED, "sketch_left_csr: pad2 too large");
        SRLU_CUDA(cudaFuncSetAttribute(csr_col_project_kernel<kCsrColCap>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        csr_col_project_kernel<kCsrColCap><<<(unsigned)(grid < 148 ? grid : 148), 256, smem, s>>>(
            w.colptr, w.ent, w.mode, n, (int)l2, (int)pad2, phase2, idx2, (int)k2, mult2, out, ldo,
            flags, 2048, w.maxcnt);
    }
    SRLU_CHECK_LAUNCH("csr_col_project_kernel");
    return SRLU_OK;
}

}  // namespace srlu

using namespace srlu;

extern "C" size_t srlu_sketch_left_csr_workspace(int64_t rows, int64_t n, int64_t nnz, int64_t l2,
                                                 int64_t pad2) {
    (void)l2; (void)pad2;
    return csr_ws_layout(rows, n, nnz, nullptr, nullptr) + 256;
}

extern "C" int srlu_sketch_left_csr(const int64_t *indptr, const int32_t *indices,
                                    const void *vals, int dtype, int64_t rows, int64_t n,
                                    int64_t nnz, const int32_t *inv_perm, const int32_t *row_of2,
                                    const double *sign2, int64_t l2, const double *phase2,
                                    const int32_t *idx2, int64_t k2, int64_t pad2, double mult2,
                                    double *out, int64_t ldo, void *ws, size_t ws_bytes,
                                    int *flags, srlu_stream_t stream) {
    SRLU_REQUIRE(rows >= 0 && n >= 1 && l2 >= 1 && k2 >= 1 && k2 <= pad2 && pad2 >= l2 &&
                     (pad2 & (pad2 - 1)) == 0 && ldo >= k2 && nnz >= 0,
                 SRLU_ERR_ARG, "sketch_left_csr: bad sizes");
    SRLU_REQUIRE(rows < (1LL << 31) && l2 < (1LL << 31), SRLU_ERR_UNSUPPORTED,
                 "sketch_left_csr: sizes beyond int32");
    SRLU_REQUIRE(ws_bytes >= srlu_sketch_left_csr_workspace(rows, n, nnz, l2, pad2),
                 SRLU_ERR_WORKSPACE, "sketch_left_csr: workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == SRLU_F32)
        return run_csr_left<float>(indptr, indices, (const float *)vals, rows, n, nnz, inv_perm,
                                   row_of2, sign2, l2, phase2, idx2, k2, pad2, mult2, out, ldo,
                                   ws, flags, s);
    if (dtype == SRLU_F64)
        return run_csr_left<double>(indptr, indices, (const double *)vals, rows, n, nnz,
                                    inv_perm, row_of2, sign2, l2, phase2, idx2, k2, pad2, mult2,
                                    out, ldo, ws, flags, s);
    set_error("sketch_left_csr: unknown dtype %d", dtype);
    return SRLU_ERR_ARG;
}
