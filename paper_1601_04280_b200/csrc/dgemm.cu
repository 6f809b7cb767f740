// FP64 tensor-core (DMMA) GEMMs of the pipeline's tail and the fused
// approximation error (K7).
//
//  * srlu_dgemm: C = A·B, row-major fp64 — core = pinv·(Omega2 P A)
//    (reference randlu.py:267) as core^T = (Omega2 P A)^T · pinv^T, and
//    L = L1·L~ (randlu.py:272; matrix.py:219-230 matmul).  With
//    SRLU_GEMM_B_LOWER the K loop of an output column tile starts at its
//    first column (L~ is unit lower triangular: B[j][c] = 0 for j < c), which
//    halves the flops of L1·L~.
//  * srlu_lu_error_dense / _csr: ||L U - P A Q||_F (randlu.py:279-302) as
//    ||L·Ũ - P·A||_F with Ũ = U·Q^T (the column permutation moves to the
//    small factor, so A is read row by row, coalesced): the L·Ũ tile never
//    leaves the SM — the epilogue subtracts A[perm[i], j] and accumulates
//    squares; per-CTA partials are summed in a fixed order (deterministic).
//
// Mainloop: CTA tile BM x BN x 16, warps of WM x WN, each warp issuing
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4) on fragments read from padded shared
// tiles (2 wavefronts per 256-byte fragment load = the minimum); a
// STAGES-deep cp.async (LDGSTS) ring with zero fill at the edges.
//
// Fragment layouts (PTX m8n8k4 .row.col f64): A 8x4 — lane holds
// A[lane/4][lane%4]; B 4x8 — B[lane%4][lane/4]; C 8x8 — C[lane/4][2(lane%4)+{0,1}].
#include <math.h>
#include <stdlib.h>

#include <algorithm>

#include "async_copy.cuh"
#include "common.cuh"

namespace srlu {
namespace dmma {

constexpr int BK = 16;
constexpr int AST = BK;  // A/B^T tile row stride (doubles)

// XOR-swizzled shared tiles (no padding).  A 64-bit shared load is served
// per half-warp, so each half-warp's 16 fragment elements must hit 16
// different 8-byte bank slots: rows x 16 tile (A, B^T): 16-byte chunk c of
// row r lives at chunk c ^ 2(r & 3); 16 x BN tile (row-major B): chunk c of
// k-row k lives at chunk c ^ 2(k & 3).  A quarter-warp's 16-byte LDGSTS
// writes 8 consecutive chunks of one row: a permutation of the 8 positions.
__host__ __device__ constexpr int off_rk(int r, int k) {
    return r * AST + ((((k >> 1) ^ ((r & 3) << 1)) << 1) | (k & 1));
}
template <int BN>
__host__ __device__ constexpr int off_kc(int k, int n) {
    return k * BN + ((((n >> 1) ^ ((k & 3) << 1)) << 1) | (n & 1));
}

__device__ __forceinline__ void mma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

template <int BM, int BN, int WM, int WN, int STAGES, bool BT>
struct Tile {
    static constexpr int NWM = BM / WM, NWN = BN / WN;
    static constexpr int NT = NWM * NWN * 32;
    static constexpr int MI = WM / 8, NI = WN / 8;
    static constexpr int BST = BN;  // row-major B tile row stride (doubles)
    static constexpr int A_STAGE = BM * AST;
    static constexpr int B_STAGE = BT ? BN * AST : BK * BST;
    static constexpr size_t SMEM = sizeof(double) * (size_t)STAGES * (A_STAGE + B_STAGE);
    static_assert(BM % WM == 0 && BN % WN == 0 && WM % 8 == 0 && WN % 8 == 0, "tile shape");
};

__device__ __forceinline__ void cp_async_zfill(uint32_t dst, const void *src, int bytes,
                                              bool ok) {
    if (bytes == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                     "r"(ok ? 16 : 0)
                     : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src),
                     "r"(ok ? 8 : 0)
                     : "memory");
}

// Per-thread copy descriptors of a rows x 16 (k) tile of a row-major
// (rows x K) operand into shared [R][16] (off_rk): one source pointer and the
// row index of the thread's first chunk; chunk p sits NT/CPR rows further (a
// multiple of 4 rows, so its swizzled shared offset is a constant step).
// Each k-tile is then one predicate and one LDGSTS per chunk.  VEC: 16-byte
// chunks (K even, ld even, 16-byte base), else 8-byte.
template <int R, int NT, bool VEC>
struct RowsLoader {
    static constexpr int W = VEC ? 2 : 1;           // doubles per chunk
    static constexpr int CPR = BK / W;               // chunks per row
    static constexpr int RSTEP = NT / CPR;           // rows between a thread's chunks
    static constexpr int PER = (R + RSTEP - 1) / RSTEP;
    static_assert(NT % CPR == 0 && RSTEP % 4 == 0, "loader geometry");
    const double *src;
    int64_t step;
    int row, rows_left, kof;
    uint32_t dst;
    __device__ __forceinline__ void init(const double *__restrict__ a, int64_t rows, int64_t ld,
                                         int64_t r0) {
        const int r = threadIdx.x / CPR, c = (threadIdx.x % CPR) * W;
        row = r;
        rows_left = (int)(rows - r0 < (int64_t)R ? rows - r0 : (int64_t)R);
        src = a + (r0 + r) * ld + c;
        step = (int64_t)RSTEP * ld;
        kof = c;
        dst = (uint32_t)(off_rk(r, c) * sizeof(double));
    }
    __device__ __forceinline__ void load(uint32_t stage, int k0, int K,
                                         const double *__restrict__ base) const {
        const bool kok = k0 + kof < K;
        const double *p = src + k0;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            if (PER * RSTEP > R && row + q * RSTEP >= R) continue;
            const bool v = kok && row + q * RSTEP < rows_left;
            cp_async_zfill(stage + dst + q * (uint32_t)(RSTEP * AST * sizeof(double)),
                           v ? p : base, W * 8, v);
            p += step;
        }
    }
};

// Per-thread copy descriptors of a 16 (k) x BN tile of a row-major (K x N)
// operand into shared [16][BN] (off_kc): 32-bit element offsets.
template <int BN, int BST, int NT, bool VEC>
struct KColsLoader {
    static constexpr int W = VEC ? 2 : 1;
    static constexpr int CPR = BN / W;
    static constexpr int PER = (BK * CPR + NT - 1) / NT;
    int off[PER];
    uint32_t dst[PER];
    uint32_t kmask;   // bit p: chunk p's column is inside the matrix
    __device__ __forceinline__ void init(int64_t N, int64_t ld, int64_t c0) {
        kmask = 0;
#pragma unroll
        for (int p = 0; p < PER; ++p) {
            const int idx = threadIdx.x + p * NT;
            const int r = idx / CPR, c = (idx % CPR) * W;
            if (idx < BK * CPR && c0 + c < N) kmask |= 1u << p;
            off[p] = (int)(r * ld + c);
            dst[p] = (uint32_t)(off_kc<BST>(r, c) * sizeof(double));
        }
    }
    __device__ __forceinline__ void load(uint32_t stage, int k0, int K,
                                         const double *__restrict__ b, int64_t ld) const {
        const double *p0 = b + (int64_t)k0 * ld;
#pragma unroll
        for (int p = 0; p < PER; ++p) {
            if (PER * NT > BK * CPR && threadIdx.x + p * NT >= BK * CPR) continue;
            const int r = (threadIdx.x + p * NT) / CPR;
            const bool v = ((kmask >> p) & 1u) && k0 + r < K;
            cp_async_zfill(stage + dst[p], v ? p0 + off[p] : b, W * 8, v);
        }
    }
};

// acc (this warp's WM x WN sub-tile of the CTA tile at (m0, n0)) =
// A[m0:, kt_begin*16 : K] · B[kt_begin*16 : K, n0:].  B is row-major K x N,
// or (BT) given as its transpose, row-major N x K.
template <int BM, int BN, int WM, int WN, int STAGES, bool BT, bool VEC>
__device__ __forceinline__ void mainloop(double *smem, const double *__restrict__ A, int64_t lda,
                                         const double *__restrict__ B, int64_t ldb, int64_t M,
                                         int64_t N, int K, int64_t m0, int64_t n0, int kt_begin,
                                         double (&acc)[WM / 8][WN / 8][2]) {
    using T = Tile<BM, BN, WM, WN, STAGES, BT>;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm0 = (warp / T::NWN) * WM, wn0 = (warp % T::NWN) * WN;
    const int kt_end = (K + BK - 1) / BK;
#pragma unroll
    for (int i = 0; i < T::MI; ++i)
#pragma unroll
        for (int j = 0; j < T::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const uint32_t sA = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t sB = sA + (uint32_t)(STAGES * T::A_STAGE * sizeof(double));
    RowsLoader<BM, T::NT, VEC> la;
    la.init(A, M, lda, m0);
    RowsLoader<BN, T::NT, VEC> lbt;
    KColsLoader<BN, T::BST, T::NT, VEC> lb;
    const double *Bc = B + (BT ? 0 : n0);   // row-major B: this tile's first column
    if (BT)
        lbt.init(B, N, ldb, n0);
    else
        lb.init(N, ldb, n0);
    auto load = [&](int slot, int kt) {
        const int k0 = kt * BK;
        la.load(sA + slot * (uint32_t)(T::A_STAGE * sizeof(double)), k0, K, A);
        const uint32_t sb = sB + slot * (uint32_t)(T::B_STAGE * sizeof(double));
        if (BT)
            lbt.load(sb, k0, K, B);
        else
            lb.load(sb, k0, K, Bc, ldb);
    };
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (kt_begin + s < kt_end) load(s, kt_begin + s);
        cp_async_commit();
    }
    const int ar = lane >> 2, ac = lane & 3;
    // per-thread fragment offsets (off_rk / off_kc at the lane's element):
    // A element (wm0 + 8i + ar, kk + ac) = offA[kk/4] + 8i*16; row-major B
    // element (kk + ac, wn0 + 8j + ar) = kk*BN + offB[j]
    int offA[BK / 4], offB[BT ? BK / 4 : T::NI];
#pragma unroll
    for (int q = 0; q < BK / 4; ++q) offA[q] = off_rk(wm0 + ar, 4 * q + ac);
    if (BT) {
#pragma unroll
        for (int q = 0; q < BK / 4; ++q) offB[q] = off_rk(wn0 + ar, 4 * q + ac);
    } else {
#pragma unroll
        for (int j = 0; j < T::NI; ++j) offB[j] = off_kc<T::BST>(ac, wn0 + 8 * j + ar);
    }
    const double *as0 = smem;
    const double *bs0 = smem + STAGES * T::A_STAGE;
    int rslot = 0, wslot = STAGES - 1;
    for (int kt = kt_begin; kt < kt_end; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        if (kt + STAGES - 1 < kt_end) load(wslot, kt + STAGES - 1);
        cp_async_commit();
        wslot = wslot == STAGES - 1 ? 0 : wslot + 1;
        const double *as = as0 + rslot * T::A_STAGE;
        const double *bs = bs0 + rslot * T::B_STAGE;
        rslot = rslot == STAGES - 1 ? 0 : rslot + 1;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[T::MI], bf[T::NI];
#pragma unroll
            for (int i = 0; i < T::MI; ++i) af[i] = as[offA[kk / 4] + i * 8 * AST];
#pragma unroll
            for (int j = 0; j < T::NI; ++j)
                bf[j] = BT ? bs[offB[kk / 4] + j * 8 * AST] : bs[kk * T::BST + offB[j]];
#pragma unroll
            for (int i = 0; i < T::MI; ++i)
#pragma unroll
                for (int j = 0; j < T::NI; ++j) mma884(acc[i][j], af[i], bf[j]);
        }
    }
    cp_async_wait<0>();
    __syncthreads();  // the ring may be reused by the caller's next tile / epilogue
}

// ---------------------------------------------------------------------------
// C = A·B

template <int BM, int BN, int WM, int WN, int STAGES, bool VEC, int MINB>
__global__ void __launch_bounds__(Tile<BM, BN, WM, WN, STAGES, false>::NT, MINB)
    gemm_kernel(const double *__restrict__ A, int64_t lda, const double *__restrict__ B,
                int64_t ldb, double *__restrict__ C, int64_t ldc, int64_t M, int64_t N, int K,
                int b_lower) {
    using T = Tile<BM, BN, WM, WN, STAGES, false>;
    extern __shared__ __align__(16) double smem[];
    const int64_t n0 = (int64_t)blockIdx.x * BN;
    const int64_t m0 = (int64_t)blockIdx.y * BM;
    // B lower triangular: rows j < n0 of B are zero in this column tile
    const int kt_begin = b_lower ? (int)(n0 / BK) : 0;
    double acc[T::MI][T::NI][2];
    mainloop<BM, BN, WM, WN, STAGES, false, VEC>(smem, A, lda, B, ldb, M, N, K, m0, n0, kt_begin,
                                                 acc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = m0 + (warp / T::NWN) * WM + (lane >> 2);
    const int64_t c0 = n0 + (warp % T::NWN) * WN + 2 * (lane & 3);
#pragma unroll
    for (int i = 0; i < T::MI; ++i) {
        const int64_t r = r0 + i * 8;
        if (r >= M) continue;
#pragma unroll
        for (int j = 0; j < T::NI; ++j) {
            const int64_t c = c0 + j * 8;
            double *dst = C + r * ldc + c;
            if (VEC && c + 1 < N) {
                *reinterpret_cast<double2 *>(dst) = make_double2(acc[i][j][0], acc[i][j][1]);
            } else {
                if (c < N) dst[0] = acc[i][j][0];
                if (c + 1 < N) dst[1] = acc[i][j][1];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// K7: sum over the tile of (L·Ũ - P·A)^2; L (m x k, positions), ŨT (n x k).

template <typename V>
__device__ __forceinline__ double to_f64(V v) { return (double)v; }

template <int BM, int BN, int WM, int WN, int STAGES, bool VEC, typename V>
__global__ void __launch_bounds__(Tile<BM, BN, WM, WN, STAGES, true>::NT)
    err_dense_kernel(const double *__restrict__ L, int64_t ldl, const double *__restrict__ UtT,
                     int64_t ldu, const int64_t *__restrict__ perm, const V *__restrict__ a,
                     int64_t lda, int64_t m, int64_t n, int k, double *__restrict__ partial) {
    using T = Tile<BM, BN, WM, WN, STAGES, true>;
    extern __shared__ __align__(16) double smem[];
    __shared__ double red[T::NT / 32];
    const int64_t n0 = (int64_t)blockIdx.x * BN;
    const int64_t m0 = (int64_t)blockIdx.y * BM;
    double acc[T::MI][T::NI][2];
    mainloop<BM, BN, WM, WN, STAGES, true, VEC>(smem, L, ldl, UtT, ldu, m, n, k, m0, n0, 0, acc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = m0 + (warp / T::NWN) * WM + (lane >> 2);
    const int64_t c0 = n0 + (warp % T::NWN) * WN + 2 * (lane & 3);
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < T::MI; ++i) {
        const int64_t r = r0 + i * 8;
        if (r >= m) continue;
        const V *arow = a + perm[r] * lda;
#pragma unroll
        for (int j = 0; j < T::NI; ++j) {
            const int64_t c = c0 + j * 8;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                if (c + e < n) {
                    const double d = __dsub_rn(acc[i][j][e], to_f64(arow[c + e]));
                    s = __dadd_rn(s, __dmul_rn(d, d));
                }
            }
        }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < T::NT / 32; ++w) t += red[w];
        partial[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}

// CSR A: one CTA per BM positions walks every column tile; each row's CSR
// cursor only moves forward (columns ascending), so the sparse entries of
// P·A are subtracted from the tile in shared memory without a search.
template <int BM, int BN, int WM, int WN, int STAGES, bool VEC, typename V>
__global__ void __launch_bounds__(Tile<BM, BN, WM, WN, STAGES, true>::NT)
    err_csr_kernel(const double *__restrict__ L, int64_t ldl, const double *__restrict__ UtT,
                   int64_t ldu, const int64_t *__restrict__ perm,
                   const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                   const V *__restrict__ vals, int64_t m, int64_t n, int k,
                   double *__restrict__ partial) {
    using T = Tile<BM, BN, WM, WN, STAGES, true>;
    constexpr int TS = BN + 1;
    extern __shared__ __align__(16) double smem[];
    double *tile = smem + STAGES * (T::A_STAGE + T::B_STAGE);
    __shared__ int64_t cur[BM], lim[BM];
    __shared__ double red[T::NT / 32];
    const int64_t m0 = (int64_t)blockIdx.x * BM;
    for (int t = threadIdx.x; t < BM; t += T::NT) {
        if (m0 + t < m) {
            const int64_t r = perm[m0 + t];
            cur[t] = indptr[r];
            lim[t] = indptr[r + 1];
        } else {
            cur[t] = lim[t] = 0;
        }
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rl0 = (warp / T::NWN) * WM + (lane >> 2);
    const int cl0 = (warp % T::NWN) * WN + 2 * (lane & 3);
    const int rows = (int)(m - m0 < BM ? m - m0 : BM);
    double s = 0.0;
    for (int64_t n0 = 0; n0 < n; n0 += BN) {
        double acc[T::MI][T::NI][2];
        mainloop<BM, BN, WM, WN, STAGES, true, VEC>(smem, L, ldl, UtT, ldu, m, n, k, m0, n0, 0,
                                                    acc);
#pragma unroll
        for (int i = 0; i < T::MI; ++i)
#pragma unroll
            for (int j = 0; j < T::NI; ++j) {
                tile[(rl0 + i * 8) * TS + cl0 + j * 8] = acc[i][j][0];
                tile[(rl0 + i * 8) * TS + cl0 + j * 8 + 1] = acc[i][j][1];
            }
        __syncthreads();
        const int64_t n1 = n0 + BN;
        for (int t = threadIdx.x; t < rows; t += T::NT) {
            int64_t p = cur[t];
            const int64_t e = lim[t];
            while (p < e && indices[p] < n1) {
                double *d = tile + t * TS + (indices[p] - n0);
                *d = __dsub_rn(*d, to_f64(vals[p]));
                ++p;
            }
            cur[t] = p;
        }
        __syncthreads();
        const int cols = (int)(n - n0 < BN ? n - n0 : BN);
        for (int idx = threadIdx.x; idx < rows * BN; idx += T::NT) {
            const int r = idx / BN, c = idx % BN;
            if (c < cols) {
                const double d = tile[r * TS + c];
                s = __dadd_rn(s, __dmul_rn(d, d));
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < T::NT / 32; ++w) t += red[w];
        partial[blockIdx.x] = t;
    }
}

// ŨT[q[c], :] = UT[c, :]  (Ũ = U Q^T)
__global__ void scatter_rows_kernel(const double *__restrict__ ut, int64_t ldut,
                                    const int64_t *__restrict__ q, double *__restrict__ out,
                                    int64_t ldo, int64_t n, int k) {
    for (int64_t c = blockIdx.x; c < n; c += gridDim.x) {
        const double *src = ut + c * ldut;
        double *dst = out + q[c] * ldo;
        for (int j = threadIdx.x; j < k; j += blockDim.x) dst[j] = src[j];
    }
}

// fixed-order sum of the per-CTA partials (one CTA): deterministic
__global__ void sum_partials_kernel(const double *__restrict__ partial, int64_t count,
                                    double *__restrict__ out) {
    __shared__ double red[32];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < count; i += blockDim.x) s += partial[i];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        *out = t;
    }
}

// tile configurations (measured on B200 against cuBLAS DMMA, tools/bench_dgemm.py;
// profiles/r02/dgemm_tiles.txt): 4 warps of 32 x (BN/2), 16-deep k steps,
// XOR-swizzled shared tiles, 3 or 4 CTAs per SM
struct Cfg64x64 { static constexpr int BM = 64, BN = 64, WM = 32, WN = 32, ST = 3, MB = 4; };
struct Cfg64x80 { static constexpr int BM = 64, BN = 80, WM = 32, WN = 40, ST = 3, MB = 3; };
struct Cfg64x112 { static constexpr int BM = 64, BN = 112, WM = 32, WN = 56, ST = 3, MB = 3; };
struct Cfg128x64 { static constexpr int BM = 128, BN = 64, WM = 32, WN = 32, ST = 3, MB = 2; };
using ErrCfg = Cfg128x64;

template <class C, bool VEC>
static int launch_gemm(const double *A, int64_t lda, const double *B, int64_t ldb, double *Cm,
                       int64_t ldc, int64_t M, int64_t N, int64_t K, int b_lower,
                       cudaStream_t st) {
    using T = Tile<C::BM, C::BN, C::WM, C::WN, C::ST, false>;
    auto kern = gemm_kernel<C::BM, C::BN, C::WM, C::WN, C::ST, VEC, C::MB>;
    SRLU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)T::SMEM));
    dim3 grid((unsigned)ceil_div(N, C::BN), (unsigned)ceil_div(M, C::BM));
    SRLU_REQUIRE(grid.y <= 65535u, SRLU_ERR_UNSUPPORTED, "dgemm: M too large (%lld)",
                 (long long)M);
    kern<<<grid, T::NT, T::SMEM, st>>>(A, lda, B, ldb, Cm, ldc, M, N, (int)K, b_lower);
    SRLU_CHECK_LAUNCH("dgemm gemm_kernel");
    return SRLU_OK;
}

static inline bool al16(const void *p) { return ((uintptr_t)p & 15) == 0; }

// tile choice: BN = 80 when it pads N less than BN = 64 (N = 220, 550), else
// 64 x 64 (also for the triangular L~ products, whose skipped blocks favour
// narrow column tiles)
static int pick_cfg(int64_t N, int b_lower) {
    const char *e = getenv("SRLU_DGEMM_TILE");
    if (e && *e) return atoi(e);
    if (b_lower) return 0;
    return ceil_div(N, 80) * 80 < ceil_div(N, 64) * 64 ? 1 : 0;
}

template <bool VEC>
static int gemm_dispatch(const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                         int64_t ldc, int64_t M, int64_t N, int64_t K, int b_lower,
                         cudaStream_t st) {
    switch (pick_cfg(N, b_lower)) {
    case 1: return launch_gemm<Cfg64x80, VEC>(A, lda, B, ldb, C, ldc, M, N, K, b_lower, st);
    case 2: return launch_gemm<Cfg64x112, VEC>(A, lda, B, ldb, C, ldc, M, N, K, b_lower, st);
    case 3: return launch_gemm<Cfg128x64, VEC>(A, lda, B, ldb, C, ldc, M, N, K, b_lower, st);
    default: return launch_gemm<Cfg64x64, VEC>(A, lda, B, ldb, C, ldc, M, N, K, b_lower, st);
    }
}

template <bool VEC, typename V>
static int launch_err_dense(const double *L, int64_t ldl, const double *UtT, int64_t ldu,
                            const int64_t *perm, const V *a, int64_t lda, int64_t m, int64_t n,
                            int64_t k, double *partial, cudaStream_t st, dim3 grid) {
    using C = ErrCfg;
    using T = Tile<C::BM, C::BN, C::WM, C::WN, C::ST, true>;
    auto kern = err_dense_kernel<C::BM, C::BN, C::WM, C::WN, C::ST, VEC, V>;
    SRLU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)T::SMEM));
    kern<<<grid, T::NT, T::SMEM, st>>>(L, ldl, UtT, ldu, perm, a, lda, m, n, (int)k, partial);
    SRLU_CHECK_LAUNCH("err_dense_kernel");
    return SRLU_OK;
}

template <bool VEC, typename V>
static int launch_err_csr(const double *L, int64_t ldl, const double *UtT, int64_t ldu,
                          const int64_t *perm, const int64_t *indptr, const int32_t *indices,
                          const V *vals, int64_t m, int64_t n, int64_t k, double *partial,
                          cudaStream_t st, unsigned grid) {
    using C = ErrCfg;
    using T = Tile<C::BM, C::BN, C::WM, C::WN, C::ST, true>;
    const size_t smem = T::SMEM + sizeof(double) * (size_t)C::BM * (C::BN + 1);
    auto kern = err_csr_kernel<C::BM, C::BN, C::WM, C::WN, C::ST, VEC, V>;
    SRLU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, T::NT, smem, st>>>(L, ldl, UtT, ldu, perm, indptr, indices, vals, m, n, (int)k,
                                    partial);
    SRLU_CHECK_LAUNCH("err_csr_kernel");
    return SRLU_OK;
}

static size_t err_layout(int64_t m, int64_t n, int64_t k, int64_t *ldu, int64_t *nparts) {
    *ldu = (k + 1) & ~int64_t(1);  // even row pitch: 16-byte copies
    *nparts = ceil_div(n, ErrCfg::BN) * ceil_div(m, ErrCfg::BM);
    return sizeof(double) * ((size_t)n * *ldu + (size_t)*nparts + 2);
}

}  // namespace dmma
}  // namespace srlu

using namespace srlu;
using namespace srlu::dmma;

extern "C" int srlu_dgemm_ex(const double *A, int64_t lda, const double *B, int64_t ldb,
                             double *C, int64_t ldc, int64_t M, int64_t N, int64_t K, int flags,
                             srlu_stream_t stream) {
    SRLU_REQUIRE(M >= 0 && N >= 0 && K >= 0 && N < (1 << 30) && K < (1 << 30), SRLU_ERR_ARG,
                 "dgemm: bad sizes");
    SRLU_REQUIRE(lda >= K && ldb >= N && ldc >= N, SRLU_ERR_ARG, "dgemm: bad leading dimension");
    if (M == 0 || N == 0) return SRLU_OK;
    const int b_lower = (flags & SRLU_GEMM_B_LOWER) ? 1 : 0;
    cudaStream_t st = (cudaStream_t)stream;
    if (K == 0) {
        SRLU_CUDA(cudaMemset2DAsync(C, ldc * sizeof(double), 0, N * sizeof(double), M, st));
        return SRLU_OK;
    }
    const bool vec = al16(A) && al16(B) && al16(C) && !(lda & 1) && !(ldb & 1) && !(ldc & 1) &&
                     !(K & 1) && !(N & 1);
    return vec ? gemm_dispatch<true>(A, lda, B, ldb, C, ldc, M, N, K, b_lower, st)
               : gemm_dispatch<false>(A, lda, B, ldb, C, ldc, M, N, K, b_lower, st);
}

extern "C" int srlu_dgemm(const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                          int64_t ldc, int64_t M, int64_t N, int64_t K, srlu_stream_t stream) {
    return srlu_dgemm_ex(A, lda, B, ldb, C, ldc, M, N, K, 0, stream);
}

extern "C" size_t srlu_lu_error_workspace(int64_t m, int64_t n, int64_t k) {
    int64_t ldu, np;
    if (m <= 0 || n <= 0 || k <= 0) return 16;
    return err_layout(m, n, k, &ldu, &np);
}

static int lu_error_common(const double *L, int64_t ldl, const double *UT, int64_t ldut,
                           const int64_t *q, int64_t m, int64_t n, int64_t k, void *ws,
                           size_t ws_bytes, cudaStream_t st, double **utt, int64_t *ldu,
                           int64_t *np, double **partial) {
    SRLU_REQUIRE(m >= 1 && n >= 1 && k >= 1 && k < (1 << 30) && ldl >= k && ldut >= k,
                 SRLU_ERR_ARG, "lu_error: bad sizes");
    const size_t need = err_layout(m, n, k, ldu, np);
    SRLU_REQUIRE(ws != nullptr && ws_bytes >= need, SRLU_ERR_WORKSPACE,
                 "lu_error: workspace %zu < %zu bytes", ws_bytes, need);
    *utt = (double *)ws;
    *partial = *utt + (size_t)n * *ldu;
    if (*ldu != k)
        SRLU_CUDA(cudaMemsetAsync(*utt, 0, sizeof(double) * (size_t)n * *ldu, st));
    scatter_rows_kernel<<<(unsigned)std::min<int64_t>(n, 148 * 64), 128, 0, st>>>(
        UT, ldut, q, *utt, *ldu, n, (int)k);
    SRLU_CHECK_LAUNCH("scatter_rows_kernel");
    return SRLU_OK;
}

extern "C" int srlu_lu_error_dense(const double *L, int64_t ldl, const double *UT, int64_t ldut,
                                   const int64_t *perm, const int64_t *q, const void *a,
                                   int dtype, int64_t m, int64_t n, int64_t lda, int64_t k,
                                   double *sq, void *ws, size_t ws_bytes, srlu_stream_t stream) {
    SRLU_REQUIRE(dtype == SRLU_F32 || dtype == SRLU_F64, SRLU_ERR_ARG, "lu_error: dtype");
    SRLU_REQUIRE(lda >= n, SRLU_ERR_ARG, "lu_error: lda < n");
    cudaStream_t st = (cudaStream_t)stream;
    double *utt, *partial;
    int64_t ldu, np;
    int rc = lu_error_common(L, ldl, UT, ldut, q, m, n, k, ws, ws_bytes, st, &utt, &ldu, &np,
                             &partial);
    if (rc) return rc;
    dim3 grid((unsigned)ceil_div(n, ErrCfg::BN), (unsigned)ceil_div(m, ErrCfg::BM));
    SRLU_REQUIRE(grid.y <= 65535u, SRLU_ERR_UNSUPPORTED, "lu_error: m too large");
    const bool vec = al16(L) && !(ldl & 1) && !(ldu & 1) && !(k & 1);
    const int64_t kk = k;
    if (dtype == SRLU_F32)
        rc = vec ? launch_err_dense<true, float>(L, ldl, utt, ldu, perm, (const float *)a, lda, m,
                                                 n, kk, partial, st, grid)
                 : launch_err_dense<false, float>(L, ldl, utt, ldu, perm, (const float *)a, lda,
                                                  m, n, kk, partial, st, grid);
    else
        rc = vec ? launch_err_dense<true, double>(L, ldl, utt, ldu, perm, (const double *)a, lda,
                                                  m, n, kk, partial, st, grid)
                 : launch_err_dense<false, double>(L, ldl, utt, ldu, perm, (const double *)a,
                                                   lda, m, n, kk, partial, st, grid);
    if (rc) return rc;
    sum_partials_kernel<<<1, 1024, 0, st>>>(partial, np, sq);
    SRLU_CHECK_LAUNCH("sum_partials_kernel");
    return SRLU_OK;
}

extern "C" int srlu_lu_error_csr(const double *L, int64_t ldl, const double *UT, int64_t ldut,
                                 const int64_t *perm, const int64_t *q, const int64_t *indptr,
                                 const int32_t *indices, const void *vals, int dtype, int64_t m,
                                 int64_t n, int64_t k, double *sq, void *ws, size_t ws_bytes,
                                 srlu_stream_t stream) {
    SRLU_REQUIRE(dtype == SRLU_F32 || dtype == SRLU_F64, SRLU_ERR_ARG, "lu_error: dtype");
    cudaStream_t st = (cudaStream_t)stream;
    double *utt, *partial;
    int64_t ldu, np;
    int rc = lu_error_common(L, ldl, UT, ldut, q, m, n, k, ws, ws_bytes, st, &utt, &ldu, &np,
                             &partial);
    if (rc) return rc;
    const unsigned grid = (unsigned)ceil_div(m, ErrCfg::BM);
    const bool vec = al16(L) && !(ldl & 1) && !(ldu & 1) && !(k & 1);
    if (dtype == SRLU_F32)
        rc = vec ? launch_err_csr<true, float>(L, ldl, utt, ldu, perm, indptr, indices,
                                               (const float *)vals, m, n, k, partial, st, grid)
                 : launch_err_csr<false, float>(L, ldl, utt, ldu, perm, indptr, indices,
                                                (const float *)vals, m, n, k, partial, st, grid);
    else
        rc = vec ? launch_err_csr<true, double>(L, ldl, utt, ldu, perm, indptr, indices,
                                                (const double *)vals, m, n, k, partial, st, grid)
                 : launch_err_csr<false, double>(L, ldl, utt, ldu, perm, indptr, indices,
                                                 (const double *)vals, m, n, k, partial, st,
                                                 grid);
    if (rc) return rc;
    sum_partials_kernel<<<1, 1024, 0, st>>>(partial, (int64_t)grid, sq);
    SRLU_CHECK_LAUNCH("sum_partials_kernel");
    return SRLU_OK;
}
