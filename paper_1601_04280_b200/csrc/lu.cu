// K2 / K5 — exact replays of the reference's pivoted LUs
//   MODE_ROW: lu_row_pivot(Y)      factor.py:49-77   (Y: m x k, tall)
//   MODE_COL: lu_col_pivot(core)   factor.py:80-109  (core: k x n, wide,
//             handled through its transpose: one "entity" per column)
//
// Both are k sequential pivot steps over M "entities" (rows of Y / columns
// of core) of k values each.  One persistent cooperative kernel, one CTA
// per SM; each CTA owns a contiguous block of entities.  Columns are
// processed in panels of b (b = k when the whole matrix fits in shared
// memory, e.g. BASELINE config 2):
//   * per step: local argmax of |w| over the CTA's active entities (ties:
//     smallest current position, like numpy argmax on the swapped array),
//     publish {|w|, position, entity, panel row} to global memory, ONE grid
//     barrier, every CTA reduces the 1-per-CTA candidates to the same
//     winner, swaps positions, and applies the step to its own entities'
//     panel columns (mul then sub, never fused: __dmul_rn/__dsub_rn, like
//     numpy's `w -= outer(l, u)`; division correctly rounded);
//   * after the panel: the b deferred rank-1 updates are applied to the
//     trailing columns of every active entity in the same order s = J..J+b-1
//     (each element sees exactly the reference's sequence of roundings),
//     with the pivot entities' trailing vectors obtained by the small
//     in-panel triangular recurrence.
// Result: P/Q and L/U bit-identical to the reference on the same input.
#include <stdlib.h>

#include "common.cuh"

namespace srlu {

enum { MODE_ROW = 0, MODE_COL = 1 };

constexpr int kLuThreads = 256;
constexpr int kLuMaxGrid = 256;
constexpr int kLuXC = 64;  // trailing columns per chunk
constexpr double kPivotRtol = 1e-14;  // factor.py:19

struct Cand {
    unsigned long long absbits;
    unsigned int pos;
    int entity;
};

struct LuParams {
    double *w;  // M x k entity-major, ld
    int64_t M;
    int k;
    int64_t ld;
    int b;    // panel width
    int bs;   // smem stride of the panel (odd)
    int rpc;  // entities per CTA
    int64_t *perm;
    double *out_main;  // ROW: L (M x k pos order); COL: UT (M x k pos order)
    int64_t ld_main;
    double *out_small;  // ROW: U (k x k) or null; COL: Lt (k x k)
    int64_t ld_small;
    unsigned *bar;
    double *partial;
    Cand *cand;       // [2][G]
    double *candrow;  // [2][G][k]
    double *piv;      // [k][k] trailing parts of pivot entities
};

__device__ inline bool better(unsigned long long a_abs, unsigned a_pos, unsigned long long b_abs,
                              unsigned b_pos) {
    return a_abs > b_abs || (a_abs == b_abs && a_pos < b_pos);
}

// block-wide argmax; returns result in all threads via smem
__device__ inline void block_best(unsigned long long &abs, unsigned &pos, int &ent,
                                  unsigned long long *s_abs, unsigned *s_pos, int *s_ent) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        unsigned long long oa = __shfl_down_sync(0xffffffffu, abs, off);
        unsigned op = __shfl_down_sync(0xffffffffu, pos, off);
        int oe = __shfl_down_sync(0xffffffffu, ent, off);
        if (better(oa, op, abs, pos)) { abs = oa; pos = op; ent = oe; }
    }
    if (lane == 0) { s_abs[warp] = abs; s_pos[warp] = pos; s_ent[warp] = ent; }
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        abs = lane < nw ? s_abs[lane] : 0ULL;
        pos = lane < nw ? s_pos[lane] : 0xFFFFFFFFu;
        ent = lane < nw ? s_ent[lane] : -1;
#pragma unroll
        for (int off = 16; off; off >>= 1) {
            unsigned long long oa = __shfl_down_sync(0xffffffffu, abs, off);
            unsigned op = __shfl_down_sync(0xffffffffu, pos, off);
            int oe = __shfl_down_sync(0xffffffffu, ent, off);
            if (better(oa, op, abs, pos)) { abs = oa; pos = op; ent = oe; }
        }
        if (lane == 0) { s_abs[0] = abs; s_pos[0] = pos; s_ent[0] = ent; }
    }
    __syncthreads();
    abs = s_abs[0]; pos = s_pos[0]; ent = s_ent[0];
    __syncthreads();
}

template <int MODE>
__global__ void __launch_bounds__(kLuThreads, 1) lu_kernel(LuParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ unsigned long long s_abs[32];
    __shared__ unsigned s_pos[32];
    __shared__ int s_ent[32];
    __shared__ double s_thresh;
    __shared__ int s_wcta;

    const int tid = threadIdx.x;
    const int G = gridDim.x;
    const int k = p.k, b = p.b, bs = p.bs, rpc = p.rpc;
    const int64_t e0 = (int64_t)blockIdx.x * rpc;
    const int ne = (int)max((int64_t)0, min((int64_t)rpc, p.M - e0));

    // smem carve-up
    double *panel = reinterpret_cast<double *>(smem_raw);          // rpc x bs
    double *PR = panel + (size_t)rpc * bs;                          // b x b
    double *u = PR + (size_t)b * b;                                 // b
    double *Ach = u + b;                                            // b x kLuXC
    int *pos = reinterpret_cast<int *>(Ach + (size_t)b * kLuXC);    // rpc
    int *pw_ent = pos + rpc;                                        // b
    unsigned bar_target = 0;

    // ---- thresh = PIVOT_RTOL * ||w||_F (deterministic two-level sum) ----
    {
        double ss = 0.0;
        for (int64_t w = tid; w < (int64_t)ne * k; w += blockDim.x) {
            int64_t e = w / k;
            int x = (int)(w % k);
            double v = p.w[(e0 + e) * p.ld + x];
            ss += v * v;
        }
        // block reduce (fixed tree order)
        __shared__ double s_red[kLuThreads];
        s_red[tid] = ss;
        __syncthreads();
        for (int off = blockDim.x >> 1; off; off >>= 1) {
            if (tid < off) s_red[tid] += s_red[tid + off];
            __syncthreads();
        }
        if (tid == 0) p.partial[blockIdx.x] = s_red[0];
        bar_target += G;
        grid_arrive_wait(p.bar, bar_target);
        if (tid == 0) {
            double tot = 0.0;
            for (int c = 0; c < G; ++c) tot += __ldcg(p.partial + c);
            s_thresh = kPivotRtol * sqrt(tot);
        }
        for (int e = tid; e < ne; e += blockDim.x) pos[e] = (int)(e0 + e);
        __syncthreads();
    }
    const double thresh = s_thresh;

    for (int J = 0; J < k; J += b) {
        const int bw = min(b, k - J);  // this panel's width
        // load panel columns [J, J+bw) of own entities
        for (int w = tid; w < ne * bw; w += blockDim.x) {
            int e = w / bw, x = w % bw;
            panel[e * bs + x] = p.w[(e0 + e) * p.ld + J + x];
        }
        __syncthreads();

        for (int ls = 0; ls < bw; ++ls) {
            const int s = J + ls;
            const int slot = s & 1;
            // 1. local candidate
            unsigned long long babs = 0ULL;
            unsigned bpos = 0xFFFFFFFFu;
            int bent = -1;
            for (int e = tid; e < ne; e += blockDim.x) {
                if (pos[e] >= s) {
                    unsigned long long a =
                        (unsigned long long)__double_as_longlong(fabs(panel[e * bs + ls]));
                    if (better(a, (unsigned)pos[e], babs, bpos)) {
                        babs = a; bpos = (unsigned)pos[e]; bent = e;
                    }
                }
            }
            block_best(babs, bpos, bent, s_abs, s_pos, s_ent);
            // 2. publish
            Cand *cs = p.cand + (size_t)slot * G;
            double *crow = p.candrow + ((size_t)slot * G + blockIdx.x) * k;
            if (tid == 0) {
                Cand c;
                c.absbits = babs;
                c.pos = bpos;
                c.entity = bent >= 0 ? (int)(e0 + bent) : -1;
                cs[blockIdx.x] = c;
            }
            if (bent >= 0)
                for (int x = tid; x < bw; x += blockDim.x) crow[x] = panel[bent * bs + x];
            // 3. one grid barrier per pivot step
            bar_target += G;
            grid_arrive_wait(p.bar, bar_target);
            // 4. global winner
            {
                unsigned long long ga = 0ULL;
                unsigned gp = 0xFFFFFFFFu;
                int gc = -1;
                for (int c = tid; c < G; c += blockDim.x) {
                    const Cand *cp = cs + c;
                    unsigned long long a = __ldcg(&cp->absbits);
                    unsigned pp = __ldcg(&cp->pos);
                    if (better(a, pp, ga, gp)) { ga = a; gp = pp; gc = c; }
                }
                block_best(ga, gp, gc, s_abs, s_pos, s_ent);
                if (tid == 0) s_wcta = gc;
                const double *wrow = p.candrow + ((size_t)slot * G + gc) * k;
                for (int x = tid; x < bw; x += blockDim.x) u[x] = __ldcg(wrow + x);
                if (tid == 0) {
                    pw_ent[ls] = __ldcg(&cs[gc].entity);
                    s_pos[1] = gp;  // winner's old position
                }
                __syncthreads();
            }
            const int went = pw_ent[ls];
            const int wpos = (int)s_pos[1];
            const double pivv = u[ls];
            const bool big = fabs(pivv) > thresh;
            if (b < k)
                for (int x = tid; x < bw; x += blockDim.x) PR[ls * b + x] = u[x];
            // 5. swap positions s <-> wpos
            for (int e = tid; e < ne; e += blockDim.x) {
                if (pos[e] == s) pos[e] = wpos;
                if (e0 + e == went) pos[e] = s;
            }
            __syncthreads();
            // 6. apply the step to own panel columns
            if (MODE == MODE_ROW) {
                for (int e = tid; e < ne; e += blockDim.x) {
                    if (pos[e] <= s) continue;
                    double *we = panel + e * bs;
                    if (big) {
                        const double l = we[ls] / pivv;
                        we[ls] = l;
                        for (int x = ls + 1; x < bw; ++x) we[x] = __dsub_rn(we[x], __dmul_rn(l, u[x]));
                    } else {
                        we[ls] = 0.0;
                    }
                }
            } else {
                // multipliers of the pivot column: L[x] = u[x] / piv
                for (int x = ls + 1 + tid; x < bw; x += blockDim.x) u[x] = big ? u[x] / pivv : 0.0;
                __syncthreads();
                for (int e = tid; e < ne; e += blockDim.x) {
                    double *we = panel + e * bs;
                    if (e0 + e == went) {
                        for (int x = ls + 1; x < bw; ++x) we[x] = u[x];
                        continue;
                    }
                    if (pos[e] <= s || !big) continue;
                    const double c = we[ls];
                    for (int x = ls + 1; x < bw; ++x) we[x] = __dsub_rn(we[x], __dmul_rn(u[x], c));
                }
                if (b < k)
                    for (int x = ls + 1 + tid; x < bw; x += blockDim.x) PR[ls * b + x] = u[x];
            }
            __syncthreads();
        }

        // write the panel back
        for (int w = tid; w < ne * bw; w += blockDim.x) {
            int e = w / bw, x = w % bw;
            p.w[(e0 + e) * p.ld + J + x] = panel[e * bs + x];
        }

        // deferred trailing update of columns [J+bw, k)
        for (int x0 = J + bw; x0 < k; x0 += kLuXC) {
            const int xc = min(kLuXC, k - x0);
            // A_s[x] for the panel's pivots (tiny triangular recurrence)
            for (int c = tid; c < xc; c += blockDim.x) {
                const int x = x0 + c;
                for (int ls = 0; ls < bw; ++ls) {
                    double v = __ldcg(p.w + (int64_t)pw_ent[ls] * p.ld + x);
                    const double *pr = PR + ls * b;
                    if (MODE == MODE_ROW) {
                        for (int l2 = 0; l2 < ls; ++l2)
                            v = __dsub_rn(v, __dmul_rn(pr[l2], Ach[l2 * kLuXC + c]));
                    } else {
                        for (int l2 = 0; l2 < ls; ++l2)
                            v = __dsub_rn(v, __dmul_rn(Ach[l2 * kLuXC + c], pr[l2]));
                        const double pv = pr[ls];
                        v = fabs(pv) > thresh ? v / pv : 0.0;
                    }
                    Ach[ls * kLuXC + c] = v;
                    if (blockIdx.x == 0) p.piv[(int64_t)(J + ls) * k + x] = v;
                }
            }
            __syncthreads();
            for (int w = tid; w < ne * xc; w += blockDim.x) {
                const int e = w / xc, c = w % xc;
                if (pos[e] < J + bw) continue;  // pivots are frozen
                double *gp = p.w + (e0 + e) * p.ld + x0 + c;
                double v = *gp;
                const double *pe = panel + e * bs;
                if (MODE == MODE_ROW) {
                    for (int ls = 0; ls < bw; ++ls)
                        v = __dsub_rn(v, __dmul_rn(pe[ls], Ach[ls * kLuXC + c]));
                } else {
                    for (int ls = 0; ls < bw; ++ls)
                        v = __dsub_rn(v, __dmul_rn(Ach[ls * kLuXC + c], pe[ls]));
                }
                *gp = v;
            }
            __syncthreads();
        }
    }

    // ---- final assembly (after everyone's write-backs and CTA 0's piv rows)
    bar_target += G;
    grid_arrive_wait(p.bar, bar_target);
    for (int w = tid; w < ne * k; w += blockDim.x) {
        const int e = w / k, x = w % k;
        const int q = pos[e];
        double v;
        if (q < k) {
            const int pend = min(k, (q / b) * b + b);
            v = x < pend ? __ldcg(p.w + (e0 + e) * p.ld + x) : __ldcg(p.piv + (int64_t)q * k + x);
        } else {
            v = p.w[(e0 + e) * p.ld + x];
        }
        if (MODE == MODE_ROW) {
            double lv = q >= k ? v : (x < q ? v : (x == q ? 1.0 : 0.0));
            p.out_main[(int64_t)q * p.ld_main + x] = lv;
            if (q < k && p.out_small) p.out_small[(int64_t)q * p.ld_small + x] = x >= q ? v : 0.0;
        } else {
            p.out_main[(int64_t)q * p.ld_main + x] = (q >= k || x <= q) ? v : 0.0;
            if (q < k) p.out_small[(int64_t)x * p.ld_small + q] = x > q ? v : (x == q ? 1.0 : 0.0);
        }
    }
    for (int e = tid; e < ne; e += blockDim.x) p.perm[pos[e]] = e0 + e;
}

static size_t lu_smem_bytes(int rpc, int b, int bs) {
    return sizeof(double) * ((size_t)rpc * bs + (size_t)b * b + b + (size_t)b * kLuXC) +
           sizeof(int) * ((size_t)rpc + b) + 16;
}

static int sm_count() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 1;
}

template <int MODE>
static int run_lu(double *w, int64_t M, int64_t k, int64_t ld, int64_t *perm, double *out_main,
                  int64_t ld_main, double *out_small, int64_t ld_small, int reserve_sms,
                  void *ws, size_t ws_bytes, cudaStream_t stream) {
    SRLU_REQUIRE(M >= 1 && k >= 1 && ld >= k, SRLU_ERR_ARG, "lu: bad sizes M=%lld k=%lld",
                 (long long)M, (long long)k);
    SRLU_REQUIRE(M < (1LL << 31) - 1 && k <= 8192, SRLU_ERR_UNSUPPORTED, "lu: sizes too large");
    SRLU_REQUIRE(ws_bytes >= srlu_lu_workspace(M, k), SRLU_ERR_WORKSPACE, "lu: workspace too small");
    SRLU_REQUIRE(reserve_sms >= 0, SRLU_ERR_ARG, "lu: reserve_sms < 0");
    int G = sm_count() - reserve_sms;
    if (G < 1) G = 1;
    if (const char *env = getenv("SRLU_LU_MAX_GRID")) {  // testing knob
        int cap = atoi(env);
        if (cap >= 1 && cap < G) G = cap;
    }
    if (G > kLuMaxGrid) G = kLuMaxGrid;
    if (G > M) G = (int)M;
    int rpc = (int)ceil_div(M, G);
    G = (int)ceil_div(M, rpc);
    // widest panel that fits the shared-memory budget
    const size_t budget = 200 * 1024;
    int b = (int)k;
    while (b > 1 && lu_smem_bytes(rpc, b, b | 1) > budget) --b;
    int bs = b | 1;
    size_t smem = lu_smem_bytes(rpc, b, bs);
    SRLU_REQUIRE(smem <= budget, SRLU_ERR_UNSUPPORTED,
                 "lu: %lld entities per CTA do not fit in shared memory", (long long)rpc);
    auto kern = lu_kernel<MODE>;
    SRLU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    SRLU_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kLuThreads, smem));
    SRLU_REQUIRE(per_sm >= 1, SRLU_ERR_UNSUPPORTED, "lu: kernel cannot be resident");

    char *wsb = (char *)ws;
    LuParams prm;
    prm.w = w; prm.M = M; prm.k = (int)k; prm.ld = ld; prm.b = b; prm.bs = bs; prm.rpc = rpc;
    prm.perm = perm; prm.out_main = out_main; prm.ld_main = ld_main;
    prm.out_small = out_small; prm.ld_small = ld_small;
    prm.bar = (unsigned *)wsb;
    prm.partial = (double *)(wsb + 256);
    prm.cand = (Cand *)(wsb + 256 + sizeof(double) * kLuMaxGrid);
    prm.candrow = (double *)((char *)prm.cand + sizeof(Cand) * 2 * kLuMaxGrid);
    prm.piv = prm.candrow + (size_t)2 * kLuMaxGrid * k;
    SRLU_CUDA(cudaMemsetAsync(prm.bar, 0, 256, stream));
    void *args[] = {&prm};
    SRLU_CUDA(cudaLaunchCooperativeKernel((const void *)kern, dim3(G), dim3(kLuThreads), args, smem,
                                          stream));
    return SRLU_OK;
}

}  // namespace srlu

using namespace srlu;

extern "C" size_t srlu_lu_workspace(int64_t M, int64_t k) {
    (void)M;
    return 256 + sizeof(double) * kLuMaxGrid + sizeof(Cand) * 2 * kLuMaxGrid +
           sizeof(double) * ((size_t)2 * kLuMaxGrid * k + (size_t)k * k) + 256;
}

extern "C" int srlu_lu_rowpiv(double *y, int64_t m, int64_t k, int64_t ldy, int64_t *perm,
                              double *L, int64_t ldl, double *U, int64_t ldu, int reserve_sms,
                              void *ws, size_t ws_bytes, srlu_stream_t stream) {
    SRLU_REQUIRE(m >= k, SRLU_ERR_ARG, "lu_row_pivot: need rows >= cols, got %lld x %lld",
                 (long long)m, (long long)k);
    SRLU_REQUIRE(ldl >= k && (U == nullptr || ldu >= k), SRLU_ERR_ARG, "lu_row_pivot: bad ld");
    return run_lu<MODE_ROW>(y, m, k, ldy, perm, L, ldl, U, ldu, reserve_sms, ws, ws_bytes,
                            (cudaStream_t)stream);
}

extern "C" int srlu_lu_colpiv(double *ct, int64_t n, int64_t k, int64_t ldc, int64_t *q,
                              double *Lt, int64_t ldlt, double *UT, int64_t ldut, int reserve_sms,
                              void *ws, size_t ws_bytes, srlu_stream_t stream) {
    SRLU_REQUIRE(k <= n, SRLU_ERR_ARG, "lu_col_pivot: need rows <= cols, got %lld x %lld",
                 (long long)k, (long long)n);
    SRLU_REQUIRE(Lt != nullptr && ldlt >= k && ldut >= k, SRLU_ERR_ARG, "lu_col_pivot: bad ld");
    return run_lu<MODE_COL>(ct, n, k, ldc, q, UT, ldut, Lt, ldlt, reserve_sms, ws, ws_bytes,
                            (cudaStream_t)stream);
}
