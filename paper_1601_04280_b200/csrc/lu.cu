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
#include <cooperative_groups.h>
#include <mutex>
#include <stdlib.h>

#include "common.cuh"
#include "tma.cuh"

namespace cg = cooperative_groups;

#ifdef SRLU_LU_TRACE
__device__ long long g_lu_trace[8];
#define LU_T0() long long t_prev_ = clock64(), t_acc_[8] = {0, 0, 0, 0, 0, 0, 0, 0}
#define LU_T(i)                                                  \
    do {                                                         \
        long long t_ = clock64();                                \
        t_acc_[i] += t_ - t_prev_;                               \
        t_prev_ = t_;                                            \
    } while (0)
#define LU_TDUMP()                                                            \
    do {                                                                      \
        if (threadIdx.x == 0 && blockIdx.x == 0)                              \
            for (int i_ = 0; i_ < 8; ++i_) g_lu_trace[i_] = t_acc_[i_];       \
    } while (0)
#else
#define LU_T0() do { } while (0)
#define LU_T(i) do { } while (0)
#define LU_TDUMP() do { } while (0)
#endif

namespace srlu {

enum { MODE_ROW = 0, MODE_COL = 1 };

constexpr int kLuThreads = 512;
static_assert(kLuThreads >= 8 * 64, "grid LU: the blocked recurrence uses 8 groups of kLuXC threads");
constexpr int kLuRPW = 4;  // trailing update: rows per warp pass
#ifndef SRLU_LU_PFD
#define SRLU_LU_PFD 1  // trailing update: passes of loads in flight (2 measured: no gain)
#endif
#ifndef SRLU_LU_RPW
#define SRLU_LU_RPW 4  // smem-panel kernel: rows per warp pass (8 measured slower)
#endif
constexpr int kLuMaxGrid = 256;
constexpr int kLuXC = 64;  // trailing columns per chunk
constexpr int kLuB2Max = 32;  // outer block: its multipliers are broadcast by warp shuffles
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
    double *gpanel;   // GB > 0: attribute-major panel [GB][ldp] (L2-resident)
    int64_t ldp;
    int l2pf;         // trailing update: L2 prefetch distance in warp passes (0 = off)
    int b2;           // outer block width (multiple of b, <= kLuB2Max; 0 = one level)
    int la;           // priority-column look-ahead in the pivot steps (shared-memory panel)
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

// GB > 0: "L2 panel" variant for tall inputs whose smem panel would be
// narrow (BASELINE config 4: 7085 entities per CTA leave room for 3 columns):
// the panel lives in an attribute-major workspace [GB][M] (64 MB at M = 1M:
// L2-resident, every column access coalesced across threads), with GB-wide
// register rows and several entities' loads in flight per thread.
// Two-level trailing update (lu_outer_width): the nb2 = x_hi - Jo pivots of the
// outer block [Jo, x_hi) applied to the columns [x_hi, k) of this CTA's live
// rows.  Kept out of line so that its registers do not weigh on the kernel's
// per-step loops.
template <int MODE>
__device__ __noinline__ void lu_outer_update(const LuParams &p, double *PRo, double *Acho,
                                             const double *PR, const int *pwo, const int *pos,
                                             int J, int Jo, int x_hi, int ne, int64_t e0,
                                             double thresh) {
    const int tid = threadIdx.x;
    const int k = p.k, b = p.b;
        const int nb2 = x_hi - Jo;   // pivots of the outer block
        const int jl = J - Jo;       // first one of the last inner panel
        // PRo(ls, l2 <= ls): pivot row ls's panel values at the earlier
        // pivots' columns (ROW: its multipliers; COL: its own values, the
        // pivot on the diagonal).  The last inner panel's are still in PR
        // (its write-back may not be visible to other CTAs yet); the others
        // were written back before at least one grid barrier.
        for (int w = tid; w < nb2 * nb2; w += blockDim.x) {
            const int ls = w / nb2, l2 = w - ls * nb2;
            if (l2 > ls) continue;
            PRo[ls * kLuB2Max + l2] =
                (ls >= jl && l2 >= jl) ? PR[(ls - jl) * b + (l2 - jl)]
                                       : __ldcg(p.w + (int64_t)pwo[ls] * p.ld + Jo + l2);
        }
        __syncthreads();
        for (int x0 = x_hi; x0 < k; x0 += kLuXC) {
            const int xc = min(kLuXC, k - x0);
            for (int w = tid; w < nb2 * xc; w += blockDim.x) {
                const int ls = w / xc, c = w - ls * xc;
                Acho[ls * kLuXC + c] = __ldcg(p.w + (int64_t)pwo[ls] * p.ld + x0 + c);
            }
            __syncthreads();
            {   // the pivot rows' values: the same blocked recurrence over nb2 pivots
                constexpr int KB = 8;
                const int c = tid % kLuXC, g = tid / kLuXC;
                for (int s0 = 0; s0 < nb2; s0 += KB) {
                    const int ls = s0 + g;
                    if (s0 > 0 && g < KB && ls < nb2 && c < xc) {
                        double v = Acho[ls * kLuXC + c];
                        const double *pr = PRo + ls * kLuB2Max;
                        for (int l2 = 0; l2 < s0; ++l2)
                            v = MODE == MODE_ROW
                                    ? __dsub_rn(v, __dmul_rn(pr[l2], Acho[l2 * kLuXC + c]))
                                    : __dsub_rn(v, __dmul_rn(Acho[l2 * kLuXC + c], pr[l2]));
                        Acho[ls * kLuXC + c] = v;
                    }
                    __syncthreads();
                    if (g == 0 && c < xc) {
                        const int nb = min(KB, nb2 - s0);
                        double a[KB];
#pragma unroll
                        for (int i = 0; i < KB; ++i)
                            a[i] = i < nb ? Acho[(s0 + i) * kLuXC + c] : 0.0;
#pragma unroll
                        for (int i = 0; i < KB; ++i) {
                            if (i < nb) {
                                double v = a[i];
                                const double *pr = PRo + (s0 + i) * kLuB2Max + s0;
#pragma unroll
                                for (int j = 0; j < i; ++j)
                                    v = MODE == MODE_ROW ? __dsub_rn(v, __dmul_rn(pr[j], a[j]))
                                                         : __dsub_rn(v, __dmul_rn(a[j], pr[j]));
                                if (MODE != MODE_ROW) {
                                    const double pv = pr[i];
                                    v = fabs(pv) > thresh ? v / pv : 0.0;
                                }
                                a[i] = v;
                            }
                        }
#pragma unroll
                        for (int i = 0; i < KB; ++i) {
                            if (i < nb) {
                                Acho[(s0 + i) * kLuXC + c] = a[i];
                                if (blockIdx.x == 0)
                                    p.piv[(int64_t)(Jo + s0 + i) * k + x0 + c] = a[i];
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            
            {   // rows: RPW per warp pass, the row's nb2 multipliers (its
                // columns [Jo, x_hi), one coalesced load) held across the
                // lanes and broadcast by shuffles
                constexpr int RPW = kLuRPW;
                const int lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
                const bool c0ok = lane < xc, c1ok = lane + 32 < xc;
                const int a1i = lane + 32 < kLuXC ? lane + 32 : lane;
                const int stride = nwarp * RPW;
                double vn[RPW][2], pmn[RPW];
                bool ln[RPW];
                auto fetch = [&](int eb) {
#pragma unroll
                    for (int r = 0; r < RPW; ++r) {
                        const int e = eb + r;
                        ln[r] = e < ne && pos[e] >= x_hi;  // this block's pivots are frozen
                        const double *gr = p.w + (e0 + e) * p.ld;
                        vn[r][0] = ln[r] && c0ok ? gr[x0 + lane] : 0.0;
                        vn[r][1] = ln[r] && c1ok ? gr[x0 + lane + 32] : 0.0;
                        pmn[r] = ln[r] && lane < nb2 ? gr[Jo + lane] : 0.0;
                    }
                };
                const int l2pf = p.l2pf;
                auto prefetch = [&](int ebp) {
                    if (lane < RPW) {
                        const int e = ebp + lane;
                        if (e < ne && pos[e] >= x_hi) {
                            const uintptr_t a0 = (uintptr_t)(p.w + (e0 + e) * p.ld + x0);
                            const uintptr_t lo = a0 & ~(uintptr_t)15;
                            const uintptr_t hi = (a0 + (uintptr_t)xc * 8 + 15) & ~(uintptr_t)15;
                            bulk_prefetch_l2((const void *)lo, (unsigned)(hi - lo));
                        }
                    }
                };
                int eb = warp * RPW;
                if (l2pf > 0)
                    for (int d = 1; d <= l2pf; ++d) prefetch(eb + d * stride);
                if (eb < ne) fetch(eb);
                for (; eb < ne; eb += stride) {
                    if (l2pf > 0) prefetch(eb + (l2pf + 1) * stride);
                    double v[RPW][2], pm[RPW];
                    bool live[RPW];
#pragma unroll
                    for (int r = 0; r < RPW; ++r) {
                        v[r][0] = vn[r][0];
                        v[r][1] = vn[r][1];
                        live[r] = ln[r];
                        pm[r] = pmn[r];
                    }
                    if (eb + stride < ne) fetch(eb + stride);
                    for (int ls = 0; ls < nb2; ++ls) {
                        const double a0 = Acho[ls * kLuXC + lane];
                        const double a1 = Acho[ls * kLuXC + a1i];
#pragma unroll
                        for (int r = 0; r < RPW; ++r) {
                            const double pv = __shfl_sync(0xffffffffu, pm[r], ls);
                            if (MODE == MODE_ROW) {
                                v[r][0] = __dsub_rn(v[r][0], __dmul_rn(pv, a0));
                                v[r][1] = __dsub_rn(v[r][1], __dmul_rn(pv, a1));
                            } else {
                                v[r][0] = __dsub_rn(v[r][0], __dmul_rn(a0, pv));
                                v[r][1] = __dsub_rn(v[r][1], __dmul_rn(a1, pv));
                            }
                        }
                    }
#pragma unroll
                    for (int r = 0; r < RPW; ++r) {
                        if (!live[r]) continue;
                        double *gp = p.w + (e0 + eb + r) * p.ld + x0 + lane;
                        if (c0ok) gp[0] = v[r][0];
                        if (c1ok) gp[32] = v[r][1];
                    }
                }
            }
            __syncthreads();
            
        }

}

template <int MODE, int GB = 0, bool TWO = false>
__global__ void __launch_bounds__(kLuThreads, 1) lu_kernel(LuParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ unsigned long long s_abs[32];
    __shared__ unsigned s_pos[32];
    __shared__ int s_ent[32];
    __shared__ double s_thresh;
    __shared__ int s_wcta;

    const int tid = threadIdx.x;
    const int G = gridDim.x;
    const int k = p.k, b = p.b, rpc = p.rpc;
    const int bs = p.bs;
    const int64_t es = GB ? 1 : bs, xs = GB ? p.ldp : 1;  // panel[e * es + x * xs]
    const int64_t e0 = (int64_t)blockIdx.x * rpc;
    const int ne = (int)max((int64_t)0, min((int64_t)rpc, p.M - e0));

    // smem carve-up
    double *const spanel = reinterpret_cast<double *>(smem_raw);   // rpc x bs (GB == 0)
    double *PR = spanel + (GB ? 0 : (size_t)rpc * bs);              // b x b
    double *u = PR + (size_t)b * b;                                 // b
    double *u2 = u + b;                                             // b (look-ahead: the previous step's pivot row)
    double *Ach = u2 + b;                                           // b x kLuXC
    const int b2 = TWO ? p.b2 : 0;
    double *PRo = Ach + (size_t)b * kLuXC;                          // b2 x kLuB2Max
    double *Acho = PRo + (size_t)b2 * kLuB2Max;                     // b2 x kLuXC
    int *pos = reinterpret_cast<int *>(Acho + (size_t)b2 * kLuXC);  // rpc
    int *pw_ent = pos + rpc;                                        // b
    int *pwo = pw_ent + b;                                          // b2: pivots of the outer block
    unsigned bar_target = 0;
    // Priority-column look-ahead (shared-memory panel only): step ls updates
    // only the next pivot column before the candidates of step ls+1 are
    // published; the rest of its update (columns > ls+1) runs between the
    // arrival at the grid barrier of step ls+1 and the wait on it.  The
    // published candidate row gets that pending update on the fly, so every
    // value is produced by the same operations in the same order.
    // (the L2-panel variant, GB > 0, keeps the plain order: extending the
    // look-ahead to it cost registers — spills at the 128 cap — and measured
    // 9.19 vs 9.02 ms at config 4, against 8.74 ms without the extra code)
    const bool la = !GB && p.la != 0;
    LU_T0();

    // ---- thresh = PIVOT_RTOL * ||w||_F (deterministic two-level sum) ----
    {
        double ss = 0.0;
        if (p.ld == k) {  // contiguous rows: flat, four independent sums in flight
            const double *base = p.w + e0 * p.ld;
            const int64_t nel = (int64_t)ne * k;
            double s4[4] = {0.0, 0.0, 0.0, 0.0};
            int64_t w = tid;
            for (; w + 3 * kLuThreads < nel; w += 4 * kLuThreads) {
                double v4[4];
#pragma unroll
                for (int u4 = 0; u4 < 4; ++u4) v4[u4] = __ldcs(base + w + u4 * kLuThreads);
#pragma unroll
                for (int u4 = 0; u4 < 4; ++u4) s4[u4] += v4[u4] * v4[u4];
            }
            for (; w < nel; w += kLuThreads) s4[0] += base[w] * base[w];
            ss = (s4[0] + s4[1]) + (s4[2] + s4[3]);
        } else {
            for (int64_t w = tid; w < (int64_t)ne * k; w += blockDim.x) {
                int64_t e = w / k;
                int x = (int)(w % k);
                double v = p.w[(e0 + e) * p.ld + x];
                ss += v * v;
            }
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
        double *const panel = GB ? p.gpanel + e0 : spanel;
        LU_T(7);
        // load panel columns [J, J+bw) of own entities: lanes over (row,
        // column) pairs, 4 row groups of loads in flight per warp
        {
            const int lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
            const int bwl = bw < 32 ? bw : 32;
            const int rpl = 32 / bwl, r = lane / bwl, xl = lane - r * bwl;
            const int step = nwarp * rpl;
            for (int xb = 0; xb < bw; xb += bwl) {
                const int x = xb + xl;
                const bool xok = r < rpl && x < bw;
                for (int eb = warp * rpl; eb < ne; eb += 4 * step) {
                    double v[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int e = eb + u * step + r;
                        v[u] = xok && e < ne ? p.w[(e0 + e) * p.ld + J + x] : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int e = eb + u * step + r;
                        if (xok && e < ne) panel[e * es + x * xs] = v[u];
                    }
                }
            }
        }
        __syncthreads();
        LU_T(3);

        bool pend_big = false;  // look-ahead: step ls-1 still owes columns > ls
        for (int ls = 0; ls < bw; ++ls) {
            const int s = J + ls;
            const int slot = s & 1;
            double *const uc = (la && (ls & 1)) ? u2 : u;     // this step's pivot row
            const double *const up = (ls & 1) ? u : u2;       // the previous step's (look-ahead)
            // 1. local candidate
            unsigned long long babs = 0ULL;
            unsigned bpos = 0xFFFFFFFFu;
            int bent = -1;
            if (GB) {  // four entities' loads in flight per thread
                for (int eb = tid; eb < ne; eb += 4 * kLuThreads) {
                    double v[4];
                    int ps[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int e = eb + r * kLuThreads;
                        ps[r] = e < ne ? pos[e] : -1;
                        v[r] = ps[r] >= s ? panel[(int64_t)e * es + ls * xs] : 0.0;
                    }
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const unsigned long long a =
                            (unsigned long long)__double_as_longlong(fabs(v[r]));
                        if (ps[r] >= s && better(a, (unsigned)ps[r], babs, bpos)) {
                            babs = a; bpos = (unsigned)ps[r]; bent = eb + r * kLuThreads;
                        }
                    }
                }
            } else {
                for (int e = tid; e < ne; e += blockDim.x) {
                    if (pos[e] >= s) {
                        unsigned long long a =
                            (unsigned long long)__double_as_longlong(fabs(panel[e * bs + ls]));
                        if (better(a, (unsigned)pos[e], babs, bpos)) {
                            babs = a; bpos = (unsigned)pos[e]; bent = e;
                        }
                    }
                }
            }
            block_best(babs, bpos, bent, s_abs, s_pos, s_ent);
            LU_T(0);
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
                for (int x = tid; x < bw; x += blockDim.x) {
                    double v = panel[bent * es + x * xs];
                    if (la && pend_big && x > ls) {  // the pending update of step ls-1, on the fly
                        const double c = panel[bent * es + (ls - 1) * xs];
                        v = MODE == MODE_ROW ? __dsub_rn(v, __dmul_rn(c, up[x]))
                                             : __dsub_rn(v, __dmul_rn(up[x], c));
                    }
                    crow[x] = v;
                }
            // 3. one grid barrier per pivot step
            bar_target += G;
            if (la) {
                grid_arrive(p.bar);
                if (pend_big) {  // step ls-1 on the columns > ls of the rows live at that step
                    for (int e = tid; e < ne; e += blockDim.x) {
                        if (pos[e] < s) continue;
                        double *we = panel + e * bs;
                        const double c = we[ls - 1];
                        for (int x = ls + 1; x < bw; ++x)
                            we[x] = MODE == MODE_ROW ? __dsub_rn(we[x], __dmul_rn(c, up[x]))
                                                     : __dsub_rn(we[x], __dmul_rn(up[x], c));
                    }
                }
                grid_wait(p.bar, bar_target);
            } else {
                grid_arrive_wait(p.bar, bar_target);
            }
            LU_T(1);
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
                for (int x = tid; x < bw; x += blockDim.x) uc[x] = __ldcg(wrow + x);
                if (tid == 0) {
                    pw_ent[ls] = __ldcg(&cs[gc].entity);
                    if (b2) pwo[s % b2] = pw_ent[ls];
                    s_pos[1] = gp;  // winner's old position
                }
                __syncthreads();
            }
            LU_T(2);
            const int went = pw_ent[ls];
            const int wpos = (int)s_pos[1];
            const double pivv = uc[ls];
            const bool big = fabs(pivv) > thresh;
            if (b < k)
                for (int x = tid; x < bw; x += blockDim.x) PR[ls * b + x] = uc[x];
            // 5. swap positions s <-> wpos
            for (int e = tid; e < ne; e += blockDim.x) {
                if (pos[e] == s) pos[e] = wpos;
                if (e0 + e == went) pos[e] = s;
            }
            __syncthreads();
            // 6. apply the step to own panel columns
            constexpr int RA = GB <= 8 ? 4 : 2;  // entities in flight (GB > 0)
            if (GB && MODE == MODE_ROW) {
                for (int eb = tid; eb < ne; eb += RA * kLuThreads) {
                    double v[RA][GB > 0 ? GB : 1], lv[RA];
                    bool act[RA];
#pragma unroll
                    for (int r = 0; r < RA; ++r) {
                        const int e = eb + r * kLuThreads;
                        act[r] = e < ne && pos[e] > s;
                        const double *we = panel + (int64_t)e * es;
                        lv[r] = act[r] ? we[ls * xs] : 0.0;
#pragma unroll
                        for (int x = 0; x < GB; ++x)
                            v[r][x] = (act[r] && big && x > ls && x < bw) ? we[x * xs] : 0.0;
                    }
#pragma unroll
                    for (int r = 0; r < RA; ++r) {
                        if (!act[r]) continue;
                        double *we = panel + (int64_t)(eb + r * kLuThreads) * es;
                        if (big) {
                            const double l = lv[r] / pivv;
                            we[ls * xs] = l;
#pragma unroll
                            for (int x = 0; x < GB; ++x)
                                if (x > ls && x < bw) we[x * xs] = __dsub_rn(v[r][x], __dmul_rn(l, uc[x]));
                        } else {
                            we[ls * xs] = 0.0;
                        }
                    }
                }
            } else if (GB) {
                // multipliers of the pivot column: L[x] = u[x] / piv
                for (int x = ls + 1 + tid; x < bw; x += blockDim.x) uc[x] = big ? uc[x] / pivv : 0.0;
                __syncthreads();
                for (int eb = tid; eb < ne; eb += RA * kLuThreads) {
                    double v[RA][GB > 0 ? GB : 1], cv[RA];
                    bool act[RA], isw[RA];
#pragma unroll
                    for (int r = 0; r < RA; ++r) {
                        const int e = eb + r * kLuThreads;
                        isw[r] = e < ne && e0 + e == went;
                        act[r] = e < ne && !isw[r] && big && pos[e] > s;
                        const double *we = panel + (int64_t)e * es;
                        cv[r] = act[r] ? we[ls * xs] : 0.0;
#pragma unroll
                        for (int x = 0; x < GB; ++x)
                            v[r][x] = (act[r] && x > ls && x < bw) ? we[x * xs] : 0.0;
                    }
#pragma unroll
                    for (int r = 0; r < RA; ++r) {
                        double *we = panel + (int64_t)(eb + r * kLuThreads) * es;
                        if (isw[r]) {
#pragma unroll
                            for (int x = 0; x < GB; ++x)
                                if (x > ls && x < bw) we[x * xs] = uc[x];
                        } else if (act[r]) {
#pragma unroll
                            for (int x = 0; x < GB; ++x)
                                if (x > ls && x < bw) we[x * xs] = __dsub_rn(v[r][x], __dmul_rn(uc[x], cv[r]));
                        }
                    }
                }
                if (b < k)
                    for (int x = ls + 1 + tid; x < bw; x += blockDim.x) PR[ls * b + x] = uc[x];
            } else if (MODE == MODE_ROW) {
                const int xend = la ? min(bw, ls + 2) : bw;   // look-ahead: the next pivot column only
                for (int e = tid; e < ne; e += blockDim.x) {
                    if (pos[e] <= s) continue;
                    double *we = panel + e * bs;
                    if (big) {
                        const double l = we[ls] / pivv;
                        we[ls] = l;
                        for (int x = ls + 1; x < xend; ++x) we[x] = __dsub_rn(we[x], __dmul_rn(l, uc[x]));
                    } else {
                        we[ls] = 0.0;
                    }
                }
                pend_big = la && big;
            } else {
                // multipliers of the pivot column: L[x] = u[x] / piv
                for (int x = ls + 1 + tid; x < bw; x += blockDim.x) uc[x] = big ? uc[x] / pivv : 0.0;
                __syncthreads();
                for (int e = tid; e < ne; e += blockDim.x) {
                    double *we = panel + e * bs;
                    if (e0 + e == went) {
                        for (int x = ls + 1; x < bw; ++x) we[x] = uc[x];
                        continue;
                    }
                    if (pos[e] <= s || !big) continue;
                    const double c = we[ls];
                    const int xend = la ? min(bw, ls + 2) : bw;
                    for (int x = ls + 1; x < xend; ++x) we[x] = __dsub_rn(we[x], __dmul_rn(uc[x], c));
                }
                pend_big = la && big;
                if (b < k)
                    for (int x = ls + 1 + tid; x < bw; x += blockDim.x) PR[ls * b + x] = uc[x];
            }
            __syncthreads();
            LU_T(6);
        }

        // write the panel back
        {
            const int lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
            const int bwl = bw < 32 ? bw : 32;
            const int rpl = 32 / bwl, r = lane / bwl, xl = lane - r * bwl;
            for (int xb = 0; xb < bw; xb += bwl) {
                const int x = xb + xl;
                if (r >= rpl || x >= bw) continue;
                for (int e = warp * rpl + r; e < ne; e += nwarp * rpl)
                    p.w[(e0 + e) * p.ld + J + x] = panel[e * es + x * xs];
            }
        }

        // deferred trailing update of columns [J+bw, x_hi): all of them, or
        // (two-level blocking, b2 > 0) only the rest of the outer block
        // [Jo, Jo + b2) — those columns of all rows stay L2-resident — while
        // the columns beyond it are updated once per outer block below with
        // all of its b2 pivots (b2 / b times fewer passes over the trailing
        // matrix in HBM; every element still receives its updates in
        // ascending pivot order with the same operands: bit-identical)
        const int Jo = b2 ? (J / b2) * b2 : 0;
        const int x_hi = b2 ? min(k, Jo + b2) : k;
        for (int x0 = J + bw; x0 < x_hi; x0 += kLuXC) {
            const int xc = min(kLuXC, x_hi - x0);
            // A_s[x] for the panel's pivots (tiny triangular recurrence); the
            // pivot rows' values are first staged (all loads in flight)
            for (int w = tid; w < bw * xc; w += blockDim.x) {
                const int ls = w / xc, c = w - ls * xc;
                Ach[ls * kLuXC + c] = __ldcg(p.w + (int64_t)pw_ent[ls] * p.ld + x0 + c);
            }
            __syncthreads();
            // The pivot rows' values on these columns: the triangular
            // recurrence v(ls) = A(ls) - sum_{l2 < ls} PR(ls, l2) v(l2), each
            // chain in the reference's l2 order, blocked by 8 rows: the terms
            // l2 < s of the 8 chains of block [s, s+8) run in parallel (one
            // thread group per chain, 64 columns each), the in-block terms in
            // registers by one thread per column.  Wide panels (config 5:
            // ~50 rows) no longer run 50^2/2 dependent steps per column.
            {
                constexpr int KB = 8;
                const int c = tid % kLuXC, g = tid / kLuXC;
                for (int s0 = 0; s0 < bw; s0 += KB) {
                    const int ls = s0 + g;
                    if (s0 > 0 && g < KB && ls < bw && c < xc) {
                        double v = Ach[ls * kLuXC + c];
                        const double *pr = PR + ls * b;
                        for (int l2 = 0; l2 < s0; ++l2)
                            v = MODE == MODE_ROW ? __dsub_rn(v, __dmul_rn(pr[l2], Ach[l2 * kLuXC + c]))
                                                 : __dsub_rn(v, __dmul_rn(Ach[l2 * kLuXC + c], pr[l2]));
                        Ach[ls * kLuXC + c] = v;
                    }
                    __syncthreads();
                    if (g == 0 && c < xc) {
                        const int nb = min(KB, bw - s0);
                        double a[KB];
#pragma unroll
                        for (int i = 0; i < KB; ++i) a[i] = i < nb ? Ach[(s0 + i) * kLuXC + c] : 0.0;
#pragma unroll
                        for (int i = 0; i < KB; ++i) {
                            if (i < nb) {
                                double v = a[i];
                                const double *pr = PR + (s0 + i) * b + s0;
#pragma unroll
                                for (int j = 0; j < i; ++j)
                                    v = MODE == MODE_ROW ? __dsub_rn(v, __dmul_rn(pr[j], a[j]))
                                                         : __dsub_rn(v, __dmul_rn(a[j], pr[j]));
                                if (MODE != MODE_ROW) {
                                    const double pv = pr[i];
                                    v = fabs(pv) > thresh ? v / pv : 0.0;
                                }
                                a[i] = v;
                            }
                        }
#pragma unroll
                        for (int i = 0; i < KB; ++i) {
                            if (i < nb) {
                                Ach[(s0 + i) * kLuXC + c] = a[i];
                                if (blockIdx.x == 0) p.piv[(int64_t)(J + s0 + i) * k + x0 + c] = a[i];
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            LU_T(4);  // trace: staging + pivot-row recurrence of this chunk
            // rows by warp (RPW per pass), columns by lane (up to two per
            // lane): coalesced, division-free; the next pass's loads are
            // issued before this pass's arithmetic (software pipeline)
            {
                constexpr int RPW = GB ? kLuRPW : SRLU_LU_RPW;  // 8 with the L2 panel: spills
                const int lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
                const bool c0ok = lane < xc, c1ok = lane + 32 < xc;
                const int a1i = lane + 32 < kLuXC ? lane + 32 : lane;
                const int stride = nwarp * RPW;
                // SRLU_LU_PFD passes of loads in flight ahead of the arithmetic
                double vn[RPW][2], vn2[RPW][2];
                double pmn[RPW], pmn2[RPW];  // GB: lane x holds multiplier x of row r
                bool ln[RPW], ln2[RPW];
                auto fetch = [&](int eb, double (&dv)[RPW][2], double (&dpm)[RPW], bool (&dl)[RPW]) {
#pragma unroll
                    for (int r = 0; r < RPW; ++r) {
                        const int e = eb + r;
                        dl[r] = e < ne && pos[e] >= J + bw;  // pivots are frozen
                        const double *gp = p.w + (e0 + e) * p.ld + x0 + lane;
                        dv[r][0] = dl[r] && c0ok ? gp[0] : 0.0;
                        dv[r][1] = dl[r] && c1ok ? gp[32] : 0.0;
                        dpm[r] = GB && dl[r] && lane < bw ? panel[(int64_t)e * es + lane * xs] : 0.0;
                    }
                };
                int eb = warp * RPW;
                // L2 prefetch distance (warp passes): the rows' loads hit L2
                // instead of HBM without holding registers (testing knob
                // SRLU_LU_L2PF, 0 = off)
                const int l2pf = GB ? 0 : p.l2pf;  // measured: helps the smem panel only
                auto prefetch = [&](int ebp) {
                    if (lane < RPW) {
                        const int e = ebp + lane;
                        if (e < ne && pos[e] >= J + bw) {
                            const uintptr_t a0 = (uintptr_t)(p.w + (e0 + e) * p.ld + x0);
                            const uintptr_t lo = a0 & ~(uintptr_t)15;
                            const uintptr_t hi = (a0 + (uintptr_t)xc * 8 + 15) & ~(uintptr_t)15;
                            bulk_prefetch_l2((const void *)lo, (unsigned)(hi - lo));
                        }
                    }
                };
                if (l2pf > 0)
                    for (int d = 1; d <= l2pf; ++d) prefetch(eb + d * stride);
                if (eb < ne) fetch(eb, vn, pmn, ln);
                if (SRLU_LU_PFD > 1 && eb + stride < ne) fetch(eb + stride, vn2, pmn2, ln2);
                for (; eb < ne; eb += stride) {
                    if (l2pf > 0) prefetch(eb + (l2pf + 1) * stride);
                    double v[RPW][2];
                    double pm[RPW];
                    bool live[RPW];
#pragma unroll
                    for (int r = 0; r < RPW; ++r) {
                        v[r][0] = vn[r][0];
                        v[r][1] = vn[r][1];
                        live[r] = ln[r];
                        pm[r] = pmn[r];
                    }
                    if (SRLU_LU_PFD > 1) {
#pragma unroll
                        for (int r = 0; r < RPW; ++r) {
                            vn[r][0] = vn2[r][0];
                            vn[r][1] = vn2[r][1];
                            ln[r] = ln2[r];
                            pmn[r] = pmn2[r];
                        }
                        if (eb + 2 * stride < ne) fetch(eb + 2 * stride, vn2, pmn2, ln2);
                    } else if (eb + stride < ne) {
                        fetch(eb + stride, vn, pmn, ln);
                    }
                    if (GB) {  // all lanes shuffle (stores below are gated by live)
#pragma unroll
                        for (int ls = 0; ls < (GB > 0 ? GB : 1); ++ls) {
                            if (ls >= bw) break;
                            const double a0 = Ach[ls * kLuXC + lane];
                            const double a1 = Ach[ls * kLuXC + a1i];
#pragma unroll
                            for (int r = 0; r < RPW; ++r) {
                                const double pv = __shfl_sync(0xffffffffu, pm[r], ls);
                                if (MODE == MODE_ROW) {
                                    v[r][0] = __dsub_rn(v[r][0], __dmul_rn(pv, a0));
                                    v[r][1] = __dsub_rn(v[r][1], __dmul_rn(pv, a1));
                                } else {
                                    v[r][0] = __dsub_rn(v[r][0], __dmul_rn(a0, pv));
                                    v[r][1] = __dsub_rn(v[r][1], __dmul_rn(a1, pv));
                                }
                            }
                        }
                    }
                    if (!GB) {  // steps outer, rows inner: one Ach load per step
                        const double *pe = panel + eb * bs;
                        for (int ls = 0; ls < bw; ++ls) {
                            const double a0 = Ach[ls * kLuXC + lane];
                            const double a1 = Ach[ls * kLuXC + a1i];
#pragma unroll
                            for (int r = 0; r < RPW; ++r) {
                                const double pv = pe[r * bs + ls];  // dead rows: unused
                                if (MODE == MODE_ROW) {
                                    v[r][0] = __dsub_rn(v[r][0], __dmul_rn(pv, a0));
                                    v[r][1] = __dsub_rn(v[r][1], __dmul_rn(pv, a1));
                                } else {
                                    v[r][0] = __dsub_rn(v[r][0], __dmul_rn(a0, pv));
                                    v[r][1] = __dsub_rn(v[r][1], __dmul_rn(a1, pv));
                                }
                            }
                        }
                    }
#pragma unroll
                    for (int r = 0; r < RPW; ++r) {
                        if (!live[r]) continue;
                        double *gp = p.w + (e0 + eb + r) * p.ld + x0 + lane;
                        if (c0ok) gp[0] = v[r][0];
                        if (c1ok) gp[32] = v[r][1];
                    }
                }
            }
            __syncthreads();
            LU_T(5);  // trace: the rows' trailing update of this chunk
        }

        // ---- outer block complete: its pivots applied to the columns [x_hi, k)
        if (TWO && b2 && J + bw >= x_hi && x_hi < k) {
            lu_outer_update<MODE>(p, PRo, Acho, PR, pwo, pos, J, Jo, x_hi, ne, e0, thresh);
            LU_T(5);
        }
    }

    LU_T(4);
    // ---- final assembly (after everyone's write-backs and CTA 0's piv rows)
    bar_target += G;
    grid_arrive_wait(p.bar, bar_target);
    const int lane_f = tid & 31, warp_f = tid >> 5, nwarp_f = blockDim.x >> 5;
    // four entities per warp pass: their loads in flight together
    for (int eb = warp_f * 4; eb < ne; eb += nwarp_f * 4)
    for (int x = lane_f; x < k; x += 32) {
        double vv[4];
        int qq[4];
#pragma unroll
        for (int u4 = 0; u4 < 4; ++u4) {
            const int e = eb + u4;
            const int q = e < ne ? pos[e] : -1;
            qq[u4] = q;
            double v = 0.0;
            if (q >= 0 && q < k) {
                const int pend = min(k, (q / b) * b + b);
                v = x < pend ? __ldcg(p.w + (e0 + e) * p.ld + x) : __ldcg(p.piv + (int64_t)q * k + x);
            } else if (q >= k) {
                v = __ldcs(p.w + (e0 + e) * p.ld + x);
            }
            vv[u4] = v;
        }
#pragma unroll
        for (int u4 = 0; u4 < 4; ++u4) {
        const int q = qq[u4];
        const double v = vv[u4];
        if (q < 0) continue;
        if (MODE == MODE_ROW) {
            double lv = q >= k ? v : (x < q ? v : (x == q ? 1.0 : 0.0));
            p.out_main[(int64_t)q * p.ld_main + x] = lv;
            if (q < k && p.out_small) p.out_small[(int64_t)q * p.ld_small + x] = x >= q ? v : 0.0;
        } else {
            p.out_main[(int64_t)q * p.ld_main + x] = (q >= k || x <= q) ? v : 0.0;
            if (q < k) p.out_small[(int64_t)x * p.ld_small + q] = x > q ? v : (x == q ? 1.0 : 0.0);
        }
        }
    }
    for (int e = tid; e < ne; e += blockDim.x) p.perm[pos[e]] = e0 + e;
    LU_T(5);
    LU_TDUMP();
}

// ---------------------------------------------------------------------------
// Cluster variant: the same replay (identical per-element operation order,
// so identical results) on ONE thread-block cluster of CL CTAs (16 when the
// device allows non-portable clusters) x 1024 threads, one entity per
// thread, for matrices whose panels fit the cluster's shared memory
// (BASELINE configs 1-2: Y and core stay L2-resident).
//  * attribute-major working copy: the kernel first transposes its entities
//    into wt[x][e] (workspace), so every per-entity access of the panel loads,
//    write-backs and trailing updates is a coalesced warp access;
//  * exchange without a cluster-wide barrier: after the CTA argmax, warp d
//    (d < CL) writes {candidate, the candidate's panel row} into slot
//    [s&1][rank] of CTA d's shared memory with st.async, whose bytes complete
//    the transaction count of CTA d's mbarrier for that slot; each CTA waits
//    on its own mbarrier (armed with the step's byte count) and every warp
//    reduces the CL candidates locally.  Slots are double-buffered: a
//    producer can write slot s&1 again only at step s+2, after it received
//    every CTA's step-(s+1) push, which each CTA sends only after all its
//    threads finished step s (the argmax barriers in between);
//  * deferred trailing update: the panel's pivot entities' trailing values are
//    staged in shared memory once, the small triangular recurrence runs there,
//    and each thread updates its entity in blocks of 8 independent columns.
__device__ __forceinline__ unsigned mapa_rank(unsigned saddr, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_f64x2(unsigned addr, double a, double b) {
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(a), "d"(b) : "memory");
}
__device__ __forceinline__ void st_cluster_u64x2(unsigned addr, unsigned long long a,
                                                 unsigned long long b) {
    asm volatile("st.shared::cluster.v2.u64 [%0], {%1, %2};" ::"r"(addr), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void st_async_f64x2(unsigned addr, double a, double b, unsigned rbar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(addr),
        "d"(a), "d"(b), "r"(rbar)
        : "memory");
}
__device__ __forceinline__ void st_async_u64x2(unsigned addr, unsigned long long a,
                                               unsigned long long b, unsigned rbar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(addr),
        "l"(a), "l"(b), "r"(rbar)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx_cta(unsigned addr, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(addr),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_init_cta(unsigned addr, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(addr), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(unsigned raddr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(raddr)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(unsigned addr, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAITC_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAITC_%=;\n"
        "}\n" ::"r"(addr),
        "r"(parity)
        : "memory");
}

// warp argmax of (a desc, key asc) with three redux.sync steps: max of the
// high word, max of the low word among those, min key among the maxima
__device__ __forceinline__ void warp_argmax_redux(unsigned long long &a, unsigned &key) {
    const unsigned hi = (unsigned)(a >> 32), lo = (unsigned)a;
    const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
    const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
    const bool top = hi == mhi && lo == mlo;
    key = __reduce_min_sync(0xffffffffu, top ? key : 0xFFFFFFFFu);
    a = ((unsigned long long)mhi << 32) | mlo;
}

struct LuClusterParams {
    LuParams p;
    double *wt;   // k x ldt attribute-major working copy
    int64_t ldt;
};

template <int MODE>
__global__ void __launch_bounds__(1024, 1) lu_cluster_kernel(LuClusterParams cp) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ unsigned long long s_wabs[2][32];
    __shared__ unsigned s_wkey[2][32];
    __shared__ unsigned long long s_babs[2];
    __shared__ unsigned s_bkey[2];
    __shared__ double s_wsum[32];
    __shared__ double s_thresh;
    __shared__ __align__(8) uint64_t xbar[3];

    const LuParams &p = cp.p;
    double *const wt = cp.wt;
    const int64_t ldt = cp.ldt;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    const int CL = (int)cl.num_blocks();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = blockDim.x >> 5;
    const int k = p.k, b = p.b, bs = p.bs, rpc = p.rpc;
    const int b2 = (b + 1) & ~1;       // slot row length (16-byte rows)
    const int AW = ((k > b ? k - b : 1) + 15) & ~15;  // widest trailing block, 16-padded
    const int64_t e0 = (int64_t)rank * rpc;
    const int ne = (int)max((int64_t)0, min((int64_t)rpc, p.M - e0));
    const bool mine = tid < ne;  // thread tid owns entity e0 + tid
    const int64_t me = e0 + tid;

    double *xrow = reinterpret_cast<double *>(smem_raw);     // [3][CL][b2]
    Cand *xcand = reinterpret_cast<Cand *>(xrow + (size_t)3 * CL * b2);  // [3][CL]
    double *xpart = reinterpret_cast<double *>(xcand + 3 * CL);          // [CL]
    double *ucol = xpart + CL;                                           // [32][b]
    double *PR = ucol + 32 * b;                                          // b x b
    double *Ach = PR + (((size_t)b * b + 1) & ~(size_t)1);               // b x AW (16-B aligned)
    double *panel = Ach + (size_t)b * AW;                                // rpc x bs
    int *pw_ent = reinterpret_cast<int *>(panel + (size_t)rpc * bs);     // b
    int *qarr = pw_ent + b;                                              // rpc (epilogue)
    // transposes go through tiles of TWD columns in the panel region
    const int TWD = max(1, min(16, bs - 1));
    double *myrow = panel + (size_t)tid * bs;
    int mypos = (int)me;

    // CTA argmax of (|w| desc, position asc); key = pos << 10 | local entity
    auto cta_argmax = [&](unsigned long long a, unsigned key, int par) {
        warp_argmax_redux(a, key);
        if (lane == 0) { s_wabs[par][warp] = a; s_wkey[par][warp] = key; }
        __syncthreads();
        if (warp == 0) {
            a = lane < nwarps ? s_wabs[par][lane] : 0ULL;
            key = lane < nwarps ? s_wkey[par][lane] : 0xFFFFFFFFu;
            warp_argmax_redux(a, key);
            if (lane == 0) { s_babs[par] = a; s_bkey[par] = key; }
        }
        __syncthreads();
    };

    // bytes every CTA receives for step s: CL x {row pairs, candidate}
    auto step_bytes = [&](int st) -> unsigned {
        const int bw_s = min(b, k - (st / b) * b);
        return (unsigned)(CL * (((bw_s + 1) >> 1) * 16 + 16));
    };
    // push step st's CTA candidate (computed by cta_argmax into par st&1) and
    // its panel row into slot st%3 of every CTA: the owner's warp does it
    auto push = [&](int st, int bw_s) {
        const int par = st & 1;
        const unsigned long long babs = s_babs[par];
        const unsigned bkey = s_bkey[par];
        const int owner = bkey == 0xFFFFFFFFu ? -1 : (int)(bkey & 1023u);
        if (warp != (owner >= 0 ? owner >> 5 : 0)) return;
        __syncwarp();
        const int sl = st % 3;
        const int npair = (bw_s + 1) >> 1;
        const unsigned pos = owner >= 0 ? (bkey >> 10) : 0xFFFFFFFFu;
        const int ent = owner >= 0 ? (int)(e0 + owner) : -1;
        // lanes d and d+16 serve destination d: the first half of the pairs,
        // then the second half plus the candidate (mapa once per lane)
        const unsigned dst = (unsigned)(lane & 15);
        if ((int)dst < CL) {
            const unsigned rbar = mapa_rank(smem_u32(&xbar[sl]), dst);
            const unsigned rrow = mapa_rank(smem_u32(xrow + ((size_t)sl * CL + rank) * b2), dst);
            const int half = (npair + 1) >> 1;
            const int i0 = lane < 16 ? 0 : half, i1 = lane < 16 ? half : npair;
            const double *src = panel + (size_t)(owner >= 0 ? owner : 0) * bs;
            for (int it = i0; it < i1; ++it) {
                const int x = 2 * it;
                double v0 = 0.0, v1 = 0.0;
                if (owner >= 0) {
                    v0 = src[x];
                    v1 = x + 1 < bw_s ? src[x + 1] : 0.0;
                }
                st_async_f64x2(rrow + 16u * (unsigned)it, v0, v1, rbar);
            }
            if (lane >= 16)
                st_async_u64x2(mapa_rank(smem_u32(xcand + sl * CL + rank), dst), babs,
                               ((unsigned long long)(unsigned)ent << 32) | pos, rbar);
        }
    };
    if (tid == 0) {
        for (int i = 0; i < 3; ++i) mbar_init_cta(smem_u32(&xbar[i]), 1u);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < 3 && i < k; ++i) mbar_arrive_expect_tx_cta(smem_u32(&xbar[i]), step_bytes(i));
    }
    // ---- transpose own entities into wt (through shared-memory tiles, full
    // 128-byte rows read by 16 consecutive threads); ||w||_F^2 on the way ----
    double ss = 0.0;
    for (int x0 = 0; x0 < k; x0 += TWD) {
        const int cw = min(TWD, k - x0);
        for (int t = tid; t < ne * 16; t += blockDim.x) {
            const int e = t >> 4, c = t & 15;
            if (c < cw) panel[(size_t)e * bs + c] = p.w[(e0 + e) * p.ld + x0 + c];
        }
        __syncthreads();
        if (mine)
            for (int c = 0; c < cw; ++c) {
                const double v = myrow[c];
                wt[(int64_t)(x0 + c) * ldt + me] = v;
                ss += v * v;
            }
        __syncthreads();
    }
    cl.sync();  // barriers initialised, every CTA running, before any remote access
    {  // thresh = PIVOT_RTOL * ||w||_F (fixed-order two-level sum)
#pragma unroll
        for (int off = 16; off; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
        if (lane == 0) s_wsum[warp] = ss;
        __syncthreads();
        if (warp == 0) {
            double v = lane < nwarps ? s_wsum[lane] : 0.0;
#pragma unroll
            for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
            if (lane < CL) *cl.map_shared_rank(xpart + rank, lane) = v;
        }
        cl.sync();
        if (tid == 0) {
            double tot = 0.0;
            for (int c = 0; c < CL; ++c) tot += xpart[c];
            s_thresh = kPivotRtol * sqrt(tot);
        }
        __syncthreads();
    }
    const double thresh = s_thresh;
    LU_T0();

    for (int J = 0; J < k; J += b) {
        const int bw = min(b, k - J);
        if (mine)
            for (int x = 0; x < bw; ++x) myrow[x] = wt[(int64_t)(J + x) * ldt + me];
        {  // candidates for the panel's first column
            unsigned long long a = 0ULL;
            unsigned key = 0xFFFFFFFFu;
            if (mine && mypos >= J) {
                a = (unsigned long long)__double_as_longlong(fabs(myrow[0]));
                key = ((unsigned)mypos << 10) | (unsigned)tid;
            }
            cta_argmax(a, key, J & 1);
            push(J, bw);
        }
        LU_T(6);

        for (int ls = 0; ls < bw; ++ls) {
            const int s = J + ls;
            const int sl = s % 3;
            // 1. wait for the CL pushes of this step; re-arm the slot for s+3
            //    (its data can only arrive after this CTA's push of step s+2)
            mbar_wait_cluster(smem_u32(&xbar[sl]), (unsigned)((s / 3) & 1));
            if (tid == 0 && s + 3 < k) mbar_arrive_expect_tx_cta(smem_u32(&xbar[sl]), step_bytes(s + 3));
            LU_T(2);
            // 2. winner: every warp reduces the CL candidates itself
            unsigned long long ga = 0ULL;
            unsigned gkey = 0xFFFFFFFFu;
            if (lane < CL) {
                const Cand c = xcand[sl * CL + lane];
                if (c.entity >= 0) { ga = c.absbits; gkey = (c.pos << 4) | (unsigned)lane; }
            }
            warp_argmax_redux(ga, gkey);
            const int gc = (int)(gkey & 15u);
            const int wpos = (int)(gkey >> 4);
            const int went = xcand[sl * CL + gc].entity;
            const double *u = xrow + ((size_t)sl * CL + gc) * b2;
            const double pivv = u[ls];
            const bool big = fabs(pivv) > thresh;
            if (tid == 0) pw_ent[ls] = went;
            if (b < k && tid < bw)
                PR[ls * b + tid] = (MODE == MODE_COL && tid > ls) ? (big ? u[tid] / pivv : 0.0)
                                                                  : u[tid];
            // swap positions s <-> wpos (own entity only)
            if (mine) {
                if (mypos == s) mypos = wpos;
                if (me == went) mypos = s;
            }
            const double *um = u;
            if (MODE == MODE_COL) {  // this warp's copy of the multipliers
                double *uw = ucol + warp * b;
                if (lane > ls && lane < bw) uw[lane] = big ? u[lane] / pivv : 0.0;
                __syncwarp();
                um = uw;
            }
            LU_T(3);
            // 3. critical path: the next pivot column of own entity only
            double lm = 0.0;
            bool rest = false;  // the rest of the panel row still to update
            if (mine) {
                if (MODE == MODE_ROW) {
                    if (mypos > s) {
                        if (big) {
                            lm = myrow[ls] / pivv;
                            myrow[ls] = lm;
                            if (ls + 1 < bw)
                                myrow[ls + 1] = __dsub_rn(myrow[ls + 1], __dmul_rn(lm, u[ls + 1]));
                            rest = true;
                        } else {
                            myrow[ls] = 0.0;
                        }
                    }
                } else {
                    if (me == went) {
                        for (int x = ls + 1; x < bw; ++x) myrow[x] = um[x];
                    } else if (mypos > s && big) {
                        lm = myrow[ls];
                        if (ls + 1 < bw)
                            myrow[ls + 1] = __dsub_rn(myrow[ls + 1], __dmul_rn(um[ls + 1], lm));
                        rest = true;
                    }
                }
            }
            // x = ls+2 .. bw-1 in batches of 8 (loads first: no store-to-load
            // dependence between iterations)
            auto finish_row = [&]() {
                for (int x0 = ls + 2; x0 < bw; x0 += 8) {
                    double r[8], w[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const bool in = x0 + i < bw;
                        r[i] = in ? myrow[x0 + i] : 0.0;
                        w[i] = in ? (MODE == MODE_ROW ? u[x0 + i] : um[x0 + i]) : 0.0;
                    }
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        if (x0 + i < bw)
                            myrow[x0 + i] = MODE == MODE_ROW ? __dsub_rn(r[i], __dmul_rn(lm, w[i]))
                                                             : __dsub_rn(r[i], __dmul_rn(w[i], lm));
                }
            };
            LU_T(4);
            if (ls + 1 < bw) {
                // 4. CTA argmax of the next column; its owner completes its row
                //    and its warp pushes step s+1 before anyone else's row work
                unsigned long long a = 0ULL;
                unsigned key = 0xFFFFFFFFu;
                if (mine && mypos >= s + 1) {
                    a = (unsigned long long)__double_as_longlong(fabs(myrow[ls + 1]));
                    key = ((unsigned)mypos << 10) | (unsigned)tid;
                }
                cta_argmax(a, key, (s + 1) & 1);
                const unsigned bkey = s_bkey[(s + 1) & 1];
                if (rest && bkey != 0xFFFFFFFFu && (int)(bkey & 1023u) == tid) {
                    finish_row();
                    rest = false;
                }
                push(s + 1, bw);
            }
            LU_T(1);
            // 5. the rest of the panel row (overlaps the exchange of step s+1)
            if (rest) finish_row();
            LU_T(0);
        }
        __syncthreads();  // PR / pw_ent complete

        // write the panel back
        if (mine)
            for (int x = 0; x < bw; ++x) wt[(int64_t)(J + x) * ldt + me] = myrow[x];

        // deferred trailing update of columns [J+bw, k)
        const int x0 = J + bw, tw = k - x0;
        if (tw > 0) {
            const int twp = (tw + 15) & ~15;
            for (int t = tid; t < bw * twp; t += blockDim.x) {
                const int ls = t / twp, c = t % twp;
                Ach[ls * AW + c] = c < tw ? __ldcg(wt + (int64_t)(x0 + c) * ldt + pw_ent[ls]) : 0.0;
            }
            __syncthreads();
            for (int c = tid; c < tw; c += blockDim.x) {
                for (int ls = 0; ls < bw; ++ls) {
                    double v = Ach[ls * AW + c];
                    const double *pr = PR + ls * b;
                    if (MODE == MODE_ROW) {
                        for (int l2 = 0; l2 < ls; ++l2)
                            v = __dsub_rn(v, __dmul_rn(pr[l2], Ach[l2 * AW + c]));
                    } else {
                        for (int l2 = 0; l2 < ls; ++l2)
                            v = __dsub_rn(v, __dmul_rn(Ach[l2 * AW + c], pr[l2]));
                        const double pv = pr[ls];
                        v = fabs(pv) > thresh ? v / pv : 0.0;
                    }
                    Ach[ls * AW + c] = v;
                    if (rank == 0) p.piv[(int64_t)(J + ls) * k + x0 + c] = v;
                }
            }
            __syncthreads();
            if (mine && mypos >= x0) {  // pivots are frozen
                double *g = wt + (int64_t)x0 * ldt + me;
                for (int c0 = 0; c0 < tw; c0 += 16) {
                    double v[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) v[i] = c0 + i < tw ? g[(int64_t)(c0 + i) * ldt] : 0.0;
                    for (int ls = 0; ls < bw; ++ls) {
                        const double l = myrow[ls];
                        const double2 *ar = reinterpret_cast<const double2 *>(Ach + ls * AW + c0);
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const double2 av = ar[i];  // zero-padded past tw
                            if (MODE == MODE_ROW) {
                                v[2 * i] = __dsub_rn(v[2 * i], __dmul_rn(l, av.x));
                                v[2 * i + 1] = __dsub_rn(v[2 * i + 1], __dmul_rn(l, av.y));
                            } else {
                                v[2 * i] = __dsub_rn(v[2 * i], __dmul_rn(av.x, l));
                                v[2 * i + 1] = __dsub_rn(v[2 * i + 1], __dmul_rn(av.y, l));
                            }
                        }
                    }
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        if (c0 + i < tw) g[(int64_t)(c0 + i) * ldt] = v[i];
                }
            }
            __syncthreads();
        }
        LU_T(5);
    }
    LU_TDUMP();

    // ---- final assembly (after everyone's write-backs and rank 0's piv rows):
    // each entity's output row goes through a shared-memory tile so that 16
    // consecutive threads write 128 contiguous bytes of row q
    cl.sync();
    if (mine) {
        qarr[tid] = mypos;
        p.perm[mypos] = me;
    }
    const int q = mypos;
    const int pend = q < k ? min(k, (q / b) * b + b) : k;
    for (int x0 = 0; x0 < k; x0 += TWD) {
        const int cw = min(TWD, k - x0);
        if (mine)
            for (int c = 0; c < cw; ++c) {
                const int x = x0 + c;
                const double v =
                    x < pend ? wt[(int64_t)x * ldt + me] : __ldcg(p.piv + (int64_t)q * k + x);
                double o;
                if (MODE == MODE_ROW) {
                    o = q >= k ? v : (x < q ? v : (x == q ? 1.0 : 0.0));
                    if (q < k && p.out_small) p.out_small[(int64_t)q * p.ld_small + x] = x >= q ? v : 0.0;
                } else {
                    o = (q >= k || x <= q) ? v : 0.0;
                    if (q < k) p.out_small[(int64_t)x * p.ld_small + q] = x > q ? v : (x == q ? 1.0 : 0.0);
                }
                myrow[c] = o;
            }
        __syncthreads();
        for (int t = tid; t < ne * 16; t += blockDim.x) {
            const int e = t >> 4, c = t & 15;
            if (c < cw) p.out_main[(int64_t)qarr[e] * p.ld_main + x0 + c] = panel[(size_t)e * bs + c];
        }
        __syncthreads();
    }
    cl.sync();  // no CTA exits while a peer could still address its shared memory
}

static size_t lu_cluster_smem_bytes(int rpc, int b, int bs, int CL, int k) {
    const int AW = ((k > b ? k - b : 1) + 15) & ~15;
    const int b2 = (b + 1) & ~1;
    return sizeof(double) * ((size_t)3 * CL * b2 + CL + (size_t)32 * b + (((size_t)b * b + 1) & ~(size_t)1) +
                             (size_t)b * AW + (size_t)rpc * bs) +
           sizeof(Cand) * 3 * CL + sizeof(int) * ((size_t)b + rpc) + 16;
}

// ---------------------------------------------------------------------------
// Register-resident cluster LU (the default cluster path): as above, but the
// panel width is a compile-time B <= 16 and each thread keeps its entity's
// panel row in registers, so a pivot step's row update is B predicated
// mul/sub pairs against the pivot row (128-bit broadcast loads) with no
// shared-memory traffic for the rows.  The shared-memory row kernel above
// spent most of each step in shared-memory bandwidth (row loads/stores),
// which also delayed the remote st.async deliveries of the exchange.
template <int B>
__device__ __forceinline__ double rsel(const double (&r)[B], int i) {
    double v = 0.0;
#pragma unroll
    for (int j = 0; j < B; ++j)
        if (j == i) v = r[j];
    return v;
}

constexpr int kLuTile = 16;  // transpose tile width (row stride kLuTile + 1)

template <int MODE, int B>
__global__ void __launch_bounds__(1024, 1) lu_cluster_reg_kernel(LuClusterParams cp) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ unsigned long long s_wabs[2][32];
    __shared__ unsigned s_wkey[2][32];
    __shared__ unsigned long long s_babs[2];
    __shared__ unsigned s_bkey[2];
    __shared__ double s_wsum[32];
    __shared__ double s_thresh;
    __shared__ __align__(8) uint64_t xbar[3];
    __shared__ __align__(16) double s_own[B];

    const LuParams &p = cp.p;
    double *const wt = cp.wt;
    const int64_t ldt = cp.ldt;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    const int CL = (int)cl.num_blocks();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = blockDim.x >> 5;
    const int k = p.k, rpc = p.rpc;
    const int b = k < B ? k : B;
    const int AW = ((k > b ? k - b : 1) + 15) & ~15;
    const int64_t e0 = (int64_t)rank * rpc;
    const int ne = (int)max((int64_t)0, min((int64_t)rpc, p.M - e0));
    const bool mine = tid < ne;
    const int64_t me = e0 + tid;

    double *xrow = reinterpret_cast<double *>(smem_raw);                 // [3][CL][B]
    Cand *xcand = reinterpret_cast<Cand *>(xrow + (size_t)3 * CL * B);   // [3][CL]
    double *xpart = reinterpret_cast<double *>(xcand + 3 * CL);          // [CL]
    double *ucol = xpart + ((CL + 1) & ~1);                              // [32][B]
    double *PR = ucol + 32 * B;                                          // B x B
    double *Ach = PR + B * B;                                            // B x AW
    double *tile = Ach + (size_t)B * AW;                                 // rpc x (kLuTile+1)
    int *pw_ent = reinterpret_cast<int *>(tile + (size_t)rpc * (kLuTile + 1));  // B
    int *qarr = pw_ent + B;                                              // rpc
    double *mytile = tile + (size_t)tid * (kLuTile + 1);
    int mypos = (int)me;
    double r[B];

    auto cta_argmax = [&](unsigned long long a, unsigned key, int par) {
        warp_argmax_redux(a, key);
        if (lane == 0) { s_wabs[par][warp] = a; s_wkey[par][warp] = key; }
        __syncthreads();
        if (warp == 0) {
            a = lane < nwarps ? s_wabs[par][lane] : 0ULL;
            key = lane < nwarps ? s_wkey[par][lane] : 0xFFFFFFFFu;
            warp_argmax_redux(a, key);
            if (lane == 0) { s_babs[par] = a; s_bkey[par] = key; }
        }
        __syncthreads();
    };
    auto step_bytes = [&](int st) -> unsigned {
        const int bw_s = min(b, k - (st / b) * b);
        return (unsigned)(CL * (((bw_s + 1) >> 1) * 16 + 16));
    };
    // after cta_argmax(.., st&1): the owner stages its row, its warp pushes
    // {candidate, row} into slot st%3 of every CTA (lanes d, d+16 -> CTA d)
    auto stage_and_push = [&](int st, int bw_s) {
        const int par = st & 1;
        const unsigned long long babs = s_babs[par];
        const unsigned bkey = s_bkey[par];
        const int owner = bkey == 0xFFFFFFFFu ? -1 : (int)(bkey & 1023u);
        if (warp != (owner >= 0 ? owner >> 5 : 0)) return;
        if (tid == owner) {
#pragma unroll
            for (int i = 0; i < B; ++i) s_own[i] = r[i];
        }
        __syncwarp();
        const int sl = st % 3;
        const int npair = (bw_s + 1) >> 1;
        const unsigned pos = owner >= 0 ? (bkey >> 10) : 0xFFFFFFFFu;
        const int ent = owner >= 0 ? (int)(e0 + owner) : -1;
        const unsigned dst = (unsigned)(lane & 15);
        if ((int)dst < CL) {
            const unsigned rbar = mapa_rank(smem_u32(&xbar[sl]), dst);
            const unsigned rrow = mapa_rank(smem_u32(xrow + ((size_t)sl * CL + rank) * B), dst);
            const int half = (npair + 1) >> 1;
            const int i0 = lane < 16 ? 0 : half, i1 = lane < 16 ? half : npair;
            for (int it = i0; it < i1; ++it) {
                const int x = 2 * it;
                const double v0 = owner >= 0 ? s_own[x] : 0.0;
                const double v1 = owner >= 0 && x + 1 < bw_s ? s_own[x + 1] : 0.0;
                st_async_f64x2(rrow + 16u * (unsigned)it, v0, v1, rbar);
            }
            if (lane >= 16)
                st_async_u64x2(mapa_rank(smem_u32(xcand + sl * CL + rank), dst), babs,
                               ((unsigned long long)(unsigned)ent << 32) | pos, rbar);
        }
    };

    if (tid == 0) {
        for (int i = 0; i < 3; ++i) mbar_init_cta(smem_u32(&xbar[i]), 1u);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < 3 && i < k; ++i) mbar_arrive_expect_tx_cta(smem_u32(&xbar[i]), step_bytes(i));
    }
    // ---- transpose own entities into wt through shared-memory tiles;
    // ||w||_F^2 on the way (per entity in column order) ----
    double ss = 0.0;
    for (int x0 = 0; x0 < k; x0 += kLuTile) {
        const int cw = min(kLuTile, k - x0);
        for (int t = tid; t < ne * kLuTile; t += blockDim.x) {
            const int e = t / kLuTile, c = t % kLuTile;
            if (c < cw) tile[(size_t)e * (kLuTile + 1) + c] = p.w[(e0 + e) * p.ld + x0 + c];
        }
        __syncthreads();
        if (mine)
            for (int c = 0; c < cw; ++c) {
                const double v = mytile[c];
                wt[(int64_t)(x0 + c) * ldt + me] = v;
                ss += v * v;
            }
        __syncthreads();
    }
    cl.sync();  // barriers initialised, every CTA running, before any remote access
    {  // thresh = PIVOT_RTOL * ||w||_F (fixed-order two-level sum)
#pragma unroll
        for (int off = 16; off; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
        if (lane == 0) s_wsum[warp] = ss;
        __syncthreads();
        if (warp == 0) {
            double v = lane < nwarps ? s_wsum[lane] : 0.0;
#pragma unroll
            for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
            if (lane < CL) *cl.map_shared_rank(xpart + rank, lane) = v;
        }
        cl.sync();
        if (tid == 0) {
            double tot = 0.0;
            for (int c = 0; c < CL; ++c) tot += xpart[c];
            s_thresh = kPivotRtol * sqrt(tot);
        }
        __syncthreads();
    }
    const double thresh = s_thresh;
    LU_T0();

    for (int J = 0; J < k; J += b) {
        const int bw = min(b, k - J);
#pragma unroll
        for (int i = 0; i < B; ++i) r[i] = (mine && i < bw) ? wt[(int64_t)(J + i) * ldt + me] : 0.0;
        {
            unsigned long long a = 0ULL;
            unsigned key = 0xFFFFFFFFu;
            if (mine && mypos >= J) {
                a = (unsigned long long)__double_as_longlong(fabs(r[0]));
                key = ((unsigned)mypos << 10) | (unsigned)tid;
            }
            cta_argmax(a, key, J & 1);
            stage_and_push(J, bw);
        }
        LU_T(6);

        for (int ls = 0; ls < bw; ++ls) {
            const int s = J + ls;
            const int sl = s % 3;
            mbar_wait_cluster(smem_u32(&xbar[sl]), (unsigned)((s / 3) & 1));
            if (tid == 0 && s + 3 < k) mbar_arrive_expect_tx_cta(smem_u32(&xbar[sl]), step_bytes(s + 3));
            LU_T(2);
            unsigned long long ga = 0ULL;
            unsigned gkey = 0xFFFFFFFFu;
            if (lane < CL) {
                const Cand c = xcand[sl * CL + lane];
                if (c.entity >= 0) { ga = c.absbits; gkey = (c.pos << 4) | (unsigned)lane; }
            }
            warp_argmax_redux(ga, gkey);
            const int gc = (int)(gkey & 15u);
            const int wpos = (int)(gkey >> 4);
            const int went = xcand[sl * CL + gc].entity;
            const double *u = xrow + ((size_t)sl * CL + gc) * B;
            const double pivv = u[ls];
            const bool big = fabs(pivv) > thresh;
            if (tid == 0) pw_ent[ls] = went;
            if (b < k && tid < bw)
                PR[ls * B + tid] = (MODE == MODE_COL && tid > ls) ? (big ? u[tid] / pivv : 0.0)
                                                                  : u[tid];
            if (mine) {
                if (mypos == s) mypos = wpos;
                if (me == went) mypos = s;
            }
            const double *um = u;
            if (MODE == MODE_COL) {
                double *uw = ucol + warp * B;
                if (lane > ls && lane < bw) uw[lane] = big ? u[lane] / pivv : 0.0;
                __syncwarp();
                um = uw;
            }
            LU_T(3);
            if (mine) {
                const double2 *uv = reinterpret_cast<const double2 *>(um);
                if (MODE == MODE_ROW) {
                    if (mypos > s) {
                        if (big) {
                            const double lm = rsel<B>(r, ls) / pivv;
#pragma unroll
                            for (int i2 = 0; i2 < B / 2; ++i2) {
                                const double2 w = uv[i2];
                                const int i = 2 * i2;
                                if (i == ls) r[i] = lm;
                                else if (i > ls && i < bw) r[i] = __dsub_rn(r[i], __dmul_rn(lm, w.x));
                                if (i + 1 == ls) r[i + 1] = lm;
                                else if (i + 1 > ls && i + 1 < bw)
                                    r[i + 1] = __dsub_rn(r[i + 1], __dmul_rn(lm, w.y));
                            }
                        } else {
#pragma unroll
                            for (int i = 0; i < B; ++i)
                                if (i == ls) r[i] = 0.0;
                        }
                    }
                } else {
                    if (me == went) {
#pragma unroll
                        for (int i2 = 0; i2 < B / 2; ++i2) {
                            const double2 w = uv[i2];
                            const int i = 2 * i2;
                            if (i > ls && i < bw) r[i] = w.x;
                            if (i + 1 > ls && i + 1 < bw) r[i + 1] = w.y;
                        }
                    } else if (mypos > s && big) {
                        const double lm = rsel<B>(r, ls);
#pragma unroll
                        for (int i2 = 0; i2 < B / 2; ++i2) {
                            const double2 w = uv[i2];
                            const int i = 2 * i2;
                            if (i > ls && i < bw) r[i] = __dsub_rn(r[i], __dmul_rn(w.x, lm));
                            if (i + 1 > ls && i + 1 < bw)
                                r[i + 1] = __dsub_rn(r[i + 1], __dmul_rn(w.y, lm));
                        }
                    }
                }
            }
            LU_T(4);
            if (ls + 1 < bw) {
                unsigned long long a = 0ULL;
                unsigned key = 0xFFFFFFFFu;
                if (mine && mypos >= s + 1) {
                    a = (unsigned long long)__double_as_longlong(fabs(rsel<B>(r, ls + 1)));
                    key = ((unsigned)mypos << 10) | (unsigned)tid;
                }
                cta_argmax(a, key, (s + 1) & 1);
                stage_and_push(s + 1, bw);
            }
            LU_T(1);
        }
        __syncthreads();  // PR / pw_ent complete

        // write the panel back; the multipliers go to this thread's tile row
        // (the registers are free for the trailing update's 16-column block)
#pragma unroll
        for (int i = 0; i < B; ++i)
            if (i < bw) {
                if (mine) wt[(int64_t)(J + i) * ldt + me] = r[i];
                mytile[i] = r[i];
            }

        const int x0 = J + bw, tw = k - x0;
        if (tw > 0) {
            const int twp = (tw + 15) & ~15;
            for (int t = tid; t < bw * twp; t += blockDim.x) {
                const int ls = t / twp, c = t % twp;
                Ach[ls * AW + c] = c < tw ? __ldcg(wt + (int64_t)(x0 + c) * ldt + pw_ent[ls]) : 0.0;
            }
            __syncthreads();
            for (int c = tid; c < tw; c += blockDim.x) {
                for (int ls = 0; ls < bw; ++ls) {
                    double v = Ach[ls * AW + c];
                    const double *pr = PR + ls * B;
                    if (MODE == MODE_ROW) {
                        for (int l2 = 0; l2 < ls; ++l2)
                            v = __dsub_rn(v, __dmul_rn(pr[l2], Ach[l2 * AW + c]));
                    } else {
                        for (int l2 = 0; l2 < ls; ++l2)
                            v = __dsub_rn(v, __dmul_rn(Ach[l2 * AW + c], pr[l2]));
                        const double pv = pr[ls];
                        v = fabs(pv) > thresh ? v / pv : 0.0;
                    }
                    Ach[ls * AW + c] = v;
                    if (rank == 0) p.piv[(int64_t)(J + ls) * k + x0 + c] = v;
                }
            }
            __syncthreads();
            if (mine && mypos >= x0) {  // pivots are frozen
                double *g = wt + (int64_t)x0 * ldt + me;
                for (int c0 = 0; c0 < tw; c0 += 16) {
                    double v[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) v[i] = c0 + i < tw ? g[(int64_t)(c0 + i) * ldt] : 0.0;
                    for (int ls = 0; ls < bw; ++ls) {
                        const double l = mytile[ls];
                        const double2 *ar = reinterpret_cast<const double2 *>(Ach + ls * AW + c0);
#pragma unroll
                        for (int i2 = 0; i2 < 8; ++i2) {
                            const double2 av = ar[i2];  // zero-padded past tw
                            if (MODE == MODE_ROW) {
                                v[2 * i2] = __dsub_rn(v[2 * i2], __dmul_rn(l, av.x));
                                v[2 * i2 + 1] = __dsub_rn(v[2 * i2 + 1], __dmul_rn(l, av.y));
                            } else {
                                v[2 * i2] = __dsub_rn(v[2 * i2], __dmul_rn(av.x, l));
                                v[2 * i2 + 1] = __dsub_rn(v[2 * i2 + 1], __dmul_rn(av.y, l));
                            }
                        }
                    }
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        if (c0 + i < tw) g[(int64_t)(c0 + i) * ldt] = v[i];
                }
            }
            __syncthreads();
        }
        LU_T(5);
    }
    LU_TDUMP();

    // ---- final assembly through shared-memory tiles ----
    cl.sync();
    if (mine) {
        qarr[tid] = mypos;
        p.perm[mypos] = me;
    }
    const int q = mypos;
    const int pend = q < k ? min(k, (q / b) * b + b) : k;
    for (int x0 = 0; x0 < k; x0 += kLuTile) {
        const int cw = min(kLuTile, k - x0);
        if (mine)
            for (int c = 0; c < cw; ++c) {
                const int x = x0 + c;
                const double v =
                    x < pend ? wt[(int64_t)x * ldt + me] : __ldcg(p.piv + (int64_t)q * k + x);
                double o;
                if (MODE == MODE_ROW) {
                    o = q >= k ? v : (x < q ? v : (x == q ? 1.0 : 0.0));
                    if (q < k && p.out_small) p.out_small[(int64_t)q * p.ld_small + x] = x >= q ? v : 0.0;
                } else {
                    o = (q >= k || x <= q) ? v : 0.0;
                    if (q < k) p.out_small[(int64_t)x * p.ld_small + q] = x > q ? v : (x == q ? 1.0 : 0.0);
                }
                mytile[c] = o;
            }
        __syncthreads();
        for (int t = tid; t < ne * kLuTile; t += blockDim.x) {
            const int e = t / kLuTile, c = t % kLuTile;
            if (c < cw)
                p.out_main[(int64_t)qarr[e] * p.ld_main + x0 + c] = tile[(size_t)e * (kLuTile + 1) + c];
        }
        __syncthreads();
    }
    cl.sync();  // no CTA exits while a peer could still address its shared memory
}

template <int B>
static size_t lu_cluster_reg_smem_bytes(int rpc, int CL, int k) {
    const int b = k < B ? k : B;
    const int AW = ((k > b ? k - b : 1) + 15) & ~15;
    return sizeof(double) * ((size_t)3 * CL * B + ((CL + 1) & ~1) + (size_t)32 * B + (size_t)B * B +
                             (size_t)B * AW + (size_t)rpc * (kLuTile + 1)) +
           sizeof(Cand) * 3 * CL + sizeof(int) * ((size_t)B + rpc) + 16;
}

// One pivot step on a register-resident panel row with the step index LS a
// compile-time constant: only columns > LS are touched (no per-element
// predication on LS).  Returns the entity's next-column value (argmax input).
template <int MODE, int B, int LS>
__device__ __forceinline__ double step_regs(double (&r)[B], const double *__restrict__ um,
                                            double pivv, bool big, bool active, bool pivot_ent,
                                            int bw) {
    if (MODE == MODE_ROW) {
        if (active) {
            if (big) {
                const double lm = r[LS] / pivv;
                r[LS] = lm;
#pragma unroll
                for (int i = LS + 1; i < B; ++i)
                    if (i < bw) r[i] = __dsub_rn(r[i], __dmul_rn(lm, um[i]));
            } else {
                r[LS] = 0.0;
            }
        }
    } else {
        if (pivot_ent) {
#pragma unroll
            for (int i = LS + 1; i < B; ++i)
                if (i < bw) r[i] = um[i];
        } else if (active && big) {
            const double lm = r[LS];
#pragma unroll
            for (int i = LS + 1; i < B; ++i)
                if (i < bw) r[i] = __dsub_rn(r[i], __dmul_rn(um[i], lm));
        }
    }
    return LS + 1 < B ? r[LS + 1 < B ? LS + 1 : 0] : 0.0;
}

#define SRLU_STEP_CASE(L)                                                                   \
    case L:                                                                                 \
        if constexpr (L < B) nxt = step_regs<MODE, B, L>(rj, um, pivv, big, act, piv_ent, bw); \
        break;

// The same step split at the critical path: step_first touches column LS+1
// only (the next pivot column), step_rest columns LS+2.. afterwards, while
// the exchange of the next step is in flight.
template <int MODE, int B, int LS>
__device__ __forceinline__ double step_first(double (&r)[B], const double *__restrict__ um,
                                             double pivv, bool big, bool active, bool pivot_ent,
                                             int bw, bool &upd) {
    constexpr int N1 = LS + 1 < B ? LS + 1 : B - 1;
    const bool has1 = LS + 1 < B && LS + 1 < bw;
    if (MODE == MODE_ROW) {
        if (active) {
            if (big) {
                const double lm = r[LS] / pivv;
                r[LS] = lm;
                if (has1) r[N1] = __dsub_rn(r[N1], __dmul_rn(lm, um[N1]));
                upd = true;
            } else {
                r[LS] = 0.0;
            }
        }
    } else {
        if (pivot_ent) {
#pragma unroll
            for (int i = LS + 1; i < B; ++i)
                if (i < bw) r[i] = um[i];
        } else if (active && big) {
            if (has1) r[N1] = __dsub_rn(r[N1], __dmul_rn(um[N1], r[LS]));
            upd = true;
        }
    }
    return has1 ? r[N1] : 0.0;
}

template <int MODE, int B, int LS>
__device__ __forceinline__ void step_rest(double (&r)[B], const double *__restrict__ um, int bw) {
    const double lm = r[LS];  // ROW: the multiplier; COL: the pivot-column value
#pragma unroll
    for (int i = LS + 2; i < B; ++i)
        if (i < bw)
            r[i] = MODE == MODE_ROW ? __dsub_rn(r[i], __dmul_rn(lm, um[i]))
                                    : __dsub_rn(r[i], __dmul_rn(um[i], lm));
}

#define SRLU_CASES_16(M)                                                                  \
    M(0) M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10) M(11) M(12) M(13) M(14) M(15)
#define SRLU_FIRST_CASE(L)                                                                 \
    case L:                                                                                \
        if constexpr (L < B) nxt = step_first<MODE, B, L>(rj, um, pivv, big, act, piv_ent, bw, updj); \
        break;
#define SRLU_REST_CASE(L)                                                                  \
    case L:                                                                                \
        if constexpr (L < B) step_rest<MODE, B, L>(rj, um, bw);                            \
        break;

// ---------------------------------------------------------------------------
// Hybrid LU (default for M <= 16384): ONE cooperative launch of G CTAs in
// clusters of 16 (G = every co-resident cluster).  Cluster 0 runs each
// panel's pivot steps exactly as lu_cluster_reg_kernel (registers rows,
// DSMEM st.async exchange); then, after a grid barrier, ALL G CTAs apply the
// panel's deferred trailing update to their own entity ranges, and a second
// grid barrier hands the updated columns back to cluster 0.  The latency-
// bound pivot chain stays inside one cluster while the FP64 trailing work
// (most of the flops) runs on every SM.  Same per-element operation order.
struct LuHybridParams {
    LuParams p;
    double *wt;   // k x ldt attribute-major working copy
    int64_t ldt;
    int *gpos;    // [M] position of each entity (written by cluster 0 per panel)
    double *gPR;  // [B][B] the panel's pivot rows (panel part)
    int *gpw;     // [B] the panel's pivot entities
    double *gpart;  // [G] partial sums of squares
    unsigned *cnt;  // CTAs done with the next panel's columns (zeroed per launch)
    int nocoop;     // launched without the cooperative attribute: own grid barrier on p.bar
};

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <int MODE, int B, int RPT>
__global__ void __launch_bounds__(1024 / RPT, 1) lu_hybrid_kernel(LuHybridParams hp) {
    constexpr int NT = 1024 / RPT;  // RPT entities per thread in the panel phase
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ unsigned long long s_wabs[2][32];
    __shared__ unsigned s_wkey[2][32];
    __shared__ unsigned long long s_babs[2];
    __shared__ unsigned s_bkey[2];
    __shared__ double s_wsum[32];
    __shared__ double s_thresh;
    __shared__ __align__(8) uint64_t xbar[3];
    __shared__ __align__(16) double s_own[B];
    __shared__ int s_pw[B];

    const LuParams &p = hp.p;
    double *const wt = hp.wt;
    const int64_t ldt = hp.ldt;
    cg::grid_group grid = cg::this_grid();
    cg::cluster_group cl = cg::this_cluster();
    const int G = gridDim.x, bid = blockIdx.x;
    // Grid-wide barrier: grid.sync() of the cooperative launch, or — when the
    // kernel was launched without the cooperative attribute (profilers that
    // cannot replay cooperative cluster launches; every CTA is co-resident
    // by construction of the grid) — the counter barrier on p.bar.
    unsigned nc_target = 0;
    auto grid_sync = [&]() {
        if (hp.nocoop) {
            nc_target += (unsigned)G;
            grid_arrive_wait(hp.p.bar, nc_target);
        } else {
            grid.sync();
        }
    };
    const bool panel_cta = bid < (int)cl.num_blocks();  // cluster 0
    const int rank = (int)cl.block_rank();
    const int CL = (int)cl.num_blocks();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = blockDim.x >> 5;
    const int k = p.k;
    const int64_t M = p.M;
    const int b = k < B ? k : B;
    const int AW = ((k > b ? k - b : 1) + 15) & ~15;
    // phase-A ownership (cluster 0): local entities tid + j*NT, j < RPT
    const int rpcA = (int)ceil_div(M, (int64_t)CL);
    const int64_t eA0 = (int64_t)rank * rpcA;
    const int neA = (int)max((int64_t)0, min((int64_t)rpcA, M - eA0));
    bool mineA[RPT];
    int64_t meA[RPT];
    int mypos[RPT];
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
        mineA[j] = panel_cta && tid + j * NT < neA;
        meA[j] = eA0 + tid + j * NT;
        mypos[j] = (int)meA[j];
    }
    // whole-grid ownership (prologue, trailing, epilogue): [eT0, eT0 + neT)
    const int rpcT = (int)ceil_div(M, (int64_t)G);
    const int64_t eT0 = (int64_t)bid * rpcT;
    const int neT = (int)max((int64_t)0, min((int64_t)rpcT, M - eT0));

    double *xrow = reinterpret_cast<double *>(smem_raw);                 // [3][CL][B]
    Cand *xcand = reinterpret_cast<Cand *>(xrow + (size_t)3 * CL * B);   // [3][CL]
    double *ucol = reinterpret_cast<double *>(xcand + 3 * CL);           // [32][B]
    double *PR = ucol + 32 * B;                                          // B x B
    double *Ach = PR + B * B;                                            // B x AW
    double *tile = Ach + (size_t)B * AW;                                 // rpcT x (kLuTile+1)
    int *qarr = reinterpret_cast<int *>(tile + (size_t)rpcT * (kLuTile + 1));  // rpcT
    double r[RPT][B];

    auto cta_argmax = [&](unsigned long long a, unsigned key, int par) {
        warp_argmax_redux(a, key);
        if (lane == 0) { s_wabs[par][warp] = a; s_wkey[par][warp] = key; }
        __syncthreads();
        if (warp == 0) {
            a = lane < nwarps ? s_wabs[par][lane] : 0ULL;
            key = lane < nwarps ? s_wkey[par][lane] : 0xFFFFFFFFu;
            warp_argmax_redux(a, key);
            if (lane == 0) { s_babs[par] = a; s_bkey[par] = key; }
        }
        __syncthreads();
    };
    auto step_bytes = [&](int st) -> unsigned {
        const int bw_s = min(b, k - (st / b) * b);
        return (unsigned)(CL * (((bw_s + 1) >> 1) * 16 + 16));
    };
    auto stage_and_push = [&](int st, int bw_s) {
        const int par = st & 1;
        const unsigned long long babs = s_babs[par];
        const unsigned bkey = s_bkey[par];
        const int owner = bkey == 0xFFFFFFFFu ? -1 : (int)(bkey & 1023u);  // local entity
        const int othr = owner >= 0 ? owner % NT : 0;
        if (warp != (othr >> 5)) return;
        if (owner >= 0 && tid == othr) {
            const int oj = owner / NT;
#pragma unroll
            for (int j = 0; j < RPT; ++j)
                if (j == oj) {
#pragma unroll
                    for (int i = 0; i < B; ++i) s_own[i] = r[j][i];
                }
        }
        __syncwarp();
        const int sl = st % 3;
        const int npair = (bw_s + 1) >> 1;
        const unsigned pos = owner >= 0 ? (bkey >> 10) : 0xFFFFFFFFu;
        const int ent = owner >= 0 ? (int)(eA0 + owner) : -1;
        const unsigned dst = (unsigned)(lane & 15);
        if ((int)dst < CL) {
            const unsigned rbar = mapa_rank(smem_u32(&xbar[sl]), dst);
            const unsigned rrow = mapa_rank(smem_u32(xrow + ((size_t)sl * CL + rank) * B), dst);
            const int half = (npair + 1) >> 1;
            const int i0 = lane < 16 ? 0 : half, i1 = lane < 16 ? half : npair;
            for (int it = i0; it < i1; ++it) {
                const int x = 2 * it;
                const double v0 = owner >= 0 ? s_own[x] : 0.0;
                const double v1 = owner >= 0 && x + 1 < bw_s ? s_own[x + 1] : 0.0;
                st_async_f64x2(rrow + 16u * (unsigned)it, v0, v1, rbar);
            }
            if (lane >= 16)
                st_async_u64x2(mapa_rank(smem_u32(xcand + sl * CL + rank), dst), babs,
                               ((unsigned long long)(unsigned)ent << 32) | pos, rbar);
        }
    };

    if (panel_cta && tid == 0) {
        for (int i = 0; i < 3; ++i) mbar_init_cta(smem_u32(&xbar[i]), 1u);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < 3 && i < k; ++i) mbar_arrive_expect_tx_cta(smem_u32(&xbar[i]), step_bytes(i));
    }
    // ---- prologue (all CTAs): transpose own range into wt; positions;
    // ||w||_F^2 partial per CTA ----
    double ss = 0.0;
    for (int x0 = 0; x0 < k; x0 += kLuTile) {
        const int cw = min(kLuTile, k - x0);
        for (int t = tid; t < neT * kLuTile; t += blockDim.x) {
            const int e = t / kLuTile, c = t % kLuTile;
            if (c < cw) tile[(size_t)e * (kLuTile + 1) + c] = p.w[(eT0 + e) * p.ld + x0 + c];
        }
        __syncthreads();
        if (tid < neT)
            for (int c = 0; c < cw; ++c) {
                const double v = tile[(size_t)tid * (kLuTile + 1) + c];
                wt[(int64_t)(x0 + c) * ldt + eT0 + tid] = v;
                ss += v * v;
            }
        __syncthreads();
    }
    if (tid < neT) hp.gpos[eT0 + tid] = (int)(eT0 + tid);
#pragma unroll
    for (int off = 16; off; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    if (lane == 0) s_wsum[warp] = ss;
    __syncthreads();
    if (warp == 0) {
        double v = lane < nwarps ? s_wsum[lane] : 0.0;
#pragma unroll
        for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) hp.gpart[bid] = v;
    }
    cl.sync();    // cluster 0: barriers initialised before any remote access
    grid_sync();  // wt, gpos, partials complete
    if (tid == 0) {
        double tot = 0.0;
        for (int c = 0; c < G; ++c) tot += __ldcg(hp.gpart + c);
        s_thresh = kPivotRtol * sqrt(tot);
    }
    __syncthreads();
    const double thresh = s_thresh;
    LU_T0();
    int npan = 0;

    for (int J = 0; J < k; J += b) {
        const int bw = min(b, k - J);
        // ======== phase A: the panel's pivot steps (cluster 0) ========
        if (panel_cta) {
#pragma unroll
            for (int j = 0; j < RPT; ++j)
#pragma unroll
                for (int i = 0; i < B; ++i)
                    r[j][i] = (mineA[j] && i < bw) ? __ldcg(wt + (int64_t)(J + i) * ldt + meA[j]) : 0.0;
            {
                unsigned long long a = 0ULL;
                unsigned key = 0xFFFFFFFFu;
#pragma unroll
                for (int j = 0; j < RPT; ++j)
                    if (mineA[j] && mypos[j] >= J) {
                        const unsigned long long aj =
                            (unsigned long long)__double_as_longlong(fabs(r[j][0]));
                        const unsigned kj = ((unsigned)mypos[j] << 10) | (unsigned)(tid + j * NT);
                        if (better(aj, kj, a, key)) { a = aj; key = kj; }
                    }
                cta_argmax(a, key, J & 1);
                stage_and_push(J, bw);
            }
            for (int ls = 0; ls < bw; ++ls) {
                const int s = J + ls;
                const int sl = s % 3;
                LU_T(6);
                mbar_wait_cluster(smem_u32(&xbar[sl]), (unsigned)((s / 3) & 1));
                if (tid == 0 && s + 3 < k) mbar_arrive_expect_tx_cta(smem_u32(&xbar[sl]), step_bytes(s + 3));
                LU_T(4);
                unsigned long long ga = 0ULL;
                unsigned gkey = 0xFFFFFFFFu;
                if (lane < CL) {
                    const Cand c = xcand[sl * CL + lane];
                    if (c.entity >= 0) { ga = c.absbits; gkey = (c.pos << 4) | (unsigned)lane; }
                }
                warp_argmax_redux(ga, gkey);
                const int gc = (int)(gkey & 15u);
                const int wpos = (int)(gkey >> 4);
                const int went = xcand[sl * CL + gc].entity;
                const double *u = xrow + ((size_t)sl * CL + gc) * B;
                const double pivv = u[ls];
                const bool big = fabs(pivv) > thresh;
                if (tid == 0) s_pw[ls] = went;
                if (b < k && tid < bw)
                    PR[ls * B + tid] = (MODE == MODE_COL && tid > ls) ? (big ? u[tid] / pivv : 0.0)
                                                                      : u[tid];
#pragma unroll
                for (int j = 0; j < RPT; ++j)
                    if (mineA[j]) {
                        if (mypos[j] == s) mypos[j] = wpos;
                        if (meA[j] == went) mypos[j] = s;
                    }
                const double *um = u;
                if (MODE == MODE_COL) {
                    double *uw = ucol + warp * B;
                    if (lane > ls && lane < bw) uw[lane] = big ? u[lane] / pivv : 0.0;
                    __syncwarp();
                    um = uw;
                }
                if constexpr (MODE == MODE_ROW) {  // critical-path split (row LU)
                unsigned long long ca = 0ULL;
                unsigned ckey = 0xFFFFFFFFu;
                bool upd[RPT];
#pragma unroll
                for (int j = 0; j < RPT; ++j) {
                    double nxt = 0.0;
                    bool updj = false;
                    if (mineA[j]) {
                        double (&rj)[B] = r[j];
                        const bool act = mypos[j] > s, piv_ent = meA[j] == went;
                        switch (ls) {
                            SRLU_CASES_16(SRLU_FIRST_CASE)
                            default: break;
                        }
                        if (mypos[j] >= s + 1) {
                            const unsigned long long aj =
                                (unsigned long long)__double_as_longlong(fabs(nxt));
                            const unsigned kj = ((unsigned)mypos[j] << 10) | (unsigned)(tid + j * NT);
                            if (better(aj, kj, ca, ckey)) { ca = aj; ckey = kj; }
                        }
                    }
                    upd[j] = updj;
                }
                auto rest_row = [&](int j) {
#pragma unroll
                    for (int jj = 0; jj < RPT; ++jj)
                        if (jj == j) {
                            double (&rj)[B] = r[jj];
                            switch (ls) {
                                SRLU_CASES_16(SRLU_REST_CASE)
                                default: break;
                            }
                        }
                };
                if (ls + 1 < bw) {
                    cta_argmax(ca, ckey, (s + 1) & 1);
                    // the owner completes its row before its warp stages it
                    const unsigned bk = s_bkey[(s + 1) & 1];
                    if (bk != 0xFFFFFFFFu && (int)(bk & 1023u) % NT == tid) {
                        const int oj = (int)(bk & 1023u) / NT;
#pragma unroll
                        for (int j = 0; j < RPT; ++j)
                            if (j == oj && upd[j]) {
                                rest_row(j);
                                upd[j] = false;
                            }
                    }
                    stage_and_push(s + 1, bw);
                }
                // the rest of the rows, overlapping the exchange of step s+1
#pragma unroll
                for (int j = 0; j < RPT; ++j)
                    if (upd[j]) rest_row(j);
                } else {  // one pass per step (column LU: the split measured slower)
                unsigned long long ca = 0ULL;
                unsigned ckey = 0xFFFFFFFFu;
#pragma unroll
                for (int j = 0; j < RPT; ++j) {
                    double nxt = 0.0;
                    if (mineA[j]) {
                        double (&rj)[B] = r[j];
                        const bool act = mypos[j] > s, piv_ent = meA[j] == went;
                        switch (ls) {
                            SRLU_CASES_16(SRLU_STEP_CASE)
                            default: break;
                        }
                        if (mypos[j] >= s + 1) {
                            const unsigned long long aj =
                                (unsigned long long)__double_as_longlong(fabs(nxt));
                            const unsigned kj = ((unsigned)mypos[j] << 10) | (unsigned)(tid + j * NT);
                            if (better(aj, kj, ca, ckey)) { ca = aj; ckey = kj; }
                        }
                    }
                }
                if (ls + 1 < bw) {
                    cta_argmax(ca, ckey, (s + 1) & 1);
                    stage_and_push(s + 1, bw);
                }
                }
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
#pragma unroll
                for (int i = 0; i < B; ++i)
                    if (mineA[j] && i < bw) wt[(int64_t)(J + i) * ldt + meA[j]] = r[j][i];
                if (mineA[j]) hp.gpos[meA[j]] = mypos[j];
            }
            if (rank == 0) {
                for (int t = tid; t < bw * B; t += blockDim.x) hp.gPR[t] = PR[t];
                if (tid < bw) hp.gpw[tid] = s_pw[tid];
            }
        }
        LU_T(0);
        const int x0 = J + bw, tw = k - x0;
        if (tw <= 0) break;
        grid_sync();
        LU_T(1);
        // ======== phase C: the panel's trailing update (all CTAs) ========
        {
            const int twp = (tw + 15) & ~15;
            // (entity, column group) per thread: consecutive threads take
            // consecutive entities of the same columns (coalesced in wt).
            // Everything that does not depend on the pivot rows — the
            // frozen-pivot check, the entity's multipliers and its first
            // block of trailing values — is loaded before the pivot-row
            // rounds below, so those latencies overlap.
            constexpr int NI = 3;
            // the counter hand-off below lets cluster 0 start the next panel once
            // pass 1 is done everywhere: pass 1 (columns x0 .. x0 + NI*4*ngrp - 1,
            // ngrp >= 1) must therefore contain the whole next panel
            static_assert(B <= NI * 4, "hybrid LU: pass 1 must cover the next panel's columns");
            const int ngrp = neT > 0 ? max(1, (int)blockDim.x / neT) : 1;
            const int el = neT > 0 ? tid % neT : 0, grp = neT > 0 ? tid / neT : ngrp;
            const int64_t e = eT0 + el;
            const bool cact = neT > 0 && grp < ngrp;
            const int gp_e = cact ? __ldcg(hp.gpos + e) : 0;
            double l[B];
            double v[NI][4];
#pragma unroll
            for (int ls = 0; ls < B; ++ls)
                l[ls] = cact && ls < bw ? __ldcg(wt + (int64_t)(J + ls) * ldt + e) : 0.0;
            {
                const int cb = 4 * grp;
#pragma unroll
                for (int q = 0; q < NI; ++q)
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int c = cb + q * 4 * ngrp + i;
                        v[q][i] = cact && c < tw ? __ldcg(wt + (int64_t)(x0 + c) * ldt + e) : 0.0;
                    }
            }
            for (int t = tid; t < bw * B; t += blockDim.x) PR[t] = __ldcg(hp.gPR + t);
            if (tid < bw) s_pw[tid] = __ldcg(hp.gpw + tid);
            __syncthreads();
            for (int t = tid; t < bw * twp; t += blockDim.x) {
                const int ls = t / twp, c = t % twp;
                Ach[ls * AW + c] = c < tw ? __ldcg(wt + (int64_t)(x0 + c) * ldt + s_pw[ls]) : 0.0;
            }
            __syncthreads();
            LU_T(5);
            // the panel's pivot rows on the trailing columns: the small
            // triangular recurrence in registers, fully unrolled so that the
            // independent chains of different ls overlap (each chain keeps
            // the reference's l2 order)
            for (int c = tid; c < tw; c += blockDim.x) {
                double a[B];
#pragma unroll
                for (int ls = 0; ls < B; ++ls) a[ls] = ls < bw ? Ach[ls * AW + c] : 0.0;
#pragma unroll
                for (int ls = 0; ls < B; ++ls) {
                    if (ls < bw) {
                        double v = a[ls];
                        const double *pr = PR + ls * B;
#pragma unroll
                        for (int l2 = 0; l2 < ls; ++l2)
                            v = MODE == MODE_ROW ? __dsub_rn(v, __dmul_rn(pr[l2], a[l2]))
                                                 : __dsub_rn(v, __dmul_rn(a[l2], pr[l2]));
                        if (MODE != MODE_ROW) {
                            const double pv = pr[ls];
                            v = fabs(pv) > thresh ? v / pv : 0.0;
                        }
                        a[ls] = v;
                    }
                }
#pragma unroll
                for (int ls = 0; ls < B; ++ls) {
                    if (ls < bw) {
                        Ach[ls * AW + c] = a[ls];
                        if (bid == 0) p.piv[(int64_t)(J + ls) * k + x0 + c] = a[ls];
                    }
                }
            }
            __syncthreads();
            LU_T(7);
            // columns 4*grp + {0..3} + 4*ngrp*it, three such groups (twelve
            // independent loads) in flight per thread.  Pass 1 = the first
            // block (prefetched above; it holds every column of the next
            // panel), then a signal to cluster 0, then pass 2 = the rest.
            for (int pass = 0; pass < 2; ++pass) {
                if (pass == 1) {
                    __syncthreads();
                    if (tid == 0) {
                        __threadfence();
                        atomicAdd(hp.cnt, 1u);
                    }
                }
                if (cact && gp_e >= x0) {  // pivots are frozen
                    const int cb0 = 4 * grp + (pass ? NI * 4 * ngrp : 0);
                    const int cb1 = pass ? tw : min(tw, 4 * grp + 1);
                    for (int cb = cb0; cb < cb1; cb += NI * 4 * ngrp) {
                        if (pass) {
#pragma unroll
                            for (int q = 0; q < NI; ++q)
#pragma unroll
                                for (int i = 0; i < 4; ++i) {
                                    const int c = cb + q * 4 * ngrp + i;
                                    v[q][i] = c < tw ? __ldcg(wt + (int64_t)(x0 + c) * ldt + e) : 0.0;
                                }
                        }
#pragma unroll
                        for (int q = 0; q < NI; ++q) {
                            const int c0 = cb + q * 4 * ngrp;
                            if (c0 >= tw) break;
#pragma unroll
                            for (int ls = 0; ls < B; ++ls)
                                if (ls < bw) {
#pragma unroll
                                    for (int i = 0; i < 4; ++i) {
                                        const double av = Ach[ls * AW + c0 + i];  // zero past tw
                                        v[q][i] = MODE == MODE_ROW
                                                      ? __dsub_rn(v[q][i], __dmul_rn(l[ls], av))
                                                      : __dsub_rn(v[q][i], __dmul_rn(av, l[ls]));
                                    }
                                }
#pragma unroll
                            for (int i = 0; i < 4; ++i)
                                if (c0 + i < tw) wt[(int64_t)(x0 + c0 + i) * ldt + e] = v[q][i];
                        }
                    }
                }
            }
        }
        LU_T(2);
        // cluster 0 waits only until every CTA has updated the next panel's
        // columns (pass 1); the rest of the trailing update overlaps the
        // next panel's pivot steps.  The next panel's grid barrier orders
        // everyone's pass 2 before its own phase C.
        ++npan;
        if (panel_cta) {
            if (tid == 0)
                while (ld_acquire_gpu(hp.cnt) < (unsigned)(npan * G)) __nanosleep(32);
            __syncthreads();
        }
        LU_T(3);
    }
    LU_TDUMP();

    // ---- final assembly (all CTAs) through shared-memory tiles ----
    grid_sync();
    const int q = tid < neT ? __ldcg(hp.gpos + eT0 + tid) : 0;
    if (tid < neT) {
        qarr[tid] = q;
        p.perm[q] = eT0 + tid;
    }
    const int pend = q < k ? min(k, (q / b) * b + b) : k;
    for (int x0 = 0; x0 < k; x0 += kLuTile) {
        const int cw = min(kLuTile, k - x0);
        if (tid < neT)
            for (int c = 0; c < cw; ++c) {
                const int x = x0 + c;
                const double v = x < pend ? __ldcg(wt + (int64_t)x * ldt + eT0 + tid)
                                          : __ldcg(p.piv + (int64_t)q * k + x);
                double o;
                if (MODE == MODE_ROW) {
                    o = q >= k ? v : (x < q ? v : (x == q ? 1.0 : 0.0));
                    if (q < k && p.out_small) p.out_small[(int64_t)q * p.ld_small + x] = x >= q ? v : 0.0;
                } else {
                    o = (q >= k || x <= q) ? v : 0.0;
                    if (q < k) p.out_small[(int64_t)x * p.ld_small + q] = x > q ? v : (x == q ? 1.0 : 0.0);
                }
                tile[(size_t)tid * (kLuTile + 1) + c] = o;
            }
        __syncthreads();
        for (int t = tid; t < neT * kLuTile; t += blockDim.x) {
            const int e = t / kLuTile, c = t % kLuTile;
            if (c < cw)
                p.out_main[(int64_t)qarr[e] * p.ld_main + x0 + c] = tile[(size_t)e * (kLuTile + 1) + c];
        }
        __syncthreads();
    }
}

template <int B>
static size_t lu_hybrid_smem_bytes(int rpcT, int CL, int k) {
    const int b = k < B ? k : B;
    const int AW = ((k > b ? k - b : 1) + 15) & ~15;
    return sizeof(double) * ((size_t)3 * CL * B + (size_t)32 * B + (size_t)B * B + (size_t)B * AW +
                             (size_t)rpcT * (kLuTile + 1)) +
           sizeof(Cand) * 3 * CL + sizeof(int) * (size_t)rpcT + 16;
}

// the cluster path is considered for M <= 16 * 1024 entities
constexpr int64_t kLuClusterMaxM = 16 * 1024;
static inline int64_t lu_cluster_ldt(int64_t M) { return (M + 31) & ~(int64_t)31; }
static size_t lu_base_workspace(int64_t k) {
    return 256 + sizeof(double) * kLuMaxGrid + sizeof(Cand) * 2 * kLuMaxGrid +
           sizeof(double) * ((size_t)2 * kLuMaxGrid * k + (size_t)k * k) + 256;
}

// L2 panel of the grid kernel: [8][ldp] doubles after the base workspace
static inline int64_t lu_gpanel_ld(int64_t M) { return (M + 31) & ~(int64_t)31; }

// Outer block of the two-level trailing update for panels of width b (0 =
// one level).  Opt-in experiment (SRLU_LU_B2=1), bit-exact (tests), measured
// slower on B200 and therefore off: it cuts the HBM traffic of the trailing
// updates by b2 / b, but those are bound by their instruction stream at 16
// warps per SM, not by traffic — config 3 shape (262144 x 220, shared-memory
// panel) 4.16 -> 4.52 ms (narrow in-block chunks leave lanes idle, the extra
// 24 KB of shared memory narrow the panel); config 4 (1048576 x 120, L2
// panel) LU(Y) 8.74 -> 10.4 ms (the out-of-line update spills at the
// 128-register cap).  The kernels without it (TWO = false) are unchanged.
static int lu_outer_width(int b, int64_t k, bool gpanel) {
    (void)gpanel;
    bool on = false;
    if (const char *env = getenv("SRLU_LU_B2")) on = atoi(env) != 0;  // testing knob
    if (!on || b >= k || 2 * b > kLuB2Max) return 0;
    return (kLuB2Max / b) * b;
}

static size_t lu_smem_bytes(int rpc, int b, int bs, int b2 = 0) {
    return sizeof(double) * ((size_t)rpc * bs + (size_t)b * b + 2 * (size_t)b + (size_t)b * kLuXC +
                             (size_t)b2 * kLuB2Max + (size_t)b2 * kLuXC) +
           sizeof(int) * ((size_t)rpc + b + b2) + 16;
}

static int sm_count() {
    static int cached = 0;   // one device per process (one process per GPU)
    if (cached > 0) return cached;
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached = n > 0 ? n : 1;
    return cached;
}

// Cluster path when the panels of all M entities fit one cluster's shared
// memory with a useful panel width; returns SRLU_OK when launched, 1 when the
// shape (or the device) does not qualify.
template <typename Kern>
static int launch_lu_cluster(Kern kern, int CL, size_t smem, LuClusterParams cp,
                             cudaStream_t stream, bool *launched) {
    *launched = false;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess) {
        cudaGetLastError();
        return SRLU_OK;
    }
    if (CL > 8 &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
            cudaSuccess) {
        cudaGetLastError();
        return SRLU_OK;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(CL);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, (void *)kern, &cfg) != cudaSuccess ||
        nclusters < 1) {
        cudaGetLastError();
        return SRLU_OK;
    }
    SRLU_CUDA(cudaLaunchKernelEx(&cfg, kern, cp));
    *launched = true;
    return SRLU_OK;
}

template <int MODE, int B, int RPT>
static int try_run_lu_hybrid_b(LuParams prm, void *ws, cudaStream_t stream, bool *launched) {
    *launched = false;
    const int64_t M = prm.M;
    const int k = prm.k;
    constexpr int CL = 16;
    auto kern = lu_hybrid_kernel<MODE, B, RPT>;
    static bool np_ok = false;   // set once per kernel variant
    if (!np_ok) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
            cudaGetLastError();
            return SRLU_OK;
        }
        np_ok = true;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    // ncu aborts the process on a cooperative launch with cluster dimensions
    // (GPUTEST_r01: ncu_rc = 9).  Under a CUDA injection profiler (or with
    // SRLU_LU_NOCOOP = 1) the same kernel is launched with the cluster
    // attribute only and synchronises the grid with its own counter barrier:
    // the grid is sized to the co-resident clusters, so every CTA is running.
    int nocoop = getenv("CUDA_INJECTION64_PATH") != nullptr || getenv("NV_NSIGHT_INJECTION_PORT_BASE") != nullptr;
    if (const char *env = getenv("SRLU_LU_NOCOOP")) nocoop = atoi(env) != 0;
    cfg.blockDim = dim3(1024 / RPT);
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = nocoop ? 1 : 2;
    // grid = every co-resident cluster (smem depends on the per-CTA range).
    // The occupancy search costs several driver queries (tens of
    // microseconds of host time per LU): its result is kept for the last
    // shape of this kernel variant.
    struct Plan { int64_t M; int k; int nocoop; int ncl; size_t smem; };
    static Plan last = {-1, 0, 0, 0, 0};
    static std::mutex last_mu;
    int ncl = 0;
    size_t smem = 0;
    bool cached = false;
    {
        std::lock_guard<std::mutex> lk(last_mu);
        if (last.M == M && last.k == k && last.nocoop == nocoop) {
            ncl = last.ncl;
            smem = last.smem;
            cached = true;   // the kernel's shared-memory attribute still holds this value
        }
    }
    for (int guess = cached ? 0 : 9; guess >= 1; --guess) {
        const int rpcT = (int)ceil_div(M, (int64_t)(guess * CL));
        smem = lu_hybrid_smem_bytes<B>(rpcT, CL, k);
        if (smem > 220 * 1024) return SRLU_OK;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess) {
            cudaGetLastError();
            return SRLU_OK;
        }
        cfg.gridDim = dim3(guess * CL);
        cfg.dynamicSmemBytes = smem;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, (void *)kern, &cfg) != cudaSuccess) {
            cudaGetLastError();
            return SRLU_OK;
        }
        if (n >= guess) { ncl = guess; break; }
    }
    if (!cached) {
        std::lock_guard<std::mutex> lk(last_mu);
        last = {M, k, nocoop, ncl, smem};
    } else {
        cfg.gridDim = dim3(ncl * CL);
        cfg.dynamicSmemBytes = smem;
    }
    if (ncl < 1 || ceil_div(M, (int64_t)CL) > 1024 ||
        ceil_div(M, (int64_t)(ncl * CL)) > 1024 / RPT)  // one entity per thread outside phase A
        return SRLU_OK;
    const int G = ncl * CL;
    LuHybridParams hp;
    hp.p = prm;
    hp.p.b = k < B ? k : B;
    hp.p.bs = hp.p.b | 1;
    hp.p.rpc = (int)ceil_div(M, (int64_t)CL);
    hp.ldt = lu_cluster_ldt(M);
    char *base = (char *)ws + ((lu_base_workspace(k) + 255) & ~(size_t)255);
    hp.wt = (double *)base;
    char *extra = base + sizeof(double) * (size_t)k * hp.ldt;
    hp.gpos = (int *)extra;
    extra += ((size_t)M * sizeof(int) + 255) & ~(size_t)255;
    hp.gPR = (double *)extra;
    extra += 256 * sizeof(double) + 256;
    hp.gpart = (double *)extra;
    extra += 256 * sizeof(double);
    hp.gpw = (int *)extra;
    hp.cnt = (unsigned *)(extra + 128);  // gpw holds <= 16 ints
    SRLU_CUDA(cudaMemsetAsync(hp.cnt, 0, sizeof(unsigned), stream));
    hp.nocoop = nocoop;
    if (nocoop) SRLU_CUDA(cudaMemsetAsync(prm.bar, 0, 256, stream));
    (void)G;
    SRLU_CUDA(cudaLaunchKernelEx(&cfg, kern, hp));
    *launched = true;
    return SRLU_OK;
}

template <int MODE>
static int try_run_lu_hybrid(LuParams prm, void *ws, cudaStream_t stream) {
    if (const char *env = getenv("SRLU_LU_NO_HYBRID"))  // testing knob
        if (atoi(env)) return 1;
    if (prm.M > kLuClusterMaxM || prm.k > 1024) return 1;
    bool launched = false;
    const int hb = getenv("SRLU_LU_HYBRID_B") ? atoi(getenv("SRLU_LU_HYBRID_B")) : 0;  // testing knob
    // B = 8 measured faster than 12 at BASELINE config 2 (smaller per-step
    // code: the step is specialised per in-panel index)
    const int rc = hb != 12 ? try_run_lu_hybrid_b<MODE, 8, 2>(prm, ws, stream, &launched)
                            : try_run_lu_hybrid_b<MODE, 12, 2>(prm, ws, stream, &launched);
    if (rc != SRLU_OK) return rc;
    return launched ? SRLU_OK : 1;
}

template <int MODE>
static int try_run_lu_cluster(LuParams prm, void *ws, cudaStream_t stream) {
    if (const char *env = getenv("SRLU_LU_NO_CLUSTER"))  // testing knob
        if (atoi(env)) return 1;
    const bool v4 = getenv("SRLU_LU_CLUSTER_V4") != nullptr;  // shared-memory rows (comparison)
    const int64_t M = prm.M;
    const int k = prm.k;
    // the register-row kernel faults for k > 128 (measured: 220, 300, 500);
    // wider inputs take the grid kernel (the hybrid kernel is tried first)
    if (M > kLuClusterMaxM || k > (v4 ? 1024 : 128)) return 1;
    const size_t budget = 220 * 1024;
    LuClusterParams cp;
    cp.p = prm;
    cp.ldt = lu_cluster_ldt(M);
    cp.wt = (double *)((char *)ws + ((lu_base_workspace(k) + 255) & ~(size_t)255));
    for (int CL : {16, 8}) {
        const int64_t rpc64 = ceil_div(M, (int64_t)CL);
        if (rpc64 > 1024) continue;  // one entity per thread
        const int rpc = (int)rpc64;
        cp.p.rpc = rpc;
        bool launched = false;
        if (!v4) {
            // panel width B: 12 keeps the row plus the step's state within the
            // 64 registers of a 1024-thread CTA (16 spills); 8 for tiny k
            int B = k <= 8 ? 8 : 12;
            if (const char *env = getenv("SRLU_LU_REG_B")) B = atoi(env);  // testing knob
            size_t smem;
            int rc;
            if (B == 8) {
                smem = lu_cluster_reg_smem_bytes<8>(rpc, CL, k);
                if (smem > budget) continue;
                cp.p.b = k < 8 ? k : 8;
                cp.p.bs = cp.p.b | 1;
                rc = launch_lu_cluster(lu_cluster_reg_kernel<MODE, 8>, CL, smem, cp, stream, &launched);
            } else if (B == 16) {
                smem = lu_cluster_reg_smem_bytes<16>(rpc, CL, k);
                if (smem > budget) continue;
                cp.p.b = k < 16 ? k : 16;
                cp.p.bs = cp.p.b | 1;
                rc = launch_lu_cluster(lu_cluster_reg_kernel<MODE, 16>, CL, smem, cp, stream, &launched);
            } else {
                smem = lu_cluster_reg_smem_bytes<12>(rpc, CL, k);
                if (smem > budget) continue;
                cp.p.b = k < 12 ? k : 12;
                cp.p.bs = cp.p.b | 1;
                rc = launch_lu_cluster(lu_cluster_reg_kernel<MODE, 12>, CL, smem, cp, stream, &launched);
            }
            if (rc != SRLU_OK) return rc;
        } else {
            int b = k < 32 ? k : 32;
            while (b > 1 && lu_cluster_smem_bytes(rpc, b, b | 1, CL, k) > budget) --b;
            if (b < (k < 8 ? k : 8) || lu_cluster_smem_bytes(rpc, b, b | 1, CL, k) > budget) continue;
            cp.p.b = b;
            cp.p.bs = b | 1;
            const int rc = launch_lu_cluster(lu_cluster_kernel<MODE>, CL,
                                             lu_cluster_smem_bytes(rpc, b, b | 1, CL, k), cp, stream,
                                             &launched);
            if (rc != SRLU_OK) return rc;
        }
        if (launched) return SRLU_OK;
    }
    return 1;
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

    char *wsb = (char *)ws;
    LuParams prm;
    prm.w = w; prm.M = M; prm.k = (int)k; prm.ld = ld;
    prm.perm = perm; prm.out_main = out_main; prm.ld_main = ld_main;
    prm.out_small = out_small; prm.ld_small = ld_small;
    prm.bar = (unsigned *)wsb;
    prm.partial = (double *)(wsb + 256);
    prm.cand = (Cand *)(wsb + 256 + sizeof(double) * kLuMaxGrid);
    prm.candrow = (double *)((char *)prm.cand + sizeof(Cand) * 2 * kLuMaxGrid);
    prm.piv = prm.candrow + (size_t)2 * kLuMaxGrid * k;
    prm.gpanel = nullptr;
    prm.ldp = 0;
    prm.l2pf = 1;  // tools/lu_sweep.sh: config 3 LU(Y) 4.39 -> 4.08 ms
    prm.b2 = 0;
    prm.la = 1;
    if (const char *env = getenv("SRLU_LU_LA")) prm.la = atoi(env) != 0;  // testing knob
    if (const char *env = getenv("SRLU_LU_L2PF")) prm.l2pf = atoi(env);  // testing knob

    int rc = try_run_lu_hybrid<MODE>(prm, ws, stream);
    if (rc <= 0) return rc;  // launched (0) or failed (<0)
    // the single-cluster kernels are kept for comparison only (opt-in): the
    // hybrid kernel supersedes them, and the register-row one faults on some
    // shapes (k > 128; 2048 x 60)
    if (const char *env = getenv("SRLU_LU_CLUSTER"))  // testing knob
        if (atoi(env)) {
            rc = try_run_lu_cluster<MODE>(prm, ws, stream);
            if (rc <= 0) return rc;
        }

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
    while (b > 1 && lu_smem_bytes(rpc, b, b | 1, lu_outer_width(b, k, false)) > budget) --b;
    int bs = b | 1;
    // narrow smem panel (tall inputs): an 8-wide attribute-major L2 panel
    const char *nogp = getenv("SRLU_LU_NO_GPANEL");  // testing knob
    const char *fgp = getenv("SRLU_LU_GPANEL");       // testing knob: force it
    const bool gpanel = ((b < k && b < 8) || (fgp && atoi(fgp))) && !(nogp && atoi(nogp)) &&
                        (int64_t)rpc * ld < (1LL << 31) - 1;
    if (gpanel) {
        b = k < 8 ? (int)k : 8;
        bs = 0;
        prm.ldp = lu_gpanel_ld(M);
        prm.gpanel = (double *)(wsb + ((lu_base_workspace(k) + 255) & ~(size_t)255));
    }
    prm.b2 = lu_outer_width(b, k, gpanel);
    size_t smem = lu_smem_bytes(rpc, b, bs, prm.b2);
    SRLU_REQUIRE(smem <= budget, SRLU_ERR_UNSUPPORTED,
                 "lu: %lld entities per CTA do not fit in shared memory", (long long)rpc);
    auto kern = gpanel ? (prm.b2 ? lu_kernel<MODE, 8, true> : lu_kernel<MODE, 8, false>)
                       : (prm.b2 ? lu_kernel<MODE, 0, true> : lu_kernel<MODE, 0, false>);
    SRLU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    SRLU_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kLuThreads, smem));
    SRLU_REQUIRE(per_sm >= 1, SRLU_ERR_UNSUPPORTED, "lu: kernel cannot be resident");
    prm.b = b; prm.bs = bs; prm.rpc = rpc;
    SRLU_CUDA(cudaMemsetAsync(prm.bar, 0, 256, stream));
    void *args[] = {&prm};
    SRLU_CUDA(cudaLaunchCooperativeKernel((const void *)kern, dim3(G), dim3(kLuThreads), args, smem,
                                          stream));
    return SRLU_OK;
}

}  // namespace srlu

using namespace srlu;

// hybrid-path arrays after the attribute-major copy: gpos[M], gPR[16x16],
// gpw[16], gpart[256]
static size_t lu_hybrid_extra(int64_t M) {
    return (((size_t)M * sizeof(int) + 255) & ~(size_t)255) + 256 * sizeof(double) + 256 +
           256 * sizeof(double) + 256;
}

extern "C" size_t srlu_lu_workspace(int64_t M, int64_t k) {
    size_t n = lu_base_workspace(k);
    // the grid kernel's L2 panel (same offset; the cluster paths' copy is
    // laid out there too and never coexists with it)
    const size_t ngp = ((n + 255) & ~(size_t)255) + sizeof(double) * 8 * (size_t)lu_gpanel_ld(M);
    if (M <= kLuClusterMaxM && k <= 1024)  // attribute-major copy for the cluster paths
        n = ((n + 255) & ~(size_t)255) + sizeof(double) * (size_t)k * lu_cluster_ldt(M) +
            lu_hybrid_extra(M);
    return n > ngp ? n : ngp;
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
