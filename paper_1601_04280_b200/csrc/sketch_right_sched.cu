// K1 v4 — scheduled, warp-specialised stage-1 sketch  Y = A · Omega1^*
// (reference: sketch.py:362-368 apply_sketch_right = _fast.pyx:44-54
// sem_gather_dense + sketch.py:322-335 _fast_adjoint_right + _fast.pyx:23-41
// fwht_rows), for dense A whose rows span at most kMaxChunks TMA chunks.
//
// Why a schedule.  Every (row, bucket) sum must be accumulated in ascending
// source column (the reference's loop order) to be bit-identical, so one
// lane owns one bucket and walks its sources.  Walked naively (k1v2) the
// lanes of a warp diverge (Poisson bucket sizes) and their shared-memory
// gathers hit random banks (~3.5-way conflicts).  The schedule, computed
// once per sketch on the device, turns each warp's walk into a fixed number
// of uniform steps: in every step each lane either takes its bucket's next
// source or reads a zero word, and no two lanes of a step touch the same
// shared-memory bank (per half-warp for 8-byte elements) — one wavefront
// per gather.  Lanes with the longest remaining queue win bank collisions.
// Codes are 16 bits (chunk-local column | sign << 15), two steps per u32,
// staged in shared memory when they fit.
//
// Kernel structure (persistent, one CTA per SM, 1024 threads):
//   * a ring of NS stages of RB rows x C columns, filled by 1-D bulk copies
//     (cp.async.bulk + mbarrier); the last gather warp to release a stage
//     refills it, so the stream never waits on a CTA-wide barrier;
//   * 28 gather warps: fp64 register accumulators acc[BPT][RB] persisting
//     across the chunks of a row block, then +-phase and the FWHT stages
//     h < 32 by shuffles (lane = bucket bits 0..4) into a double-buffered
//     scratch xs;
//   * per row block, all 32 warps then run the stages 32 <= h < 512 (one
//     thread per in-block column, registers) and the output-pruned stages
//     h >= 512 for the k sampled outputs only (x mult, Y store, non-finite
//     flag), between two CTA barriers — the bulk copies of the next stages
//     stay in flight meanwhile.
#include <limits.h>
#include <stdlib.h>

#include <algorithm>

#include "fwht_warp.cuh"
#include "tma.cuh"

namespace srlu {

namespace k1s {

constexpr int kGW = 28;                 // gather warps (of 32)
constexpr int kNT = 1024;
constexpr int kMaxChunks = 4;          // codes staged in shared memory
constexpr int kMaxChunksG = 32;        // codes read from global memory (L2-resident)
constexpr int kMaxStages = 8;
constexpr int kZeroBytes = 128;         // zero tail per staged row: one word per bank
constexpr size_t kSmemMax = 232448 - 1024;
constexpr int kHeader = 16;             // int32 header words

struct Cfg {
    int es, rb, bpt, c, nch, ns, ng, zpad, d2, sorted, joint, xpad;
    int64_t stage_bytes, row_stride, xs_bytes, code_cap, smem;
    // workspace offsets (bytes)
    int64_t off_grp, off_np, off_wsched, off_codes, ws_bytes;
};

static int env_int(const char *name, int dflt) {
    const char *s = getenv(name);
    return (s && *s) ? atoi(s) : dflt;
}

// SM count of the process's device (one process per GPU), queried once
static int device_sms() {
    static int cached = 0;
    if (cached > 0) return cached;
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached = n > 0 ? n : 148;
    return cached;
}

// Deterministic from (n, l, pad, es): the schedule and the kernel agree.
// One geometry (rows per block rb, stage target bytes); false if it does
// not fit the shared-memory budget with at least two stages.
static bool config_try(int64_t n, int64_t l, int64_t pad, int es, int bpt, int rb,
                       int64_t stage_target, Cfg *cf) {
    int64_t cmax = stage_target / (rb * es);
    cmax &= ~31LL;
    if (cmax < 32) return false;
    int64_t nch = ceil_div(n, cmax);
    if (nch > kMaxChunksG) return false;
    int64_t c = ((ceil_div(n, nch) + 31) / 32) * 32;
    if (c + kZeroBytes / es > 32767) return false;
    Cfg f{};
    f.es = es; f.rb = rb; f.bpt = bpt; f.c = (int)c; f.nch = (int)nch;
    f.ng = kGW * bpt; f.zpad = kZeroBytes / es;
    f.d2 = env_int("SRLU_K1_D", 2) >= 2 ? 2 : 1;
    // several slots per lane: buckets sorted by count into groups (similar
    // queues per warp step), heavy and light groups paired per warp (snake),
    // each slot on its own step sequence.  One slot: consecutive buckets, so
    // the FWHT stages h < 32 run on the accumulators directly.
    f.sorted = env_int("SRLU_K1_SORT", bpt >= 2 ? 1 : 0) != 0;
    // joint = the slots of a warp step together (one code stream per warp and
    // chunk).  Codes in shared memory: separate sequences per slot (fewer
    // padded steps).  Codes read from L2 (more than kMaxChunks chunks): joint,
    // because each slot sequence is a dependent L2 round trip and the kernel
    // is bound by that latency (config 5: 14.2 -> 10.4 ms)
    f.joint = env_int("SRLU_K1_JOINT", (f.sorted && nch <= kMaxChunks) ? 0 : 1) != 0;
    f.row_stride = (c + f.zpad) * es;
    f.stage_bytes = rb * f.row_stride;
    // FWHT scratch: only the bsize-point blocks that hold buckets (blocks
    // past ceil(l / bsize) stay zero through the in-block stages and enter
    // the output-pruned cross-block stages as zeros)
    {
        const int64_t bs = pad < 512 ? pad : 512;
        f.xpad = (int)(ceil_div(l, bs) * bs);
    }
    f.xs_bytes = 2LL * rb * f.xpad * 8;
    // leave room for the codes (~64 B per warp step, ~n/16 steps); more than
    // kMaxChunks chunks: the codes stay in global memory
    const int64_t code_est = (env_int("SRLU_K1_GCODES", 0) || nch > kMaxChunks) ? 0 : 4 * n + 4096;
    int ns = env_int("SRLU_K1_NS", 4);
    if (ns < 2) ns = 2;
    if (ns > kMaxStages) ns = kMaxStages;
    while (ns > 2 && (size_t)(ns * f.stage_bytes + f.xs_bytes + code_est) > kSmemMax) --ns;
    f.ns = ns;
    int64_t used = ns * f.stage_bytes + f.xs_bytes;
    if ((size_t)used + (code_est ? 8192 : 256) > kSmemMax) return false;
    f.code_cap = ((int64_t)kSmemMax - used) & ~15LL;
    f.smem = used + f.code_cap;
    // workspace: header | grp[ng*32] | np[nch*ng] | wsched[nch*ng*2] | codes
    auto al = [](int64_t v) { return (v + 15) & ~15LL; };
    f.off_grp = al(kHeader * 4);
    f.off_np = al(f.off_grp + (int64_t)f.ng * 32 * 4);
    f.off_wsched = al(f.off_np + (int64_t)nch * f.ng * 4);
    f.off_codes = al(f.off_wsched + (int64_t)nch * f.ng * 8);
    // a step advances >= 1 source of its group; pairs round up; slots of a
    // warp are padded to the longest: <= bpt * 16 * (n + 2 nch ng) words
    f.ws_bytes = f.off_codes + 64LL * bpt * (n + 2 * nch * (int64_t)f.ng) + 64;
    *cf = f;
    return true;
}

// Deterministic from (n, l, pad, es): the schedule and the kernel agree.
// Preferred geometry (measured on B200, tools/k1_sweep.py): two rows per
// block from 8 KB rows up (four below), stages of up to 64 KB (longer chunks
// = fewer idle lane-steps); smaller blocks/stages when the FWHT scratch of a
// long transform leaves no room.
static bool config(int64_t n, int64_t l, int64_t pad, int es, Cfg *cf) {
    if (getenv("SRLU_K1_NOSCHED") != nullptr) return false;
    if (pad < 32 || pad > 8192 || l < 1 || l > pad || n < 1) return false;
    const int64_t groups = ceil_div(l, 32);
    int bpt = 0;
    for (int b : {1, 2, 4, 5, 8})
        if ((int64_t)kGW * b >= groups) { bpt = b; break; }
    if (!bpt) return false;
    const int64_t row_bytes = n * es;
    const int rb_env = env_int("SRLU_K1_RB", 0);
    const int st_env = env_int("SRLU_K1_STAGE", 0);
    if (rb_env || st_env) {
        const int rb = rb_env ? rb_env : (row_bytes <= 8192 ? 4 : 2);
        if (rb != 1 && rb != 2 && rb != 4) return false;
        return config_try(n, l, pad, es, bpt, rb, st_env ? st_env : 65536, cf);
    }
    for (int rb = row_bytes <= 8192 ? 4 : 2; rb >= 1; rb >>= 1)
        for (int64_t st = 65536; st >= 16384; st >>= 1)
            if (config_try(n, l, pad, es, bpt, rb, st, cf) && cf->nch <= kMaxChunks) return true;
    // long rows (codes read from L2): one row per block, the widest chunks
    // (fewest idle lane-steps per chunk; measured at config 5: 64 KB stages
    // 13.9 ms, 32 KB 24 ms, 16 KB 43 ms, two-row blocks of 2048 columns 32 ms)
    return config_try(n, l, pad, es, bpt, 1, 65536, cf);
}

// warp w, slot b -> group (snake order over the slots)
__host__ __device__ inline int group_of(int w, int b) { return b * kGW + ((b & 1) ? kGW - 1 - w : w); }

// ---------------------------------------------------------------------------
// schedule construction

// slot -> bucket (-1 = empty lane).  sorted: buckets in descending order of
// their source count (stable), so that the 32 lanes of a group have similar
// queue lengths (fewer idle lane-steps); the snake map group_of() then pairs
// heavy and light groups in one warp.  Otherwise consecutive buckets.
// One CTA of 1024 threads: counting sort on min(count, 1023).
__global__ void __launch_bounds__(1024) group_kernel(const int32_t *__restrict__ bptr, int l,
                                                     int ng, int sorted, int32_t *grp) {
    __shared__ int hist[1024];
    __shared__ int cursor[1024];
    const int tid = threadIdx.x;
    for (int s = tid; s < ng * 32; s += blockDim.x) grp[s] = (!sorted && s < l) ? s : -1;
    if (!sorted) return;
    hist[tid] = 0;
    __syncthreads();
    for (int t = tid; t < l; t += blockDim.x) atomicAdd(&hist[1023 - min(bptr[t + 1] - bptr[t], 1023)], 1);
    __syncthreads();
    if (tid == 0) {  // exclusive scan (descending count = ascending key)
        int run = 0;
        for (int k = 0; k < 1024; ++k) {
            cursor[k] = run;
            run += hist[k];
        }
    }
    __syncthreads();
    // stable scatter: warp 0 walks the buckets in order, 32 at a time
    if (tid < 32) {
        const unsigned lt = (1u << tid) - 1u;
        for (int t0 = 0; t0 < l; t0 += 32) {
            const int t = t0 + tid;
            const bool ok = t < l;
            const int key = ok ? 1023 - min(bptr[t + 1] - bptr[t], 1023) : 1024 + tid;
            const unsigned peers = __match_any_sync(0xffffffffu, key);
            if (ok) {
                const int pos = cursor[key] + __popc(peers & lt);
                grp[pos] = t;
            }
            __syncwarp();
            if (ok && (peers & lt) == 0) cursor[key] += __popc(peers);
            __syncwarp();
        }
    }
}

// One warp per group simulates the walk of its 32 lanes chunk by chunk: in
// each step every pending lane proposes its next source; per bank (per
// half-warp bank pair for 8-byte elements) the D lanes with the longest
// remaining queue win, the others read a zero word in a bank nobody uses.
// PASS 0 counts step pairs per (chunk, group).  PASS 1 pads the slots of each
// warp to a common pair count per chunk and writes the codes at
// [chunk][warp][pair][slot][lane] (u32 = two 16-bit codes).
constexpr int kSchedListCap = 4096;  // staged source codes per group (ints)

// One pass of the simulation for group g (see sched_kernel).  src[0..cnt) =
// this lane's bucket sources (ascending, sign in bit 31).
// Two 16-bit step codes (column | sign << 15) as one word, laid out for a
// cheap decode in gather_pair: bits 2-16 column of the first step, bit 0 its
// sign, bit 1 the second step's sign, bits 17-31 its column.
__device__ __forceinline__ uint32_t pack_pair(uint32_t lo, uint32_t hi) {
    return ((lo & 0x7fffu) << 2) | (lo >> 15) | ((hi >> 15) << 1) | ((hi & 0x7fffu) << 17);
}

template <int PASS>
__device__ __forceinline__ void sched_pass(const int32_t *src, int cnt, int g, int c, int nch,
                                           int ch0, int ch1,
                                           int es8, int bpt, int d2, int joint, int32_t *np_tab,
                                           int32_t *wsched, uint32_t *codes, int32_t *header,
                                           unsigned *best, unsigned *best2) {
    const int lane = threadIdx.x;
    const int ng = kGW * bpt;
    const int b = g / kGW, w = (b & 1) ? kGW - 1 - (g % kGW) : (g % kGW);
    const unsigned FULL = 0xffffffffu;
    // chunks [ch0, ch1) of this group: the lane's first source at or beyond the
    // first chunk's first column (its list is ascending in the column)
    int cur = 0;
    if (ch0 > 0) {
        int lo = 0, hi = cnt;
        const int c_first = ch0 * c;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if ((src[mid] & 0x7fffffff) < c_first) lo = mid + 1; else hi = mid;
        }
        cur = lo;
    }
    int nxt = cur < cnt ? src[cur] : INT_MAX;
    auto joint_np = [&](int ch, int ww) {  // common pairs of warp ww in chunk ch
        int mx = 0;
        for (int bb = 0; bb < bpt; ++bb) mx = max(mx, np_tab[ch * ng + group_of(ww, bb)]);
        return mx;
    };
    for (int ch = ch0; ch < ch1; ++ch) {
        const int c0 = ch * c, c1 = c0 + c;
        uint32_t *out = nullptr;
        int npj = 0;
        int pstride = 32;  // words between consecutive pairs of this group
        if (PASS == 1 && joint) {
            // base of (ch, w): all (ch', w') before it in [chunk][warp] order
            const int idx = ch * kGW + w;
            int s = 0;
            for (int i = lane; i < idx; i += 32) s += joint_np(i / kGW, i % kGW);
#pragma unroll
            for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
            npj = joint_np(ch, w);
            const int base = s * bpt * 32;
            if (lane == 0 && b == 0) {
                wsched[2 * idx] = base;
                wsched[2 * idx + 1] = npj;
                if (idx == nch * kGW - 1) header[0] = base + npj * bpt * 32;
            }
            out = codes + base + b * 32 + lane;
            pstride = bpt * 32;
        } else if (PASS == 1) {
            // base of (ch, g): all (ch', g') before it in [chunk][group] order
            const int idx = ch * ng + g;
            int s = 0;
            for (int i = lane; i < idx; i += 32) s += np_tab[i];
#pragma unroll
            for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
            npj = np_tab[idx];
            const int base = s * 32;
            if (lane == 0) {
                wsched[2 * idx] = base;
                wsched[2 * idx + 1] = npj;
                if (idx == nch * ng - 1) header[0] = base + npj * 32;
            }
            out = codes + base + lane;
        }
        int step = 0;
        uint32_t pairw = 0;
        auto emit = [&](uint32_t code) {
            if (PASS == 1) {
                if (step & 1) out[(size_t)(step >> 1) * pstride] = pack_pair(pairw, code);
                else pairw = code;
            }
            ++step;
        };
        while (true) {
            const int col = nxt & 0x7fffffff;
            const bool pend = nxt != INT_MAX && col < c1;
            if (!__any_sync(FULL, pend)) break;
            const int lc = col - c0;
            const int key = es8 ? ((lc & 15) | (lane & 16)) : (lc & 31);
            const int rem = cnt - cur;
            const unsigned prio = ((unsigned)min(rem, 1 << 20) << 5) | (unsigned)(31 - lane);
            if (pend) atomicMax(&best[key], prio);
            __syncwarp();
            bool win = pend && best[key] == prio;
            if (d2 >= 2) {
                if (pend && !win) atomicMax(&best2[key], prio);
                __syncwarp();
                win = win || (pend && best2[key] == prio);
            }
            __syncwarp();
            if (pend) {
                best[key] = 0;
                best2[key] = 0;
            }
            const unsigned used = __reduce_or_sync(FULL, win ? (1u << key) : 0u);
            uint32_t code;
            if (win) {
                code = (uint32_t)lc | (nxt < 0 ? 0x8000u : 0u);
            } else {
                unsigned freem = ~used;
                if (es8) freem = (lane & 16) ? (freem >> 16) & 0xffffu : freem & 0xffffu;
                const int fk = __ffs((int)freem) - 1;  // exists: this lane did not win
                code = (uint32_t)(c + fk);             // a zero word in that bank
            }
            emit(code);
            if (win) {
                ++cur;
                nxt = cur < cnt ? src[cur] : INT_MAX;
            }
            __syncwarp();
        }
        // pad to the warp's common pair count with broadcast no-ops (every
        // lane reads the same zero word)
        const int target = PASS == 1 ? 2 * npj : step + (step & 1);
        while (step < target) emit((uint32_t)c);
        if (PASS == 0 && lane == 0) np_tab[ch * ng + g] = step >> 1;
    }
}

// One warp (CTA) per group simulates the walk of its 32 lanes chunk by
// chunk: in each step every pending lane proposes its next source; per bank
// (per half-warp bank pair for 8-byte elements) the D lanes with the longest
// remaining queue win, the others read a zero word in a bank nobody uses.
// Pass 0 counts step pairs per (chunk, group); after a grid barrier (cooperative
// launch) pass 1 lays the codes out: joint = the slots of each warp padded to
// a common pair count per chunk, [chunk][warp][pair][slot][lane]; otherwise
// [chunk][group][pair][lane].  u32 = two 16-bit codes.  The group's source
// lists are staged in shared memory when they fit.
__global__ void __launch_bounds__(32) sched_kernel(const int32_t *__restrict__ sorted,
                                                   const int32_t *__restrict__ bptr, int l, int c,
                                                   int nch, int es8, int bpt, int d2, int joint,
                                                   const int32_t *__restrict__ grp,
                                                   int32_t *np_tab, int32_t *wsched,
                                                   uint32_t *codes, int32_t *header,
                                                   unsigned *barrier, int cpb) {
    __shared__ unsigned best[32], best2[32];
    __shared__ int32_t lists[kSchedListCap];
    // one warp per (group, slice of cpb chunks): blockIdx.x = slice * ng + group
    const int ngrp = kGW * bpt;
    const int g = blockIdx.x % ngrp, lane = threadIdx.x;
    const int chq = (blockIdx.x / ngrp) * cpb, chr = min(nch, chq + cpb);
    const unsigned FULL = 0xffffffffu;
    const int t = grp ? grp[g * 32 + lane] : (g * 32 + lane < l ? g * 32 + lane : -1);
    const int beg = t >= 0 ? bptr[t] : 0;
    const int cnt = t >= 0 ? bptr[t + 1] - beg : 0;
    int off = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(FULL, off, o);
        if (lane >= o) off += v;
    }
    const int total = __shfl_sync(FULL, off, 31);
    off -= cnt;
    const bool staged = total <= kSchedListCap;
    if (staged) {
        for (int j = 0; j < 32; ++j) {
            const int bj = __shfl_sync(FULL, beg, j), nj = __shfl_sync(FULL, cnt, j);
            const int oj = __shfl_sync(FULL, off, j);
            for (int i = lane; i < nj; i += 32) lists[oj + i] = __ldg(sorted + bj + i);
        }
    }
    best[lane] = 0;
    best2[lane] = 0;
    __syncwarp();
    const int32_t *src = staged ? lists + off : sorted + beg;
    sched_pass<0>(src, cnt, g, c, nch, chq, chr, es8, bpt, d2, joint, np_tab, wsched, codes, header, best,
                  best2);
    grid_arrive_wait(barrier, gridDim.x);
    sched_pass<1>(src, cnt, g, c, nch, chq, chr, es8, bpt, d2, joint, np_tab, wsched, codes, header, best,
                  best2);
}

// ---------------------------------------------------------------------------
// the sketch kernel

struct Dev {
    int c, nch, ns, ng, dbg, pf, sorted, joint, xpad;
    int row_stride, stage_bytes;
    int xs_off, code_off, code_cap;
};

__device__ __forceinline__ void named_bar(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// One element: the sign bit (bit 31 of smask) goes into the element's own
// sign bit before the widening (exact), then acc + v — bit-identical to the
// reference's out += s * a.
template <typename T>
__device__ __forceinline__ double signed_elem(const unsigned char *p, uint32_t smask) {
    if (sizeof(T) == 4) {
        const uint32_t f = *reinterpret_cast<const uint32_t *>(p) ^ (smask & 0x80000000u);
        return (double)__uint_as_float(f);
    } else {
        const uint2 d = *reinterpret_cast<const uint2 *>(p);
        return __hiloint2double((int)(d.y ^ (smask & 0x80000000u)), (int)d.x);
    }
}

// Two consecutive steps of one lane from a pack_pair word (first step first).
template <typename T, int RB>
__device__ __forceinline__ void gather_pair(const unsigned char *st, int row_stride, uint32_t w,
                                            double (&acc)[RB]) {
    const uint32_t off0 = sizeof(T) == 4 ? (w & 0x1fffcu) : ((w << 1) & 0x3fff8u);
    const uint32_t off1 = sizeof(T) == 4 ? ((w >> 15) & 0x1fffcu) : ((w >> 14) & 0x3fff8u);
    const uint32_t m0 = w << 31, m1 = w << 30;
    const unsigned char *p0 = st + off0, *p1 = st + off1;
    double v0[RB], v1[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        v0[r] = signed_elem<T>(p0 + r * row_stride, m0);
        v1[r] = signed_elem<T>(p1 + r * row_stride, m1);
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) acc[r] = __dadd_rn(__dadd_rn(acc[r], v0[r]), v1[r]);
}

// One gather warp's stream: per row block, per chunk, the warp's joint
// schedule (all BPT slots step together); then +-phase, the FWHT stages
// h < 32 by shuffles (slot g*32 + lane holds bucket g*32 + lane, zero if
// empty) and the hand-off of the block to the epilogue warps.
template <typename T, int RB, int BPT, typename Codes, typename Issue>
__device__ __forceinline__ void gather_warp(unsigned char *smem, Codes cw,
                                            const int32_t *__restrict__ grp,
                                            const int2 *__restrict__ wsched,
                                            const double *__restrict__ phase, const Dev &d,
                                            int64_t my_nrb, int64_t nitems, uint64_t *full,
                                            uint64_t *xs_full, uint64_t *xs_empty, unsigned *rel,
                                            double *xs_base, int xpad, int l, const Issue &issue) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int bt[BPT];
    bool bneg[BPT];
#pragma unroll
    for (int b = 0; b < BPT; ++b) {
        const int slot = group_of(warp, b) * 32 + lane;
        bt[b] = d.sorted ? grp[slot] : (slot < l ? slot : -1);
        bneg[b] = bt[b] >= 0 && phase[bt[b]] < 0.0;
    }
    int stage = 0;
    unsigned ph = 0;
    int64_t it = 0;
    for (int64_t rbi = 0; rbi < my_nrb; ++rbi) {
        double acc[BPT][RB];
#pragma unroll
        for (int b = 0; b < BPT; ++b)
#pragma unroll
            for (int r = 0; r < RB; ++r) acc[b][r] = 0.0;
        for (int ch = 0; ch < d.nch; ++ch, ++it) {
            if (!(d.dbg & 8)) mbar_wait_suspend(&full[stage], ph);
            // the stage base as one opaque shared address (keeps the compiler
            // from re-deriving smem + stage * bytes for every code)
            uint32_t stb = smem_u32(smem + stage * d.stage_bytes);
            asm volatile("" : "+r"(stb));
            const unsigned char *st = (const unsigned char *)__cvta_shared_to_generic(stb);
            if (BPT == 1 || d.joint) {
                const int2 sc = __ldg(wsched + ch * kGW + warp);
                const int np = sc.y;
                const int base = sc.x + lane;
#pragma unroll(BPT == 1 ? 4 : (BPT == 2 ? 2 : 1))
                for (int s2 = 0; s2 < np; ++s2) {
#pragma unroll
                    for (int b = 0; b < BPT; ++b) {
                        const uint32_t w = cw[base + (s2 * BPT + b) * 32];
                        gather_pair<T, RB>(st, d.row_stride, w, acc[b]);
                    }
                }
            } else {
#pragma unroll
                for (int b = 0; b < BPT; ++b) {
                    const int2 sc = __ldg(wsched + ch * d.ng + group_of(warp, b));
                    const int np = sc.y;
                    const int base = sc.x + lane;
#pragma unroll 4
                    for (int s2 = 0; s2 < np; ++s2) {
                        const uint32_t w = cw[base + s2 * 32];
                        gather_pair<T, RB>(st, d.row_stride, w, acc[b]);
                    }
                }
            }
            // release the stage; the last of the kGW warps refills it
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                const unsigned old = atomicAdd(&rel[stage], 1u);
                if ((old + 1) % kGW == 0 && it + d.ns < nitems && !(d.dbg & 8)) {
                    fence_proxy_async_smem();
                    issue(it + d.ns, stage);
                }
            }
            if (++stage == d.ns) {
                stage = 0;
                ph ^= 1u;
            }
        }
        const int buf = (int)(rbi & 1);
        if (rbi >= 2) {
            const unsigned par = (unsigned)(((rbi >> 1) - 1) & 1);
            if (d.dbg & 32) mbar_wait_sleep(&xs_empty[buf], par, 256);
            else mbar_wait_suspend(&xs_empty[buf], par);
        }
        double *xs = xs_base + (size_t)buf * RB * xpad;
        // +-phase, scatter by bucket, then (after all gather warps wrote) the
        // FWHT stages h < 32 by shuffles on 32-aligned blocks of buckets;
        // positions >= l (no bucket) enter as zeros
        if (d.sorted) {
#pragma unroll
            for (int b = 0; b < BPT; ++b) {
                if (bt[b] >= 0) {
                    const int pos = fwht_sw(bt[b]);
#pragma unroll
                    for (int r = 0; r < RB; ++r)
                        xs[r * xpad + pos] = bneg[b] ? -acc[b][r] : acc[b][r];
                }
            }
            named_bar(2, kGW * 32);
            for (int q = warp; q * 32 < l; q += kGW) {
                const int pos = fwht_sw(q * 32 + lane);
                const bool live = q * 32 + lane < l;
#pragma unroll
                for (int r = 0; r < RB; ++r)
                    xs[r * xpad + pos] = fwht_lane_stages(live ? xs[r * xpad + pos] : 0.0, lane);
            }
        } else {
            // consecutive buckets: slot g*32 + lane holds bucket g*32 + lane
#pragma unroll
            for (int b = 0; b < BPT; ++b) {
                const int g = group_of(warp, b);
                const int pos = fwht_sw(g * 32 + lane);
#pragma unroll
                for (int r = 0; r < RB; ++r) {
                    const double v = fwht_lane_stages(bneg[b] ? -acc[b][r] : acc[b][r], lane);
                    if (g * 32 < xpad) xs[r * xpad + pos] = v;
                }
            }
        }
        mbar_arrive(&xs_full[buf]);
    }
}

template <typename T, int RB, int BPT>
__global__ void __launch_bounds__(kNT, 1) k1s_kernel(
    const T *__restrict__ a, int64_t m, int64_t n, int64_t lda, const unsigned char *__restrict__ ws,
    int64_t off_grp, int64_t off_wsched, int64_t off_codes, int l, const double *__restrict__ phase,
    const int32_t *__restrict__ idx, int k, int pad, double mult, double *__restrict__ y,
    int64_t ldy, int *nonfinite, Dev d) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t full[kMaxStages];
    __shared__ __align__(8) uint64_t xs_full[2], xs_empty[2];
    __shared__ unsigned rel[kMaxStages];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int es = (int)sizeof(T);
    const int64_t nrb = ceil_div(m, RB);
    const int64_t my_nrb = (int64_t)blockIdx.x < nrb ? ceil_div(nrb - blockIdx.x, gridDim.x) : 0;
    const int64_t nitems = my_nrb * d.nch;
    const int32_t *grp = reinterpret_cast<const int32_t *>(ws + off_grp);
    const int2 *wsched = reinterpret_cast<const int2 *>(ws + off_wsched);
    const uint32_t *codes_g = reinterpret_cast<const uint32_t *>(ws + off_codes);
    const int total_words = reinterpret_cast<const int32_t *>(ws)[0];
    double *xs_base = reinterpret_cast<double *>(smem + d.xs_off);
    uint32_t *codes_s = reinterpret_cast<uint32_t *>(smem + d.code_off);
    const bool codes_in_smem = (int64_t)total_words * 4 <= d.code_cap && !(d.dbg & 4);

    if (tid == 0) {
        for (int s = 0; s < d.ns; ++s) mbar_init(&full[s], 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&xs_full[b], kGW * 32);
            mbar_init(&xs_empty[b], (kNT / 32 - kGW) * 32);
        }
        fence_mbar_init();
    }
    if (tid < kMaxStages) rel[tid] = 0;
    // zero tails of every staged row (never written by the bulk copies)
    {
        const int zw = kZeroBytes / 4;
        for (int i = tid; i < d.ns * RB * zw; i += kNT) {
            const int sr = i / zw, w = i % zw;
            reinterpret_cast<uint32_t *>(smem + (size_t)sr * d.row_stride + (size_t)d.c * es)[w] = 0u;
        }
    }
    const int xpad = d.xpad;
    for (int i = tid; i < 2 * RB * xpad; i += kNT) xs_base[i] = 0.0;
    if (codes_in_smem) {
        const uint4 *src = reinterpret_cast<const uint4 *>(codes_g);
        uint4 *dst = reinterpret_cast<uint4 *>(codes_s);
        const int nv = (total_words + 3) / 4;
        for (int i = tid; i < nv; i += kNT) dst[i] = __ldg(src + i);
    }
    __syncthreads();

    uint64_t *fullp = full;
    const int nch = d.nch, cc = d.c, sbytes = d.stage_bytes, rstride = d.row_stride;
    const int64_t bid = blockIdx.x, gdim = gridDim.x;
    const int pf = d.pf;
    // item it -> (rows, column range) of A; PF > 0: also prefetch item it + PF
    // into L2 so that the ring's bulk copies hit L2 (keeps more HBM bytes in
    // flight than the shared-memory ring holds)
    auto prefetch = [=](int64_t it) {
        if (it >= nitems) return;
        const int64_t rbi = it / nch;
        const int ch = (int)(it - rbi * nch);
        const int64_t row0 = (bid + rbi * gdim) * RB;
        const int nrows = (int)min((int64_t)RB, m - row0);
        const int64_t c0 = (int64_t)ch * cc;
        const unsigned bytes = (unsigned)min((int64_t)cc, n - c0) * es;
        for (int r = 0; r < nrows; ++r) bulk_prefetch_l2(a + (row0 + r) * lda + c0, bytes);
    };
    auto issue = [=](int64_t it, int stage) {
        const int64_t rbi = it / nch;
        const int ch = (int)(it - rbi * nch);
        const int64_t row0 = (bid + rbi * gdim) * RB;
        const int nrows = (int)min((int64_t)RB, m - row0);
        const int64_t c0 = (int64_t)ch * cc;
        const int cols = (int)min((int64_t)cc, n - c0);
        const unsigned bytes = (unsigned)cols * es;
        unsigned char *st = smem + (size_t)stage * sbytes;
        mbar_arrive_expect_tx(&fullp[stage], bytes * nrows);
        for (int r = 0; r < nrows; ++r)
            bulk_g2s(st + (size_t)r * rstride, a + (row0 + r) * lda + c0, bytes, &fullp[stage]);
        if (pf > 0) prefetch(it + pf);
    };
    if (tid == 0 && !(d.dbg & 16)) {
        for (int64_t it = d.ns; pf > 0 && it < d.ns + pf - 1; ++it) prefetch(it);
        for (int64_t it = 0; it < d.ns && it < nitems; ++it) issue(it, (int)it);
    }

    if (warp < kGW) {
        if (codes_in_smem)
            gather_warp<T, RB, BPT>(smem, codes_s, grp, wsched, phase, d, my_nrb, nitems, full,
                                    xs_full, xs_empty, rel, xs_base, xpad, l, issue);
        else
            gather_warp<T, RB, BPT>(smem, codes_g, grp, wsched, phase, d, my_nrb, nitems, full,
                                    xs_full, xs_empty, rel, xs_base, xpad, l, issue);
        return;
    }
    // ---------------------------------------------------------------- epilogue
    constexpr int kEW = kNT / 32 - kGW;
    const int ew = warp - kGW, etid = tid - kGW * 32;
    const int bsize = pad < 512 ? pad : 512;
    const int nb = pad / bsize;
    const int nzb = (l + bsize - 1) / bsize;
    bool bad = false;
    for (int64_t rbi = 0; rbi < my_nrb; ++rbi) {
        const int buf = (int)(rbi & 1);
        if (d.dbg & 32) mbar_wait_sleep(&xs_full[buf], (unsigned)((rbi >> 1) & 1), 32);
        else mbar_wait_suspend(&xs_full[buf], (unsigned)((rbi >> 1) & 1));
        double *xs = xs_base + (size_t)buf * RB * xpad;
        // stages 32 <= h < bsize (the gather warps applied h < 32)
        for (int item = ew; !(d.dbg & 1) && item < RB * nzb; item += kEW) {
            const int r = item / nzb, bb = item % nzb;
            fwht_block_warp_hi_dyn512(xs + (size_t)r * xpad + (size_t)bb * bsize, bsize, lane);
        }
        named_bar(1, kEW * 32);
        // output-pruned stages h >= bsize for the k sampled outputs only
        const int64_t row0 = ((int64_t)blockIdx.x + rbi * gridDim.x) * RB;
        const int nrows = (int)min((int64_t)RB, m - row0);
        for (int kk = etid; !(d.dbg & 2) && kk < k; kk += kEW * 32) {
            const int q = idx[kk];
            const int o = fwht_sw(q & (bsize - 1)), B = q / bsize;
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                if (r < nrows) {
                    const double *row = xs + (size_t)r * xpad;
                    double f;
                    switch (nb) {
                        case 1: f = row[o]; break;
                        case 2: f = wht_pick<2>(row, bsize, o, B, nzb); break;
                        case 4: f = wht_pick<4>(row, bsize, o, B, nzb); break;
                        case 8: f = wht_pick<8>(row, bsize, o, B, nzb); break;
                        default: f = wht_pick<16>(row, bsize, o, B, nzb); break;
                    }
                    const double v = __dmul_rn(f, mult);
                    y[(row0 + r) * ldy + kk] = v;
                    bad |= !isfinite(v);
                }
            }
        }
        named_bar(1, kEW * 32);
        // positions in [ng*32, nzb*bsize) are not rewritten by the gather
        // warps but were transformed in place: re-zero them
        const int z0 = d.sorted ? (l + 31) / 32 * 32 : d.ng * 32, z1 = nzb * bsize;
        for (int i = etid; z1 > z0 && i < RB * (z1 - z0); i += kEW * 32) {
            const int r = i / (z1 - z0), t = z0 + i % (z1 - z0);
            xs[(size_t)r * xpad + fwht_sw(t)] = 0.0;
        }
        mbar_arrive(&xs_empty[buf]);
    }
    if (bad) atomicOr(nonfinite, 1);
}

template <typename T, int RB, int BPT>
static int launch(const Cfg &f, const T *a, int64_t m, int64_t n, int64_t lda,
                  const unsigned char *ws, int64_t l, const double *phase, const int32_t *idx,
                  int64_t k, int64_t pad, double mult, double *y, int64_t ldy, int *nonfinite,
                  cudaStream_t s) {
    Dev d;
    d.c = f.c; d.nch = f.nch; d.ns = f.ns; d.ng = f.ng;
    d.sorted = f.sorted; d.joint = f.joint; d.xpad = f.xpad;
    d.pf = env_int("SRLU_K1_PF", 0);  // L2 prefetch distance in ring items (measured: no gain)
    d.dbg = env_int("SRLU_K1_DBG", 0);  // experiments: 1 no FWHT, 2 no outputs, 8 no waits, 32 sleep-polling hand-off waits
    d.row_stride = (int)f.row_stride; d.stage_bytes = (int)f.stage_bytes;
    d.xs_off = (int)(f.ns * f.stage_bytes);
    d.code_off = (int)(d.xs_off + f.xs_bytes);
    d.code_cap = (int)f.code_cap;
    auto kern = k1s_kernel<T, RB, BPT>;
    // host time matters here (the stage-1 prologue is host-bound): the
    // attribute is set again only when the size changes, the SM count once
    static int64_t smem_set = -1;   // per kernel variant
    if (smem_set != f.smem) {
        SRLU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f.smem));
        smem_set = f.smem;
    }
    const int sms = device_sms();
    const int64_t nrb = ceil_div(m, RB);
    const unsigned grid = (unsigned)(nrb < sms ? nrb : sms);
    kern<<<grid, kNT, (size_t)f.smem, s>>>(a, m, n, lda, ws, f.off_grp, f.off_wsched,
                                           f.off_codes, (int)l, phase, idx, (int)k, (int)pad,
                                           mult, y, ldy, nonfinite, d);
    SRLU_CHECK_LAUNCH("k1s_kernel");
    return SRLU_OK;
}

template <typename T>
static int dispatch(const Cfg &f, const T *a, int64_t m, int64_t n, int64_t lda,
                    const unsigned char *ws, int64_t l, const double *phase, const int32_t *idx,
                    int64_t k, int64_t pad, double mult, double *y, int64_t ldy, int *nonfinite,
                    cudaStream_t s) {
#define K1S_CASE(RB_, BPT_)                                                                   \
    if (f.rb == RB_ && f.bpt == BPT_)                                                         \
        return launch<T, RB_, BPT_>(f, a, m, n, lda, ws, l, phase, idx, k, pad, mult, y, ldy, \
                                    nonfinite, s);
    K1S_CASE(1, 1) K1S_CASE(1, 2) K1S_CASE(1, 4)
    K1S_CASE(2, 1) K1S_CASE(2, 2) K1S_CASE(2, 4)
    K1S_CASE(4, 1) K1S_CASE(4, 2) K1S_CASE(4, 4)
    K1S_CASE(1, 5) K1S_CASE(2, 5) K1S_CASE(1, 8) K1S_CASE(2, 8)
#undef K1S_CASE
    set_error("sketch_right_dense_sched: no kernel for rb=%d bpt=%d", f.rb, f.bpt);
    return SRLU_ERR_UNSUPPORTED;
}

}  // namespace k1s
}  // namespace srlu

using namespace srlu;

static int es_of(int dtype) { return dtype == SRLU_F32 ? 4 : (dtype == SRLU_F64 ? 8 : 0); }

// sketch_right_tmem.cu: the TMEM-accumulator kernel takes over whenever its
// geometry applies (128 <= pad1 <= 1024); same plan buffer protocol
size_t srlu_k1t_plan_bytes(int64_t n, int64_t l1, int64_t pad1, int es);
int srlu_k1t_info(int64_t n, int64_t l1, int64_t pad1, int es, int64_t info[8]);
int srlu_k1t_plan(const int32_t *sorted1, const int32_t *bptr1, int64_t n, int64_t l1,
                  int64_t pad1, int es, void *plan, size_t plan_bytes, cudaStream_t s);
int srlu_k1t_run(const void *a, int es, int64_t m, int64_t n, int64_t lda, const void *plan,
                 size_t plan_bytes, int64_t l1, const double *phase1, const int32_t *idx1,
                 int64_t k1, int64_t pad1, double mult1, double *y, int64_t ldy, int *nonfinite,
                 cudaStream_t s);

extern "C" size_t srlu_k1_schedule_bytes(int64_t n, int64_t l1, int64_t pad1, int dtype) {
    const int es = es_of(dtype);
    k1s::Cfg f;
    if (es) {
        const size_t tb = srlu_k1t_plan_bytes(n, l1, pad1, es);
        if (tb) return tb;
    }
    if (!es || !k1s::config(n, l1, pad1, es, &f)) return 0;
    return (size_t)f.ws_bytes;
}

extern "C" int srlu_k1_config(int64_t n, int64_t l1, int64_t pad1, int dtype, int64_t info[8]) {
    const int es = es_of(dtype);
    k1s::Cfg f;
    SRLU_REQUIRE(info != nullptr, SRLU_ERR_ARG, "k1_config: null info");
    if (es && srlu_k1t_info(n, l1, pad1, es, info) == SRLU_OK) return SRLU_OK;
    if (!es || !k1s::config(n, l1, pad1, es, &f)) {
        for (int i = 0; i < 8; ++i) info[i] = 0;
        return SRLU_ERR_UNSUPPORTED;
    }
    info[0] = f.rb; info[1] = f.bpt; info[2] = f.c; info[3] = f.nch;
    info[4] = f.ns; info[5] = f.code_cap; info[6] = f.smem; info[7] = f.d2;
    return SRLU_OK;
}

extern "C" int srlu_k1_schedule(const int32_t *sorted1, const int32_t *bptr1, int64_t n,
                                int64_t l1, int64_t pad1, int dtype, void *sched,
                                size_t sched_bytes, srlu_stream_t stream) {
    const int es = es_of(dtype);
    k1s::Cfg f;
    if (es && srlu_k1t_plan_bytes(n, l1, pad1, es))
        return srlu_k1t_plan(sorted1, bptr1, n, l1, pad1, es, sched, sched_bytes,
                             (cudaStream_t)stream);
    SRLU_REQUIRE(es && k1s::config(n, l1, pad1, es, &f), SRLU_ERR_UNSUPPORTED,
                 "k1_schedule: shape not supported by the scheduled kernel");
    SRLU_REQUIRE(sched_bytes >= (size_t)f.ws_bytes, SRLU_ERR_WORKSPACE,
                 "k1_schedule: buffer too small");
    cudaStream_t s = (cudaStream_t)stream;
    unsigned char *ws = (unsigned char *)sched;
    int32_t *header = (int32_t *)ws;
    int32_t *grp = (int32_t *)(ws + f.off_grp);
    int32_t *np = (int32_t *)(ws + f.off_np);
    int32_t *wsc = (int32_t *)(ws + f.off_wsched);
    uint32_t *codes = (uint32_t *)(ws + f.off_codes);
    if (f.sorted) {
        k1s::group_kernel<<<1, 1024, 0, s>>>(bptr1, (int)l1, f.ng, f.sorted, grp);
        SRLU_CHECK_LAUNCH("k1s_group_kernel");
    }
    SRLU_CUDA(cudaMemsetAsync(header, 0, k1s::kHeader * sizeof(int32_t), s));
    const int32_t *grp_arg = f.sorted ? grp : nullptr;
    int l_arg = (int)l1, c_arg = f.c, nch_arg = f.nch, es8 = es == 8, bpt_arg = f.bpt,
        d2_arg = f.d2, joint_arg = f.joint;
    unsigned *bar = (unsigned *)(header + 1);
    // one warp per (group, slice of chunks): the simulation of a chunk only
    // needs each lane's cursor at the chunk's first column (binary search),
    // so the chunks of a group run in parallel — as many as stay co-resident
    // (cooperative launch; config 2: 28 x 2 warps, 31 -> 17 us)
    static int per_sm = 0;   // queried once
    const int sms = k1s::device_sms();
    if (per_sm == 0)
        SRLU_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k1s::sched_kernel, 32, 0));
    int cpb = 1;
    while ((int64_t)f.ng * ceil_div(f.nch, cpb) > (int64_t)per_sm * sms && cpb < f.nch) ++cpb;
    const int nslices = (int)ceil_div(f.nch, cpb);
    void *args[] = {(void *)&sorted1, (void *)&bptr1, &l_arg,   &c_arg, &nch_arg, &es8,
                    &bpt_arg,         &d2_arg,        &joint_arg, (void *)&grp_arg, &np,
                    &wsc,             &codes,         &header,  &bar, &cpb};
    SRLU_CUDA(cudaLaunchCooperativeKernel((const void *)k1s::sched_kernel, dim3(f.ng * nslices),
                                          dim3(32), args, 0, s));
    SRLU_CHECK_LAUNCH("k1s_sched_kernel");
    return SRLU_OK;
}

extern "C" int srlu_sketch_right_dense_sched(const void *a, int dtype, int64_t m, int64_t n,
                                             int64_t lda, const void *sched, size_t sched_bytes,
                                             int64_t l1, const double *phase1, const int32_t *idx1,
                                             int64_t k1, int64_t pad1, double mult1, double *y,
                                             int64_t ldy, int *nonfinite, srlu_stream_t stream) {
    const int es = es_of(dtype);
    k1s::Cfg f;
    SRLU_REQUIRE(m >= 1 && n >= 1 && lda >= n && l1 >= 1 && l1 <= n && k1 >= 1 && k1 <= pad1 &&
                     ldy >= k1,
                 SRLU_ERR_ARG, "sketch_right_dense_sched: bad sizes");
    if (es && srlu_k1t_plan_bytes(n, l1, pad1, es)) {
        SRLU_REQUIRE((uintptr_t)a % 16 == 0 && (lda * es) % 16 == 0, SRLU_ERR_UNSUPPORTED,
                     "sketch_right_dense_sched: A must be 16-byte aligned with 16-byte row pitch");
        return srlu_k1t_run(a, es, m, n, lda, sched, sched_bytes, l1, phase1, idx1, k1, pad1, mult1,
                            y, ldy, nonfinite, (cudaStream_t)stream);
    }
    SRLU_REQUIRE(es && k1s::config(n, l1, pad1, es, &f), SRLU_ERR_UNSUPPORTED,
                 "sketch_right_dense_sched: shape not supported by the scheduled kernel");
    SRLU_REQUIRE(sched_bytes >= (size_t)f.ws_bytes, SRLU_ERR_WORKSPACE,
                 "sketch_right_dense_sched: schedule buffer too small");
    SRLU_REQUIRE((uintptr_t)a % 16 == 0 && (lda * es) % 16 == 0 && (n * es) % 16 == 0,
                 SRLU_ERR_UNSUPPORTED,
                 "sketch_right_dense_sched: A must be 16-byte aligned with 16-byte row pitch");
    cudaStream_t s = (cudaStream_t)stream;
    const unsigned char *ws = (const unsigned char *)sched;
    if (dtype == SRLU_F32)
        return k1s::dispatch<float>(f, (const float *)a, m, n, lda, ws, l1, phase1, idx1, k1, pad1,
                                    mult1, y, ldy, nonfinite, s);
    return k1s::dispatch<double>(f, (const double *)a, m, n, lda, ws, l1, phase1, idx1, k1, pad1,
                                 mult1, y, ldy, nonfinite, s);
}
