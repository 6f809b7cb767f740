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
//   * a ring of kNS stages of RB rows x C columns, filled by 1-D bulk
//     copies (cp.async.bulk + mbarrier); the last gather warp to release a
//     stage refills it (no CTA-wide barrier in the stream);
//   * 28 gather warps: fp64 register accumulators acc[BPT][RB], persisting
//     across the chunks of a row block; then +-phase into a double-buffered
//     FWHT scratch (mbarrier hand-off);
//   * 4 epilogue warps: register FWHT per 512-point block, output-pruned
//     cross-block stages, x mult, Y write, non-finite flag — overlapping the
//     gathers of the next row block.
#include <limits.h>
#include <stdlib.h>

#include "fwht_warp.cuh"
#include "tma.cuh"

namespace srlu {

namespace k1s {

constexpr int kGW = 28;                 // gather warps
constexpr int kEW = 4;                  // epilogue warps
constexpr int kNT = (kGW + kEW) * 32;   // 1024 threads
constexpr int kMaxChunks = 4;
constexpr int kMaxStages = 8;
constexpr int kZeroBytes = 128;         // zero tail per staged row: one word per bank
constexpr size_t kSmemMax = 232448 - 1024;
constexpr int kHeader = 16;             // int32 header words

struct Cfg {
    int es, rb, bpt, c, nch, ns, ng, zpad;
    int64_t stage_bytes, row_stride, xs_bytes, code_cap, smem;
    // workspace offsets (bytes)
    int64_t off_grp, off_np, off_sched, off_codes, ws_bytes;
};

static int env_int(const char *name, int dflt) {
    const char *s = getenv(name);
    return (s && *s) ? atoi(s) : dflt;
}

// Deterministic from (n, l, pad, es): the schedule and the kernel agree.
static bool config(int64_t n, int64_t l, int64_t pad, int es, Cfg *cf) {
    if (getenv("SRLU_K1_NOSCHED") != nullptr) return false;
    if (pad < 32 || pad > 8192 || l < 1 || l > pad || n < 1) return false;
    const int64_t groups = ceil_div(l, 32);
    int bpt = 0;
    for (int b : {1, 2, 4})
        if ((int64_t)kGW * b >= groups) { bpt = b; break; }
    if (!bpt) return false;
    const int64_t row_bytes = n * es;
    int rb = env_int("SRLU_K1_RB", row_bytes <= 8192 ? 4 : (row_bytes <= 16384 ? 2 : 1));
    if (rb != 1 && rb != 2 && rb != 4) return false;
    const int64_t stage_target = env_int("SRLU_K1_STAGE", 32768);
    int64_t cmax = stage_target / (rb * es);
    cmax &= ~31LL;
    if (cmax < 32) return false;
    int64_t nch = ceil_div(n, cmax);
    if (nch > kMaxChunks) return false;
    int64_t c = ((ceil_div(n, nch) + 31) / 32) * 32;
    if (c + kZeroBytes / es > 32767) return false;
    Cfg f{};
    f.es = es; f.rb = rb; f.bpt = bpt; f.c = (int)c; f.nch = (int)nch;
    f.ng = kGW * bpt; f.zpad = kZeroBytes / es;
    f.row_stride = (c + f.zpad) * es;
    f.stage_bytes = rb * f.row_stride;
    f.xs_bytes = 2LL * rb * pad * 8;
    int ns = env_int("SRLU_K1_NS", 4);
    if (ns < 2) ns = 2;
    if (ns > kMaxStages) ns = kMaxStages;
    while (ns > 2 && (size_t)(ns * f.stage_bytes + f.xs_bytes + 16384) > kSmemMax) --ns;
    f.ns = ns;
    int64_t used = ns * f.stage_bytes + f.xs_bytes;
    if ((size_t)used + 4096 > kSmemMax) return false;
    f.code_cap = ((int64_t)kSmemMax - used) & ~15LL;
    f.smem = used + f.code_cap;
    // workspace: header | grp_bucket[ng*32] | np[nch*ng] | sched[nch*ng*2] | codes
    auto al = [](int64_t v) { return (v + 15) & ~15LL; };
    f.off_grp = al(kHeader * 4);
    f.off_np = al(f.off_grp + (int64_t)f.ng * 32 * 4);
    f.off_sched = al(f.off_np + (int64_t)nch * f.ng * 4);
    f.off_codes = al(f.off_sched + (int64_t)nch * f.ng * 8);
    // every step advances >= 1 source; + one odd-padding step per (chunk, group)
    f.ws_bytes = f.off_codes + 64 * (n + 2 * nch * (int64_t)f.ng) + 64;
    *cf = f;
    return true;
}

// ---------------------------------------------------------------------------
// schedule construction

// slot -> bucket (identity grouping of consecutive buckets; -1 = empty lane)
__global__ void group_kernel(int l, int ng, int32_t *grp) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < ng * 32; s += gridDim.x * blockDim.x)
        grp[s] = s < l ? s : -1;
}

// One warp per group simulates the walk of its 32 lanes chunk by chunk.
// PASS 0 counts steps (np = step pairs per (chunk, group)); PASS 1 recomputes
// the layout offsets (chunk-major, then group) and writes the codes.
template <int PASS>
__global__ void __launch_bounds__(32) sched_kernel(const int32_t *__restrict__ sorted,
                                                   const int32_t *__restrict__ bptr, int c,
                                                   int nch, int es8, int ng,
                                                   const int32_t *__restrict__ grp,
                                                   int32_t *np_tab, int32_t *sched,
                                                   uint32_t *codes, int32_t *header) {
    __shared__ unsigned best[32];
    const int g = blockIdx.x, lane = threadIdx.x;
    const unsigned FULL = 0xffffffffu;
    const int t = grp[g * 32 + lane];
    int cur = t >= 0 ? bptr[t] : 0;
    const int end = t >= 0 ? bptr[t + 1] : 0;
    int nxt = cur < end ? sorted[cur] : INT_MAX;
    best[lane] = 0;
    __syncwarp();
    for (int ch = 0; ch < nch; ++ch) {
        const int c0 = ch * c, c1 = c0 + c;
        const int idx = ch * ng + g;
        uint32_t *out = nullptr;
        if (PASS == 1) {
            int s = 0;
            for (int i = lane; i < idx; i += 32) s += np_tab[i];
#pragma unroll
            for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
            const int base = s * 32;
            if (lane == 0) {
                sched[2 * idx] = base;
                sched[2 * idx + 1] = np_tab[idx];
                if (idx == nch * ng - 1) header[0] = base + np_tab[idx] * 32;
            }
            out = codes + base;
        }
        int step = 0;
        uint32_t pairw = 0;
        while (true) {
            const int col = nxt & 0x7fffffff;
            const bool pend = nxt != INT_MAX && col < c1;
            if (!__any_sync(FULL, pend)) break;
            const int lc = col - c0;
            const int key = es8 ? ((lc & 15) | (lane & 16)) : (lc & 31);
            const int rem = end - cur;
            const unsigned prio = ((unsigned)min(rem, 1 << 20) << 5) | (unsigned)(31 - lane);
            if (pend) atomicMax(&best[key], prio);
            __syncwarp();
            const bool win = pend && best[key] == prio;
            __syncwarp();
            if (pend) best[key] = 0;
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
            if (PASS == 1) {
                if (step & 1) out[(step >> 1) * 32 + lane] = pairw | (code << 16);
                else pairw = code;
            }
            if (win) {
                ++cur;
                nxt = cur < end ? __ldg(sorted + cur) : INT_MAX;
            }
            __syncwarp();
            ++step;
        }
        if (step & 1) {  // pad the pair with a broadcast no-op (same zero word for all lanes)
            if (PASS == 1) out[(step >> 1) * 32 + lane] = pairw | ((uint32_t)c << 16);
            ++step;
        }
        if (PASS == 0 && lane == 0) np_tab[idx] = step >> 1;
    }
}

// ---------------------------------------------------------------------------
// the sketch kernel

struct Dev {
    int c, nch, ns, ng;
    int row_stride, stage_bytes;
    int xs_off, code_off, code_cap;
};

__device__ __forceinline__ void named_bar(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <typename T, int RB>
__device__ __forceinline__ void gather_step(const unsigned char *st, int row_stride, uint32_t c,
                                            double (&acc)[RB]) {
    const uint32_t col = c & 0x7fffu;
    const uint32_t sg = (c & 0x8000u) << 16;
    const unsigned char *p = st + col * sizeof(T);
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        if constexpr (sizeof(T) == 4) {
            const uint32_t bits = *reinterpret_cast<const uint32_t *>(p + r * row_stride) ^ sg;
            acc[r] = __dadd_rn(acc[r], (double)__uint_as_float(bits));
        } else {
            const uint2 bits = *reinterpret_cast<const uint2 *>(p + r * row_stride);
            acc[r] = __dadd_rn(acc[r], __hiloint2double((int)(bits.y ^ sg), (int)bits.x));
        }
    }
}

template <typename T, int RB, int BPT>
__global__ void __launch_bounds__(kNT, 1) k1s_kernel(
    const T *__restrict__ a, int64_t m, int64_t n, int64_t lda, const unsigned char *__restrict__ ws,
    int64_t off_grp, int64_t off_sched, int64_t off_codes, int l, const double *__restrict__ phase,
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
    const int2 *sched = reinterpret_cast<const int2 *>(ws + off_sched);
    const uint32_t *codes_g = reinterpret_cast<const uint32_t *>(ws + off_codes);
    const int total_words = reinterpret_cast<const int32_t *>(ws)[0];
    double *xs_base = reinterpret_cast<double *>(smem + d.xs_off);
    uint32_t *codes_s = reinterpret_cast<uint32_t *>(smem + d.code_off);
    const bool codes_in_smem = (int64_t)total_words * 4 <= d.code_cap;

    if (tid == 0) {
        for (int s = 0; s < d.ns; ++s) mbar_init(&full[s], 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&xs_full[b], kGW * 32);
            mbar_init(&xs_empty[b], kEW * 32);
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
    for (int i = tid; i < 2 * RB * pad; i += kNT) xs_base[i] = 0.0;
    if (codes_in_smem) {
        const uint4 *src = reinterpret_cast<const uint4 *>(codes_g);
        uint4 *dst = reinterpret_cast<uint4 *>(codes_s);
        const int nv = (total_words + 3) / 4;
        for (int i = tid; i < nv; i += kNT) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    const uint32_t *cw = codes_in_smem ? codes_s : codes_g;

    auto issue = [&](int64_t it) {
        const int stage = (int)(it % d.ns);
        const int64_t rbi = it / d.nch;
        const int ch = (int)(it % d.nch);
        const int64_t row0 = ((int64_t)blockIdx.x + rbi * gridDim.x) * RB;
        const int nrows = (int)min((int64_t)RB, m - row0);
        const int64_t c0 = (int64_t)ch * d.c;
        const int cols = (int)min((int64_t)d.c, n - c0);
        const unsigned bytes = (unsigned)cols * es;
        unsigned char *st = smem + (size_t)stage * d.stage_bytes;
        mbar_arrive_expect_tx(&full[stage], bytes * nrows);
        for (int r = 0; r < nrows; ++r)
            bulk_g2s(st + (size_t)r * d.row_stride, a + (row0 + r) * lda + c0, bytes, &full[stage]);
    };
    if (tid == 0)
        for (int64_t it = 0; it < d.ns && it < nitems; ++it) issue(it);

    if (warp < kGW) {
        // ------------------------------------------------------------ gather
        int bt[BPT], gid[BPT];
        bool bneg[BPT];
#pragma unroll
        for (int b = 0; b < BPT; ++b) {
            const int g = b * kGW + ((b & 1) ? kGW - 1 - warp : warp);
            gid[b] = g;
            bt[b] = grp[g * 32 + lane];
            bneg[b] = bt[b] >= 0 && phase[bt[b]] < 0.0;
        }
        for (int64_t rbi = 0; rbi < my_nrb; ++rbi) {
            double acc[BPT][RB];
#pragma unroll
            for (int b = 0; b < BPT; ++b)
#pragma unroll
                for (int r = 0; r < RB; ++r) acc[b][r] = 0.0;
            for (int ch = 0; ch < d.nch; ++ch) {
                const int64_t it = rbi * d.nch + ch;
                const int stage = (int)(it % d.ns);
                mbar_wait(&full[stage], (unsigned)((it / d.ns) & 1));
                const unsigned char *st = smem + (size_t)stage * d.stage_bytes;
#pragma unroll
                for (int b = 0; b < BPT; ++b) {
                    const int2 sc = __ldg(sched + ch * d.ng + gid[b]);
                    const uint32_t *cp = cw + sc.x + lane;
                    const int np = sc.y;
#pragma unroll 4
                    for (int s2 = 0; s2 < np; ++s2) {
                        const uint32_t w = cp[s2 * 32];
                        gather_step<T, RB>(st, d.row_stride, w & 0xffffu, acc[b]);
                        gather_step<T, RB>(st, d.row_stride, w >> 16, acc[b]);
                    }
                }
                // release the stage; the last of the kGW warps refills it
                __syncwarp();
                if (lane == 0) {
                    __threadfence_block();
                    const unsigned old = atomicAdd(&rel[stage], 1u);
                    if ((old + 1) % kGW == 0 && it + d.ns < nitems) {
                        fence_proxy_async_smem();
                        issue(it + d.ns);
                    }
                }
            }
            const int buf = (int)(rbi & 1);
            if (rbi >= 2) mbar_wait(&xs_empty[buf], (unsigned)(((rbi >> 1) - 1) & 1));
            double *xs = xs_base + (size_t)buf * RB * pad;
#pragma unroll
            for (int b = 0; b < BPT; ++b) {
                if (bt[b] >= 0) {
                    const int pos = fwht_sw(bt[b]);
#pragma unroll
                    for (int r = 0; r < RB; ++r) xs[r * pad + pos] = bneg[b] ? -acc[b][r] : acc[b][r];
                }
            }
            mbar_arrive(&xs_full[buf]);
        }
    } else {
        // ---------------------------------------------------------- epilogue
        const int ew = warp - kGW, etid = tid - kGW * 32;
        const int bsize = pad < 512 ? pad : 512;
        const int nb = pad / bsize;
        const int nzb = (l + bsize - 1) / bsize;
        bool bad = false;
        for (int64_t rbi = 0; rbi < my_nrb; ++rbi) {
            const int buf = (int)(rbi & 1);
            mbar_wait(&xs_full[buf], (unsigned)((rbi >> 1) & 1));
            double *xs = xs_base + (size_t)buf * RB * pad;
            for (int item = ew; item < RB * nzb; item += kEW) {
                const int r = item / nzb, bb = item % nzb;
                fwht_block_warp_dyn512(xs + (size_t)r * pad + (size_t)bb * bsize, bsize, lane);
            }
            named_bar(1, kEW * 32);
            const int64_t row0 = ((int64_t)blockIdx.x + rbi * gridDim.x) * RB;
            const int nrows = (int)min((int64_t)RB, m - row0);
            for (int w = etid; w < nrows * k; w += kEW * 32) {
                const int r = w / k, kk = w % k;
                const double v =
                    __dmul_rn(fwht_combine_blocks(xs + (size_t)r * pad, bsize, nb, idx[kk]), mult);
                y[(row0 + r) * ldy + kk] = v;
                bad |= !isfinite(v);
            }
            named_bar(1, kEW * 32);
            // the transformed blocks hold nonzeros at t >= l: re-zero them
            const int tz = nzb * bsize;
            for (int i = etid; i < RB * (tz - l); i += kEW * 32) {
                const int r = i / (tz - l), t = l + i % (tz - l);
                xs[(size_t)r * pad + fwht_sw(t)] = 0.0;
            }
            mbar_arrive(&xs_empty[buf]);
        }
        if (bad) atomicOr(nonfinite, 1);
    }
}

template <typename T, int RB, int BPT>
static int launch(const Cfg &f, const T *a, int64_t m, int64_t n, int64_t lda,
                  const unsigned char *ws, int64_t l, const double *phase, const int32_t *idx,
                  int64_t k, int64_t pad, double mult, double *y, int64_t ldy, int *nonfinite,
                  cudaStream_t s) {
    Dev d;
    d.c = f.c; d.nch = f.nch; d.ns = f.ns; d.ng = f.ng;
    d.row_stride = (int)f.row_stride; d.stage_bytes = (int)f.stage_bytes;
    d.xs_off = (int)(f.ns * f.stage_bytes);
    d.code_off = (int)(d.xs_off + f.xs_bytes);
    d.code_cap = (int)f.code_cap;
    auto kern = k1s_kernel<T, RB, BPT>;
    SRLU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f.smem));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t nrb = ceil_div(m, RB);
    const unsigned grid = (unsigned)(nrb < sms ? nrb : sms);
    kern<<<grid, kNT, (size_t)f.smem, s>>>(a, m, n, lda, ws, f.off_grp, f.off_sched, f.off_codes,
                                           (int)l, phase, idx, (int)k, (int)pad, mult, y, ldy,
                                           nonfinite, d);
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
#undef K1S_CASE
    set_error("sketch_right_dense_sched: no kernel for rb=%d bpt=%d", f.rb, f.bpt);
    return SRLU_ERR_UNSUPPORTED;
}

}  // namespace k1s
}  // namespace srlu

using namespace srlu;

static int es_of(int dtype) { return dtype == SRLU_F32 ? 4 : (dtype == SRLU_F64 ? 8 : 0); }

extern "C" size_t srlu_k1_schedule_bytes(int64_t n, int64_t l1, int64_t pad1, int dtype) {
    const int es = es_of(dtype);
    k1s::Cfg f;
    if (!es || !k1s::config(n, l1, pad1, es, &f)) return 0;
    return (size_t)f.ws_bytes;
}

extern "C" int srlu_k1_schedule(const int32_t *sorted1, const int32_t *bptr1, int64_t n,
                                int64_t l1, int64_t pad1, int dtype, void *sched,
                                size_t sched_bytes, srlu_stream_t stream) {
    const int es = es_of(dtype);
    k1s::Cfg f;
    SRLU_REQUIRE(es && k1s::config(n, l1, pad1, es, &f), SRLU_ERR_UNSUPPORTED,
                 "k1_schedule: shape not supported by the scheduled kernel");
    SRLU_REQUIRE(sched_bytes >= (size_t)f.ws_bytes, SRLU_ERR_WORKSPACE,
                 "k1_schedule: buffer too small");
    cudaStream_t s = (cudaStream_t)stream;
    unsigned char *ws = (unsigned char *)sched;
    int32_t *header = (int32_t *)ws;
    int32_t *grp = (int32_t *)(ws + f.off_grp);
    int32_t *np = (int32_t *)(ws + f.off_np);
    int32_t *sc = (int32_t *)(ws + f.off_sched);
    uint32_t *codes = (uint32_t *)(ws + f.off_codes);
    k1s::group_kernel<<<(unsigned)ceil_div((int64_t)f.ng * 32, 256), 256, 0, s>>>((int)l1, f.ng,
                                                                                 grp);
    SRLU_CHECK_LAUNCH("k1s_group_kernel");
    k1s::sched_kernel<0><<<f.ng, 32, 0, s>>>(sorted1, bptr1, f.c, f.nch, es == 8, f.ng, grp, np,
                                             sc, codes, header);
    SRLU_CHECK_LAUNCH("k1s_sched_kernel<0>");
    k1s::sched_kernel<1><<<f.ng, 32, 0, s>>>(sorted1, bptr1, f.c, f.nch, es == 8, f.ng, grp, np,
                                             sc, codes, header);
    SRLU_CHECK_LAUNCH("k1s_sched_kernel<1>");
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
