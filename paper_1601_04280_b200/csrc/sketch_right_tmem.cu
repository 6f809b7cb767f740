// K1T — stage-1 sketch  Y = A · Omega1^*  with the bucket accumulators in
// TENSOR MEMORY (reference: sketch.py:362-368 apply_sketch_right =
// _fast.pyx:44-54 sem_gather_dense + sketch.py:322-335 _fast_adjoint_right +
// _fast.pyx:23-41 fwht_rows), for dense A and 128 <= pad1 <= 1024.
//
// Why.  Every (row, bucket) sum must be accumulated in ascending source
// column to be bit-identical to the reference, so the parallelism is across
// (row, bucket) pairs.  The scheduled kernel (sketch_right_sched.cu) puts
// one BUCKET per lane: the lanes of a warp then want different columns of
// the same row in every step (bank conflicts, padded schedules: 57% of the
// lane-steps carry a source at config 2).  Here one ROW sits in each lane:
// the 32 lanes of a warp walk the SAME list of source columns, so a step is
// one shared-memory read of one column of 32 rows, there is no divergence
// and no schedule padding.  The price is 32 x l1 live fp64 accumulators per
// row block (225 KB at l1 = 880) — exactly what the 256 KB of tensor memory
// hold: TMEM lane = row, two 32-bit TMEM columns = one fp64 accumulator, a
// bucket's slot = its index within the lane quarter that owns it.  No
// tensor-core instruction is involved: TMEM is used as a second register
// file (tcgen05.ld / tcgen05.st, 32x32b shape).
//
// Layout.  A row block of R <= 32 rows is streamed in chunks of C columns
// (248 fp32 / 124 fp64) through a ring of stages filled by 2-D tensor-map
// bulk copies (TMA): one box of 8 rows x 1008 bytes per row group g = r / 8.
// The row pitch of 252 words maps the 8 rows of a box to the 8 bank quads;
// TMA can only place 16-byte units (measured: an inner coordinate that is
// not a multiple of 16 bytes is an illegal instruction), so three skew warps
// then shift the rows of group g by g words in place (fp64: g & 1 doubles):
// after that one column of all 32 rows falls into 32 distinct banks and
// every gather is one wavefront.  The words a shift frees (and the last
// word of the unshifted rows) are zeroed: the empty entries of the schedule
// point there and add +0.0 (exact) with no branch.  Consumer warp w = 4 i + q (i < 7, q = lane quarter) owns the
// slots [start(i), start(i+1)) of quarter q, i.e. buckets q * pad/4 + slot.
// Its schedule (built once per sketch, k1t_plan_kernel) lists, per chunk,
// its source columns in ascending order, packed four to a 64-bit word (no
// two of a word in the same slot): the warp loads the four accumulators
// (tcgen05.ld), adds the four columns (sign applied to the element's own
// sign bit, exact), and stores them back — four independent read-modify-
// write chains in flight per wait.
//
// Epilogue per row block, on the accumulators in place: +-phase and the
// FWHT stages h < pad/4 run inside each lane quarter (register passes of 16
// values per lane = row, tcgen05.ld/st), then the two cross-quarter stages
// are output-pruned to the k1 sampled indices (wht_pick order), exchanged
// through a small shared-memory tile so that the Y stores are coalesced.
// The ring keeps filling with the next row block meanwhile.
#include <cuda.h>
#include <limits.h>
#include <stdlib.h>

#include "fwht_warp.cuh"
#include "tma.cuh"

namespace srlu {
namespace k1t {

constexpr int kNT = 1024;
constexpr int kQW = 7;                    // consumer warps per lane quarter
constexpr int kCW = 4 * kQW;              // consumer warps
constexpr int kProducer = kCW;            // warp 28 issues the bulk copies
constexpr int kRowBytes = 1008;           // staged row: 252 fp32 / 126 fp64
constexpr int kBoxBytes = 8 * kRowBytes;        // one 8-row box = 63 * 128 bytes
constexpr int kGroupBytes = kBoxBytes + 128;    // + a zero pad behind the last row
constexpr int kStageBytes = 4 * kGroupBytes;    // 32 rows
constexpr int kSkewWarps = 3;                   // warps 29..31 shift row groups 1..3
constexpr int kXR = 16;                   // sampled outputs per exchange round
constexpr int kXPitch = 4 * 32 + 1;       // doubles per output in the exchange tile
constexpr int kMaxStages = 6;
constexpr int kHeader = 16;               // int32 header words of the plan
constexpr size_t kSmemMax = 232448 - 1024;

static int env_int(const char *name, int dflt) {
    const char *s = getenv(name);
    return (s && *s) ? atoi(s) : dflt;
}

struct Cfg {
    int es, c, nch, qs;
    int64_t off_info, off_table, off_quads, ws_bytes;
};

// Deterministic from (n, l, pad, es): the plan and the kernel agree.
static bool config(int64_t n, int64_t l, int64_t pad, int es, Cfg *cf) {
    // opt-in experiment (SRLU_K1_TMEM=1): bit-exact, but 0.49 ms at config 2
    // against 0.247 ms for the scheduled kernel (issue-bound: ~19 instructions
    // per 32-row gather step plus the skew pass; profiles/r02/k1t_*.txt)
    if (env_int("SRLU_K1_TMEM", 0) == 0) return false;
    if (pad < 128 || pad > 1024 || l < 1 || l > pad || n < 1 || n > (1 << 23)) return false;
    if (es != 4 && es != 8) return false;
    Cfg f{};
    f.es = es;
    f.c = es == 4 ? 248 : 124;
    f.nch = (int)ceil_div(n, f.c);
    f.qs = (int)(pad / 4);
    if ((int64_t)f.nch * kCW * 4 > 64 * 1024) return false;   // chunk table staged in smem
    auto al = [](int64_t v) { return (v + 15) & ~15LL; };
    f.off_info = al(kHeader * 4);
    f.off_table = al(f.off_info + n * 4);
    f.off_quads = al(f.off_table + (int64_t)f.nch * kCW * 4);
    f.ws_bytes = f.off_quads + 8 * (n + 4) + 64;     // <= one quad per source
    *cf = f;
    return true;
}

__host__ __device__ inline int slot_start(int i, int qs) { return (i * qs + kQW - 1) / kQW; }

// ---------------------------------------------------------------------------
// plan

// column -> bucket | negative sign << 31, from the bucket-sorted source lists
__global__ void k1t_invert_kernel(const int32_t *sorted, const int32_t *bptr, int l,
                                  uint32_t *info) {
    const int b = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x & 31;
    if (b >= l) return;
    for (int p = bptr[b] + lane; p < bptr[b + 1]; p += 32) {
        const uint32_t e = (uint32_t)sorted[p];
        info[e & 0x7fffffffu] = (uint32_t)b | (e & 0x80000000u);
    }
}

// One CTA per chunk, one warp per consumer warp: the warp's sources of the
// chunk in ascending column, greedily packed four to a quad (a quad closes
// early when the next source's slot is already in it).  Entry (16 bits):
// column in the chunk (bits 0-7; `dummy` = empty, a zeroed word) | slot relative to the warp's
// first slot (bits 8-13) | negative sign (bit 15).
__global__ void __launch_bounds__(32 * kCW) k1t_plan_kernel(const uint32_t *info, int n, int c,
                                                            int qs, unsigned dummy, int *total,
                                                            uint32_t *table,
                                                            unsigned long long *quads) {
    __shared__ uint16_t lst[kCW][256];
    const int ch = blockIdx.x, w = threadIdx.x / 32, lane = threadIdx.x & 31;
    const int q = w & 3, i = w >> 2;
    const int s0 = slot_start(i, qs), s1 = slot_start(i + 1, qs);
    const int c0 = ch * c, cw = min(c, n - c0);
    int cnt = 0;
    for (int cc0 = 0; cc0 < cw; cc0 += 32) {
        const int cc = cc0 + lane;
        uint32_t e = cc < cw ? info[c0 + cc] : 0u;
        const int b = (int)(e & 0x7fffffffu);
        const int sl = b % qs;
        const bool mine = cc < cw && b / qs == q && sl >= s0 && sl < s1;
        const unsigned mask = __ballot_sync(0xffffffffu, mine);
        if (mine)
            lst[w][cnt + __popc(mask & ((1u << lane) - 1u))] =
                (uint16_t)(cc | ((sl - s0) << 8) | ((e >> 31) << 15));
        cnt += __popc(mask);
    }
    __syncwarp();
    if (lane == 0) {
        // pass 1: number of quads
        int nq = 0, fill = 0;
        unsigned long long used = 0;
        for (int t = 0; t < cnt; ++t) {
            const unsigned long long bit = 1ull << ((lst[w][t] >> 8) & 63);
            if (fill == 4 || (used & bit)) { ++nq; fill = 0; used = 0; }
            used |= bit; ++fill;
        }
        if (fill) ++nq;
        const int off = nq ? atomicAdd(total, nq) : 0;
        table[ch * kCW + w] = ((uint32_t)off << 8) | (uint32_t)nq;
        // pass 2: write them; the empty entries of a quad get the dummy column
        // (a zeroed word: the kernel adds +0.0, exact) and a slot of the warp that is not in
        // the quad (four independent read-modify-writes, no branches)
        const int nslots = s1 - s0;
        auto flush = [&](unsigned long long cur, int fill, unsigned long long used) {
            int free_slot = 0;
            for (int u = fill; u < 4; ++u) {
                while (free_slot < nslots - 1 && ((used >> free_slot) & 1ull)) ++free_slot;
                used |= 1ull << free_slot;
                cur = (cur & ~(0xffffull << (16 * u))) |
                      ((unsigned long long)(dummy | (free_slot << 8)) << (16 * u));
            }
            return cur;
        };
        unsigned long long cur = 0;
        int k = 0;
        fill = 0; used = 0;
        for (int t = 0; t < cnt; ++t) {
            const unsigned long long bit = 1ull << ((lst[w][t] >> 8) & 63);
            if (fill == 4 || (used & bit)) {
                quads[off + k++] = flush(cur, fill, used);
                cur = 0; fill = 0; used = 0;
            }
            cur |= (unsigned long long)lst[w][t] << (16 * fill);
            used |= bit; ++fill;
        }
        if (fill) quads[off + k++] = flush(cur, fill, used);
    }
}

// ---------------------------------------------------------------------------
// tensor memory helpers (32x32b shape: lane = thread of the warp's quarter)

__device__ __forceinline__ void tm_ld2(unsigned taddr, unsigned &lo, unsigned &hi) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
                 : "=r"(lo), "=r"(hi) : "r"(taddr));
}
__device__ __forceinline__ void tm_st2(unsigned taddr, unsigned lo, unsigned hi) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};"
                 :: "r"(taddr), "r"(lo), "r"(hi));
}
__device__ __forceinline__ void tm_wait_st() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// wait for the loads AND pin the destination registers behind the wait
__device__ __forceinline__ void tm_wait_ld2(unsigned &a, unsigned &b) {
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(a), "+r"(b)::"memory");
}
__device__ __forceinline__ void tm_wait_ld8(unsigned (&v)[8]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                   "+r"(v[6]), "+r"(v[7])::"memory");
}
__device__ __forceinline__ void tm_ld32(unsigned taddr, unsigned (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
        "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
        "%30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
          "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
          "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tm_st32(unsigned taddr, const unsigned (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
        "%29, %30, %31, %32};"
        ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
          "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]),
          "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]),
          "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
          "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
}
__device__ __forceinline__ void tm_wait_ld32(unsigned (&v)[32]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                   "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]),
                   "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]), "+r"(v[16]), "+r"(v[17]),
                   "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]),
                   "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]),
                   "+r"(v[30]), "+r"(v[31])::"memory");
}
__device__ __forceinline__ void tm_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tm_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// 2-D tensor-map bulk copy of one box, completion counted on `bar`
__device__ __forceinline__ void tma_box_2d(void *dst, const CUtensorMap *tm, int x, int y,
                                           uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], "
        "[%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(tm), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// 16 values: butterflies of the bits 0..3 of the value index (a + b, a - b)
__device__ __forceinline__ void butterflies16(double (&v)[16]) {
#pragma unroll
    for (int h = 1; h < 16; h <<= 1) {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            if ((e & h) == 0) {
                const double a = v[e], b = v[e + h];
                v[e] = __dadd_rn(a, b);
                v[e + h] = __dsub_rn(a, b);
            }
        }
    }
}

// FWHT stages h = 16 .. qs/2 of a lane quarter: NV = qs/16 values of stride
// 16 slots per group c0 (one tcgen05.ld/st per value)
template <int NV>
__device__ __forceinline__ void quarter_pass_b(unsigned qbase, int i) {
    for (int c0 = i; c0 < 16; c0 += kQW) {
        unsigned lo[NV], hi[NV];
#pragma unroll
        for (int e = 0; e < NV; ++e) tm_ld2(qbase + 2 * (c0 + 16 * e), lo[e], hi[e]);
#pragma unroll
        for (int e = 0; e < NV; ++e) tm_wait_ld2(lo[e], hi[e]);
        double v[NV];
#pragma unroll
        for (int e = 0; e < NV; ++e) v[e] = __hiloint2double((int)hi[e], (int)lo[e]);
#pragma unroll
        for (int h = 1; h < NV; h <<= 1) {
#pragma unroll
            for (int e = 0; e < NV; ++e) {
                if ((e & h) == 0) {
                    const double a = v[e], b = v[e + h];
                    v[e] = __dadd_rn(a, b);
                    v[e + h] = __dsub_rn(a, b);
                }
            }
        }
#pragma unroll
        for (int e = 0; e < NV; ++e)
            tm_st2(qbase + 2 * (c0 + 16 * e), (unsigned)__double2loint(v[e]),
                   (unsigned)__double2hiint(v[e]));
    }
}

struct Dev {
    int c, nch, ns, qs, rows;        // rows per block R
    int nfull, tail;                 // 8-row boxes per stage, rows of the tail box
    int stage_tx;                    // bytes per stage
    int off_table, off_quads, off_xch, quad_cap;   // smem offsets (bytes), quad capacity
    int dbg;                         // experiments (wrong results): 1 no quads, 2 no epilogue, 4 no skew
};

template <typename T>
__global__ void __launch_bounds__(kNT, 1)
k1t_kernel(const __grid_constant__ CUtensorMap tm8, const __grid_constant__ CUtensorMap tmt,
           int64_t m, const unsigned char *ws, int64_t ws_table, int64_t ws_quads, int l,
           const double *__restrict__ phase, const int32_t *__restrict__ idx, int k, int pad,
           double mult, double *__restrict__ y, int64_t ldy, int *nonfinite, Dev d) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint64_t full[kMaxStages], ready[kMaxStages], empty[kMaxStages];
    __shared__ unsigned tmem_base_s;
    __shared__ unsigned phw[32];                 // phase sign bits of the pad buckets
    constexpr int ES = (int)sizeof(T);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int R = d.rows, qs = d.qs;
    const int64_t nblk = ceil_div(m, (int64_t)R);
    const int64_t my_nblk = (nblk - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int total_quads = ((const int *)ws)[0];
    const bool staged = total_quads <= d.quad_cap;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         smem_u32(&tmem_base_s))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 32) {
        for (int s = 0; s < d.ns; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&ready[s], kSkewWarps);
            mbar_init(&empty[s], kCW);
        }
        fence_mbar_init();
    }
    // chunk table (and the quads when they fit) into shared memory
    uint32_t *table_s = (uint32_t *)(smem + d.off_table);
    {
        const uint32_t *tg = (const uint32_t *)(ws + ws_table);
        for (int t = tid; t < d.nch * kCW; t += kNT) table_s[t] = tg[t];
        if (staged) {
            const uint2 *qg = (const uint2 *)(ws + ws_quads);
            uint2 *qsm = (uint2 *)(smem + d.off_quads);
            for (int t = tid; t < total_quads; t += kNT) qsm[t] = qg[t];
        }
    }
    // phase sign bits
    for (int b = tid; b < pad; b += kNT) {
        const bool neg = b < l && phase[b] < 0.0;
        const unsigned mask = __ballot_sync(0xffffffffu, neg);
        if (lane == 0) phw[b >> 5] = mask;
    }
    // zero pad behind every row group (the bulk copies never write it)
    for (int t = tid; t < d.ns * 4 * 32; t += kNT)
        *(unsigned *)(smem + (size_t)(t / 32) * kGroupBytes + kBoxBytes + (t % 32) * 4) = 0u;
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    const unsigned tbase = tmem_base_s;
    const uint2 *quads = staged ? (const uint2 *)(smem + d.off_quads)
                                : (const uint2 *)(ws + ws_quads);

    if (warp == kProducer) {
        // ---------------- producer: one lane issues the bulk copies ----------------
        if (lane == 0) {
            int64_t it = 0;
            for (int64_t bi = 0; bi < my_nblk; ++bi) {
                const int64_t row0 = ((int64_t)blockIdx.x + bi * gridDim.x) * R;
                for (int ch = 0; ch < d.nch; ++ch, ++it) {
                    const int s = (int)(it % d.ns);
                    if (it >= d.ns) mbar_wait(&empty[s], (unsigned)(((it / d.ns) - 1) & 1));
                    mbar_arrive_expect_tx(&full[s], (unsigned)d.stage_tx);
                    unsigned char *st = smem + (size_t)s * kStageBytes;
                    const int c0 = ch * d.c;
#pragma unroll 1
                    for (int g = 0; g < d.nfull; ++g)
                        tma_box_2d(st + g * kGroupBytes, &tm8, c0, (int)(row0 + 8 * g), &full[s]);
                    if (d.tail)
                        tma_box_2d(st + d.nfull * kGroupBytes, &tmt, c0, (int)(row0 + 8 * d.nfull),
                                   &full[s]);
                }
            }
        }
    } else if (warp > kProducer) {
        // ---------------- skew warps: row group j + 1 shifted in place ----------------
        const int j = warp - kProducer - 1;            // 0..2
        const int g = j + 1;
        const int skew = ES == 4 ? g : (g & 1);        // elements
        constexpr int EPR = kRowBytes / ES;            // elements per staged row
        constexpr int NV = (EPR + 31) / 32;
        const int64_t items = my_nblk * d.nch;
        for (int64_t it = 0; it < items; ++it) {
            const int s = (int)(it % d.ns);
            mbar_wait(&full[s], (unsigned)((it / d.ns) & 1));
            unsigned char *st = smem + (size_t)s * kStageBytes;
            if (skew && 8 * g < R && !(d.dbg & 4)) {
                T *grp = (T *)(st + g * kGroupBytes);
#pragma unroll 1
                for (int r0 = 0; r0 < 8; r0 += 2) {
                    T v[2][NV];
#pragma unroll
                    for (int rr = 0; rr < 2; ++rr)
#pragma unroll
                        for (int t = 0; t < NV; ++t) {
                            const int c = t * 32 + lane;
                            v[rr][t] = c < EPR ? grp[(r0 + rr) * EPR + c] : T(0);
                        }
                    __syncwarp();
#pragma unroll
                    for (int rr = 0; rr < 2; ++rr)
#pragma unroll
                        for (int t = 0; t < NV; ++t) {
                            const int c = t * 32 + lane + skew;
                            if (c < EPR) grp[(r0 + rr) * EPR + c] = v[rr][t];
                        }
                    if (lane < 2 * skew) grp[(r0 + lane / skew) * EPR + lane % skew] = T(0);
                }
            }
            // unshifted rows: their last element is the dummy column
            if (lane < 8) {
                if (j == 0) ((T *)st)[lane * EPR + EPR - 1] = T(0);
                if (ES == 8 && j == 1) ((T *)(st + 2 * kGroupBytes))[lane * EPR + EPR - 1] = T(0);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&ready[s]);
        }
    } else if (warp < kCW) {
        // ---------------- consumers ----------------
        const int q = warp & 3, i = warp >> 2;
        const int s0 = slot_start(i, qs), s1 = slot_start(i + 1, qs);
        const unsigned qbase = tbase + ((unsigned)(32 * q) << 16);
        const unsigned wbase = qbase + 2 * s0;
        // zero the own slots
        for (int s = s0; s < s1; ++s) tm_st2(qbase + 2 * s, 0u, 0u);
        tm_wait_st();
        const int g = lane >> 3;
        const unsigned lane_off =
            (unsigned)(g * kGroupBytes + (lane & 7) * kRowBytes + (ES == 4 ? g : (g & 1)) * ES);
        double *xch = (double *)(smem + d.off_xch);
        bool bad = false;
        int64_t it = 0;
        for (int64_t bi = 0; bi < my_nblk; ++bi) {
            const int64_t row0 = ((int64_t)blockIdx.x + bi * gridDim.x) * R;
            const int nrows = (int)min((int64_t)R, m - row0);
            for (int ch = 0; ch < d.nch; ++ch, ++it) {
                const int s = (int)(it % d.ns);
                const uint32_t te = table_s[ch * kCW + warp];
                const int nq = (int)(te & 0xffu);
                const uint2 *qp = quads + (te >> 8);
                mbar_wait(&ready[s], (unsigned)((it / d.ns) & 1));
                const unsigned char *row = smem + (size_t)s * kStageBytes + lane_off;
#pragma unroll 1
                for (int t = 0; t < ((d.dbg & 1) ? 0 : nq); ++t) {
                    const uint2 qd = qp[t];
                    unsigned e[4] = {qd.x & 0xffffu, qd.x >> 16, qd.y & 0xffffu, qd.y >> 16};
                    unsigned acc[8], ta[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        ta[u] = wbase + ((e[u] >> 7) & 0x7eu);
                        tm_ld2(ta[u], acc[2 * u], acc[2 * u + 1]);
                    }
                    double x[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const unsigned off = (e[u] & 0xffu) * ES;
                        if (ES == 4) {
                            unsigned bits = *(const unsigned *)(row + off);
                            bits ^= (e[u] & 0x8000u) << 16;
                            x[u] = (double)__uint_as_float(bits);
                        } else {
                            uint2 bits = *(const uint2 *)(row + off);
                            bits.y ^= (e[u] & 0x8000u) << 16;
                            x[u] = __hiloint2double((int)bits.y, (int)bits.x);
                        }
                    }
                    tm_wait_ld8(acc);
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const double a = __hiloint2double((int)acc[2 * u + 1], (int)acc[2 * u]);
                        const double r = __dadd_rn(a, x[u]);
                        tm_st2(ta[u], (unsigned)__double2loint(r), (unsigned)__double2hiint(r));
                    }
                }
                // this warp is done reading the stage
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }
            // ---------------- epilogue of the row block ----------------
            if (d.dbg & 2) continue;
            tm_wait_st();
            tm_fence_before();
            named_bar(1 + q, 32 * kQW);
            tm_fence_after();
            // pass A: +-phase, stages h = 1, 2, 4, 8 on 16 consecutive slots
            for (int grp = i; grp < qs / 16; grp += kQW) {
                unsigned r[32];
                tm_ld32(qbase + 32 * grp, r);
                const int b0 = q * qs + 16 * grp;
                const unsigned bits = (phw[b0 >> 5] >> (b0 & 31)) & 0xffffu;
                tm_wait_ld32(r);
                double v[16];
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    v[e] = __hiloint2double((int)(r[2 * e + 1] ^ ((bits << (31 - e)) & 0x80000000u)),
                                            (int)r[2 * e]);
                butterflies16(v);
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    r[2 * e] = (unsigned)__double2loint(v[e]);
                    r[2 * e + 1] = (unsigned)__double2hiint(v[e]);
                }
                tm_st32(qbase + 32 * grp, r);
            }
            tm_wait_st();
            tm_fence_before();
            named_bar(1 + q, 32 * kQW);
            tm_fence_after();
            // pass B: stages h = 16 .. qs/2
            switch (qs) {
                case 256: quarter_pass_b<16>(qbase, i); break;
                case 128: quarter_pass_b<8>(qbase, i); break;
                case 64: quarter_pass_b<4>(qbase, i); break;
                default: quarter_pass_b<2>(qbase, i); break;
            }
            tm_wait_st();
            tm_fence_before();
            named_bar(1 + q, 32 * kQW);
            tm_fence_after();
            // cross-quarter stages h = qs, 2 qs for the k sampled outputs only
            for (int kb = 0; kb < k; kb += kXR) {
                const int nk = min(kXR, k - kb);
                for (int kk = i; kk < nk; kk += kQW) {
                    const int o = __ldg(idx + kb + kk) & (qs - 1);
                    unsigned lo, hi;
                    tm_ld2(qbase + 2 * o, lo, hi);
                    tm_wait_ld2(lo, hi);
                    xch[kk * kXPitch + q * 32 + lane] = __hiloint2double((int)hi, (int)lo);
                }
                named_bar(5, 32 * kCW);
                if (tid < kXR * 32) {
                    const int kk = tid & (kXR - 1), r = tid / kXR;
                    if (kk < nk && r < nrows) {
                        const int B = __ldg(idx + kb + kk) / qs;
                        const double *xp = xch + kk * kXPitch + r;
                        const double sg0 = pm_one(B & 1), sg1 = pm_one((B >> 1) & 1);
                        const double u0 = __fma_rn(sg0, xp[32], xp[0]);
                        const double u1 = __fma_rn(sg0, xp[96], xp[64]);
                        const double v = __dmul_rn(__fma_rn(sg1, u1, u0), mult);
                        y[(row0 + r) * ldy + kb + kk] = v;
                        bad |= !isfinite(v);
                    }
                }
                named_bar(5, 32 * kCW);
            }
            // fresh accumulators for the next row block
            for (int s = s0; s < s1; ++s) tm_st2(qbase + 2 * s, 0u, 0u);
            tm_wait_st();
        }
        if (bad) atomicOr(nonfinite, 1);
    }
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase)
                     : "memory");
}

// ---------------------------------------------------------------------------
// host

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) ==
                cudaSuccess &&
            qr == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    }
    return fn;
}

static int make_map(CUtensorMap *tm, const void *a, int es, int64_t m, int64_t n, int64_t lda,
                    int box_rows) {
    EncodeTiledFn fn = encode_fn();
    SRLU_REQUIRE(fn != nullptr, SRLU_ERR_CUDA, "k1t: cuTensorMapEncodeTiled not available");
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)m};
    cuuint64_t strides[1] = {(cuuint64_t)(lda * es)};
    cuuint32_t box[2] = {(cuuint32_t)(kRowBytes / es), (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(tm, es == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                    2, const_cast<void *>(a), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    SRLU_REQUIRE(r == CUDA_SUCCESS, SRLU_ERR_CUDA, "k1t: cuTensorMapEncodeTiled failed (%d)", (int)r);
    return SRLU_OK;
}

// rows per block: the R <= 32 with the shortest makespan (waves x R) on
// `sms` persistent CTAs, larger R on ties
static int pick_rows(int64_t m, int sms) {
    const int forced = env_int("SRLU_K1T_ROWS", 0);
    if (forced >= 1 && forced <= 32) return forced;
    int best = 32;
    int64_t best_cost = LLONG_MAX;
    for (int r = 32; r >= 8; --r) {
        const int64_t nblk = ceil_div(m, (int64_t)r);
        const int64_t cost = ceil_div(nblk, (int64_t)sms) * r;
        if (cost < best_cost) { best_cost = cost; best = r; }
    }
    return best;
}

template <typename T>
static int launch(const Cfg &f, const T *a, int64_t m, int64_t n, int64_t lda,
                  const unsigned char *ws, int64_t l, const double *phase, const int32_t *idx,
                  int64_t k, int64_t pad, double mult, double *y, int64_t ldy, int *nonfinite,
                  cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    Dev d{};
    d.c = f.c; d.nch = f.nch; d.qs = f.qs;
    d.rows = pick_rows(m, sms);
    d.dbg = env_int("SRLU_K1T_DBG", 0);
    d.nfull = d.rows / 8;
    d.tail = d.rows % 8;
    d.stage_tx = d.nfull * kBoxBytes + d.tail * kRowBytes;
    const int64_t table_bytes = ((int64_t)f.nch * kCW * 4 + 15) & ~15LL;
    const int64_t xch_bytes = ((int64_t)kXR * kXPitch * 8 + 15) & ~15LL;
    // ring stages: as many as leave room for the expected quads (n / 3)
    int ns = env_int("SRLU_K1T_NS", 0);
    if (ns < 2 || ns > kMaxStages) {
        ns = kMaxStages;
        const int64_t want = table_bytes + xch_bytes + 8 * (n / 3 + 64);
        while (ns > 3 && (int64_t)ns * kStageBytes + want > (int64_t)kSmemMax) --ns;
    }
    const int64_t fixed = (int64_t)ns * kStageBytes + table_bytes + xch_bytes;
    SRLU_REQUIRE(fixed + 64 <= (int64_t)kSmemMax, SRLU_ERR_UNSUPPORTED, "k1t: shared memory");
    d.ns = ns;
    d.off_table = ns * kStageBytes;
    d.off_xch = (int)(d.off_table + table_bytes);
    d.off_quads = (int)(d.off_xch + xch_bytes);
    d.quad_cap = (int)(((int64_t)kSmemMax - d.off_quads) / 8);
    CUtensorMap tm8, tmt;
    int rc = make_map(&tm8, a, (int)sizeof(T), m, n, lda, 8);
    if (rc != SRLU_OK) return rc;
    rc = make_map(&tmt, a, (int)sizeof(T), m, n, lda, d.tail ? d.tail : 8);
    if (rc != SRLU_OK) return rc;
    auto kern = k1t_kernel<T>;
    SRLU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax));
    const int64_t nblk = ceil_div(m, (int64_t)d.rows);
    const unsigned grid = (unsigned)(nblk < sms ? nblk : sms);
    kern<<<grid, kNT, kSmemMax, s>>>(tm8, tmt, m, ws, f.off_table, f.off_quads, (int)l, phase, idx,
                                     (int)k, (int)pad, mult, y, ldy, nonfinite, d);
    SRLU_CHECK_LAUNCH("k1t_kernel");
    return SRLU_OK;
}

}  // namespace k1t
}  // namespace srlu

using namespace srlu;

// Entry points used by sketch_right_sched.cu's C ABI (srlu_k1_schedule_bytes,
// srlu_k1_config, srlu_k1_schedule, srlu_sketch_right_dense_sched): the
// TMEM kernel takes over whenever its geometry applies.

size_t srlu_k1t_plan_bytes(int64_t n, int64_t l1, int64_t pad1, int es) {
    k1t::Cfg f;
    return k1t::config(n, l1, pad1, es, &f) ? (size_t)f.ws_bytes : 0;
}

int srlu_k1t_info(int64_t n, int64_t l1, int64_t pad1, int es, int64_t info[8]) {
    k1t::Cfg f;
    if (!k1t::config(n, l1, pad1, es, &f)) return SRLU_ERR_UNSUPPORTED;
    info[0] = 32; info[1] = 2;   // [1] >= 2: the plan is two kernel launches (launch accounting)
    info[2] = f.c; info[3] = f.nch;
    info[4] = k1t::kMaxStages; info[5] = 0; info[6] = (int64_t)k1t::kSmemMax; info[7] = 100;
    return SRLU_OK;
}

int srlu_k1t_plan(const int32_t *sorted1, const int32_t *bptr1, int64_t n, int64_t l1,
                  int64_t pad1, int es, void *plan, size_t plan_bytes, cudaStream_t s) {
    k1t::Cfg f;
    SRLU_REQUIRE(k1t::config(n, l1, pad1, es, &f), SRLU_ERR_UNSUPPORTED, "k1t_plan: unsupported shape");
    SRLU_REQUIRE(plan_bytes >= (size_t)f.ws_bytes, SRLU_ERR_WORKSPACE, "k1t_plan: buffer too small");
    unsigned char *ws = (unsigned char *)plan;
    SRLU_CUDA(cudaMemsetAsync(ws, 0, k1t::kHeader * sizeof(int32_t), s));
    uint32_t *info = (uint32_t *)(ws + f.off_info);
    k1t::k1t_invert_kernel<<<(unsigned)ceil_div(l1 * 32, 256), 256, 0, s>>>(sorted1, bptr1, (int)l1, info);
    SRLU_CHECK_LAUNCH("k1t_invert_kernel");
    k1t::k1t_plan_kernel<<<f.nch, 32 * k1t::kCW, 0, s>>>(
        info, (int)n, f.c, f.qs, (unsigned)(k1t::kRowBytes / es - 1), (int *)ws, (uint32_t *)(ws + f.off_table),
        (unsigned long long *)(ws + f.off_quads));
    SRLU_CHECK_LAUNCH("k1t_plan_kernel");
    return SRLU_OK;
}

int srlu_k1t_run(const void *a, int es, int64_t m, int64_t n, int64_t lda, const void *plan,
                 size_t plan_bytes, int64_t l1, const double *phase1, const int32_t *idx1,
                 int64_t k1, int64_t pad1, double mult1, double *y, int64_t ldy, int *nonfinite,
                 cudaStream_t s) {
    k1t::Cfg f;
    SRLU_REQUIRE(k1t::config(n, l1, pad1, es, &f), SRLU_ERR_UNSUPPORTED, "k1t_run: unsupported shape");
    SRLU_REQUIRE(plan_bytes >= (size_t)f.ws_bytes, SRLU_ERR_WORKSPACE, "k1t_run: plan buffer too small");
    const unsigned char *ws = (const unsigned char *)plan;
    if (es == 4)
        return k1t::launch<float>(f, (const float *)a, m, n, lda, ws, l1, phase1, idx1, k1, pad1,
                                  mult1, y, ldy, nonfinite, s);
    return k1t::launch<double>(f, (const double *)a, m, n, lda, ws, l1, phase1, idx1, k1, pad1,
                               mult1, y, ldy, nonfinite, s);
}
