// K4 for large reduced systems: Householder QR of M = Omega2·L1 (k2 x k1,
// k1 up to 576) on one thread-block cluster, and the exact singular-value
// fallback of the rank test.  Reference: factor.py:112-130
// (left_pseudo_inverse: numpy.linalg.qr, numpy.linalg.svd of R, the
// sv[-1] <= 1e-10 sv[0] decision, solve_triangular).
//
//  * qr_cluster_kernel: the columns of M are dealt cyclically to the C CTAs
//    of one cluster (column c lives in CTA c mod C's shared memory: 35
//    columns of 558 rows = 156 KB per CTA at config 5).  Reflector j is
//    formed (LAPACK dgeqr2/dlarfg conventions) by the CTA that owns column j
//    and pushed with st.async into a receive slot of every CTA's shared
//    memory, completing the transaction count of that CTA's mbarrier; every
//    CTA applies it to its own columns.  Lookahead: the owner of column j+1
//    applies reflector j to that column first, forms reflector j+1 and
//    pushes it, then updates its other columns — so the critical path per
//    reflector is one column update + one dlarfg + one push.  Two receive
//    slots; a slot is rewritten (reflector j+2) only after every CTA
//    released it (remote mbarrier arrivals on the next owner's free
//    barrier).  Output: the packed QR (column-major, reflectors below the
//    diagonal), tau and R row-major — the layout of the one-CTA kernels in
//    small_dense.cu, so the pinv tail and the rank test are shared.
//  * jacobi_sv_kernel: one-sided (Hestenes) Jacobi on the columns of R in
//    global memory (L2-resident), round-robin pair ordering, one grid
//    barrier per round, until a sweep rotates nothing; sigma_i = column
//    norms.  Run only when the certified bounds of the rank test cannot
//    decide (srlu_qr_rank_certified flag 2): the decision is then made on
//    the singular values themselves, like the reference.
#include <math.h>
#include <stdlib.h>

#include "common.cuh"
#include "tma.cuh"

namespace srlu {
namespace qrc {

constexpr int NT = 512;
constexpr int NW = NT / 32;

__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_size() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
                 ::: "memory");
}
__device__ __forceinline__ unsigned mapa(unsigned saddr, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async2(unsigned addr, double a, double b, unsigned rbar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
            addr),
        "d"(a), "d"(b), "r"(rbar)
        : "memory");
}
__device__ __forceinline__ void arrive_remote(unsigned raddr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(raddr)
                 : "memory");
}
__device__ __forceinline__ void wait_cluster(unsigned addr, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WQC_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WQC_%=;\n"
        "}\n" ::"r"(addr),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// one warp: col[j:] -= tau * v * (v^T col[j:]), v[j] = 1 (dlarf)
__device__ __forceinline__ void apply_col(double *col, const double *v, double tau, int j, int k2p) {
    const int lane = threadIdx.x & 31;
    double w = lane == 0 ? col[j] : 0.0;
    for (int i = j + 1 + lane; i < k2p; i += 32) w = __fma_rn(v[i], col[i], w);
    const double f = tau * warp_sum(w);
    if (lane == 0) col[j] -= f;
    for (int i = j + 1 + lane; i < k2p; i += 32) col[i] = __fma_rn(-f, v[i], col[i]);
    __syncwarp();
}

// one warp: dlarfg on col[j:] (alpha = col[j]); col[j] <- beta, col[j+1:]
// <- v (scaled by 1/(alpha - beta)); returns tau (0: H = I, col unchanged)
__device__ __forceinline__ double dlarfg_col(double *col, int j, int k2p) {
    const int lane = threadIdx.x & 31;
    double part = 0.0;
    for (int i = j + 1 + lane; i < k2p; i += 32) part = __fma_rn(col[i], col[i], part);
    part = warp_sum(part);
    const double alpha = col[j];
    __syncwarp();
    if (!(part > 0.0)) return 0.0;
    const double beta = -copysign(sqrt(__fma_rn(alpha, alpha, part)), alpha);
    const double tau = (beta - alpha) / beta;
    const double scal = 1.0 / (alpha - beta);
    for (int i = j + 1 + lane; i < k2p; i += 32) col[i] *= scal;
    if (lane == 0) col[j] = beta;
    __syncwarp();
    return tau;
}

struct QrLayout {
    int k2p, ncl;
    __host__ __device__ static int ncl_max(int k1, int C) { return (k1 + C - 1) / C; }
    __host__ __device__ static size_t bytes(int k1, int k2, int C) {
        const int k2p = (k2 + 1) & ~1, nc = ncl_max(k1, C);
        return 64 + sizeof(double) * ((size_t)((nc + 1) & ~1) + 2 * (size_t)(2 + k2p) +
                                      (size_t)nc * k2p);
    }
};

__global__ void __launch_bounds__(NT, 1) qr_cluster_kernel(const double *__restrict__ mT, int k1,
                                                         int k2, int64_t ldm,
                                                         double *__restrict__ qa,
                                                         double *__restrict__ qtau,
                                                         double *__restrict__ rrow) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const unsigned C = cluster_size(), rank = cluster_rank();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int k2p = (k2 + 1) & ~1;
    const int ncl = k1 > (int)rank ? (k1 - (int)rank + (int)C - 1) / (int)C : 0;
    const int ncm = QrLayout::ncl_max(k1, (int)C);
    uint64_t *rbar = reinterpret_cast<uint64_t *>(smem_raw);  // [2] reflector arrived
    uint64_t *fbar = rbar + 2;                                 // [2] slot released (owner)
    double *taus = reinterpret_cast<double *>(smem_raw + 64);
    double *vbuf = taus + ((ncm + 1) & ~1);                    // [2][2 + k2p]
    double *cols = vbuf + 2 * (2 + k2p);                       // [ncl][k2p]
    const int VS = 2 + k2p;

    for (int i = tid; i < ncl * k2p; i += NT) {
        const int lc = i / k2p, r = i % k2p;
        const int c = (int)rank + (int)C * lc;
        cols[i] = r < k2 ? mT[(int64_t)c * ldm + r] : 0.0;
    }
    if (tid == 0) {
        mbar_init(&rbar[0], 1);
        mbar_init(&rbar[1], 1);
        mbar_init(&fbar[0], C);
        mbar_init(&fbar[1], C);
        fence_mbar_init();
    }
    __syncthreads();
    cluster_sync_all();

    auto push = [&](int j, const double *col, double tau) {
        const int s = j & 1, j0 = j & ~1;
        const int units = 1 + (k2p - j0) / 2;
        const unsigned slot = smem_u32(vbuf + s * VS), bar = smem_u32(&rbar[s]);
        for (int idx = tid; idx < (int)C * units; idx += NT) {
            const unsigned d = (unsigned)(idx / units);
            const int u = idx % units;
            const unsigned rb = mapa(bar, d);
            if (u == 0) {
                st_async2(mapa(slot, d), tau, 0.0, rb);
            } else {
                const int r = j0 + 2 * (u - 1);
                st_async2(mapa(slot + 8u * (unsigned)(2 + r), d), col[r], col[r + 1], rb);
            }
        }
    };

    unsigned fuse0 = 0u, fuse1 = 0u;  // waits done on this CTA's free barriers
    if (rank == 0) {
        if (warp == 0) {
            const double t = dlarfg_col(cols, 0, k2p);
            if (lane == 0) taus[0] = t;
        }
        __syncthreads();
        push(0, cols, taus[0]);
    }
    for (int j = 0; j < k1; ++j) {
        const int s = j & 1;
        if (tid == 0)
            mbar_arrive_expect_tx(&rbar[s], 16u * (unsigned)(1 + (k2p - (j & ~1)) / 2));
        wait_cluster(smem_u32(&rbar[s]), (unsigned)(j >> 1) & 1u);
        const double *vs = vbuf + s * VS;
        const double tau = vs[0];
        const double *v = vs + 2;
        int lc0 = j < (int)rank ? 0 : (j - (int)rank) / (int)C + 1;
        const int jn = j + 1;
        if (jn < k1 && jn % (int)C == (int)rank) {
            // the critical column: reflector j, then form and push reflector j+1
            double *col = cols + (size_t)lc0 * k2p;
            if (warp == 0) {
                if (tau != 0.0) apply_col(col, v, tau, j, k2p);
                const double t = dlarfg_col(col, jn, k2p);
                if (lane == 0) taus[lc0] = t;
            }
            __syncthreads();
            if (jn >= 2) {
                const int sn = jn & 1;
                unsigned &fu = sn ? fuse1 : fuse0;
                wait_cluster(smem_u32(&fbar[sn]), fu & 1u);
                ++fu;
            }
            push(jn, col, taus[lc0]);
            ++lc0;
        }
        if (tau != 0.0)
            for (int lc = lc0 + warp; lc < ncl; lc += NW)
                apply_col(cols + (size_t)lc * k2p, v, tau, j, k2p);
        __syncthreads();
        if (tid == 0 && j + 2 < k1) arrive_remote(mapa(smem_u32(&fbar[s]), (unsigned)((j + 2) % (int)C)));
    }
    // packed QR (column-major, ld = k2|1), tau, R row-major
    const int ld = k2 | 1;
    for (int i = tid; i < ncl * k2; i += NT) {
        const int lc = i / k2, r = i % k2;
        const int c = (int)rank + (int)C * lc;
        qa[(int64_t)c * ld + r] = cols[(size_t)lc * k2p + r];
    }
    for (int lc = tid; lc < ncl; lc += NT) qtau[(int)rank + (int)C * lc] = taus[lc];
    for (int i = tid; i < ncl * k1; i += NT) {
        const int lc = i / k1, r = i % k1;
        const int c = (int)rank + (int)C * lc;
        rrow[(int64_t)r * k1 + c] = r <= c ? cols[(size_t)lc * k2p + r] : 0.0;
    }
    cluster_sync_all();
}

// ---------------------------------------------------------------------------
// Exact singular values of R (k x k upper triangular): one-sided Jacobi.

struct JacobiParams {
    const double *rrow;  // R row-major, ld k
    double *a;           // workspace: column-major copy, ld = kp (k rounded up to even)
    unsigned *bar;       // grid-barrier counter (zeroed by the host)
    int *rot;            // [2] rotations in the current / previous sweep
    double *stats;       // out: [0] sigma_max, [1] sigma_min, [2] cond, [3] singular flag
    int k;
};

__global__ void __launch_bounds__(256) jacobi_sv_kernel(JacobiParams jp, int kp, int max_sweeps) {
    const int k = jp.k;
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int npairs = kp / 2;
    unsigned target = 0;
    // column-major copy of R (padding column kp-1 = 0 when k is odd)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kp * kp; i += gridDim.x * blockDim.x) {
        const int c = i / kp, r = i % kp;
        jp.a[i] = (r < k && c < k && r <= c) ? jp.rrow[(int64_t)r * k + c] : 0.0;
    }
    target += gridDim.x;
    grid_arrive_wait(jp.bar, target);
    const double tol = 1e-15;
    for (int sweep = 0; sweep < max_sweeps; ++sweep) {
        for (int rnd = 0; rnd < kp - 1; ++rnd) {
            for (int pi = gw; pi < npairs; pi += nw) {
                // circle method: positions 0..kp-1, position kp-1 fixed
                int a, b;
                if (pi == 0) {
                    a = kp - 1;
                    b = rnd;
                } else {
                    a = (rnd + pi) % (kp - 1);
                    b = (rnd - pi + (kp - 1)) % (kp - 1);
                }
                double *ca = jp.a + (int64_t)a * kp, *cb = jp.a + (int64_t)b * kp;
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int r = lane; r < kp; r += 32) {
                    const double x = ca[r], y = cb[r];
                    al = __fma_rn(x, x, al);
                    be = __fma_rn(y, y, be);
                    ga = __fma_rn(x, y, ga);
                }
                al = qrc::warp_sum(al);
                be = qrc::warp_sum(be);
                ga = qrc::warp_sum(ga);
                if (fabs(ga) > tol * sqrt(al * be) && ga != 0.0) {
                    const double zeta = (be - al) / (2.0 * ga);
                    const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                    const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
                    for (int r = lane; r < kp; r += 32) {
                        const double x = ca[r], y = cb[r];
                        ca[r] = c * x - s * y;
                        cb[r] = s * x + c * y;
                    }
                    if (lane == 0) atomicAdd(&jp.rot[sweep & 1], 1);
                }
            }
            target += gridDim.x;
            grid_arrive_wait(jp.bar, target);
        }
        const int done = atomicAdd(&jp.rot[sweep & 1], 0) == 0;
        target += gridDim.x;
        grid_arrive_wait(jp.bar, target);
        if (blockIdx.x == 0 && threadIdx.x == 0) jp.rot[(sweep + 1) & 1] = 0;
        target += gridDim.x;
        grid_arrive_wait(jp.bar, target);
        if (done) break;
    }
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        double smax = 0.0, smin = INFINITY;
        for (int c = 0; c < k; ++c) {
            const double *cc = jp.a + (int64_t)c * kp;
            double ss = 0.0;
            for (int r = lane; r < kp; r += 32) ss = __fma_rn(cc[r], cc[r], ss);
            ss = qrc::warp_sum(ss);
            const double sv = sqrt(ss);
            smax = fmax(smax, sv);
            smin = fmin(smin, sv);
        }
        if (lane == 0) {
            jp.stats[0] = smax;
            jp.stats[1] = smin;
            jp.stats[2] = smin > 0.0 ? smax / smin : INFINITY;
            jp.stats[3] = (smax == 0.0 || smin <= 1e-10 * smax) ? 1.0 : 0.0;  // factor.py:123-124
        }
    }
}

}  // namespace qrc

// host side, used by small_dense.cu's srlu_qr_pinv
int qr_cluster_launch(const double *mT, int64_t k1, int64_t k2, int64_t ldm, double *qa,
                      double *qtau, double *rrow, cudaStream_t st) {
    using namespace qrc;
    int C = 0;
    size_t smem = 0;
    for (int c = 2; c <= 16; c *= 2) {
        smem = QrLayout::bytes((int)k1, (int)k2, c);
        if (smem <= 200 * 1024) {
            C = c;
            break;
        }
    }
    SRLU_REQUIRE(C > 0, SRLU_ERR_UNSUPPORTED,
                 "qr_pinv: %lld x %lld does not fit one 16-CTA cluster", (long long)k2,
                 (long long)k1);
    SRLU_CUDA(cudaFuncSetAttribute(qr_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    if (C > 8)
        SRLU_CUDA(cudaFuncSetAttribute(qr_cluster_kernel,
                                       cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((unsigned)C);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SRLU_CUDA(cudaLaunchKernelEx(&cfg, qr_cluster_kernel, mT, (int)k1, (int)k2, ldm, qa, qtau,
                                 rrow));
    return SRLU_OK;
}

size_t jacobi_workspace(int64_t k) {
    const int64_t kp = (k + 1) & ~int64_t(1);
    return sizeof(double) * (size_t)(kp * kp) + 64;
}

int jacobi_launch(const double *rrow, int64_t k, void *ws, double *stats, cudaStream_t st) {
    using namespace qrc;
    const int kp = (int)((k + 1) & ~int64_t(1));
    JacobiParams jp;
    jp.rrow = rrow;
    jp.a = (double *)ws;
    jp.bar = (unsigned *)((char *)ws + sizeof(double) * (size_t)kp * kp);
    jp.rot = (int *)(jp.bar + 4);
    jp.stats = stats;
    jp.k = (int)k;
    SRLU_CUDA(cudaMemsetAsync(jp.bar, 0, 64, st));
    int dev = 0, nsm = 0, per = 0;
    SRLU_CUDA(cudaGetDevice(&dev));
    SRLU_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    SRLU_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, jacobi_sv_kernel, 256, 0));
    const int need = (kp / 2 + 7) / 8;  // one warp per pair
    int grid = need < nsm * (per > 0 ? per : 1) ? need : nsm * (per > 0 ? per : 1);
    if (grid < 1) grid = 1;
    int max_sweeps = 60;
    void *args[] = {&jp, (void *)&kp, &max_sweeps};
    SRLU_CUDA(cudaLaunchCooperativeKernel((void *)jacobi_sv_kernel, dim3(grid), dim3(256), args, 0,
                                          st));
    return SRLU_OK;
}

}  // namespace srlu
