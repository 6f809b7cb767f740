// All-to-all exchange latency inside one 16-CTA cluster, as the cluster LU
// does it per pivot step: every CTA pushes NP 16-byte items to every CTA
// with st.async (complete_tx on the receiver's mbarrier), then waits on its
// own mbarrier.  Three slots, re-armed after each wait.
// nvcc -cudart shared -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/bench_xchg.cu -o tools/bin/bench_xchg
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ long long g_cyc;
__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa_rank(unsigned a, unsigned r) {
    unsigned o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o;
}

template <int MODE>
__global__ void kern(int iters, int np) {
    __shared__ __align__(16) double buf[3][16][34];
    __shared__ __align__(8) uint64_t bar[3];
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank(), CL = cl.num_blocks();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned bytes = CL * np * 16;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 3; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < 3; ++i)
            asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[i])), "r"(bytes) : "memory");
    }
    cl.sync();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int sl = it % 3;
        if (warp == (it % (blockDim.x >> 5)) && lane < (int)CL) {  // one warp, lane = destination
            const unsigned rb = mapa_rank(su32(&bar[sl]), lane);
            const unsigned rr = mapa_rank(su32(&buf[sl][rank][0]), lane);
            for (int i = 0; i < np; ++i)
                asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
                             ::"r"(rr + 16u * i), "d"((double)it), "d"(1.0), "r"(rb) : "memory");
        }
        asm volatile("{ .reg .pred p; W_%=: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1; @!p bra W_%=; }"
                     ::"r"(su32(&bar[sl])), "r"((unsigned)((it / 3) & 1)) : "memory");
        if (threadIdx.x == 0)
            asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[sl])), "r"(bytes) : "memory");
        if (MODE == 1) __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && rank == 0) g_cyc = (t1 - t0) / iters;
    cl.sync();
}

int main() {
    for (int mode = 0; mode < 2; ++mode)
        for (int threads : {256, 1024})
            for (int np : {1, 6, 12}) {
                cudaLaunchConfig_t cfg = {};
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = 16; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
                cfg.gridDim = dim3(16); cfg.blockDim = dim3(threads); cfg.attrs = attr; cfg.numAttrs = 1;
                auto k = mode ? kern<1> : kern<0>;
                cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                cudaLaunchKernelEx(&cfg, k, 3000, np);
                cudaDeviceSynchronize();
                long long c; cudaMemcpyFromSymbol(&c, g_cyc, sizeof(c));
                printf("mode %d (%s) threads %4d items/dst %2d: %lld cycles per exchange  %s\n", mode,
                       mode ? "+syncthreads" : "plain", threads, np, c, cudaGetErrorString(cudaGetLastError()));
            }
    return 0;
}
