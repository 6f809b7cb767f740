// Cluster barrier cost on B200: bare cluster.sync, with a one-warp DSMEM push
// before it, and with the arrive/wait split (relaxed arrive + wait).
// nvcc -cudart shared -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/bench_cluster.cu -o tools/bin/bench_cluster
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ long long g_t[4];

template <int MODE>
__global__ void kern(int iters, int items) {
    __shared__ double buf[2][16][32];
    cg::cluster_group cl = cg::this_cluster();
    const int rank = cl.block_rank(), CL = cl.num_blocks();
    cl.sync();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int slot = it & 1;
        if (MODE >= 1 && (threadIdx.x >> 5) == (it % (blockDim.x >> 5))) {
            const int lane = threadIdx.x & 31;
            for (int t = lane; t < CL * items; t += 32) {
                const int dst = t / items, i = t % items;
                double *r = cl.map_shared_rank(&buf[slot][rank][0], dst);
                r[i] = (double)it;
            }
        }
        if (MODE == 2) {
            asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
            asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
        } else {
            cl.sync();
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && rank == 0) g_t[MODE] = (t1 - t0) / iters;
}

int main() {
    for (int threads : {256, 1024}) {
        for (int mode = 0; mode < 3; ++mode) {
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 16;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.gridDim = dim3(16);
            cfg.blockDim = dim3(threads);
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            void (*k)(int, int) = mode == 0 ? kern<0> : mode == 1 ? kern<1> : kern<2>;
            cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, k, 2000, 23);
            cudaDeviceSynchronize();
            long long t[4];
            cudaMemcpyFromSymbol(t, g_t, sizeof(t));
            printf("threads %4d mode %d (%s): %lld cycles/iter  %s\n", threads, mode,
                   mode == 0 ? "bare cluster.sync" : mode == 1 ? "push 368 + sync" : "push + relaxed arrive/wait",
                   t[mode], cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
