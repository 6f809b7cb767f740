// Can a cooperative launch carry cluster dimensions on this device, how many
// 16-/8-CTA clusters (1024 threads, ~170 KB smem) are co-resident, and does
// grid.sync() work across them?
// nvcc -cudart shared -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/probe_coop_cluster.cu -o tools/bin/probe_coop_cluster
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__device__ int g_count[4];
__global__ void kern(int rounds) {
    extern __shared__ double sm[];
    cg::grid_group g = cg::this_grid();
    cg::cluster_group cl = cg::this_cluster();
    for (int r = 0; r < rounds; ++r) {
        if (threadIdx.x == 0) atomicAdd(&g_count[r & 3], 1);
        g.sync();
        cl.sync();
    }
    sm[threadIdx.x] = 1.0;
}
int main() {
    int dev = 0, nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = 170 * 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int CL : {16, 8, 4}) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CL; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeCooperative;
        attr[1].val.cooperative = 1;
        cfg.blockDim = dim3(1024);
        cfg.dynamicSmemBytes = smem;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(CL);
        int ncl = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, (void *)kern, &cfg);
        printf("CL=%d: max active clusters %d (%s) -> %d CTAs of %d SMs\n", CL, ncl, cudaGetErrorString(e), ncl * CL, nsm);
        if (ncl < 1) continue;
        cfg.gridDim = dim3(ncl * CL);
        cfg.numAttrs = 2;
        int zero[4] = {0, 0, 0, 0};
        cudaMemcpyToSymbol(g_count, zero, sizeof(zero));
        e = cudaLaunchKernelEx(&cfg, kern, 8);
        cudaError_t e2 = cudaDeviceSynchronize();
        int c[4];
        cudaMemcpyFromSymbol(c, g_count, sizeof(c));
        printf("   coop+cluster launch of %d CTAs: launch=%s sync=%s counts %d %d %d %d\n", ncl * CL,
               cudaGetErrorString(e), cudaGetErrorString(e2), c[0], c[1], c[2], c[3]);
    }
    return 0;
}
