// Cluster occupancy and SM -> GPC grouping on this GPU (development probe):
// max active clusters of size CS for a 1-CTA/SM kernel (227 KB smem, 512
// threads), and the SM ids that share a 16-CTA cluster (one GPC each).
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__global__ void k_dummy(int* out) {
    extern __shared__ double s[];
    if (threadIdx.x == 0) {
        unsigned smid, cid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
        s[0] = smid;
        out[2 * blockIdx.x] = smid;
        out[2 * blockIdx.x + 1] = cid;
    }
}

int main() {
    int* d;
    cudaMalloc(&d, 4096 * 8);
    const size_t smem = 227 * 1024;
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int sizes[] = {1, 2, 3, 4, 5, 6, 8, 9, 10, 12, 16};
    for (int cs : sizes) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs * 16);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_dummy, &cfg);
        printf("cluster %2d: max active clusters %3d -> %3d CTAs (%s)\n", cs, n, n * cs, cudaGetErrorString(e));
    }
    // GPC grouping: clusters of 16 (each within one GPC)
    for (int cs : {16, 8}) {
        int ncl = 0;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = smem;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(cs);
        cudaOccupancyMaxActiveClusters(&ncl, k_dummy, &cfg);
        cfg.gridDim = dim3(cs * ncl);
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_dummy, d);
        cudaDeviceSynchronize();
        int h[4096];
        cudaMemcpy(h, d, 8 * cs * ncl, cudaMemcpyDeviceToHost);
        printf("clusters of %d (%d, %s): smids per cluster\n", cs, ncl, cudaGetErrorString(e));
        for (int c = 0; c < ncl; ++c) {
            printf("  ");
            for (int i = 0; i < cs; ++i) printf("%d ", h[2 * (c * cs + i)]);
            printf("\n");
        }
    }
    return 0;
}
