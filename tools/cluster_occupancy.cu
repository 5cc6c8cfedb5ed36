// How many thread-block clusters of size CS (1 CTA per SM, 256 threads, ~200 KB shared memory)
// can be co-resident on this GPU: cudaOccupancyMaxActiveClusters (next-step sizing for a
// hierarchical cluster exchange).   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/cluster_occupancy tools/cluster_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dummy(int *p) { if (p) p[threadIdx.x] = 0; }
int main() {
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(cs * 64);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = 200 * 1024;
        cfg.attrs = at; cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_dummy, &cfg);
        printf("cluster size %2d: max active clusters %3d -> %3d SMs busy (%s)\n", cs, n, n * cs, cudaGetErrorString(e));
    }
    return 0;
}
