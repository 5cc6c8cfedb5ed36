// microbench.cu -- K7: B200 building-block latencies/bandwidths that set
// the roofline denominators and the exchange design of the persistent solve kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
// Prints one "name value unit" line per measurement.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

namespace cg = cooperative_groups;

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e = (x);                                                       \
        if (e != cudaSuccess) {                                                    \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                               \
        }                                                                          \
    } while (0)

__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t *p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// 1) ping-pong between CTA 0 and CTA b through global memory: round trip per iteration
__global__ void k_pingpong(uint64_t *flags, int iters, long long *out) {
    if (threadIdx.x != 0) return;
    if (blockIdx.x != 0 && blockIdx.x != gridDim.x - 1) return;
    uint64_t *a = flags, *b = flags + 32;
    long long t0 = clock64();
    for (int i = 1; i <= iters; ++i) {
        if (blockIdx.x == 0) {
            st_relaxed(a, i);
            while (ld_relaxed(b) != (uint64_t)i) {
            }
        } else {
            while (ld_relaxed(a) != (uint64_t)i) {
            }
            st_relaxed(b, i);
        }
    }
    if (blockIdx.x == 0) out[0] = clock64() - t0;
}

// 2) all-to-all push exchange among G CTAs (our solve exchange without payload)
__global__ void k_alltoall(uint64_t *inbox, int iters, long long *out) {
    const int G = gridDim.x, c = blockIdx.x, lane = threadIdx.x;
    long long t0 = clock64();
    for (int i = 1; i <= iters; ++i) {
        uint64_t *par = inbox + (size_t)(i & 1) * G * G * 8;
        for (int r = lane; r < G; r += 32) st_relaxed(par + ((size_t)r * G + c) * 8, i);
        for (int w = lane; w < G; w += 32)
            while (ld_relaxed(par + ((size_t)c * G + w) * 8) != (uint64_t)i) {
            }
        __syncwarp();
    }
    if (c == 0 && lane == 0) out[0] = clock64() - t0;
}

// 3) central-counter barrier (atomicAdd + spin) among G CTAs
__global__ void k_counter(unsigned int *ctr, int iters, long long *out) {
    const int G = gridDim.x;
    long long t0 = clock64();
    for (int i = 1; i <= iters; ++i) {
        if (threadIdx.x == 0) {
            atomicAdd(ctr, 1u);
            while (atomicAdd(ctr, 0u) < (unsigned)(i * G)) {
            }
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

// 4) cooperative-groups grid sync
__global__ void k_gridsync(int iters, long long *out) {
    cg::grid_group g = cg::this_grid();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

// 5) cluster barrier latency
__global__ void k_clusterbar(int iters, long long *out) {
    cg::cluster_group cl = cg::this_cluster();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) cl.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

// 6) DSMEM ping-pong between rank 0 and rank 1 of a cluster
__global__ void k_dsmem_pingpong(int iters, long long *out) {
    __shared__ volatile uint64_t flag[2];
    cg::cluster_group cl = cg::this_cluster();
    if (threadIdx.x == 0) { flag[0] = 0; flag[1] = 0; }
    cl.sync();
    const unsigned rank = cl.block_rank();
    long long t0 = clock64();
    if (threadIdx.x == 0 && rank < 2) {
        volatile uint64_t *peer = (volatile uint64_t *)cl.map_shared_rank((uint64_t *)flag, rank ^ 1);
        for (int i = 1; i <= iters; ++i) {
            if (rank == 0) {
                peer[0] = i;
                while (flag[1] != (uint64_t)i) {
                }
            } else {
                while (flag[0] != (uint64_t)i) {
                }
                peer[1] = i;
            }
        }
    }
    if (rank == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
    cl.sync();
}

// 7) streaming read bandwidth: every CTA reads its slice `reps` times
__global__ void k_read(const double2 *__restrict__ a, size_t n2, int reps, double *sink) {
    double s = 0.0;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
            double2 v;
            asm("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(a + i));
            s += v.x + v.y;
        }
    if (s == 12345.678) *sink = s;
}

// 8) shared-memory read bandwidth per SM
__global__ void k_smem(int reps, double *sink) {
    extern __shared__ double2 buf[];
    const int nb = 12288;  // 192 KB
    for (int i = threadIdx.x; i < nb; i += blockDim.x) buf[i] = make_double2(i, i);
    __syncthreads();
    double s = 0.0;
    for (int r = 0; r < reps; ++r)
        for (int i = threadIdx.x; i < nb; i += blockDim.x) {
            double2 v = buf[i];
            s += v.x + v.y;
        }
    if (s == 12345.678) *sink = s;
}

static float time_kernel(void (*launch)(void *), void *arg) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    launch(arg);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a));
    launch(arg);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms;
}

int main() {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    const int sms = prop.multiProcessorCount;
    int clk_khz = 0;
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
    printf("device %s sms %d l2_bytes %d smem_optin %zu clock_khz %d\n", prop.name, sms, prop.l2CacheSize,
           prop.sharedMemPerBlockOptin, clk_khz);
    long long *out;
    CK(cudaMallocManaged(&out, 64));
    uint64_t *flags;
    CK(cudaMalloc(&flags, 2 * 160 * 160 * 64));
    const int iters = 2000;

    for (int far : {1, 74, 147}) {
        CK(cudaMemset(flags, 0, 4096));
        // CTA b lands on some SM; the grid is 2 CTAs but we vary which is the partner via grid size
        int grid = far + 1;
        k_pingpong<<<grid, 32>>>(flags, iters, out);  // CTA 0 <-> CTA grid-1
        CK(cudaDeviceSynchronize());
        printf("pingpong_rt_cycles_grid%d %.1f cycles\n", grid, (double)out[0] / iters);
    }
    for (int G : {8, 16, 32, 74, 148}) {
        CK(cudaMemset(flags, 0, (size_t)2 * G * G * 64));
        k_alltoall<<<G, 32>>>(flags, iters, out);
        CK(cudaDeviceSynchronize());
        printf("alltoall_push_G%d %.1f cycles/iter\n", G, (double)out[0] / iters);
    }
    for (int G : {16, 148}) {
        CK(cudaMemset(flags, 0, 64));
        k_counter<<<G, 32>>>((unsigned *)flags, iters, out);
        CK(cudaDeviceSynchronize());
        printf("counter_barrier_G%d %.1f cycles/iter\n", G, (double)out[0] / iters);
    }
    {
        int it = iters;
        void *args[] = {&it, &out};
        CK(cudaLaunchCooperativeKernel((void *)k_gridsync, dim3(sms), dim3(256), args, 0, 0));
        CK(cudaDeviceSynchronize());
        printf("grid_sync_G%d %.1f cycles/iter\n", sms, (double)out[0] / iters);
    }
    for (int cs : {2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(128);
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (cs > 8) CK(cudaFuncSetAttribute(k_clusterbar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_clusterbar, iters, out);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("cluster_sync_cs%d error %s\n", cs, cudaGetErrorString(e)); cudaGetLastError(); continue; }
        printf("cluster_sync_cs%d %.1f cycles/iter\n", cs, (double)out[0] / iters);
        int ncl = 0;
        cfg.gridDim = dim3(cs * 64);
        cfg.dynamicSmemBytes = 0;
        CK(cudaOccupancyMaxActiveClusters(&ncl, (void *)k_clusterbar, &cfg));
        printf("max_active_clusters_cs%d_smallsmem %d\n", cs, ncl);
    }
    {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(2);
        cfg.blockDim = dim3(32);
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, k_dsmem_pingpong, iters, out));
        CK(cudaDeviceSynchronize());
        printf("dsmem_pingpong_rt %.1f cycles\n", (double)out[0] / iters);
    }
    // occupancy of big-smem clusters
    for (int cs : {2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(cs * 64);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = 200 * 1024;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CK(cudaFuncSetAttribute(k_clusterbar, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        int ncl = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, (void *)k_clusterbar, &cfg);
        printf("max_active_clusters_cs%d_200KB %d %s\n", cs, ncl, e == cudaSuccess ? "" : cudaGetErrorString(e));
        cudaGetLastError();
    }
    // bandwidths
    double *sink;
    CK(cudaMalloc(&sink, 8));
    for (size_t mb : {16, 48, 80, 100, 4096}) {
        size_t bytes = mb << 20;
        double2 *a;
        CK(cudaMalloc(&a, bytes));
        CK(cudaMemset(a, 0, bytes));
        size_t n2 = bytes / 16;
        int reps = mb >= 1024 ? 3 : 40;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        k_read<<<sms * 4, 512>>>(a, n2, 1, sink);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        k_read<<<sms * 4, 512>>>(a, n2, reps, sink);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("read_bw_%zuMB %.1f GB/s\n", mb, (double)bytes * reps / (ms * 1e-3) / 1e9);
        CK(cudaFree(a));
    }
    {
        CK(cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        int reps = 200;
        k_smem<<<sms, 1024, 200 * 1024>>>(1, sink);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        k_smem<<<sms, 1024, 200 * 1024>>>(reps, sink);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("smem_read_bw_chip %.1f GB/s\n", (double)sms * 192 * 1024 * reps / (ms * 1e-3) / 1e9);
    }
    return 0;
}
