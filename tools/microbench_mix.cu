// microbench_mix.cu -- do TMEM reads (tcgen05.ld) and shared-memory reads (LDS.128) share a
// per-SM bottleneck?  One CTA of 8 warps per SM.  Mode 0: 8 warps read TMEM; mode 1: 8 warps read
// shared memory; mode 2: warps 0-3 read TMEM while warps 4-7 read shared memory.  Each warp
// folds what it reads (xor) so the loads cannot be dropped; bytes / cycle per SM per group.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_mix tools/microbench_mix.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void __launch_bounds__(256, 1) k_mix(int mode, int reps, unsigned long long *cycles, double *sink) {
    extern __shared__ __align__(16) unsigned char sm[];  // 128 KB
    __shared__ uint32_t taddr_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 128 * 1024 / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(sm)[i] = make_uint4(i, i + 1, i + 2, i + 3);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(&taddr_s)))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t base = taddr_s;
    const bool tm = mode == 0 || (mode == 2 && warp < 4);
    uint32_t acc = 0;
    __syncthreads();
    const long long t0 = clock64();
    if (tm) {
        const uint32_t lane_base = static_cast<uint32_t>(32 * (warp & 3)) << 16;
        const uint32_t col0 = static_cast<uint32_t>((warp >> 2) * 256) & 511u;
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int c = 0; c < 256; c += 32) {
                uint32_t v[32];
                const uint32_t ta = base + lane_base + ((col0 + c) & 511u);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                      "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                      "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                      "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                      "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                    : "r"(ta));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int i = 0; i < 32; ++i) acc ^= v[i];
            }
        }
    } else {
        // the same bytes per warp per rep as the TMEM path (8 x 4 KB), conflict-free LDS.128
        const uint4 *p = reinterpret_cast<const uint4 *>(sm) + (warp & 3) * 2048 + lane;
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int c = 0; c < 64; ++c) {
                const uint4 v = p[((c + r) * 32) & 2047];
                acc ^= v.x ^ v.y ^ v.z ^ v.w;
            }
        }
    }
    const long long t1 = clock64();
    cycles[blockIdx.x * 8 + warp] = static_cast<unsigned long long>(t1 - t0);
    if (acc == 0x12345678u) *sink = acc;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base) : "memory");
}

int main() {
    unsigned long long *cyc;
    double *sink;
    cudaMallocManaged(&cyc, 148 * 8 * sizeof(unsigned long long));
    cudaMalloc(&sink, 8);
    cudaFuncSetAttribute(k_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
    const int reps = 2000;
    const char *names[] = {"tmem x8", "lds x8", "tmem x4 + lds x4"};
    for (int mode = 0; mode < 3; ++mode) {
        k_mix<<<148, 256, 128 * 1024>>>(mode, 10, cyc, sink);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        k_mix<<<148, 256, 128 * 1024>>>(mode, reps, cyc, sink);
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        double mt = 0, ml = 0;  // slowest warp of each kind (SM 0)
        for (int w = 0; w < 8; ++w) {
            const bool tm = mode == 0 || (mode == 2 && w < 4);
            double c = static_cast<double>(cyc[w]);
            if (tm) mt = c > mt ? c : mt; else ml = c > ml ? c : ml;
        }
        const double per_warp = static_cast<double>(reps) * 8 * 4096.0;
        const int nt = mode == 0 ? 8 : mode == 2 ? 4 : 0, nl = 8 - nt;
        printf("%-18s TMEM %.1f B/clk (%d warps, %.0f cyc)  LDS %.1f B/clk (%d warps, %.0f cyc)\n", names[mode],
               nt ? nt * per_warp / mt : 0.0, nt, mt, nl ? nl * per_warp / ml : 0.0, nl, ml);
    }
    return 0;
}
