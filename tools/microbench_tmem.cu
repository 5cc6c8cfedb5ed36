// microbench_tmem.cu -- K7: tensor-memory (TMEM) read bandwidth per SM with tcgen05.ld, to
// decide whether A~ rows beyond shared memory can live in TMEM (C4 at 1 GPU: 80 MB of A~ vs
// 148 x 227 KB SMEM).  One CTA per SM; 4/8/16 warps; each warp repeatedly loads its lane
// quarter (32 lanes x 32 columns x 4 B = 4 KB per tcgen05.ld.32x32b.x32).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_tmem tools/microbench_tmem.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void k_tmem_read(int reps, unsigned long long *cycles, double *sink) {
    __shared__ uint32_t taddr_s;
    const int warp = threadIdx.x >> 5;
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
    const uint32_t lane_base = static_cast<uint32_t>(32 * (warp & 3)) << 16;
    // each warp of the same quadrant reads a different 128-column slice
    const uint32_t col0 = static_cast<uint32_t>((warp >> 2) * 128) & 511u;
    uint32_t acc = 0;
    __syncthreads();
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int c = 0; c < 128; c += 32) {
            uint32_t v[32];
            const uint32_t ta = base + lane_base + ((col0 + c) & 511u);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                  "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                  "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(ta));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < 32; ++i) acc ^= v[i];
        }
    }
    const long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) cycles[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
    if (acc == 0x12345678u) *sink = acc;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base) : "memory");
}

int main() {
    unsigned long long *cyc;
    double *sink;
    cudaMallocManaged(&cyc, 148 * sizeof(unsigned long long));
    cudaMalloc(&sink, 8);
    const int reps = 2000;
    for (int warps : {4, 8, 16}) {
        k_tmem_read<<<148, warps * 32>>>(10, cyc, sink);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        k_tmem_read<<<148, warps * 32>>>(reps, cyc, sink);
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        double mx = 0;
        for (int i = 0; i < 148; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
        const double bytes = static_cast<double>(warps) * reps * 4 * 4096.0;  // per CTA
        printf("tmem_read warps=%d bytes_per_cycle_per_SM %.1f\n", warps, bytes / mx);
    }
    return 0;
}
