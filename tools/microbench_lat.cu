// microbench_lat.cu -- K7: dependent-chain latencies (cycles) of the instructions on the
// persistent loop's critical path: DFMA, DADD, DDIV, SHFL (double), REDUX, LDS, L2 load.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_lat tools/microbench_lat.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void k_lat(double *out, long long *cyc, const double *g, double a0) {
    __shared__ double sm[256];
    sm[threadIdx.x] = threadIdx.x * 1e-3;
    __syncthreads();
    const int N = 256;
    double a = a0 + threadIdx.x * 1e-9, b = 1.0000001;
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) a = __fma_rn(a, b, 1e-7);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0);
    // DADD chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) a = a + b;
    t1 = clock64();
    if (threadIdx.x == 0) cyc[1] = (t1 - t0);
    // DDIV chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) a = 1.5 / (a + 1.0);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[2] = (t1 - t0);
    // SHFL (double) + DADD chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) a = a + __shfl_xor_sync(0xffffffffu, a, 1);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[3] = (t1 - t0);
    // REDUX chain
    unsigned u = threadIdx.x;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) u = __reduce_max_sync(0xffffffffu, u) + (threadIdx.x & 1);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[4] = (t1 - t0);
    // LDS chain
    int idx = threadIdx.x;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) idx = static_cast<int>(sm[idx & 255]) + ((idx + 1) & 255);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[5] = (t1 - t0);
    // L2 load chain (pointer chase over a small L2-resident array, .cg)
    const double *pp = g;
    long long j = 0;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 64; ++i) {
        double v;
        asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(pp + j));
        j = (static_cast<long long>(v) + 4099 * (i + 1)) & ((1 << 20) - 1);
    }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[6] = (t1 - t0) * 4;  // x4: report per 256 for uniform scaling
    // __syncthreads alone
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) __syncthreads();
    t1 = clock64();
    if (threadIdx.x == 0) cyc[7] = (t1 - t0);
    // clock64 overhead
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) { long long t = clock64(); if (t == 0) a += 1; }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[8] = (t1 - t0);
    // DFMA throughput: 8 independent chains x 256 threads
    double c[8];
    for (int q = 0; q < 8; ++q) c[q] = a + q;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int q = 0; q < 8; ++q) c[q] = __fma_rn(c[q], b, 1e-7);
    }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[9] = (t1 - t0);
    for (int q = 0; q < 8; ++q) a += c[q];
    out[threadIdx.x] = a + u + idx + static_cast<double>(j);
}

int main() {
    double *out, *g;
    long long *cyc;
    cudaMalloc(&out, 4096 * 8);
    cudaMalloc(&g, (1 << 20) * 8);
    cudaMemset(g, 0, (1 << 20) * 8);
    cudaMallocManaged(&cyc, 16 * 8);
    for (int thr : {32, 256}) {
        k_lat<<<1, thr>>>(out, cyc, g, 1.0);
        k_lat<<<1, thr>>>(out, cyc, g, 1.0);
        cudaDeviceSynchronize();
        const char *nm[] = {"dfma", "dadd", "ddiv", "shfl64+dadd", "redux+iadd", "lds(+cvt)", "l2_load(.cg)", "syncthreads",
                            "clock64", "dfma_tput_8chains(per 8 FMA)"};
        printf("threads=%d:", thr);
        for (int i = 0; i < 10; ++i) printf(" %s=%.1f", nm[i], cyc[i] / 256.0);
        printf("  (cycles per op)\n");
    }
    return 0;
}
