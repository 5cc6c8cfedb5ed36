// microbench_dfma.cu -- K7: FP64 FMA (DFMA) throughput per SM on B200: 148 CTAs, W warps,
// 8 independent fma chains per thread.  Prints DFMA/clk/SM and the chip FP64 TFLOP/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_dfma tools/microbench_dfma.cu
#include <cuda_runtime.h>
#include <stdio.h>

__global__ void k_dfma(int reps, long long *cyc, double *out) {
    double c[8];
    for (int q = 0; q < 8; ++q) c[q] = threadIdx.x * 1e-3 + q;
    const double b = 1.0000001, a = 1e-9;
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int q = 0; q < 8; ++q) c[q] = __fma_rn(c[q], b, a);
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    double s = 0;
    for (int q = 0; q < 8; ++q) s += c[q];
    if (s == 1234.5) *out = s;
}

int main() {
    long long *cyc;
    double *out;
    cudaMallocManaged(&cyc, 148 * 8);
    cudaMalloc(&out, 8);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int thr : {128, 256, 512, 1024}) {
        const int reps = 4096;
        k_dfma<<<148, thr>>>(16, cyc, out);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k_dfma<<<148, thr>>>(reps, cyc, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
        const double fma_per_sm = (double)thr * reps * 8;
        printf("dfma threads=%d: %.1f DFMA/clk/SM, %.2f TFLOP/s (events, %.0f MHz nominal clock)\n", thr,
               fma_per_sm / mx, 2.0 * fma_per_sm * 148 / (ms * 1e-3) / 1e12, clk / 1e3);
    }
    return 0;
}
