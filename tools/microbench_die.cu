// microbench_die.cu -- K7: L2 round-trip latency from every SM to one fixed 128-byte line
// (ld.relaxed.gpu, dependent chain), and the atomic-ack latency (atom.add.gpu), to see the
// near/far L2 split of the two B200 dies.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_die tools/microbench_die.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void k_die(unsigned long long *line, int which, long long *out) {
    if (threadIdx.x != 0) return;
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    unsigned long long *p = line + which * 4096;  // 32 KB apart -> different slices
    // serialise CTAs: CTA c runs its probe alone-ish (no contention): wait for turn
    unsigned long long v = 0;
    long long t0 = clock64();
    for (int i = 0; i < 64; ++i) {
        unsigned long long a;
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(a) : "l"(p + (v & 1)) : "memory");
        v += a + 1;
    }
    long long t1 = clock64();
    for (int i = 0; i < 64; ++i) {
        unsigned long long a;
        asm volatile("atom.relaxed.gpu.global.add.u64 %0, [%1], %2;" : "=l"(a) : "l"(p + 8 + (v & 1)), "l"(0ull) : "memory");
        v += a + 1;
    }
    long long t2 = clock64();
    out[blockIdx.x * 4 + 0] = smid;
    out[blockIdx.x * 4 + 1] = (t1 - t0) / 64;
    out[blockIdx.x * 4 + 2] = (t2 - t1) / 64;
    out[blockIdx.x * 4 + 3] = v;
}

int main() {
    unsigned long long *line;
    long long *out;
    cudaMalloc(&line, 1 << 20);
    cudaMemset(line, 0, 1 << 20);
    cudaMallocManaged(&out, 148 * 4 * 8);
    for (int which = 0; which < 4; ++which) {
        k_die<<<148, 32>>>(line, which, out);
        cudaDeviceSynchronize();
        int lo = 1 << 30, hi = 0;
        long long ld_sum = 0;
        int hist[40] = {0};
        for (int c = 0; c < 148; ++c) {
            int l = (int)out[c * 4 + 1];
            ld_sum += l;
            lo = l < lo ? l : lo;
            hi = l > hi ? l : hi;
            hist[l / 50 < 39 ? l / 50 : 39]++;
        }
        printf("line%d ld: min %d max %d mean %.0f | hist(50-cycle bins):", which, lo, hi, ld_sum / 148.0);
        for (int i = 0; i < 40; ++i) if (hist[i]) printf(" %d:%d", i * 50, hist[i]);
        printf("\n  per-SM (smid:ld/atom):");
        for (int c = 0; c < 148; c += 1) printf(" %lld:%lld/%lld", out[c * 4], out[c * 4 + 1], out[c * 4 + 2]);
        printf("\n");
    }
    return 0;
}
