// microbench_xdie.cu -- K7: the per-iteration atomic exchange (red.max key + red.release.add
// count, spin on a 16-byte {count, max} pair) with ONE pair vs one pair PER DIE (each CTA
// updates the pair homed on its own die and polls both), G = 148 CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_xdie tools/microbench_xdie.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ void red_max(unsigned long long *p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add_rel(unsigned long long *p, unsigned long long v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void ld2(const unsigned long long *p, unsigned long long &a, unsigned long long &b) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ void st2(unsigned long long *p, unsigned long long a, unsigned long long b) {
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1,%2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ long long atom_lat(unsigned long long *p) {
    // 16 dependent atomics (the address depends on the previous result), mean latency
    unsigned long long v = 0;
    long long t0 = clock64();
    for (int i = 0; i < 16; ++i) {
        unsigned long long a;
        asm volatile("atom.relaxed.gpu.global.add.u64 %0, [%1], %2;" : "=l"(a) : "l"(p + (v & 1)), "l"(0ull) : "memory");
        v += a + 2;
    }
    long long t1 = clock64();
    return (t1 - t0) / 16 + (long long)(v & 0x100000000000ull);
}

// lines: [0] probe line A, [16*j] pairs. die[c] computed in-kernel (staggered probes).
// MODE 0: one pair for all; MODE 1: pair per die; MODE 2: MODE 1 + slot store before release
template <int MODE>
__global__ void k_x(unsigned long long *w, int iters, long long *out, int *dies) {
    const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
    __shared__ int die_s, gd0, gd1;
    if (tid == 0) {
        int *turn = (int *)(w + 8192 + 48);
        while (atomicAdd(turn, 0) != c) {
        }
        long long la = atom_lat(w + 4096);  // line A defines die 0 (= SMs near line A)
        die_s = la < 520 ? 0 : 1;
        dies[c] = die_s;
        if (c == 0) {
            // pair lines: home(L) == home(A) iff near(me, L) == near(me, A)
            int f0 = -1, f1 = -1;
            for (int j = 1; j < 64 && (f0 < 0 || f1 < 0); ++j) {
                const bool near = atom_lat(w + 4096 + 16 * 3 * j) < 520;
                const bool same = near == (die_s == 0);
                if (same && f0 < 0) f0 = j;
                if (!same && f1 < 0) f1 = j;
            }
            ((int *)(w + 8192 + 64))[0] = f0;
            ((int *)(w + 8192 + 64))[1] = f1;
        }
        atomicAdd((int *)(w + 8192 + die_s * 16), 1);
        __threadfence();
        atomicAdd(turn, 1);
        while (atomicAdd(turn, 0) < G) {
        }
        gd0 = atomicAdd((int *)(w + 8192), 0);
        gd1 = atomicAdd((int *)(w + 8192 + 16), 0);
    }
    __syncthreads();
    const int die = die_s;
    const bool PD = MODE == 1 || MODE == 2;
    const unsigned long long G0 = PD ? gd0 : G, G1 = PD ? gd1 : 0;
    // pair lines: die 0 pairs must be homed on die 0: line A (w+4096) is near die 0 by definition;
    // find a die-1 line: we use lines A + 16*j and let die-1 CTAs... (simplification: pair bases)
    const int f0 = ((volatile int *)(w + 8192 + 64))[0], f1 = ((volatile int *)(w + 8192 + 64))[1];
    unsigned long long *base0 = w + 4096 + 16 * 3 * (PD ? f0 : 1);   // homed on die 0
    unsigned long long *base1 = w + 4096 + 16 * 3 * (f1 < 0 ? 2 : f1);  // homed on die 1
    long long t0 = clock64();
    for (int it = 1; it <= iters; ++it) {
        const int e = it % 3;
        unsigned long long *p0 = base0 + e * 2;
        unsigned long long *p1 = base1 + e * 2;
        if (tid == 0) {
            unsigned long long *mine = (PD && die) ? p1 : p0;
            if (c == 0) {
                st2(base0 + ((it + 1) % 3) * 2, 0, 0);
                if (PD) st2(base1 + ((it + 1) % 3) * 2, 0, 0);
            }
            if (MODE == 2) st2(w + 12288 + c * 4, it, it);
            const unsigned long long key = ((unsigned long long)((c * 2654435761u) ^ (it * 40503u)) << 16) | (unsigned)c;
            if (MODE != 5 && MODE != 6) red_max(mine + 1, key);
            if (MODE == 4 || MODE == 6) asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(mine), "l"(1ull) : "memory");
            else red_add_rel(mine, 1ull);
            unsigned long long a0, m0, a1 = 0, m1 = 0;
            do {
                ld2(p0, a0, m0);
                if (PD) ld2(p1, a1, m1);
            } while (a0 < G0 || a1 < G1);
            if (MODE != 3) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        __syncthreads();
    }
    if (c == 0 && tid == 0) out[0] = clock64() - t0;
}

int main() {
    unsigned long long *w;
    long long *out;
    int *dies;
    cudaMalloc(&w, 1 << 20);
    cudaMallocManaged(&out, 64);
    cudaMallocManaged(&dies, 148 * 4);
    const int iters = 4000;
    for (int mode = 0; mode < 7; ++mode) {
        for (int rep = 0; rep < 1; ++rep) {
            cudaMemset(w, 0, 1 << 20);
            void *args[] = {&w, (void *)&iters, &out, &dies};
            int it = iters;
            args[1] = &it;
            void *fns[] = {(void *)k_x<0>, (void *)k_x<1>, (void *)k_x<2>, (void *)k_x<3>, (void *)k_x<4>, (void *)k_x<5>, (void *)k_x<6>};
            void *fn = fns[mode];
            cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(148), dim3(256), args, 0, 0);
            if (e == cudaSuccess) e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            int n0 = 0;
            for (int c = 0; c < 148; ++c) n0 += dies[c] == 0;
            int f0 = 0, f1 = 0;
            cudaMemcpy(&f0, (int *)(w + 8192 + 64), 4, cudaMemcpyDeviceToHost);
            cudaMemcpy(&f1, (int *)(w + 8192 + 64) + 1, 4, cudaMemcpyDeviceToHost);
            printf("lines f0=%d f1=%d ", f0, f1);
            printf("mode %d (%s): %.0f cycles/iter  (die0 CTAs %d)\n", mode,
                   (const char *[]){"one pair", "pair per die", "pair per die + slot store", "one pair, no fence", "one pair, relaxed add", "count only (release)", "count only (relaxed)"}[mode], (double)out[0] / iters, n0);
        }
    }
    return 0;
}
