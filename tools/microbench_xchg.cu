// microbench_xchg.cu -- K7: latency of the per-iteration global exchange patterns a flat
// (cluster-free) persistent CSK loop would use, at G CTAs (1 per SM), 256 threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_xchg tools/microbench_xchg.cu
// Each iteration: every CTA publishes a tagged 64-byte slot (LL-style: tag in every 8-byte
// word), warp 0 polls all G slots until every tag is current, combines (argmax), then
// __syncthreads.  Variants add the winner-row fetch (n doubles from an L2-resident matrix).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e = (x);                                                                   \
        if (e != cudaSuccess) {                                                                \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);     \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

__device__ __forceinline__ void st_v2(uint64_t *p, uint64_t a, uint64_t b) {
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1,%2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_v2(const uint64_t *p, uint64_t &a, uint64_t &b) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

// mode 0: warp 0 polls all slots.  mode 1: every warp polls G/W slots, combine via smem.
// fetch_n > 0: after the winner is known, every thread loads its share of a row of fetch_n
// doubles (index = winner) from `mat` and sums it (the x update).
template <int MODE>
__global__ void k_flat(uint64_t *slots, const double *mat, int fetch_n, int iters, long long *out,
                       double *sink) {
    const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W = blockDim.x >> 5;
    __shared__ uint64_t best[32];
    __shared__ int winner;
    double acc = 0.0;
    long long t0 = clock64();
    for (int it = 1; it <= iters; ++it) {
        const uint32_t tag = static_cast<uint32_t>(it);
        uint64_t *par = slots + static_cast<size_t>(it & 1) * G * 8;
        // pseudo-random candidate key per CTA
        const uint32_t key = (c * 2654435761u) ^ (it * 40503u);
        if (tid == 0) {
            uint64_t *s = par + static_cast<size_t>(c) * 8;
            const uint64_t w = (static_cast<uint64_t>(key) << 32) | tag;
            const uint64_t wi = (static_cast<uint64_t>(c) << 32) | tag;
            st_v2(s, w, w);
            st_v2(s + 2, w, w);
            st_v2(s + 4, w, w);
            st_v2(s + 6, wi, w);
        }
        if (MODE == 0) {
            if (warp == 0) {
                uint64_t bk = 0;
                for (int j = lane; j < G; j += 32) {
                    uint64_t a, b, c2, d, e, f, g, h;
                    do {
                        ld_v2(par + static_cast<size_t>(j) * 8, a, b);
                        ld_v2(par + static_cast<size_t>(j) * 8 + 2, c2, d);
                        ld_v2(par + static_cast<size_t>(j) * 8 + 4, e, f);
                        ld_v2(par + static_cast<size_t>(j) * 8 + 6, g, h);
                    } while ((uint32_t)a != tag || (uint32_t)b != tag || (uint32_t)c2 != tag || (uint32_t)d != tag ||
                             (uint32_t)e != tag || (uint32_t)f != tag || (uint32_t)g != tag || (uint32_t)h != tag);
                    const uint64_t k2 = ((a >> 32) << 32) | (g >> 32);
                    if (k2 > bk) bk = k2;
                }
                for (int o = 16; o; o >>= 1) {
                    uint64_t v = __shfl_xor_sync(0xffffffffu, bk, o);
                    if (v > bk) bk = v;
                }
                if (lane == 0) winner = static_cast<int>(bk & 0xffffffffu);
            }
        } else {
            uint64_t bk = 0;
            for (int j = tid; j < G; j += blockDim.x) {
                uint64_t a, b, c2, d, e, f, g, h;
                do {
                    ld_v2(par + static_cast<size_t>(j) * 8, a, b);
                    ld_v2(par + static_cast<size_t>(j) * 8 + 2, c2, d);
                    ld_v2(par + static_cast<size_t>(j) * 8 + 4, e, f);
                    ld_v2(par + static_cast<size_t>(j) * 8 + 6, g, h);
                } while ((uint32_t)a != tag || (uint32_t)b != tag || (uint32_t)c2 != tag || (uint32_t)d != tag ||
                         (uint32_t)e != tag || (uint32_t)f != tag || (uint32_t)g != tag || (uint32_t)h != tag);
                const uint64_t k2 = ((a >> 32) << 32) | (g >> 32);
                if (k2 > bk) bk = k2;
            }
            for (int o = 16; o; o >>= 1) {
                uint64_t v = __shfl_xor_sync(0xffffffffu, bk, o);
                if (v > bk) bk = v;
            }
            if (lane == 0) best[warp] = bk;
            __syncthreads();
            if (warp == 0) {
                bk = lane < W ? best[lane] : 0;
                for (int o = 16; o; o >>= 1) {
                    uint64_t v = __shfl_xor_sync(0xffffffffu, bk, o);
                    if (v > bk) bk = v;
                }
                if (lane == 0) winner = static_cast<int>(bk & 0xffffffffu);
            }
        }
        __syncthreads();
        if (fetch_n > 0) {
            const double *row = mat + static_cast<size_t>(winner * 7919 % 5000) * fetch_n;
            for (int q = tid; q < fetch_n; q += blockDim.x) {
                double v;
                asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(row + q));
                acc += v;
            }
            __syncthreads();
        }
    }
    if (c == 0 && tid == 0) out[0] = clock64() - t0;
    if (acc == 1234.5) *sink = acc;
}


// atomic exchange: red.max of a 64-bit key + red.release.add of a counter in the same 16-byte
// pair, spin with a 16-byte acquire load of {count, max}.  PAIR=false: count and max in
// different lines, a second (relaxed) load of max after the count completes.
// fetch_n > 0: then every thread loads its share of the winner row (the x update).
template <bool PAIR>
__global__ void k_atomic(unsigned long long *w, const double *mat, int fetch_n, int iters, long long *out,
                         double *sink) {
    const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
    __shared__ unsigned long long win;
    double acc = 0.0;
    long long t0 = clock64();
    for (int it = 1; it <= iters; ++it) {
        unsigned long long *cnt = w + (PAIR ? 0 : 0);
        unsigned long long *mx = w + (PAIR ? 1 + 2 * (it % 3) : 64 + 16 * (it % 3));
        if (PAIR) cnt = w + 2 * (it % 3);
        else cnt = w + 16 * (it % 3);
        if (tid == 0) {
            if (c == 0) {  // reset the slot two iterations ahead
                unsigned long long *nc = PAIR ? w + 2 * ((it + 1) % 3) : w + 16 * ((it + 1) % 3);
                unsigned long long *nm = PAIR ? nc + 1 : w + 64 + 16 * ((it + 1) % 3);
                asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(nc), "l"(0ull) : "memory");
                asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(nm), "l"(0ull) : "memory");
            }
            const unsigned long long key = ((unsigned long long)((c * 2654435761u) ^ (it * 40503u)) << 16) | (unsigned)c;
            asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(mx), "l"(key) : "memory");
            asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(cnt), "l"(1ull) : "memory");
            unsigned long long a, b;
            if (PAIR) {
                do {
                    asm volatile("ld.acquire.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(cnt) : "memory");
                } while (a < (unsigned long long)G);
            } else {
                do {
                    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(a) : "l"(cnt) : "memory");
                } while (a < (unsigned long long)G);
                asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(b) : "l"(mx) : "memory");
            }
            win = b;
        }
        __syncthreads();
        if (fetch_n > 0) {
            const double *row = mat + static_cast<size_t>((win & 0xffff) * 7919 % 5000) * fetch_n;
            for (int q = tid; q < fetch_n; q += blockDim.x) {
                double v;
                asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(row + q));
                acc += v;
            }
            __syncthreads();
        }
    }
    if (c == 0 && tid == 0) out[0] = clock64() - t0;
    if (acc == 1234.5) *sink = acc;
}


// LL exchange: every CTA stores a SW-byte slot (SW/8 words, each = 32 data bits | 32-bit tag);
// warp 0 lane l polls slots l, l+32, ... all in flight at once, re-polling only the stale
// ones (optional __nanosleep backoff).  No fences, no atomics.
template <int SW, int SLEEP>
__global__ void k_ll(uint64_t *slots, const double *mat, int fetch_n, int iters, long long *out, double *sink) {
    constexpr int NW = SW / 8;
    const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ int winner;
    double acc = 0.0;
    long long t0 = clock64();
    for (int it = 1; it <= iters; ++it) {
        const uint32_t tag = static_cast<uint32_t>(it);
        uint64_t *par = slots + static_cast<size_t>(it & 1) * 160 * NW;
        const uint32_t key = (c * 2654435761u) ^ (it * 40503u);
        if (tid == 0) {
            uint64_t *s = par + static_cast<size_t>(c) * NW;
#pragma unroll
            for (int j = 0; j < NW; j += 2) st_v2(s + j, (static_cast<uint64_t>(key) << 32) | tag, (static_cast<uint64_t>(c) << 32) | tag);
        }
        if (warp == 0) {
            uint64_t best = 0;
            uint32_t pend = 0;
            uint64_t got[5];
#pragma unroll
            for (int j = 0; j < 5; ++j) { got[j] = 0; if (lane + 32 * j < G) pend |= 1u << j; }
            while (true) {
#pragma unroll
                for (int j = 0; j < 5; ++j) {
                    if (pend & (1u << j)) {
                        uint64_t w[NW];
#pragma unroll
                        for (int q = 0; q < NW; q += 2) ld_v2(par + static_cast<size_t>(lane + 32 * j) * NW + q, w[q], w[q + 1]);
                        bool ok = true;
#pragma unroll
                        for (int q = 0; q < NW; ++q) ok = ok && static_cast<uint32_t>(w[q]) == tag;
                        if (ok) { pend &= ~(1u << j); got[j] = ((w[0] >> 32) << 32) | (w[1] >> 32); }
                    }
                }
                if (__all_sync(0xffffffffu, pend == 0)) break;
                if (SLEEP) __nanosleep(SLEEP);
            }
#pragma unroll
            for (int j = 0; j < 5; ++j) if (got[j] > best) best = got[j];
            for (int o = 16; o; o >>= 1) {
                uint64_t v = __shfl_xor_sync(0xffffffffu, best, o);
                if (v > best) best = v;
            }
            if (lane == 0) winner = static_cast<int>(best & 0xffffffffu);
        }
        __syncthreads();
        if (fetch_n > 0) {
            const double *row = mat + static_cast<size_t>(winner * 7919 % 5000) * fetch_n;
            for (int q = tid; q < fetch_n; q += blockDim.x) {
                double v;
                asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(row + q));
                acc += v;
            }
            __syncthreads();
        }
    }
    if (c == 0 && tid == 0) out[0] = clock64() - t0;
    if (acc == 1234.5) *sink = acc;
}


// MODE 0: red.max + red.add both relaxed (ordering NOT guaranteed -- timing only)
// MODE 1: atom.max (returns: performed at L2) then red.relaxed.add
// (timing only: parity pairs with cumulative counts, no resets; the max is not used)
template <int MODE>
__global__ void k_atomic2(unsigned long long *w, const double *mat, int fetch_n, int iters, long long *out, double *sink) {
    const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
    __shared__ unsigned long long win;
    double acc = 0.0;
    long long t0 = clock64();
    for (int it = 1; it <= iters; ++it) {
        unsigned long long *cnt = w + 2 * (it & 1), *mx = cnt + 1;
        const unsigned long long target = static_cast<unsigned long long>((it + 1) >> 1) * G;
        if (tid == 0) {
            const unsigned long long key = ((unsigned long long)((c * 2654435761u) ^ (it * 40503u)) << 16) | (unsigned)c;
            if (MODE == 0) {
                asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(mx), "l"(key) : "memory");
                asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(cnt), "l"(1ull) : "memory");
            } else {
                unsigned long long old;
                asm volatile("atom.relaxed.gpu.global.max.u64 %0, [%1], %2;" : "=l"(old) : "l"(mx), "l"(key) : "memory");
                asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(cnt), "l"(1ull + (old >> 63)) : "memory");
            }
            unsigned long long a, b;
            const long long ts = clock64();
            do {
                asm volatile("ld.acquire.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(cnt) : "memory");
            } while (a < target && clock64() - ts < 2000000000ll);
            win = b;
        }
        __syncthreads();
        if (fetch_n > 0) {
            const double *row = mat + static_cast<size_t>((win & 0xffff) * 7919 % 5000) * fetch_n;
            for (int q = tid; q < fetch_n; q += blockDim.x) {
                double v;
                asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(row + q));
                acc += v;
            }
            __syncthreads();
        }
    }
    if (c == 0 && tid == 0) out[0] = clock64() - t0;
    if (acc == 1234.5) *sink = acc;
}

// root gather + LL broadcast: every CTA stores a 16-byte LL slot; CTA 0's warp 0 polls all
// G slots (single reader), reduces, stores one 16-byte LL winner word; all CTAs poll it.
__global__ void k_root(uint64_t *slots, const double *mat, int fetch_n, int iters, long long *out, double *sink) {
    const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ unsigned long long win;
    double acc = 0.0;
    long long t0 = clock64();
    for (int it = 1; it <= iters; ++it) {
        const uint32_t tag = static_cast<uint32_t>(it);
        uint64_t *par = slots + static_cast<size_t>(it & 1) * 160 * 2;
        uint64_t *bc = slots + 4 * 160 + (it & 1) * 16;
        const uint32_t key = (c * 2654435761u) ^ (it * 40503u);
        if (tid == 0) st_v2(par + 2 * c, (static_cast<uint64_t>(key) << 32) | tag, (static_cast<uint64_t>(c) << 32) | tag);
        if (c == 0 && warp == 0) {
            uint64_t best = 0;
            uint32_t pend = 0;
            uint64_t got[5];
#pragma unroll
            for (int j = 0; j < 5; ++j) { got[j] = 0; if (lane + 32 * j < G) pend |= 1u << j; }
            const long long ts0 = clock64();
            while (clock64() - ts0 < 2000000000ll) {
#pragma unroll
                for (int j = 0; j < 5; ++j) {
                    if (pend & (1u << j)) {
                        uint64_t a, b;
                        ld_v2(par + 2 * (lane + 32 * j), a, b);
                        if ((uint32_t)a == tag && (uint32_t)b == tag) { pend &= ~(1u << j); got[j] = ((a >> 32) << 32) | (b >> 32); }
                    }
                }
                if (__all_sync(0xffffffffu, pend == 0)) break;
            }
#pragma unroll
            for (int j = 0; j < 5; ++j) if (got[j] > best) best = got[j];
            for (int o = 16; o; o >>= 1) {
                uint64_t v = __shfl_xor_sync(0xffffffffu, best, o);
                if (v > best) best = v;
            }
            if (lane == 0) st_v2(bc, (best & 0xffffffff00000000ull) | tag, (best << 32) | tag);
        }
        if (tid == 0) {
            uint64_t a, b;
            const long long ts1 = clock64();
            do { ld_v2(bc, a, b); } while (((uint32_t)a != tag || (uint32_t)b != tag) && clock64() - ts1 < 2000000000ll);
            win = (b >> 32);
        }
        __syncthreads();
        if (fetch_n > 0) {
            const double *row = mat + static_cast<size_t>((win & 0xffff) * 7919 % 5000) * fetch_n;
            for (int q = tid; q < fetch_n; q += blockDim.x) {
                double v;
                asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(row + q));
                acc += v;
            }
            __syncthreads();
        }
    }
    if (c == 0 && tid == 0) out[0] = clock64() - t0;
    if (acc == 1234.5) *sink = acc;
}

// counter barrier reference (one atomic per CTA + spin) at the same G
__global__ void k_counter(unsigned int *ctr, int iters, long long *out) {
    const int G = gridDim.x;
    long long t0 = clock64();
    for (int i = 1; i <= iters; ++i) {
        if (threadIdx.x == 0) {
            atomicAdd(ctr, 1u);
            unsigned v;
            do {
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
            } while (v < static_cast<unsigned>(i * G));
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

int main() {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    const int sms = prop.multiProcessorCount;
    long long *out;
    CK(cudaMallocManaged(&out, 64));
    uint64_t *slots;
    CK(cudaMalloc(&slots, 2 * 160 * 64));
    double *mat, *sink;
    CK(cudaMalloc(&mat, 5000ull * 2000 * 8));
    CK(cudaMemset(mat, 0, 5000ull * 2000 * 8));
    CK(cudaMalloc(&sink, 8));
    const int iters = 4000;
    for (int G : {16, 64, 128, sms}) {
        const int thr = 512;
        double r[12];
        int i = 0;
        for (int fn : {0, 500}) {
#define RUN(K)                                                        \
    CK(cudaMemset(slots, 0, 2 * 160 * 64));                           \
    K<<<G, thr>>>(slots, mat, fn, iters, out, sink);                  \
    CK(cudaDeviceSynchronize());                                      \
    r[i++] = (double)out[0] / iters;
            RUN(k_root)
            CK(cudaMemset(slots, 0, 2 * 160 * 64));
            k_atomic<true><<<G, thr>>>((unsigned long long *)slots, mat, fn, iters, out, sink);
            CK(cudaDeviceSynchronize());
            r[i++] = (double)out[0] / iters;
            CK(cudaMemset(slots, 0, 2 * 160 * 64));
            k_atomic2<0><<<G, thr>>>((unsigned long long *)slots, mat, fn, iters, out, sink);
            CK(cudaDeviceSynchronize());
            r[i++] = (double)out[0] / iters;
            CK(cudaMemset(slots, 0, 2 * 160 * 64));
            k_atomic2<1><<<G, thr>>>((unsigned long long *)slots, mat, fn, iters, out, sink);
            CK(cudaDeviceSynchronize());
            r[i++] = (double)out[0] / iters;
            CK(cudaMemset(slots, 0, 64));
            k_counter<<<G, thr>>>((unsigned *)slots, iters, out);
            CK(cudaDeviceSynchronize());
            r[i++] = (double)out[0] / iters;
        }
        printf("G=%d root %.0f atomic_release %.0f atomic_relaxed %.0f atom_then_red %.0f counter %.0f | +row500: %.0f %.0f %.0f %.0f %.0f\n", G,
               r[0], r[1], r[2], r[3], r[4], r[5], r[6], r[7], r[8], r[9]);
    }
    return 0;
}
