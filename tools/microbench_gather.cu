// microbench_gather.cu -- the floor of C5's CSR sketch access pattern: every row of a 4M x 2000
// CSR matrix (10 stored pairs per row, int64 row_ptr, int32 col, fp64 val, fp64 b) read once in
// a random row order (the bucket-sorted perm), nothing folded.  One thread per row at full
// occupancy gives the most memory-level parallelism this pattern can have; the "+write" variant
// adds the 640 MB coalesced output stream of the sketch (160 B per row).  A sequential perm shows
// what the same bytes cost in address order.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_gather tools/microbench_gather.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <numeric>
#include <random>
#include <vector>

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e = (x);                                                                   \
        if (e != cudaSuccess) {                                                                \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);     \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

template <bool WRITE>
__global__ void __launch_bounds__(256) k_gather(const int32_t *__restrict__ perm, const int64_t *__restrict__ row_ptr,
                                                const int32_t *__restrict__ col, const double *__restrict__ val,
                                                const double *__restrict__ b, int64_t m, double *__restrict__ out,
                                                double *__restrict__ out2) {
    const int64_t T = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < m; t += T) {
        const int64_t r = perm[t];
        const int64_t rs = __ldg(row_ptr + r), re = __ldg(row_ptr + r + 1);
        double acc = __ldg(b + r);
        for (int64_t q = rs; q < re; ++q) acc += __ldg(val + q) + static_cast<double>(__ldg(col + q));
        out[t] = acc;
        if (WRITE) {
#pragma unroll
            for (int j = 0; j < 20; ++j) out2[j * m + t] = acc;
        }
    }
}

int main() {
    const int64_t m = 4000000, nnz_row = 10, n = 2000, nnz = m * nnz_row;
    std::vector<int64_t> rp(m + 1);
    for (int64_t i = 0; i <= m; ++i) rp[i] = i * nnz_row;
    std::vector<int32_t> col(nnz);
    std::mt19937_64 g(7);
    for (int64_t i = 0; i < nnz; ++i) col[i] = static_cast<int32_t>(g() % n);
    std::vector<int32_t> rnd(m), seq(m);
    std::iota(seq.begin(), seq.end(), 0);
    rnd = seq;
    std::shuffle(rnd.begin(), rnd.end(), g);
    int64_t *d_rp;
    int32_t *d_col, *d_rnd, *d_seq;
    double *d_val, *d_b, *d_out, *d_out2;
    char *flush;
    CK(cudaMalloc(&d_rp, (m + 1) * 8));
    CK(cudaMalloc(&d_col, nnz * 4));
    CK(cudaMalloc(&d_val, nnz * 8));
    CK(cudaMalloc(&d_b, m * 8));
    CK(cudaMalloc(&d_rnd, m * 4));
    CK(cudaMalloc(&d_seq, m * 4));
    CK(cudaMalloc(&d_out, m * 8));
    CK(cudaMalloc(&d_out2, 20 * m * 8));
    CK(cudaMalloc(&flush, 256 << 20));
    CK(cudaMemcpy(d_rp, rp.data(), (m + 1) * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_col, col.data(), nnz * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(d_val, 0, nnz * 8));
    CK(cudaMemset(d_b, 0, m * 8));
    CK(cudaMemcpy(d_rnd, rnd.data(), m * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_seq, seq.data(), m * 4, cudaMemcpyHostToDevice));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const double rd = 12.0 * nnz + 8.0 * (m + 1) + 8.0 * m + 4.0 * m;  // CSR + b + perm
    const double wr = 160.0 * m;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int v = 0; v < 4; ++v) {
        const bool write = v & 1;
        const int32_t *perm = (v & 2) ? d_seq : d_rnd;
        float best = 1e30f;
        for (int rep = 0; rep < 6; ++rep) {
            CK(cudaMemset(flush, rep, 256 << 20));  // flush L2
            CK(cudaEventRecord(e0));
            if (write)
                k_gather<true><<<sms * 8, 256>>>(perm, d_rp, d_col, d_val, d_b, m, d_out, d_out2);
            else
                k_gather<false><<<sms * 8, 256>>>(perm, d_rp, d_col, d_val, d_b, m, d_out, d_out2);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (rep > 0) best = std::min(best, ms);
        }
        const double by = rd + 8.0 * m + (write ? wr : 0.0);
        printf("%-10s perm %-10s %.3f ms  %.0f GB/s algorithmic (%.0f MB)\n", write ? "+write" : "read only",
               (v & 2) ? "sequential" : "random", best, by / (best * 1e-3) / 1e9, by / 1e6);
    }
    return 0;
}
