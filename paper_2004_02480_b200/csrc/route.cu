// route.cu -- S9 for CSR input by ROW ROUTING (the C5 variant of the sharded
// sketch).  Rank p holds the contiguous input rows [row_offset, row_offset + m_local) of a CSR
// matrix.  Every row i is hashed with its GLOBAL index (Definition 1: bucket h(i), sign
// D_ii) and sent whole -- (global row, b_i, its stored (col, val) pairs) -- to the rank owning
// bucket h(i) (csk_shard_range: owner = h / ceil(d/P)).  Rows leave each rank in ascending order
// and arrive ordered by source rank, so every owner receives its rows in ascending GLOBAL order
// and folds each bucket exactly as the single-GPU sketch does (Algorithm 1 "Initialize", P:60;
// S:140 source-row order): A~ and b~ are bit-identical to P = 1, and the wire carries the CSR
// bytes (~12 nnz) instead of partial A~ rows (8 d n / P per rank, 9x more at C5).
//
//   k_route_count    per 256-row block and destination: rows and stored pairs
//   k_route_scan     (one CTA) block offsets within each destination's segment, and totals
//   k_route_scatter  rows to their destination segment, stable (ascending row): header (global
//                    row, b, pair offset within the segment) and the pairs
//   k_route_rowptr   (receiver) row_ptr of the received rows from the per-source pair bases
//   k_route_hash     (receiver) local bucket (h - d_lo) and sign of every received row
// The receiver then runs the ordinary plan (explicit map) and CSR sketch on its bucket range.
#include "csk_internal.cuh"

namespace csk {

namespace {

constexpr int kRT = 256;  // rows per block (one per thread)

__device__ __forceinline__ uint32_t route_bucket(uint64_t seed, uint64_t c, uint32_t d, uint32_t &neg) {
    neg = static_cast<uint32_t>(sm64(seed, 2 * c + 1) >> 63);
    return static_cast<uint32_t>(__umul64hi(sm64(seed, 2 * c), static_cast<uint64_t>(d)));
}

// Block-wide exclusive scan of (a, b) in thread order; returns the block totals in (ta, tb).
__device__ __forceinline__ void block_scan2(int64_t a, int64_t b, int64_t &ea, int64_t &eb, int64_t &ta, int64_t &tb,
                                            int64_t *sh) {  // sh: 2 * (kRT / 32) + 2 int64
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t ia = a, ib = b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t ya = __shfl_up_sync(0xffffffffu, ia, o), yb = __shfl_up_sync(0xffffffffu, ib, o);
        if (lane >= o) { ia += ya; ib += yb; }
    }
    if (lane == 31) { sh[2 * warp] = ia; sh[2 * warp + 1] = ib; }
    __syncthreads();
    int64_t wa = 0, wb = 0;
    ta = 0; tb = 0;
    for (int w = 0; w < kRT / 32; ++w) {
        if (w == warp) { wa = ta; wb = tb; }
        ta += sh[2 * w]; tb += sh[2 * w + 1];
    }
    ea = wa + ia - a;
    eb = wb + ib - b;
    __syncthreads();  // sh reused by the next scan
}

}  // namespace

__global__ void k_route_count(const int64_t *__restrict__ row_ptr, int64_t m, int64_t row_offset, uint64_t seed,
                              uint32_t d, int64_t chunk, int P, int64_t *__restrict__ blk) {
    __shared__ unsigned long long cnt[2 * kMaxRanks];
    if (threadIdx.x < 2 * kMaxRanks) cnt[threadIdx.x] = 0ull;
    __syncthreads();
    const int64_t i = static_cast<int64_t>(blockIdx.x) * kRT + threadIdx.x;
    if (i < m) {
        uint32_t neg;
        const uint32_t h = route_bucket(seed, static_cast<uint64_t>(row_offset + i), d, neg);
        const int o = static_cast<int>(h / static_cast<uint64_t>(chunk));
        atomicAdd(&cnt[2 * o], 1ull);
        atomicAdd(&cnt[2 * o + 1], static_cast<unsigned long long>(row_ptr[i + 1] - row_ptr[i]));
    }
    __syncthreads();
    if (threadIdx.x < 2 * P) blk[static_cast<int64_t>(blockIdx.x) * 2 * P + threadIdx.x] = static_cast<int64_t>(cnt[threadIdx.x]);
}

// one CTA: blk[b][o][2] -> exclusive offsets over blocks (per destination); tot[o][2] totals
__global__ void k_route_scan(int64_t *blk, int64_t nblocks, int P, int64_t *tot) {
    const int t = threadIdx.x;  // one thread per (destination, quantity)
    if (t < 2 * P) {
        int64_t run = 0;
        for (int64_t b = 0; b < nblocks; ++b) {
            const int64_t v = blk[b * 2 * P + t];
            blk[b * 2 * P + t] = run;
            run += v;
        }
        tot[t] = run;
    }
}

// seg[o][2]: start of destination o's segment in the row / pair send buffers
__global__ void k_route_scatter(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                const double *__restrict__ val, const double *__restrict__ b, int64_t m,
                                int64_t row_offset, uint64_t seed, uint32_t d, int64_t chunk, int P,
                                const int64_t *__restrict__ blk, const int64_t *__restrict__ seg,
                                int32_t *__restrict__ srow, double *__restrict__ sb, int64_t *__restrict__ soff,
                                int32_t *__restrict__ scol, double *__restrict__ sval) {
    __shared__ int64_t sh[2 * (kRT / 32) + 2];
    const int64_t i = static_cast<int64_t>(blockIdx.x) * kRT + threadIdx.x;
    int o = -1;
    int64_t nnz = 0;
    if (i < m) {
        uint32_t neg;
        const uint32_t h = route_bucket(seed, static_cast<uint64_t>(row_offset + i), d, neg);
        o = static_cast<int>(h / static_cast<uint64_t>(chunk));
        nnz = row_ptr[i + 1] - row_ptr[i];
    }
    for (int q = 0; q < P; ++q) {  // stable: rows of destination q keep their order
        int64_t er, ep, tr, tp;
        block_scan2(o == q ? 1 : 0, o == q ? nnz : 0, er, ep, tr, tp, sh);
        if (o == q) {
            const int64_t* bo = blk + static_cast<int64_t>(blockIdx.x) * 2 * P + 2 * q;
            const int64_t pr = seg[2 * q] + bo[0] + er;   // row slot in the send buffer
            CSK_DCHECK(pr >= seg[2 * q] && (q + 1 == P || pr < seg[2 * q + 2]));
            const int64_t pin = bo[1] + ep;               // pair offset within q's segment
            srow[pr] = static_cast<int32_t>(row_offset + i);
            sb[pr] = b[i];
            soff[pr] = pin;
            const int64_t src = row_ptr[i], dst = seg[2 * q + 1] + pin;
            for (int64_t k = 0; k < nnz; ++k) {
                scol[dst + k] = col[src + k];
                sval[dst + k] = val[src + k];
            }
        }
    }
}

// receiver: rows of source s occupy [rbase[s], rbase[s+1]); their pair offsets are relative to
// the source's segment, which starts at pbase[s] of the received pairs
__global__ void k_route_rowptr(const int64_t *__restrict__ roff, int64_t M, int P, const int64_t *__restrict__ rbase,
                               const int64_t *__restrict__ pbase, int64_t *__restrict__ row_ptr) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i <= M;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (i == M) {
            row_ptr[M] = pbase[P];
        } else {
            int s = 0;
            while (s + 1 < P && rbase[s + 1] <= i) ++s;
            row_ptr[i] = pbase[s] + roff[i];
        }
    }
}

__global__ void k_route_hash(const int32_t *__restrict__ grow, int64_t M, uint64_t seed, uint32_t d, int64_t d_lo,
                             int32_t *__restrict__ h, int8_t *__restrict__ sign) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < M;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint32_t neg;
        const uint32_t hh = route_bucket(seed, static_cast<uint64_t>(grow[i]), d, neg);
        h[i] = static_cast<int32_t>(static_cast<int64_t>(hh) - d_lo);
        sign[i] = neg ? int8_t(-1) : int8_t(1);
    }
}

// ---- host side ---------------------------------------------------------------------------------

csk_status_t route_pack(csk_ctx_t ctx, const int64_t *row_ptr, const int32_t *col, const double *val, const double *b,
                        int64_t m_local, int64_t row_offset, int64_t d, uint64_t seed, int P, RoutePack &pk,
                        cudaStream_t s) {
    const int64_t chunk = (d + P - 1) / P;
    const int64_t nb = (m_local + kRT - 1) / kRT;
    pk.P = P;
    pk.owned.clear();
    auto alloc = [&](void **p, size_t bytes) -> csk_status_t {
        CSK_CUDA(ctx, cudaMallocAsync(p, bytes > 0 ? bytes : 16, s));
        pk.owned.push_back(*p);
        return CSK_OK;
    };
    int64_t *blk = nullptr, *tot = nullptr;
    CSK_CHECK(alloc(reinterpret_cast<void **>(&blk), static_cast<size_t>(nb > 0 ? nb : 1) * 2 * P * 8));
    CSK_CHECK(alloc(reinterpret_cast<void **>(&tot), static_cast<size_t>(4 * kMaxRanks + 2) * 8));
    if (m_local > 0) {
        k_route_count<<<static_cast<unsigned>(nb), kRT, 0, s>>>(row_ptr, m_local, row_offset, seed,
                                                                static_cast<uint32_t>(d), chunk, P, blk);
        k_route_scan<<<1, 32, 0, s>>>(blk, nb, P, tot);
    } else {
        CSK_CUDA(ctx, cudaMemsetAsync(tot, 0, static_cast<size_t>(2 * P) * 8, s));
    }
    CSK_CUDA(ctx, cudaGetLastError());
    CSK_CUDA(ctx, cudaMemcpyAsync(pk.cnt, tot, static_cast<size_t>(2 * P) * 8, cudaMemcpyDeviceToHost, s));
    CSK_CUDA(ctx, cudaStreamSynchronize(s));
    int64_t seg[2 * kMaxRanks];
    int64_t rows = 0, pairs = 0;
    for (int q = 0; q < P; ++q) {
        seg[2 * q] = rows;
        seg[2 * q + 1] = pairs;
        rows += pk.cnt[2 * q];
        pairs += pk.cnt[2 * q + 1];
    }
    for (int q = 0; q < 2 * P; ++q) pk.seg[q] = seg[q];
    CSK_CHECK(alloc(reinterpret_cast<void **>(&pk.row), static_cast<size_t>(rows) * 4));
    CSK_CHECK(alloc(reinterpret_cast<void **>(&pk.b), static_cast<size_t>(rows) * 8));
    CSK_CHECK(alloc(reinterpret_cast<void **>(&pk.off), static_cast<size_t>(rows) * 8));
    CSK_CHECK(alloc(reinterpret_cast<void **>(&pk.col), static_cast<size_t>(pairs) * 4));
    CSK_CHECK(alloc(reinterpret_cast<void **>(&pk.val), static_cast<size_t>(pairs) * 8));
    if (m_local > 0) {
        int64_t *segd = tot + 2 * kMaxRanks;
        CSK_CUDA(ctx, cudaMemcpyAsync(segd, seg, static_cast<size_t>(2 * P) * 8, cudaMemcpyHostToDevice, s));
        k_route_scatter<<<static_cast<unsigned>(nb), kRT, 0, s>>>(row_ptr, col, val, b, m_local, row_offset, seed,
                                                                  static_cast<uint32_t>(d), chunk, P, blk, segd,
                                                                  pk.row, pk.b, pk.off, pk.col, pk.val);
        CSK_CUDA(ctx, cudaGetLastError());
    }
    return CSK_OK;
}

csk_status_t route_unpack_sketch(csk_ctx_t ctx, const RouteRecv &rv, int64_t n, int64_t d, int64_t d_lo, int64_t d_hi,
                                 uint64_t seed, double *At_local, double *bt_local, double *nsq_local,
                                 cudaStream_t s) {
    const int64_t dl = d_hi - d_lo;
    const int64_t M = rv.rbase[rv.P];
    if (dl <= 0) return CSK_OK;
    if (M == 0) {  // no rows hashed into this rank's buckets: A~ rows are zero
        CSK_CUDA(ctx, cudaMemsetAsync(At_local, 0, static_cast<size_t>(dl) * n * 8, s));
        CSK_CUDA(ctx, cudaMemsetAsync(bt_local, 0, static_cast<size_t>(dl) * 8, s));
        if (nsq_local) CSK_CUDA(ctx, cudaMemsetAsync(nsq_local, 0, static_cast<size_t>(dl) * 8, s));
        return CSK_OK;
    }
    std::vector<void *> owned;
    auto cleanup = [&]() {
        for (void *p : owned) cudaFreeAsync(p, s);
    };
    auto alloc = [&](void **p, size_t bytes) -> csk_status_t {
        CSK_CUDA(ctx, cudaMallocAsync(p, bytes > 0 ? bytes : 16, s));
        owned.push_back(*p);
        return CSK_OK;
    };
    int64_t *row_ptr = nullptr, *bases = nullptr;
    int32_t *h = nullptr;
    int8_t *sign = nullptr;
    csk_status_t st = alloc(reinterpret_cast<void **>(&row_ptr), static_cast<size_t>(M + 1) * 8);
    if (st == CSK_OK) st = alloc(reinterpret_cast<void **>(&bases), static_cast<size_t>(2 * (kMaxRanks + 1)) * 8);
    if (st == CSK_OK) st = alloc(reinterpret_cast<void **>(&h), static_cast<size_t>(M) * 4);
    if (st == CSK_OK) st = alloc(reinterpret_cast<void **>(&sign), static_cast<size_t>(M));
    if (st != CSK_OK) { cleanup(); return st; }
    int64_t hb[2 * (kMaxRanks + 1)];
    for (int q = 0; q <= rv.P; ++q) {
        hb[q] = rv.rbase[q];
        hb[kMaxRanks + 1 + q] = rv.pbase[q];
    }
    CSK_CUDA(ctx, cudaMemcpyAsync(bases, hb, sizeof(hb), cudaMemcpyHostToDevice, s));
    const int grid = static_cast<int>(std::min<int64_t>((M + 256) / 256, int64_t(ctx->num_sms) * 8));
    k_route_rowptr<<<grid, 256, 0, s>>>(rv.off, M, rv.P, bases, bases + kMaxRanks + 1, row_ptr);
    k_route_hash<<<grid, 256, 0, s>>>(rv.row, M, seed, static_cast<uint32_t>(d), d_lo, h, sign);
    CSK_CUDA(ctx, cudaGetLastError());
    int32_t *perm = nullptr, *offsets = nullptr;
    st = build_plan(ctx, 0, 0, M, dl, h, sign, &perm, &offsets, s);
    if (st == CSK_OK)
        st = launch_sketch_csr(ctx, row_ptr, rv.col, rv.val, rv.b, M, n, dl, perm, offsets, At_local, bt_local,
                               nsq_local, s);
    cleanup();
    return st;
}

void route_free(RoutePack &pk, cudaStream_t s) {
    for (void *p : pk.owned) cudaFreeAsync(p, s);
    pk.owned.clear();
}

}  // namespace csk

using namespace csk;

// P virtual ranks on one GPU (test hook): the whole routing decomposition with device copies as
// the transport; A_tilde (d x n), b_tilde, nsq receive every owner's bucket rows.
extern "C" csk_status_t csk_sketch_csr_routed_virtual(csk_ctx_t ctx, const int64_t *row_ptr, const int32_t *col,
                                                      const double *val, const double *b, int64_t m, int64_t n,
                                                      int64_t d, uint64_t seed, int32_t nranks, double *A_tilde,
                                                      double *b_tilde, double *nsq, void *stream) {
    CSK_NVTX("csk_sketch_csr_routed_virtual");
    if (!ctx) return CSK_E_ARG;
    if (!row_ptr || !col || !val || !b || !A_tilde || !b_tilde || m < 1 || m >= (int64_t(1) << 31) || n < 1 || d < 1 ||
        d >= m || nranks < 1 || nranks > kMaxRanks || d < nranks)
        return fail(ctx, CSK_E_ARG, "csk_sketch_csr_routed_virtual: bad arguments (1 <= nranks <= min(8, d), d < m)");
    CSK_CUDA(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = as_stream(stream);
    const int P = nranks;
    std::vector<RoutePack> packs(P);
    int64_t rp_h[kMaxRanks + 1];
    for (int q = 0; q <= P; ++q) rp_h[q] = m * q / P;  // contiguous input row shards (any split works)
    for (int q = 0; q < P; ++q) {
        // shard q's rows [rp_h[q], rp_h[q+1]) index the global col/val through row_ptr + rp_h[q]
        csk_status_t st = route_pack(ctx, row_ptr + rp_h[q], col, val, b + rp_h[q], rp_h[q + 1] - rp_h[q], rp_h[q], d,
                                     seed, P, packs[q], s);
        if (st != CSK_OK) {
            for (auto &pk : packs) route_free(pk, s);
            return st;
        }
    }
    csk_status_t st = CSK_OK;
    for (int o = 0; o < P && st == CSK_OK; ++o) {
        int64_t lo, hi;
        csk_shard_range(d, P, o, &lo, &hi);
        RouteRecv rv;
        rv.P = P;
        rv.rbase[0] = rv.pbase[0] = 0;
        for (int q = 0; q < P; ++q) {
            rv.rbase[q + 1] = rv.rbase[q] + packs[q].cnt[2 * o];
            rv.pbase[q + 1] = rv.pbase[q] + packs[q].cnt[2 * o + 1];
        }
        const int64_t M = rv.rbase[P], NNZ = rv.pbase[P];
        void *buf[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
        const size_t sz[5] = {static_cast<size_t>(M) * 4, static_cast<size_t>(M) * 8, static_cast<size_t>(M) * 8,
                              static_cast<size_t>(NNZ) * 4, static_cast<size_t>(NNZ) * 8};
        for (int a = 0; a < 5 && st == CSK_OK; ++a)
            if (cudaMallocAsync(&buf[a], sz[a] > 0 ? sz[a] : 16, s) != cudaSuccess) st = fail(ctx, CSK_E_NOMEM, "routed: cudaMallocAsync");
        // the "transport": source q's segment for owner o, in source order
        for (int q = 0; q < P && st == CSK_OK; ++q) {
            const RoutePack &pk = packs[q];
            const int64_t r0 = pk.seg[2 * o], nr = pk.cnt[2 * o], p0 = pk.seg[2 * o + 1], np = pk.cnt[2 * o + 1];
            cudaMemcpyAsync(static_cast<int32_t *>(buf[0]) + rv.rbase[q], pk.row + r0, nr * 4, cudaMemcpyDeviceToDevice, s);
            cudaMemcpyAsync(static_cast<double *>(buf[1]) + rv.rbase[q], pk.b + r0, nr * 8, cudaMemcpyDeviceToDevice, s);
            cudaMemcpyAsync(static_cast<int64_t *>(buf[2]) + rv.rbase[q], pk.off + r0, nr * 8, cudaMemcpyDeviceToDevice, s);
            cudaMemcpyAsync(static_cast<int32_t *>(buf[3]) + rv.pbase[q], pk.col + p0, np * 4, cudaMemcpyDeviceToDevice, s);
            cudaMemcpyAsync(static_cast<double *>(buf[4]) + rv.pbase[q], pk.val + p0, np * 8, cudaMemcpyDeviceToDevice, s);
        }
        rv.row = static_cast<int32_t *>(buf[0]);
        rv.b = static_cast<double *>(buf[1]);
        rv.off = static_cast<int64_t *>(buf[2]);
        rv.col = static_cast<int32_t *>(buf[3]);
        rv.val = static_cast<double *>(buf[4]);
        if (st == CSK_OK)
            st = route_unpack_sketch(ctx, rv, n, d, lo, hi, seed, A_tilde + lo * n, b_tilde + lo, nsq ? nsq + lo : nullptr, s);
        for (void *p : buf)
            if (p) cudaFreeAsync(p, s);
    }
    for (auto &pk : packs) route_free(pk, s);
    cudaError_t e = cudaStreamSynchronize(s);
    if (st == CSK_OK && e != cudaSuccess) st = cuda_fail(ctx, e, "csk_sketch_csr_routed_virtual");
    return st;
}
