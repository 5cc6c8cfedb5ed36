// comm.cu -- S9/S10: the row-sharded multi-GPU path (north_star: "rows of A are sharded for
// the sketch (NCCL reduce-scatter of partial A~ by bucket range) and rows of A~ are sharded
// for the loop (a per-iteration max-loc exchange plus the winning n-vector)").
//
// Sketch (S9): rank p hashes its rows of A with GLOBAL row indices (row_offset), folds them
// into a full partial (A~ | b~) of d x (n+1) with the single-GPU kernels, and one grouped
// ncclReduceScatter(sum) leaves rank p with bucket rows [p*c, min((p+1)*c, d)), c = ceil(d/P)
// (equal blocks: reduce-scatter needs equal counts; the tail block is zero-padded).
//
// Loop (S10), per iteration k, identical on every rank:
//   k_shard_candidate  local GEMV r = b~ - A~ x_k over the rank's rows, scores, argmax (ties
//                      -> lowest GLOBAL row), writes (score, idx, lambda, sum r^2, row[n]);
//   ncclAllGather      of that (n + 4)-double record -- the allreduce max-loc and the
//                      broadcast of the winning row fused into one exchange (the winner's
//                      owner is unknown before the exchange, so a rooted broadcast would
//                      need another round);
//   k_shard_apply      every rank picks the same winner from the P records in rank order,
//                      x += lambda row, RES / residual test -> device-side stop flag.
// Kernels become no-ops once the flag is set; the host polls it every kBatch iterations.
// The loopback exchange (csk_solve_virtual_ranks) runs the same kernels for P virtual ranks
// on one GPU, with the gather done by the candidate kernels writing straight into the
// gathered buffer -- the 1-GPU test of the sharded decomposition.
#include <nccl.h>
#include <stdlib.h>
#include <string.h>

#include <cuda.h>

#include <map>
#include <string>
#include <vector>

#include "csk_internal.cuh"

namespace csk {

struct Comm {
    ncclComm_t nccl = nullptr;
    int nranks = 1, rank = 0;
    // peer mappings (cudaIpcOpenMemHandle) of the other ranks' allocations, by handle bytes
    std::map<std::string, void *> peer_open;
    // the fused S10 setup of the last solve (peer pointers, probed): reused when every rank calls
    // again with the same A~ shard and exchange buffer
    struct FusedSetup {
        bool valid = false;
        const void *a = nullptr;
        void *slots = nullptr;
        int gr = 0;
        int64_t d_lo = 0, d_hi = 0;
        RankSetup rs;
    } fused;
};

namespace {

constexpr int kBatch = 16;   // iterations per host poll of the stop flag
constexpr int kRecHead = 4;  // record head: score, idx (as double), lambda, sum r^2

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ bool better(double sa, int64_t ia, double sb, int64_t ib) {
    return sa > sb || (sa == sb && ia < ib);
}

// Device state of a sharded solve (one per rank): [0] iterations, [1] termination (-1 running),
// [2] final res bits, [3] last index.
struct ShardState {
    int64_t it, term, res_bits, last;
};

// One CTA per 32 rows (warp per row pair of lanes over columns), block candidates reduced by
// the last CTA to finish (ticket), fixed order -> deterministic.
__global__ void __launch_bounds__(256) k_shard_candidate(
    const double *__restrict__ At, const double *__restrict__ bt, const double *__restrict__ nsq,
    int64_t rows, int64_t row0_global, int64_t n, const double *__restrict__ x,
    double *__restrict__ blk, unsigned int *ticket, double *__restrict__ rec,
    const ShardState *st) {
    if (st->term >= 0) return;
    __shared__ double s_s[8], s_l[8], s_rr[8];
    __shared__ int64_t s_i[8];
    __shared__ bool s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double bs = -2.0, bl = 0.0, rr = 0.0;
    int64_t bi = INT64_MAX;
    for (int64_t l = static_cast<int64_t>(blockIdx.x) * 8 + warp; l < rows; l += static_cast<int64_t>(gridDim.x) * 8) {
        const double *row = At + l * n;
        double acc = 0.0;
        for (int64_t k = lane; k < n; k += 32) acc = __fma_rn(row[k], x[k], acc);
        acc = warp_sum(acc);
        const double ri = bt[l] - acc;
        const double ns = nsq[l];
        const double sc = ns > 0.0 ? (ri * ri) / ns : -1.0;
        rr = __fma_rn(ri, ri, rr);
        if (better(sc, row0_global + l, bs, bi)) { bs = sc; bi = row0_global + l; bl = ns > 0.0 ? ri / ns : 0.0; }
    }
    if (lane == 0) { s_s[warp] = bs; s_i[warp] = bi; s_l[warp] = bl; s_rr[warp] = rr; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double cs = s_s[0], cl = s_l[0], crr = s_rr[0];
        int64_t ci = s_i[0];
        for (int w = 1; w < 8; ++w) {
            if (better(s_s[w], s_i[w], cs, ci)) { cs = s_s[w]; ci = s_i[w]; cl = s_l[w]; }
            crr = crr + s_rr[w];
        }
        double *b = blk + static_cast<size_t>(blockIdx.x) * 4;
        b[0] = cs; b[1] = static_cast<double>(ci); b[2] = cl; b[3] = crr;
        __threadfence();
        s_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // last block: combine all block candidates in block order, copy the winner's row
    __shared__ double w_s, w_l, w_rr;
    __shared__ int64_t w_i;
    if (threadIdx.x == 0) {
        double cs = -2.0, cl = 0.0, crr = 0.0;
        int64_t ci = INT64_MAX;
        for (unsigned b = 0; b < gridDim.x; ++b) {
            const volatile double *p = blk + static_cast<size_t>(b) * 4;
            const double s = p[0], l = p[2], r = p[3];
            const int64_t i = p[0] < -1.5 ? INT64_MAX : static_cast<int64_t>(p[1]);
            if (better(s, i, cs, ci)) { cs = s; ci = i; cl = l; }
            crr = crr + r;
        }
        w_s = cs; w_i = ci; w_l = cl; w_rr = crr;
        rec[0] = cs;
        rec[1] = static_cast<double>(ci == INT64_MAX ? -1 : ci);
        rec[2] = cl;
        rec[3] = crr;
        *ticket = 0;
    }
    __syncthreads();
    const int64_t li = (w_i == INT64_MAX) ? -1 : w_i - row0_global;
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) rec[kRecHead + k] = li >= 0 ? At[li * n + k] : 0.0;
}

// One CTA: winner over P records (rank order), x update, stop test.  bb: ||b~||^2 (residual
// mode) or ||x*||^2 (RES mode) precomputed.
__global__ void __launch_bounds__(256) k_shard_apply(
    const double *__restrict__ gathered, int P, int64_t n, double *__restrict__ x,
    const double *__restrict__ x_star, double denom, double tol, int64_t max_iters,
    ShardState *st, int64_t *idx_trace, int64_t trace_cap) {
    if (st->term >= 0) return;
    __shared__ double s_l, s_red[8];
    __shared__ int64_t s_i, s_p;
    __shared__ int s_stop;
    const int64_t rl = kRecHead + n;
    const int64_t k = st->it;
    if (threadIdx.x == 0) {
        double cs = -2.0, cl = 0.0, rr = 0.0;
        int64_t ci = INT64_MAX, cp = -1;
        for (int p = 0; p < P; ++p) {
            const double *r = gathered + p * rl;
            const int64_t i = r[1] < 0 ? INT64_MAX : static_cast<int64_t>(r[1]);
            if (better(r[0], i, cs, ci)) { cs = r[0]; ci = i; cl = r[2]; cp = p; }
            rr = rr + r[3];
        }
        int stop = -1;
        if (!x_star) {  // residual mode: test r_k before the update
            const double res = denom > 0.0 ? rr / denom : rr;
            if (res <= tol) stop = CSK_CONVERGED;
            else if (k == max_iters) stop = CSK_MAX_ITERS;
            if (stop >= 0) st->res_bits = __double_as_longlong(res);
        }
        if (stop < 0 && cs < 0.0) stop = -2;
        if (stop < 0 && cs == 0.0) stop = CSK_STAGNATED;
        s_stop = stop;
        s_l = cl; s_i = ci; s_p = cp;
    }
    __syncthreads();
    if (s_stop != -1) {
        if (threadIdx.x == 0) st->term = s_stop;
        return;
    }
    const double *row = gathered + s_p * rl + kRecHead;
    double e2 = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
        const double xn = __fma_rn(s_l, row[j], x[j]);
        x[j] = xn;
        if (x_star) {
            const double e = xn - x_star[j];
            e2 = __fma_rn(e, e, e2);
        }
    }
    if (x_star) {
        e2 = warp_sum(e2);
        if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = e2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (idx_trace && k < trace_cap) idx_trace[k] = s_i;
        st->it = k + 1;
        st->last = s_i;
        if (x_star) {
            double t = s_red[0];
            for (int w = 1; w < 8; ++w) t = t + s_red[w];
            const double res = denom > 0.0 ? t / denom : t;
            st->res_bits = __double_as_longlong(res);
            if (res <= tol) st->term = CSK_CONVERGED;
            else if (k + 1 == max_iters) st->term = CSK_MAX_ITERS;
        }
    }
}

// RES_0 (RES mode) and the stop test before the first update; denominators.
__global__ void k_shard_init(const double *x, const double *x_star, const double *bt, int64_t rows,
                             int64_t n, double tol, int64_t max_iters, ShardState *st,
                             double *denoms) {
    __shared__ double red[3][8];
    double a = 0.0, b = 0.0, c = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
        if (x_star) {
            a = __fma_rn(x_star[j], x_star[j], a);
            const double e = x[j] - x_star[j];
            b = __fma_rn(e, e, b);
        }
    }
    for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) c = __fma_rn(bt[i], bt[i], c);
    a = warp_sum(a); b = warp_sum(b); c = warp_sum(c);
    if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = a; red[1][threadIdx.x >> 5] = b; red[2][threadIdx.x >> 5] = c; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double A = red[0][0], B = red[1][0], C = red[2][0];
        for (int w = 1; w < 8; ++w) { A = A + red[0][w]; B = B + red[1][w]; C = C + red[2][w]; }
        denoms[0] = A;  // ||x*||^2
        denoms[1] = C;  // local ||b~||^2 (summed over ranks by the host-side allreduce)
        st->it = 0; st->term = -1; st->last = -1;
        if (x_star) {
            const double res = A > 0.0 ? B / A : B;
            st->res_bits = __double_as_longlong(res);
            if (res <= tol) st->term = CSK_CONVERGED;
            else if (max_iters == 0) st->term = CSK_MAX_ITERS;
        }
    }
}

__global__ void k_zero_rows(double *p, int64_t count) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = 0.0;
}

csk_status_t nccl_fail(csk_ctx_t ctx, ncclResult_t r, const char *what) {
    return fail(ctx, CSK_E_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

#define CSK_NCCL(ctx, call)                                          \
    do {                                                             \
        ncclResult_t _r = (call);                                    \
        if (_r != ncclSuccess) return nccl_fail((ctx), _r, #call);   \
    } while (0)

// Exchange abstraction: NCCL all-gather, or loopback (virtual ranks on one device).
struct Gather {
    csk_ctx_t ctx;
    Comm *comm;  // nullptr -> loopback
};

struct ShardBufs {
    double *blk = nullptr;
    unsigned int *ticket = nullptr;
    double *send = nullptr;
    double *gathered = nullptr;
    ShardState *st = nullptr;
    double *denoms = nullptr;
};

int cand_grid(csk_ctx_t ctx, int64_t rows) {
    int64_t g = (rows + 7) / 8;
    if (g > ctx->num_sms * 4) g = ctx->num_sms * 4;
    if (g < 1) g = 1;
    return static_cast<int>(g);
}

}  // namespace

// ---------------------------------------------------------------- sharded loop driver
struct RankView {
    const double *At, *bt, *nsq;
    int64_t rows, row0;
    double *x;
    ShardBufs b;
};

static csk_status_t run_sharded_loop(csk_ctx_t ctx, std::vector<RankView> &ranks, Comm *comm, int64_t n,
                                     const double *x_star, double tol, int64_t max_iters,
                                     csk_report_t *report, cudaStream_t s) {
    const int P = comm ? comm->nranks : static_cast<int>(ranks.size());
    const int64_t rl = kRecHead + n;
    // init (per local rank view) and denominators
    for (auto &r : ranks) {
        k_shard_init<<<1, 256, 0, s>>>(r.x, x_star, r.bt, r.rows, n, tol, max_iters, r.b.st, r.b.denoms);
        CSK_CUDA(ctx, cudaGetLastError());
    }
    double denom_res = 0.0;
    {
        double d2[2];
        CSK_CUDA(ctx, cudaMemcpyAsync(d2, ranks[0].b.denoms, sizeof(d2), cudaMemcpyDeviceToHost, s));
        double bsum = 0.0;
        if (comm) {
            CSK_NCCL(ctx, ncclAllReduce(ranks[0].b.denoms + 1, ranks[0].b.denoms + 1, 1, ncclFloat64, ncclSum, comm->nccl, s));
            CSK_CUDA(ctx, cudaMemcpyAsync(&bsum, ranks[0].b.denoms + 1, sizeof(double), cudaMemcpyDeviceToHost, s));
            CSK_CUDA(ctx, cudaStreamSynchronize(s));
        } else {
            CSK_CUDA(ctx, cudaStreamSynchronize(s));
            for (auto &r : ranks) {  // rank order
                double v;
                CSK_CUDA(ctx, cudaMemcpy(&v, r.b.denoms + 1, sizeof(double), cudaMemcpyDeviceToHost));
                bsum = bsum + v;
            }
        }
        denom_res = x_star ? d2[0] : bsum;
    }
    ShardState hs{};
    for (int64_t k0 = 0;; k0 += kBatch) {
        for (int t = 0; t < kBatch; ++t) {
            for (size_t q = 0; q < ranks.size(); ++q) {
                auto &r = ranks[q];
                double *dst = comm ? r.b.send : ranks[0].b.gathered + q * rl;
                k_shard_candidate<<<cand_grid(ctx, r.rows), 256, 0, s>>>(
                    r.At, r.bt, r.nsq, r.rows, r.row0, n, r.x, r.b.blk, r.b.ticket, dst, r.b.st);
            }
            if (comm) {
                auto &r = ranks[0];
                CSK_NCCL(ctx, ncclAllGather(r.b.send, r.b.gathered, rl, ncclFloat64, comm->nccl, s));
            }
            for (auto &r : ranks) {
                k_shard_apply<<<1, 256, 0, s>>>(comm ? r.b.gathered : ranks[0].b.gathered, P, n, r.x, x_star,
                                                denom_res, tol, max_iters, r.b.st, nullptr, 0);
            }
            CSK_CUDA(ctx, cudaGetLastError());
        }
        CSK_CUDA(ctx, cudaMemcpyAsync(&hs, ranks[0].b.st, sizeof(hs), cudaMemcpyDeviceToHost, s));
        CSK_CUDA(ctx, cudaStreamSynchronize(s));
        if (hs.term >= 0 || hs.term == -2) break;
    }
    if (hs.term == -2) return fail(ctx, CSK_E_ZERO_SKETCH, "csk_solve_sharded: every row of A~ is zero");
    report->iterations = hs.it;
    double fr;
    memcpy(&fr, &hs.res_bits, sizeof(double));
    report->final_res = fr;
    report->termination = static_cast<int32_t>(hs.term);
    report->stop_mode = x_star ? CSK_STOP_RES : CSK_STOP_RESIDUAL;
    report->last_index = hs.last;
    return CSK_OK;
}

static csk_status_t alloc_shard_bufs(csk_ctx_t ctx, int64_t n, int P, int grid, ShardBufs &b,
                                     std::vector<void *> &owned) {
    const int64_t rl = kRecHead + n;
    auto get = [&](size_t bytes, void **out) -> csk_status_t {
        CSK_CUDA(ctx, cudaMalloc(out, bytes));
        owned.push_back(*out);
        return CSK_OK;
    };
    void *p;
    CSK_CHECK(get(static_cast<size_t>(grid) * 4 * 8, &p)); b.blk = static_cast<double *>(p);
    CSK_CHECK(get(64, &p)); b.ticket = static_cast<unsigned int *>(p);
    CSK_CUDA(ctx, cudaMemset(b.ticket, 0, 64));
    CSK_CHECK(get(static_cast<size_t>(rl) * 8, &p)); b.send = static_cast<double *>(p);
    CSK_CHECK(get(static_cast<size_t>(rl) * P * 8, &p)); b.gathered = static_cast<double *>(p);
    CSK_CHECK(get(sizeof(ShardState), &p)); b.st = static_cast<ShardState *>(p);
    CSK_CHECK(get(64, &p)); b.denoms = static_cast<double *>(p);
    return CSK_OK;
}

}  // namespace csk

using namespace csk;

extern "C" {

csk_status_t csk_shard_range(int64_t total, int32_t nranks, int32_t rank, int64_t *lo, int64_t *hi) {
    if (total < 0 || nranks < 1 || rank < 0 || rank >= nranks || !lo || !hi) return CSK_E_ARG;
    const int64_t c = (total + nranks - 1) / nranks;
    int64_t a = c * rank, e = c * (rank + 1);
    if (a > total) a = total;
    if (e > total) e = total;
    *lo = a;
    *hi = e;
    return CSK_OK;
}

csk_status_t csk_comm_unique_id(void *uid_out) {
    if (!uid_out) return CSK_E_ARG;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return CSK_E_NCCL;
    memcpy(uid_out, &id, sizeof(id));
    return CSK_OK;
}

csk_status_t csk_comm_create(csk_ctx_t ctx, const void *uid, int32_t nranks, int32_t rank) {
    if (!ctx || !uid || nranks < 1 || rank < 0 || rank >= nranks) return CSK_E_ARG;
    CSK_CUDA(ctx, cudaSetDevice(ctx->device));
    if (ctx->comm) return fail(ctx, CSK_E_ARG, "csk_comm_create: ctx already has a communicator");
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    auto *c = new Comm();
    ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, id, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_fail(ctx, r, "ncclCommInitRank");
    }
    c->nranks = nranks;
    c->rank = rank;
    ctx->comm = c;
    return CSK_OK;
}

csk_status_t csk_comm_destroy(csk_ctx_t ctx) {
    if (!ctx) return CSK_E_ARG;
    if (ctx->comm) {
        ncclCommDestroy(ctx->comm->nccl);
        delete ctx->comm;
        ctx->comm = nullptr;
    }
    return CSK_OK;
}

csk_status_t csk_sketch_sharded(csk_ctx_t ctx, const double *A_local, int64_t lda, const double *b_local,
                                int64_t m_local, int64_t row_offset, int64_t m, int64_t n, int64_t d,
                                uint64_t seed, double *A_tilde_local, double *b_tilde_local,
                                double *nsq_local, int64_t *d_lo, int64_t *d_hi, void *stream) {
    CSK_NVTX("csk_sketch_sharded");
    if (!ctx || !ctx->comm) return ctx ? fail(ctx, CSK_E_ARG, "csk_sketch_sharded: call csk_comm_create first") : CSK_E_ARG;
    if (!A_local || !b_local || !A_tilde_local || !b_tilde_local || !d_lo || !d_hi || m_local < 1 ||
        row_offset < 0 || row_offset + m_local > m || n < 1 || d < 1 || d >= m || lda < n)
        return fail(ctx, CSK_E_ARG, "csk_sketch_sharded: bad arguments (need 1 <= d < m, shard inside [0, m))");
    CSK_CUDA(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = as_stream(stream);
    Comm *c = ctx->comm;
    const int P = c->nranks;
    const int64_t chunk = (d + P - 1) / P;
    const int64_t dpad = chunk * P;
    // partial (A~ | b~) over all d buckets, rows >= d zero
    CSK_CHECK(ensure(ctx, ctx->a_tilde, static_cast<size_t>(dpad) * n * 8 + static_cast<size_t>(chunk) * n * 8));
    CSK_CHECK(ensure(ctx, ctx->b_tilde, static_cast<size_t>(dpad) * 8 + static_cast<size_t>(chunk) * 8));
    double *partA = static_cast<double *>(ctx->a_tilde.ptr);
    double *recvA = partA + dpad * n;
    double *partb = static_cast<double *>(ctx->b_tilde.ptr);
    double *recvb = partb + dpad;
    if (dpad > d) {
        k_zero_rows<<<64, 256, 0, s>>>(partA + d * n, (dpad - d) * n);
        k_zero_rows<<<1, 256, 0, s>>>(partb + d, dpad - d);
    }
    int32_t *perm = nullptr, *offsets = nullptr;
    CSK_CHECK(build_plan(ctx, seed, row_offset, m_local, d, nullptr, nullptr, &perm, &offsets, s));
    CSK_CHECK(launch_sketch_dense(ctx, A_local, lda, b_local, m_local, n, d, perm, offsets, partA, partb, nullptr, s));
    CSK_NCCL(ctx, ncclGroupStart());
    CSK_NCCL(ctx, ncclReduceScatter(partA, recvA, chunk * n, ncclFloat64, ncclSum, c->nccl, s));
    CSK_NCCL(ctx, ncclReduceScatter(partb, recvb, chunk, ncclFloat64, ncclSum, c->nccl, s));
    CSK_NCCL(ctx, ncclGroupEnd());
    int64_t lo, hi;
    csk_shard_range(d, P, c->rank, &lo, &hi);
    *d_lo = lo;
    *d_hi = hi;
    if (hi > lo) {
        CSK_CUDA(ctx, cudaMemcpyAsync(A_tilde_local, recvA, static_cast<size_t>(hi - lo) * n * 8, cudaMemcpyDeviceToDevice, s));
        CSK_CUDA(ctx, cudaMemcpyAsync(b_tilde_local, recvb, static_cast<size_t>(hi - lo) * 8, cudaMemcpyDeviceToDevice, s));
        if (nsq_local) CSK_CHECK(launch_row_norms(ctx, A_tilde_local, hi - lo, n, nsq_local, s));
    }
    return CSK_OK;
}

// S9 for CSR input.  CSK_SHARD_REDUCE_SCATTER: this rank's rows folded into a partial (A~ | b~)
// over all d buckets (global hashing), then the same grouped ncclReduceScatter as the dense path.
// CSK_SHARD_ROUTE_ROWS: every row goes to its bucket's owner (route.cu): the counts by an
// ncclAllGather, the rows and their pairs by grouped ncclSend/ncclRecv (self included), then the
// owner's plan + CSR sketch over its bucket range -- bit-identical to one GPU.
csk_status_t csk_sketch_csr_sharded(csk_ctx_t ctx, const int64_t *row_ptr, const int32_t *col, const double *val,
                                    const double *b_local, int64_t m_local, int64_t row_offset, int64_t m, int64_t n,
                                    int64_t d, uint64_t seed, int32_t mode, double *A_tilde_local,
                                    double *b_tilde_local, double *nsq_local, int64_t *d_lo, int64_t *d_hi,
                                    void *stream) {
    CSK_NVTX("csk_sketch_csr_sharded");
    if (!ctx || !ctx->comm) return ctx ? fail(ctx, CSK_E_ARG, "csk_sketch_csr_sharded: call csk_comm_create first") : CSK_E_ARG;
    if (!row_ptr || !col || !val || !b_local || !A_tilde_local || !b_tilde_local || !d_lo || !d_hi || m_local < 0 ||
        row_offset < 0 || row_offset + m_local > m || m >= (int64_t(1) << 31) || n < 1 || d < 1 || d >= m ||
        (mode != CSK_SHARD_REDUCE_SCATTER && mode != CSK_SHARD_ROUTE_ROWS))
        return fail(ctx, CSK_E_ARG, "csk_sketch_csr_sharded: bad arguments (need 1 <= d < m < 2^31, shard inside [0, m))");
    CSK_CUDA(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = as_stream(stream);
    Comm *c = ctx->comm;
    const int P = c->nranks, me = c->rank;
    if (P > kMaxRanks || d < P) return fail(ctx, CSK_E_UNSUPPORTED, "csk_sketch_csr_sharded: need P <= 8 and d >= P");
    int64_t lo, hi;
    csk_shard_range(d, P, me, &lo, &hi);
    *d_lo = lo;
    *d_hi = hi;
    if (mode == CSK_SHARD_REDUCE_SCATTER) {
        const int64_t chunk = (d + P - 1) / P;
        const int64_t dpad = chunk * P;
        CSK_CHECK(ensure(ctx, ctx->a_tilde, static_cast<size_t>(dpad) * n * 8 + static_cast<size_t>(chunk) * n * 8));
        CSK_CHECK(ensure(ctx, ctx->b_tilde, static_cast<size_t>(dpad) * 8 + static_cast<size_t>(chunk) * 8));
        double *partA = static_cast<double *>(ctx->a_tilde.ptr);
        double *recvA = partA + dpad * n;
        double *partb = static_cast<double *>(ctx->b_tilde.ptr);
        double *recvb = partb + dpad;
        if (dpad > d) {
            k_zero_rows<<<64, 256, 0, s>>>(partA + d * n, (dpad - d) * n);
            k_zero_rows<<<1, 256, 0, s>>>(partb + d, dpad - d);
        }
        if (m_local > 0) {
            int32_t *perm = nullptr, *offsets = nullptr;
            CSK_CHECK(build_plan(ctx, seed, row_offset, m_local, d, nullptr, nullptr, &perm, &offsets, s));
            CSK_CHECK(launch_sketch_csr(ctx, row_ptr, col, val, b_local, m_local, n, d, perm, offsets, partA, partb,
                                        nullptr, s));
        } else {
            k_zero_rows<<<64, 256, 0, s>>>(partA, d * n);
            k_zero_rows<<<1, 256, 0, s>>>(partb, d);
        }
        CSK_NCCL(ctx, ncclGroupStart());
        CSK_NCCL(ctx, ncclReduceScatter(partA, recvA, chunk * n, ncclFloat64, ncclSum, c->nccl, s));
        CSK_NCCL(ctx, ncclReduceScatter(partb, recvb, chunk, ncclFloat64, ncclSum, c->nccl, s));
        CSK_NCCL(ctx, ncclGroupEnd());
        if (hi > lo) {
            CSK_CUDA(ctx, cudaMemcpyAsync(A_tilde_local, recvA, static_cast<size_t>(hi - lo) * n * 8, cudaMemcpyDeviceToDevice, s));
            CSK_CUDA(ctx, cudaMemcpyAsync(b_tilde_local, recvb, static_cast<size_t>(hi - lo) * 8, cudaMemcpyDeviceToDevice, s));
            if (nsq_local) CSK_CHECK(launch_row_norms(ctx, A_tilde_local, hi - lo, n, nsq_local, s));
        }
        return CSK_OK;
    }
    // ---- row routing ----
    RoutePack pk;
    CSK_CHECK(route_pack(ctx, row_ptr, col, val, b_local, m_local, row_offset, d, seed, P, pk, s));
    int64_t *cnts = nullptr;  // [P][2P] every rank's per-destination counts, + this rank's at the end
    CSK_CUDA(ctx, cudaMallocAsync(reinterpret_cast<void **>(&cnts), static_cast<size_t>(P + 1) * 2 * P * 8, s));
    CSK_CUDA(ctx, cudaMemcpyAsync(cnts + static_cast<size_t>(P) * 2 * P, pk.cnt, static_cast<size_t>(2 * P) * 8,
                                  cudaMemcpyHostToDevice, s));
    CSK_NCCL(ctx, ncclAllGather(cnts + static_cast<size_t>(P) * 2 * P, cnts, 2 * P, ncclInt64, c->nccl, s));
    std::vector<int64_t> all(static_cast<size_t>(P) * 2 * P);
    CSK_CUDA(ctx, cudaMemcpyAsync(all.data(), cnts, all.size() * 8, cudaMemcpyDeviceToHost, s));
    CSK_CUDA(ctx, cudaStreamSynchronize(s));
    CSK_CUDA(ctx, cudaFreeAsync(cnts, s));
    RouteRecv rv;
    rv.P = P;
    for (int q = 0; q < P; ++q) {
        rv.rbase[q + 1] = rv.rbase[q] + all[static_cast<size_t>(q) * 2 * P + 2 * me];
        rv.pbase[q + 1] = rv.pbase[q] + all[static_cast<size_t>(q) * 2 * P + 2 * me + 1];
    }
    const int64_t M = rv.rbase[P], NNZ = rv.pbase[P];
    void *buf[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    const size_t sz[5] = {static_cast<size_t>(M) * 4, static_cast<size_t>(M) * 8, static_cast<size_t>(M) * 8,
                          static_cast<size_t>(NNZ) * 4, static_cast<size_t>(NNZ) * 8};
    for (int a = 0; a < 5; ++a) CSK_CUDA(ctx, cudaMallocAsync(&buf[a], sz[a] > 0 ? sz[a] : 16, s));
    CSK_NCCL(ctx, ncclGroupStart());
    for (int q = 0; q < P; ++q) {
        const int64_t sr = pk.seg[2 * q], nr = pk.cnt[2 * q], sp = pk.seg[2 * q + 1], np = pk.cnt[2 * q + 1];
        const int64_t rr = rv.rbase[q], mr = rv.rbase[q + 1] - rr, rp = rv.pbase[q], mp = rv.pbase[q + 1] - rp;
        CSK_NCCL(ctx, ncclSend(pk.row + sr, nr, ncclInt32, q, c->nccl, s));
        CSK_NCCL(ctx, ncclSend(pk.b + sr, nr, ncclFloat64, q, c->nccl, s));
        CSK_NCCL(ctx, ncclSend(pk.off + sr, nr, ncclInt64, q, c->nccl, s));
        CSK_NCCL(ctx, ncclSend(pk.col + sp, np, ncclInt32, q, c->nccl, s));
        CSK_NCCL(ctx, ncclSend(pk.val + sp, np, ncclFloat64, q, c->nccl, s));
        CSK_NCCL(ctx, ncclRecv(static_cast<int32_t *>(buf[0]) + rr, mr, ncclInt32, q, c->nccl, s));
        CSK_NCCL(ctx, ncclRecv(static_cast<double *>(buf[1]) + rr, mr, ncclFloat64, q, c->nccl, s));
        CSK_NCCL(ctx, ncclRecv(static_cast<int64_t *>(buf[2]) + rr, mr, ncclInt64, q, c->nccl, s));
        CSK_NCCL(ctx, ncclRecv(static_cast<int32_t *>(buf[3]) + rp, mp, ncclInt32, q, c->nccl, s));
        CSK_NCCL(ctx, ncclRecv(static_cast<double *>(buf[4]) + rp, mp, ncclFloat64, q, c->nccl, s));
    }
    CSK_NCCL(ctx, ncclGroupEnd());
    rv.row = static_cast<int32_t *>(buf[0]);
    rv.b = static_cast<double *>(buf[1]);
    rv.off = static_cast<int64_t *>(buf[2]);
    rv.col = static_cast<int32_t *>(buf[3]);
    rv.val = static_cast<double *>(buf[4]);
    csk_status_t st = route_unpack_sketch(ctx, rv, n, d, lo, hi, seed, A_tilde_local, b_tilde_local, nsq_local, s);
    for (void *p : buf) cudaFreeAsync(p, s);
    route_free(pk, s);
    return st;
}

// ---- S10 fused across GPUs: every rank runs the persistent k_loop on its rows; all P x Gr
//      CTAs take part in ONE exchange whose {count, max} pair lives in rank 0's memory and is
//      updated with system-scope atomics over NVLink; the winner's slot and row are read from
//      the owner's memory through peer mappings (CUDA IPC handles swapped with ncclAllGather).
constexpr int kXchWordsComm = 16;  // mirrors loop.cu's exchange layout (one 128-B line per pair)

struct IpcRec {
    cudaIpcMemHandle_t a;  // allocation holding this rank's A~ rows
    long long a_off;       // offset of A~_local inside it
    cudaIpcMemHandle_t x;  // this rank's exchange buffer (ctx->slots)
    long long x_off;       // offset of the exchange buffer inside its allocation
    long long ok;          // 1: both handles exported (0: e.g. a VMM allocation -- every rank falls back)
};

static csk_status_t ipc_handle(csk_ctx_t ctx, const void *ptr, cudaIpcMemHandle_t *h, long long *off) {
    // driver entry point through the runtime (no link-time dependency on libcuda)
    using GetRange = CUresult (*)(CUdeviceptr *, size_t *, CUdeviceptr);
    static GetRange get_range = nullptr;
    if (!get_range) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            return fail(ctx, CSK_E_CUDA, "cudaGetDriverEntryPoint(cuMemGetAddressRange) failed");
        get_range = reinterpret_cast<GetRange>(fn);
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
        return fail(ctx, CSK_E_CUDA, "cuMemGetAddressRange failed");
    CSK_CUDA(ctx, cudaIpcGetMemHandle(h, reinterpret_cast<void *>(base)));
    *off = static_cast<long long>(reinterpret_cast<uintptr_t>(ptr) - static_cast<uintptr_t>(base));
    return CSK_OK;
}

static csk_status_t ipc_open(csk_ctx_t ctx, const cudaIpcMemHandle_t &h, void **out) {
    const std::string key(reinterpret_cast<const char *>(&h), sizeof(h));
    auto it = ctx->comm->peer_open.find(key);
    if (it != ctx->comm->peer_open.end()) {
        *out = it->second;
        return CSK_OK;
    }
    void *p = nullptr;
    CSK_CUDA(ctx, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    ctx->comm->peer_open[key] = p;
    *out = p;
    return CSK_OK;
}

__global__ void k_sumsq_shard(const double *v, int64_t len, double *out) {
    // single CTA, fixed order: thread-strided fma, warp butterfly, warps in order
    __shared__ double red[32];
    double a = 0.0;
    for (int64_t i = threadIdx.x; i < len; i += blockDim.x) a = __fma_rn(v[i], v[i], a);
    a = warp_sum(a);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = red[0];
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) t = t + red[w];
        *out = t;
    }
}

// P2P sanity probe: rank r's word (r+1) * gamma must be readable by every rank through its
// peer mapping (system-scope loads).  bad = 1 on any mismatch.
__global__ void k_peer_probe(const unsigned long long *const *words, int P, int *bad) {
    const int r = threadIdx.x;
    if (r < P) {
        unsigned long long v;
        asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(words[r]) : "memory");
        if (v != static_cast<unsigned long long>(r + 1) * 0x9E3779B97F4A7C15ull) atomicExch(bad, 1);
    }
}

static csk_status_t solve_sharded_fused(csk_ctx_t ctx, const double *A_tilde_local, const double *b_tilde_local,
                                        const double *nsq_local, int64_t d_lo, int64_t d_hi, int64_t d, int64_t n,
                                        double *x, const double *x_star, double tol, int64_t max_iters,
                                        csk_report_t *report, cudaStream_t s) {
    Comm *cm = ctx->comm;
    const int P = cm->nranks, me = cm->rank;
    if (P > kMaxRanks) return fail(ctx, CSK_E_UNSUPPORTED, "csk_solve_sharded: more than 8 ranks");
    RankSetup rs;
    rs.P = P;
    rs.rank = me;
    // every SM of every GPU: the CTAs of a rank meet in that rank's memory, and only one key per
    // rank crosses NVLink (loop.cu, SYS), so the participant count does not grow with P
    rs.Gr = ctx->num_sms;
    rs.sys = 1;
    for (int r = 0; r < P; ++r) {
        int64_t lo, hi;
        csk_shard_range(d, P, r, &lo, &hi);
        rs.dlo[r] = lo;
        rs.dlo[r + 1] = hi;
    }
    if (rs.dlo[me] != d_lo || rs.dlo[me + 1] != d_hi)
        return fail(ctx, CSK_E_ARG, "csk_solve_sharded: [d_lo, d_hi) must be csk_shard_range(d, P, rank)");
    for (int r = 0; r < P; ++r)
        if (rs.dlo[r + 1] <= rs.dlo[r]) return fail(ctx, CSK_E_ARG, "csk_solve_sharded: a rank owns no rows (d < P)");
    // this rank's exchange buffer: [3 pairs][2][Gr] LL slots (rank 0's pairs are the global ones)
    const size_t ex = loop_exchange_bytes(rs.Gr);
    CSK_CHECK(ensure(ctx, ctx->slots, ex));
    CSK_CHECK(ensure(ctx, ctx->scalars, 8 * 8));
    const size_t xch_bytes = ex - static_cast<size_t>(2) * rs.Gr * 8 * 8;
    // the peer setup of the previous solve, if every rank calls again with the same buffers
    // (agreed by one all-reduce; any miss redoes the exchange of handles and the probe everywhere)
    {
        Comm::FusedSetup &fc = cm->fused;
        int hit = (fc.valid && fc.a == A_tilde_local && fc.slots == ctx->slots.ptr && fc.gr == rs.Gr &&
                   fc.d_lo == d_lo && fc.d_hi == d_hi)
                      ? 1
                      : 0;
        int *dflag = reinterpret_cast<int *>(static_cast<double *>(ctx->scalars.ptr) + 1);
        CSK_CUDA(ctx, cudaMemcpyAsync(dflag, &hit, sizeof(int), cudaMemcpyHostToDevice, s));
        CSK_NCCL(ctx, ncclAllReduce(dflag, dflag, 1, ncclInt32, ncclMin, cm->nccl, s));
        int all_hit = 0;
        CSK_CUDA(ctx, cudaMemcpyAsync(&all_hit, dflag, sizeof(int), cudaMemcpyDeviceToHost, s));
        CSK_CUDA(ctx, cudaStreamSynchronize(s));
        if (all_hit) {
            RankSetup rc = fc.rs;
            rc.bt_r[me] = b_tilde_local;
            rc.nsq_r[me] = nsq_local;
            rc.x_r[me] = x;
            CSK_CUDA(ctx, cudaMemsetAsync(ctx->slots.ptr, 0, ex, s));
            double *bb = static_cast<double *>(ctx->scalars.ptr);
            CSK_CUDA(ctx, cudaMemsetAsync(bb, 0, 8, s));
            rc.bb = nullptr;
            if (x_star == nullptr) {
                k_sumsq_shard<<<1, 1024, 0, s>>>(b_tilde_local, d_hi - d_lo, bb);
                rc.bb = bb;
            }
            CSK_NCCL(ctx, ncclAllReduce(bb, bb, 1, ncclFloat64, ncclSum, cm->nccl, s));  // + the barrier
            rc.exchange_zeroed = true;
            return run_loop(ctx, A_tilde_local, b_tilde_local, nsq_local, d_hi - d_lo, n, x, x_star, tol, max_iters,
                            nullptr, report, s, &rc);
        }
        fc.valid = false;
    }
    // swap IPC handles (A~ rows, exchange buffer) through NCCL.  An export failure is not an
    // error here: every rank sees every rank's `ok` after the all-gather and all of them take the
    // host-driven NCCL loop together
    IpcRec mine{};
    mine.ok = (ipc_handle(ctx, A_tilde_local, &mine.a, &mine.a_off) == CSK_OK &&
               ipc_handle(ctx, ctx->slots.ptr, &mine.x, &mine.x_off) == CSK_OK)
                  ? 1
                  : 0;
    if (!mine.ok) cudaGetLastError();  // clear a sticky-free runtime error of the failed export
    std::vector<IpcRec> all(P);
    void *dbuf = nullptr;
    CSK_CUDA(ctx, cudaMallocAsync(&dbuf, sizeof(IpcRec) * (P + 1), s));
    CSK_CUDA(ctx, cudaMemcpyAsync(static_cast<char *>(dbuf) + sizeof(IpcRec) * P, &mine, sizeof(IpcRec),
                                  cudaMemcpyHostToDevice, s));
    CSK_NCCL(ctx, ncclAllGather(static_cast<char *>(dbuf) + sizeof(IpcRec) * P, dbuf, sizeof(IpcRec), ncclUint8,
                                cm->nccl, s));
    CSK_CUDA(ctx, cudaMemcpyAsync(all.data(), dbuf, sizeof(IpcRec) * P, cudaMemcpyDeviceToHost, s));
    CSK_CUDA(ctx, cudaStreamSynchronize(s));
    for (int r = 0; r < P; ++r)
        if (!all[r].ok) {
            CSK_CUDA(ctx, cudaFreeAsync(dbuf, s));
            return CSK_E_UNSUPPORTED;  // every rank returns here: the host-driven loop
        }
    int open_bad = 0;  // a failed peer mapping is agreed on through the probe's all-reduce below
    for (int r = 0; r < P; ++r) {
        unsigned char *xb = nullptr;
        if (r == me) {
            rs.At_r[r] = A_tilde_local;
            xb = static_cast<unsigned char *>(ctx->slots.ptr);
        } else {
            void *a = nullptr, *xp = nullptr;
            if (ipc_open(ctx, all[r].a, &a) != CSK_OK || ipc_open(ctx, all[r].x, &xp) != CSK_OK) {
                cudaGetLastError();
                open_bad = 1;
                rs.At_r[r] = A_tilde_local;  // placeholders, never dereferenced
                xb = static_cast<unsigned char *>(ctx->slots.ptr);
            } else {
                rs.At_r[r] = reinterpret_cast<const double *>(static_cast<unsigned char *>(a) + all[r].a_off);
                xb = static_cast<unsigned char *>(xp) + all[r].x_off;
            }
        }
        rs.slots_r[r] = reinterpret_cast<unsigned long long *>(xb + xch_bytes);
    }
    rs.bt_r[me] = b_tilde_local;
    rs.nsq_r[me] = nsq_local;
    rs.x_r[me] = x;
    // probe the peer mappings once per solve: every rank writes a word into its exchange buffer,
    // reads every rank's word through the mappings, and all ranks agree (all-reduce max) on the
    // outcome; a failure selects the host-driven NCCL loop on every rank
    {
        const size_t probe_off = (2 * kXchWordsComm + 8) * 8;  // unused word of the third pair line
        const unsigned long long mine_w = static_cast<unsigned long long>(me + 1) * 0x9E3779B97F4A7C15ull;
        CSK_CUDA(ctx, cudaMemcpyAsync(static_cast<unsigned char *>(ctx->slots.ptr) + probe_off, &mine_w, 8,
                                      cudaMemcpyHostToDevice, s));
        const unsigned long long *words[kMaxRanks];
        for (int r = 0; r < P; ++r)
            words[r] = reinterpret_cast<const unsigned long long *>(
                reinterpret_cast<const unsigned char *>(rs.slots_r[r]) - xch_bytes + probe_off);
        void *pb = nullptr;
        CSK_CUDA(ctx, cudaMallocAsync(&pb, sizeof(words) + 16, s));
        CSK_CUDA(ctx, cudaMemcpyAsync(pb, words, sizeof(words), cudaMemcpyHostToDevice, s));
        int *bad = reinterpret_cast<int *>(static_cast<unsigned char *>(pb) + sizeof(words));
        CSK_CUDA(ctx, cudaMemcpyAsync(bad, &open_bad, sizeof(int), cudaMemcpyHostToDevice, s));
        CSK_NCCL(ctx, ncclAllReduce(bad, bad, 1, ncclInt32, ncclMax, cm->nccl, s));  // barrier: all words written
        if (!open_bad) k_peer_probe<<<1, 32, 0, s>>>(reinterpret_cast<const unsigned long long *const *>(pb), P, bad);
        CSK_NCCL(ctx, ncclAllReduce(bad, bad, 1, ncclInt32, ncclMax, cm->nccl, s));
        int bad_h = 0;
        CSK_CUDA(ctx, cudaMemcpyAsync(&bad_h, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
        CSK_CUDA(ctx, cudaStreamSynchronize(s));
        CSK_CUDA(ctx, cudaFreeAsync(pb, s));
        if (bad_h) return CSK_E_UNSUPPORTED;  // caller falls back to the host-driven loop
    }
    // zero the exchange memory, and the global ||b~||^2 for residual mode; the all-reduce is
    // also the barrier that keeps every rank's kernel behind rank 0's zeroed pairs
    CSK_CUDA(ctx, cudaMemsetAsync(ctx->slots.ptr, 0, ex, s));
    double *bb = static_cast<double *>(ctx->scalars.ptr);
    CSK_CUDA(ctx, cudaMemsetAsync(bb, 0, 8, s));
    if (x_star == nullptr) {
        k_sumsq_shard<<<1, 1024, 0, s>>>(b_tilde_local, d_hi - d_lo, bb);
        rs.bb = bb;
    }
    CSK_NCCL(ctx, ncclAllReduce(bb, bb, 1, ncclFloat64, ncclSum, cm->nccl, s));
    CSK_CUDA(ctx, cudaFreeAsync(dbuf, s));
    rs.exchange_zeroed = true;
    cm->fused.valid = true;  // peers mapped and probed: reusable while the buffers stay the same
    cm->fused.a = A_tilde_local;
    cm->fused.slots = ctx->slots.ptr;
    cm->fused.gr = rs.Gr;
    cm->fused.d_lo = d_lo;
    cm->fused.d_hi = d_hi;
    cm->fused.rs = rs;
    return run_loop(ctx, A_tilde_local, b_tilde_local, nsq_local, d_hi - d_lo, n, x, x_star, tol, max_iters, nullptr,
                    report, s, &rs);
}

csk_status_t csk_solve_sharded(csk_ctx_t ctx, const double *A_tilde_local, const double *b_tilde_local,
                               const double *nsq_local, int64_t d_lo, int64_t d_hi, int64_t d, int64_t n,
                               double *x, const double *x_star, double tol, int64_t max_iters,
                               csk_report_t *report, void *stream) {
    CSK_NVTX("csk_solve_sharded");
    if (!ctx || !ctx->comm) return ctx ? fail(ctx, CSK_E_ARG, "csk_solve_sharded: call csk_comm_create first") : CSK_E_ARG;
    if (!report || !x || n < 1 || d < 1 || d_lo < 0 || d_hi < d_lo || d_hi > d || !(tol > 0.0) || max_iters < 0 ||
        (d_hi > d_lo && (!A_tilde_local || !b_tilde_local || !nsq_local)))
        return fail(ctx, CSK_E_ARG, "csk_solve_sharded: bad arguments");
    CSK_CUDA(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = as_stream(stream);
    // default: the fused persistent loop over peer memory; CSK_SHARDED_NCCL=1 selects the
    // host-driven loop (local candidate kernel + ncclAllGather + apply kernel per iteration)
    static const bool host_nccl = getenv("CSK_SHARDED_NCCL") != nullptr;
    if (!host_nccl) {
        const csk_status_t fst = solve_sharded_fused(ctx, A_tilde_local, b_tilde_local, nsq_local, d_lo, d_hi, d, n,
                                                     x, x_star, tol, max_iters, report, s);
        if (fst != CSK_E_UNSUPPORTED) return fst;
        // peer memory unusable (probe failed / no P2P): the host-driven NCCL loop below
    }
    std::vector<void *> owned;
    std::vector<RankView> rv(1);
    rv[0] = RankView{A_tilde_local, b_tilde_local, nsq_local, d_hi - d_lo, d_lo, x, {}};
    csk_status_t st = alloc_shard_bufs(ctx, n, ctx->comm->nranks, cand_grid(ctx, d_hi - d_lo), rv[0].b, owned);
    if (st == CSK_OK) st = run_sharded_loop(ctx, rv, ctx->comm, n, x_star, tol, max_iters, report, s);
    cudaStreamSynchronize(s);
    for (void *p : owned) cudaFree(p);
    return st;
}

// P virtual ranks on this device: A_tilde is the full d x n sketch; rank p owns rows
// csk_shard_range(d, P, p); every virtual rank keeps its own copy of x (all must agree).
csk_status_t csk_solve_virtual_ranks(csk_ctx_t ctx, const double *A_tilde, const double *b_tilde,
                                     const double *nsq, int64_t d, int64_t n, int32_t nranks, double *x,
                                     const double *x_star, double tol, int64_t max_iters,
                                     double *x_copies, csk_report_t *report, void *stream) {
    return csk_solve_virtual_ranks_ex(ctx, A_tilde, b_tilde, nsq, d, n, nranks, x, x_star, tol, max_iters,
                                      x_copies, nullptr, report, stream);
}

csk_status_t csk_solve_virtual_ranks_ex(csk_ctx_t ctx, const double *A_tilde, const double *b_tilde,
                                        const double *nsq, int64_t d, int64_t n, int32_t nranks, double *x,
                                        const double *x_star, double tol, int64_t max_iters,
                                        double *x_copies, const csk_solve_opts_t *opts, csk_report_t *report,
                                        void *stream) {
    CSK_NVTX("csk_solve_virtual_ranks_ex");
    if (!ctx || !A_tilde || !b_tilde || !nsq || !x || !report || nranks < 1 || d < 1 || n < 1 || !(tol > 0.0) ||
        max_iters < 0)
        return ctx ? fail(ctx, CSK_E_ARG, "csk_solve_virtual_ranks: bad arguments") : CSK_E_ARG;
    if (nranks > kMaxRanks)
        return fail(ctx, CSK_E_UNSUPPORTED, "csk_solve_virtual_ranks: more than 8 ranks");
    CSK_CUDA(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = as_stream(stream);
    // The fused S10 loop with P virtual ranks in ONE cooperative launch: rank r's CTAs own the
    // rows of csk_shard_range(d, P, r) and run the same grid-wide exchange the P-GPU launch runs
    // (there with peer-mapped memory); every virtual rank writes its own copy of x.
    void *tmp = nullptr;
    double *copies = x_copies;
    if (!copies) {
        if (cudaMalloc(&tmp, static_cast<size_t>(nranks) * n * 8) != cudaSuccess)
            return fail(ctx, CSK_E_NOMEM, "csk_solve_virtual_ranks: cudaMalloc");
        copies = static_cast<double *>(tmp);
    }
    RankSetup rs;
    rs.P = nranks;
    rs.rank = -1;
    rs.Gr = ctx->num_sms / nranks;
    rs.sys = 0;
    for (int p = 0; p < nranks; ++p) {
        int64_t lo, hi;
        csk_shard_range(d, nranks, p, &lo, &hi);
        rs.dlo[p] = lo;
        rs.dlo[p + 1] = hi;
        rs.At_r[p] = A_tilde + lo * n;
        rs.bt_r[p] = b_tilde + lo;
        rs.nsq_r[p] = nsq + lo;
        rs.x_r[p] = copies + static_cast<size_t>(p) * n;
        cudaMemcpyAsync(rs.x_r[p], x, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToDevice, s);
    }
    for (int p = 0; p < nranks; ++p)
        if (rs.dlo[p + 1] <= rs.dlo[p])
            return fail(ctx, CSK_E_ARG, "csk_solve_virtual_ranks: a rank owns no rows (d < P)");
    // only the traces of opts apply (the geometry is the sharded one)
    csk_solve_opts_t tr{};
    if (opts) {
        tr.trace_cap = opts->trace_cap;
        tr.idx_trace = opts->idx_trace;
        tr.res_trace = opts->res_trace;
        tr.x_trace = opts->x_trace;
        tr.r_trace = opts->r_trace;
        tr.r_trace_cap = opts->r_trace_cap;
    }
    csk_status_t st = run_loop(ctx, A_tilde, b_tilde, nsq, d, n, x, x_star, tol, max_iters, opts ? &tr : nullptr,
                               report, s, &rs);
    if (st == CSK_OK) cudaMemcpyAsync(x, copies, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToDevice, s);
    cudaStreamSynchronize(s);
    if (tmp) cudaFree(tmp);
    return st;
}

}  // extern "C"
