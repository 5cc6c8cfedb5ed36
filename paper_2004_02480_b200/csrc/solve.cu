// solve.cu -- S5..S8: the Algorithm 1 loop as ONE persistent kernel.
//
// Every iteration k (all steps fused, no per-iteration launch):
//   S6  r_i = b~_i - A~^(i) x_k for the CTA's rows (P:62 numerator).  Each warp keeps
//       a private copy of x in registers (lane l holds column pairs l + 32v), so the
//       GEMV streams only A~: from shared memory for the rows resident there, from
//       L2/HBM (ld.global.nc, no L1 allocate) for the rest.
//   S7  score_i = r_i^2 / nsq_i (squared form), masked rows score -1;
//       warp argmax -> CTA argmax (smem) -> grid argmax through a one-round-trip
//       exchange: every CTA publishes (score, lambda, idx, sum r^2) as eight 64-bit
//       words each carrying the iteration tag in its low half (LL-style: every
//       8-byte store is single-copy atomic, so a reader that sees the tag in all
//       words has consistent data), double-buffered by iteration parity; one warp
//       per CTA polls all G slots.  Ties -> lowest row index (north_star).
//   S8  lambda = r_ik / nsq_ik (computed by the owning CTA); every warp of every CTA
//       applies x += lambda * A~^(ik) to its register copy with the same fma in the
//       same order, so all copies stay bit-identical and every CTA takes the same
//       stop decision without further communication.
//   S5  RES_{k+1} = ||x - x*||^2/||x*||^2 per warp (butterfly), or in
//       residual mode ||r||^2/||b~||^2 from the exchanged partial sums.
// Launch: cooperative (all CTAs co-resident, required by the spin exchange).
#include <cooperative_groups.h>

#include <string.h>

#include "csk_internal.cuh"

namespace csk {

namespace {

constexpr int kMaxSlotsPerLane = 5;  // G <= 160 CTAs
constexpr int kMaxG = 32 * kMaxSlotsPerLane;
constexpr int kSlotWords = 8;        // 64-byte slot

struct SolveParams {
    const double *At;
    const double *bt;
    const double *nsq;
    int64_t d, n;
    double *x;
    const double *x_star;
    double tol;
    int64_t max_iters;
    uint64_t *slots;        // [2][G][8] words
    int64_t *report;        // [0]=iterations, [1]=final_res bits, [2]=termination, [3]=last idx
    const double *bb;       // residual mode: ||b~||^2 (device scalar)
    int smem_rows_cap;      // rows per CTA kept in shared memory
    int64_t trace_cap;
    int64_t *idx_trace;
    double *res_trace;
    double *x_trace;
};

struct Cand {
    double score;
    double lambda;
    double rr;
    int64_t idx;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// (score desc, idx asc) total order; `better(a, b)` = a should win over b.
__device__ __forceinline__ bool better(double sa, int64_t ia, double sb, int64_t ib) {
    return sa > sb || (sa == sb && ia < ib);
}

__device__ __forceinline__ void warp_argmax(double &score, int64_t &idx, double &lambda) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, score, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, idx, o);
        const double ol = __shfl_xor_sync(0xffffffffu, lambda, o);
        if (better(os, oi, score, idx)) {
            score = os;
            idx = oi;
            lambda = ol;
        }
    }
}

__device__ __forceinline__ uint64_t pack(uint32_t data, uint32_t tag) {
    return (static_cast<uint64_t>(data) << 32) | tag;
}

template <bool EVEN>
__device__ __forceinline__ double2 load_pair_global(const double *row, int64_t q, int64_t n) {
    if (EVEN) return ldg_stream2(row + 2 * q);
    double2 v;
    v.x = ldg_stream1(row + 2 * q);
    v.y = (2 * q + 1 < n) ? ldg_stream1(row + 2 * q + 1) : 0.0;
    return v;
}

template <int NV, int R, int W, bool EVEN, bool RESMODE>
__global__ void __launch_bounds__(W * 32, 1) k_solve(const SolveParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, cta = blockIdx.x;
    const int64_t d = p.d, n = p.n;
    const int64_t npairs = (n + 1) >> 1;
    const int64_t npairs_pad = 32 * NV;
    const int64_t r0 = d * cta / G, r1 = d * (cta + 1) / G;
    const int rows = static_cast<int>(r1 - r0);
    const int srows = rows < p.smem_rows_cap ? rows : p.smem_rows_cap;

    // shared-memory carve-up
    double2 *xs2 = reinterpret_cast<double2 *>(smem);            // x* pairs   [npairs_pad]
    double2 *wrow = xs2 + npairs_pad;                             // winner row [npairs_pad]
    double *bt_loc = reinterpret_cast<double *>(wrow + npairs_pad);  // [rows]
    double *nsq_loc = bt_loc + rows;                              // [rows]
    Cand *cand = reinterpret_cast<Cand *>(nsq_loc + rows);                     // [W]
    volatile int64_t *win_i = reinterpret_cast<int64_t *>(cand + W);        // [4]
    double2 *arows = reinterpret_cast<double2 *>(cand + W) + 2;  // [srows][npairs]

    // ---- prologue: stage resident rows, b~, nsq, x* ----
    for (int64_t e = tid; e < static_cast<int64_t>(srows) * npairs; e += blockDim.x) {
        const int64_t l = e / npairs, q = e - l * npairs;
        const double *src = p.At + (r0 + l) * n;
        double2 v;
        if (EVEN) {
            v = *reinterpret_cast<const double2 *>(src + 2 * q);
        } else {
            v.x = src[2 * q];
            v.y = (2 * q + 1 < n) ? src[2 * q + 1] : 0.0;
        }
        arows[e] = v;
    }
    for (int l = tid; l < rows; l += blockDim.x) {
        bt_loc[l] = p.bt[r0 + l];
        nsq_loc[l] = p.nsq[r0 + l];
    }
    for (int64_t q = tid; q < npairs_pad; q += blockDim.x) {
        double2 v = make_double2(0.0, 0.0);
        if (!RESMODE && q < npairs) {
            v.x = p.x_star[2 * q];
            if (2 * q + 1 < n) v.y = p.x_star[2 * q + 1];
        }
        xs2[q] = v;
    }
    // x_0 into registers (every warp holds the whole vector, lane-strided pairs)
    double2 xr[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const int64_t q = lane + 32 * v;
        xr[v] = make_double2(0.0, 0.0);
        if (q < npairs) {
            xr[v].x = p.x[2 * q];
            if (2 * q + 1 < n) xr[v].y = p.x[2 * q + 1];
        }
    }
    __syncthreads();

    // ||x*||^2 and RES_0 (per warp, identical everywhere)
    double xs_nrm = 0.0;
    double res = 0.0;
    if (!RESMODE) {
        double a = 0.0, bnum = 0.0;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const double2 s = xs2[lane + 32 * v];
            a = __fma_rn(s.x, s.x, a);
            a = __fma_rn(s.y, s.y, a);
            const double ex = xr[v].x - s.x, ey = xr[v].y - s.y;
            bnum = __fma_rn(ex, ex, bnum);
            bnum = __fma_rn(ey, ey, bnum);
        }
        xs_nrm = warp_sum(a);
        bnum = warp_sum(bnum);
        res = xs_nrm > 0.0 ? bnum / xs_nrm : bnum;
    }
    const double bb = RESMODE ? *p.bb : 0.0;

    int64_t k = 0;
    int64_t last = -1;
    int term = -1;
    for (;; ++k) {
        // trace x_k (CTA 0, warp 0)
        if (cta == 0 && warp == 0 && k < p.trace_cap) {
            if (p.x_trace) {
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const int64_t q = lane + 32 * v;
                    if (q < npairs) {
                        p.x_trace[k * n + 2 * q] = xr[v].x;
                        if (2 * q + 1 < n) p.x_trace[k * n + 2 * q + 1] = xr[v].y;
                    }
                }
            }
            if (!RESMODE && p.res_trace && lane == 0) p.res_trace[k] = res;
        }
        if (!RESMODE) {
            if (res <= p.tol) { term = CSK_CONVERGED; break; }
            if (k == p.max_iters) { term = CSK_MAX_ITERS; break; }
        }

        // ---- S6/S7 local: GEMV over this warp's rows, warp argmax ----
        double best_s = -2.0, best_l = 0.0, rr = 0.0;
        int64_t best_i = INT64_MAX;
        for (int l0 = warp * R; l0 < rows; l0 += W * R) {
            double acc[R];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = 0.0;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const int64_t q = lane + 32 * v;
                if (q < npairs) {
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int l = l0 + r;
                        if (l < rows) {
                            const double2 a = (l < srows)
                                                  ? arows[static_cast<int64_t>(l) * npairs + q]
                                                  : load_pair_global<EVEN>(p.At + (r0 + l) * n, q, n);
                            acc[r] = __fma_rn(a.x, xr[v].x, acc[r]);
                            acc[r] = __fma_rn(a.y, xr[v].y, acc[r]);
                        }
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int l = l0 + r;
                const double dot = warp_sum(acc[r]);
                if (l < rows) {
                    const double ri = bt_loc[l] - dot;
                    const double ns = nsq_loc[l];
                    const double sc = ns > 0.0 ? (ri * ri) / ns : -1.0;
                    if (RESMODE) rr = __fma_rn(ri, ri, rr);
                    if (sc > best_s) {  // rows visited in ascending order: keep the first max
                        best_s = sc;
                        best_i = r0 + l;
                        best_l = ns > 0.0 ? ri / ns : 0.0;
                    }
                }
            }
        }
        if (lane == 0) cand[warp] = Cand{best_s, best_l, rr, best_i};
        __syncthreads();

        // ---- S7 grid: CTA candidate -> exchange -> global winner (warp 0) ----
        if (warp == 0) {
            double cs = -2.0, cl = 0.0;
            int64_t ci = INT64_MAX;
            if (lane < W) {
                cs = cand[lane].score;
                cl = cand[lane].lambda;
                ci = cand[lane].idx;
            }
            warp_argmax(cs, ci, cl);
            double crr = 0.0;
            if (RESMODE) {
                for (int w = 0; w < W; ++w) crr = crr + cand[w].rr;  // fixed order
            }
            const uint32_t tag = static_cast<uint32_t>(k + 1);
            uint64_t *slot_base = p.slots + static_cast<size_t>(k & 1) * G * kSlotWords;
            if (lane == 0) {
                const uint64_t sb = __double_as_longlong(cs), lb = __double_as_longlong(cl),
                               rb = __double_as_longlong(crr);
                uint64_t *s = slot_base + static_cast<size_t>(cta) * kSlotWords;
                st_relaxed_v2u64(s + 0, pack(static_cast<uint32_t>(sb >> 32), tag),
                                 pack(static_cast<uint32_t>(sb), tag));
                st_relaxed_v2u64(s + 2, pack(static_cast<uint32_t>(lb >> 32), tag),
                                 pack(static_cast<uint32_t>(lb), tag));
                st_relaxed_v2u64(s + 4, pack(static_cast<uint32_t>(rb >> 32), tag),
                                 pack(static_cast<uint32_t>(rb), tag));
                st_relaxed_v2u64(s + 6, pack(static_cast<uint32_t>(ci), tag), pack(0u, tag));
            }
            // poll every CTA's slot (lane l owns slots l, l+32, ...)
            double gs[kMaxSlotsPerLane], gl[kMaxSlotsPerLane], gr[kMaxSlotsPerLane];
            int64_t gi[kMaxSlotsPerLane];
            uint32_t pending = 0;
#pragma unroll
            for (int j = 0; j < kMaxSlotsPerLane; ++j) {
                gs[j] = -2.0; gl[j] = 0.0; gr[j] = 0.0; gi[j] = INT64_MAX;
                if (lane + 32 * j < G) pending |= 1u << j;
            }
            while (true) {
#pragma unroll
                for (int j = 0; j < kMaxSlotsPerLane; ++j) {
                    if (pending & (1u << j)) {
                        const uint64_t *s = slot_base + static_cast<size_t>(lane + 32 * j) * kSlotWords;
                        uint64_t w0, w1, w2, w3, w4, w5, w6, w7;
                        ld_relaxed_v2u64(s + 0, w0, w1);
                        ld_relaxed_v2u64(s + 2, w2, w3);
                        ld_relaxed_v2u64(s + 4, w4, w5);
                        ld_relaxed_v2u64(s + 6, w6, w7);
                        const bool ok = static_cast<uint32_t>(w0) == tag &&
                                        static_cast<uint32_t>(w1) == tag &&
                                        static_cast<uint32_t>(w2) == tag &&
                                        static_cast<uint32_t>(w3) == tag &&
                                        static_cast<uint32_t>(w4) == tag &&
                                        static_cast<uint32_t>(w5) == tag &&
                                        static_cast<uint32_t>(w6) == tag;
                        if (ok) {
                            gs[j] = __longlong_as_double(static_cast<long long>((w0 >> 32) << 32 | (w1 >> 32)));
                            gl[j] = __longlong_as_double(static_cast<long long>((w2 >> 32) << 32 | (w3 >> 32)));
                            gr[j] = __longlong_as_double(static_cast<long long>((w4 >> 32) << 32 | (w5 >> 32)));
                            const uint32_t iw = static_cast<uint32_t>(w6 >> 32);
                            gi[j] = (iw == 0xffffffffu) ? INT64_MAX : static_cast<int64_t>(iw);
                            pending &= ~(1u << j);
                        }
                    }
                }
                if (__all_sync(0xffffffffu, pending == 0)) break;
            }
            // combine in a fixed order: lane's slots ascending, then butterfly
            double ws = -2.0, wl = 0.0, wr = 0.0;
            int64_t wi = INT64_MAX;
#pragma unroll
            for (int j = 0; j < kMaxSlotsPerLane; ++j) {
                if (better(gs[j], gi[j], ws, wi)) { ws = gs[j]; wi = gi[j]; wl = gl[j]; }
                if (RESMODE) wr = wr + gr[j];
            }
            warp_argmax(ws, wi, wl);
            if (RESMODE) wr = warp_sum(wr);
            if (lane == 0) {
                win_i[0] = wi;
                win_i[1] = __double_as_longlong(wl);
                win_i[2] = __double_as_longlong(ws);
                win_i[3] = __double_as_longlong(wr);
            }
            // stage the winner row A~^(ik) in shared memory
            if (ws > 0.0) {
                const double *src = p.At + wi * n;
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const int64_t q = lane + 32 * v;
                    if (q < npairs) wrow[q] = load_pair_global<EVEN>(src, q, n);
                }
            }
        }
        __syncthreads();

        const int64_t wi = win_i[0];
        const double wl = __longlong_as_double(win_i[1]);
        const double ws = __longlong_as_double(win_i[2]);
        if (RESMODE) {
            const double rrt = __longlong_as_double(win_i[3]);
            res = bb > 0.0 ? rrt / bb : rrt;
            if (cta == 0 && tid == 0 && p.res_trace && k < p.trace_cap) p.res_trace[k] = res;
            if (res <= p.tol) { term = CSK_CONVERGED; break; }
            if (k == p.max_iters) { term = CSK_MAX_ITERS; break; }
        }
        if (ws < 0.0) { term = -2; break; }            // every row masked: zero sketch
        if (ws == 0.0) { term = CSK_STAGNATED; break; }
        if (cta == 0 && tid == 0 && p.idx_trace && k < p.trace_cap) p.idx_trace[k] = wi;

        // ---- S8: x_{k+1} = x_k + lambda A~^(ik)T ----
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const int64_t q = lane + 32 * v;
            if (q < npairs) {
                const double2 a = wrow[q];
                xr[v].x = __fma_rn(wl, a.x, xr[v].x);
                xr[v].y = __fma_rn(wl, a.y, xr[v].y);
            }
        }
        last = wi;
        // ---- S5: RES_{k+1} ----
        if (!RESMODE) {
            double bnum = 0.0;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const double2 s = xs2[lane + 32 * v];
                const double ex = xr[v].x - s.x, ey = xr[v].y - s.y;
                bnum = __fma_rn(ex, ex, bnum);
                bnum = __fma_rn(ey, ey, bnum);
            }
            bnum = warp_sum(bnum);
            res = xs_nrm > 0.0 ? bnum / xs_nrm : bnum;
        }
    }

    // ---- epilogue: CTA 0 writes x and the report ----
    if (cta == 0 && warp == 0) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const int64_t q = lane + 32 * v;
            if (q < npairs) {
                p.x[2 * q] = xr[v].x;
                if (2 * q + 1 < n) p.x[2 * q + 1] = xr[v].y;
            }
        }
        if (lane == 0) {
            p.report[0] = k;
            p.report[1] = __double_as_longlong(res);
            p.report[2] = term;
            p.report[3] = last;
        }
    }
}

__global__ void k_sumsq(const double *v, int64_t len, double *out) {
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

using KernelFn = void (*)(const SolveParams);

template <int NV, bool EVEN, bool RESMODE>
KernelFn pick_w() {
    constexpr int R = NV >= 32 ? 1 : 2;
    constexpr int W = NV <= 4 ? 16 : 8;
    return k_solve<NV, R, W, EVEN, RESMODE>;
}
template <int NV>
KernelFn pick_mode(bool even, bool resmode, int &warps) {
    warps = NV <= 4 ? 16 : 8;
    if (even) return resmode ? pick_w<NV, true, true>() : pick_w<NV, true, false>();
    return resmode ? pick_w<NV, false, true>() : pick_w<NV, false, false>();
}

KernelFn pick_kernel(int64_t n, bool resmode, int &nv, int &warps) {
    const int64_t npairs = (n + 1) / 2;
    const bool even = (n & 1) == 0;
    nv = 1;
    while (32 * nv < npairs) nv *= 2;
    switch (nv) {
        case 1: return pick_mode<1>(even, resmode, warps);
        case 2: return pick_mode<2>(even, resmode, warps);
        case 4: return pick_mode<4>(even, resmode, warps);
        case 8: return pick_mode<8>(even, resmode, warps);
        case 16: return pick_mode<16>(even, resmode, warps);
        case 32: return pick_mode<32>(even, resmode, warps);
        default: return nullptr;
    }
}

}  // namespace

csk_status_t run_solve(csk_ctx_t ctx, const double *At, const double *bt, const double *nsq,
                       int64_t d, int64_t n, double *x, const double *x_star, double tol,
                       int64_t max_iters, const csk_solve_opts_t *opts, csk_report_t *report,
                       cudaStream_t stream) {
    if (d < 1 || n < 1 || !At || !bt || !nsq || !x || !(tol > 0.0) || max_iters < 0 ||
        (!report && !(opts && (opts->flags & CSK_SOLVE_ASYNC))))
        return fail(ctx, CSK_E_ARG, "csk_solve: need d, n >= 1, non-null A~, b~, nsq, x, report, tol > 0, max_iters >= 0");
    if (d >= (int64_t(1) << 31) - 1) return fail(ctx, CSK_E_ARG, "csk_solve: d >= 2^31");
    if (n > CSK_MAX_N) return fail(ctx, CSK_E_UNSUPPORTED, "csk_solve: n > CSK_MAX_N");
    if ((n % 2 == 0) && !aligned16(At)) return fail(ctx, CSK_E_ARG, "csk_solve: A~ not 16-byte aligned");
    const bool resmode = (x_star == nullptr);
    int nv = 0, warps = 0;
    KernelFn fn = pick_kernel(n, resmode, nv, warps);
    if (!fn) return fail(ctx, CSK_E_UNSUPPORTED, "csk_solve: n out of range");
    const int threads = warps * 32;

    int G = ctx->num_sms;
    if (opts && opts->num_ctas > 0) G = opts->num_ctas;
    if (G > kMaxG) G = kMaxG;
    if (G > d) G = static_cast<int>(d);
    const int64_t rows_max = (d + G - 1) / G;
    const int64_t npairs = (n + 1) / 2;
    const size_t fixed = static_cast<size_t>(2 * 32 * nv) * 16 + static_cast<size_t>(rows_max) * 16 +
                         static_cast<size_t>(warps) * sizeof(Cand) + 4 * 8 + 64;
    const size_t avail = ctx->max_smem_optin > static_cast<int>(fixed) ? ctx->max_smem_optin - fixed : 0;
    int64_t srows = static_cast<int64_t>(avail / (static_cast<size_t>(npairs) * 16));
    if (srows > rows_max) srows = rows_max;
    if (opts && opts->smem_rows > 0 && opts->smem_rows < srows) srows = opts->smem_rows;
    if (opts && opts->smem_rows < 0) srows = 0;
    const size_t smem = fixed + static_cast<size_t>(srows) * npairs * 16;

    CSK_CUDA(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int per_sm = 0;
    CSK_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem));
    if (per_sm * ctx->num_sms < G)
        return fail(ctx, CSK_E_UNSUPPORTED, "csk_solve: grid cannot be co-resident");

    CSK_CHECK(ensure(ctx, ctx->slots, static_cast<size_t>(2) * G * kSlotWords * 8));
    CSK_CHECK(ensure(ctx, ctx->report, 8 * 8));
    CSK_CHECK(ensure(ctx, ctx->scalars, 8 * 8));
    CSK_CUDA(ctx, cudaMemsetAsync(ctx->slots.ptr, 0, static_cast<size_t>(2) * G * kSlotWords * 8, stream));
    double *bb = static_cast<double *>(ctx->scalars.ptr);
    if (resmode) k_sumsq<<<1, 1024, 0, stream>>>(bt, d, bb);

    SolveParams prm{};
    prm.At = At; prm.bt = bt; prm.nsq = nsq; prm.d = d; prm.n = n; prm.x = x;
    prm.x_star = x_star; prm.tol = tol; prm.max_iters = max_iters;
    prm.slots = static_cast<uint64_t *>(ctx->slots.ptr);
    prm.report = static_cast<int64_t *>(ctx->report.ptr);
    prm.bb = bb;
    prm.smem_rows_cap = static_cast<int>(srows);
    prm.trace_cap = opts ? opts->trace_cap : 0;
    prm.idx_trace = opts ? opts->idx_trace : nullptr;
    prm.res_trace = opts ? opts->res_trace : nullptr;
    prm.x_trace = opts ? opts->x_trace : nullptr;
    if (prm.trace_cap <= 0) { prm.idx_trace = nullptr; prm.res_trace = nullptr; prm.x_trace = nullptr; prm.trace_cap = 0; }

    void *args[] = {&prm};
    CSK_CUDA(ctx, cudaLaunchCooperativeKernel(reinterpret_cast<void *>(fn), dim3(G), dim3(threads), args, smem, stream));
    CSK_CHECK(ensure_host_report(ctx));
    CSK_CUDA(ctx, cudaMemcpyAsync(ctx->report_host, ctx->report.ptr, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
    ctx->pending_stream = stream;
    ctx->pending_resmode = resmode;
    ctx->pending = true;
    if (opts && (opts->flags & CSK_SOLVE_ASYNC)) return CSK_OK;
    return finish_solve(ctx, report);
}

csk_status_t ensure_host_report(csk_ctx_t ctx) {
    if (ctx->report_host) return CSK_OK;
    cudaError_t e = cudaMallocHost(&ctx->report_host, 8 * sizeof(int64_t));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMallocHost(report)");
    return CSK_OK;
}

csk_status_t finish_solve(csk_ctx_t ctx, csk_report_t *report) {
    if (!ctx->pending) return fail(ctx, CSK_E_ARG, "csk_solve_wait: no solve in flight");
    ctx->pending = false;
    CSK_CUDA(ctx, cudaStreamSynchronize(ctx->pending_stream));
    const int64_t *rep = ctx->report_host;
    if (rep[2] == -2) return fail(ctx, CSK_E_ZERO_SKETCH, "csk_solve: every row of A~ is zero");
    if (!report) return CSK_OK;
    report->iterations = rep[0];
    double fr;
    memcpy(&fr, &rep[1], sizeof(double));
    report->final_res = fr;
    report->termination = static_cast<int32_t>(rep[2]);
    report->stop_mode = ctx->pending_resmode ? CSK_STOP_RESIDUAL : CSK_STOP_RES;
    report->last_index = rep[3];
    return CSK_OK;
}

}  // namespace csk
