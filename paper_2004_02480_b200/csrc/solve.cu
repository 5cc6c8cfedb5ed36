// solve.cu -- S5..S8: the Algorithm 1 loop as ONE persistent kernel.
//
// Grid: G = CS x NC cooperative CTAs in NC thread-block clusters of CS CTAs (CS <= 16,
// one CTA per SM).  CTA c owns the contiguous rows [d c/G, d (c+1)/G) of A~; as many as
// fit stay resident in shared memory for the whole solve, the rest are re-read from
// L2/HBM every iteration.
//
// Thread layout (8 warps): warps form a Wr x Wc grid.  Column-warp cw owns the column
// pairs cw*32P + lane + 32p (p < P) and keeps those entries of x and x* in registers;
// row-team t processes the 32-row groups g = t, t + Wr, ...
//
// Every iteration k (all steps fused, no per-iteration launch):
//   S6  GEMV r = b~ - A~ x_k (P:62 numerator).  For a 32-row group each lane folds its
//       pairs into 32 row accumulators (fma, pair order), a transposed shuffle reduction
//       leaves row l's warp partial in lane l, and the Wc column-warp partials are added
//       in column order.  Fixed order => identical bits in every run.
//   S7  score_i = r_i^2 / nsq_i (squared form; masked rows -1), one division per
//       lane in parallel; argmax (ties -> lowest row index, north_star) in three hops:
//         1. CTA: warps -> shared memory;
//         2. cluster: every CTA pushes its candidate into every cluster CTA's shared
//            memory (DSMEM) and reduces the CS slots locally (same order everywhere);
//         3. grid (NC > 1): the cluster leaders push the cluster candidate into each
//            leader's global inbox, poll their own inbox, and push the winner back to
//            their members over DSMEM.
//       Every slot is eight 64-bit words carrying the iteration tag in their low half
//       (8-byte stores are single-copy atomic, so a reader that sees the tag in all
//       words has a consistent slot); slots are double-buffered by iteration parity.
//   S8  lambda = r_ik / nsq_ik (computed by the owning CTA); every CTA applies
//       x += lambda * A~^(ik) with the same fma in the same order, so all copies of x
//       stay bit-identical and every CTA takes the same stop decision locally.
//   S5  RES_k = ||x_k - x*||^2/||x*||^2 from register partials, or in residual
//       mode ||r||^2/||b~||^2 from the exchanged partial sums.
#include <stdlib.h>
#include <string.h>

#include "csk_internal.cuh"

namespace csk {

namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kMaxW = 16;  // max warps of any variant (sizes cand[] in the layout)
constexpr int kResW = 8;   // warps of the resident-only variant
constexpr int kMaxSlotsPerLane = 5;  // NC <= 160 cluster leaders
constexpr int kMaxNC = 32 * kMaxSlotsPerLane;
constexpr int kMaxCS = 16;
constexpr int kSlotWords = 8;        // 64-byte slot
constexpr int kMaxTab = 164;         // r0 table entries (>= max grid + 1, multiple of 4)

struct SolveParams {
    const double *At;
    const double *bt;
    const double *nsq;
    int64_t d, n;
    double *x;
    const double *x_star;
    double tol;
    int64_t max_iters;
    uint64_t *slots;        // global inboxes [2][NC readers][NC writers][8] words
    int64_t *report;        // [0]=iterations, [1]=final_res bits, [2]=termination, [3]=last idx
    const double *bb;       // residual mode: ||b~||^2 (device scalar)
    int smem_rows_cap;      // rows per CTA kept in shared memory
    int wc;                 // column warps of the streamed-row GEMV (1, 2, 4, 8)
    int wk;                 // column chunks of the resident-row GEMV
    int rows_max;           // max rows per CTA (sizes the uniform shared-memory layout)
    int cs;                 // cluster size
    int64_t trace_cap;
    int64_t *idx_trace;
    double *res_trace;
    double *x_trace;
    int64_t *phase_cycles;  // debug: per-phase clock64 totals of CTA 0, warps 0 and 1
};

struct Cand {
    double score;
    double r;
    double rr;
    int64_t idx;
};

// Exchange payload: score, lambda, sum r^2, row index.
struct Pay {
    double s, l, rr;
    int64_t i;
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

__device__ __forceinline__ void warp_argmax(double &score, int64_t &idx, double &v1) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, score, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, idx, o);
        const double o1 = __shfl_xor_sync(0xffffffffu, v1, o);
        if (better(os, oi, score, idx)) {
            score = os;
            idx = oi;
            v1 = o1;
        }
    }
}

// Warp-wide combine of one payload per lane: argmax of (s, i) carrying l; rr summed by a
// fixed butterfly (identical bits in every CTA that combines the same payloads).
__device__ __forceinline__ Pay warp_combine(Pay v, bool sum_rr) {
    warp_argmax(v.s, v.i, v.l);
    if (sum_rr) v.rr = warp_sum(v.rr);
    return v;
}

// Monotone 64-bit key of a score: finite scores >= 0 map to bits + 1 (order-preserving for
// non-negative doubles), masked (-1) / empty (-2) candidates to 0.
__device__ __forceinline__ uint64_t score_key(double s) {
    return s >= 0.0 ? static_cast<uint64_t>(__double_as_longlong(s)) + 1ull : 0ull;
}
__device__ __forceinline__ uint32_t idx32(int64_t i) {
    return i == INT64_MAX ? 0xffffffffu : static_cast<uint32_t>(i);
}
// Lane holding the (largest key, smallest index) of the warp -- the same total order as
// better() -- in three redux.sync reductions and a ballot instead of a 5-step butterfly.
__device__ __forceinline__ int warp_argmax_lane(uint64_t key, uint32_t idx) {
    const uint32_t kh = static_cast<uint32_t>(key >> 32), kl = static_cast<uint32_t>(key);
    const uint32_t hi = __reduce_max_sync(0xffffffffu, kh);
    const uint32_t lo = __reduce_max_sync(0xffffffffu, kh == hi ? kl : 0u);
    const bool top = kh == hi && kl == lo;
    const uint32_t mi = __reduce_min_sync(0xffffffffu, top ? idx : 0xffffffffu);
    return __ffs(__ballot_sync(0xffffffffu, top && idx == mi)) - 1;
}

__device__ __forceinline__ uint64_t pack(uint32_t data, uint32_t tag) {
    return (static_cast<uint64_t>(data) << 32) | tag;
}

__device__ __forceinline__ void encode(const Pay &v, uint32_t tag, uint64_t (&w)[8]) {
    const uint64_t sb = __double_as_longlong(v.s), lb = __double_as_longlong(v.l),
                   rb = __double_as_longlong(v.rr);
    w[0] = pack(static_cast<uint32_t>(sb >> 32), tag);
    w[1] = pack(static_cast<uint32_t>(sb), tag);
    w[2] = pack(static_cast<uint32_t>(lb >> 32), tag);
    w[3] = pack(static_cast<uint32_t>(lb), tag);
    w[4] = pack(static_cast<uint32_t>(rb >> 32), tag);
    w[5] = pack(static_cast<uint32_t>(rb), tag);
    w[6] = pack(static_cast<uint32_t>(v.i), tag);
    w[7] = pack(0u, tag);
}

__device__ __forceinline__ bool decode(const uint64_t (&w)[8], uint32_t tag, Pay &v) {
#pragma unroll
    for (int j = 0; j < 7; ++j)
        if (static_cast<uint32_t>(w[j]) != tag) return false;
    v.s = __longlong_as_double(static_cast<long long>((w[0] >> 32) << 32 | (w[1] >> 32)));
    v.l = __longlong_as_double(static_cast<long long>((w[2] >> 32) << 32 | (w[3] >> 32)));
    v.rr = __longlong_as_double(static_cast<long long>((w[4] >> 32) << 32 | (w[5] >> 32)));
    const uint32_t iw = static_cast<uint32_t>(w[6] >> 32);
    v.i = (iw == 0xffffffffu) ? INT64_MAX : static_cast<int64_t>(iw);
    return true;
}

__device__ __forceinline__ void st_global_slot(uint64_t *s, const uint64_t (&w)[8]) {
    st_relaxed_v2u64(s + 0, w[0], w[1]);
    st_relaxed_v2u64(s + 2, w[2], w[3]);
    st_relaxed_v2u64(s + 4, w[4], w[5]);
    st_relaxed_v2u64(s + 6, w[6], w[7]);
}
__device__ __forceinline__ void ld_global_slot(const uint64_t *s, uint64_t (&w)[8]) {
    ld_relaxed_v2u64(s + 0, w[0], w[1]);
    ld_relaxed_v2u64(s + 2, w[2], w[3]);
    ld_relaxed_v2u64(s + 4, w[4], w[5]);
    ld_relaxed_v2u64(s + 6, w[6], w[7]);
}
__device__ __forceinline__ void st_dsmem_slot(uint32_t a, const uint64_t (&w)[8]) {
    st_cluster_v2u64(a + 0, w[0], w[1]);
    st_cluster_v2u64(a + 16, w[2], w[3]);
    st_cluster_v2u64(a + 32, w[4], w[5]);
    st_cluster_v2u64(a + 48, w[6], w[7]);
}
__device__ __forceinline__ void ld_local_slot(uint32_t a, uint64_t (&w)[8]) {
    ld_cluster_local_v2u64(a + 0, w[0], w[1]);
    ld_cluster_local_v2u64(a + 16, w[2], w[3]);
    ld_cluster_local_v2u64(a + 32, w[4], w[5]);
    ld_cluster_local_v2u64(a + 48, w[6], w[7]);
}

template <bool EVEN>
__device__ __forceinline__ double2 load_pair_global(const double *row, int64_t q, int64_t n) {
    if (EVEN) return ldg_stream2(row + 2 * q);
    double2 v;
    v.x = ldg_stream1(row + 2 * q);
    v.y = (2 * q + 1 < n) ? ldg_stream1(row + 2 * q + 1) : 0.0;
    return v;
}

// 32 row partials per lane -> lane l holds the sum over lanes of row l (fixed tree).
__device__ __forceinline__ double transpose_reduce32(double (&v)[32], int lane) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int j = 0; j < o; ++j) {
            const double send = upper ? v[j] : v[j + o];
            const double keep = upper ? v[j + o] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0];
}

// Owner CTA of global row i under the contiguous split r0(c) = floor(d c / G).
__device__ __forceinline__ int owner_cta(int64_t i, int64_t d, int G) {
    int c = static_cast<int>((i * G) / d);
    while (c + 1 < G && (d * (c + 1)) / G <= i) ++c;
    while (c > 0 && (d * c) / G > i) --c;
    return c;
}

template <int P, bool EVEN, bool RESMODE, bool STREAM, int W>
__global__ void __launch_bounds__(W * 32, 1) k_solve(const SolveParams p) {
    constexpr int kT = W * 32;
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, cta = blockIdx.x;
    const int CS = p.cs, NC = G / CS;
    const int rank = static_cast<int>(CS > 1 ? cluster_ctarank() : 0u);
    const int clus = cta / CS;
    const int64_t d = p.d, n = p.n;
    const int64_t npairs = (n + 1) >> 1;
    const int64_t r0 = d * cta / G, r1 = d * (cta + 1) / G;
    const int rows = static_cast<int>(r1 - r0);
    const int srows = rows < p.smem_rows_cap ? rows : p.smem_rows_cap;
    // resident rows: lane-per-row GEMV over Wk column chunks (x broadcast from smem)
    const int gs = (srows + 31) >> 5;
    const int Wk = p.wk;
    const int64_t chunk = (npairs + Wk - 1) / Wk;
    const int64_t sstride = npairs | 1;  // odd 16-byte stride: lanes (= rows) hit distinct banks
    // streamed rows: column-lane GEMV (coalesced) + transposed shuffle reduction
    const int nst = rows - srows;
    const int gt = (nst + 31) >> 5;
    const int Wc = p.wc, Wr = W / Wc;
    const int cw = warp % Wc, team = warp / Wc;
    const int64_t xpad = (npairs > static_cast<int64_t>(Wc) * 32 * P) ? npairs : static_cast<int64_t>(Wc) * 32 * P;
    const double gd = static_cast<double>(G) / static_cast<double>(d);

    // ---- shared-memory carve-up: identical in every CTA (sized by rows_max), because
    //      peers address each other's resident rows over DSMEM ----
    const int rows_u = p.rows_max;
    const int srows_u = rows_u < p.smem_rows_cap ? rows_u : p.smem_rows_cap;
    const int gs_u = (srows_u + 31) >> 5, gt_u = (rows_u - srows_u + 31) >> 5;
    uint64_t *l1 = reinterpret_cast<uint64_t *>(smem);                 // [2][16][8] cluster slots
    uint64_t *rs = l1 + 2 * kMaxCS * kSlotWords;                        // [2][8] winner slot
    double2 *xsm = reinterpret_cast<double2 *>(rs + 2 * kSlotWords);   // x   [xpad] pairs
    double2 *xst = xsm + xpad;                                          // x*  [xpad] pairs
    double *part_r = reinterpret_cast<double *>(xst + xpad);           // [gs][Wk][32]
    double *part_s = part_r + static_cast<size_t>(gs_u) * Wk * 32;     // [gt][Wc][32]
    double *bt_loc = part_s + static_cast<size_t>(gt_u) * Wc * 32;     // [rows]
    double *nsq_loc = bt_loc + rows_u;                                 // [rows]
    Cand *cand = reinterpret_cast<Cand *>(nsq_loc + rows_u);            // [8] (16-byte aligned)
    volatile int64_t *win = reinterpret_cast<volatile int64_t *>(cand + W);  // [8]
    double *resp = reinterpret_cast<double *>(cand + W) + 8;      // [32] RES lane partials
    double *xs_nrm_s = resp + 32;                                      // [2]
    int32_t *r0tab = reinterpret_cast<int32_t *>(xs_nrm_s + 2);       // [G+1] first row of each CTA
    double2 *arows = reinterpret_cast<double2 *>(r0tab + kMaxTab);     // [srows][sstride]

    // ---- prologue ----
    if (tid == 0) {  // the carve-up must fit the launch's dynamic shared memory
        uint32_t dyn;
        asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
        const size_t need = reinterpret_cast<unsigned char *>(arows + static_cast<int64_t>(srows_u) * sstride) - smem;
        if (need > dyn) __trap();
    }
    for (int e = tid; e < 2 * kMaxCS * kSlotWords + 2 * kSlotWords; e += kT) l1[e] = 0;
    for (int c = tid; c <= G; c += kT) r0tab[c] = static_cast<int32_t>(d * c / G);
    for (int64_t e = tid; e < static_cast<int64_t>(srows) * npairs; e += kT) {
        const int64_t l = e / npairs, q = e - l * npairs;
        const double *src = p.At + (r0 + l) * n;
        double2 v;
        if (EVEN) {
            v = *reinterpret_cast<const double2 *>(src + 2 * q);
        } else {
            v.x = src[2 * q];
            v.y = (2 * q + 1 < n) ? src[2 * q + 1] : 0.0;
        }
        arows[l * sstride + q] = v;
    }
    for (int l = tid; l < rows; l += kT) {
        bt_loc[l] = p.bt[r0 + l];
        nsq_loc[l] = p.nsq[r0 + l];
    }
    for (int64_t q = tid; q < xpad; q += kT) {
        double2 v = make_double2(0.0, 0.0), w = make_double2(0.0, 0.0);
        if (q < npairs) {
            v.x = p.x[2 * q];
            if (2 * q + 1 < n) v.y = p.x[2 * q + 1];
            if (!RESMODE) {
                w.x = p.x_star[2 * q];
                if (2 * q + 1 < n) w.y = p.x_star[2 * q + 1];
            }
        }
        xsm[q] = v;
        xst[q] = w;
    }
    __syncthreads();
    // ||x*||^2 and RES_0 (warp 0; lane-strided pairs, butterfly)
    double xs_nrm = 0.0, res = 0.0;
    int64_t k = 0, last = -1;
    int term = -1;
    if (warp == 0) {
        int stop = -1;
        if (!RESMODE) {
            double a = 0.0, e2 = 0.0;
            for (int64_t q = lane; q < npairs; q += 32) {
                const double2 s = xst[q], x = xsm[q];
                a = __fma_rn(s.x, s.x, a);
                a = __fma_rn(s.y, s.y, a);
                const double ex = x.x - s.x, ey = x.y - s.y;
                e2 = __fma_rn(ex, ex, e2);
                e2 = __fma_rn(ey, ey, e2);
            }
            xs_nrm = warp_sum(a);
            e2 = warp_sum(e2);
            res = xs_nrm > 0.0 ? e2 / xs_nrm : e2;
            if (cta == 0 && lane == 0 && p.res_trace && p.trace_cap > 0) p.res_trace[0] = res;
            if (res <= p.tol) stop = CSK_CONVERGED;
            else if (p.max_iters == 0) stop = CSK_MAX_ITERS;
        }
        if (lane == 0) {
            win[0] = -1;
            win[2] = stop;
            win[3] = __double_as_longlong(res);
            win[4] = 0;
            win[5] = -1;
            xs_nrm_s[0] = xs_nrm;
        }
    }
    const double bb = RESMODE ? *p.bb : 0.0;
    if (CS > 1) cluster_sync_all();  // every CTA's slots are zeroed before any remote write
    else __syncthreads();

#if CSK_PHASE_PROF
    // debug build only (libcsk_prof.so): per-phase SM-cycle totals of CTA 0, warps 0 and 1
    const bool prof = p.phase_cycles != nullptr && cta == 0 && lane == 0 && warp < 2;
    int64_t ph[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long tp = clock64(), tf = tp;
#define CSK_PHASE(i)                    \
    if (prof) {                         \
        const long long tn = clock64(); \
        ph[i] += tn - tp;               \
        tp = tn;                        \
        tf = tn;                        \
    }
// fine-grained points inside warp 0's exchange (no barriers in between: exact)
#define CSK_FINE(i)                     \
    if (prof) {                         \
        const long long tn = clock64(); \
        ph[8 + (i)] += tn - tf;         \
        tf = tn;                        \
    }
#else
#define CSK_PHASE(i)
#define CSK_FINE(i)
#endif

    if (win[2] != -1) {
        term = static_cast<int>(win[2]);
        res = __longlong_as_double(win[3]);
    } else {
        for (;; ++k) {
            // trace x_k (CTA 0, warp 0)
            if (cta == 0 && warp == 0 && p.x_trace && k < p.trace_cap) {
                for (int64_t q = lane; q < npairs; q += 32) {
                    const double2 x = xsm[q];
                    p.x_trace[k * n + 2 * q] = x.x;
                    if (2 * q + 1 < n) p.x_trace[k * n + 2 * q + 1] = x.y;
                }
            }

            // ---- S5 (deferred): RES_k from warp 0's lane partials of the last update; the
            //      test result is read by warp 0 after B1 (warp 7 is off the critical path) ----
            if (!RESMODE && warp == W - 1 && k > 0) {
                const double e2 = warp_sum(resp[lane]);
                const double rk = xs_nrm_s[0] > 0.0 ? e2 / xs_nrm_s[0] : e2;
                int st = -1;
                if (rk <= p.tol) st = CSK_CONVERGED;
                else if (k == p.max_iters) st = CSK_MAX_ITERS;
                if (lane == 0) {
                    win[5] = st;
                    win[6] = __double_as_longlong(rk);
                    if (cta == 0 && p.res_trace && k < p.trace_cap) p.res_trace[k] = rk;
                }
            }

            // ---- S6a: resident rows, lane-per-row, work items (group, chunk) over warps ----
            for (int it = warp; it < gs * Wk; it += W) {
                const int g = it / Wk, kc = it - g * Wk;
                const int l = g * 32 + lane;
                const int64_t q0 = kc * chunk;
                const int64_t q1 = (q0 + chunk < npairs) ? q0 + chunk : npairs;
                double a0 = 0.0, a1 = 0.0;
                if (l < srows) {
                    const double2 *ar = arows + l * sstride;
                    int64_t q = q0;
                    for (; q + 2 <= q1; q += 2) {
                        const double2 u = ar[q], v = ar[q + 1];
                        const double2 xu = xsm[q], xv = xsm[q + 1];
                        a0 = __fma_rn(u.x, xu.x, a0);
                        a0 = __fma_rn(u.y, xu.y, a0);
                        a1 = __fma_rn(v.x, xv.x, a1);
                        a1 = __fma_rn(v.y, xv.y, a1);
                    }
                    if (q < q1) {
                        const double2 u = ar[q], xu = xsm[q];
                        a0 = __fma_rn(u.x, xu.x, a0);
                        a0 = __fma_rn(u.y, xu.y, a0);
                    }
                }
                part_r[static_cast<size_t>(it) * 32 + lane] = a0 + a1;
            }
            // ---- S6b: streamed rows (L2/HBM), column-lane mapping ----
            if constexpr (STREAM) for (int g = team; g < gt; g += Wr) {
                double2 xr[P];
#pragma unroll
                for (int j = 0; j < P; ++j) xr[j] = xsm[static_cast<int64_t>(cw) * 32 * P + lane + 32 * j];
                double acc[32];
#pragma unroll
                for (int r = 0; r < 32; ++r) acc[r] = 0.0;
                const int lb = srows + g * 32;
                const bool full = lb + 32 <= rows;
                const double *gbase = p.At + (r0 + lb) * n;
#pragma unroll
                for (int j = 0; j < P; ++j) {
                    const int64_t q = static_cast<int64_t>(cw) * 32 * P + lane + 32 * j;
                    if (q < npairs) {
                        if (full) {
#pragma unroll
                            for (int r = 0; r < 32; ++r) {
                                const double2 a = load_pair_global<EVEN>(gbase + static_cast<int64_t>(r) * n, q, n);
                                acc[r] = __fma_rn(a.x, xr[j].x, acc[r]);
                                acc[r] = __fma_rn(a.y, xr[j].y, acc[r]);
                            }
                        } else {
#pragma unroll
                            for (int r = 0; r < 32; ++r) {
                                if (lb + r < rows) {
                                    const double2 a = load_pair_global<EVEN>(gbase + static_cast<int64_t>(r) * n, q, n);
                                    acc[r] = __fma_rn(a.x, xr[j].x, acc[r]);
                                    acc[r] = __fma_rn(a.y, xr[j].y, acc[r]);
                                }
                            }
                        }
                    }
                }
                const double sum = transpose_reduce32(acc, lane);
                part_s[(static_cast<size_t>(g) * Wc + cw) * 32 + lane] = sum;
            }
            CSK_PHASE(0)
            __syncthreads();  // B1
            CSK_PHASE(1)

            // ---- S7 local: finalize rows (score and lambda per row), argmax ----
            // small CTAs (<= 64 rows): warp 0 alone, no second barrier; else all warps
            const bool small = rows_u <= 64;
            if (!small || warp == 0) {
                double bs = -2.0, bl = 0.0, rr = 0.0;
                int64_t bi = INT64_MAX;
                const int step = small ? 32 : kT;
                for (int l = small ? lane : tid; l - lane < rows; l += step) {
                    if (l < rows) {
                        double dot;
                        if (l < srows) {
                            const double *pp = part_r + (static_cast<size_t>(l >> 5) * Wk) * 32 + (l & 31);
                            dot = pp[0];
                            for (int c = 1; c < Wk; ++c) dot = dot + pp[c * 32];
                        } else {
                            const int ls = l - srows;
                            const double *pp = part_s + (static_cast<size_t>(ls >> 5) * Wc) * 32 + (ls & 31);
                            dot = pp[0];
                            for (int c = 1; c < Wc; ++c) dot = dot + pp[c * 32];
                        }
                        const double ri = bt_loc[l] - dot;
                        const double ns = nsq_loc[l];
                        const double sc = ns > 0.0 ? (ri * ri) / ns : -1.0;
                        const double lam = ns > 0.0 ? ri / ns : 0.0;
                        if (RESMODE) rr = __fma_rn(ri, ri, rr);
                        if (better(sc, r0 + l, bs, bi)) { bs = sc; bi = r0 + l; bl = lam; }
                    }
                }
                if (RESMODE) rr = warp_sum(rr);
                {
                    const int wl = warp_argmax_lane(score_key(bs), idx32(bi));
                    bs = __shfl_sync(0xffffffffu, bs, wl);
                    bi = __shfl_sync(0xffffffffu, bi, wl);
                    bl = __shfl_sync(0xffffffffu, bl, wl);
                }
                if (lane == 0) cand[warp] = Cand{bs, bl, rr, bi};
            }
            if (!small) __syncthreads();  // B1b
            CSK_PHASE(2)

            // ---- S7 exchange, S8 update (warp 0) ----
            if (warp == 0) {
                int stop = -1, applied = 0;
                if (!RESMODE) stop = static_cast<int>(win[5]);  // RES_k test made by warp 7
                Pay wv{-2.0, 0.0, 0.0, INT64_MAX};
                if (stop < 0) {
                // hop 1: CTA candidate (8 warp candidates, xor 4,2,1 then broadcast lane 0)
                Pay cv{-2.0, 0.0, 0.0, INT64_MAX};
                if (small) {
                    __syncwarp();
                    cv.s = cand[0].score; cv.l = cand[0].r; cv.i = cand[0].idx;
                    if (RESMODE) cv.rr = cand[0].rr;
                } else {
                    if (lane < W) { cv.s = cand[lane].score; cv.l = cand[lane].r; cv.i = cand[lane].idx; }
                    const int wl = warp_argmax_lane(score_key(cv.s), idx32(cv.i));
                    cv.s = __shfl_sync(0xffffffffu, cv.s, wl);
                    cv.i = __shfl_sync(0xffffffffu, cv.i, wl);
                    cv.l = __shfl_sync(0xffffffffu, cv.l, wl);
                    if (RESMODE) {
                        for (int w = 0; w < W; ++w) cv.rr = cv.rr + cand[w].rr;  // fixed order
                    }
                }
                const uint32_t tag = static_cast<uint32_t>(k + 1);
                const int par = static_cast<int>(k & 1);
                uint64_t w[8];
                CSK_FINE(0)
                // hop 2: cluster all-to-all over DSMEM (lane r -> rank r), combine 16 lanes
                Pay cl = cv;
                if (CS > 1) {
                    encode(cv, tag, w);
                    const uint32_t my_slot = smem_u32(l1 + (par * kMaxCS + rank) * kSlotWords);
                    if (lane < CS) st_dsmem_slot(mapa_shared(my_slot, static_cast<uint32_t>(lane)), w);
                    CSK_FINE(1)
                    Pay got{-2.0, 0.0, 0.0, INT64_MAX};
                    bool ok = lane >= CS;
                    const uint32_t rd = smem_u32(l1 + (par * kMaxCS + (lane < CS ? lane : 0)) * kSlotWords);
                    while (!__all_sync(0xffffffffu, ok)) {
                        if (!ok) {
                            uint64_t r8[8];
                            ld_local_slot(rd, r8);
                            ok = decode(r8, tag, got);
                        }
                    }
                    CSK_FINE(2)
                    if (RESMODE) {
#pragma unroll
                        for (int o = 8; o > 0; o >>= 1) got.rr = got.rr + __shfl_xor_sync(0xffffffffu, got.rr, o);
                    }
                    const int wl = warp_argmax_lane(score_key(got.s), idx32(got.i));
                    cl.s = __shfl_sync(0xffffffffu, got.s, wl);
                    cl.i = __shfl_sync(0xffffffffu, got.i, wl);
                    cl.l = __shfl_sync(0xffffffffu, got.l, wl);
                    cl.rr = __shfl_sync(0xffffffffu, got.rr, 0);
                }
                CSK_PHASE(3)
                // hop 3: grid exchange among the NC cluster leaders (global inboxes)
                wv = cl;
                if (NC > 1) {
                    if (rank == 0) {
                        encode(cl, tag, w);
                        uint64_t *gpar = p.slots + static_cast<size_t>(par) * NC * NC * kSlotWords;
#pragma unroll
                        for (int j = 0; j < kMaxSlotsPerLane; ++j) {
                            const int rdr = lane + 32 * j;
                            if (rdr < NC) st_global_slot(gpar + (static_cast<size_t>(rdr) * NC + clus) * kSlotWords, w);
                        }
                        CSK_FINE(3)
                        const uint64_t *inbox = gpar + static_cast<size_t>(clus) * NC * kSlotWords;
                        Pay g[kMaxSlotsPerLane];
                        uint32_t pending = 0;
#pragma unroll
                        for (int j = 0; j < kMaxSlotsPerLane; ++j) {
                            g[j] = Pay{-2.0, 0.0, 0.0, INT64_MAX};
                            if (lane + 32 * j < NC) pending |= 1u << j;
                        }
                        while (true) {
#pragma unroll
                            for (int j = 0; j < kMaxSlotsPerLane; ++j) {
                                if (pending & (1u << j)) {
                                    uint64_t r8[8];
                                    ld_global_slot(inbox + static_cast<size_t>(lane + 32 * j) * kSlotWords, r8);
                                    if (decode(r8, tag, g[j])) pending &= ~(1u << j);
                                }
                            }
                            if (__all_sync(0xffffffffu, pending == 0)) break;
                        }
                        CSK_FINE(4)
                        Pay acc{-2.0, 0.0, 0.0, INT64_MAX};
#pragma unroll
                        for (int j = 0; j < kMaxSlotsPerLane; ++j) {
                            if (better(g[j].s, g[j].i, acc.s, acc.i)) { acc.s = g[j].s; acc.i = g[j].i; acc.l = g[j].l; }
                            if (RESMODE) acc.rr = acc.rr + g[j].rr;
                        }
                        if (RESMODE) acc.rr = warp_sum(acc.rr);
                        {
                            const int wl = warp_argmax_lane(score_key(acc.s), idx32(acc.i));
                            wv.s = __shfl_sync(0xffffffffu, acc.s, wl);
                            wv.i = __shfl_sync(0xffffffffu, acc.i, wl);
                            wv.l = __shfl_sync(0xffffffffu, acc.l, wl);
                            wv.rr = acc.rr;
                        }
                        if (CS > 1) {
                            encode(wv, tag, w);
                            const uint32_t rslot = smem_u32(rs + par * kSlotWords);
                            if (lane < CS && lane != 0) st_dsmem_slot(mapa_shared(rslot, static_cast<uint32_t>(lane)), w);
                        }
                    } else {
                        const uint32_t rslot = smem_u32(rs + par * kSlotWords);
                        bool ok = false;
                        Pay got{-2.0, 0.0, 0.0, INT64_MAX};
                        while (!ok) {
                            uint64_t r8[8];
                            ld_local_slot(rslot, r8);
                            ok = decode(r8, tag, got);
                        }
                        wv = got;
                        CSK_FINE(5)
                    }
                }
                CSK_PHASE(4)
                if (RESMODE) {
                    res = bb > 0.0 ? wv.rr / bb : wv.rr;
                    if (cta == 0 && lane == 0 && p.res_trace && k < p.trace_cap) p.res_trace[k] = res;
                    if (res <= p.tol) stop = CSK_CONVERGED;
                    else if (k == p.max_iters) stop = CSK_MAX_ITERS;
                }
                if (stop < 0) {
                    if (wv.s < 0.0) stop = -2;                 // every row masked: zero sketch
                    else if (wv.s == 0.0) stop = CSK_STAGNATED;
                }
                if (stop < 0) {
                    if (cta == 0 && lane == 0 && p.idx_trace && k < p.trace_cap) p.idx_trace[k] = wv.i;
                    // fetch A~^(ik): from the owner's shared memory over DSMEM when it is a
                    // resident row of this cluster, else from L2/HBM; then x += lambda row
                    int co = static_cast<int>(static_cast<double>(wv.i) * gd);
                    if (co > G - 1) co = G - 1;
                    while (co + 1 < G && r0tab[co + 1] <= wv.i) ++co;
                    while (co > 0 && r0tab[co] > wv.i) --co;
                    const int64_t o0 = r0tab[co], o1 = r0tab[co + 1];
                    const int64_t lo = wv.i - o0;
                    const int64_t ocap = (o1 - o0) < p.smem_rows_cap ? (o1 - o0) : p.smem_rows_cap;
                    const bool dsm = CS > 1 && co / CS == clus && lo < ocap;
                    uint32_t rbase = 0;
                    if (dsm) rbase = mapa_shared(smem_u32(arows + lo * sstride), static_cast<uint32_t>(co % CS));
                    const double *gsrc = p.At + wv.i * n;
                    // loads in blocks of 8 independent pairs per lane (one round trip each), then the update
                    double e2 = 0.0;
                    CSK_FINE(6)
                    for (int64_t qb = 0; qb < npairs; qb += 8 * 32) {
                        double2 av[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const int64_t q = qb + lane + 32 * j;
                            if (q < npairs) av[j] = dsm ? ld_dsmem_v2f64_nc(rbase + static_cast<uint32_t>(q * 16))
                                                        : load_pair_global<EVEN>(gsrc, q, n);
                        }
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const int64_t q = qb + lane + 32 * j;
                            if (q < npairs) {
                                double2 x = xsm[q];
                                x.x = __fma_rn(wv.l, av[j].x, x.x);
                                x.y = __fma_rn(wv.l, av[j].y, x.y);
                                xsm[q] = x;
                                if (!RESMODE) {
                                    const double2 s = xst[q];
                                    const double ex = x.x - s.x, ey = x.y - s.y;
                                    e2 = __fma_rn(ex, ex, e2);
                                    e2 = __fma_rn(ey, ey, e2);
                                }
                            }
                        }
                    }
                    CSK_FINE(7)
                    applied = 1;
                    last = wv.i;
                    if (!RESMODE) resp[lane] = e2;  // reduced by warp 7 next iteration (S5)
                }
                }  // stop < 0 (RES_k test)
                if (!RESMODE && stop >= 0 && !applied) res = __longlong_as_double(win[6]);
                __syncwarp();
                if (lane == 0) {
                    win[0] = last;
                    win[2] = stop;
                    win[3] = __double_as_longlong(res);
                    win[4] = applied;
                }
                CSK_PHASE(5)
            }
            __syncthreads();  // B2
            CSK_PHASE(6)
            const int stop = static_cast<int>(win[2]);
            if (stop != -1) {
                term = stop;
                res = __longlong_as_double(win[3]);
                last = win[0];
                if (win[4]) ++k;
                break;
            }
        }
    }
#undef CSK_PHASE
#undef CSK_FINE
#if CSK_PHASE_PROF
    if (prof) {
        for (int i = 0; i < 16; ++i) p.phase_cycles[warp * 16 + i] = ph[i];
    }
#endif

    // ---- epilogue: CTA 0 writes x (and the trace of the final iterate); thread 0 the report ----
    if (cta == 0) {
        const bool tr = p.x_trace && k < p.trace_cap;
        for (int64_t q = tid; q < npairs; q += kT) {
            const double2 x = xsm[q];
            p.x[2 * q] = x.x;
            if (2 * q + 1 < n) p.x[2 * q + 1] = x.y;
            if (tr) {
                p.x_trace[k * n + 2 * q] = x.x;
                if (2 * q + 1 < n) p.x_trace[k * n + 2 * q + 1] = x.y;
            }
        }
        if (tid == 0) {
            p.report[0] = k;
            p.report[1] = __double_as_longlong(res);
            p.report[2] = term;
            p.report[3] = last;
        }
    }
    // no CTA may leave while a cluster peer could still address its shared memory
    if (CS > 1) cluster_sync_all();
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

// STREAM = some rows are re-read from L2/HBM (8 warps, the column-lane GEMV compiled in);
// otherwise every row is resident and the lighter kernel runs 16 warps for latency hiding.
template <int P>
KernelFn pick_mode(bool even, bool resmode, bool stream) {
    if (stream) {
        if (even) return resmode ? k_solve<P, true, true, true, 8> : k_solve<P, true, false, true, 8>;
        return resmode ? k_solve<P, false, true, true, 8> : k_solve<P, false, false, true, 8>;
    }
    if (even) return resmode ? k_solve<P, true, true, false, kResW> : k_solve<P, true, false, false, kResW>;
    return resmode ? k_solve<P, false, true, false, kResW> : k_solve<P, false, false, false, kResW>;
}

// P = column pairs per lane (power of two), Wc = column warps (power of two <= 8) of the
// streamed-row GEMV.
KernelFn pick_kernel(int64_t n, bool resmode, bool stream, int &P, int &wc) {
    const int64_t npairs = (n + 1) / 2;
    P = 1;
    while (32 * kWarps * P < npairs) P *= 2;
    wc = 1;
    while (wc < kWarps && 32 * P * wc < npairs) wc *= 2;
    const bool even = (n & 1) == 0;
    switch (P) {
        case 1: return pick_mode<1>(even, resmode, stream);
        case 2: return pick_mode<2>(even, resmode, stream);
        case 4: return pick_mode<4>(even, resmode, stream);
        default: return nullptr;
    }
}

// Bytes of the kernel's shared-memory carve-up for a given split (mirrors k_solve).
size_t smem_layout(int64_t rows_max, int64_t srows, int64_t npairs, int64_t wc, int64_t P, int64_t wk) {
    const int64_t xpad = npairs > wc * 32 * P ? npairs : wc * 32 * P;
    const int64_t gs = (srows + 31) / 32, gt = (rows_max - srows + 31) / 32;
    return static_cast<size_t>(2 * kMaxCS * kSlotWords + 2 * kSlotWords) * 8 +  // slots
           static_cast<size_t>(2 * xpad) * 16 +                                // x, x*
           static_cast<size_t>(gs * wk + gt * wc) * 32 * 8 +                   // partials
           static_cast<size_t>(rows_max) * 16 + kMaxW * sizeof(Cand) +         // b~, nsq, cand
           8 * 8 + 32 * 8 + 2 * 8 + kMaxTab * 4 +                              // win, resp, xs_nrm, r0tab
           static_cast<size_t>(srows) * (npairs | 1) * 16 + 64;                // resident rows
}

// Column chunks for the resident-row GEMV: enough (group, chunk) items to occupy the 8
// warps, chunks of at least 8 pairs.
int pick_wk(int64_t rows_res, int64_t npairs, int warps = kMaxW);
// Largest number of resident rows whose layout fits `cap` bytes.
int64_t fit_srows(int64_t rows_max, int64_t npairs, int64_t wc, int64_t P, size_t cap) {
    int64_t lo = 0, hi = rows_max;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) / 2;
        if (smem_layout(rows_max, mid, npairs, wc, P, pick_wk(mid, npairs, kMaxW)) <= cap) lo = mid; else hi = mid - 1;
    }
    return lo;
}

int pick_wk(int64_t rows_res, int64_t npairs, int warps) {
    const int64_t groups = (rows_res + 31) / 32;
    int wk = 1;
    while (wk < warps && groups * wk < warps && npairs / (2 * wk) >= 8) wk *= 2;
    return wk;
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
    if (ctx->pending) return fail(ctx, CSK_E_ARG, "csk_solve: a CSK_SOLVE_ASYNC solve is still in flight (call csk_solve_wait)");
    if (!(opts && (opts->flags & CSK_SOLVE_LEGACY)))
        return run_loop(ctx, At, bt, nsq, d, n, x, x_star, tol, max_iters, opts, report, stream);
    const bool resmode = (x_star == nullptr);
    int P = 0, wc = 0;
    KernelFn fn = pick_kernel(n, resmode, true, P, wc);  // geometry probe (8-warp variant)
    if (!fn) return fail(ctx, CSK_E_UNSUPPORTED, "csk_solve: n out of range");
    const int64_t npairs = (n + 1) / 2;
    CSK_CHECK(raise_smem(ctx, reinterpret_cast<const void *>(fn)));

    // ---- launch geometry: cluster size CS, number of clusters NC ----
    int CS = opts && opts->cluster_size > 0 ? opts->cluster_size : 0;
    if (CS > kMaxCS || (CS & (CS - 1)) != 0) return fail(ctx, CSK_E_ARG, "csk_solve: cluster_size must be a power of two <= 16");
    int G = opts && opts->num_ctas > 0 ? opts->num_ctas : 0;
    auto smem_for = [&](int g, bool all_rows) -> size_t {
        const int64_t rows_max = (d + g - 1) / g;
        if (all_rows) return smem_layout(rows_max, rows_max, npairs, wc, P, pick_wk(rows_max, npairs));
        return static_cast<size_t>(ctx->max_smem_optin);
    };
    auto max_clusters = [&](int cs, size_t smem, int &out) -> csk_status_t {
        return max_resident(ctx, reinterpret_cast<const void *>(fn), cs, kThreads, smem, &out);
    };
    if (CS == 0) {
        // auto: the smallest number of 16-CTA clusters that keeps all of A~ on chip; if none
        // does, the largest co-resident grid of 16-CTA clusters (rows streamed from L2/HBM)
        CS = 16;
        int mc = 0;
        CSK_CHECK(max_clusters(16, static_cast<size_t>(ctx->max_smem_optin), mc));
        if (mc < 1) { CS = 1; }
        if (G == 0) {
            if (CS == 16) {
                int nc = 1;
                while (nc < mc && smem_for(nc * 16, true) > static_cast<size_t>(ctx->max_smem_optin)) ++nc;
                G = nc * 16;
            } else {
                G = ctx->num_sms;
            }
        }
    }
    if (G == 0) G = ctx->num_sms;
    if (G > d) G = static_cast<int>(d);
    if (G > kMaxTab - 1) G = kMaxTab - 1;
    if (CS > G) CS = 1;
    G = (G / CS) * CS;
    const int NC = G / CS;
    if (NC > kMaxNC) return fail(ctx, CSK_E_UNSUPPORTED, "csk_solve: too many clusters");

    const int64_t rows_max = (d + G - 1) / G;
    int64_t srows = fit_srows(rows_max, npairs, wc, P, static_cast<size_t>(ctx->max_smem_optin));
    if (opts && opts->smem_rows > 0 && opts->smem_rows < srows) srows = opts->smem_rows;
    if (opts && opts->smem_rows < 0) srows = 0;
    const bool streamed = srows < rows_max;
    const int W = streamed ? kWarps : kResW;
    fn = pick_kernel(n, resmode, streamed, P, wc);
    const int wk = pick_wk(srows, npairs, W);
    const size_t smem = smem_layout(rows_max, srows, npairs, wc, P, wk);
    if (smem > static_cast<size_t>(ctx->max_smem_optin))
        return fail(ctx, CSK_E_UNSUPPORTED, "csk_solve: too many rows per CTA for shared memory (use more CTAs)");

    int per = 0;
    CSK_CHECK(max_resident(ctx, reinterpret_cast<const void *>(fn), CS, W * 32, smem, &per));
    if (per < (CS > 1 ? NC : G)) return fail(ctx, CSK_E_UNSUPPORTED, "csk_solve: grid cannot be co-resident");

    const size_t slot_bytes = static_cast<size_t>(2) * NC * NC * kSlotWords * 8;
    CSK_CHECK(ensure(ctx, ctx->slots, slot_bytes));
    CSK_CHECK(ensure(ctx, ctx->report, 8 * 8));
    CSK_CHECK(ensure(ctx, ctx->scalars, 8 * 8));
    CSK_CUDA(ctx, cudaMemsetAsync(ctx->slots.ptr, 0, slot_bytes, stream));
    double *bb = static_cast<double *>(ctx->scalars.ptr);
    if (resmode) k_sumsq<<<1, 1024, 0, stream>>>(bt, d, bb);

    SolveParams prm{};
    prm.At = At; prm.bt = bt; prm.nsq = nsq; prm.d = d; prm.n = n; prm.x = x;
    prm.x_star = x_star; prm.tol = tol; prm.max_iters = max_iters;
    prm.slots = static_cast<uint64_t *>(ctx->slots.ptr);
    prm.report = static_cast<int64_t *>(ctx->report.ptr);
    prm.bb = bb;
    prm.smem_rows_cap = static_cast<int>(srows);
    prm.wc = wc;
    prm.wk = wk;
    prm.rows_max = static_cast<int>(rows_max);
    prm.cs = CS;
    prm.trace_cap = opts ? opts->trace_cap : 0;
    prm.idx_trace = opts ? opts->idx_trace : nullptr;
    prm.res_trace = opts ? opts->res_trace : nullptr;
    prm.x_trace = opts ? opts->x_trace : nullptr;
    prm.phase_cycles = opts ? opts->phase_cycles : nullptr;
    if (prm.trace_cap <= 0) { prm.idx_trace = nullptr; prm.res_trace = nullptr; prm.x_trace = nullptr; prm.trace_cap = 0; }

    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = CS;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(W * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cfg.attrs = at;
    cfg.numAttrs = CS > 1 ? 2 : 1;
    // Profiling only: ncu cannot launch cooperative + cluster kernels, so CSK_PROFILE_NONCOOP=1
    // launches the same kernel and geometry without the cooperative attribute (residency is
    // still checked above against the occupancy API; the GPU must be otherwise idle).
    static const bool noncoop = getenv("CSK_PROFILE_NONCOOP") != nullptr;
    if (noncoop) { cfg.attrs = at + 1; cfg.numAttrs = CS > 1 ? 1 : 0; }
    CSK_CUDA(ctx, cudaLaunchKernelEx(&cfg, fn, prm));
    ctx->last_solve_geom[0] = G;
    ctx->last_solve_geom[1] = CS;
    ctx->last_solve_geom[2] = static_cast<int>(srows);
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
    if (rep[2] == -3)
        return fail(ctx, CSK_E_CUDA, "csk_solve: exchange watchdog -- not every CTA / rank arrived within "
                                     "CSK_EXCHANGE_TIMEOUT_S (default 30 s)");
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
