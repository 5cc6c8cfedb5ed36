// solve.cu -- S5..S8: the Algorithm 1 loop as ONE persistent kernel.
//
// Grid: G cooperative CTAs (<= 1 per SM), CTA c owns the contiguous rows
// [d c/G, d (c+1)/G) of A~; as many of them as fit stay resident in shared memory for
// the whole solve, the rest are re-read from L2/HBM every iteration.
//
// Thread layout (8 warps): warps form a Wr x Wc grid.  Column-warp cw owns the column
// pairs cw*32P + lane + 32p (p < P), and keeps those entries of x and x* in registers;
// row-team t processes the 32-row groups g = t, t + Wr, ...
//
// Every iteration k (all steps fused, no per-iteration launch):
//   S6  GEMV r = b~ - A~ x_k (P:62 numerator).  For a 32-row group each lane folds its
//       pairs into 32 row accumulators (fma, pair order), a transposed shuffle reduction
//       leaves row l's warp partial in lane l, partials of the Wc column-warps are added
//       in column order.  Fixed order => identical bits in every run.
//   S7  score_i = r_i^2 / nsq_i (squared form; masked rows -1), one division per
//       lane in parallel; warp argmax -> CTA argmax -> grid argmax through a PUSH
//       exchange: each CTA writes (score, lambda, idx, sum r^2) into every CTA's private
//       inbox slot (eight 64-bit words, each carrying the iteration tag in its low half:
//       8-byte stores are single-copy atomic, so a reader that sees the tag in all words
//       has a consistent slot), double-buffered by iteration parity; each CTA polls only
//       its own inbox, so no L2 line is hammered by more than one reader.
//       Ties -> lowest row index (north_star).
//   S8  lambda = r_ik / nsq_ik (computed by the owning CTA); every CTA applies
//       x += lambda * A~^(ik) with the same fma in the same order, so all copies of x
//       stay bit-identical and every CTA takes the same stop decision locally.
//   S5  RES_k = ||x_k - x*||^2/||x*||^2 from register partials, or in residual
//       mode ||r||^2/||b~||^2 from the exchanged partial sums.
#include <string.h>

#include "csk_internal.cuh"

namespace csk {

namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
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
    uint64_t *slots;        // [2][G readers][G writers][8] words
    int64_t *report;        // [0]=iterations, [1]=final_res bits, [2]=termination, [3]=last idx
    const double *bb;       // residual mode: ||b~||^2 (device scalar)
    int smem_rows_cap;      // rows per CTA kept in shared memory (multiple of 32 unless all)
    int wc;                 // column warps (1, 2, 4, 8)
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

template <int P, bool EVEN, bool RESMODE>
__global__ void __launch_bounds__(kThreads, 1) k_solve(const SolveParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, cta = blockIdx.x;
    const int64_t d = p.d, n = p.n;
    const int64_t npairs = (n + 1) >> 1;
    const int64_t r0 = d * cta / G, r1 = d * (cta + 1) / G;
    const int rows = static_cast<int>(r1 - r0);
    const int srows = rows < p.smem_rows_cap ? rows : p.smem_rows_cap;
    const int ngroups = (rows + 31) >> 5;
    const int Wc = p.wc, Wr = kWarps / Wc;
    const int cw = warp % Wc, team = warp / Wc;
    const int64_t npairs_pad = static_cast<int64_t>(Wc) * 32 * P;

    // ---- shared-memory carve-up (16-byte aligned pieces) ----
    double2 *wrow = reinterpret_cast<double2 *>(smem);                 // winner row [npairs_pad]
    double *part = reinterpret_cast<double *>(wrow + npairs_pad);      // [ngroups][Wc][32]
    double *bt_loc = part + static_cast<size_t>(ngroups) * Wc * 32;    // [rows]
    double *nsq_loc = bt_loc + rows;                                   // [rows]
    double *res_w = nsq_loc + rows;                                    // [8]
    Cand *cand = reinterpret_cast<Cand *>(res_w + 8);                  // [8]
    volatile int64_t *win = reinterpret_cast<volatile int64_t *>(cand + kWarps);  // [8]
    double2 *arows = reinterpret_cast<double2 *>(cand + kWarps) + 4;   // [srows][npairs]

    // ---- prologue: stage resident rows, b~, nsq; x, x* pairs into registers ----
    for (int64_t e = tid; e < static_cast<int64_t>(srows) * npairs; e += kThreads) {
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
    for (int l = tid; l < rows; l += kThreads) {
        bt_loc[l] = p.bt[r0 + l];
        nsq_loc[l] = p.nsq[r0 + l];
    }
    double2 xr[P], xs[P];
#pragma unroll
    for (int j = 0; j < P; ++j) {
        const int64_t q = static_cast<int64_t>(cw) * 32 * P + lane + 32 * j;
        xr[j] = make_double2(0.0, 0.0);
        xs[j] = make_double2(0.0, 0.0);
        if (q < npairs) {
            xr[j].x = p.x[2 * q];
            if (2 * q + 1 < n) xr[j].y = p.x[2 * q + 1];
            if (!RESMODE) {
                xs[j].x = p.x_star[2 * q];
                if (2 * q + 1 < n) xs[j].y = p.x_star[2 * q + 1];
            }
        }
    }
    // ||x*||^2 (team 0 partials; summed in column-warp order by every thread below)
    if (!RESMODE && team == 0) {
        double a = 0.0;
#pragma unroll
        for (int j = 0; j < P; ++j) {
            a = __fma_rn(xs[j].x, xs[j].x, a);
            a = __fma_rn(xs[j].y, xs[j].y, a);
        }
        a = warp_sum(a);
        if (lane == 0) res_w[cw] = a;  // scratch before the loop
    }
    __syncthreads();
    double xs_nrm = 0.0;
    if (!RESMODE) {
        xs_nrm = res_w[0];
        for (int c = 1; c < Wc; ++c) xs_nrm = xs_nrm + res_w[c];
    }
    const double bb = RESMODE ? *p.bb : 0.0;
    __syncthreads();

    const bool prof = p.phase_cycles != nullptr && cta == 0 && lane == 0 && warp < 2;
    int64_t ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tp = clock64();
#define CSK_PHASE(i)                    \
    if (prof) {                         \
        const long long tn = clock64(); \
        ph[i] += tn - tp;               \
        tp = tn;                        \
    }

    int64_t k = 0, last = -1;
    int term = -1;
    double res = 0.0;
    for (;; ++k) {
        // ---- S5 partial: ||x_k - x*||^2 over team 0's pairs; trace x_k ----
        if (team == 0) {
            if (!RESMODE) {
                double a = 0.0;
#pragma unroll
                for (int j = 0; j < P; ++j) {
                    const double ex = xr[j].x - xs[j].x, ey = xr[j].y - xs[j].y;
                    a = __fma_rn(ex, ex, a);
                    a = __fma_rn(ey, ey, a);
                }
                a = warp_sum(a);
                if (lane == 0) res_w[cw] = a;
            }
            if (cta == 0 && p.x_trace && k < p.trace_cap) {
#pragma unroll
                for (int j = 0; j < P; ++j) {
                    const int64_t q = static_cast<int64_t>(cw) * 32 * P + lane + 32 * j;
                    if (q < npairs) {
                        p.x_trace[k * n + 2 * q] = xr[j].x;
                        if (2 * q + 1 < n) p.x_trace[k * n + 2 * q + 1] = xr[j].y;
                    }
                }
            }
        }

        // ---- S6: GEMV partials for this team's 32-row groups ----
        for (int g = team; g < ngroups; g += Wr) {
            double acc[32];
#pragma unroll
            for (int r = 0; r < 32; ++r) acc[r] = 0.0;
            const int lbase = g * 32;
            const bool in_smem = lbase + 32 <= srows || (srows == rows);
            const bool full = lbase + 32 <= rows;
#pragma unroll
            for (int j = 0; j < P; ++j) {
                const int64_t q = static_cast<int64_t>(cw) * 32 * P + lane + 32 * j;
                if (q < npairs) {
                    if (in_smem) {
                        const double2 *src = arows + static_cast<int64_t>(lbase) * npairs + q;
                        if (full) {
#pragma unroll
                            for (int r = 0; r < 32; ++r) {
                                const double2 a = src[static_cast<int64_t>(r) * npairs];
                                acc[r] = __fma_rn(a.x, xr[j].x, acc[r]);
                                acc[r] = __fma_rn(a.y, xr[j].y, acc[r]);
                            }
                        } else {
#pragma unroll
                            for (int r = 0; r < 32; ++r) {
                                if (lbase + r < rows) {
                                    const double2 a = src[static_cast<int64_t>(r) * npairs];
                                    acc[r] = __fma_rn(a.x, xr[j].x, acc[r]);
                                    acc[r] = __fma_rn(a.y, xr[j].y, acc[r]);
                                }
                            }
                        }
                    } else {
                        const double *src = p.At + (r0 + lbase) * n;
                        if (full) {
#pragma unroll
                            for (int r = 0; r < 32; ++r) {
                                const double2 a = load_pair_global<EVEN>(src + static_cast<int64_t>(r) * n, q, n);
                                acc[r] = __fma_rn(a.x, xr[j].x, acc[r]);
                                acc[r] = __fma_rn(a.y, xr[j].y, acc[r]);
                            }
                        } else {
#pragma unroll
                            for (int r = 0; r < 32; ++r) {
                                if (lbase + r < rows) {
                                    const double2 a = load_pair_global<EVEN>(src + static_cast<int64_t>(r) * n, q, n);
                                    acc[r] = __fma_rn(a.x, xr[j].x, acc[r]);
                                    acc[r] = __fma_rn(a.y, xr[j].y, acc[r]);
                                }
                            }
                        }
                    }
                }
            }
            const double s = transpose_reduce32(acc, lane);
            part[(static_cast<size_t>(g) * Wc + cw) * 32 + lane] = s;
        }
        CSK_PHASE(0)
        __syncthreads();  // B1
        CSK_PHASE(1)

        // ---- S7 local: finalize rows (one per lane), warp argmax ----
        {
            double bs = -2.0, br = 0.0, rr = 0.0;
            int64_t bi = INT64_MAX;
            for (int l = warp * 32 + lane; l - lane < rows; l += kThreads) {
                if (l < rows) {
                    const int g = l >> 5, ln = l & 31;
                    double dot = part[(static_cast<size_t>(g) * Wc) * 32 + ln];
                    for (int c = 1; c < Wc; ++c) dot = dot + part[(static_cast<size_t>(g) * Wc + c) * 32 + ln];
                    const double ri = bt_loc[l] - dot;
                    const double ns = nsq_loc[l];
                    const double sc = ns > 0.0 ? (ri * ri) / ns : -1.0;
                    if (RESMODE) rr = __fma_rn(ri, ri, rr);
                    if (better(sc, r0 + l, bs, bi)) { bs = sc; bi = r0 + l; br = ri; }
                }
            }
            if (RESMODE) rr = warp_sum(rr);
            warp_argmax(bs, bi, br);
            if (lane == 0) cand[warp] = Cand{bs, br, rr, bi};
        }
        __syncthreads();  // B1b
        CSK_PHASE(2)

        // ---- S5 stop test + S7 grid exchange (warp 0) ----
        if (warp == 0) {
            int stop = -1;
            if (!RESMODE) {
                double a = res_w[0];
                for (int c = 1; c < Wc; ++c) a = a + res_w[c];
                res = xs_nrm > 0.0 ? a / xs_nrm : a;
                if (cta == 0 && lane == 0 && p.res_trace && k < p.trace_cap) p.res_trace[k] = res;
                if (res <= p.tol) stop = CSK_CONVERGED;
                else if (k == p.max_iters) stop = CSK_MAX_ITERS;
            }
            double ws = -2.0, wl = 0.0, wrr = 0.0;
            int64_t wi = INT64_MAX;
            if (stop < 0) {
                double cs = -2.0, cr = 0.0, crr = 0.0;
                int64_t ci = INT64_MAX;
                if (lane < kWarps) { cs = cand[lane].score; cr = cand[lane].r; ci = cand[lane].idx; }
                warp_argmax(cs, ci, cr);
                if (RESMODE) {
                    for (int w = 0; w < kWarps; ++w) crr = crr + cand[w].rr;  // fixed order
                }
                const double cl = (cs > 0.0) ? cr / nsq_loc[ci - r0] : 0.0;
                const uint32_t tag = static_cast<uint32_t>(k + 1);
                const uint64_t sb = __double_as_longlong(cs), lb = __double_as_longlong(cl),
                               rb = __double_as_longlong(crr);
                const uint64_t w0 = pack(static_cast<uint32_t>(sb >> 32), tag), w1 = pack(static_cast<uint32_t>(sb), tag);
                const uint64_t w2 = pack(static_cast<uint32_t>(lb >> 32), tag), w3 = pack(static_cast<uint32_t>(lb), tag);
                const uint64_t w4 = pack(static_cast<uint32_t>(rb >> 32), tag), w5 = pack(static_cast<uint32_t>(rb), tag);
                const uint64_t w6 = pack(static_cast<uint32_t>(ci), tag), w7 = pack(0u, tag);
                uint64_t *par = p.slots + static_cast<size_t>(k & 1) * G * G * kSlotWords;
                // push: this CTA's candidate into every reader's inbox (lane l -> readers l + 32j)
#pragma unroll
                for (int j = 0; j < kMaxSlotsPerLane; ++j) {
                    const int rd = lane + 32 * j;
                    if (rd < G) {
                        uint64_t *s = par + (static_cast<size_t>(rd) * G + cta) * kSlotWords;
                        st_relaxed_v2u64(s + 0, w0, w1);
                        st_relaxed_v2u64(s + 2, w2, w3);
                        st_relaxed_v2u64(s + 4, w4, w5);
                        st_relaxed_v2u64(s + 6, w6, w7);
                    }
                }
                CSK_PHASE(3)
                // poll own inbox (lane l owns writers l, l+32, ...)
                const uint64_t *inbox = par + static_cast<size_t>(cta) * G * kSlotWords;
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
                            const uint64_t *s = inbox + static_cast<size_t>(lane + 32 * j) * kSlotWords;
                            uint64_t a0, a1, a2, a3, a4, a5, a6, a7;
                            ld_relaxed_v2u64(s + 0, a0, a1);
                            ld_relaxed_v2u64(s + 2, a2, a3);
                            ld_relaxed_v2u64(s + 4, a4, a5);
                            ld_relaxed_v2u64(s + 6, a6, a7);
                            const bool ok = static_cast<uint32_t>(a0) == tag && static_cast<uint32_t>(a1) == tag &&
                                            static_cast<uint32_t>(a2) == tag && static_cast<uint32_t>(a3) == tag &&
                                            static_cast<uint32_t>(a4) == tag && static_cast<uint32_t>(a5) == tag &&
                                            static_cast<uint32_t>(a6) == tag;
                            if (ok) {
                                gs[j] = __longlong_as_double(static_cast<long long>((a0 >> 32) << 32 | (a1 >> 32)));
                                gl[j] = __longlong_as_double(static_cast<long long>((a2 >> 32) << 32 | (a3 >> 32)));
                                gr[j] = __longlong_as_double(static_cast<long long>((a4 >> 32) << 32 | (a5 >> 32)));
                                const uint32_t iw = static_cast<uint32_t>(a6 >> 32);
                                gi[j] = (iw == 0xffffffffu) ? INT64_MAX : static_cast<int64_t>(iw);
                                pending &= ~(1u << j);
                            }
                        }
                    }
                    if (__all_sync(0xffffffffu, pending == 0)) break;
                }
                CSK_PHASE(4)
                // combine in a fixed order: lane's slots ascending, then butterfly
#pragma unroll
                for (int j = 0; j < kMaxSlotsPerLane; ++j) {
                    if (better(gs[j], gi[j], ws, wi)) { ws = gs[j]; wi = gi[j]; wl = gl[j]; }
                    if (RESMODE) wrr = wrr + gr[j];
                }
                warp_argmax(ws, wi, wl);
                if (RESMODE) {
                    wrr = warp_sum(wrr);
                    res = bb > 0.0 ? wrr / bb : wrr;
                    if (cta == 0 && lane == 0 && p.res_trace && k < p.trace_cap) p.res_trace[k] = res;
                    if (res <= p.tol) stop = CSK_CONVERGED;
                    else if (k == p.max_iters) stop = CSK_MAX_ITERS;
                }
                if (stop < 0) {
                    if (ws < 0.0) stop = -2;                 // every row masked: zero sketch
                    else if (ws == 0.0) stop = CSK_STAGNATED;
                }
                if (stop < 0) {
                    // stage the winner row A~^(ik) in shared memory
                    const double *src = p.At + wi * n;
                    for (int64_t q = lane; q < npairs; q += 32) wrow[q] = load_pair_global<EVEN>(src, q, n);
                    if (cta == 0 && lane == 0 && p.idx_trace && k < p.trace_cap) p.idx_trace[k] = wi;
                }
            }
            if (lane == 0) {
                win[0] = wi;
                win[1] = __double_as_longlong(wl);
                win[2] = stop;
                win[3] = __double_as_longlong(res);
            }
            CSK_PHASE(5)
        }
        __syncthreads();  // B2
        CSK_PHASE(6)
        const int stop = static_cast<int>(win[2]);
        if (stop >= 0 || stop == -2) {
            term = stop;
            res = __longlong_as_double(win[3]);
            break;
        }
        // ---- S8: x_{k+1} = x_k + lambda A~^(ik)T ----
        const double wl = __longlong_as_double(win[1]);
        last = win[0];
#pragma unroll
        for (int j = 0; j < P; ++j) {
            const int64_t q = static_cast<int64_t>(cw) * 32 * P + lane + 32 * j;
            if (q < npairs) {
                const double2 a = wrow[q];
                xr[j].x = __fma_rn(wl, a.x, xr[j].x);
                xr[j].y = __fma_rn(wl, a.y, xr[j].y);
            }
        }
        CSK_PHASE(7)
    }
#undef CSK_PHASE
    if (prof) {
        for (int i = 0; i < 8; ++i) p.phase_cycles[warp * 8 + i] = ph[i];
    }

    // ---- epilogue: CTA 0 team 0 writes x; thread 0 the report ----
    if (cta == 0 && team == 0) {
#pragma unroll
        for (int j = 0; j < P; ++j) {
            const int64_t q = static_cast<int64_t>(cw) * 32 * P + lane + 32 * j;
            if (q < npairs) {
                p.x[2 * q] = xr[j].x;
                if (2 * q + 1 < n) p.x[2 * q + 1] = xr[j].y;
            }
        }
        if (tid == 0) {
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

template <int P>
KernelFn pick_mode(bool even, bool resmode) {
    if (even) return resmode ? k_solve<P, true, true> : k_solve<P, true, false>;
    return resmode ? k_solve<P, false, true> : k_solve<P, false, false>;
}

// P = column pairs per lane (power of two), Wc = column warps (power of two <= 8).
KernelFn pick_kernel(int64_t n, bool resmode, int &P, int &wc) {
    const int64_t npairs = (n + 1) / 2;
    P = 1;
    while (32 * kWarps * P < npairs) P *= 2;
    wc = 1;
    while (wc < kWarps && 32 * P * wc < npairs) wc *= 2;
    const bool even = (n & 1) == 0;
    switch (P) {
        case 1: return pick_mode<1>(even, resmode);
        case 2: return pick_mode<2>(even, resmode);
        case 4: return pick_mode<4>(even, resmode);
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
    if (ctx->pending) return fail(ctx, CSK_E_ARG, "csk_solve: a CSK_SOLVE_ASYNC solve is still in flight (call csk_solve_wait)");
    const bool resmode = (x_star == nullptr);
    int P = 0, wc = 0;
    KernelFn fn = pick_kernel(n, resmode, P, wc);
    if (!fn) return fail(ctx, CSK_E_UNSUPPORTED, "csk_solve: n out of range");

    int G = ctx->num_sms;
    if (opts && opts->num_ctas > 0) G = opts->num_ctas;
    if (G > kMaxG) G = kMaxG;
    if (G > d) G = static_cast<int>(d);
    const int64_t rows_max = (d + G - 1) / G;
    const int64_t ngroups = (rows_max + 31) / 32;
    const int64_t npairs = (n + 1) / 2;
    const int64_t npairs_pad = static_cast<int64_t>(wc) * 32 * P;
    const size_t fixed = static_cast<size_t>(npairs_pad) * 16 + static_cast<size_t>(ngroups) * wc * 32 * 8 +
                         static_cast<size_t>(rows_max) * 16 + 8 * 8 + kWarps * sizeof(Cand) + 64 + 64;
    const size_t avail = ctx->max_smem_optin > static_cast<int>(fixed) ? ctx->max_smem_optin - fixed : 0;
    int64_t srows = static_cast<int64_t>(avail / (static_cast<size_t>(npairs) * 16));
    if (srows >= rows_max) {
        srows = rows_max;
    } else {
        srows = (srows / 32) * 32;  // whole 32-row groups so every group has one source
    }
    if (opts && opts->smem_rows > 0 && opts->smem_rows < srows) srows = (opts->smem_rows / 32) * 32;
    if (opts && opts->smem_rows < 0) srows = 0;
    const size_t smem = fixed + static_cast<size_t>(srows) * npairs * 16;

    CSK_CUDA(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int per_sm = 0;
    CSK_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem));
    if (per_sm * ctx->num_sms < G)
        return fail(ctx, CSK_E_UNSUPPORTED, "csk_solve: grid cannot be co-resident");

    const size_t slot_bytes = static_cast<size_t>(2) * G * G * kSlotWords * 8;
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
    prm.trace_cap = opts ? opts->trace_cap : 0;
    prm.idx_trace = opts ? opts->idx_trace : nullptr;
    prm.res_trace = opts ? opts->res_trace : nullptr;
    prm.x_trace = opts ? opts->x_trace : nullptr;
    prm.phase_cycles = opts ? opts->phase_cycles : nullptr;
    if (prm.trace_cap <= 0) { prm.idx_trace = nullptr; prm.res_trace = nullptr; prm.x_trace = nullptr; prm.trace_cap = 0; }

    void *args[] = {&prm};
    CSK_CUDA(ctx, cudaLaunchCooperativeKernel(reinterpret_cast<void *>(fn), dim3(G), dim3(kThreads), args, smem, stream));
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
