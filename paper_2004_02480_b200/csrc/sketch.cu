// sketch.cu -- S3 count-sketch application A~ = S A, b~ = S b and S4 row norms.
//
// Algorithm 1 "Initialize": A~ = S A, b~ = S b with S = Phi D (Def. 1,
// P:50).  Row j of A~ is the signed sum of the rows of A hashed to bucket j, added in
// ascending row order from +0.0, i.e. exactly the fp64 adds of the dense
// product Phi D A -- so every A~ / b~ entry is bit-identical to the CPU oracle.
//
// Dense kernel (B200 design):
//   * persistent grid, one CTA per SM; CTA c owns the buckets whose first row falls in
//     rows [c m/G, (c+1) m/G) of the bucket-sorted order, so the work per CTA is a
//     contiguous range of `perm` (balanced by rows, not by buckets);
//   * a producer warp streams the gathered rows of A into a shared-memory ring with
//     1-D TMA bulk copies (cp.async.bulk, completion on an mbarrier per slot);
//     each row of A is read from HBM exactly once, as one contiguous 8n-byte burst;
//   * consumer warps own column pairs (16-byte lanes) and fold the ring rows into
//     fp64 register accumulators in ring (= row) order; at a bucket boundary they
//     store the row of A~ (coalesced) and reduce its squared norm (S4, fused);
//   * a b-warp folds b~ for the same buckets, one bucket per lane, row order.
// Short rows (n <= 256, the paper's Table-1 shapes): warp per bucket, rows loaded straight
//   from HBM with R rows in flight per warp (k_sketch_dense_wpb).
// CSR kernel (config C5): warp per bucket range, dense shared-memory accumulator row, the
//   (col, val) pairs gathered by cp.async into per-warp stages, several batches in flight.
#include "csk_internal.cuh"

namespace csk {

namespace {

constexpr int kPmax = 4;               // column pairs per consumer thread (template max)
constexpr int kMaxConsumers = 256;     // consumer threads per CTA
constexpr int kMaxStages = 32;         // ring depth cap
constexpr int kMaxRB = 32;             // rows per stage cap
constexpr int kRingBudget = 200 * 1024;
constexpr int kStageTarget = 16 * 1024;  // bytes per stage (TMA batch)

struct DenseGeom {
    int tc;          // consumer threads (multiple of 32)
    int p;           // pairs per consumer thread (1, 2 or 4)
    int chunk_cols;  // columns per chunk (even), = 2 * tc * p
    int chunks;      // ceil(n / chunk_cols)
    int slot_bytes;  // bytes per row slot (multiple of 128)
    int rb;          // rows per ring stage
    int stages;      // ring depth
    size_t header;   // barriers + metadata
    size_t smem;     // dynamic shared memory
};

size_t dense_header(int stages, int rb) {
    // full[stages], empty[stages] (8 B), meta[stages][kMaxRB] (4 B), red[2][8] doubles (last 128 B)
    (void)rb;
    size_t h = static_cast<size_t>(stages) * 16 + static_cast<size_t>(stages) * kMaxRB * 4 + 2 * 8 * 8;
    return (h + 127) / 128 * 128;
}

DenseGeom dense_geom(int64_t n, bool tma) {
    DenseGeom g{};
    const int64_t pairs = (n + 1) / 2;
    int64_t tc = ((pairs + 31) / 32) * 32;
    if (tc > kMaxConsumers) tc = kMaxConsumers;
    int64_t p = (pairs + tc - 1) / tc;
    if (p > kPmax) p = kPmax;
    if (p == 3) p = 4;
    g.tc = static_cast<int>(tc);
    g.p = static_cast<int>(p);
    g.chunk_cols = 2 * g.tc * g.p;
    g.chunks = static_cast<int>((n + g.chunk_cols - 1) / g.chunk_cols);
    const int64_t cols0 = n < g.chunk_cols ? n : g.chunk_cols;
    g.slot_bytes = tma ? static_cast<int>(((cols0 * 8 + 127) / 128) * 128) : 0;
    int rb = tma ? kStageTarget / g.slot_bytes : 8;
    if (rb < 1) rb = 1;
    if (rb > kMaxRB) rb = kMaxRB;
    while (rb & (rb - 1)) rb &= rb - 1;  // power of two: whole stages per 32-row perm window
    g.rb = rb;
    int stages = tma ? kRingBudget / (rb * g.slot_bytes) : 4;
    if (stages > kMaxStages) stages = kMaxStages;
    if (stages < 2) stages = 2;
    g.stages = stages;
    g.header = dense_header(stages, rb);
    g.smem = g.header + static_cast<size_t>(stages) * rb * g.slot_bytes;
    return g;
}

// lower_bound(a[0..len), v) by one warp: 32 probes per step (log32 len dependent loads instead of
// log2 len); every lane returns the same index
__device__ __forceinline__ int64_t warp_lower_bound(const int32_t *a, int64_t len, int64_t v, int lane) {
    int64_t lo = 0, hi = len;
    while (hi - lo > 32) {
        const int64_t step = (hi - lo + 31) / 32;
        const int64_t pk = lo + lane * step;
        const bool below = pk < hi && static_cast<int64_t>(__ldg(a + pk)) < v;
        const int c = __popc(__ballot_sync(0xffffffffu, below));
        if (c == 0) return lo;
        const int64_t nhi = lo + c * step < hi ? lo + c * step : hi;
        lo = lo + (c - 1) * step + 1;
        hi = nhi;
    }
    const bool below = lo + lane < hi && static_cast<int64_t>(__ldg(a + lo + lane)) < v;
    return lo + __popc(__ballot_sync(0xffffffffu, below));
}


// Warp-level butterfly sum: every lane ends with the same bits (IEEE + is commutative).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// TMA = true: rows staged by 1-D bulk copies (A 16-byte aligned, lda even).
// TMA = false: any alignment; the producer only publishes the row order and the
// consumers read their columns straight from global memory (same adds, same order).
// The CTA's rows are the contiguous range [t0, t1) of `perm`; the ring moves them in
// stages of `rb` rows (one full/empty mbarrier pair per stage); slot and phase are
// tracked incrementally (no division on the per-row path).
template <int P, bool TMA, int RB>
__global__ void __launch_bounds__(kMaxConsumers + 64, 1)
k_sketch_dense(const double *__restrict__ A, int64_t lda, const double *__restrict__ b, int64_t m,
               int64_t n, int64_t d, const int32_t *__restrict__ perm,
               const int32_t *__restrict__ offsets, double *__restrict__ At,
               double *__restrict__ bt, int tc, int chunk_cols,
               int chunks, int slot_bytes, int rb, int stages, int header) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *empty = full + stages;
    int32_t *meta = reinterpret_cast<int32_t *>(empty + stages);   // [stages][kMaxRB] row | sign bit
    unsigned char *ring = smem + header;
    const int stage_bytes = rb * slot_bytes;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const int wc = tc >> 5;  // consumer warps

    __shared__ int64_t s_j0, s_j1;
    // the CTA's bucket range: warps 0 and 1 search for its two ends side by side (32 probes per
    // step: ~3 dependent L2 loads each instead of two serial ~13-step binary searches)
    if (warp < 2) {
        const int G = static_cast<int>(gridDim.x), c = static_cast<int>(blockIdx.x) + warp;
        const int64_t j = (c == G) ? d : warp_lower_bound(offsets, d, m * c / G, lane);
        if (lane == 0) (warp == 0 ? s_j0 : s_j1) = j;
    }
    if (tid == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], wc);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int64_t j0 = s_j0, j1 = s_j1;
    if (j0 >= j1) return;
    const int64_t t0 = offsets[j0];
    const int64_t t1 = offsets[j1];
    const int64_t nrows = t1 - t0;
    const int64_t nst = (nrows + rb - 1) / rb;  // stages per chunk

    if (warp == wc) {
        // ------------------------------------------------ producer warp (TMA)
        int s = 0;
        uint32_t ph = 0;   // phase of the current use of stage s
        int64_t use = 0;   // total stage uses so far
        for (int c = 0; c < chunks; ++c) {
            const int64_t c0 = static_cast<int64_t>(c) * chunk_cols;
            const int64_t c1 = (c0 + chunk_cols < n) ? c0 + chunk_cols : n;
            const uint32_t bytes = TMA ? static_cast<uint32_t>(((c1 - c0) & ~int64_t(1)) * 8) : 0u;
            // perm is read 32 rows (32/rb whole stages) at a time, one window ahead
            int32_t cur = (t0 + lane < t1) ? __ldg(perm + t0 + lane) : 0;
            int32_t nxt = 0;
            for (int64_t u = 0; u < nst; ++u, ++use) {
                const int64_t tb = t0 + u * rb;
                const int wofs = static_cast<int>((u * rb) & 31);
                if (wofs == 0) {
                    if (u > 0) cur = nxt;
                    const int64_t tn = tb + 32 + lane;
                    nxt = (tn < t1) ? __ldg(perm + tn) : 0;
                }
                const int cnt = static_cast<int>((t1 - tb) < rb ? (t1 - tb) : rb);
                const int32_t mine = __shfl_sync(0xffffffffu, cur, (wofs + lane) & 31);
                if (use >= stages) mbar_wait(&empty[s], ph ^ 1u);
                if (lane < cnt) meta[s * kMaxRB + lane] = mine;
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive_expect_tx(&full[s], bytes * static_cast<uint32_t>(cnt));
                }
                __syncwarp();
                if (bytes && lane < cnt) {
                    const int64_t row = mine & 0x7fffffff;
                    bulk_g2s(ring + static_cast<size_t>(s) * stage_bytes + static_cast<size_t>(lane) * slot_bytes,
                             A + row * lda + c0, bytes, &full[s]);
                }
                if (++s == stages) { s = 0; ph ^= 1u; }
            }
        }
        return;
    }
    if (warp == wc + 1) {
        // ------------------------------------------------ b~ warp: one bucket per lane
        for (int64_t j = j0 + lane; j < j1; j += 32) {
            const int64_t a = offsets[j], e = offsets[j + 1];
            double acc = 0.0;
            int64_t t = a;
            for (; t + 4 <= e; t += 4) {
                int32_t p4[4];
                double v4[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) p4[q] = __ldg(perm + t + q);
#pragma unroll
                for (int q = 0; q < 4; ++q) v4[q] = __ldg(b + (p4[q] & 0x7fffffff));
#pragma unroll
                for (int q = 0; q < 4; ++q) acc = acc + (p4[q] < 0 ? -v4[q] : v4[q]);
            }
            for (; t < e; ++t) {
                const int32_t pr = __ldg(perm + t);
                const double v = __ldg(b + (pr & 0x7fffffff));
                acc = acc + (pr < 0 ? -v : v);
            }
            bt[j] = acc;
        }
        return;
    }

    // ---------------------------------------------------- consumer warps
    int s = 0;
    uint32_t ph = 0;
    for (int c = 0; c < chunks; ++c) {
        const int64_t c0 = static_cast<int64_t>(c) * chunk_cols;
        const int64_t c1 = (c0 + chunk_cols < n) ? c0 + chunk_cols : n;
        const int64_t ce = TMA ? c0 + ((c1 - c0) & ~int64_t(1)) : c0;  // end of the TMA-copied columns
        int64_t j = j0;
        int64_t e = offsets[j + 1];  // end (exclusive) of bucket j in perm order
        double2 acc[P];
#pragma unroll
        for (int q = 0; q < P; ++q) acc[q] = make_double2(0.0, 0.0);

        // bucket epilogue: store the row of A~ and (fused S4) its squared norm
        auto flush = [&](int64_t jj) {
            double *dst = At + jj * n;
#pragma unroll
            for (int q = 0; q < P; ++q) {
                const int qq = tid + tc * q;
                const int64_t col = c0 + 2 * static_cast<int64_t>(qq);
                if (col + 1 < c1) {
                    if ((n & 1) == 0) {
                        *reinterpret_cast<double2 *>(dst + col) = acc[q];
                    } else {
                        dst[col] = acc[q].x;
                        dst[col + 1] = acc[q].y;
                    }
                } else if (col < c1) {
                    dst[col] = acc[q].x;
                }
                acc[q] = make_double2(0.0, 0.0);
            }
        };

        int64_t t = t0;
        // leading empty buckets
        while (j < j1 && e == t) { flush(j); ++j; if (j < j1) e = offsets[j + 1]; }
        for (int64_t u = 0; u < nst; ++u) {
            const int cnt = static_cast<int>((t1 - t) < rb ? (t1 - t) : rb);
            mbar_wait(&full[s], ph);
            const int32_t *mrow = meta + s * kMaxRB;
            const unsigned char *sbase = ring + static_cast<size_t>(s) * stage_bytes;
            if (TMA && RB > 1 && cnt == RB && rb == RB && e - t >= RB && ce == c1) {
                // fast path: full stage, no bucket boundary inside, every column in the copy:
                // issue all loads of the stage, then fold them in row order
                double2 v[RB][P];
                uint64_t sg[RB];
#pragma unroll
                for (int r = 0; r < RB; ++r) {
                    sg[r] = mrow[r] < 0 ? 0x8000000000000000ULL : 0ULL;
                    const double2 *srow = reinterpret_cast<const double2 *>(sbase + static_cast<size_t>(r) * slot_bytes);
#pragma unroll
                    for (int q = 0; q < P; ++q) {
                        const int qq = tid + tc * q;
                        v[r][q] = (c0 + 2 * static_cast<int64_t>(qq) < c1) ? srow[qq] : make_double2(0.0, 0.0);
                    }
                }
#pragma unroll
                for (int r = 0; r < RB; ++r) {
#pragma unroll
                    for (int q = 0; q < P; ++q) {
                        // sign flip = xor of the sign bit (exact, same bits as -v)
                        acc[q].x = acc[q].x + __longlong_as_double(__double_as_longlong(v[r][q].x) ^ sg[r]);
                        acc[q].y = acc[q].y + __longlong_as_double(__double_as_longlong(v[r][q].y) ^ sg[r]);
                    }
                }
                t += RB;
                while (j < j1 && e == t) { flush(j); ++j; if (j < j1) e = offsets[j + 1]; }
            } else {
            for (int r = 0; r < cnt; ++r, ++t) {
                const int32_t pr = mrow[r];
                const bool neg = pr < 0;
                const double2 *srow = reinterpret_cast<const double2 *>(sbase + static_cast<size_t>(r) * slot_bytes);
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    const int qq = tid + tc * q;
                    const int64_t col = c0 + 2 * static_cast<int64_t>(qq);
                    if (col + 1 < ce) {
                        double2 v = srow[qq];
                        if (neg) { v.x = -v.x; v.y = -v.y; }
                        acc[q].x = acc[q].x + v.x;
                        acc[q].y = acc[q].y + v.y;
                    } else if (col < c1) {  // columns not in the bulk copy: read directly
                        const double *src = A + static_cast<int64_t>(pr & 0x7fffffff) * lda + col;
                        double v = src[0];
                        if (neg) v = -v;
                        acc[q].x = acc[q].x + v;
                        if (col + 1 < c1) {
                            double w = src[1];
                            if (neg) w = -w;
                            acc[q].y = acc[q].y + w;
                        }
                    }
                }
                // bucket boundary after row t (and any empty buckets that follow)
                while (j < j1 && e == t + 1) { flush(j); ++j; if (j < j1) e = offsets[j + 1]; }
            }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == stages) { s = 0; ph ^= 1u; }
        }
    }
}

// Standalone S4: the same per-row arithmetic as the fused epilogue above
// (thread t sums pairs t + tc*p, p ascending, then warp butterfly, then warps in
// order, then chunks in order), one CTA of `tc` threads per row.

// Short rows (n <= 256): one warp per bucket.  The row-per-CTA ring above moves each gathered
// row with its own bulk copy, and for rows of a few hundred bytes the copy issue rate, not HBM,
// bounds it (one consumer warp per CTA at n <= 64).  Here every warp owns whole buckets: lane l
// holds column pairs l + 32 v (v < V), the bucket's rows are folded in ascending order (the same
// adds as the oracle), R rows' loads in flight per warp, b~ folded alongside by every lane.  The
// fused norm keeps the standalone k_row_norms order (for n <= 256 its team is tc = 32 V' threads,
// thread t = 32 v + l holding pair t): a partial per v, butterfly, then v ascending.

template <int V, bool VEC>
__global__ void __launch_bounds__(256, 2)
k_sketch_dense_wpb(const double *__restrict__ A, int64_t lda, const double *__restrict__ b, int64_t m, int64_t n, int64_t d,
                   const int32_t *__restrict__ perm, const int32_t *__restrict__ offsets, double *__restrict__ At,
                   double *__restrict__ bt, int tcw) {
    constexpr int R = V == 1 ? 16 : V == 2 ? 8 : 4;  // rows in flight per warp
    const int lane = threadIdx.x & 31;
    const int W = static_cast<int>((static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5);
    const int w = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    // warp w: the buckets whose first row lies in [w m / W, (w + 1) m / W) of the sorted order
    // (contiguous, balanced by rows); their rows are one contiguous range of perm, streamed in
    // batches of R rows that may span bucket boundaries
    int64_t j = warp_lower_bound(offsets, d, m * w / W, lane);
    int64_t je = (w == W - 1) ? d : warp_lower_bound(offsets, d, m * (w + 1) / W, lane);
    if (j >= je) return;
    const int64_t T1 = offsets[je];
    int64_t t = offsets[j];
    // bucket ends in a lane-distributed window: lane l holds offsets[wb + 1 + l]
    int64_t wb = j;
    int32_t owin = (wb + 1 + lane <= je) ? __ldg(offsets + wb + 1 + lane) : static_cast<int32_t>(T1);
    auto end_of = [&](int64_t jj) -> int64_t {  // offsets[jj + 1] (warp-uniform jj >= wb)
        if (jj - wb >= 32) {
            wb = jj;
            owin = (wb + 1 + lane <= je) ? __ldg(offsets + wb + 1 + lane) : static_cast<int32_t>(T1);
        }
        return __shfl_sync(0xffffffffu, owin, static_cast<int>(jj - wb));
    };
    int64_t e = end_of(j);  // end of bucket j in perm order
    double2 acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = make_double2(0.0, 0.0);
    double bacc = 0.0;
    // bucket epilogue: the row of A~, b~_j, and the fused norm in the standalone order
    auto flush = [&]() {
        double *dst = At + j * n;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const int64_t col = 2 * static_cast<int64_t>(lane + 32 * v);
            if (col + 1 < n) {
                if (VEC) *reinterpret_cast<double2 *>(dst + col) = acc[v];
                else { dst[col] = acc[v].x; dst[col + 1] = acc[v].y; }
            } else if (col < n) {
                dst[col] = acc[v].x;
            }
            acc[v] = make_double2(0.0, 0.0);
        }
        if (lane == 0) bt[j] = bacc;
        bacc = 0.0;
        ++j;
        e = (j < je) ? end_of(j) : T1;
    };
    while (j < je && e == t) flush();  // leading empty buckets
    int32_t prn = (t + lane < T1) ? __ldg(perm + t + lane) : 0;  // the next batch's perm window
    for (; t < T1; t += R) {
        const int cnt = (T1 - t) < R ? static_cast<int>(T1 - t) : R;
        // lane r holds the batch's r-th perm entry and its b value; the next window is in flight
        const int32_t prl = prn;
        prn = (t + R + lane < T1) ? __ldg(perm + t + R + lane) : 0;
        const double bl = lane < cnt ? __ldg(b + (prl & 0x7fffffff)) : 0.0;
        int32_t pr[R];
#pragma unroll
        for (int r = 0; r < R; ++r) pr[r] = __shfl_sync(0xffffffffu, prl, r);
        double2 val[R][V];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const double *src = A + static_cast<int64_t>(pr[r] & 0x7fffffff) * lda;
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const int64_t col = 2 * static_cast<int64_t>(lane + 32 * v);
                double2 x2 = make_double2(0.0, 0.0);
                if (r < cnt && col < n) {
                    if (VEC && col + 1 < n) {
                        x2 = __ldg(reinterpret_cast<const double2 *>(src + col));
                    } else {
                        x2.x = __ldg(src + col);
                        if (col + 1 < n) x2.y = __ldg(src + col + 1);
                    }
                }
                val[r][v] = x2;
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (r < cnt) {  // ascending row order; the sign flip is exact
                const bool neg = pr[r] < 0;
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    acc[v].x = acc[v].x + (neg ? -val[r][v].x : val[r][v].x);
                    acc[v].y = acc[v].y + (neg ? -val[r][v].y : val[r][v].y);
                }
                const double bvr = __shfl_sync(0xffffffffu, bl, r);
                bacc = bacc + (neg ? -bvr : bvr);
                while (j < je && e == t + r + 1) flush();  // bucket boundary (and empty buckets)
            }
        }
    }
}


// ---- CSR sketch (config C5): warp pair per bucket range, dense shared-memory accumulator row ----
//
// Pair w (a producer warp and a consumer warp) owns the buckets whose first row lies in
// [w m/W, (w+1) m/W) of the bucket-sorted order: one contiguous range of `perm`.  The pair stream
// of a bucket (its rows' stored (col, val) pairs, rows ascending, pairs in stored order) is cut
// into batches of <= kCsrSP pairs (whole rows, or a slice of one long row).  The PRODUCER forms
// each batch: row descriptors (perm entry, row_ptr pair, b) 32 rows at a time, one window ahead
// (perm two windows ahead), a scan of the rows' pair counts, and the GATHER with cp.async (LDGSTS:
// 8-byte val, 4-byte col, no registers held) into one of kCsrS shared-memory stages; it folds b~
// (row order) and writes empty buckets itself.  The stage's `full` mbarrier completes when every
// producer lane's copies have landed (cp.async.mbarrier.arrive.noinc) and its meta is written.
// The CONSUMER folds 32 pairs per step into its accumulator row and releases the stage (`empty`).
// Two pairs of one step can hit the same column only if they come from different rows (a row's
// columns are distinct): a per-pair byte array of lane stamps (every lane writes its id at its
// column, then reads it back) detects that case in four instructions, and only such steps take
// the ordered path (__match_any_sync ranks, earlier pair = earlier row first), so every column is
// the ascending-row fold.  At a bucket's last batch the consumer stores the A~ row (coalesced
// 16-byte stores) and clears the accumulator; the norms follow in k_row_norms_exact.
// Round 2 split the former single-warp loop (formation and fold interleaved in one warp, at most
// 16 warps per SM) into this pair: the fold's add chain no longer waits behind the formation's
// descriptor loads, 0.90 -> 0.60 ms at C5.
#ifndef CSK_CSR_STAGES
#define CSK_CSR_STAGES 2
#endif
#ifndef CSK_CSR_STAGE_PAIRS
#define CSK_CSR_STAGE_PAIRS 256
#endif
constexpr int kCsrS = CSK_CSR_STAGES;                          // stages (batches in flight) per pair
constexpr int kCsrSP = CSK_CSR_STAGE_PAIRS;                    // pairs per stage
constexpr int kCsrStageBytes = kCsrSP * (8 + 4 + 1);           // val | col | sign
constexpr int kCsrMetaBytes = kCsrS * 16 + kCsrS * 16;  // batch meta + the full / empty mbarriers
constexpr int kCsrMaxWarps = 16;                                 // 8 pairs

__device__ __forceinline__ void cp_async4(uint32_t dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
// the mbarrier receives one arrival once all of this thread's earlier cp.async copies have landed
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t *bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(kCsrMaxWarps * 32, 1)
k_sketch_csr(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col, const double *__restrict__ val,
             const double *__restrict__ b, int64_t m, int64_t n, int64_t d, const int32_t *__restrict__ perm,
             const int32_t *__restrict__ offsets, double *__restrict__ At, double *__restrict__ bt,
             int64_t acc_stride, int stamp_bytes, int warp_bytes, int vec) {
    // warp specialisation: warp p < NP forms and issues batches (producer), warp NP + p folds them
    // into its accumulator row (consumer); they meet on kCsrS stages with a full / empty mbarrier
    // pair each, so the formation (descriptor loads, gathers, b~) overlaps the fold's add chain
    extern __shared__ __align__(16) unsigned char csr_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int NP = static_cast<int>(blockDim.x >> 6);
    const bool producer = warp < NP;
    const int pw = producer ? warp : warp - NP;  // the pair
    unsigned char *ws = csr_smem + static_cast<size_t>(pw) * warp_bytes;
    double *acc = reinterpret_cast<double *>(ws);
    unsigned char *stamp = ws + acc_stride * 8;  // [stamp_bytes]: lane id per column (conflict test)
    unsigned char *stg = stamp + stamp_bytes;
    int *meta = reinterpret_cast<int *>(stg + kCsrS * kCsrStageBytes);  // [kCsrS][4]: pairs, bucket, end
    uint64_t *full = reinterpret_cast<uint64_t *>(meta + kCsrS * 4);   // [kCsrS]: 32 gather + 32 plain arrivals
    uint64_t *empty = full + kCsrS;                                    // [kCsrS]: the consumer's release
    if (!producer) {
        for (int64_t k = lane; k < acc_stride; k += 32) acc[k] = 0.0;
    } else if (lane == 0) {
        for (int q = 0; q < kCsrS; ++q) {
            mbar_init(full + q, 64);
            mbar_init(empty + q, 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    if (!producer) {
        // ---- consumer: fold batch after batch until the producer's sentinel (pairs = -1) ----
        for (int folded = 0;; ++folded) {
            const int slot = folded % kCsrS;
            mbar_wait(full + slot, static_cast<uint32_t>((folded / kCsrS) & 1));
            const int P = meta[slot * 4 + 0];
            if (P < 0) break;
            const int64_t jb = meta[slot * 4 + 1];
            const bool end = meta[slot * 4 + 2] != 0;
            const double *sv = reinterpret_cast<const double *>(stg + slot * kCsrStageBytes);
            const int32_t *sc = reinterpret_cast<const int32_t *>(stg + slot * kCsrStageBytes + kCsrSP * 8);
            const unsigned char *sg = stg + slot * kCsrStageBytes + kCsrSP * 12;
            int c0 = lane < P ? sc[lane] : -1;
            double v0 = lane < P ? sv[lane] : 0.0;
            if (lane < P && sg[lane]) v0 = -v0;
            for (int q0 = 0; q0 < P; q0 += 32) {
                const int q1 = q0 + 32 + lane;
                int c1 = -1;
                double v1 = 0.0;
                if (q1 < P) {
                    c1 = sc[q1];
                    v1 = sv[q1];
                    if (sg[q1]) v1 = -v1;
                }
                if (c0 >= 0) stamp[c0] = static_cast<unsigned char>(lane);
                __syncwarp();
                const bool clash = c0 >= 0 && stamp[c0] != lane;
                CSK_DCHECK(c0 < static_cast<int>(n));
                if (!__any_sync(0xffffffffu, clash)) {
                    if (c0 >= 0) acc[c0] = acc[c0] + v0;  // distinct columns: one step
                } else {
                    const unsigned same = __match_any_sync(0xffffffffu, c0 >= 0 ? c0 : -1 - lane);
                    const unsigned rank = __popc(same & lt);
                    const unsigned maxr = __reduce_max_sync(0xffffffffu, rank);
                    for (unsigned rr = 0; rr <= maxr; ++rr) {
                        if (c0 >= 0 && rank == rr) acc[c0] = acc[c0] + v0;
                        __syncwarp();
                    }
                }
                __syncwarp();
                c0 = c1;
                v0 = v1;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + slot);  // the stage may be refilled
            if (end) {  // bucket jb complete: store the A~ row, clear the accumulator
                double *dst = At + jb * n;
                if (vec) {
                    double2 *a2 = reinterpret_cast<double2 *>(acc);
                    double2 *d2 = reinterpret_cast<double2 *>(dst);
                    for (int64_t k2 = lane; k2 < n / 2; k2 += 32) {
                        d2[k2] = a2[k2];
                        a2[k2] = make_double2(0.0, 0.0);
                    }
                } else {
                    for (int64_t k = 2 * lane; k < n; k += 64) {
                        dst[k] = acc[k];
                        acc[k] = 0.0;
                        if (k + 1 < n) {
                            dst[k + 1] = acc[k + 1];
                            acc[k + 1] = 0.0;
                        }
                    }
                }
                __syncwarp();
            }
        }
        return;
    }
    // ---- producer ----
    const int W = static_cast<int>(gridDim.x) * NP;
    const int w = static_cast<int>(blockIdx.x) * NP + pw;
    int64_t fj = warp_lower_bound(offsets, d, m * w / W, lane);
    const int64_t je = (w == W - 1) ? d : warp_lower_bound(offsets, d, m * (w + 1) / W, lane);
    auto finish = [&](int slot) {  // the sentinel: this pair has no more batches
        if (lane == 0) meta[slot * 4 + 0] = -1;
        cp_async_arrive_noinc(full + slot);
        mbar_arrive(full + slot);
    };
    if (fj >= je) {
        finish(0);
        return;
    }
    const int64_t T1 = offsets[je];
    int64_t t = offsets[fj];  // perm position of the next row to take
    // bucket ends, lane-distributed: lane l holds offsets[ob + 1 + l]
    int64_t ob = fj;
    int32_t owin = (ob + 1 + lane <= je) ? __ldg(offsets + ob + 1 + lane) : static_cast<int32_t>(T1);
    auto end_of = [&](int64_t jj) -> int64_t {  // offsets[jj + 1] (warp-uniform jj >= ob)
        if (jj - ob >= 32) {
            ob = jj;
            owin = (ob + 1 + lane <= je) ? __ldg(offsets + ob + 1 + lane) : static_cast<int32_t>(T1);
        }
        return __shfl_sync(0xffffffffu, owin, static_cast<int>(jj - ob));
    };
    auto zero_row = [&](int64_t jj) {  // an empty bucket: A~ row 0, b~ 0, nsq 0
        double *dst = At + jj * n;
        for (int64_t k = lane; k < n; k += 32) dst[k] = 0.0;
        if (lane == 0) {
            bt[jj] = 0.0;
        }
    };
    int64_t fe = end_of(fj);  // end (perm position) of the bucket being formed
    while (fj < je && fe == t) {
        zero_row(fj);
        ++fj;
        if (fj < je) fe = end_of(fj);
    }
    // ---- row-descriptor windows: lane l describes the row at perm position wbase + l ----
    auto load_pr = [&](int64_t base) -> int32_t { return (base + lane < T1) ? __ldg(perm + base + lane) : 0; };
    int64_t wbase = t;
    int32_t pr = load_pr(wbase);
    const int32_t pr1 = load_pr(wbase + 32);
    int32_t pr2 = load_pr(wbase + 64);
    auto desc = [&](int64_t base, int32_t p, int64_t &rs, int64_t &re, double &bv) {
        const int64_t r = p & 0x7fffffff;
        const bool ok = base + lane < T1;
        rs = ok ? __ldg(row_ptr + r) : 0;
        re = ok ? __ldg(row_ptr + r + 1) : 0;
        bv = ok ? __ldg(b + r) : 0.0;
    };
    int64_t rs, re, nrs, nre;
    double bv, nbv;
    desc(wbase, pr, rs, re, bv);
    int32_t npr = pr1;
    desc(wbase + 32, npr, nrs, nre, nbv);
    int64_t roff = 0;  // pairs of the row at t already taken (a long row split over batches)
    double bacc = 0.0;
    int issued = 0;
    // ---- form one batch of bucket fj into stage `slot` and issue its gathers ----
    auto form = [&](int slot) {
        if (t - wbase >= 32) {  // next window (its descriptors are already in flight)
            wbase += 32;
            pr = npr; rs = nrs; re = nre; bv = nbv;
            npr = pr2;
            desc(wbase + 32, npr, nrs, nre, nbv);
            pr2 = load_pr(wbase + 64);
        }
        const int cur = static_cast<int>(t - wbase);
        const int64_t wend = (wbase + 32 < fe) ? wbase + 32 : fe;
        const int ra = static_cast<int>(wend - t);  // rows of bucket fj left in this window (>= 1)
        const bool inr = lane >= cur && lane < cur + ra;
        const int64_t skip = (lane == cur) ? roff : 0;
        const int64_t rem = re - rs - skip;
        // pair counts clamped to kCsrSP + 1 (a longer row is taken in kCsrSP slices), inclusive scan
        int cnt = inr ? static_cast<int>(rem < kCsrSP + 1 ? rem : kCsrSP + 1) : 0;
        int inc = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        const int first = __shfl_sync(0xffffffffu, cnt, cur);
        const bool partial = first > kCsrSP;  // a slice of the (long) row at cur
        const int k = partial ? 0 : __popc(__ballot_sync(0xffffffffu, inr && inc <= kCsrSP));  // whole rows
        const int P = partial ? kCsrSP : __shfl_sync(0xffffffffu, inc, cur + k - 1);
        const bool mine = lane >= cur && lane < cur + (partial ? 1 : k);
        const int mcnt = mine ? (partial ? kCsrSP : cnt) : 0;
        const int moff = inc - cnt;  // first stage slot of this lane's row
        const int64_t mstart = rs + skip;
        const bool neg = pr < 0;
        double *sv = reinterpret_cast<double *>(stg + slot * kCsrStageBytes);
        int32_t *sc = reinterpret_cast<int32_t *>(stg + slot * kCsrStageBytes + kCsrSP * 8);
        unsigned char *sg = stg + slot * kCsrStageBytes + kCsrSP * 12;
        const int maxc = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(mcnt)));
        if (maxc <= 32) {
            // short rows: lane r gathers the pairs of its own row (pair kk of every row per step;
            // .ca: a row's later pairs come from the line the first one brought into L1)
            const uint32_t dv = smem_u32(sv + moff), dc = smem_u32(sc + moff);
            const double *gv = val + mstart;
            const int32_t *gc = col + mstart;
            unsigned char *gs = sg + moff;
            const unsigned char ngb = neg ? 1 : 0;
            for (int kk = 0; kk < maxc; ++kk) {
                if (kk < mcnt) {
                    CSK_DCHECK(moff + kk < kCsrSP && mstart + kk < row_ptr[m]);
                    cp_async8(dv + 8u * kk, gv + kk);
                    cp_async4(dc + 4u * kk, gc + kk);
                    gs[kk] = ngb;
                }
            }
        } else {
            // long rows: the warp strides over one row at a time
            for (int r = cur; r < cur + (partial ? 1 : k); ++r) {
                const int64_t s0 = __shfl_sync(0xffffffffu, mstart, r);
                const int c0 = __shfl_sync(0xffffffffu, mcnt, r);
                const int o0 = __shfl_sync(0xffffffffu, moff, r);
                const bool ng = __shfl_sync(0xffffffffu, neg, r);
                for (int q = lane; q < c0; q += 32) {
                    cp_async8(smem_u32(sv + o0 + q), val + s0 + q);
                    cp_async4(smem_u32(sc + o0 + q), col + s0 + q);
                    sg[o0 + q] = ng ? 1 : 0;
                }
            }
        }
        // b~: the rows that START in this batch, ascending (the oracle's fold order); the
        // shuffles are batched ahead of the dependent adds
        const double bs = neg ? -bv : bv;
        const int rf = roff > 0 ? cur + 1 : cur, rl = partial ? cur + 1 : cur + k;
        for (int r0 = rf; r0 < rl; r0 += 8) {
            double bb[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) bb[u] = __shfl_sync(0xffffffffu, bs, (r0 + u) & 31);
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (r0 + u < rl) bacc = bacc + bb[u];
        }
        if (partial) {
            roff += kCsrSP;
        } else {
            t += k;
            roff = 0;
        }
        const int64_t jb = fj;
        const bool end = (t == fe);
        if (end) {
            if (lane == 0) bt[fj] = bacc;
            bacc = 0.0;
            ++fj;
            if (fj < je) fe = end_of(fj);
            while (fj < je && fe == t) {
                zero_row(fj);
                ++fj;
                if (fj < je) fe = end_of(fj);
            }
        }
        if (lane == 0) {
            meta[slot * 4 + 0] = static_cast<int>(P);
            meta[slot * 4 + 1] = static_cast<int>(jb);
            meta[slot * 4 + 2] = end ? 1 : 0;
        }
    };
    for (issued = 0;; ++issued) {
        const int slot = issued % kCsrS;
        if (issued >= kCsrS) mbar_wait(empty + slot, static_cast<uint32_t>(((issued / kCsrS) - 1) & 1));
        if (fj >= je) {
            finish(slot);
            break;
        }
        form(slot);
        cp_async_arrive_noinc(full + slot);  // the gathers of this lane
        mbar_arrive(full + slot);            // the meta / sign bytes of this lane (release)
    }
}

// S4 in the oracle's exact order (SURVEY §8(c) acceptance 2): nsq_j = fma-accumulated
// a_j0^2, a_j1^2, ... left to right from +0.0, one thread per row (the chain is sequential by
// definition; rows run in parallel).  The row streams through four 16-double register stages
// (16-byte loads): the loads of the stage three ahead are in flight while one stage is folded,
// so the n-long fma chain, not the load latency, bounds a thread.
__device__ __forceinline__ void norm_stage_load(const double *r, int64_t k, int64_t n, double2 (&v)[8]) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
        v[u] = (k + 2 * u + 1 < n) ? __ldg(reinterpret_cast<const double2 *>(r + k + 2 * u)) : make_double2(0.0, 0.0);
}
__device__ __forceinline__ double norm_stage_fold(const double2 (&v)[8], int64_t k, int64_t n, double acc) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        if (k + 2 * u + 1 < n) {  // (a zero pad would not change acc, but keep the chain exact: skip it)
            acc = __fma_rn(v[u].x, v[u].x, acc);
            acc = __fma_rn(v[u].y, v[u].y, acc);
        }
    }
    return acc;
}
__global__ void __launch_bounds__(32) k_row_norms_exact(const double *__restrict__ At, int64_t d, int64_t n,
                                                        double *__restrict__ nsq) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= d) return;
    const double *r = At + j * n;
    double acc = 0.0;
    int64_t k = 0;
    if ((reinterpret_cast<uintptr_t>(r) & 15) == 0 && n >= 64) {
        const int64_t ne = n & ~int64_t(15);  // whole 16-double stages
        double2 s0[8], s1[8], s2[8], s3[8];
        norm_stage_load(r, 0, ne, s0);
        norm_stage_load(r, 16, ne, s1);
        norm_stage_load(r, 32, ne, s2);
        norm_stage_load(r, 48, ne, s3);
        for (; k < ne; k += 64) {
            acc = norm_stage_fold(s0, k, ne, acc);
            norm_stage_load(r, k + 64, ne, s0);
            acc = norm_stage_fold(s1, k + 16, ne, acc);
            norm_stage_load(r, k + 80, ne, s1);
            acc = norm_stage_fold(s2, k + 32, ne, acc);
            norm_stage_load(r, k + 96, ne, s2);
            acc = norm_stage_fold(s3, k + 48, ne, acc);
            norm_stage_load(r, k + 112, ne, s3);
        }
        k = ne;
    }
    for (; k < n; ++k) {
        const double v = __ldg(r + k);
        acc = __fma_rn(v, v, acc);
    }
    nsq[j] = acc;
}

#ifndef CSK_NORM_COLS
#define CSK_NORM_COLS 64
#endif
#ifndef CSK_NORM_STAGES
#define CSK_NORM_STAGES 4
#endif
// The same chains with the rows staged through shared memory: CTA = one warp = 32 consecutive
// rows, lane l the chain of row r0 + l.  A stage holds kNC = 64 columns of the 32 rows, copied by
// cp.async (LDGSTS, 16 bytes per lane: one coalesced 512-byte row chunk per warp instruction);
// the stage's mbarrier completes when every lane's copies have landed
// (cp.async.mbarrier.arrive.noinc), and kNS stages are in flight, so the HBM stream runs ahead of
// the chains.  (One 1-D bulk copy per row chunk instead was bound by the TMA issue rate for
// 512-byte copies: C3 16 us, C5 131 us.)  Rows sit kNP doubles apart, kNP / 2 odd: the 32 lanes'
// 16-byte reads of one column pair fall in distinct bank groups (4 wavefronts for 512 bytes, the
// minimum).  Needs n even and a 16-byte aligned A~.
constexpr int kNC = CSK_NORM_COLS, kNS = CSK_NORM_STAGES, kNP = kNC + 2;
static_assert((kNP / 2) % 2 == 1, "conflict-free row stride");
static_assert(kNC == 64, "one 16-byte copy per lane per row chunk");
constexpr size_t kNormSmem = static_cast<size_t>(kNS) * 32 * kNP * 8 + kNS * 8;
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__global__ void __launch_bounds__(32) k_row_norms_staged(const double *__restrict__ At, int64_t d, int64_t n,
                                                         double *__restrict__ nsq) {
    extern __shared__ __align__(16) unsigned char norm_smem[];
    double *buf = reinterpret_cast<double *>(norm_smem);  // [kNS][32][kNP]
    uint64_t *full = reinterpret_cast<uint64_t *>(norm_smem + static_cast<size_t>(kNS) * 32 * kNP * 8);
    const int lane = threadIdx.x;
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32;
    const int rows = static_cast<int>(d - r0 < 32 ? d - r0 : 32);
    const bool act = lane < rows;
    const int nch = static_cast<int>((n + kNC - 1) / kNC);
    if (lane == 0) {
        for (int q = 0; q < kNS; ++q) mbar_init(full + q, 32);
        fence_mbar_init();
    }
    __syncwarp();
    auto issue = [&](int ch) {
        const int st = ch % kNS;
        const int64_t c0 = static_cast<int64_t>(ch) * kNC;
        const int cw = static_cast<int>(n - c0 < kNC ? n - c0 : kNC);
        if (2 * lane < cw) {
            const double *src = At + r0 * n + c0 + 2 * lane;
            const uint32_t dst = smem_u32(buf + static_cast<size_t>(st) * 32 * kNP + 2 * lane);
            for (int r = 0; r < rows; ++r) cp_async16(dst + static_cast<uint32_t>(r * kNP * 8), src + r * n);
        }
        cp_async_arrive_noinc(full + st);
    };
    for (int ch = 0; ch < kNS && ch < nch; ++ch) issue(ch);
    double acc = 0.0;
    for (int ch = 0; ch < nch; ++ch) {
        const int st = ch % kNS;
        mbar_wait(full + st, static_cast<uint32_t>((ch / kNS) & 1));
        const int cw = static_cast<int>(n - static_cast<int64_t>(ch) * kNC < kNC ? n - static_cast<int64_t>(ch) * kNC : kNC);
        const double2 *rp = reinterpret_cast<const double2 *>(buf + (static_cast<size_t>(st) * 32 + lane) * kNP);
        if (act) {
            if (cw == kNC) {
                // the next pair's load is issued before this pair's two fmas (the chain, not the
                // shared-memory latency, sets the pace)
                double2 v = rp[0];
#pragma unroll
                for (int u = 0; u < kNC / 2; ++u) {
                    const double2 w = rp[u + 1 < kNC / 2 ? u + 1 : u];
                    acc = __fma_rn(v.x, v.x, acc);
                    acc = __fma_rn(v.y, v.y, acc);
                    v = w;
                }
            } else {
                for (int u = 0; u < cw / 2; ++u) {
                    const double2 v = rp[u];
                    acc = __fma_rn(v.x, v.x, acc);
                    acc = __fma_rn(v.y, v.y, acc);
                }
            }
        }
        __syncwarp();  // every lane is done with stage st before it is refilled
        if (ch + kNS < nch) issue(ch + kNS);
    }
    if (act) nsq[r0 + lane] = acc;
}

}  // namespace

int norm_team_threads(int64_t n) { return dense_geom(n, true).tc; }

csk_status_t launch_sketch_dense(csk_ctx_t ctx, const double *A, int64_t lda, const double *b,
                                 int64_t m, int64_t n, int64_t d, const int32_t *perm,
                                 const int32_t *offsets, double *At, double *bt, double *nsq,
                                 cudaStream_t stream) {
    const bool tma = aligned16(A) && (lda % 2 == 0);
    const DenseGeom g = dense_geom(n, tma);
    static const bool no_wpb = getenv("CSK_SKETCH_NO_WPB") != nullptr;
    if (n <= 256 && !no_wpb) {  // short rows: warp per bucket
        const int tcw = g.tc / 32;  // the standalone norm team (k_row_norms) in warps
        const int V = static_cast<int>((n + 63) / 64);
        const int64_t grid = int64_t(ctx->num_sms) * 2;  // persistent, 16 warps per SM
        time_mark(ctx, 0, false, stream);
#define CSK_WPB(VV)                                                                                       \
        if (tma) k_sketch_dense_wpb<VV, true><<<static_cast<int>(grid), 256, 0, stream>>>(                 \
            A, lda, b, m, n, d, perm, offsets, At, bt, tcw);                                              \
        else k_sketch_dense_wpb<VV, false><<<static_cast<int>(grid), 256, 0, stream>>>(                   \
            A, lda, b, m, n, d, perm, offsets, At, bt, tcw);
        switch (V) {
            case 1: CSK_WPB(1) break;
            case 2: CSK_WPB(2) break;
            case 3: CSK_WPB(3) break;
            default: CSK_WPB(4) break;
        }
#undef CSK_WPB
        time_mark(ctx, 0, true, stream);
        CSK_CUDA(ctx, cudaGetLastError());
        return nsq ? launch_row_norms(ctx, At, d, n, nsq, stream) : CSK_OK;  // S4, the oracle's order
    }
    int grid = ctx->num_sms;
    if (grid > d) grid = static_cast<int>(d);
    const int threads = g.tc + 64;
#define CSK_LAUNCH_DENSE_RB(PP, T, R)                                                                   \
    {                                                                                                   \
        CSK_CHECK(raise_smem(ctx, reinterpret_cast<const void *>(k_sketch_dense<PP, T, R>)));           \
        time_mark(ctx, 0, false, stream);                                                              \
        k_sketch_dense<PP, T, R><<<grid, threads, g.smem, stream>>>(                                    \
            A, lda, b, m, n, d, perm, offsets, At, bt, g.tc, g.chunk_cols, g.chunks,                    \
            g.slot_bytes, g.rb, g.stages, static_cast<int>(g.header));                                  \
    }
#define CSK_LAUNCH_DENSE(PP, T)                                        \
    {                                                                  \
        if (T && g.rb == 2) CSK_LAUNCH_DENSE_RB(PP, T, 2)              \
        else if (T && g.rb == 4) CSK_LAUNCH_DENSE_RB(PP, T, 4)         \
        else if (T && g.rb >= 8) CSK_LAUNCH_DENSE_RB(PP, T, 8)         \
        else CSK_LAUNCH_DENSE_RB(PP, T, 1)                             \
    }
    switch (g.p * 2 + (tma ? 1 : 0)) {
        case 3: CSK_LAUNCH_DENSE(1, true) break;
        case 2: CSK_LAUNCH_DENSE(1, false) break;
        case 5: CSK_LAUNCH_DENSE(2, true) break;
        case 4: CSK_LAUNCH_DENSE(2, false) break;
        case 9: CSK_LAUNCH_DENSE(4, true) break;
        case 8: CSK_LAUNCH_DENSE(4, false) break;
        default: return fail(ctx, CSK_E_UNSUPPORTED, "sketch geometry");
    }
#undef CSK_LAUNCH_DENSE
#undef CSK_LAUNCH_DENSE_RB
    time_mark(ctx, 0, true, stream);
    CSK_CUDA(ctx, cudaGetLastError());
    return nsq ? launch_row_norms(ctx, At, d, n, nsq, stream) : CSK_OK;  // S4, the oracle's order
}

csk_status_t launch_row_norms(csk_ctx_t ctx, const double *At, int64_t d, int64_t n, double *nsq,
                              cudaStream_t stream) {
    // S4 in the oracle's order (bit-exact): one thread per row, sequential fma chain; the rows
    // staged through shared memory when they are 16-byte aligned (n even), else read by the threads
    static const bool plain = getenv("CSK_NORMS_PLAIN") != nullptr;  // A/B
    const unsigned grid = static_cast<unsigned>((d + 31) / 32);
    if (!plain && n % 2 == 0 && aligned16(At)) {
        CSK_CHECK(raise_smem(ctx, reinterpret_cast<const void *>(k_row_norms_staged)));
        k_row_norms_staged<<<grid, 32, kNormSmem, stream>>>(At, d, n, nsq);
    } else {
        k_row_norms_exact<<<grid, 32, 0, stream>>>(At, d, n, nsq);
    }
    CSK_CUDA(ctx, cudaGetLastError());
    return CSK_OK;
}

csk_status_t launch_sketch_csr(csk_ctx_t ctx, const int64_t *row_ptr, const int32_t *col,
                               const double *val, const double *b, int64_t m, int64_t n,
                               int64_t d, const int32_t *perm, const int32_t *offsets,
                               double *At, double *bt, double *nsq, cudaStream_t stream) {
    const int64_t stride = (n + 1) & ~int64_t(1);  // accumulator doubles (16-byte multiple)
    const int64_t stampb = (n + 15) & ~int64_t(15);  // conflict stamps: one byte per column
    const int64_t wb = ((stride * 8 + stampb + kCsrS * kCsrStageBytes + kCsrMetaBytes) + 127) & ~int64_t(127);
    int pairs = static_cast<int>(ctx->max_smem_optin / wb);  // producer / consumer warp pairs per CTA
    if (pairs > kCsrMaxWarps / 2) pairs = kCsrMaxWarps / 2;
    if (pairs < 1) return fail(ctx, CSK_E_UNSUPPORTED, "csk_sketch_csr: n too large for shared accumulators");
    const int warps = 2 * pairs;
    const size_t smem = static_cast<size_t>(pairs) * wb;
    CSK_CHECK(raise_smem(ctx, reinterpret_cast<const void *>(k_sketch_csr)));
    const int vec = (n % 2 == 0 && aligned16(At)) ? 1 : 0;
    // experiment knob: the L2 fetch granularity for the random (col, val) / row_ptr / b gathers
    static const char *gran = getenv("CSK_L2_FETCH_GRAN");
    if (gran) CSK_CUDA(ctx, cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, static_cast<size_t>(atoi(gran))));
    time_mark(ctx, 0, false, stream);
    k_sketch_csr<<<ctx->num_sms, warps * 32, smem, stream>>>(row_ptr, col, val, b, m, n, d, perm, offsets, At, bt,
                                                            stride, static_cast<int>(stampb), static_cast<int>(wb), vec);
    time_mark(ctx, 0, true, stream);
    CSK_CUDA(ctx, cudaGetLastError());
    return nsq ? launch_row_norms(ctx, At, d, n, nsq, stream) : CSK_OK;  // S4, the oracle's order
}

}  // namespace csk
