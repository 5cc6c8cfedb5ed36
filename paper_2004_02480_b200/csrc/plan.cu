// plan.cu -- S1 hash and S2 stable bucketing of rows (the count-sketch "plan").
//
// Definition 1: S = Phi D, Phi_{h(i),i} = 1, D = diag(+-1), h uniform
// on [d].  h and D come from the counter form of SplitMix64 (reading R-1 of
// DESIGN.md): z_h = SM64(seed, 2c), z_s = SM64(seed, 2c+1) for GLOBAL row c,
// h = floor(z_h * d / 2^64) (one UMULHI), sign = top bit of z_s.
//
// Bucketing (S2): perm lists the rows grouped by bucket, ascending row index inside each
// bucket -- the order Algorithm 1's sketch sums in; offsets[j] = first position of
// bucket j, offsets[d] = m.  Default: the one-launch counting plan k_plan_fused below.  Only
// when buckets average > 512 rows (m > 512 d, e.g. d = 1) a stable LSD radix sort of
// (key = h, value = row | sign<<31) (CUB onesweep) is used instead.
#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>

#include "csk_internal.cuh"

namespace csk {

__global__ void k_hash_keys(uint64_t seed, int64_t row_offset, int32_t m, uint32_t d,
                            uint32_t *keys, uint32_t *vals, int32_t *h_out, int8_t *sign_out) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        const uint64_t c = static_cast<uint64_t>(row_offset) + static_cast<uint64_t>(i);
        const uint64_t zh = sm64(seed, 2 * c);
        const uint64_t zs = sm64(seed, 2 * c + 1);
        const uint32_t h = static_cast<uint32_t>(__umul64hi(zh, static_cast<uint64_t>(d)));
        const uint32_t neg = static_cast<uint32_t>(zs >> 63);
        if (keys) {
            keys[i] = h;
            vals[i] = static_cast<uint32_t>(i) | (neg << 31);
        }
        if (h_out) h_out[i] = static_cast<int32_t>(h);
        if (sign_out) sign_out[i] = neg ? int8_t(-1) : int8_t(1);
    }
}

__global__ void k_map_keys(const int32_t *h, const int8_t *sign, int32_t m, int32_t d,
                           uint32_t *keys, uint32_t *vals, int *bad) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        const int32_t hi = h[i];
        const int8_t si = sign[i];
        if (hi < 0 || hi >= d || (si != 1 && si != -1)) {
            atomicExch(bad, 1);
        }
        keys[i] = static_cast<uint32_t>(hi < 0 ? 0 : (hi >= d ? d - 1 : hi));
        vals[i] = static_cast<uint32_t>(i) | (si < 0 ? 0x80000000u : 0u);
    }
}

// offsets[j] = lower_bound(sorted_keys, j) for j in [0, d]; each j written exactly once.
__global__ void k_offsets(const uint32_t *sorted_keys, int32_t m, int32_t d, int32_t *offsets) {
    for (int32_t t = blockIdx.x * blockDim.x + threadIdx.x; t <= m; t += gridDim.x * blockDim.x) {
        const int32_t prev = t > 0 ? static_cast<int32_t>(sorted_keys[t - 1]) : -1;
        const int32_t cur = t < m ? static_cast<int32_t>(sorted_keys[t]) : d;
        for (int32_t j = prev + 1; j <= cur; ++j) offsets[j] = t;
    }
}

// One-launch plan (the default): a cooperative kernel over G CTAs (one per SM; fewer for small m).
//   P1  count[h(i)] += 1 for every row (global atomics; count zeroed by the caller); with an
//       explicit map (csk_sketch_with_map, the routing receiver) h/sign are read and validated
//   P2  offsets = exclusive scan of count: CTA c scans its slice of the d counts, the CTA
//       totals are added in CTA order; cursor = offsets
//   P3  perm[atomicAdd(cursor[h(i)], 1)] = i | sign << 31   (arbitrary order within a bucket)
//   P4  each bucket's segment sorted by row (warp bitonic sort per bucket; rows are distinct
//       keys, so the result is unique: exactly the stable order a radix sort produces)
// Four grid barriers in one launch instead of the ~6 launches (and their gaps) of a radix sort.
// Warp bitonic sort of N = 32 EPL unsigned keys (element g = lane EPL + e), ascending.
template <int EPL>
__device__ __forceinline__ void warp_bitonic(uint32_t (&v)[EPL], int lane) {
#pragma unroll
    for (int k = 2; k <= 32 * EPL; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= EPL) {  // partner in lane ^ (j / EPL), same slot
                const int lj = j / EPL;
                const bool lower = (lane & lj) == 0;
#pragma unroll
                for (int e = 0; e < EPL; ++e) {
                    const uint32_t o = __shfl_xor_sync(0xffffffffu, v[e], lj);
                    const bool up = ((lane * EPL + e) & k) == 0;
                    v[e] = (lower == up) ? min(v[e], o) : max(v[e], o);
                }
            } else {  // partner slot e | j in this lane
#pragma unroll
                for (int e = 0; e < EPL; ++e) {
                    if ((e & j) == 0) {
                        const bool up = ((lane * EPL + e) & k) == 0;
                        const uint32_t a = v[e], b = v[e | j];
                        v[e] = up ? min(a, b) : max(a, b);
                        v[e | j] = up ? max(a, b) : min(a, b);
                    }
                }
            }
        }
    }
}

// One bucket segment perm[a, a + sz) (sz <= 32 EPL) sorted by row: the entry is rotated so the
// row index is in the high 31 bits and the sign bit in bit 0 (distinct rows: a total order).
template <int EPL>
__device__ __forceinline__ void sort_segment(int32_t *perm, int32_t a, int32_t sz, int lane) {
    uint32_t v[EPL];
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
        const int g = lane * EPL + e;
        const uint32_t x = g < sz ? static_cast<uint32_t>(perm[a + g]) : 0xffffffffu;
        v[e] = g < sz ? ((x << 1) | (x >> 31)) : 0xffffffffu;
    }
    warp_bitonic<EPL>(v, lane);
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
        const int g = lane * EPL + e;
        if (g < sz) perm[a + g] = static_cast<int32_t>((v[e] >> 1) | (v[e] << 31));
    }
}

constexpr int kPlanThreads = 512;
constexpr int kPlanDirtyCap = 1024;  // k_plan_hist: listed (bucket, CTA) groups per CTA
constexpr int kPlanColPer = 8;       // k_plan_hist P2a, warp per bucket: CTAs per lane (G <= 256)
__global__ void __launch_bounds__(kPlanThreads, 1)
k_plan_fused(uint64_t seed, int64_t row_offset, int32_t m, uint32_t d, const int32_t *h_in, const int8_t *sign_in,
             int32_t *count, int32_t *cursor, int32_t *offsets, int32_t *perm, int32_t *scratch, int32_t *ctot,
             int *bad) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ int32_t wsum[32];
    __shared__ int32_t sbase;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t gtid = static_cast<int64_t>(blockIdx.x) * blockDim.x + tid;
    const int64_t gthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
    auto bucket = [&](int32_t i, uint32_t &neg) -> uint32_t {
        if (h_in) {
            const int32_t hi = h_in[i];
            const int8_t si = sign_in[i];
            neg = si < 0 ? 1u : 0u;
            if (hi < 0 || hi >= static_cast<int32_t>(d) || (si != 1 && si != -1)) {
                *bad = 1;
                return hi < 0 ? 0u : d - 1u;
            }
            return static_cast<uint32_t>(hi);
        }
        const uint64_t c = static_cast<uint64_t>(row_offset) + static_cast<uint64_t>(i);
        neg = static_cast<uint32_t>(sm64(seed, 2 * c + 1) >> 63);
        return static_cast<uint32_t>(__umul64hi(sm64(seed, 2 * c), static_cast<uint64_t>(d)));
    };
    // P1
    for (int64_t i = gtid; i < m; i += gthreads) {
        uint32_t neg;
        atomicAdd(count + bucket(static_cast<int32_t>(i), neg), 1);
    }
    grid.sync();
    // P2: CTA c scans the counts [j0, j1) (each thread a contiguous run, block scan of the runs)
    const int64_t G = gridDim.x;
    const int64_t j0 = static_cast<int64_t>(d) * blockIdx.x / G, j1 = static_cast<int64_t>(d) * (blockIdx.x + 1) / G;
    const int64_t per = (j1 - j0 + kPlanThreads - 1) / kPlanThreads;
    const int64_t r0 = j0 + per * tid, r1 = (r0 + per < j1) ? r0 + per : j1;
    int32_t run = 0;
    for (int64_t j = r0; j < r1; ++j) run += count[j];
    int32_t incl = run;  // inclusive warp scan, then warps
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int32_t w = lane < kPlanThreads / 32 ? wsum[lane] : 0, wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        wsum[lane] = wi - w;  // exclusive over warps
        if (lane == 31) ctot[blockIdx.x] = wi;  // this CTA's total
    }
    __syncthreads();
    const int32_t local = wsum[warp] + incl - run;
    grid.sync();
    if (tid == 0) {  // base of this CTA's slice: the totals of the CTAs before it, in CTA order
        int32_t bsum = 0;
        for (int c = 0; c < static_cast<int>(blockIdx.x); ++c) bsum += ctot[c];
        sbase = bsum;
    }
    __syncthreads();
    int32_t base = sbase + local;
    for (int64_t j = r0; j < r1; ++j) {
        offsets[j] = base;
        cursor[j] = base;
        base += count[j];
    }
    if (gtid == 0) offsets[d] = m;
    if (blockIdx.x == gridDim.x - 1 && tid == kPlanThreads - 1) CSK_DCHECK(base == m || r1 < j1);  // counts sum to m
    grid.sync();
    // P3 (four rows per thread per step: four cursor round trips in flight)
    for (int64_t i0 = gtid; i0 < m; i0 += 4 * gthreads) {
        uint32_t hh[4], ng[4];
        int32_t pos[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = i0 + u * gthreads;
            hh[u] = i < m ? bucket(static_cast<int32_t>(i), ng[u]) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (i0 + u * gthreads < m) pos[u] = atomicAdd(cursor + hh[u], 1);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = i0 + u * gthreads;
            if (i < m) {
                CSK_DCHECK(pos[u] >= 0 && pos[u] < m && hh[u] < d);
                perm[pos[u]] = static_cast<int32_t>(static_cast<uint32_t>(i) | (ng[u] << 31));
            }
        }
    }
    grid.sync();
    // P4: sort each bucket by row (keys distinct): a warp bitonic sort in registers for up to
    // 1024 rows, a rank sort through global scratch beyond (degenerate inputs only)
    const int64_t gw = gtid >> 5, nw = gthreads >> 5;
    for (int64_t j = gw; j < d; j += nw) {
        const int32_t a = offsets[j], e = offsets[j + 1], sz = e - a;
        if (sz <= 1) continue;
        if (sz <= 32) sort_segment<1>(perm, a, sz, lane);
        else if (sz <= 64) sort_segment<2>(perm, a, sz, lane);
        else if (sz <= 128) sort_segment<4>(perm, a, sz, lane);
        else if (sz <= 256) sort_segment<8>(perm, a, sz, lane);
        else if (sz <= 512) sort_segment<16>(perm, a, sz, lane);
        else if (sz <= 1024) sort_segment<32>(perm, a, sz, lane);
        else {
            for (int t = lane; t < sz; t += 32) scratch[a + t] = perm[a + t];
            __syncwarp();
            __threadfence_block();
            const int32_t *src = scratch + a;
            for (int t = lane; t < sz; t += 32) {
                const int32_t v = src[t], key = v & 0x7fffffff;
                int32_t rank = 0;
                for (int u = 0; u < sz; ++u) rank += (src[u] & 0x7fffffff) < key ? 1 : 0;
                perm[a + rank] = v;
            }
            __syncwarp();
        }
    }
}


// Histogram plan (default when the d bucket counts fit in shared memory): CTA c owns the
// contiguous rows [c m/G, (c+1) m/G).  Because a CTA's rows are consecutive, placing every
// (bucket, CTA) group after the groups of lower CTAs already yields ascending rows inside each
// bucket; only rows of one CTA that share a bucket need ordering, and those groups are tiny.
//   P1  per-CTA histogram of its rows' buckets in shared memory (shared atomics), stored as
//       hist[c][j] (coalesced)
//   P2  hist[c][j] := sum_{c' < c} hist[c'][j] (column prefix, one thread per bucket), bucket
//       totals -> offsets by the multi-CTA scan of k_plan_fused
//   P3  cursors in shared memory start at offsets[j] + hist[c][j]; rows take slots chunk by
//       chunk in row order (warp-ranked by __match_any_sync, one shared atomic per bucket per
//       warp), and only the (bucket, CTA) groups two warps of one chunk claimed are sorted
// Three grid barriers, no global atomics, no per-bucket sort pass.
__global__ void __launch_bounds__(kPlanThreads, 1)
k_plan_hist(uint64_t seed, int64_t row_offset, int32_t m, uint32_t d, const int32_t *h_in, const int8_t *sign_in,
            int32_t *hist, int32_t *count, int32_t *offsets, int32_t *perm, int32_t *ctot, int *bad) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ int32_t sh[];  // [d]: histogram, then cursors
    __shared__ int32_t wsum[32];
    __shared__ int32_t sbase;
    __shared__ int32_t ndirty;
    __shared__ int32_t dirty[kPlanDirtyCap];  // buckets whose group needs the row-order sort
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x;
    const int64_t gtid = static_cast<int64_t>(c) * blockDim.x + tid;
    const int64_t gthreads = static_cast<int64_t>(G) * blockDim.x;
    const int32_t i0 = static_cast<int32_t>(static_cast<int64_t>(m) * c / G);
    const int32_t i1 = static_cast<int32_t>(static_cast<int64_t>(m) * (c + 1) / G);
    auto bucket = [&](int32_t i, uint32_t &neg) -> uint32_t {
        if (h_in) {
            const int32_t hi = h_in[i];
            const int8_t si = sign_in[i];
            neg = si < 0 ? 1u : 0u;
            if (hi < 0 || hi >= static_cast<int32_t>(d) || (si != 1 && si != -1)) {
                *bad = 1;
                return hi < 0 ? 0u : d - 1u;
            }
            return static_cast<uint32_t>(hi);
        }
        const uint64_t cc = static_cast<uint64_t>(row_offset) + static_cast<uint64_t>(i);
        neg = static_cast<uint32_t>(sm64(seed, 2 * cc + 1) >> 63);
        return static_cast<uint32_t>(__umul64hi(sm64(seed, 2 * cc), static_cast<uint64_t>(d)));
    };
    // P1
    for (int64_t j = tid; j < d; j += kPlanThreads) sh[j] = 0;
    __syncthreads();
    for (int32_t i = i0 + tid; i < i1; i += kPlanThreads) {
        uint32_t neg;
        atomicAdd(&sh[bucket(i, neg)], 1);
    }
    __syncthreads();
    int32_t *hc = hist + static_cast<int64_t>(c) * d;
    for (int64_t j = tid; j < d; j += kPlanThreads) hc[j] = sh[j];
    grid.sync();
    // P2a: column prefix over the CTAs, bucket totals.  Few buckets (d <= threads / 32): a warp
    // per bucket, lane l the CTAs [l per, (l+1) per) (one round of loads, a warp scan); else a
    // thread per bucket walking the G CTAs with 16 loads in flight
    if (static_cast<int64_t>(d) * 32 <= gthreads && G <= 32 * kPlanColPer) {
        const int per = (G + 31) / 32;
        for (int64_t j = gtid >> 5; j < d; j += gthreads >> 5) {
            int32_t v[kPlanColPer];
            int32_t run = 0;
#pragma unroll
            for (int u = 0; u < kPlanColPer; ++u) {
                const int cq = lane * per + u;
                v[u] = (u < per && cq < G) ? hist[static_cast<int64_t>(cq) * d + j] : 0;
                run += v[u];
            }
            int32_t incl = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            int32_t ex = incl - run;
#pragma unroll
            for (int u = 0; u < kPlanColPer; ++u) {
                const int cq = lane * per + u;
                if (u < per && cq < G) hist[static_cast<int64_t>(cq) * d + j] = ex;
                ex += v[u];
            }
            if (lane == 31) count[j] = incl;
        }
    } else
    // thread per bucket; consecutive warps of buckets go to consecutive CTAs (warp-major over the
    // grid), so the d / 32 busy warps spread over every SM instead of filling the first few CTAs
    for (int64_t j = ((static_cast<int64_t>(warp) * G + c) << 5) + lane; j < d; j += gthreads) {
        int32_t run = 0;
        for (int q0 = 0; q0 < G; q0 += 16) {  // 16 loads in flight, then the prefix and the stores
            int32_t v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) v[u] = q0 + u < G ? hist[static_cast<int64_t>(q0 + u) * d + j] : 0;
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                if (q0 + u < G) hist[static_cast<int64_t>(q0 + u) * d + j] = run;
                run += v[u];
            }
        }
        count[j] = run;
    }
    grid.sync();
    // P2b: offsets = exclusive scan of the totals (CTA c scans its slice, CTA totals in order)
    const int64_t j0 = static_cast<int64_t>(d) * c / G, j1 = static_cast<int64_t>(d) * (c + 1) / G;
    const int64_t per = (j1 - j0 + kPlanThreads - 1) / kPlanThreads;
    const int64_t r0 = j0 + per * tid, r1 = (r0 + per < j1) ? r0 + per : j1;
    int32_t run = 0;
    for (int64_t j = r0; j < r1; ++j) run += count[j];
    int32_t incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int32_t w = lane < kPlanThreads / 32 ? wsum[lane] : 0, wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        wsum[lane] = wi - w;
        if (lane == 31) ctot[c] = wi;
    }
    __syncthreads();
    const int32_t local = wsum[warp] + incl - run;
    grid.sync();
    if (warp == 0) {  // base of this CTA's slice: the totals of the CTAs before it (a warp sum)
        int32_t bsum = 0;
        for (int q = lane; q < c; q += 32) bsum += ctot[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) bsum += __shfl_xor_sync(0xffffffffu, bsum, o);
        if (lane == 0) sbase = bsum;
    }
    __syncthreads();
    int32_t base = sbase + local;
    for (int64_t j = r0; j < r1; ++j) {
        offsets[j] = base;
        base += count[j];
    }
    if (gtid == 0) offsets[d] = m;
    grid.sync();
    // P3: this CTA's slots.  Rows are taken in chunks of kPlanThreads, in row order: inside a
    // warp, rows of one bucket get consecutive slots in lane (= row) order (__match_any_sync
    // ranks, one shared atomic per bucket per warp); chunks follow one another (a barrier), so
    // only two warps of one chunk claiming the same bucket can land out of row order.  The claim
    // detects that (its cursor moved since the chunk began) and lists the bucket; only the listed
    // (bucket, CTA) groups are sorted afterwards.  (A full list falls back to sorting every group.)
    for (int64_t j = tid; j < d; j += kPlanThreads) sh[j] = offsets[j] + hc[j];
    if (tid == 0) ndirty = 0;
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    for (int32_t base = i0; base < i1; base += kPlanThreads) {
        const int32_t i = base + tid;
        const bool valid = i < i1;
        uint32_t neg = 0u, h = 0u;
        if (valid) h = bucket(i, neg);
        const unsigned same = __match_any_sync(0xffffffffu, valid ? h : (0x80000000u | static_cast<uint32_t>(lane)));
        const int leader = __ffs(same) - 1;
        int32_t start = 0;
        if (valid && lane == leader) start = sh[h];
        __syncthreads();  // every warp has read its cursors before any warp claims
        int32_t pos = 0;
        if (valid && lane == leader) {
            pos = atomicAdd(&sh[h], __popc(same));
            if (pos != start) {
                const int q = atomicAdd(&ndirty, 1);
                if (q < kPlanDirtyCap) dirty[q] = static_cast<int32_t>(h);
            }
        }
        pos = __shfl_sync(0xffffffffu, pos, leader) + __popc(same & lt);
        if (valid) {
            CSK_DCHECK(pos >= 0 && pos < m);
            perm[pos] = static_cast<int32_t>(static_cast<uint32_t>(i) | (neg << 31));
        }
        __syncthreads();  // this chunk's claims are done before the next chunk reads its cursors
    }
    auto sort_group = [&](int32_t a, int32_t e) {  // insertion sort by row (rows are distinct)
        for (int32_t t = a + 1; t < e; ++t) {
            const int32_t v = perm[t], key = v & 0x7fffffff;
            int32_t s = t - 1;
            while (s >= a && (perm[s] & 0x7fffffff) > key) {
                perm[s + 1] = perm[s];
                --s;
            }
            perm[s + 1] = v;
        }
    };
    if (ndirty <= kPlanDirtyCap) {
        // the listed groups (a bucket may be listed more than once: the first to set the cursor's
        // sign bit sorts it)
        for (int q = tid; q < ndirty; q += kPlanThreads) {
            const int32_t j = dirty[q];
            const int32_t e = atomicOr(&sh[j], static_cast<int32_t>(0x80000000u));
            if (e < 0) continue;
            sort_group(offsets[j] + hc[j], e);
        }
    } else {
        for (int64_t j0 = tid; j0 < d; j0 += 8 * kPlanThreads) {
            int32_t ga[8], ge[8];  // group bounds of 8 buckets (their loads in flight together)
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t j = j0 + static_cast<int64_t>(u) * kPlanThreads;
                ga[u] = j < d ? offsets[j] + hc[j] : 0;
                ge[u] = j < d ? sh[j] : 0;
            }
#pragma unroll 1
            for (int u = 0; u < 8; ++u) sort_group(ga[u], ge[u]);
        }
    }
}

static int grid_for(int64_t items, int threads, int num_sms) {
    int64_t g = (items + threads - 1) / threads;
    const int64_t cap = static_cast<int64_t>(num_sms) * 16;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return static_cast<int>(g);
}

csk_status_t build_plan(csk_ctx_t ctx, uint64_t seed, int64_t row_offset, int64_t m, int64_t d,
                        const int32_t *h_in, const int8_t *sign_in, int32_t **perm_out,
                        int32_t **offsets_out, cudaStream_t stream) {
    const size_t mb = static_cast<size_t>(m) * 4;
    CSK_CHECK(ensure(ctx, ctx->keys_in, mb));
    CSK_CHECK(ensure(ctx, ctx->keys_out, mb));
    CSK_CHECK(ensure(ctx, ctx->vals_in, mb));
    CSK_CHECK(ensure(ctx, ctx->vals_out, mb));
    CSK_CHECK(ensure(ctx, ctx->offsets, static_cast<size_t>(d + 1) * 4));
    auto *keys_in = static_cast<uint32_t *>(ctx->keys_in.ptr);
    auto *keys_out = static_cast<uint32_t *>(ctx->keys_out.ptr);
    auto *vals_in = static_cast<uint32_t *>(ctx->vals_in.ptr);
    auto *vals_out = static_cast<uint32_t *>(ctx->vals_out.ptr);
    auto *offsets = static_cast<int32_t *>(ctx->offsets.ptr);
    const int threads = 256;
    const int grid = grid_for(m, threads, ctx->num_sms);

    // the one-launch plan (hand-written, deterministic) for every input whose buckets average
    // <= 512 rows (its per-bucket rank sort is quadratic in the bucket size); the CUB radix sort
    // only for the degenerate m >> d case (e.g. d = 1) or on request (CSK_PLAN_CUB=1, A/B)
    static const bool use_cub = getenv("CSK_PLAN_CUB") != nullptr;
    static const bool no_hist = getenv("CSK_PLAN_ATOMIC") != nullptr;  // A/B: the global-atomic plan
    // histogram plan: the d counts fit in shared memory and the CTA groups stay small
    const size_t hist_smem = static_cast<size_t>(d) * 4;
    if (!use_cub && !no_hist && hist_smem + 1024 + kPlanDirtyCap * 4 <= static_cast<size_t>(ctx->max_smem_optin) &&
        m <= 512 * d) {
        int G = static_cast<int>((m + 255) / 256);
        if (G > ctx->num_sms) G = ctx->num_sms;
        static const int gcap = getenv("CSK_PLAN_G") ? atoi(getenv("CSK_PLAN_G")) : 0;  // A/B knob
        if (gcap > 0 && G > gcap) G = gcap;
        if (G < 1) G = 1;
        CSK_CHECK(ensure(ctx, ctx->keys_in, static_cast<size_t>(d + 1) * 4 + 2 * static_cast<size_t>(ctx->num_sms) * 4 + 64));
        int32_t *count = static_cast<int32_t *>(ctx->keys_in.ptr);
        int32_t *ctot = count + d + 1;
        int *bad = reinterpret_cast<int *>(ctot + ctx->num_sms + 1);
        CSK_CHECK(ensure(ctx, ctx->cub_tmp, static_cast<size_t>(G) * d * 4));  // hist[G][d]
        int32_t *hist = static_cast<int32_t *>(ctx->cub_tmp.ptr);
        int32_t *perm = reinterpret_cast<int32_t *>(static_cast<uint32_t *>(ctx->vals_out.ptr));
        if (h_in) CSK_CUDA(ctx, cudaMemsetAsync(bad, 0, sizeof(int), stream));
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        cfg.gridDim = dim3(G);
        cfg.blockDim = dim3(kPlanThreads);
        cfg.dynamicSmemBytes = hist_smem;
        cfg.stream = stream;
        CSK_CHECK(raise_smem(ctx, reinterpret_cast<const void *>(k_plan_hist)));
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CSK_CUDA(ctx, cudaLaunchKernelEx(&cfg, k_plan_hist, seed, row_offset, static_cast<int32_t>(m),
                                         static_cast<uint32_t>(d), h_in, sign_in, hist, count, offsets, perm, ctot,
                                         bad));
        if (h_in) {
            int bad_h = 0;
            CSK_CUDA(ctx, cudaMemcpyAsync(&bad_h, bad, sizeof(int), cudaMemcpyDeviceToHost, stream));
            CSK_CUDA(ctx, cudaStreamSynchronize(stream));
            if (bad_h) return fail(ctx, CSK_E_ARG, "explicit map: h outside [0,d) or sign not +-1");
        }
        *perm_out = perm;
        *offsets_out = offsets;
        return CSK_OK;
    }
    if (!use_cub && m <= 512 * d) {
        CSK_CHECK(ensure(ctx, ctx->keys_in, static_cast<size_t>(d + 1) * 4 + 2 * static_cast<size_t>(ctx->num_sms) * 4 + 64));
        int32_t *count = static_cast<int32_t *>(ctx->keys_in.ptr);
        int32_t *ctot = count + d + 1;
        int *bad = reinterpret_cast<int *>(ctot + ctx->num_sms + 1);
        CSK_CHECK(ensure(ctx, ctx->vals_in, static_cast<size_t>(d > m ? d : m) * 4));
        int32_t *cursor = static_cast<int32_t *>(ctx->vals_in.ptr);
        int32_t *perm = reinterpret_cast<int32_t *>(vals_out);
        int32_t *scratch = reinterpret_cast<int32_t *>(keys_out);
        CSK_CUDA(ctx, cudaMemsetAsync(count, 0, static_cast<size_t>(d) * 4, stream));
        if (h_in) CSK_CUDA(ctx, cudaMemsetAsync(bad, 0, sizeof(int), stream));
        // grid: one CTA per SM, fewer for small m (a grid barrier over fewer CTAs is cheaper)
        int G = static_cast<int>((m + 255) / 256);
        if (G > ctx->num_sms) G = ctx->num_sms;
        if (G < 1) G = 1;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        cfg.gridDim = dim3(G);
        cfg.blockDim = dim3(kPlanThreads);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = stream;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CSK_CUDA(ctx, cudaLaunchKernelEx(&cfg, k_plan_fused, seed, row_offset, static_cast<int32_t>(m),
                                         static_cast<uint32_t>(d), h_in, sign_in, count, cursor, offsets, perm,
                                         scratch, ctot, bad));
        if (h_in) {
            int bad_h = 0;
            CSK_CUDA(ctx, cudaMemcpyAsync(&bad_h, bad, sizeof(int), cudaMemcpyDeviceToHost, stream));
            CSK_CUDA(ctx, cudaStreamSynchronize(stream));
            if (bad_h) return fail(ctx, CSK_E_ARG, "explicit map: h outside [0,d) or sign not +-1");
        }
        *perm_out = perm;
        *offsets_out = offsets;
        return CSK_OK;
    }
    if (h_in == nullptr) {
        k_hash_keys<<<grid, threads, 0, stream>>>(seed, row_offset, static_cast<int32_t>(m),
                                                  static_cast<uint32_t>(d), keys_in, vals_in,
                                                  nullptr, nullptr);
    } else {
        CSK_CHECK(ensure(ctx, ctx->flag, sizeof(int)));
        int *bad = static_cast<int *>(ctx->flag.ptr);
        CSK_CUDA(ctx, cudaMemsetAsync(bad, 0, sizeof(int), stream));
        k_map_keys<<<grid, threads, 0, stream>>>(h_in, sign_in, static_cast<int32_t>(m),
                                                 static_cast<int32_t>(d), keys_in, vals_in, bad);
        int bad_h = 0;
        CSK_CUDA(ctx, cudaMemcpyAsync(&bad_h, bad, sizeof(int), cudaMemcpyDeviceToHost, stream));
        CSK_CUDA(ctx, cudaStreamSynchronize(stream));
        if (bad_h) return fail(ctx, CSK_E_ARG, "explicit map: h outside [0,d) or sign not +-1");
    }
    CSK_CUDA(ctx, cudaGetLastError());

    int end_bit = 1;
    while ((int64_t(1) << end_bit) < d) ++end_bit;
    size_t tmp_bytes = 0;
    if (ctx->cub_key_m == m && ctx->cub_key_bits == end_bit) {
        tmp_bytes = ctx->cub_bytes;
    } else {
        CSK_CUDA(ctx, cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys_in, keys_out, vals_in,
                                                      vals_out, static_cast<int>(m), 0, end_bit,
                                                      stream));
        ctx->cub_key_m = m;
        ctx->cub_key_bits = end_bit;
        ctx->cub_bytes = tmp_bytes;
    }
    CSK_CHECK(ensure(ctx, ctx->cub_tmp, tmp_bytes));
    CSK_CUDA(ctx, cub::DeviceRadixSort::SortPairs(ctx->cub_tmp.ptr, tmp_bytes, keys_in, keys_out,
                                                  vals_in, vals_out, static_cast<int>(m), 0,
                                                  end_bit, stream));
    k_offsets<<<grid_for(m + 1, threads, ctx->num_sms), threads, 0, stream>>>(
        keys_out, static_cast<int32_t>(m), static_cast<int32_t>(d), offsets);
    CSK_CUDA(ctx, cudaGetLastError());
    *perm_out = reinterpret_cast<int32_t *>(vals_out);
    *offsets_out = offsets;
    return CSK_OK;
}

}  // namespace csk

using namespace csk;

extern "C" csk_status_t csk_hash(csk_ctx_t ctx, uint64_t seed, int64_t row_offset, int64_t m,
                                 int64_t d, int32_t *h, int8_t *sign, void *stream) {
    if (!ctx) return CSK_E_ARG;
    if (m < 0 || m >= (int64_t(1) << 31) || d < 1 || d >= (int64_t(1) << 31) || row_offset < 0)
        return fail(ctx, CSK_E_ARG, "csk_hash: need 0 <= m < 2^31, 1 <= d < 2^31, row_offset >= 0");
    if (m == 0) return CSK_OK;
    if (!h && !sign) return fail(ctx, CSK_E_ARG, "csk_hash: h and sign are both NULL");
    CSK_CUDA(ctx, cudaSetDevice(ctx->device));
    k_hash_keys<<<grid_for(m, 256, ctx->num_sms), 256, 0, as_stream(stream)>>>(
        seed, row_offset, static_cast<int32_t>(m), static_cast<uint32_t>(d), nullptr, nullptr, h,
        sign);
    CSK_CUDA(ctx, cudaGetLastError());
    return CSK_OK;
}

extern "C" csk_status_t csk_plan(csk_ctx_t ctx, uint64_t seed, int64_t row_offset, int64_t m,
                                 int64_t d, const int32_t *h_in, const int8_t *sign_in,
                                 int32_t *perm, int32_t *offsets, void *stream) {
    CSK_NVTX("csk_plan");
    if (!ctx) return CSK_E_ARG;
    if (m < 1 || m >= (int64_t(1) << 31) || d < 1 || d > m || row_offset < 0)
        return fail(ctx, CSK_E_ARG, "csk_plan: need 1 <= d <= m < 2^31");
    if ((h_in == nullptr) != (sign_in == nullptr))
        return fail(ctx, CSK_E_ARG, "csk_plan: h_in and sign_in must both be given or both NULL");
    if (!perm || !offsets) return fail(ctx, CSK_E_ARG, "csk_plan: null output");
    CSK_CUDA(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = as_stream(stream);
    int32_t *p = nullptr, *o = nullptr;
    CSK_CHECK(build_plan(ctx, seed, row_offset, m, d, h_in, sign_in, &p, &o, s));
    CSK_CUDA(ctx, cudaMemcpyAsync(perm, p, static_cast<size_t>(m) * 4, cudaMemcpyDeviceToDevice, s));
    CSK_CUDA(ctx, cudaMemcpyAsync(offsets, o, static_cast<size_t>(d + 1) * 4,
                                  cudaMemcpyDeviceToDevice, s));
    return CSK_OK;
}
