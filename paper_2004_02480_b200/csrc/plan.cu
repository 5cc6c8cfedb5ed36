// plan.cu -- S1 hash and S2 stable bucketing of rows (the count-sketch "plan").
//
// Definition 1: S = Phi D, Phi_{h(i),i} = 1, D = diag(+-1), h uniform
// on [d].  h and D come from the counter form of SplitMix64 (reading R-1 of
// DESIGN.md): z_h = SM64(seed, 2c), z_s = SM64(seed, 2c+1) for GLOBAL row c,
// h = floor(z_h * d / 2^64) (one UMULHI), sign = top bit of z_s.
//
// Bucketing = a stable LSD radix sort of (key = h, value = row | sign<<31) over the
// ceil(log2 d) key bits (CUB onesweep), so rows of one bucket stay in ascending row
// order -- the order Algorithm 1's sketch sums in.  offsets[j] = first
// position of bucket j (lower_bound), offsets[d] = m.
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

// One-launch plan (default for the seeded hash): a cooperative kernel, one CTA per SM.
//   P1  count[h(i)] += 1 for every row (global atomics; count zeroed by the caller)
//   P2  CTA 0: offsets = exclusive scan of count, cursor = offsets
//   P3  perm[atomicAdd(cursor[h(i)], 1)] = i | sign << 31   (arbitrary order within a bucket)
//   P4  each bucket's segment sorted by row (warp per bucket; rows are distinct keys, so the
//       result is unique: exactly the stable order the radix sort produces)
// Three grid barriers instead of the ~6 launches (and their gaps) of the CUB path.
constexpr int kPlanThreads = 1024;
constexpr int kPlanSegSmem = 1024;  // bucket sizes sorted in shared memory (ints per warp)
__global__ void __launch_bounds__(kPlanThreads, 1)
k_plan_fused(uint64_t seed, int64_t row_offset, int32_t m, uint32_t d, int32_t *count, int32_t *cursor,
             int32_t *offsets, int32_t *perm, int32_t *scratch) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ int32_t seg_all[];  // [warps][kPlanSegSmem]
    __shared__ int32_t wsum[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t gtid = static_cast<int64_t>(blockIdx.x) * blockDim.x + tid;
    const int64_t gthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
    auto bucket = [&](int32_t i, uint32_t &neg) {
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
    // P2: one CTA scans d counts (each thread a contiguous run, block scan of the run sums)
    if (blockIdx.x == 0) {
        const int64_t per = (static_cast<int64_t>(d) + kPlanThreads - 1) / kPlanThreads;
        const int64_t j0 = per * tid, j1 = (j0 + per < d) ? j0 + per : d;
        int32_t run = 0;
        for (int64_t j = j0; j < j1; ++j) run += count[j];
        int32_t incl = run;  // inclusive warp scan, then warps
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            int32_t w = wsum[lane], wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += y;
            }
            wsum[lane] = wi - w;  // exclusive over warps
        }
        __syncthreads();
        int32_t base = wsum[warp] + incl - run;
        for (int64_t j = j0; j < j1; ++j) {
            offsets[j] = base;
            cursor[j] = base;
            base += count[j];
        }
        if (tid == 0) offsets[d] = m;
    }
    grid.sync();
    // P3
    for (int64_t i = gtid; i < m; i += gthreads) {
        uint32_t neg;
        const uint32_t h = bucket(static_cast<int32_t>(i), neg);
        const int32_t pos = atomicAdd(cursor + h, 1);
        perm[pos] = static_cast<int32_t>(static_cast<uint32_t>(i) | (neg << 31));
    }
    grid.sync();
    // P4: rank sort of each bucket by row (keys distinct)
    const int64_t gw = gtid >> 5, nw = gthreads >> 5;
    int32_t *sw = seg_all + static_cast<size_t>(warp) * kPlanSegSmem;
    for (int64_t j = gw; j < d; j += nw) {
        const int32_t a = offsets[j], e = offsets[j + 1], sz = e - a;
        if (sz <= 1) continue;
        if (sz <= 32) {
            const int32_t v = lane < sz ? perm[a + lane] : 0x7fffffff;
            const int32_t key = v & 0x7fffffff;
            int32_t rank = 0;
            for (int l = 0; l < sz; ++l) {
                const int32_t kl = __shfl_sync(0xffffffffu, key, l);
                rank += kl < key ? 1 : 0;
            }
            if (lane < sz) perm[a + rank] = v;
        } else {
            const int32_t *src;
            if (sz <= kPlanSegSmem) {
                for (int t = lane; t < sz; t += 32) sw[t] = perm[a + t];
                __syncwarp();
                src = sw;
            } else {  // rare (a bucket of > 1024 rows): stage in global scratch
                for (int t = lane; t < sz; t += 32) scratch[a + t] = perm[a + t];
                __syncwarp();
                __threadfence_block();
                src = scratch + a;
            }
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

    // the one-launch plan wins in the middle (measured, tools/plan_time.py: 14 vs ~30 us of CUB
    // kernels at m = 2e4, 26 vs ~38 at 1e5); below ~1e4 rows its three grid barriers cost more
    // than the small CUB passes, above ~2e5 its bucket atomics and per-bucket sorts do
    static const bool use_cub = getenv("CSK_PLAN_CUB") != nullptr;
    static const bool use_fused = getenv("CSK_PLAN_FUSED") != nullptr;
    if (h_in == nullptr && !use_cub && ((m > 8192 && m <= 200000 && m <= 256 * d) || use_fused)) {
        CSK_CHECK(ensure(ctx, ctx->keys_in, static_cast<size_t>(d + 1) * 4));  // count[d]
        int32_t *count = static_cast<int32_t *>(ctx->keys_in.ptr);
        int32_t *cursor = reinterpret_cast<int32_t *>(vals_in);  // m >= d
        int32_t *perm = reinterpret_cast<int32_t *>(vals_out);
        int32_t *scratch = reinterpret_cast<int32_t *>(keys_out);
        CSK_CUDA(ctx, cudaMemsetAsync(count, 0, static_cast<size_t>(d) * 4, stream));
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        cfg.gridDim = dim3(ctx->num_sms);  // every SM: P4 is one latency chain per bucket per warp
        cfg.blockDim = dim3(kPlanThreads);
        cfg.dynamicSmemBytes = static_cast<size_t>(kPlanThreads / 32) * kPlanSegSmem * 4;
        cfg.stream = stream;
        CSK_CHECK(raise_smem(ctx, reinterpret_cast<const void *>(k_plan_fused)));
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CSK_CUDA(ctx, cudaLaunchKernelEx(&cfg, k_plan_fused, seed, row_offset, static_cast<int32_t>(m),
                                         static_cast<uint32_t>(d), count, cursor, offsets, perm, scratch));
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
