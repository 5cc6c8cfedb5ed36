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
#include <cub/device/device_radix_sort.cuh>
#include <stdlib.h>

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

// ---- one-pass "scan" bucketing for m <= kScanMaxM (replaces the radix sort + offsets) ----
// CTA c owns the buckets [j0, j1) = [d c/Gp, d (c+1)/Gp).  Its 8 warps read all m keys once
// (coalesced; warp w takes the rows [w m/8, (w+1) m/8)), count the rows below j0 (= the
// CTA's start in perm) and stage the rows of its buckets in ascending row order (warp
// ballots; warp segments concatenated in warp order).  Warp 0 then scatters the staged rows
// to perm with __match_any_sync ranks: stable, so each bucket keeps ascending row order.
// A CTA whose staging overflows redoes its buckets one at a time (correct, slow; only for
// maps far from uniform).
constexpr int kScanMaxM = 262144;
constexpr int kScanCapW = 1024;   // staged rows per warp
constexpr int kScanMaxNb = 8192;  // buckets per CTA

__global__ void __launch_bounds__(256) k_plan_scan(const uint32_t *__restrict__ keys, const uint32_t *__restrict__ vals,
                                                   int32_t m, int32_t d, int32_t *perm, int32_t *offsets) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int Gp = gridDim.x, c = blockIdx.x;
    const int32_t j0 = static_cast<int32_t>(static_cast<int64_t>(d) * c / Gp);
    const int32_t j1 = static_cast<int32_t>(static_cast<int64_t>(d) * (c + 1) / Gp);
    const int nb = j1 - j0;
    int *run = reinterpret_cast<int *>(sm);                          // [nb]: counts, then running positions
    uint32_t *stg_v = reinterpret_cast<uint32_t *>(run + kScanMaxNb);  // [8][kScanCapW]
    uint32_t *stg_b = stg_v + 8 * kScanCapW;                         // [8][kScanCapW]
    __shared__ int cnt_w[8], below_w[8], ovf;
    for (int t = tid; t < nb; t += blockDim.x) run[t] = 0;
    if (tid == 0) ovf = 0;
    __syncthreads();
    const int32_t w0 = static_cast<int32_t>(static_cast<int64_t>(m) * warp / 8);
    const int32_t w1 = static_cast<int32_t>(static_cast<int64_t>(m) * (warp + 1) / 8);
    const unsigned lt = (1u << lane) - 1u;
    int cnt = 0, below = 0;
    for (int32_t i0 = w0; i0 < w1; i0 += 32) {
        const int32_t i = i0 + lane;
        const uint32_t h = i < w1 ? keys[i] : 0xffffffffu;
        below += __popc(__ballot_sync(0xffffffffu, h < static_cast<uint32_t>(j0)));
        const bool sel = h >= static_cast<uint32_t>(j0) && h < static_cast<uint32_t>(j1);
        const unsigned bal = __ballot_sync(0xffffffffu, sel);
        if (sel) {
            const int pos = cnt + __popc(bal & lt);
            if (pos < kScanCapW) {
                stg_v[warp * kScanCapW + pos] = vals[i];
                stg_b[warp * kScanCapW + pos] = h - static_cast<uint32_t>(j0);
            }
            atomicAdd(&run[h - static_cast<uint32_t>(j0)], 1);
        }
        cnt += __popc(bal);
    }
    if (lane == 0) {
        cnt_w[warp] = cnt;
        below_w[warp] = below;
        if (cnt > kScanCapW) atomicExch(&ovf, 1);
    }
    __syncthreads();
    int start = 0;
    for (int w = 0; w < 8; ++w) start += below_w[w];
    // exclusive scan of the bucket counts (warp 0, in chunks of 32) -> offsets and positions
    if (warp == 0) {
        int carry = 0;
        for (int t0 = 0; t0 < nb; t0 += 32) {
            const int t = t0 + lane;
            const int v = t < nb ? run[t] : 0;
            int incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += u;
            }
            const int excl = carry + incl - v;
            if (t < nb) {
                run[t] = start + excl;
                offsets[j0 + t] = start + excl;
            }
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (c == Gp - 1 && lane == 0) offsets[d] = m;
    }
    __syncthreads();
    if (!ovf) {
        if (warp == 0) {  // stable scatter in staging (= ascending row) order
            for (int w = 0; w < 8; ++w) {
                const int cw = cnt_w[w];
                for (int e0 = 0; e0 < cw; e0 += 32) {
                    const int e = e0 + lane;
                    const bool ok = e < cw;
                    const uint32_t bkt = ok ? stg_b[w * kScanCapW + e] : 0xffffffffu;
                    const unsigned grp = __match_any_sync(0xffffffffu, bkt);
                    if (ok) {
                        const int base = run[bkt];
                        perm[base + __popc(grp & lt)] = static_cast<int32_t>(stg_v[w * kScanCapW + e]);
                    }
                    __syncwarp();
                    // the highest lane of each bucket group advances that bucket's position
                    if (ok && (grp >> lane) == 1u) run[bkt] += __popc(grp);
                    __syncwarp();
                }
            }
        }
        return;
    }
    // overflow: one bucket at a time, the whole CTA rescans the keys in row order
    __shared__ int cnt2[8];
    for (int lb = 0; lb < nb; ++lb) {
        const uint32_t hb = static_cast<uint32_t>(j0 + lb);
        int cw = 0;
        for (int32_t i0 = w0; i0 < w1; i0 += 32) {
            const int32_t i = i0 + lane;
            cw += __popc(__ballot_sync(0xffffffffu, i < w1 && keys[i] == hb));
        }
        if (lane == 0) cnt2[warp] = cw;
        __syncthreads();
        int base = run[lb];
        for (int w = 0; w < warp; ++w) base += cnt2[w];
        for (int32_t i0 = w0; i0 < w1; i0 += 32) {
            const int32_t i = i0 + lane;
            const bool sel = i < w1 && keys[i] == hb;
            const unsigned bal = __ballot_sync(0xffffffffu, sel);
            if (sel) perm[base + __popc(bal & lt)] = static_cast<int32_t>(vals[i]);
            base += __popc(bal);
        }
        __syncthreads();
    }
}

size_t plan_scan_smem() { return static_cast<size_t>(kScanMaxNb) * 4 + static_cast<size_t>(16) * kScanCapW * 4; }

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

    if (h_in == nullptr) {
        k_hash_keys<<<grid, threads, 0, stream>>>(seed, row_offset, static_cast<int32_t>(m),
                                                  static_cast<uint32_t>(d), keys_in, vals_in,
                                                  nullptr, nullptr);
        const int gp = static_cast<int>(d < ctx->num_sms ? d : ctx->num_sms);
        if (m <= kScanMaxM && (d + gp - 1) / gp <= kScanMaxNb && !getenv("CSK_PLAN_CUB")) {
            static bool raised = false;
            if (!raised) {
                CSK_CUDA(ctx, cudaFuncSetAttribute(k_plan_scan, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(plan_scan_smem())));
                raised = true;
            }
            k_plan_scan<<<gp, 256, plan_scan_smem(), stream>>>(keys_in, vals_in, static_cast<int32_t>(m),
                                                               static_cast<int32_t>(d),
                                                               reinterpret_cast<int32_t *>(vals_out), offsets);
            CSK_CUDA(ctx, cudaGetLastError());
            *perm_out = reinterpret_cast<int32_t *>(vals_out);
            *offsets_out = offsets;
            return CSK_OK;
        }
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
