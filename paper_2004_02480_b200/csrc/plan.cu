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
