// csk_internal.cuh -- shared internals of libcsk (context, error plumbing, PTX helpers).
// Product code only: nothing here is shared with oracle/ (the CPU oracle is independent).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <map>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/csk.h"

// NVTX range over one public entry point (SURVEY section 5 tracing): the host span of the call,
// visible in nsys / ncu --nvtx timelines; a no-op unless a tool is attached
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};
#define CSK_NVTX(name) ::NvtxRange csk_nvtx_range_(name)

// Device-side bounds checks of the checked build (libcsk_checked.so, -DCSK_CHECKED=1; compute-
// sanitizer is not available on the GPU pool): a failed check traps the kernel, which surfaces
// as a CUDA error in the calling test.  Compiled out of the product library.
#if defined(CSK_CHECKED) && CSK_CHECKED
#define CSK_DCHECK(cond)       \
    do {                       \
        if (!(cond)) __trap(); \
    } while (0)
#else
#define CSK_DCHECK(cond) \
    do {                 \
    } while (0)
#endif

namespace csk {

// ---------------------------------------------------------------- context
struct Workspace {
    void *ptr = nullptr;
    size_t bytes = 0;
};

struct Comm;  // sharded path (comm.cu)

}  // namespace csk

struct csk_ctx_s {
    int device = 0;
    int num_sms = 148;
    int max_smem_optin = 227 * 1024;
    std::string last_error;
    // plan workspaces
    csk::Workspace keys_in, keys_out, vals_in, vals_out, cub_tmp, offsets, flag;
    // csk_run workspaces
    csk::Workspace a_tilde, b_tilde, nsq, x_dev, xs_dev, a_dev, b_dev;
    // solve workspaces
    csk::Workspace slots, report, scalars;
    csk::Comm *comm = nullptr;
    // in-flight solve (CSK_SOLVE_ASYNC)
    int64_t *report_host = nullptr;  // pinned
    cudaStream_t pending_stream = nullptr;
    bool pending = false;
    bool pending_resmode = false;
    int last_solve_geom[5] = {0, 0, 0, 0, 0};  // CTAs, cluster size, smem rows, register rows, warps/group
    int last_solve_tiers[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // csk_last_solve_tiers
    // host-side memo of driver queries that would otherwise sit between short kernels
    std::set<const void *> smem_raised;                              // kernels set to max dyn smem
    std::map<std::tuple<const void *, int, size_t>, int> occ_cache;  // (fn, cluster, smem) -> n
    int64_t cub_key_m = -1, cub_key_bits = -1;
    size_t cub_bytes = 0;
    // csk_sketch as a replayed CUDA graph (hash, radix-sort plan, offsets, sketch: one submit)
    // per argument tuple: the first call runs eagerly (sizes the workspaces), the second captures
    struct PlanGraph {  // a captured plan (S2) and the workspaces it writes
        cudaGraphExec_t exec;
        int32_t *perm, *offsets;
    };
    std::map<std::string, PlanGraph> sketch_graphs;
    std::set<std::string> sketch_seen;
    cudaStream_t cap_stream = nullptr;  // private stream the graph is captured on
    // per-kernel CUDA-event timing (csk_ctx_set_timing): [0,1] sketch kernel, [2,3] loop kernel
    bool timing = false;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    bool ev_recorded[2] = {false, false};
};

namespace csk {

csk_status_t fail(csk_ctx_t ctx, csk_status_t st, const std::string &msg);
csk_status_t cuda_fail(csk_ctx_t ctx, cudaError_t e, const char *what);
// Grow-only device workspace.
csk_status_t ensure(csk_ctx_t ctx, Workspace &w, size_t bytes);
// Raise a kernel's dynamic shared-memory limit to the device opt-in maximum (once).
csk_status_t raise_smem(csk_ctx_t ctx, const void *fn);
// cudaOccupancyMaxActiveClusters (cs > 1) or blocks-per-SM x SMs (cs == 1), memoised.
csk_status_t max_resident(csk_ctx_t ctx, const void *fn, int cs, int threads, size_t smem, int *out);
// Kernel timing hooks: record event 2*which (before) / 2*which+1 (after) when timing is on.
inline void time_mark(csk_ctx_t ctx, int which, bool after, cudaStream_t s) {
    if (!ctx->timing) return;
    cudaEventRecord(ctx->ev[2 * which + (after ? 1 : 0)], s);
    if (after) ctx->ev_recorded[which] = true;
}

#define CSK_CUDA(ctx, call)                                   \
    do {                                                      \
        cudaError_t _e = (call);                              \
        if (_e != cudaSuccess) return csk::cuda_fail((ctx), _e, #call); \
    } while (0)

#define CSK_CHECK(call)                        \
    do {                                       \
        csk_status_t _s = (call);              \
        if (_s != CSK_OK) return _s;           \
    } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }
inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---------------------------------------------------------------- plan
// Internal plan build used by every sketch entry point.  perm/offsets may point
// into the ctx workspace.  See plan.cu.
csk_status_t build_plan(csk_ctx_t ctx, uint64_t seed, int64_t row_offset, int64_t m, int64_t d,
                        const int32_t *h_in, const int8_t *sign_in, int32_t **perm_out,
                        int32_t **offsets_out, cudaStream_t stream);

// ---------------------------------------------------------------- sketch (sketch.cu)
csk_status_t launch_sketch_dense(csk_ctx_t ctx, const double *A, int64_t lda, const double *b,
                                 int64_t m, int64_t n, int64_t d, const int32_t *perm,
                                 const int32_t *offsets, double *At, double *bt, double *nsq,
                                 cudaStream_t stream);
csk_status_t launch_sketch_csr(csk_ctx_t ctx, const int64_t *row_ptr, const int32_t *col,
                               const double *val, const double *b, int64_t m, int64_t n,
                               int64_t d, const int32_t *perm, const int32_t *offsets,
                               double *At, double *bt, double *nsq, cudaStream_t stream);
csk_status_t launch_row_norms(csk_ctx_t ctx, const double *At, int64_t d, int64_t n,
                              double *nsq, cudaStream_t stream);
// Team size used by the row-norm arithmetic (shared by fused and standalone paths).
int norm_team_threads(int64_t n);

// ---------------------------------------------------------------- solve (api.cu -> loop.cu)
csk_status_t run_solve(csk_ctx_t ctx, const double *At, const double *bt, const double *nsq,
                       int64_t d, int64_t n, double *x, const double *x_star, double tol,
                       int64_t max_iters, const csk_solve_opts_t *opts, csk_report_t *report,
                       cudaStream_t stream);
// (loop.cu) register-resident loop with the flat atomic exchange (default).
// RankSetup (optional) shards the rows of A~ over P ranks for the same persistent kernel:
//   rank = -1: P virtual ranks in ONE cooperative launch on this GPU (the 1-GPU test of S10);
//   rank >= 0: this process is rank `rank` of P GPUs; the other ranks' A~ rows and slots are
//              peer-mapped (sys = 1: system-scope exchange over NVLink).
constexpr int kMaxRanks = 8;
struct RankSetup {
    int P = 1, rank = 0, Gr = 0, sys = 0;
    int64_t dlo[kMaxRanks + 1] = {};
    const double *At_r[kMaxRanks] = {};
    const double *bt_r[kMaxRanks] = {};
    const double *nsq_r[kMaxRanks] = {};
    unsigned long long *slots_r[kMaxRanks] = {};  // null: carved from ctx->slots (virtual ranks); real
                                                  // ranks: each buffer is [exchange region][slots]
    double *x_r[kMaxRanks] = {};
    const double *bb = nullptr;                   // residual mode: global ||b~||^2 (device), null: computed
    bool exchange_zeroed = false;                 // the caller zeroed xch/slots (and synchronised the ranks)
};
size_t loop_exchange_bytes(int total_ctas);  // bytes of ctx->slots a launch of total_ctas needs

// ---------------------------------------------------------------- CSR row routing (route.cu)
// A rank's rows packed by destination owner (ascending row inside each segment): segment q holds
// cnt[2q] rows starting at seg[2q] (global row, b, pair offset in the segment) and cnt[2q+1]
// (col, val) pairs starting at seg[2q+1].  Device buffers (cudaMallocAsync) freed by route_free.
struct RoutePack {
    int P = 0;
    int64_t cnt[2 * kMaxRanks] = {}, seg[2 * kMaxRanks] = {};
    int32_t *row = nullptr;
    double *b = nullptr;
    int64_t *off = nullptr;
    int32_t *col = nullptr;
    double *val = nullptr;
    std::vector<void *> owned;
};
// What an owner received: the segments of sources 0..P-1 concatenated in source order (rows of
// source q at [rbase[q], rbase[q+1]), their pairs at [pbase[q], pbase[q+1])).
struct RouteRecv {
    int P = 0;
    int64_t rbase[kMaxRanks + 1] = {}, pbase[kMaxRanks + 1] = {};
    const int32_t *row = nullptr;
    const double *b = nullptr;
    const int64_t *off = nullptr;
    const int32_t *col = nullptr;
    const double *val = nullptr;
};
csk_status_t route_pack(csk_ctx_t ctx, const int64_t *row_ptr, const int32_t *col, const double *val, const double *b,
                        int64_t m_local, int64_t row_offset, int64_t d, uint64_t seed, int P, RoutePack &pk,
                        cudaStream_t s);
csk_status_t route_unpack_sketch(csk_ctx_t ctx, const RouteRecv &rv, int64_t n, int64_t d, int64_t d_lo, int64_t d_hi,
                                 uint64_t seed, double *At_local, double *bt_local, double *nsq_local, cudaStream_t s);
void route_free(RoutePack &pk, cudaStream_t s);
csk_status_t run_loop(csk_ctx_t ctx, const double *At, const double *bt, const double *nsq, int64_t d,
                      int64_t n, double *x, const double *x_star, double tol, int64_t max_iters,
                      const csk_solve_opts_t *opts, csk_report_t *report, cudaStream_t stream,
                      const RankSetup *ranks = nullptr);
csk_status_t ensure_host_report(csk_ctx_t ctx);
csk_status_t finish_solve(csk_ctx_t ctx, csk_report_t *report);

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ uint64_t splitmix64_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
// Counter form of SplitMix64: output number c (0-based) of the stream seeded with `seed`.
__device__ __forceinline__ uint64_t sm64(uint64_t seed, uint64_t c) {
    return splitmix64_mix(seed + (c + 1ULL) * 0x9E3779B97F4A7C15ULL);
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile(
        "{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
            smem_u32(bar)),
        "r"(bytes)
        : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
// 1-D TMA bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void *dst_smem, const void *src_gmem, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// The same copy with an L2 eviction priority (createpolicy, whole-line fraction 1.0): `keep`
// marks the lines evict_last (they stay in the 126 MB L2 between loop iterations), otherwise
// evict_first (a streamed row that will not be re-read before L2 has turned over).
__device__ __forceinline__ void bulk_g2s_l2(void *dst_smem, const void *src_gmem, uint32_t bytes,
                                            uint64_t *bar, bool keep) {
    uint64_t pol;
    if (keep)
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    else
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// Streaming read-only 16-byte load that does not allocate in L1.  Deliberately not
// `volatile`: the data is immutable for the kernel's lifetime, and a volatile asm
// would pin the loads in program order and serialise them.
__device__ __forceinline__ double2 ldg_stream2(const double *p) {
    double2 v;
    asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ double ldg_stream1(const double *p) {
    double v;
    asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

// Relaxed gpu-scope 16-byte accesses used by the cross-CTA candidate exchange.
__device__ __forceinline__ void st_relaxed_v2u64(uint64_t *p, uint64_t a, uint64_t b) {
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b)
                 : "memory");
}
__device__ __forceinline__ void ld_relaxed_v2u64(const uint64_t *p, uint64_t &a, uint64_t &b) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
                 : "=l"(a), "=l"(b)
                 : "l"(p)
                 : "memory");
}

// ---- thread-block-cluster / DSMEM helpers (sm_90+) ----
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// Address of the same shared-memory offset in cluster CTA `rank`.
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_v2u64(uint32_t addr, uint64_t a, uint64_t b) {
    asm volatile("st.relaxed.cluster.shared::cluster.v2.u64 [%0], {%1, %2};" ::"r"(addr), "l"(a), "l"(b)
                 : "memory");
}
__device__ __forceinline__ void ld_cluster_local_v2u64(uint32_t addr, uint64_t &a, uint64_t &b) {
    asm volatile("ld.relaxed.cluster.shared::cta.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "r"(addr)
                 : "memory");
}
__device__ __forceinline__ double2 ld_dsmem_v2f64(uint32_t addr) {
    double2 v;
    asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
    return v;
}
// Same, for data that is immutable while the kernel runs (not volatile: may be batched).
__device__ __forceinline__ double2 ld_dsmem_v2f64_nc(uint32_t addr) {
    double2 v;
    asm("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

}  // namespace csk
