// api.cu -- the C ABI of include/csk.h: argument validation, workspaces, dispatch.
// Every compute step runs in the kernels of plan.cu / sketch.cu / loop.cu; this file
// only checks arguments (SURVEY.md §8(b) error table) and sequences launches.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "csk_internal.cuh"

namespace csk {

csk_status_t fail(csk_ctx_t ctx, csk_status_t st, const std::string &msg) {
    if (ctx) ctx->last_error = msg;
    return st;
}

csk_status_t cuda_fail(csk_ctx_t ctx, cudaError_t e, const char *what) {
    std::string m = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    return fail(ctx, e == cudaErrorMemoryAllocation ? CSK_E_NOMEM : CSK_E_CUDA, m);
}

csk_status_t ensure(csk_ctx_t ctx, Workspace &w, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (w.bytes >= bytes) return CSK_OK;
    if (w.ptr) {
        // captured sketch graphs hold the old workspace pointers
        for (auto &kv : ctx->sketch_graphs) cudaGraphExecDestroy(kv.second.exec);
        ctx->sketch_graphs.clear();
        ctx->sketch_seen.clear();
        // the old buffer may still be in use by queued work on any stream
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaDeviceSynchronize");
        cudaFree(w.ptr);
        w.ptr = nullptr;
        w.bytes = 0;
    }
    size_t grow = bytes + bytes / 8;
    cudaError_t e = cudaMalloc(&w.ptr, grow);
    if (e != cudaSuccess) {
        w.ptr = nullptr;
        return cuda_fail(ctx, e, "cudaMalloc(workspace)");
    }
    w.bytes = grow;
    return CSK_OK;
}

csk_status_t raise_smem(csk_ctx_t ctx, const void *fn) {
    if (ctx->smem_raised.count(fn)) return CSK_OK;
    cudaFuncAttributes fa;
    CSK_CUDA(ctx, cudaFuncGetAttributes(&fa, fn));
    const int dyn = ctx->max_smem_optin - static_cast<int>(fa.sharedSizeBytes);
    CSK_CUDA(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
    CSK_CUDA(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    ctx->smem_raised.insert(fn);
    return CSK_OK;
}

csk_status_t max_resident(csk_ctx_t ctx, const void *fn, int cs, int threads, size_t smem, int *out) {
    const auto key = std::make_tuple(fn, cs, smem);
    auto it = ctx->occ_cache.find(key);
    if (it != ctx->occ_cache.end()) {
        *out = it->second;
        return CSK_OK;
    }
    CSK_CHECK(raise_smem(ctx, fn));
    int v = 0;
    if (cs > 1) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CSK_CUDA(ctx, cudaOccupancyMaxActiveClusters(&v, fn, &cfg));
    } else {
        int per = 0;
        CSK_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, smem));
        v = per * ctx->num_sms;
    }
    ctx->occ_cache[key] = v;
    *out = v;
    return CSK_OK;
}

static void release(Workspace &w) {
    if (w.ptr) cudaFree(w.ptr);
    w.ptr = nullptr;
    w.bytes = 0;
}

static csk_status_t check_dense(csk_ctx_t ctx, const char *fn, const double *A, int64_t lda,
                                const double *b, int64_t m, int64_t n, int64_t d, bool allow_d_eq_m,
                                const double *At, const double *bt) {
    char buf[256];
    if (!A || !b || !At || !bt) {
        snprintf(buf, sizeof buf, "%s: null pointer argument", fn);
        return fail(ctx, CSK_E_ARG, buf);
    }
    if (m < 1 || m >= (int64_t(1) << 31) || n < 1 || d < 1 || (allow_d_eq_m ? d > m : d >= m)) {
        snprintf(buf, sizeof buf, "%s: need n >= 1 and 1 <= d %s m < 2^31 (Algorithm 1, P:60); got m=%lld n=%lld d=%lld",
                 fn, allow_d_eq_m ? "<=" : "<", (long long)m, (long long)n, (long long)d);
        return fail(ctx, CSK_E_ARG, buf);
    }
    if (lda < n || (reinterpret_cast<uintptr_t>(A) & 7) || !aligned16(At)) {
        snprintf(buf, sizeof buf, "%s: need lda >= n, A 8-byte and A~ 16-byte aligned", fn);
        return fail(ctx, CSK_E_ARG, buf);
    }
    return CSK_OK;
}

// csk_solve / csk_solve_ex: argument checks (SURVEY.md §8(b) error table), then the persistent
// loop kernel of loop.cu.
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
    if ((reinterpret_cast<uintptr_t>(At) | reinterpret_cast<uintptr_t>(bt) | reinterpret_cast<uintptr_t>(nsq) |
         reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(x_star)) & 7)
        return fail(ctx, CSK_E_ARG, "csk_solve: fp64 arrays must be 8-byte aligned");
    if (opts && (opts->flags & CSK_SOLVE_LEGACY))
        return fail(ctx, CSK_E_UNSUPPORTED, "csk_solve: CSK_SOLVE_LEGACY was removed in ABI 2");
    if (opts && opts->r_trace_cap < 0) return fail(ctx, CSK_E_ARG, "csk_solve: r_trace_cap < 0");
    if (ctx->pending) return fail(ctx, CSK_E_ARG, "csk_solve: a CSK_SOLVE_ASYNC solve is still in flight (call csk_solve_wait)");
    return run_loop(ctx, At, bt, nsq, d, n, x, x_star, tol, max_iters, opts, report, stream);
}

csk_status_t ensure_host_report(csk_ctx_t ctx) {
    if (ctx->report_host) return CSK_OK;
    cudaError_t e = cudaMallocHost(&ctx->report_host, 8 * sizeof(int64_t));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMallocHost(report)");
    return CSK_OK;
}

// The loop kernel's report: [0] iterations, [1] final stop quantity (bits), [2] termination
// (-2 every row masked, -3 exchange watchdog), [3] last index.
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

using namespace csk;

extern "C" {

int csk_abi_version(void) { return CSK_ABI_VERSION; }

const char *csk_status_string(csk_status_t s) {
    switch (s) {
        case CSK_OK: return "CSK_OK";
        case CSK_E_ARG: return "CSK_E_ARG";
        case CSK_E_ZERO_SKETCH: return "CSK_E_ZERO_SKETCH";
        case CSK_E_UNSUPPORTED: return "CSK_E_UNSUPPORTED";
        case CSK_E_CUDA: return "CSK_E_CUDA";
        case CSK_E_NCCL: return "CSK_E_NCCL";
        case CSK_E_NOMEM: return "CSK_E_NOMEM";
    }
    return "CSK_E_UNKNOWN";
}

csk_status_t csk_ctx_create(int device, csk_ctx_t *out) {
    if (!out) return CSK_E_ARG;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) return CSK_E_CUDA;
    if (cudaSetDevice(device) != cudaSuccess) return CSK_E_CUDA;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return CSK_E_CUDA;
    if (prop.major < 10) return CSK_E_UNSUPPORTED;  // built for sm_100a only
    auto *c = new csk_ctx_s();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    c->max_smem_optin = static_cast<int>(prop.sharedMemPerBlockOptin);
    *out = c;
    return CSK_OK;
}

csk_status_t csk_ctx_destroy(csk_ctx_t ctx) {
    if (!ctx) return CSK_E_ARG;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    Workspace *all[] = {&ctx->keys_in, &ctx->keys_out, &ctx->vals_in, &ctx->vals_out, &ctx->cub_tmp,
                        &ctx->offsets, &ctx->flag, &ctx->a_tilde, &ctx->b_tilde, &ctx->nsq,
                        &ctx->x_dev, &ctx->xs_dev, &ctx->a_dev, &ctx->b_dev, &ctx->slots,
                        &ctx->report, &ctx->scalars};
    for (Workspace *w : all) release(*w);
    if (ctx->report_host) cudaFreeHost(ctx->report_host);
    for (auto &e : ctx->ev)
        if (e) cudaEventDestroy(e);
    for (auto &kv : ctx->sketch_graphs) cudaGraphExecDestroy(kv.second.exec);
    if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
    delete ctx;
    return CSK_OK;
}

const char *csk_last_error(csk_ctx_t ctx) { return ctx ? ctx->last_error.c_str() : "null context"; }

csk_status_t csk_sketch(csk_ctx_t ctx, const double *A, int64_t lda, const double *b, int64_t m,
                        int64_t n, int64_t d, uint64_t seed, double *A_tilde, double *b_tilde,
                        double *nsq, void *stream) {
    CSK_NVTX("csk_sketch");
    if (!ctx) return CSK_E_ARG;
    CSK_CHECK(check_dense(ctx, "csk_sketch", A, lda, b, m, n, d, false, A_tilde, b_tilde));
    CSK_CUDA(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = as_stream(stream);
    static const bool no_graph = getenv("CSK_NO_GRAPH") != nullptr;
    int32_t *perm = nullptr, *offsets = nullptr;
    if (no_graph) {
        CSK_CHECK(build_plan(ctx, seed, 0, m, d, nullptr, nullptr, &perm, &offsets, s));
        return launch_sketch_dense(ctx, A, lda, b, m, n, d, perm, offsets, A_tilde, b_tilde, nsq, s);
    }
    // The plan (hash + CUB radix sort + bucket offsets, ~6 launches) depends only on (seed, m, d):
    // from the second identical call on it is replayed as a CUDA graph (one submit, no host gaps
    // between its kernels); the sketch kernel is launched after it on `s` as usual
    char kb[128];
    snprintf(kb, sizeof(kb), "%lld,%lld,%llu,%p", static_cast<long long>(m), static_cast<long long>(d),
             static_cast<unsigned long long>(seed), static_cast<void *>(s));
    const std::string key(kb);
    auto it = ctx->sketch_graphs.find(key);
    cudaStreamCaptureStatus cs;
    CSK_CUDA(ctx, cudaStreamIsCapturing(s, &cs));
    if (it != ctx->sketch_graphs.end()) {
        CSK_CUDA(ctx, cudaGraphLaunch(it->second.exec, s));
        perm = it->second.perm;
        offsets = it->second.offsets;
    } else if (!ctx->sketch_seen.count(key) || cs != cudaStreamCaptureStatusNone) {
        // first time (sizes every workspace), or the caller is capturing: inline
        ctx->sketch_seen.insert(key);
        CSK_CHECK(build_plan(ctx, seed, 0, m, d, nullptr, nullptr, &perm, &offsets, s));
    } else {
        // capture on a private stream (the legacy default stream cannot capture); launch on `s`
        if (!ctx->cap_stream) CSK_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
        CSK_CUDA(ctx, cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
        const csk_status_t st = build_plan(ctx, seed, 0, m, d, nullptr, nullptr, &perm, &offsets, ctx->cap_stream);
        cudaGraph_t g = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(ctx->cap_stream, &g);
        if (st != CSK_OK) {
            if (g) cudaGraphDestroy(g);
            return st;
        }
        if (ce != cudaSuccess) return cuda_fail(ctx, ce, "cudaStreamEndCapture(csk_sketch plan)");
        cudaGraphExec_t ex = nullptr;
        const cudaError_t ie = cudaGraphInstantiate(&ex, g, 0);
        cudaGraphDestroy(g);
        if (ie != cudaSuccess) return cuda_fail(ctx, ie, "cudaGraphInstantiate(csk_sketch plan)");
        ctx->sketch_graphs[key] = {ex, perm, offsets};
        CSK_CUDA(ctx, cudaGraphLaunch(ex, s));
    }
    return launch_sketch_dense(ctx, A, lda, b, m, n, d, perm, offsets, A_tilde, b_tilde, nsq, s);
}

csk_status_t csk_sketch_with_map(csk_ctx_t ctx, const double *A, int64_t lda, const double *b,
                                 int64_t m, int64_t n, int64_t d, const int32_t *h,
                                 const int8_t *sign, double *A_tilde, double *b_tilde, double *nsq,
                                 void *stream) {
    CSK_NVTX("csk_sketch_with_map");
    if (!ctx) return CSK_E_ARG;
    CSK_CHECK(check_dense(ctx, "csk_sketch_with_map", A, lda, b, m, n, d, true, A_tilde, b_tilde));
    if (!h || !sign) return fail(ctx, CSK_E_ARG, "csk_sketch_with_map: null map");
    CSK_CUDA(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = as_stream(stream);
    int32_t *perm = nullptr, *offsets = nullptr;
    CSK_CHECK(build_plan(ctx, 0, 0, m, d, h, sign, &perm, &offsets, s));
    return launch_sketch_dense(ctx, A, lda, b, m, n, d, perm, offsets, A_tilde, b_tilde, nsq, s);
}

csk_status_t csk_sketch_planned(csk_ctx_t ctx, const double *A, int64_t lda, const double *b, int64_t m,
                                int64_t n, int64_t d, const int32_t *perm, const int32_t *offsets,
                                double *A_tilde, double *b_tilde, double *nsq, void *stream) {
    CSK_NVTX("csk_sketch_planned");
    if (!ctx) return CSK_E_ARG;
    CSK_CHECK(check_dense(ctx, "csk_sketch_planned", A, lda, b, m, n, d, true, A_tilde, b_tilde));
    if (!perm || !offsets) return fail(ctx, CSK_E_ARG, "csk_sketch_planned: null plan");
    CSK_CUDA(ctx, cudaSetDevice(ctx->device));
    return launch_sketch_dense(ctx, A, lda, b, m, n, d, perm, offsets, A_tilde, b_tilde, nsq, as_stream(stream));
}

csk_status_t csk_sketch_csr(csk_ctx_t ctx, const int64_t *row_ptr, const int32_t *col,
                            const double *val, const double *b, int64_t m, int64_t n, int64_t d,
                            uint64_t seed, double *A_tilde, double *b_tilde, double *nsq,
                            void *stream) {
    CSK_NVTX("csk_sketch_csr");
    if (!ctx) return CSK_E_ARG;
    if (!row_ptr || !col || !val || !b || !A_tilde || !b_tilde)
        return fail(ctx, CSK_E_ARG, "csk_sketch_csr: null pointer argument");
    if (m < 1 || m >= (int64_t(1) << 31) || n < 1 || d < 1 || d >= m)
        return fail(ctx, CSK_E_ARG, "csk_sketch_csr: need n >= 1 and 1 <= d < m < 2^31 (P:60)");
    CSK_CUDA(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = as_stream(stream);
    int32_t *perm = nullptr, *offsets = nullptr;
    CSK_CHECK(build_plan(ctx, seed, 0, m, d, nullptr, nullptr, &perm, &offsets, s));
    return launch_sketch_csr(ctx, row_ptr, col, val, b, m, n, d, perm, offsets, A_tilde, b_tilde, nsq, s);
}

csk_status_t csk_row_norms(csk_ctx_t ctx, const double *A_tilde, int64_t d, int64_t n, double *nsq,
                           void *stream) {
    CSK_NVTX("csk_row_norms");
    if (!ctx) return CSK_E_ARG;
    if (!A_tilde || !nsq || d < 1 || n < 1) return fail(ctx, CSK_E_ARG, "csk_row_norms: bad arguments");
    CSK_CUDA(ctx, cudaSetDevice(ctx->device));
    return launch_row_norms(ctx, A_tilde, d, n, nsq, as_stream(stream));
}

csk_status_t csk_solve(csk_ctx_t ctx, const double *A_tilde, const double *b_tilde, const double *nsq,
                       int64_t d, int64_t n, double *x, const double *x_star, double tol,
                       int64_t max_iters, csk_report_t *report, void *stream) {
    return csk_solve_ex(ctx, A_tilde, b_tilde, nsq, d, n, x, x_star, tol, max_iters, nullptr, report, stream);
}

csk_status_t csk_solve_ex(csk_ctx_t ctx, const double *A_tilde, const double *b_tilde,
                          const double *nsq, int64_t d, int64_t n, double *x, const double *x_star,
                          double tol, int64_t max_iters, const csk_solve_opts_t *opts,
                          csk_report_t *report, void *stream) {
    CSK_NVTX("csk_solve_ex");
    if (!ctx) return CSK_E_ARG;
    CSK_CUDA(ctx, cudaSetDevice(ctx->device));
    return run_solve(ctx, A_tilde, b_tilde, nsq, d, n, x, x_star, tol, max_iters, opts, report,
                     as_stream(stream));
}

csk_status_t csk_solve_wait(csk_ctx_t ctx, csk_report_t *report) {
    CSK_NVTX("csk_solve_wait");
    if (!ctx) return CSK_E_ARG;
    CSK_CUDA(ctx, cudaSetDevice(ctx->device));
    return finish_solve(ctx, report);
}

csk_status_t csk_ctx_set_timing(csk_ctx_t ctx, int32_t on) {
    if (!ctx) return CSK_E_ARG;
    CSK_CUDA(ctx, cudaSetDevice(ctx->device));
    if (on && !ctx->ev[0])
        for (auto &e : ctx->ev) CSK_CUDA(ctx, cudaEventCreate(&e));
    ctx->timing = on != 0;
    ctx->ev_recorded[0] = ctx->ev_recorded[1] = false;
    return CSK_OK;
}

csk_status_t csk_last_kernel_ms(csk_ctx_t ctx, int32_t which, float *ms) {
    if (!ctx || !ms || which < 0 || which > 1) return ctx ? fail(ctx, CSK_E_ARG, "csk_last_kernel_ms: bad arguments") : CSK_E_ARG;
    if (!ctx->ev_recorded[which]) return fail(ctx, CSK_E_ARG, "csk_last_kernel_ms: no timed launch yet (csk_ctx_set_timing)");
    CSK_CUDA(ctx, cudaEventSynchronize(ctx->ev[2 * which + 1]));
    CSK_CUDA(ctx, cudaEventElapsedTime(ms, ctx->ev[2 * which], ctx->ev[2 * which + 1]));
    return CSK_OK;
}

csk_status_t csk_last_solve_geometry(csk_ctx_t ctx, int32_t *num_ctas, int32_t *cluster_size,
                                     int32_t *smem_rows) {
    if (!ctx) return CSK_E_ARG;
    if (num_ctas) *num_ctas = ctx->last_solve_geom[0];
    if (cluster_size) *cluster_size = ctx->last_solve_geom[1];
    if (smem_rows) *smem_rows = ctx->last_solve_geom[2];
    return CSK_OK;
}

csk_status_t csk_last_solve_tiers(csk_ctx_t ctx, int32_t *out) {
    if (!ctx || !out) return CSK_E_ARG;
    for (int i = 0; i < 8; ++i) out[i] = ctx->last_solve_tiers[i];
    return CSK_OK;
}

csk_status_t csk_run(csk_ctx_t ctx, const double *A, int64_t lda, const double *b, int64_t m,
                     int64_t n, int64_t d, uint64_t seed, double *x, const double *x_star,
                     double tol, int64_t max_iters, csk_report_t *report, void *stream) {
    CSK_NVTX("csk_run");
    if (!ctx) return CSK_E_ARG;
    CSK_CUDA(ctx, cudaSetDevice(ctx->device));
    CSK_CHECK(ensure(ctx, ctx->a_tilde, static_cast<size_t>(d) * n * 8));
    CSK_CHECK(ensure(ctx, ctx->b_tilde, static_cast<size_t>(d) * 8));
    CSK_CHECK(ensure(ctx, ctx->nsq, static_cast<size_t>(d) * 8));
    double *At = static_cast<double *>(ctx->a_tilde.ptr);
    double *bt = static_cast<double *>(ctx->b_tilde.ptr);
    double *ns = static_cast<double *>(ctx->nsq.ptr);
    CSK_CHECK(csk_sketch(ctx, A, lda, b, m, n, d, seed, At, bt, ns, stream));
    return csk_solve_ex(ctx, At, bt, ns, d, n, x, x_star, tol, max_iters, nullptr, report, stream);
}

csk_status_t csk_run_host(csk_ctx_t ctx, const double *A_host, int64_t lda, const double *b_host,
                          int64_t m, int64_t n, int64_t d, uint64_t seed, double *x_host,
                          const double *x_star_host, double tol, int64_t max_iters,
                          csk_report_t *report, void *stream) {
    CSK_NVTX("csk_run_host");
    if (!ctx) return CSK_E_ARG;
    if (!A_host || !b_host || !x_host) return fail(ctx, CSK_E_ARG, "csk_run_host: null host buffer");
    if (m < 1 || n < 1 || lda < n) return fail(ctx, CSK_E_ARG, "csk_run_host: bad sizes");
    CSK_CUDA(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = as_stream(stream);
    const size_t abytes = static_cast<size_t>(m) * lda * 8;
    CSK_CHECK(ensure(ctx, ctx->a_dev, abytes));
    CSK_CHECK(ensure(ctx, ctx->b_dev, static_cast<size_t>(m) * 8));
    CSK_CHECK(ensure(ctx, ctx->x_dev, static_cast<size_t>(n) * 8));
    CSK_CHECK(ensure(ctx, ctx->xs_dev, static_cast<size_t>(n) * 8));
    double *Ad = static_cast<double *>(ctx->a_dev.ptr);
    double *bd = static_cast<double *>(ctx->b_dev.ptr);
    double *xd = static_cast<double *>(ctx->x_dev.ptr);
    double *xsd = x_star_host ? static_cast<double *>(ctx->xs_dev.ptr) : nullptr;
    CSK_CUDA(ctx, cudaMemcpyAsync(Ad, A_host, abytes, cudaMemcpyHostToDevice, s));
    CSK_CUDA(ctx, cudaMemcpyAsync(bd, b_host, static_cast<size_t>(m) * 8, cudaMemcpyHostToDevice, s));
    CSK_CUDA(ctx, cudaMemcpyAsync(xd, x_host, static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice, s));
    if (xsd) CSK_CUDA(ctx, cudaMemcpyAsync(xsd, x_star_host, static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice, s));
    CSK_CHECK(csk_run(ctx, Ad, lda, bd, m, n, d, seed, xd, xsd, tol, max_iters, report, stream));
    CSK_CUDA(ctx, cudaMemcpyAsync(x_host, xd, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost, s));
    CSK_CUDA(ctx, cudaStreamSynchronize(s));
    return CSK_OK;
}

}  // extern "C"
