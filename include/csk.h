/*
 * csk.h -- C ABI of the B200-native Count-Sketch Kaczmarz (CSK) hot path.
 *
 * Method: Zhang & Li, "A Count Sketch Kaczmarz Method for Solving Large
 * Overdetermined Linear Systems", arXiv 2004.02480 (/root/reference/PAPER.md,
 * cited as P:<line>).  The library computes, on an sm_100a GPU:
 *   (1) the count sketch  A~ = S A,  b~ = S b,  S = Phi D   (Def. 1);
 *   (2) the row norms     nsq_j = ||A~^(j)||_2^2             (P:62 denominator);
 *   (3) the Algorithm 1 loop  i_k = argmax r_i^2/nsq_i,  x += (r_ik/nsq_ik) A~^(ik)T
 *       with r = b~ - A~ x_k, stopped by RES <= tol or an iteration cap
 *       (P:180).
 *
 * Conventions for every entry point:
 *   - Every array argument is a DEVICE pointer unless the name ends in _host.
 *     Floating point is IEEE fp64; matrices are row-major with the given leading
 *     dimension; indices are 0-based (the paper's [m], [d] are 1-based).
 *   - Ownership: the caller allocates and frees every input and output; the
 *     library owns only the scratch workspaces inside a csk_ctx_t.
 *   - Ordering: calls are asynchronous on `stream` (a cudaStream_t passed as
 *     void*) unless stated otherwise; csk_solve* and *_host block until done
 *     because they return a termination reason.
 *   - Errors: every call returns a csk_status_t; no exception crosses the ABI.
 *     csk_last_error(ctx) returns a human-readable reason for the last failure
 *     on that context.  There is no CPU fallback: a call that cannot run on the
 *     GPU fails.
 *   - Alignment: A~ must be 16-byte aligned, A 8-byte aligned.  The sketch
 *     streams rows of A with TMA bulk copies when A is 16-byte aligned and lda is
 *     even (the fast path); otherwise the same kernel reads rows with plain loads.
 *   - Sizes: 1 <= d < m (Algorithm 1, "with d < m"), m < 2^31, n >= 1,
 *     n <= CSK_MAX_N for csk_solve*.
 */
#ifndef CSK_H_
#define CSK_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define CSK_API __attribute__((visibility("default")))
#else
#define CSK_API
#endif

#define CSK_ABI_VERSION 2
#define CSK_MAX_N 2048 /* solve keeps x in registers: 64 columns per lane-pair group */

typedef enum {
    CSK_OK = 0,
    CSK_E_ARG = 1,          /* bad size, null/misaligned pointer, d >= m, tol <= 0, ... */
    CSK_E_ZERO_SKETCH = 2,  /* every row of A~ is zero: nothing to select */
    CSK_E_UNSUPPORTED = 3,  /* valid input outside what this build implements (solve: n > 2048,
                               a grid that cannot be co-resident, or > ~9000 rows per CTA) */
    CSK_E_CUDA = 4,         /* a CUDA runtime error; csk_last_error has the text */
    CSK_E_NCCL = 5,         /* an NCCL error in a sharded call */
    CSK_E_NOMEM = 6         /* workspace allocation failed */
} csk_status_t;

/* Termination of the Algorithm 1 loop. */
typedef enum {
    CSK_CONVERGED = 0,  /* stop quantity <= tol */
    CSK_MAX_ITERS = 1,  /* k reached max_iters ("exceeds 20000"; configs: 50k) */
    CSK_STAGNATED = 2   /* every unmasked residual is exactly 0 while not converged */
} csk_term_t;

/* Stop quantity: RES = ||x_k - x*||^2/||x*||^2 when x_star != NULL,
 * else the solution-free relative residual ||b~ - A~ x_k||^2/||b~||^2. */
typedef enum { CSK_STOP_RES = 0, CSK_STOP_RESIDUAL = 1 } csk_stop_mode_t;

typedef struct {
    int64_t iterations;   /* IT = number of projections applied */
    double final_res;     /* stop quantity at the returned iterate */
    int32_t termination;  /* csk_term_t */
    int32_t stop_mode;    /* csk_stop_mode_t */
    int64_t last_index;   /* i_{IT-1}, or -1 if no step was taken */
} csk_report_t;

/* Optional knobs and debug traces for csk_solve_ex.  Zero-initialise for defaults. */
#define CSK_SOLVE_ASYNC 1  /* opts->flags: return right after the launch; csk_solve_wait fills the report */
#define CSK_SOLVE_LEGACY 2 /* removed in ABI 2 (the round-1 kernel left the library): CSK_E_UNSUPPORTED */
#define CSK_SOLVE_NO_TMEM 4    /* opts->flags: never keep A~ rows in tensor memory */
#define CSK_SOLVE_FORCE_TMEM 8 /* opts->flags: use the TMEM row tier whenever the layout allows (tests) */
#define CSK_SOLVE_NO_STREAM_RING 16 /* opts->flags: rows that do not fit on chip are re-read with plain loads
                                        instead of the TMA stream ring (tests, A/B) */

typedef struct {
    int32_t num_ctas;      /* persistent CTAs (<= co-resident limit); 0 = auto */
    int32_t smem_rows;     /* rows of A~ kept in shared memory per CTA: 0 = auto (max),
                              -1 = none (every row re-read from L2/HBM), k > 0 = at most k */
    int32_t flags;         /* CSK_SOLVE_ASYNC */
    int32_t cluster_size;  /* CTAs per thread-block cluster (power of two <= 16); 0 = auto */
    int64_t trace_cap;     /* capacity of the traces below (iterations) */
    int64_t *idx_trace;    /* device int64[trace_cap]: i_k, or NULL */
    double *res_trace;     /* device double[trace_cap]: stop quantity at x_k, or NULL */
    double *x_trace;       /* device double[trace_cap * n]: x_k row by row, or NULL */
    int64_t *phase_cycles; /* debug (libcsk_prof.so only): device int64[32] per-phase SM-cycle totals */
    int32_t reg_rows;      /* rows of A~ per row group kept in registers: 0 = auto (max), -1 = none,
                              k > 0 = at most k (the default kernel; smem_rows then counts rows per
                              row group kept in shared memory, the rest re-read from L2/HBM) */
    int32_t group_warps;   /* warps per row group (1, 2, 4, 8): 0 = auto (fewest with n <= 512 x warps) */
    /* ABI 2: the residual vector of the first r_trace_cap iterations (north_star "per-iteration
     * residuals within 1e-10 relative given the same x_k"; the numerator r_k = b~ - A~ x_k of
     * Algorithm 1's selection rule).  r_trace[k * d + i] = r_k[i] for every row i and
     * k < min(r_trace_cap, IT + 1) (the residual at the returned iterate x_IT is formed too: the
     * GEMV of iteration k runs before its stop test).  Written by the kernel's finalize: the very
     * values it scores.  Device double[r_trace_cap * d] or NULL (then no cost: one uniform branch). */
    double *r_trace;
    int64_t r_trace_cap;
} csk_solve_opts_t;

typedef struct csk_ctx_s *csk_ctx_t;

/* ---- context --------------------------------------------------------------- */
/* Binds the calling thread's CUDA device `device` and allocates nothing yet;
 * workspaces grow on demand and are reused.  Not thread-safe: one ctx per thread. */
CSK_API csk_status_t csk_ctx_create(int device, csk_ctx_t *out);
CSK_API csk_status_t csk_ctx_destroy(csk_ctx_t ctx);
CSK_API const char *csk_last_error(csk_ctx_t ctx);
CSK_API const char *csk_status_string(csk_status_t status);
CSK_API int csk_abi_version(void);

/* ---- S1/S2: the count-sketch plan ------------------------------------------- */
/* csk_hash: h[i] = floor(z_h * d / 2^64), sign[i] = (z_s >> 63) ? -1 : +1 with
 *   z_h = SM64(seed, 2c), z_s = SM64(seed, 2c+1), c = row_offset + i and
 *   SM64(seed, c) = splitmix64_mix(seed + (c+1) * 0x9E3779B97F4A7C15)  -- the
 *   counter form of the SplitMix64 stream (reading R-1 of DESIGN.md), realising
 *   Definition 1: h uniform on [d], D_ii = +-1 with probability 1/2.
 *   `row_offset` lets a row shard hash with GLOBAL row indices.
 *   h: int32[m], sign: int8[m] (device, caller-owned).  Requires d >= 1. */
CSK_API csk_status_t csk_hash(csk_ctx_t ctx, uint64_t seed, int64_t row_offset, int64_t m, int64_t d,
                      int32_t *h, int8_t *sign, void *stream);

/* csk_plan: the stable bucketing of rows by h ("source-row order"):
 *   perm[t] (int32[m]) lists the row indices grouped by bucket, ascending row
 *   index inside each bucket, with bit 31 set when sign = -1;
 *   offsets[j] (int32[d+1]) = first position of bucket j in perm, offsets[d] = m.
 *   h/sign are taken from the seed (h_in == NULL) or from explicit device arrays
 *   h_in int32[m] / sign_in int8[m] (the csk_sketch_with_map test hook; values
 *   outside [0,d) or not +-1 return CSK_E_ARG after a stream sync). */
CSK_API csk_status_t csk_plan(csk_ctx_t ctx, uint64_t seed, int64_t row_offset, int64_t m, int64_t d,
                      const int32_t *h_in, const int8_t *sign_in,
                      int32_t *perm, int32_t *offsets, void *stream);

/* ---- S3/S4: the sketch ------------------------------------------------------- */
/* csk_sketch: A~ = S A (d x n, ld = n), b~ = S b (d), with S = Phi D drawn from
 *   `seed` (Algorithm 1 "Initialize").  A~[j,:] = sum over rows i with
 *   h(i) = j, in ascending i, of sign_i * A[i,:], starting from +0.0 -- the same
 *   fp64 adds in the same order as the dense product Phi D A, so A~ and b~ are
 *   bit-reproducible and equal to the oracle bit for bit.  If nsq != NULL the
 *   row norms (S4) are fused into the epilogue (same arithmetic as csk_row_norms).
 *   A: m x n, leading dimension lda >= n.  1 <= d < m. */
CSK_API csk_status_t csk_sketch(csk_ctx_t ctx, const double *A, int64_t lda, const double *b,
                        int64_t m, int64_t n, int64_t d, uint64_t seed,
                        double *A_tilde, double *b_tilde, double *nsq, void *stream);

/* Test hook (Remark 1): explicit map h/sign (device int32[m] / int8[m]);
 * allows d == m, e.g. h = identity, which turns CSK into MWRK. */
CSK_API csk_status_t csk_sketch_with_map(csk_ctx_t ctx, const double *A, int64_t lda, const double *b,
                                 int64_t m, int64_t n, int64_t d,
                                 const int32_t *h, const int8_t *sign,
                                 double *A_tilde, double *b_tilde, double *nsq, void *stream);

/* CSR input (config C5): row_ptr int64[m+1], col int32[nnz] (distinct within a
 * row, any order; the stored order is the accumulation order), val fp64[nnz]. */
CSK_API csk_status_t csk_sketch_csr(csk_ctx_t ctx, const int64_t *row_ptr, const int32_t *col,
                            const double *val, const double *b,
                            int64_t m, int64_t n, int64_t d, uint64_t seed,
                            double *A_tilde, double *b_tilde, double *nsq, void *stream);

/* The sketch with a plan computed once by csk_plan for (seed, m, d) and reused (a cached plan:
 * the plan depends only on the map, not on A).  perm int32[m], offsets int32[d+1] as csk_plan
 * returns them (device).  Same results as csk_sketch with that seed. */
CSK_API csk_status_t csk_sketch_planned(csk_ctx_t ctx, const double *A, int64_t lda, const double *b,
                                        int64_t m, int64_t n, int64_t d, const int32_t *perm,
                                        const int32_t *offsets, double *A_tilde, double *b_tilde,
                                        double *nsq, void *stream);

/* nsq[j] = ||A~^(j)||_2^2 for j < d (P:62 / P:122).  Fixed summation order:
 * thread t of a row's team sums columns {2t, 2t+1} + 2T*q with fma, then a
 * fixed-shape tree -- bit-identical to the fused sketch epilogue.  A~: ld = n. */
CSK_API csk_status_t csk_row_norms(csk_ctx_t ctx, const double *A_tilde, int64_t d, int64_t n,
                           double *nsq, void *stream);

/* ---- S5-S8: the Algorithm 1 loop ---------------------------------------------- */
/* csk_solve: x is x_0 on entry and the final iterate on exit.  One
 *   persistent cooperative kernel runs every iteration: GEMV r = b~ - A~ x_k,
 *   score r_i^2/nsq_i (rows with nsq_i = 0 masked), argmax with lowest-index
 *   ties, x_{k+1} = x_k + (r_ik/nsq_ik) A~^(ik)T, stop test; A~ rows stay
 *   on chip (registers, TMEM, shared memory; the remainder streams from
 *   L2/HBM through a TMA ring each iteration).
 *   x_star != NULL: stop when RES <= tol; NULL: residual mode,
 *   available on every tier.  In residual mode on one GPU the CTA partials of
 *   ||r_k||^2 are summed in arrival order, so the last bits of RES (and, at a
 *   RES within rounding of tol, the stop iteration) may differ run to run.
 *   Stops at max_iters (>= 0).  Blocks; fills *report (host pointer).
 *   Returns CSK_E_ZERO_SKETCH if every nsq is 0. */
CSK_API csk_status_t csk_solve(csk_ctx_t ctx, const double *A_tilde, const double *b_tilde,
                       const double *nsq, int64_t d, int64_t n, double *x,
                       const double *x_star, double tol, int64_t max_iters,
                       csk_report_t *report, void *stream);

CSK_API csk_status_t csk_solve_ex(csk_ctx_t ctx, const double *A_tilde, const double *b_tilde,
                          const double *nsq, int64_t d, int64_t n, double *x,
                          const double *x_star, double tol, int64_t max_iters,
                          const csk_solve_opts_t *opts, csk_report_t *report, void *stream);

/* After csk_solve_ex(..., flags = CSK_SOLVE_ASYNC): synchronise the stream of the last
 * solve on this ctx and fill *report (host).  Returns that solve's status
 * (e.g. CSK_E_ZERO_SKETCH).  x is valid only after this returns. */
CSK_API csk_status_t csk_solve_wait(csk_ctx_t ctx, csk_report_t *report);

/* Per-kernel timing for the roofline (bench.py): with timing on, the library records CUDA
 * events on the launching stream right around the sketch kernel (k_sketch_dense, which = 0) and
 * the loop kernel (k_loop, which = 1).  csk_last_kernel_ms synchronises on the end event and
 * returns the last launch's duration in ms.  Off by default (no events recorded). */
CSK_API csk_status_t csk_ctx_set_timing(csk_ctx_t ctx, int32_t on);
CSK_API csk_status_t csk_last_kernel_ms(csk_ctx_t ctx, int32_t which, float *ms);

/* Launch geometry the last csk_solve* on this ctx used: CTAs, CTAs per cluster, rows of
 * A~ kept in shared memory per CTA (any pointer may be NULL). */
CSK_API csk_status_t csk_last_solve_geometry(csk_ctx_t ctx, int32_t *num_ctas, int32_t *cluster_size,
                                             int32_t *smem_rows);

/* Row tiers of the last csk_solve* on this ctx, per row group of a CTA (loop.cu): out[0] CTAs,
 * out[1] CTAs per cluster, out[2] register rows, out[3] TMEM rows, out[4] shared-memory rows,
 * out[5] warps per group, out[6] stream-ring stages, out[7] rows per stage (0: no ring; rows
 * past out[2] + out[3] + out[4] are re-read from L2/HBM every iteration).  out: 8 int32 (host). */
CSK_API csk_status_t csk_last_solve_tiers(csk_ctx_t ctx, int32_t *out);

/* ---- Whole Algorithm 1 (INPUT A, b, d, x0 -> OUTPUT x) ---------------- */
/* Plan + sketch + norms + loop on device buffers (workspace for A~, b~, nsq owned
 * by ctx).  Blocks; fills *report. */
CSK_API csk_status_t csk_run(csk_ctx_t ctx, const double *A, int64_t lda, const double *b,
                     int64_t m, int64_t n, int64_t d, uint64_t seed, double *x,
                     const double *x_star, double tol, int64_t max_iters,
                     csk_report_t *report, void *stream);

/* Same with HOST buffers (A_host: m x lda, b_host: m, x_host: n in/out,
 * x_star_host: n or NULL).  Copies in, runs csk_run, copies x back; pinned host
 * memory gives full PCIe bandwidth.  Blocks. */
CSK_API csk_status_t csk_run_host(csk_ctx_t ctx, const double *A_host, int64_t lda, const double *b_host,
                          int64_t m, int64_t n, int64_t d, uint64_t seed, double *x_host,
                          const double *x_star_host, double tol, int64_t max_iters,
                          csk_report_t *report, void *stream);

/* ---- S9/S10: row-sharded multi-GPU path (one process per GPU, NCCL) --------------- */
/* Bucket ownership: rank p of P owns rows [p c, min((p+1) c, total)) of A~, c = ceil(total/P)
 * (equal blocks, as ncclReduceScatter requires).  Host-only, no GPU needed. */
CSK_API csk_status_t csk_shard_range(int64_t total, int32_t nranks, int32_t rank, int64_t *lo,
                                     int64_t *hi);

/* NCCL bootstrap: rank 0 calls csk_comm_unique_id (128 host bytes), the caller broadcasts the
 * bytes (e.g. torch.distributed), every rank calls csk_comm_create.  One comm per ctx. */
CSK_API csk_status_t csk_comm_unique_id(void *uid_out);
CSK_API csk_status_t csk_comm_create(csk_ctx_t ctx, const void *uid, int32_t nranks, int32_t rank);
CSK_API csk_status_t csk_comm_destroy(csk_ctx_t ctx);

/* S9 (north_star "NCCL reduce-scatter of partial A~ by bucket range"): this rank holds rows
 * [row_offset, row_offset + m_local) of A (m rows in total) and hashes them with their GLOBAL
 * indices, so the union over ranks is exactly S A.  On return this rank owns A~ rows
 * [*d_lo, *d_hi) (csk_shard_range(d, P, rank)) in A_tilde_local ((d_hi-d_lo) x n), b~ rows in
 * b_tilde_local and, if nsq_local != NULL, their squared norms.  Partial sums are combined by
 * ncclReduceScatter(sum): A~ equals the P = 1 result up to summation order.
 * Collective: every rank must call it.  Blocks only as NCCL does. */
CSK_API csk_status_t csk_sketch_sharded(csk_ctx_t ctx, const double *A_local, int64_t lda,
                                        const double *b_local, int64_t m_local, int64_t row_offset,
                                        int64_t m, int64_t n, int64_t d, uint64_t seed,
                                        double *A_tilde_local, double *b_tilde_local,
                                        double *nsq_local, int64_t *d_lo, int64_t *d_hi,
                                        void *stream);

/* S9 for CSR input (config C5: "sketch and iteration row-sharded").  This rank holds rows
 * [row_offset, row_offset + m_local) of the CSR matrix: row_ptr (int64[m_local + 1]) indexes the
 * given col (int32) / val (fp64) arrays (absolute offsets; any base), b_local fp64[m_local].  Rows
 * are hashed with their GLOBAL index.  On return this rank owns A~ rows [*d_lo, *d_hi) =
 * csk_shard_range(d, P, rank) in A_tilde_local ((d_hi - d_lo) x n), b~ in b_tilde_local and, if
 * nsq_local != NULL, their norms.  mode:
 *   CSK_SHARD_REDUCE_SCATTER  partial (A~ | b~) over all d buckets, ncclReduceScatter(sum)
 *                             (north_star; equal to P = 1 up to summation order);
 *   CSK_SHARD_ROUTE_ROWS      every row is sent to the owner of its bucket (grouped ncclSend /
 *                             ncclRecv: the CSR bytes, not d x n partials) and the owner folds
 *                             its buckets in ascending global row order: BIT-IDENTICAL to P = 1
 *                             (the C5 variant).
 * Collective: every rank must call it with the same mode.  Blocks (a count exchange). */
#define CSK_SHARD_REDUCE_SCATTER 0
#define CSK_SHARD_ROUTE_ROWS 1
CSK_API csk_status_t csk_sketch_csr_sharded(csk_ctx_t ctx, const int64_t *row_ptr, const int32_t *col,
                                            const double *val, const double *b_local, int64_t m_local,
                                            int64_t row_offset, int64_t m, int64_t n, int64_t d,
                                            uint64_t seed, int32_t mode, double *A_tilde_local,
                                            double *b_tilde_local, double *nsq_local, int64_t *d_lo,
                                            int64_t *d_hi, void *stream);

/* The row-routing decomposition with `nranks` virtual ranks on this one GPU (test hook): the rows
 * are split into nranks contiguous shards, each shard packed by destination owner (the buffers
 * CSK_SHARD_ROUTE_ROWS hands to NCCL), moved by device copies, and every owner's bucket range
 * sketched into A_tilde (d x n) / b_tilde / nsq (full size).  Must equal csk_sketch_csr bit for bit. */
CSK_API csk_status_t csk_sketch_csr_routed_virtual(csk_ctx_t ctx, const int64_t *row_ptr, const int32_t *col,
                                                   const double *val, const double *b, int64_t m, int64_t n,
                                                   int64_t d, uint64_t seed, int32_t nranks, double *A_tilde,
                                                   double *b_tilde, double *nsq, void *stream);

/* S10: Algorithm 1 with the rows of A~ sharded across ranks (rows [d_lo, d_hi) here) and x
 * replicated.  Per iteration: local GEMV + argmax, one ncclAllGather of (score, global row,
 * lambda, sum r^2, winning local row), identical winner/update on every rank (ties -> lowest
 * global row).  Collective; blocks; fills *report (identical on every rank). */
CSK_API csk_status_t csk_solve_sharded(csk_ctx_t ctx, const double *A_tilde_local,
                                       const double *b_tilde_local, const double *nsq_local,
                                       int64_t d_lo, int64_t d_hi, int64_t d, int64_t n, double *x,
                                       const double *x_star, double tol, int64_t max_iters,
                                       csk_report_t *report, void *stream);

/* The same sharded loop with `nranks` virtual ranks on this one GPU (loopback exchange):
 * A_tilde is the full d x n sketch, virtual rank p owns csk_shard_range(d, nranks, p).
 * x_copies (optional, nranks x n) receives every virtual rank's final x (they must agree). */
CSK_API csk_status_t csk_solve_virtual_ranks(csk_ctx_t ctx, const double *A_tilde,
                                             const double *b_tilde, const double *nsq, int64_t d,
                                             int64_t n, int32_t nranks, double *x,
                                             const double *x_star, double tol, int64_t max_iters,
                                             double *x_copies, csk_report_t *report, void *stream);
/* Same with the csk_solve_opts_t traces (idx/res/x traces of virtual rank 0, r_trace indexed by
 * GLOBAL row: every virtual rank writes its own rows).  Launch knobs in opts are ignored. */
CSK_API csk_status_t csk_solve_virtual_ranks_ex(csk_ctx_t ctx, const double *A_tilde,
                                                const double *b_tilde, const double *nsq, int64_t d,
                                                int64_t n, int32_t nranks, double *x,
                                                const double *x_star, double tol, int64_t max_iters,
                                                double *x_copies, const csk_solve_opts_t *opts,
                                                csk_report_t *report, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* CSK_H_ */
