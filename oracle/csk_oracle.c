/*
 * csk_oracle.c -- plain, slow, single-threaded CPU ORACLE for the Count-Sketch
 * Kaczmarz (CSK) hot path of Zhang & Li, arXiv 2004.02480.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2004_02480_b200/) never imports, links or calls it, and this file shares
 * no header, helper, constant table or generator with csrc/.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section / equation /
 * algorithm in brackets).  "S:n" = SPEC.md line n (interfaces and worked
 * examples only).  "R-k" = a reading of the paper recorded in DESIGN.md §3.
 *
 * Build: gcc -std=c99 -O2 -ffp-contract=off -fPIC -shared (no BLAS, no OpenMP).
 * Every floating-point step is fp64; every fused multiply-add is an explicit
 * fma() call so the arithmetic is fixed by this source, not by the compiler.
 *
 * Pinning (tests/test_oracle_pins.py): every function below is pinned by
 * something other than itself -- published SplitMix64 vectors, the dense
 * definition S = Phi D (Def. 1) multiplied out by brute force, SPEC worked
 * examples, closed forms, proof identities eq:A / eq:5 / eq:6, the
 * Theorem 2 rate with the exact distortion and the paper's Table 1
 * iteration means.  See DESIGN.md §4 for the pin matrix.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* O-1  The random map h : [m] -> [d] and the diagonal D = diag(s)          */
/*      (Definition 1; PRNG fixed by BASELINE north_star "splitmix64   */
/*      of (seed, i)"; reading R-1: sequential stream, h from draw 2i,       */
/*      sign from draw 2i+1, h = floor(z * d / 2^64)).                       */
/* ------------------------------------------------------------------------ */

/* One step of the SplitMix64 generator (Steele, Lea & Flood 2014): the state
 * advances by the golden-ratio increment and the output is the mixed state. */
uint64_t oracle_splitmix64_next(uint64_t *state)
{
    uint64_t z;
    *state = *state + 0x9E3779B97F4A7C15ULL;
    z = *state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* floor(z * d / 2^64) written as a schoolbook 64x64 -> 128 bit product,
 * keeping the high word (no compiler 128-bit extension needed). */
static uint64_t oracle_mulhi64(uint64_t a, uint64_t b)
{
    uint64_t a_lo = a & 0xFFFFFFFFULL, a_hi = a >> 32;
    uint64_t b_lo = b & 0xFFFFFFFFULL, b_hi = b >> 32;
    uint64_t lo_lo = a_lo * b_lo;
    uint64_t hi_lo = a_hi * b_lo;
    uint64_t lo_hi = a_lo * b_hi;
    uint64_t hi_hi = a_hi * b_hi;
    uint64_t cross = (lo_lo >> 32) + (hi_lo & 0xFFFFFFFFULL) + lo_hi;
    return hi_hi + (hi_lo >> 32) + (cross >> 32);
}

/* Draw h[0..m) and s[0..m) from one sequential SplitMix64 stream seeded with
 * `seed`:  for i = 0..m-1: z_h = next(); z_s = next();
 *          h[i] = floor(z_h * d / 2^64);  s[i] = (z_s >> 63) ? -1 : +1.
 * Each h(i) is uniform on [0,d) up to a bias <= d/2^64 and each s[i] is +-1
 * with probability 1/2, independently per i. */
void oracle_hash(uint64_t seed, int64_t m, int64_t d, int32_t *h, int8_t *s)
{
    uint64_t state = seed;
    int64_t i;
    for (i = 0; i < m; ++i) {
        uint64_t z_h = oracle_splitmix64_next(&state);
        uint64_t z_s = oracle_splitmix64_next(&state);
        h[i] = (int32_t)oracle_mulhi64(z_h, (uint64_t)d);
        s[i] = (int8_t)((z_s >> 63) ? -1 : 1);
    }
}

/* ------------------------------------------------------------------------ */
/* O-2  A~ = S A, b~ = S b with S = Phi D (Algorithm 1 "Initialize";   */
/*      Def. 1).  Row i of A contributes s[i] * A^(i) to row h[i].     */
/*      Accumulation starts at +0.0 and follows increasing source row i     */
/*      ("accumulation in source-row order"), which is exactly the    */
/*      dense product Phi*D*A evaluated column by column in row order.       */
/* ------------------------------------------------------------------------ */
void oracle_sketch_dense(const double *A, int64_t lda, const double *b,
                         int64_t m, int64_t n, int64_t d,
                         const int32_t *h, const int8_t *s,
                         double *At, double *bt)
{
    int64_t i, j, k;
    for (j = 0; j < d * n; ++j) At[j] = 0.0;
    for (j = 0; j < d; ++j) bt[j] = 0.0;
    for (i = 0; i < m; ++i) {
        double si = (double)s[i];
        double *row = At + (int64_t)h[i] * n;
        for (k = 0; k < n; ++k) row[k] = row[k] + si * A[i * lda + k];
        bt[h[i]] = bt[h[i]] + si * b[i];
    }
}

/* Same definition for A stored as CSR (row_ptr[m+1], col[nnz], val[nnz]); a
 * row's stored (col, val) pairs are visited in stored order.  Columns within
 * one row are distinct, so per output entry the adds still follow row order. */
void oracle_sketch_csr(const int64_t *row_ptr, const int32_t *col,
                       const double *val, const double *b,
                       int64_t m, int64_t n, int64_t d,
                       const int32_t *h, const int8_t *s,
                       double *At, double *bt)
{
    int64_t i, j, t;
    for (j = 0; j < d * n; ++j) At[j] = 0.0;
    for (j = 0; j < d; ++j) bt[j] = 0.0;
    for (i = 0; i < m; ++i) {
        double si = (double)s[i];
        double *row = At + (int64_t)h[i] * n;
        for (t = row_ptr[i]; t < row_ptr[i + 1]; ++t)
            row[col[t]] = row[col[t]] + si * val[t];
        bt[h[i]] = bt[h[i]] + si * b[i];
    }
}

/* ------------------------------------------------------------------------ */
/* O-3  nsq_j = ||A~^(j)||_2^2 (P:62 denominator, squared as in P:122),     */
/*      fma-accumulated left to right over columns.                  */
/* ------------------------------------------------------------------------ */
void oracle_row_norms(const double *At, int64_t d, int64_t n, double *nsq)
{
    int64_t j, k;
    for (j = 0; j < d; ++j) {
        double acc = 0.0;
        for (k = 0; k < n; ++k) acc = fma(At[j * n + k], At[j * n + k], acc);
        nsq[j] = acc;
    }
}

/* r = b~ - A~ x, each dot product fma-accumulated left to right (P:62
 * numerator "b~^(i) - A~^(i) x_k"). */
void oracle_residual(const double *At, const double *bt, int64_t d, int64_t n,
                     const double *x, double *r)
{
    int64_t i, k;
    for (i = 0; i < d; ++i) {
        double acc = 0.0;
        for (k = 0; k < n; ++k) acc = fma(At[i * n + k], x[k], acc);
        r[i] = bt[i] - acc;
    }
}

/* ------------------------------------------------------------------------ */
/* O-4  Algorithm 1 loop with the paper's stopping rule.  */
/* ------------------------------------------------------------------------ */

/* Termination codes. */
#define ORACLE_CONVERGED 0
#define ORACLE_MAX_ITERS 1
#define ORACLE_STAGNATED 2
#define ORACLE_ERR_ZERO_SKETCH (-2)
#define ORACLE_ERR_ARG (-1)

/* RES = ||x - x*||^2 / ||x*||^2, both sums left to right.  If
 * ||x*|| = 0 the absolute squared error is used (reading R-9). */
static double oracle_res(const double *x, const double *xs, int64_t n)
{
    double num = 0.0, den = 0.0;
    int64_t k;
    for (k = 0; k < n; ++k) {
        double e = x[k] - xs[k];
        num = fma(e, e, num);
        den = fma(xs[k], xs[k], den);
    }
    return den > 0.0 ? num / den : num;
}

/*
 * oracle_solve -- x is x_0 on entry and the final iterate on exit.
 *
 * For k = 0, 1, ...:
 *   1. (x_star != NULL) RES_k = ||x_k - x*||^2/||x*||^2; RES_k <= tol ->
 *      Converged with IT = k ("RES <= 10^-6").  k == max_iters ->
 *      MaxIters (P:180 cap; configs use 50k, reading R-5).
 *   2. r_i = b~_i - A~^(i) x_k for every i;
 *      score_i = r_i^2 / nsq_i (squared form; reading R-3), rows
 *      with nsq_i = 0 are masked with score -1 (reading R-4).
 *      (x_star == NULL) residual mode: ||r_k||^2/||b~||^2 <= tol -> Converged
 *      (reading R-8); k == max_iters -> MaxIters.
 *   3. i_k = first i with the largest score (lowest-index ties, north_star).
 *      score_{i_k} == 0 while not converged -> Stagnated.
 *   4. x_{k+1} = x_k + (r_{i_k}/nsq_{i_k}) A~^(i_k)T, elementwise fma.
 *
 * Traces (optional, may be NULL): idx_trace[k] = i_k, res_trace[k] = the
 * stop quantity at iterate k (k = 0..IT), x_trace[(k)*n ..] = x_k for
 * k = 0..min(IT, trace_cap-1).  trace_cap bounds every trace.
 * Returns the termination code (>= 0) or a negative error.
 */
int oracle_solve(const double *At, const double *bt, const double *nsq,
                 int64_t d, int64_t n, double *x, const double *x_star,
                 double tol, int64_t max_iters,
                 int64_t *iters_out, double *final_res_out, int64_t *last_idx_out,
                 int64_t *idx_trace, double *res_trace, double *x_trace,
                 int64_t trace_cap, double *r_work)
{
    int64_t i, k, j, it;
    int any_row = 0;
    double bb = 0.0;
    int64_t last = -1;

    if (d <= 0 || n <= 0 || tol <= 0.0 || max_iters < 0) return ORACLE_ERR_ARG;
    for (i = 0; i < d; ++i) if (nsq[i] > 0.0) any_row = 1;
    if (!any_row) return ORACLE_ERR_ZERO_SKETCH;
    if (x_star == NULL) {
        for (i = 0; i < d; ++i) bb = fma(bt[i], bt[i], bb);
    }

    for (it = 0;; ++it) {
        double stop_val;
        double best = -2.0;
        int64_t ik = -1;
        double lambda;

        if (x_trace != NULL && it < trace_cap)
            for (j = 0; j < n; ++j) x_trace[it * n + j] = x[j];

        if (x_star != NULL) {
            stop_val = oracle_res(x, x_star, n);
            if (res_trace != NULL && it < trace_cap) res_trace[it] = stop_val;
            if (stop_val <= tol) {
                *iters_out = it; *final_res_out = stop_val; *last_idx_out = last;
                return ORACLE_CONVERGED;
            }
            if (it == max_iters) {
                *iters_out = it; *final_res_out = stop_val; *last_idx_out = last;
                return ORACLE_MAX_ITERS;
            }
        }

        oracle_residual(At, bt, d, n, x, r_work);

        if (x_star == NULL) {
            double rr = 0.0;
            for (i = 0; i < d; ++i) rr = fma(r_work[i], r_work[i], rr);
            stop_val = bb > 0.0 ? rr / bb : rr;
            if (res_trace != NULL && it < trace_cap) res_trace[it] = stop_val;
            if (stop_val <= tol) {
                *iters_out = it; *final_res_out = stop_val; *last_idx_out = last;
                return ORACLE_CONVERGED;
            }
            if (it == max_iters) {
                *iters_out = it; *final_res_out = stop_val; *last_idx_out = last;
                return ORACLE_MAX_ITERS;
            }
        }

        for (i = 0; i < d; ++i) {
            double score = nsq[i] > 0.0 ? (r_work[i] * r_work[i]) / nsq[i] : -1.0;
            if (score > best) { best = score; ik = i; }
        }
        if (best == 0.0) {
            *iters_out = it; *final_res_out = stop_val; *last_idx_out = last;
            return ORACLE_STAGNATED;
        }
        if (idx_trace != NULL && it < trace_cap) idx_trace[it] = ik;

        lambda = r_work[ik] / nsq[ik];
        for (k = 0; k < n; ++k) x[k] = fma(lambda, At[ik * n + k], x[k]);
        last = ik;
    }
}
