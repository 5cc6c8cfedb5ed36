// loop.cu -- S5..S8: the Algorithm 1 loop as ONE persistent kernel, A~ held
// on chip (registers, then TMEM, then shared memory; rows past those re-read from L2/HBM
// through a TMA ring), one flat atomic exchange per iteration.
//
// Grid: G cooperative CTAs (default: one per SM), 8 warps each (C1/C2-sized systems: one
// 16-CTA cluster with a DSMEM exchange instead).  CTA c owns the contiguous rows
// [d c/G, d (c+1)/G) of A~.  Its warps form RG = 8/WPG row groups of WPG warps (TG = 32 WPG
// threads); group g owns a balanced contiguous slice of the CTA's rows, and thread t of a group
// owns the columns c_q = t + TG q (q < CB), so every group holds all n columns and keeps its own
// copy of x_k in registers (CB doubles per thread).  Row i of a group lives in
//   i <  rr                 : registers   (a[i][q], CB doubles per row per thread)
//   rr <= i < rr + rt       : TMEM (CB = 8: 16 TMEM columns per row in the thread's lane)
//   ... < rr + rt + rs      : shared memory, [i][q/2][t][2] (16-byte words, conflict-free)
//   otherwise               : streamed from L2/HBM every iteration (TMA ring, ST variants)
//
// Iteration k (no launch, no grid barrier beyond the exchange itself):
//   S6  GEMV: thread partials sum_q fma(a[i][q], x_q) in q order; rows reduce across the warp
//       with a transposed shuffle tree (row i ends in a fixed lane group); a full TMEM tier and
//       the shared-memory rows go through one interleaved pass and one 32-row tree (C4);
//       warp partials of a row are added in warp order.  Fixed order everywhere -> identical
//       bits in every run.
//   S5  RES_k = ||x_k - x*||^2 / ||x*||^2 from the last group's registers, in every CTA
//       (identical arithmetic -> every CTA takes the same stop decision, no communication).
//   S7  score_i = r_i^2/nsq_i (masked rows never win).  A row's 64-bit key is
//       (score bits >> (b-1)) << b | (2^b - 1 - i), b = bits(d+1): max key = max score,
//       ties (equal in the kept 53-b mantissa bits) -> lowest row index (R-15).
//       CTA argmax -> one red.max.u64 of the key + one red.release.add of an arrival
//       counter on the same 16-byte pair; warp 0 polls {count, max} with relaxed 16-byte loads
//       until all G CTAs arrived (3 rotating pairs, CTA 0 clears the next; DESIGN.md section 6,
//       memory-model note).
//   S8  every CTA TMA-copies the winner's (lambda, score) slot and A~^(ik) into shared memory
//       and applies x_q += lambda a_ik[c_q] with the same fma in every copy, so all copies of x
//       stay bit-identical.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "csk_internal.cuh"

// 1: read the exchange pair the PTX-model way (an acquire fence after the poll, then a re-read)
#ifndef CSK_STRICT_ACQUIRE
#define CSK_STRICT_ACQUIRE 0
#endif

namespace csk {

namespace {

constexpr int kLW = 8;             // warps per CTA
constexpr int kTmRowsDev = 16;     // rows per thread in the TMEM tier (kTmRows)
constexpr int kLT = kLW * 32;      // threads per CTA
constexpr int kXchWords = 16;      // one 128-byte line per {count, max} pair
// after the 3 pairs: [2 parities][kMaxRanks] LL key slots (16 B each) of the cross-GPU exchange
constexpr int kKeySlotWords = 2 * kMaxRanks * 2 * 2;  // per parity and rank: the LL key, then the LL ||r||^2 sum
// then (SYS, P > 1) two row-staging buffers: one 128-B flag line, then [2][CSK_MAX_N] doubles --
// the winner's row is fetched over NVLink once per GPU, not once per CTA
constexpr size_t kStageFlagOff = static_cast<size_t>(3) * kXchWords * 8 + kKeySlotWords * 8;  // bytes
constexpr size_t kStageRowOff = kStageFlagOff + 128;
constexpr size_t kXchBytes = kStageRowOff + static_cast<size_t>(2) * CSK_MAX_N * 8;
constexpr int kSlotWords = 8;      // LL slot: lambda, score as tagged 32-bit halves + pad (64 B)

struct LoopParams {
    const double *At;
    const double *bt;
    const double *nsq;
    int64_t d, n;
    double *x;
    const double *x_star;
    double tol;
    int64_t max_iters;
    unsigned long long *xch;  // [3][kXchWords]: {count, max key}
    unsigned long long *slots;  // [2][G][kSlotWords] LL-tagged (tag = k + 1 in every 8-byte word)
    int64_t *report;          // [0]=iterations, [1]=final_res bits, [2]=termination, [3]=last idx
    const double *bb;         // residual mode: ||b~||^2 (device scalar)
    int wpg;                  // warps per row group (1, 2, 4, 8)
    int fuse_ts;              // full TMEM tier + shared-memory rows in one interleaved pass
    int npoll;                // exchange polls in flight per CTA (1: one at a time)
    int pdelay;               // cycles between their first issues
    int rr;                   // rows per group held in registers (<= RRMAX)
    int rs;                   // rows per group held in shared memory
    int rt;                   // rows per group held in tensor memory (TM variants, <= 16)
    int key_bits;             // b
    int rows_max;             // max rows per CTA (sizes the shared-memory carve-up)
    int64_t trace_cap;
    int64_t *idx_trace;
    double *res_trace;
    double *x_trace;
    double *r_trace;          // [r_trace_cap][d_glob]: r_k by GLOBAL row (csk_solve_opts_t), or null
    int64_t r_trace_cap;
    int64_t d_glob;           // rows of A~ over all ranks (the r_trace leading dimension)
    int64_t *phase_cycles;    // debug (libcsk_prof.so only): [2 warps][16] SM-cycle totals of CTA 0
    long long *skew;          // debug (libcsk_prof.so only): [64 iterations][2][G] globaltimer ns
    // ---- row sharding over P ranks (S10).  P = 1: one GPU.  rank >= 0: this launch is rank
    //      `rank` of P GPUs (the other ranks' arrays are peer-mapped; sys = 1).  rank = -1: P
    //      virtual ranks in ONE launch (rank = cta / Gr), the 1-GPU test of the decomposition.
    int P, rank, Gr, sys;
    unsigned long long timeout_ns;          // exchange watchdog
    int64_t dlo[kMaxRanks + 1];             // rank r owns the global rows [dlo[r], dlo[r+1])
    int RMr[kMaxRanks];                     // rank r's rows per CTA, ceil((dlo[r+1]-dlo[r]) / Gr)
    int st_rows, st_stages;                 // ST variants: rows per stream-ring stage, stages per row group
    int st_rest_first;                      // ST: the chunks past st_pin are copied evict_first (1) or without a hint (0)
    int st_pin;                             // ST: each group's first st_pin chunks are kept in L2 (evict_last), the rest evict_first; < 0: no hints
    unsigned long long rm_magic;            // P = 1: ceil(2^40 / RM) if (d-1) RM < 2^40 (row -> CTA by a multiply), else 0
    const double *At_r[kMaxRanks];          // rank r's rows of A~ (row dlo[r] first)
    const double *bt_r[kMaxRanks];
    const double *nsq_r[kMaxRanks];
    unsigned long long *slots_r[kMaxRanks];  // rank r's LL slots [2][Gr][kSlotWords]
    unsigned long long *xch_r[kMaxRanks];    // SYS: rank r's exchange region (its pairs, then its key slots)
    double *x_r[kMaxRanks];                 // rank r's output x (virtual: per-rank copies)
};

// ---- PTX helpers specific to the exchange ----
__device__ __forceinline__ void red_max_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add_release_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add_f64(double *p, double v) {
    asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
// {count, max, sum} of one pair in one 32-byte load (one L2 sector: read as one snapshot)
__device__ __forceinline__ void ld_relaxed_v4(const unsigned long long *p, unsigned long long &a,
                                              unsigned long long &b, unsigned long long &c) {
    unsigned long long d;
    asm volatile("ld.relaxed.gpu.global.v4.u64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p) : "memory");
}
// system-scope variants for the cross-GPU exchange (peer memory over NVLink)
__device__ __forceinline__ void red_max_u64_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("red.relaxed.sys.global.max.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add_release_u64_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void ld_relaxed_v2_sys(const unsigned long long *p, unsigned long long &a,
                                                  unsigned long long &b) {
    asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ void st_relaxed_v2_u64_sys(unsigned long long *p, unsigned long long a,
                                                      unsigned long long b) {
    asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void st_relaxed_v2_u64(unsigned long long *p, unsigned long long a,
                                                  unsigned long long b) {
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
// LL (low-latency) encoding: a double as two 8-byte words {32 data bits | 32-bit tag}; 8-byte
// aligned accesses are single-copy atomic, so a reader that sees the tag in both words holds
// a consistent value without any fence.
__device__ __forceinline__ void ll_pack(double v, uint32_t tag, unsigned long long &hi, unsigned long long &lo) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    hi = (b & 0xffffffff00000000ull) | tag;
    lo = (b << 32) | tag;
}
__device__ __forceinline__ bool ll_ok(unsigned long long hi, unsigned long long lo, uint32_t tag) {
    return static_cast<uint32_t>(hi) == tag && static_cast<uint32_t>(lo) == tag;
}
__device__ __forceinline__ double ll_val(unsigned long long hi, unsigned long long lo) {
    return __longlong_as_double(static_cast<long long>((hi & 0xffffffff00000000ull) | (lo >> 32)));
}
__device__ __forceinline__ void ld_relaxed_v2_u64(const unsigned long long *p, unsigned long long &a,
                                                  unsigned long long &b) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
// spin until the LL-tagged double at p (2 words) carries `tag` (sys: a peer GPU's memory)
__device__ __forceinline__ double ll_load(const unsigned long long *p, uint32_t tag, bool sys = false) {
    unsigned long long hi, lo;
    do {
        if (sys) ld_relaxed_v2_sys(p, hi, lo);
        else ld_relaxed_v2_u64(p, hi, lo);
    } while (!ll_ok(hi, lo, tag));
    return ll_val(hi, lo);
}
__device__ __forceinline__ void ld_relaxed_v2(const unsigned long long *p, unsigned long long &a,
                                              unsigned long long &b) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
// order this thread's generic-proxy view of global memory before its later async-proxy (TMA) reads
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ double lwarp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// 64-bit key of row i with score s (see header).  Masked rows (s < 0) -> 0.
__device__ __forceinline__ unsigned long long row_key(double s, int64_t i, int b) {
    if (!(s >= 0.0)) return 0ull;
    const unsigned long long sb = static_cast<unsigned long long>(__double_as_longlong(s));
    const unsigned long long mask = (1ull << b) - 1ull;
    return ((sb >> (b - 1)) << b) | (mask - static_cast<unsigned long long>(i));
}

// Warp max of a 64-bit key (unique per row): the lane holding it (keys 0 -> lane 0).
__device__ __forceinline__ int warp_max_key_lane(unsigned long long key, unsigned long long &kmax) {
    const uint32_t kh = static_cast<uint32_t>(key >> 32), kl = static_cast<uint32_t>(key);
    const uint32_t hi = __reduce_max_sync(0xffffffffu, kh);
    const uint32_t lo = __reduce_max_sync(0xffffffffu, kh == hi ? kl : 0u);
    kmax = (static_cast<unsigned long long>(hi) << 32) | lo;
    const unsigned bal = __ballot_sync(0xffffffffu, key == kmax);
    return bal ? __ffs(bal) - 1 : 0;
}

// Transposed reduction of V per-lane row partials over the 32 lanes: afterwards lanes
// [r 32/V, (r+1) 32/V) all hold the warp sum of row r (fixed tree, identical bits).
template <int V>
__device__ __forceinline__ double treduce(double (&v)[V], int lane) {
    int cnt = V;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        if (cnt > 1) {
            const int half = cnt >> 1;
            const bool upper = (lane & o) != 0;
#pragma unroll
            for (int j = 0; j < V / 2; ++j) {
                if (j < half) {
                    const double send = upper ? v[j] : v[j + half];
                    const double keep = upper ? v[j + half] : v[j];
                    v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
            cnt = half;
        } else {
            v[0] = v[0] + __shfl_xor_sync(0xffffffffu, v[0], o);
        }
    }
    return v[0];
}

// One level (lane mask o, cnt rows still live) of treduce<V>: the same adds in the same order,
// so a tree run level by level (interleaved with other work) gives treduce's bits.
template <int V>
__device__ __forceinline__ void treduce_level(double (&v)[V], int lane, int o, int cnt) {
    if (cnt > 1) {
        const int half = cnt >> 1;
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int j = 0; j < V / 2; ++j) {
            if (j < half) {
                const double send = upper ? v[j] : v[j + half];
                const double keep = upper ? v[j + half] : v[j];
                v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
    } else {
        v[0] = v[0] + __shfl_xor_sync(0xffffffffu, v[0], o);
    }
}

template <int N>
struct Pow2Ceil {
    static constexpr int v = N <= 1 ? 1 : N <= 2 ? 2 : N <= 4 ? 4 : N <= 8 ? 8 : N <= 16 ? 16 : 32;
};

// Shared-memory carve-up (bytes), identical on host and device.
constexpr int kCS = 16;               // cluster size of the cluster-exchange variant
constexpr int64_t kCluMaxElems = 640 * 1024;  // d n up to which one 16-SM cluster beats 148 SMs
constexpr size_t kInboxOff = 576;      // [2 parities][kCS][4] doubles: key, lambda, score, rr
constexpr size_t kXbarOff = 1600;      // 2 mbarriers (one per parity), kCS arrivals each
constexpr size_t kRowbufOff = 1664;
struct LoopSmem {
    size_t ctl, mbar, slotbuf, cand, resp, btl, invl, dotp, xs, rowbuf, arows, ring, rbar, total;
};
// Streamed rows kept resident in L2 (copied evict_last; the other streamed rows evict_first): 96 MB of
// the 126 MB L2 measured best on the B200 (C5 loop 88.5 -> 85.6 us/iteration, MWRK on C3 54.1 -> 50.5;
// 128 MB and above falls back to the unhinted time), and only for ring chunks of at least 16 KB (with
// 4.8-8 KB chunks the hinted copies measured 4-6 % slower).  profiles/r02_l2pin_ab.txt.
constexpr int kLoopL2PinMB = 96;           // CSK_LOOP_L2PIN_MB overrides (0: no hints)
constexpr int kLoopL2PinMinChunk = 16000;  // bytes; CSK_LOOP_L2PIN_MINCHUNK overrides
// Bytes of one stream-ring stage: st_rows whole rows of A~ (a 128-B multiple)
__host__ __device__ inline size_t st_stage_bytes(int64_t n, int st_rows) {
    return (static_cast<size_t>(st_rows) * static_cast<size_t>(n) * 8 + 127) & ~size_t(127);
}
__host__ __device__ inline LoopSmem loop_smem(int rows_max, int wpg, int cb, int64_t n, int rs, int st_stages = 0,
                                              int st_rows = 0) {
    // The fixed-size control words and the winner-row buffer come first, at compile-time
    // offsets: the hot loop then addresses them from the shared-memory base without keeping
    // (or rematerialising) pointers in registers.
    LoopSmem L;
    L.ctl = 0;        // 64 B
    L.mbar = 64;      // 16 B
    L.slotbuf = 128;  // 64 B
    L.cand = 192;     // kLW x 32 B
    L.resp = 448;     // 16 doubles
    L.rowbuf = kRowbufOff;
    size_t o = kRowbufOff;
    auto take = [&](size_t bytes) { size_t r = o; o += (bytes + 127) & ~size_t(127); return r; };  // 128-B aligned
    const int tg = 32 * wpg;
    const size_t np = static_cast<size_t>(tg) * cb;  // padded width: the row buffer is zero past n
    take((np > static_cast<size_t>(n) ? np : static_cast<size_t>(n)) * 8);
    L.btl = take(static_cast<size_t>(rows_max) * 8);
    L.invl = take(static_cast<size_t>(rows_max) * 8);
    L.dotp = take(static_cast<size_t>(wpg) * rows_max * 8);
    L.xs = take(np * 8);
    L.arows = take(static_cast<size_t>(rs) * cb * kLT * 8);
    // streamed rows (ST variants): per row group st_stages stages of st_rows rows, and a
    // full / empty mbarrier pair per stage
    const int rg = kLW / wpg;
    L.ring = take(static_cast<size_t>(rg) * st_stages * st_stage_bytes(n, st_rows));
    L.rbar = take(static_cast<size_t>(rg) * st_stages * 16);
    L.total = o;
    return L;
}

// ---- tensor memory (TMEM) as a row tier: each thread keeps whole A~ row slices in its own
//      TMEM lane (warp w addresses lanes 32 (w mod 4) .. +31; warps w and w + 4 split the 512
//      columns), 32-bit column pairs hold one double ----
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// Issue only; the registers are written asynchronously until tmem_wait_ld(v), which names
// them as operands so the compiler cannot read them before the wait.
__device__ __forceinline__ void tmem_ld32_async(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld(uint32_t (&v)[32]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                   "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]),
                   "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]),
                   "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]), "+r"(v[30]), "+r"(v[31])
                 :);
}
__device__ __forceinline__ void tmem_ld16_async(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld16(uint32_t (&v)[16]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                   "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15])
                 :);
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ double dbl_of(uint32_t lo, uint32_t hi) {
    return __hiloint2double(static_cast<int>(hi), static_cast<int>(lo));
}

// NB TMEM rows (NB/2 tcgen05.ld of two rows each) folded against x: the next pair's load is in
// flight while the current pair is folded; each row folds its two column halves in separate
// chains (4 chains per pair), added at the end.
template <int NB, int CB>
__device__ __forceinline__ void tmem_block(uint32_t taddr, const double (&x)[CB], double (&acc)[NB]) {
    // one row (CB doubles = 16 TMEM columns) per tcgen05.ld; the next row's load is in flight
    // while the current row is folded in two chains (column halves), added at the end
    double lo[NB], hi[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) lo[j] = hi[j] = 0.0;
    uint32_t v[16];
    tmem_ld16_async(taddr, v);
    tmem_wait_ld16(v);
#pragma unroll
    for (int j = 0; j < NB; ++j) {
        uint32_t w[16];
        if (j + 1 < NB) tmem_ld16_async(taddr + 16u * (j + 1), w);
#pragma unroll
        for (int q = 0; q < CB / 2; ++q) {
            const int q2 = q + CB / 2;
            lo[j] = __fma_rn(dbl_of(v[2 * q], v[2 * q + 1]), x[q], lo[j]);
            hi[j] = __fma_rn(dbl_of(v[2 * q2], v[2 * q2 + 1]), x[q2], hi[j]);
        }
        if (j + 1 < NB) {
            tmem_wait_ld16(w);
#pragma unroll
            for (int t = 0; t < 16; ++t) v[t] = w[t];
        }
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) acc[j] = lo[j] + hi[j];
}

// Wide variant: two rows per tcgen05.ld (x32), the next pair in flight while the current pair is
// folded (4 chains per pair) -- half the waits of the one-row form, 64 staging registers.
template <int NB, int CB>
__device__ __forceinline__ void tmem_block_wide(uint32_t taddr, const double (&x)[CB], double (&acc)[NB]) {
    double lo[NB], hi[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) lo[j] = hi[j] = 0.0;
    uint32_t v[32];
    tmem_ld32_async(taddr, v);
    tmem_wait_ld(v);
#pragma unroll
    for (int j = 0; j < NB; j += 2) {
        uint32_t w[32];
        if (j + 2 < NB) tmem_ld32_async(taddr + 16u * (j + 2), w);
#pragma unroll
        for (int q = 0; q < CB / 2; ++q) {
            const int q2 = q + CB / 2;
            lo[j] = __fma_rn(dbl_of(v[2 * q], v[2 * q + 1]), x[q], lo[j]);
            lo[j + 1] = __fma_rn(dbl_of(v[16 + 2 * q], v[16 + 2 * q + 1]), x[q], lo[j + 1]);
            hi[j] = __fma_rn(dbl_of(v[2 * q2], v[2 * q2 + 1]), x[q2], hi[j]);
            hi[j + 1] = __fma_rn(dbl_of(v[16 + 2 * q2], v[16 + 2 * q2 + 1]), x[q2], hi[j + 1]);
        }
        if (j + 2 < NB) {
            tmem_wait_ld(w);
#pragma unroll
            for (int t = 0; t < 32; ++t) v[t] = w[t];
        }
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) acc[j] = lo[j] + hi[j];
}

// The full TMEM tier (16 rows) and up to RSM shared-memory rows in ONE pass: step j issues the
// tcgen05.ld.x32 of TMEM rows j, j+1, then the step's six shared-memory (row, column pair) units
// (LDS.128 + two FMAs each), and only then waits for the load and folds the two rows (two
// column-half chains each, added) -- the TMEM load latency hides behind the shared-memory loads
// and FMAs instead of being exposed after every load.  acc[0..15] = TMEM rows, acc[16 + i] =
// shared-memory row i (i < rs; rows past rs re-read row rs-1 and are never written back), the rest
// 0: one 32-row transposed tree follows.  Every row's partial has the order of the separate tier
// passes (tmem_block_wide, smem_block), and the 32-row tree adds the lanes in the same bit order as
// two 16-row trees, so the dot products are bit-identical to theirs.
template <int RSM, int VR = 1>
__device__ __forceinline__ void tmem_smem_fused(uint32_t taddr, const double *arows, int tg, int rs, int TG,
                                                 const double (&x)[8], double (&acc)[32],
                                                 double *racc = nullptr) {
    static_assert(RSM * 4 <= 48, "six shared-memory units per TMEM row pair");
    const double2 *a2 = reinterpret_cast<const double2 *>(arows) + tg;
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = 0.0;
#pragma unroll
    for (int j = 0; j < kTmRowsDev; j += 2) {
        uint32_t v[32];
        tmem_ld32_async(taddr + 16u * j, v);
#pragma unroll
        for (int u = 3 * j; u < 3 * j + 6; ++u) {
            const int i = u >> 2, qp = u & 3;
            if (i < RSM) {
                const int ii = i < rs ? i : rs - 1;
                const double2 val = a2[(static_cast<size_t>(ii) * 4 + qp) * TG];
                acc[16 + i] = __fma_rn(val.x, x[2 * qp], acc[16 + i]);
                acc[16 + i] = __fma_rn(val.y, x[2 * qp + 1], acc[16 + i]);
            }
        }
        if constexpr (VR > 1) {
            // the register rows' tree, one level per step (levels o = 16, 8, 4, 2, 1)
            if ((j >> 1) < 5) {
                const int lvl = j >> 1;
                int cnt = VR;
#pragma unroll
                for (int t = 0; t < 5; ++t)
                    if (t < lvl && cnt > 1) cnt >>= 1;
                treduce_level<VR>(*reinterpret_cast<double(*)[VR]>(racc), threadIdx.x & 31, 16 >> lvl, cnt);
            }
        }
        tmem_wait_ld(v);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            double lo = 0.0, hi = 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                lo = __fma_rn(dbl_of(v[16 * h + 2 * q], v[16 * h + 2 * q + 1]), x[q], lo);
                hi = __fma_rn(dbl_of(v[16 * h + 2 * q + 8], v[16 * h + 2 * q + 9]), x[q + 4], hi);
            }
            acc[j + h] = lo + hi;
        }
    }
}

// NB shared-memory rows (from i0, clamped to rs-1) folded against x: columns outer, rows inner.
// Layout [row][q/2][thread][2]: a thread's columns c_q, c_{q+1} sit in one 16-byte word.
template <int NB, int CB>
__device__ __forceinline__ void smem_block(const double *arows, int tg, int i0, int rs, int TG, const double (&x)[CB],
                                           double (&acc)[NB]) {
    static_assert(CB % 2 == 0 || CB == 1, "pairs of columns");
#pragma unroll
    for (int j = 0; j < NB; ++j) acc[j] = 0.0;
    if constexpr (CB == 1) {
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            const int jj = (i0 + j < rs) ? i0 + j : rs - 1;
            acc[j] = __fma_rn(arows[static_cast<size_t>(jj) * TG + tg], x[0], acc[j]);
        }
    } else {
        const double2 *a2 = reinterpret_cast<const double2 *>(arows) + tg;
#pragma unroll
        for (int qp = 0; qp < CB / 2; ++qp) {
#pragma unroll
            for (int j = 0; j < NB; ++j) {
                const int jj = (i0 + j < rs) ? i0 + j : rs - 1;
                const double2 v = a2[(static_cast<size_t>(jj) * (CB / 2) + qp) * TG];
                acc[j] = __fma_rn(v.x, x[2 * qp], acc[j]);
                acc[j] = __fma_rn(v.y, x[2 * qp + 1], acc[j]);
            }
        }
    }
}

// ---- cluster (DSMEM) exchange helpers ----
// 16-byte asynchronous store into a peer's shared memory that completes `bytes` on the peer's
// mbarrier (no fence, no arrival: the receiver armed the barrier with expect_tx)
__device__ __forceinline__ void st_async_v2_f64(uint32_t cluster_addr, double a, double b, uint32_t cluster_mbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(cluster_addr),
                 "d"(a), "d"(b), "r"(cluster_mbar)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait_cluster(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void group_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int CB, int RRMAX, bool RESMODE, int TM, bool CLU, bool ST = false, bool SYS = false>
__global__ void __launch_bounds__(kLT, 1) k_loop(const LoopParams p) {
    // CLU: the whole grid is one kCS-CTA thread-block cluster and the exchange is an
    // all-to-all of the CTA candidates over DSMEM (no global atomics)
    // TM: 0 no TMEM tier; 1 wide (two rows per tcgen05.ld); 2 narrow (one row per load, more
    // register rows).  The TMEM tier is laid out for 8 columns (16 TMEM columns) per row.
    static_assert(TM == 0 || CB == 8, "TMEM rows hold 8 columns per thread");
    constexpr int V = Pow2Ceil<RRMAX>::v;
    constexpr int LPR = 32 / V;  // lanes per row after the transposed tree
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int cta = blockIdx.x;
    const int64_t d = p.d;
    const int n = static_cast<int>(p.n);
    const int WPG = p.wpg, TG = 32 * WPG, RG = kLW / WPG;
    const int grp = warp / WPG, wg = warp - grp * WPG, tg = tid - grp * TG;
    // rank rk owns the rows [dlo[rk], dlo[rk+1]); its CTA lc the rows [dlo + lc RMr, ...),
    // RMr = ceil(rank rows / Gr): the owner of global row i is (rank of i, (i - dlo) / RMr)
    // (non-SYS kernels serve one rank -- every multi-rank launch, virtual or real, uses SYS --
    //  but keep the general form: the single-rank values come from the parameters)
    const int rk = p.rank >= 0 ? p.rank : cta / p.Gr;
    const int lc = p.rank >= 0 ? cta : cta - rk * p.Gr;
    const int G = p.P * p.Gr;  // CTAs in the exchange (all ranks)
    const bool lead = rk == 0 && lc == 0;
    const int64_t dlo_r = p.dlo[rk], nsh = p.dlo[rk + 1] - dlo_r;
    const int64_t RMr = p.RMr[rk];
    const int64_t r0 = dlo_r + ((lc * RMr < nsh) ? lc * RMr : nsh);
    const int64_t r1 = (r0 + RMr < dlo_r + nsh) ? r0 + RMr : dlo_r + nsh;
    const double *Ash = p.At_r[rk];  // row dlo_r of A~ (this rank's rows)
    const int R = static_cast<int>(r1 - r0);
    const int lr0 = R * grp / RG, lr1 = R * (grp + 1) / RG;  // CTA-local rows of this group
    const int ng = lr1 - lr0;
    const int rr = ng < p.rr ? ng : p.rr;
    const int rt = TM != 0 ? ((ng - rr) < p.rt ? (ng - rr) : p.rt) : 0;   // rows in TMEM
    const int rs = (ng - rr - rt) < p.rs ? (ng - rr - rt) : p.rs;
    const int b = p.key_bits;
    const int RM = p.rows_max;
    // ---- ST: the rows past the on-chip tiers stream through a per-group ring of shared-memory
    //      stages filled by TMA bulk copies (SR whole rows, contiguous in A~).  Chunk g (of SC per
    //      iteration, g counted over the whole loop) holds rows s0 + (g mod SC) SR ... and lives in
    //      stage g mod SS; the copies of the next iteration's first chunks are issued as soon as
    //      their stages are drained, so they load during the exchange. ----
    const int s0 = rr + rt + rs;
    const int SR = ST ? p.st_rows : 1, SS = ST ? p.st_stages : 1;
    const int SC = ST ? (ng - s0 + SR - 1) / SR : 0;
    const bool producer = ST && wg == 0 && lane == 0;

    const LoopSmem L = loop_smem(RM, WPG, CB, n, p.rs, ST ? p.st_stages : 0, ST ? p.st_rows : 0);
    volatile int64_t *ctl = reinterpret_cast<volatile int64_t *>(smem + L.ctl);  // [0..3] B2, [4..5] RES
    uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + L.mbar);
    const unsigned long long *slotbuf = reinterpret_cast<const unsigned long long *>(smem + L.slotbuf);  // winner's slot (TMA)
    double *cand = reinterpret_cast<double *>(smem + L.cand);  // [RG][4]: key bits, lambda, score, rr
    double *resp = reinterpret_cast<double *>(smem + L.resp);
    double *btl = reinterpret_cast<double *>(smem + L.btl);
    double *invl = reinterpret_cast<double *>(smem + L.invl);  // 1/nsq (0: masked row)
    double *dotp = reinterpret_cast<double *>(smem + L.dotp);  // [WPG][RM]
    double *xs = reinterpret_cast<double *>(smem + L.xs);      // x* by padded column
    double *rowbuf = reinterpret_cast<double *>(smem + L.rowbuf);
    double *arows = reinterpret_cast<double *>(smem + L.arows) + static_cast<size_t>(grp) * p.rs * CB * TG;
    const size_t st_stride = ST ? st_stage_bytes(n, SR) / 8 : 0;  // doubles per ring stage
    double *ring = reinterpret_cast<double *>(smem + L.ring) + static_cast<size_t>(grp) * SS * st_stride;
    uint64_t *rbar = reinterpret_cast<uint64_t *>(smem + L.rbar) + 2 * grp * SS;  // [SS][full, empty]
    auto st_issue = [&](uint32_t g) {  // producer: chunk g -> stage g mod SS
        const int c = static_cast<int>(g % static_cast<uint32_t>(SC));
        const int st = static_cast<int>(g % static_cast<uint32_t>(SS));
        const int nr = min(SR, ng - s0 - c * SR);
        const uint32_t by = static_cast<uint32_t>(nr) * static_cast<uint32_t>(n) * 8u;
        mbar_arrive_expect_tx(rbar + 2 * st, by);
        if (p.st_pin < 0)
            bulk_g2s(ring + st * st_stride, Ash + (r0 - dlo_r + lr0 + s0 + c * SR) * n, by, rbar + 2 * st);
        else if (c < p.st_pin || p.st_rest_first)
            bulk_g2s_l2(ring + st * st_stride, Ash + (r0 - dlo_r + lr0 + s0 + c * SR) * n, by, rbar + 2 * st,
                        c < p.st_pin);
        else
            bulk_g2s(ring + st * st_stride, Ash + (r0 - dlo_r + lr0 + s0 + c * SR) * n, by, rbar + 2 * st);
    };

    if (tid == 0) {
        uint32_t dyn;
        asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
        if (L.total > dyn) __trap();
        mbar_init(mbar, 1);
        if (CLU) {  // one local arrival (the expect_tx) per phase; the peers' st.async bring the bytes
            mbar_init(reinterpret_cast<uint64_t *>(smem + kXbarOff), 1);
            mbar_init(reinterpret_cast<uint64_t *>(smem + kXbarOff) + 1, 1);
        }
        if constexpr (ST) {  // per stage: full (the producer's expect_tx + the bytes), empty (the group's warps)
            uint64_t *rb = reinterpret_cast<uint64_t *>(smem + L.rbar);
            for (int i = 0; i < RG * p.st_stages; ++i) {
                mbar_init(rb + 2 * i, 1);
                mbar_init(rb + 2 * i + 1, static_cast<uint32_t>(WPG));
            }
        }
        fence_mbar_init();
    }
    if (CLU) cluster_sync_all();  // every peer's exchange barriers exist before the first arrival
    uint32_t tbase = 0;  // this thread's TMEM row area: lane 32 (warp & 3) + lane, 256 columns
    if constexpr (TM != 0) {
        uint32_t *taddr_s = reinterpret_cast<uint32_t *>(const_cast<int64_t *>(ctl) + 6);
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(taddr_s))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        tbase = *taddr_s + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + static_cast<uint32_t>(256 * (warp >> 2));
    }

    // ---- prologue: x (registers), x* (smem), b~, nsq (smem), rows into their tiers ----
    double x[CB];
#pragma unroll
    for (int q = 0; q < CB; ++q) {
        const int c = tg + TG * q;
        x[q] = c < n ? p.x_r[rk][c] : 0.0;
    }
    for (int c = tid; c < TG * CB; c += kLT) {
        xs[c] = (!RESMODE && c < n) ? p.x_star[c] : 0.0;
        if (c >= n) rowbuf[c] = 0.0;  // the TMA writes [0, n); x_q += lambda * 0 past n
    }
    for (int l = tid; l < R; l += kLT) {
        btl[l] = p.bt_r[rk][r0 - dlo_r + l];
        const double ns = p.nsq_r[rk][r0 - dlo_r + l];
        invl[l] = ns > 0.0 ? 1.0 / ns : 0.0;
    }
    double a[RRMAX][CB];
#pragma unroll
    for (int i = 0; i < RRMAX; ++i) {
        const double *src = Ash + (r0 - dlo_r + lr0 + i) * n;
#pragma unroll
        for (int q = 0; q < CB; ++q) {
            const int c = tg + TG * q;
            a[i][q] = (i < rr && c < n) ? src[c] : 0.0;
        }
    }
    if constexpr (TM != 0) {
        for (int j = 0; j < rt; ++j) {  // warp-uniform
            const double *src = Ash + (r0 - dlo_r + lr0 + rr + j) * n;
            uint32_t v[16];
#pragma unroll
            for (int q = 0; q < CB; ++q) {
                const int c = tg + TG * q;
                const double a0 = c < n ? src[c] : 0.0;
                v[2 * q] = static_cast<uint32_t>(__double2loint(a0));
                v[2 * q + 1] = static_cast<uint32_t>(__double2hiint(a0));
            }
            tmem_st16(tbase + 16u * j, v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    for (int i = 0; i < rs; ++i) {
        const double *src = Ash + (r0 - dlo_r + lr0 + rr + rt + i) * n;
#pragma unroll
        for (int q = 0; q < CB; ++q) {
            const int c = tg + TG * q;
            const double v = c < n ? src[c] : 0.0;
            if (CB == 1) arows[static_cast<size_t>(i) * TG + tg] = v;
            else arows[((static_cast<size_t>(i) * (CB / 2) + q / 2) * TG + tg) * 2 + (q & 1)] = v;
        }
    }
    __syncthreads();
    if constexpr (ST) {  // the first SS chunks (barrier inits are visible after the CTA barrier)
        if (producer && SC > 0)
            for (int g = 0; g < SS; ++g) st_issue(static_cast<uint32_t>(g));
    }

    // ||x*||^2 by the last row group (every group holds all of x; fixed order: thread q-order
    // fma, warp butterfly, warps in order).  The last group also owns the RES test and the
    // x trace, keeping them off warp 0's exchange path.
    const bool resgrp = grp == RG - 1;
    if (!RESMODE && resgrp) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < CB; ++q) {
            const double v = xs[tg + TG * q];
            s = __fma_rn(v, v, s);
        }
        s = lwarp_sum(s);
        if (lane == 0) resp[8 + wg] = s;
    }
    __syncthreads();
    double xs_nrm = 0.0;
    if (!RESMODE)
        for (int w = 0; w < WPG; ++w) xs_nrm = xs_nrm + resp[8 + w];
    const double bb = RESMODE ? *p.bb : 0.0;
    const bool even = (n & 1) == 0;
    const unsigned long long kmask = (1ull << b) - 1ull;

    // finalize lanes keep their rows' b~ and 1/nsq in registers (groups of <= 32 rows; with the
    // TMEM tier <= 64: rows lane and lane + 32)
    const bool fast_fin = ng <= (TM != 0 ? 64 : 32);
    // (the narrow-TMEM variants run at the register limit: there the finalize re-reads them from
    // shared memory, measured faster at C2; the others keep them in registers)
    constexpr bool kFinReg = TM != 2;
    // wide TMEM tier with groups of up to 64 rows: two finalize warps per group (CTA-uniform)
    const bool split2 = TM == 1 && WPG >= 2 && (RM + RG - 1) / RG > 32 && (RM + RG - 1) / RG <= 64;
    const double fin_b = (kFinReg && fast_fin && lane < ng) ? btl[lr0 + lane] : 0.0;
    const double fin_i = (kFinReg && fast_fin && lane < ng) ? invl[lr0 + lane] : 0.0;
    const double fin_b2 = (TM == 1 && fast_fin && lane + 32 < ng) ? btl[lr0 + 32 + lane] : 0.0;
    const double fin_i2 = (TM == 1 && fast_fin && lane + 32 < ng) ? invl[lr0 + 32 + lane] : 0.0;
    const bool all_reg = rr == ng;  // every row of the group in registers: own partial by shuffle
    const bool fuse_ts = p.fuse_ts != 0;  // (A/B: CSK_LOOP_FUSE_TS=0 takes the separate tier passes)

    int64_t k = 0, last = -1;
    int term = -1;
    // r_k of CTA-local row l (global row r0 + l) into the residual trace (off: one uniform branch)
    auto rtrace = [&](int l, double ri) {
        if (p.r_trace != nullptr && k < p.r_trace_cap) p.r_trace[k * p.d_glob + r0 + l] = ri;
    };
    double res = 0.0;
    uint32_t mphase = 0;
    double lam = 0.0;      // lambda of the pending update x += lam A~^(prow)
    int64_t prow = -1;     // row of the pending update (-1: none)
    const double *prow_ptr = nullptr;  // its A~ row (owner rank's memory: peer-mapped across GPUs)
    int *arrive = reinterpret_cast<int *>(const_cast<int64_t *>(ctl) + 7);  // group arrivals (smem)
    if (tid == 0) *arrive = 0;
    __syncthreads();
#if CSK_PHASE_PROF
    const bool prof = p.phase_cycles != nullptr && lead && lane == 0 && (warp == 0 || warp == kLW - 1);
    long long ph[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long tp = clock64();
#define LP(i)                           \
    if (prof) {                         \
        const long long tn = clock64(); \
        ph[i] += tn - tp;               \
        tp = tn;                        \
    }
#else
#define LP(i)
#endif
#if CSK_PHASE_PROF && CSK_PROBE_GEMV
#define LPG(i) LP(i)
#define LPT(i)
#else
#define LPG(i)
#define LPT(i) LP(i)
#endif
    for (;; ++k) {
        // ---- S8 of iteration k-1, fused at the top of iteration k: x_q += lambda a_{i_{k-1}}[c_q]
        //      (the row is in the fixed-offset row buffer, zero past n; odd n: from L2) ----
        if (prow >= 0) {
            if (even && !SYS) {
                const double *rb = reinterpret_cast<const double *>(smem + kRowbufOff) + tg;
#pragma unroll
                for (int q = 0; q < CB; ++q) x[q] = __fma_rn(lam, rb[TG * q], x[q]);
            } else if (SYS && p.P > 1) {
                // the row staged in this rank's memory by its CTA 0: wait for the iteration's flag,
                // then coherent (L2) loads of this thread's columns
                const unsigned char *reg = reinterpret_cast<const unsigned char *>(p.xch_r[rk]);
                const unsigned long long *flag =
                    reinterpret_cast<const unsigned long long *>(reg + kStageFlagOff) + ((k - 1) & 1);
                const uint32_t want = static_cast<uint32_t>(k);  // the row of iteration k - 1: tag k
                unsigned long long f;
                do {  // relaxed polls, then one acquire load orders the row loads after the flag
                    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(f) : "l"(flag) : "memory");
                } while (static_cast<uint32_t>(f) != want);
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(f) : "l"(flag) : "memory");
                const double *src = reinterpret_cast<const double *>(reg + kStageRowOff) + ((k - 1) & 1) * CSK_MAX_N;
#pragma unroll
                for (int q = 0; q < CB; ++q) {
                    const int c = tg + TG * q;
                    if (c < n) x[q] = __fma_rn(lam, __ldcg(src + c), x[q]);
                }
            } else {
                const double *src = prow_ptr;
#pragma unroll
                for (int q = 0; q < CB; ++q) {
                    const int c = tg + TG * q;
                    if (c < n) x[q] = __fma_rn(lam, ldg_stream1(src + c), x[q]);
                }
            }
        }
        LP(7)
        // ---- S5 partial (last group): ||x_k - x*||^2, combined by the group's finalize warp ----
        double e2 = 0.0;
        if (resgrp && lead && p.x_trace && k < p.trace_cap) {  // both stop modes record the iterates
#pragma unroll
            for (int q = 0; q < CB; ++q) {
                const int c = tg + TG * q;
                if (c < n) p.x_trace[k * n + c] = x[q];
            }
        }
        if (!RESMODE && resgrp) {
#pragma unroll
            for (int q = 0; q < CB; ++q) {
                const double e = x[q] - xs[tg + TG * q];
                e2 = __fma_rn(e, e, e2);
            }
        }
        // ---- S6 GEMV: register rows (transposed tree: row i ends in lanes [i LPR, (i+1) LPR)) ----
        double sreg;
        // the full TMEM tier and the shared-memory rows in one interleaved pass (C4's layout)
        const bool fused = TM == 1 && !ST && rt == kTmRowsDev && rs >= 1 && rs <= 12 && fuse_ts;
        bool smem_done = false;  // the fused pass took the shared-memory rows
        double racc[V];  // register rows' partials (their tree runs inside the fused pass)
        {
#pragma unroll
            for (int i = 0; i < V; ++i) racc[i] = 0.0;
#pragma unroll
            for (int q = 0; q < CB; ++q) {
#pragma unroll
                for (int i = 0; i < RRMAX; ++i) racc[i] = __fma_rn(a[i][q], x[q], racc[i]);
            }
            if (!(TM == 1 && fused)) {
                const double s = treduce<V>(racc, lane);
                sreg = s;
                const int i = lane / LPR;
                if ((lane % LPR) == 0 && i < rr && !(all_reg && wg == 0)) dotp[wg * RM + lr0 + i] = s;
            } else {
                sreg = 0.0;  // (TMEM rows present: the finalize reads dotp)
            }
        }
        LPG(11)
        // ---- S6 GEMV: TMEM rows, blocks of 8 (two rows per tcgen05.ld), transposed tree ----
        if constexpr (TM != 0) {
            // blocks of 8 / 4 / 2 rows (a block may run one row past rt, reading an unused row
            // of this thread's TMEM area that is never written back); a full wide tier (16 rows)
            // folds both blocks into one 16-row tree (one tree depth instead of two)
            int j0 = 0;
            if (fused) {
                // full TMEM tier + the shared-memory rows in one interleaved pass, one 32-row tree
                double acc32[32];
                tmem_smem_fused<12, V>(tbase, arows, tg, rs, TG, x, acc32, racc);
                {  // the register rows' tree finished inside the pass: row i in lanes [i LPR, (i+1) LPR)
                    const int i = lane / LPR;
                    if ((lane % LPR) == 0 && i < rr) dotp[wg * RM + lr0 + i] = racc[0];
                }
                const double s = treduce<32>(acc32, lane);
                if (lane < 16) dotp[wg * RM + lr0 + rr + lane] = s;
                else if (lane - 16 < rs) dotp[wg * RM + lr0 + rr + rt + lane - 16] = s;
                j0 = rt;
                smem_done = true;
            } else if (TM == 1 && rt == kTmRowsDev) {
                double acc16[16];
                tmem_block_wide<8, CB>(tbase, x, *reinterpret_cast<double(*)[8]>(&acc16[0]));
                tmem_block_wide<8, CB>(tbase + 16u * 8, x, *reinterpret_cast<double(*)[8]>(&acc16[8]));
                const double s = treduce<16>(acc16, lane);
                const int i = lane >> 1;
                if ((lane & 1) == 0) dotp[wg * RM + lr0 + rr + i] = s;
                j0 = rt;
            }
            for (; j0 < rt;) {
                if (rt - j0 > 4) {
                    double acc8[8];
                    if constexpr (TM == 1) tmem_block_wide<8, CB>(tbase + 16u * j0, x, acc8);
                    else tmem_block<8, CB>(tbase + 16u * j0, x, acc8);
                    const double s = treduce<8>(acc8, lane);
                    const int i = lane >> 2;
                    if ((lane & 3) == 0 && j0 + i < rt) dotp[wg * RM + lr0 + rr + j0 + i] = s;
                    j0 += 8;
                } else if (rt - j0 > 2) {
                    double acc4[4];
                    if constexpr (TM == 1) tmem_block_wide<4, CB>(tbase + 16u * j0, x, acc4);
                    else tmem_block<4, CB>(tbase + 16u * j0, x, acc4);
                    const double s = treduce<4>(acc4, lane);
                    const int i = lane >> 3;
                    if ((lane & 7) == 0 && j0 + i < rt) dotp[wg * RM + lr0 + rr + j0 + i] = s;
                    j0 += 4;
                } else {
                    double acc2[2];
                    if constexpr (TM == 1) tmem_block_wide<2, CB>(tbase + 16u * j0, x, acc2);
                    else tmem_block<2, CB>(tbase + 16u * j0, x, acc2);
                    const double s = treduce<2>(acc2, lane);
                    const int i = lane >> 4;
                    if ((lane & 15) == 0 && j0 + i < rt) dotp[wg * RM + lr0 + rr + j0 + i] = s;
                    j0 += 2;
                }
            }
        }
        LPG(12)
        // ---- S6 GEMV: shared-memory rows, blocks of 8, transposed tree ----
        {
            // blocks of 8 (a tail of <= 4 rows: a block of 4), columns outer so the block's rows
            // form independent fma chains; rows past rs re-read row rs-1 (never written back).
            // 9..12 rows with the TMEM tier: one 16-row tree over a block of 8 and a block of 4
            int i0 = smem_done ? rs : 0;
            if (!smem_done && TM == 1 && rs > 8 && rs <= 12) {
                double acc16[16];
                smem_block<8, CB>(arows, tg, 0, rs, TG, x, *reinterpret_cast<double(*)[8]>(&acc16[0]));
                smem_block<4, CB>(arows, tg, 8, rs, TG, x, *reinterpret_cast<double(*)[4]>(&acc16[8]));
#pragma unroll
                for (int j = 12; j < 16; ++j) acc16[j] = 0.0;
                const double s = treduce<16>(acc16, lane);
                const int i = lane >> 1;
                if ((lane & 1) == 0 && i < rs) dotp[wg * RM + lr0 + rr + rt + i] = s;
                i0 = rs;
            }
            for (; i0 < rs;) {
                if (rs - i0 > 4) {
                    double acc8[8];
                    smem_block<8, CB>(arows, tg, i0, rs, TG, x, acc8);
                    const double s = treduce<8>(acc8, lane);
                    const int i = lane >> 2;
                    if ((lane & 3) == 0 && i0 + i < rs) dotp[wg * RM + lr0 + rr + rt + i0 + i] = s;
                    i0 += 8;
                } else {
                    double acc4[4];
                    smem_block<4, CB>(arows, tg, i0, rs, TG, x, acc4);
                    const double s = treduce<4>(acc4, lane);
                    const int i = lane >> 3;
                    if ((lane & 7) == 0 && i0 + i < rs) dotp[wg * RM + lr0 + rr + rt + i0 + i] = s;
                    i0 += 4;
                }
            }
        }
        if constexpr (ST) {
            // ---- S6 GEMV: streamed rows from the TMA ring, SR rows per stage (a multiple of 4) in
            //      passes of 4, transposed tree (row j of a pass ends in lanes [8j, 8j + 8)) ----
            for (int c = 0; c < SC; ++c) {
                const uint32_t g = static_cast<uint32_t>(k) * static_cast<uint32_t>(SC) + static_cast<uint32_t>(c);
                const int st = static_cast<int>(g % static_cast<uint32_t>(SS));
                const uint32_t par = (g / static_cast<uint32_t>(SS)) & 1u;
                const int nr = min(SR, ng - s0 - c * SR);
                mbar_wait(rbar + 2 * st, par);
                const double *rp = ring + st * st_stride;
                auto pass = [&](int p0, double (&u)[4]) {  // 4 rows of the stage against x
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) u[jj] = 0.0;
#pragma unroll
                    for (int q = 0; q < CB; ++q) {
                        const int col = tg + TG * q;
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj) {
                            const double v = (p0 + jj < nr && col < n) ? rp[(p0 + jj) * n + col] : 0.0;
                            u[jj] = __fma_rn(v, x[q], u[jj]);
                        }
                    }
                };
                const int j = lane >> 3;
                int p0 = 0;
                for (; p0 + 4 < nr; p0 += 4) {  // all passes but the last
                    double u[4];
                    pass(p0, u);
                    const double sj = treduce<4>(u, lane);
                    if ((lane & 7) == 0) dotp[wg * RM + lr0 + s0 + c * SR + p0 + j] = sj;
                }
                double u[4];
                pass(p0, u);
                __syncwarp();
                if (lane == 0) mbar_arrive(rbar + 2 * st + 1);  // this warp is done with the stage
                const double sj = treduce<4>(u, lane);
                if ((lane & 7) == 0 && p0 + j < nr) dotp[wg * RM + lr0 + s0 + c * SR + p0 + j] = sj;
                if (producer) {  // refill the stage with chunk g + SS once every warp has read it
                    mbar_wait(rbar + 2 * st + 1, par);
                    st_issue(g + static_cast<uint32_t>(SS));
                }
            }
        } else {
            // ---- S6 GEMV: streamed rows (L2/HBM), two rows per pass ----
            for (int i = rr + rt + rs; i < ng; i += 2) {
                const bool two = i + 1 < ng;
                const double *s0 = Ash + (r0 - dlo_r + lr0 + i) * n;
                const double *s1 = two ? s0 + n : s0;
                double u0 = 0.0, u1 = 0.0;
    #pragma unroll
                for (int q = 0; q < CB; ++q) {
                    const int c = tg + TG * q;
                    const double v0 = c < n ? ldg_stream1(s0 + c) : 0.0;
                    const double v1 = c < n ? ldg_stream1(s1 + c) : 0.0;
                    u0 = __fma_rn(v0, x[q], u0);
                    u1 = __fma_rn(v1, x[q], u1);
                }
                u0 = lwarp_sum(u0);
                u1 = lwarp_sum(u1);
                if (lane == 0) {
                    dotp[wg * RM + lr0 + i] = u0;
                    if (two) dotp[wg * RM + lr0 + i + 1] = u1;
                }
            }
        }
        LPG(13)
        // ---- S7 (group): r_i = b~_i - dot, score, lambda, key; group argmax -> cand[grp] ----
        if (WPG > 1) group_bar(1 + grp, TG);
        else __syncwarp();
        LPG(14)
        if (wg == 0 || (split2 && wg == 1)) {
            unsigned long long bk = 0ull;
            double bl = 0.0, bs = -1.0, rr2 = 0.0;
            if (split2) {
                // groups of 33..64 rows with the wide TMEM tier: the group's first two warps take
                // rows lane and lane + 32 side by side (one candidate each); warp 0's own partial
                // comes by shuffle when every row of the group is a register row (all_reg)
                const double own = __shfl_sync(0xffffffffu, sreg, (lane * LPR) & 31);
                const int l = lr0 + 32 * wg + lane;
                if (32 * wg + lane < ng) {
                    double dot = (all_reg && wg == 0) ? own : dotp[l];
                    for (int w = 1; w < WPG; ++w) dot = dot + dotp[w * RM + l];
                    const double fb = wg == 0 ? fin_b : fin_b2, fi = wg == 0 ? fin_i : fin_i2;
                    const double ri = fb - dot;
                    rtrace(l, ri);
                    const double sc = fi > 0.0 ? (ri * ri) * fi : -1.0;
                    if (RESMODE) rr2 = __fma_rn(ri, ri, rr2);
                    bk = row_key(sc, r0 + l, b);
                    bl = ri * fi;
                    bs = sc;
                }
            } else if (fast_fin) {
                // one row per lane; the warp's own partial of row `lane` comes by shuffle when all
                // rows are register rows, the other warps' partials from shared memory
                const double own = __shfl_sync(0xffffffffu, sreg, (lane * LPR) & 31);
                if (lane < ng) {
                    const int l = lr0 + lane;
                    double dot = all_reg ? own : dotp[l];
                    for (int w = 1; w < WPG; ++w) dot = dot + dotp[w * RM + l];
                    const double fb = kFinReg ? fin_b : btl[l], fi = kFinReg ? fin_i : invl[l];
                    const double ri = fb - dot;
                    rtrace(l, ri);
                    const double sc = fi > 0.0 ? (ri * ri) * fi : -1.0;
                    if (RESMODE) rr2 = __fma_rn(ri, ri, rr2);
                    bk = row_key(sc, r0 + l, b);
                    bl = ri * fi;
                    bs = sc;
                }
                if (TM != 0 && lane + 32 < ng) {  // second row of the lane (groups of 33..64 rows)
                    const int l = lr0 + 32 + lane;
                    double dot = dotp[l];
                    for (int w = 1; w < WPG; ++w) dot = dot + dotp[w * RM + l];
                    const double fb2 = TM == 1 ? fin_b2 : btl[l], fi2 = TM == 1 ? fin_i2 : invl[l];
                    const double ri = fb2 - dot;
                    rtrace(l, ri);
                    const double sc = fi2 > 0.0 ? (ri * ri) * fi2 : -1.0;
                    if (RESMODE) rr2 = __fma_rn(ri, ri, rr2);
                    const unsigned long long kk = row_key(sc, r0 + l, b);
                    if (kk > bk) { bk = kk; bl = ri * fi2; bs = sc; }
                }
            } else for (int l0 = 0; l0 < ng; l0 += 32) {
                const int l = lr0 + l0 + lane;
                if (l0 + lane < ng) {
                    double dot = dotp[l];
                    for (int w = 1; w < WPG; ++w) dot = dot + dotp[w * RM + l];
                    const double ri = btl[l] - dot;
                    rtrace(l, ri);
                    const double iv = invl[l];
                    // score r^2/nsq and lambda r/nsq through the precomputed 1/nsq (R-3)
                    const double sc = iv > 0.0 ? (ri * ri) * iv : -1.0;
                    if (RESMODE) rr2 = __fma_rn(ri, ri, rr2);
                    const unsigned long long kk = row_key(sc, r0 + l, b);
                    if (kk > bk) { bk = kk; bl = ri * iv; bs = sc; }
                }
            }
            if (RESMODE) rr2 = lwarp_sum(rr2);
            unsigned long long km;
            const int wl = warp_max_key_lane(bk, km);
            const int ci = split2 ? 2 * grp + wg : grp;  // candidate slot
            if (lane == wl) {
                cand[ci * 4 + 0] = __longlong_as_double(static_cast<long long>(km));
                cand[ci * 4 + 1] = bl;
                cand[ci * 4 + 2] = bs;
            }
            if (RESMODE && lane == 0) cand[ci * 4 + 3] = rr2;
            LP(0)
            // ---- arrival: the LAST group to finish combines the CTA candidate and runs the
            //      exchange (no CTA barrier before the publish) ----
        }
        __syncthreads();  // B1
        // ---- S5 (last group, beside warp 0's exchange): RES_k = ||x_k - x*||^2/||x*||^2;
        //      every CTA computes the same value from its own copy of x, so all stop at the same k
        // (RG = 1: warp 0 belongs to the only group and joins before its exchange)
        if (!RESMODE && resgrp && (RG == 1 || warp != 0)) {
            e2 = lwarp_sum(e2);
            if (WPG > 1) {
                if (lane == 0) resp[wg] = e2;
                group_bar(1 + grp, TG);
                e2 = resp[0];
                for (int w = 1; w < WPG; ++w) e2 = e2 + resp[w];
            }
            if (wg == 0 && lane == 0) {
                const double resk = xs_nrm > 0.0 ? e2 / xs_nrm : e2;
                ctl[4] = resk <= p.tol ? CSK_CONVERGED : -1;
                ctl[5] = __double_as_longlong(resk);
                if (lead && p.res_trace && k < p.trace_cap) p.res_trace[k] = resk;
            }
        }
        if (warp == 0) {
            {
                LP(1)
                int stop = (!RESMODE && k == p.max_iters) ? CSK_MAX_ITERS : -1;
                int64_t wrow = -1;
                if (stop < 0) {
                    // CTA candidate: max key over the RG group candidates
                    const int ncand = split2 ? 2 * RG : RG;
                    const unsigned long long ck =
                        lane < ncand ? static_cast<unsigned long long>(__double_as_longlong(cand[lane * 4])) : 0ull;
                    unsigned long long kc;
                    const int cl = warp_max_key_lane(ck, kc);
                    const double cl_l = cand[cl * 4 + 1], cl_s = cand[cl * 4 + 2];
                    double crr = 0.0;
                    if (RESMODE)
                        for (int g = 0; g < ncand; ++g) crr = crr + cand[g * 4 + 3];
                    const uint32_t tag = static_cast<uint32_t>(k + 1);
                    if constexpr (CLU) {
                        // ---- all-to-all over DSMEM: this CTA arms its barrier of this parity for
                        //      kCS x 32 bytes, then lane j st.async's the CTA candidate into rank j's
                        //      inbox, completing the bytes on rank j's barrier ----
                        const int par = static_cast<int>(k & 1);
                        double *inbox = reinterpret_cast<double *>(smem + kInboxOff) + par * kCS * 4;
                        uint64_t *xbar = reinterpret_cast<uint64_t *>(smem + kXbarOff) + par;
                        if (lane == 0) mbar_arrive_expect_tx(xbar, kCS * 32u);
                        if (lane < kCS) {
                            const uint32_t dst = mapa_shared(smem_u32(inbox + cta * 4), static_cast<uint32_t>(lane));
                            const uint32_t rbar = mapa_shared(smem_u32(xbar), static_cast<uint32_t>(lane));
                            st_async_v2_f64(dst, __longlong_as_double(static_cast<long long>(kc)), cl_l, rbar);
                            st_async_v2_f64(dst + 16, cl_s, crr, rbar);
                        }
                        LP(2)
                        while (!mbar_try_wait_cluster(xbar, static_cast<uint32_t>((k >> 1) & 1))) {
                        }
                        LP(3)
                        const unsigned long long kj =
                            lane < kCS ? static_cast<unsigned long long>(__double_as_longlong(inbox[lane * 4])) : 0ull;
                        unsigned long long mx;
                        const int wl = warp_max_key_lane(kj, mx);
                        const double wlam = inbox[wl * 4 + 1], wsc = inbox[wl * 4 + 2];
                        if (RESMODE) {
                            double t = 0.0;
                            for (int j = 0; j < kCS; ++j) t = t + inbox[j * 4 + 3];  // fixed order
                            res = bb > 0.0 ? t / bb : t;
                            if (lead && lane == 0 && p.res_trace && k < p.trace_cap) p.res_trace[k] = res;
                            if (res <= p.tol) stop = CSK_CONVERGED;
                            else if (k == p.max_iters) stop = CSK_MAX_ITERS;
                        }
                        if (mx != 0ull) {
                            wrow = static_cast<int64_t>(kmask - (mx & kmask));
                            if (lane == 0) {
                                // the winner's (lambda, score) go to the slot buffer, LL-tagged like
                                // the global variant's; the row comes by TMA (odd n: plain loads)
                                unsigned long long *sb = const_cast<unsigned long long *>(slotbuf);
                                ll_pack(wlam, tag, sb[0], sb[1]);
                                ll_pack(wsc, tag, sb[2], sb[3]);
                                const uint32_t rbytes = even ? static_cast<uint32_t>(n) * 8u : 0u;
                                mbar_arrive_expect_tx(mbar, rbytes);
                                if (even) bulk_g2s(rowbuf, Ash + (wrow - dlo_r) * n, rbytes, mbar);
                                sb[4] = reinterpret_cast<unsigned long long>(Ash + (wrow - dlo_r) * n);
                            }
                        }
                        if (stop < 0 && mx == 0ull) stop = -2;  // every row masked: zero sketch
                        if (stop >= 0 && wrow >= 0 && lane == 0) mbar_wait(mbar, mphase);  // drain the copy
                    } else {
                    unsigned long long *pair = p.xch + static_cast<int>(k % 3) * kXchWords;
                    const size_t par_off = static_cast<size_t>(k & 1) * p.Gr * kSlotWords;
                    if (lane == 0) {
                        // (SYS: the slots are read by the other GPUs -- system-scope stores)
                        unsigned long long *my = p.slots_r[rk] + par_off + static_cast<size_t>(lc) * kSlotWords;
                        unsigned long long h0, l0, h1, l1;
                        ll_pack(cl_l, tag, h0, l0);
                        ll_pack(cl_s, tag, h1, l1);
                        if constexpr (!SYS) {
                            if (lead) {
                                st_relaxed_v2_u64(p.xch + ((k + 1) % 3) * kXchWords, 0ull, 0ull);
                                if (RESMODE) st_relaxed_v2_u64(p.xch + ((k + 1) % 3) * kXchWords + 2, 0ull, 0ull);
                            }
                            red_max_u64(pair + 1, kc);
                            // residual stop: ||r_k||^2 accumulates beside the count (one sum,
                            // read by every CTA in the same load as the count)
                            if (RESMODE) red_add_f64(reinterpret_cast<double *>(pair + 2), crr);
                            red_add_release_u64(pair, 1ull);  // orders the max, sum (and reset) before the count
                            // the slot needs no ordering: readers validate its LL tags
                            st_relaxed_v2_u64(my, h0, l0);
                            st_relaxed_v2_u64(my + 2, h1, l1);
                        } else {
                            // across GPUs, in two levels: this rank's CTAs meet on a pair in this
                            // rank's memory (GPU scope: a system-scope release costs microseconds);
                            // the rank's leader then pushes one LL-tagged key to every rank (below)
                            unsigned long long *lp = p.xch_r[rk] + static_cast<int>(k % 3) * kXchWords;
                            if (lc == 0) {
                                st_relaxed_v2_u64(p.xch_r[rk] + ((k + 1) % 3) * kXchWords, 0ull, 0ull);
                                if (RESMODE) st_relaxed_v2_u64(p.xch_r[rk] + ((k + 1) % 3) * kXchWords + 2, 0ull, 0ull);
                            }
                            red_max_u64(lp + 1, kc);
                            if (RESMODE) red_add_f64(reinterpret_cast<double *>(lp + 2), crr);  // the rank's ||r||^2
                            red_add_release_u64(lp, 1ull);
                            st_relaxed_v2_u64_sys(my, h0, l0);
                            st_relaxed_v2_u64_sys(my + 2, h1, l1);
                        }
                    }
                    LP(2)
#if CSK_PHASE_PROF
                    if (p.skew && lane == 0 && k >= 8 && k < 72) {
                        unsigned long long gt;
                        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
                        p.skew[(k - 8) * 2 * G + cta] = static_cast<long long>(gt);
                    }
#endif
                    unsigned long long c = 0ull, mx = 0ull, rsum = 0ull;
                    unsigned long long t_spin = 0ull;
                    uint32_t spins = 0u;
                    bool timed_out = false;
                    // watchdog: a rank that never arrives (a peer that failed to launch) turns into
                    // an error instead of a hang; the clock is read only every 4096 polls
                    auto watchdog = [&]() {
                        if (((++spins) & 4095u) == 0u) {
                            const unsigned long long now = globaltimer_ns();
                            if (t_spin == 0ull) t_spin = now;
                            else if (now - t_spin > p.timeout_ns) timed_out = true;
                        }
                        return timed_out;
                    };
                    if constexpr (SYS) {
                        // the rank's leader (its CTA 0): once every local CTA has counted, push the
                        // rank's max key into every rank's key slot (LL: key halves + tag, no fence)
                        const uint32_t tag = static_cast<uint32_t>(k + 1);
                        if (lc == 0 && lane == 0) {
                            const unsigned long long *lp = p.xch_r[rk] + static_cast<int>(k % 3) * kXchWords;
                            unsigned long long lc2 = 0ull, lmx = 0ull, lsum = 0ull;
                            do {
                                if (RESMODE) ld_relaxed_v4(lp, lc2, lmx, lsum);
                                else ld_relaxed_v2(lp, lc2, lmx);
                            } while (lc2 < static_cast<unsigned long long>(p.Gr) && !watchdog());
#if CSK_STRICT_ACQUIRE
                            if (lc2 >= static_cast<unsigned long long>(p.Gr)) {  // see the single-GPU poll
                                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                                if (RESMODE) ld_relaxed_v4(lp, lc2, lmx, lsum);
                                else ld_relaxed_v2(lp, lc2, lmx);
                            }
#endif
                            unsigned long long h, l, hs = 0ull, ls = 0ull;
                            ll_pack(__longlong_as_double(static_cast<long long>(lmx)), tag, h, l);
                            if (RESMODE) ll_pack(__longlong_as_double(static_cast<long long>(lsum)), tag, hs, ls);
                            for (int q = 0; q < p.P; ++q) {
                                unsigned long long *ks = p.xch_r[q] + 3 * kXchWords + ((k & 1) * kMaxRanks + rk) * 2;
                                st_relaxed_v2_u64_sys(ks, h, l);
                                if (RESMODE) st_relaxed_v2_u64_sys(ks + 2 * kMaxRanks * 2, hs, ls);
                            }
                        }
                        // every CTA: the P rank keys from its own rank's key slots
                        for (int q = 0; q < p.P && !timed_out; ++q) {
                            const unsigned long long *ks = p.xch_r[rk] + 3 * kXchWords + ((k & 1) * kMaxRanks + q) * 2;
                            unsigned long long a0, a1;
                            do {
                                ld_relaxed_v2_sys(ks, a0, a1);
                            } while (!ll_ok(a0, a1, tag) && !watchdog());
                            const unsigned long long kq =
                                static_cast<unsigned long long>(__double_as_longlong(ll_val(a0, a1)));
                            if (kq > mx) mx = kq;
                            if (RESMODE && !timed_out) {  // the ranks' sums in rank order: every rank adds the same way
                                do {
                                    ld_relaxed_v2_sys(ks + 2 * kMaxRanks * 2, a0, a1);
                                } while (!ll_ok(a0, a1, tag) && !watchdog());
                                rsum = static_cast<unsigned long long>(__double_as_longlong(
                                    __longlong_as_double(static_cast<long long>(rsum)) + ll_val(a0, a1)));
                            }
                        }
                        timed_out = __any_sync(0xffffffffu, timed_out);
                        c = static_cast<unsigned long long>(G);
                    } else {
                        if (TM == 0 && !CLU && p.npoll > 1) {  // (not built into the TMEM-tier or cluster kernels)
                            // A/B knob CSK_LOOP_NPOLL: staggered polls, NP loads of the pair in
                            // flight, issued ~pdelay cycles apart and each re-issued as soon as it
                            // returns short of G (the count reaching G would be seen ~RT/NP after
                            // it lands).  Measured SLOWER (C3 2.87 -> 3.05 / 3.52 us at NP = 2 / 4):
                            // the extra reads of the one hot line delay the atomics on it.  The
                            // default (one poll at a time) is the loop below.
                            constexpr int NP = 4;
                            unsigned long long pc[NP], pm[NP], ps[NP];
                            const int np = p.npoll < NP ? p.npoll : NP;
                            auto issue = [&](int i) {
                                if (RESMODE) ld_relaxed_v4(pair, pc[i], pm[i], ps[i]);
                                else ld_relaxed_v2(pair, pc[i], pm[i]);
                            };
#pragma unroll
                            for (int i = 0; i < NP; ++i) {
                                if (i < np) {
                                    if (i > 0) {
                                        const long long t0 = clock64();
                                        while (clock64() - t0 < p.pdelay) {}
                                    }
                                    issue(i);
                                }
                            }
                            bool got = false;
                            while (!got) {
#pragma unroll
                                for (int i = 0; i < NP; ++i) {
                                    if (!got && i < np) {
                                        if (pc[i] >= static_cast<unsigned long long>(G)) {
                                            c = pc[i];
                                            mx = pm[i];
                                            rsum = ps[i];
                                            got = true;
                                        } else {
                                            issue(i);
                                        }
                                    }
                                }
                                if (!got && watchdog()) {
                                    c = 0ull;
                                    break;
                                }
                            }
                        } else {
                            do {  // relaxed polls (an acquire load would invalidate L1 on every poll)
                                if (RESMODE) ld_relaxed_v4(pair, c, mx, rsum);
                                else ld_relaxed_v2(pair, c, mx);
                                if (c < static_cast<unsigned long long>(G) && watchdog()) break;
                            } while (c < static_cast<unsigned long long>(G));
                        }
#if CSK_STRICT_ACQUIRE
                        // the PTX-model form of the read (memory-model note):
                        // the count seen by a relaxed poll plus an acquire fence synchronizes with
                        // every CTA's red.release of the count, so a re-read of the pair after the
                        // fence sees every CTA's red.max (and red.add of the sum) -- without relying
                        // on the 16/32-byte poll being one L2-sector snapshot.  One fence and one
                        // more L2 round trip per iteration; off by default (measured in DESIGN.md)
                        if (c >= static_cast<unsigned long long>(G)) {
                            asm volatile("fence.acq_rel.gpu;" ::: "memory");
                            if (RESMODE) ld_relaxed_v4(pair, c, mx, rsum);
                            else ld_relaxed_v2(pair, c, mx);
                        }
#endif
                    }
                    if (timed_out) {
                        stop = -3;
                        mx = 0ull;
                    }
                    // no acquire fence: A~, b~ are immutable and the slot is LL-validated (a proxy
                    // fence here would order only this thread's own accesses, not the owner's slot
                    // store, so none is issued: a stale TMA copy of the slot fails its tags)
                    LP(3)
#if CSK_PHASE_PROF
                    if (p.skew && lane == 0 && k >= 8 && k < 72) {
                        unsigned long long gt;
                        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
                        p.skew[(k - 8) * 2 * G + G + cta] = static_cast<long long>(gt);
                    }
#endif
                    LP(8)
                    if (mx != 0ull) {
                        wrow = static_cast<int64_t>(kmask - (mx & kmask));
                        CSK_DCHECK(wrow >= 0 && wrow < p.d_glob);
                        if (lane == 0) {
                            // owner: rank by the row ranges, then its CTA
                            const unsigned long long *oslot;
                            const double *orow;
                            if (p.rm_magic != 0ull) {  // one rank: CTA = row / RM by a multiply-shift
                                const uint32_t olc = static_cast<uint32_t>((static_cast<unsigned long long>(wrow) * p.rm_magic) >> 40);
                                CSK_DCHECK(olc < static_cast<uint32_t>(G));
                                oslot = p.slots + par_off + static_cast<size_t>(olc) * kSlotWords;
                                orow = p.At + wrow * n;
                            } else {
                                int orank = 0;
                                if (p.P > 1)
                                    while (orank + 1 < p.P && p.dlo[orank + 1] <= wrow) ++orank;
                                const uint32_t olrow = static_cast<uint32_t>(wrow - p.dlo[orank]);
                                const int olc = static_cast<int>(olrow / static_cast<uint32_t>(p.RMr[orank]));
                                oslot = p.slots_r[orank] + par_off + static_cast<size_t>(olc) * kSlotWords;
                                orow = p.At_r[orank] + (wrow - p.dlo[orank]) * n;
                            }
                            LPT(11)
                            unsigned long long *sb = const_cast<unsigned long long *>(slotbuf);
                            sb[4] = reinterpret_cast<unsigned long long>(orow);
                            sb[7] = reinterpret_cast<unsigned long long>(oslot);
                            if constexpr (!SYS) {
                                // winner's (lambda, score) slot and A~^(ik) -> shared memory, one
                                // mbarrier (odd n: the row is read with plain loads in the update)
                                const uint32_t rbytes = even ? static_cast<uint32_t>(n) * 8u : 0u;
                                mbar_arrive_expect_tx(mbar, rbytes + 32u);
                                LPT(12)
                                bulk_g2s(sb, oslot, 32u, mbar);
                                LPT(13)
                                if (even) bulk_g2s(rowbuf, orow, rbytes, mbar);
                                LPT(14)
                            } else {
                                // across GPUs: the slot by system-scope loads (LL-validated), the
                                // row by plain loads from the peer's memory in the update
                                const double wl = ll_load(oslot, tag, true), ws = ll_load(oslot + 2, tag, true);
                                ll_pack(wl, tag, sb[0], sb[1]);
                                ll_pack(ws, tag, sb[2], sb[3]);
                                mbar_arrive_expect_tx(mbar, 0u);
                            }
                        }
                    }
                    LP(9)
                    if (RESMODE && stop == -1) {  // (not after a watchdog timeout: stop = -3 stands)
                        // ||r_k||^2: each rank's CTA partials summed beside its count (arrival
                        // order); across ranks the ranks' sums in rank order.  The 32-byte poll
                        // reads {count, max, sum} from one L2 sector in one access (a hardware
                        // property relied on here, not a PTX guarantee: the count reaching G comes
                        // with every CTA's red.add of the sum); tests/test_gpu_parity.py
                        // test_residual_sum_complete checks RES_k against the traced r_k every
                        // iteration, where a missing CTA partial would show up as a ~1/G deficit
                        const double t = __longlong_as_double(static_cast<long long>(rsum));
                        res = bb > 0.0 ? t / bb : t;
                        if (lead && lane == 0 && p.res_trace && k < p.trace_cap) p.res_trace[k] = res;
                        if (res <= p.tol) stop = CSK_CONVERGED;
                        else if (k == p.max_iters) stop = CSK_MAX_ITERS;
                    }
                    if (stop == -1 && mx == 0ull) stop = -2;  // every row masked: zero sketch
                    if (stop >= 0 && wrow >= 0 && lane == 0) mbar_wait(mbar, mphase);  // drain the copies
                    }  // global exchange
                }
                LP(10)
                if (lane == 0) {
                    ctl[0] = stop;  // -1: copies in flight on mbar
                    ctl[1] = wrow;
                    ctl[3] = __double_as_longlong(res);
                    *arrive = 0;
                }
            }
        }
        LP(4)
        __syncthreads();  // B2
        LP(5)
        // every control word at once (independent loads, in flight during the row wait)
        int stop = static_cast<int>(ctl[0]);
        const int64_t conv = RESMODE ? 0 : ctl[4];
        const int64_t res_bits = RESMODE ? ctl[3] : ctl[5];
        const int64_t wrow_b = ctl[1];
        const double *wrow_ptr = reinterpret_cast<const double *>(slotbuf[4]);
        prow = -1;
        if (!RESMODE && conv == CSK_CONVERGED) {  // RES_k <= tol: no update
            if (stop == -1) mbar_wait(mbar, mphase);  // drain the copies of the exchange
            stop = CSK_CONVERGED;
        }
        if (stop == -1) {  // the winner's slot (and row) arrive on the mbarrier
            mbar_wait(mbar, mphase);
            mphase ^= 1u;
            const uint32_t tag = static_cast<uint32_t>(k + 1);
            double sc;
            if (ll_ok(slotbuf[0], slotbuf[1], tag) && ll_ok(slotbuf[2], slotbuf[3], tag)) {
                lam = ll_val(slotbuf[0], slotbuf[1]);
                sc = ll_val(slotbuf[2], slotbuf[3]);
            } else if (!CLU) {  // the copy raced the owner's slot store: re-read until the tags match
#if CSK_PHASE_PROF
                if (prof) ph[15] += 1000;  // (per mille of the iterations, in the probe's per-iteration print)
#endif
                const unsigned long long *gs = reinterpret_cast<const unsigned long long *>(slotbuf[7]);
                lam = ll_load(gs, tag, SYS);
                sc = ll_load(gs + 2, tag, SYS);
            }
            if (sc == 0.0) stop = CSK_STAGNATED;  // every unmasked residual is 0
        }
        LP(6)
        res = __longlong_as_double(res_bits);
        if (stop != -1) {
            term = stop;
            break;
        }
        const int64_t wrow = wrow_b;
        if (lead && tid == 0 && p.idx_trace && k < p.trace_cap) p.idx_trace[k] = wrow;
        last = wrow;
        prow = wrow;
        prow_ptr = wrow_ptr;
        if constexpr (SYS) {
            if (p.P > 1 && lc == 0) {
                // this rank's CTA 0 stages the winner's row (read over NVLink once for the GPU)
                // for the update at the top of iteration k + 1, then raises the flag (tag k + 1)
                unsigned char *reg = reinterpret_cast<unsigned char *>(p.xch_r[rk]);
                double *dst = reinterpret_cast<double *>(reg + kStageRowOff) + (k & 1) * CSK_MAX_N;
                for (int c = tid; c < n; c += kLT) dst[c] = ldg_stream1(wrow_ptr + c);
                __syncthreads();
                if (tid == 0) {
                    unsigned long long *flag = reinterpret_cast<unsigned long long *>(reg + kStageFlagOff) + (k & 1);
                    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(flag),
                                 "l"(static_cast<unsigned long long>(k + 1))
                                 : "memory");
                }
            }
        }
    }
#undef LP
#undef LPG
#undef LPT
    if constexpr (ST) {  // drain the copies already issued for the iteration that never ran
        if (producer && SC > 0) {
            const uint32_t g0 = static_cast<uint32_t>(k + 1) * static_cast<uint32_t>(SC);
            for (int i = 0; i < SS; ++i) {
                const uint32_t g = g0 + static_cast<uint32_t>(i);
                mbar_wait(rbar + 2 * (g % static_cast<uint32_t>(SS)), (g / static_cast<uint32_t>(SS)) & 1u);
            }
        }
    }
#if CSK_PHASE_PROF
    if (prof)
        for (int i = 0; i < 16; ++i) p.phase_cycles[(warp == 0 ? 0 : 1) * 16 + i] = ph[i];
#endif
    // ---- epilogue: CTA 0's last group writes x (and the trace of the final iterate) ----
    if (lc == 0 && resgrp) {  // every rank (virtual: every copy) writes its x
        const bool tr = p.x_trace && k < p.trace_cap;
#pragma unroll
        for (int q = 0; q < CB; ++q) {
            const int c = tg + TG * q;
            if (c < n) {
                p.x_r[rk][c] = x[q];
                if (tr && lead) p.x_trace[k * n + c] = x[q];
            }
        }
        if (tid == (RG - 1) * TG && (p.rank >= 0 || rk == 0)) {
            p.report[0] = k;
            p.report[1] = __double_as_longlong(res);
            p.report[2] = term;
            p.report[3] = last;
        }
    }
    if constexpr (TM != 0) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (warp == 0)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(
                             *reinterpret_cast<uint32_t *>(const_cast<int64_t *>(ctl) + 6))
                         : "memory");
    }
    if (CLU) cluster_sync_all();  // no CTA leaves while a peer could still address its shared memory
}

using LoopFn = void (*)(const LoopParams);

// rows per thread held in registers for a given column count per thread (~160 registers)
constexpr int rr_max_for(int cb) { return cb >= 16 ? 5 : cb >= 8 ? 10 : cb >= 4 ? 20 : 32; }

// Instantiated (CB, RRMAX) pairs: register-row capacities sized to the row counts per group
// that the configs produce (fewer unused register rows = fewer wasted FMAs and a shorter
// transposed tree).  Residual mode only gets the full-capacity variant.
struct LoopVariant {
    int cb, rrmax;
    LoopFn fn;
    bool tm = false;
    bool clu = false;
};
// Real multi-GPU launches (SYS: peer memory, the two-level exchange) get their own, smaller set
// of instantiations; the single-GPU kernels carry none of that code.  {cb, rrmax, fn, tm kind
// (0 none, 1 wide, 2 narrow), stream ring, residual mode}
struct SysVariant {
    int cb, rrmax, tmk;
    bool st, res;
    LoopFn fn;
};
const SysVariant kVariantsSys[] = {
    {1, 32, 0, false, false, k_loop<1, 32, false, 0, false, false, true>},
    {2, 32, 0, false, false, k_loop<2, 32, false, 0, false, false, true>},
    {4, 20, 0, false, false, k_loop<4, 20, false, 0, false, false, true>},
    {8, 10, 0, false, false, k_loop<8, 10, false, 0, false, false, true>},
    {16, 5, 0, false, false, k_loop<16, 5, false, 0, false, false, true>},
    {1, 32, 0, false, true, k_loop<1, 32, true, 0, false, false, true>},
    {2, 32, 0, false, true, k_loop<2, 32, true, 0, false, false, true>},
    {4, 20, 0, false, true, k_loop<4, 20, true, 0, false, false, true>},
    {8, 10, 0, false, true, k_loop<8, 10, true, 0, false, false, true>},
    {16, 5, 0, false, true, k_loop<16, 5, true, 0, false, false, true>},
    {8, 6, 1, false, false, k_loop<8, 6, false, 1, false, false, true>},
    {8, 6, 1, false, true, k_loop<8, 6, true, 1, false, false, true>},
    {8, 8, 2, false, false, k_loop<8, 8, false, 2, false, false, true>},
    {8, 8, 2, false, true, k_loop<8, 8, true, 2, false, false, true>},
    {1, 8, 0, true, false, k_loop<1, 8, false, 0, false, true, true>},
    {2, 8, 0, true, false, k_loop<2, 8, false, 0, false, true, true>},
    {4, 8, 0, true, false, k_loop<4, 8, false, 0, false, true, true>},
    {8, 8, 0, true, false, k_loop<8, 8, false, 0, false, true, true>},
    {8, 6, 1, true, false, k_loop<8, 6, false, 1, false, true, true>},
    {1, 8, 0, true, true, k_loop<1, 8, true, 0, false, true, true>},
    {2, 8, 0, true, true, k_loop<2, 8, true, 0, false, true, true>},
    {4, 8, 0, true, true, k_loop<4, 8, true, 0, false, true, true>},
    {8, 8, 0, true, true, k_loop<8, 8, true, 0, false, true, true>},
    {8, 6, 1, true, true, k_loop<8, 6, true, 1, false, true, true>},
};
const LoopVariant kVariants[] = {
    {1, 2, k_loop<1, 2, false, 0, false>},   {1, 8, k_loop<1, 8, false, 0, false>},   {1, 32, k_loop<1, 32, false, 0, false>},
    {2, 2, k_loop<2, 2, false, 0, false>},   {2, 8, k_loop<2, 8, false, 0, false>},   {2, 32, k_loop<2, 32, false, 0, false>},
    {4, 2, k_loop<4, 2, false, 0, false>},   {4, 4, k_loop<4, 4, false, 0, false>},   {4, 8, k_loop<4, 8, false, 0, false>},
    {4, 20, k_loop<4, 20, false, 0, false>}, {8, 2, k_loop<8, 2, false, 0, false>},   {8, 4, k_loop<8, 4, false, 0, false>},
    {8, 8, k_loop<8, 8, false, 0, false>},   {8, 9, k_loop<8, 9, false, 0, false>}, {8, 10, k_loop<8, 10, false, 0, false>}, {16, 2, k_loop<16, 2, false, 0, false>},
    {16, 4, k_loop<16, 4, false, 0, false>}, {16, 5, k_loop<16, 5, false, 0, false>},
};
// TMEM tier variants (8 columns per thread, 8 register rows + 16 TMEM rows per thread)
constexpr int kTmRows = 16;
constexpr int kTmRegRowsWide = 6, kTmRegRowsNarrow = 8;
const LoopVariant kVariantTm = {8, kTmRegRowsWide, k_loop<8, kTmRegRowsWide, false, 1, false>, true};
const LoopVariant kVariantTmRes = {8, kTmRegRowsWide, k_loop<8, kTmRegRowsWide, true, 1, false>, true};
const LoopVariant kVariantTmN = {8, kTmRegRowsNarrow, k_loop<8, kTmRegRowsNarrow, false, 2, false>, true};
const LoopVariant kVariantTmNRes = {8, kTmRegRowsNarrow, k_loop<8, kTmRegRowsNarrow, true, 2, false>, true};
// single-cluster variants (the whole problem on kCS SMs, DSMEM exchange): C1/C2-sized systems
const LoopVariant kVariantsClu[] = {
    {1, 8, k_loop<1, 8, false, 0, true>, false, true},   {2, 8, k_loop<2, 8, false, 0, true>, false, true},
    {4, 8, k_loop<4, 8, false, 0, true>, false, true},   {8, 10, k_loop<8, 10, false, 0, true>, false, true},
    {16, 5, k_loop<16, 5, false, 0, true>, false, true}, {8, kTmRegRowsWide, k_loop<8, kTmRegRowsWide, false, 1, true>, true, true},
    {8, kTmRegRowsNarrow, k_loop<8, kTmRegRowsNarrow, false, 2, true>, true, true},
};
const LoopVariant kVariantsCluRes[] = {  // the same with the residual stop (x* unknown)
    {1, 8, k_loop<1, 8, true, 0, true>, false, true},   {2, 8, k_loop<2, 8, true, 0, true>, false, true},
    {4, 8, k_loop<4, 8, true, 0, true>, false, true},   {8, 10, k_loop<8, 10, true, 0, true>, false, true},
    {16, 5, k_loop<16, 5, true, 0, true>, false, true}, {8, kTmRegRowsWide, k_loop<8, kTmRegRowsWide, true, 1, true>, true, true},
    {8, kTmRegRowsNarrow, k_loop<8, kTmRegRowsNarrow, true, 2, true>, true, true},
};
// Stream-ring variants (rows past the on-chip tiers through TMA stages):
// few register rows, so the registers go to the streamed chunk's loads
const LoopVariant kVariantsSt[] = {
    {1, 8, k_loop<1, 8, false, 0, false, true>},  {2, 8, k_loop<2, 8, false, 0, false, true>},
    {4, 8, k_loop<4, 8, false, 0, false, true>},  {8, 8, k_loop<8, 8, false, 0, false, true>},
    {8, kTmRegRowsWide, k_loop<8, kTmRegRowsWide, false, 1, false, true>, true},
};
const LoopVariant kVariantsStRes[] = {  // residual stop (no x*): the same ring, RES from the residuals
    {1, 8, k_loop<1, 8, true, 0, false, true>},  {2, 8, k_loop<2, 8, true, 0, false, true>},
    {4, 8, k_loop<4, 8, true, 0, false, true>},  {8, 8, k_loop<8, 8, true, 0, false, true>},
    {8, kTmRegRowsWide, k_loop<8, kTmRegRowsWide, true, 1, false, true>, true},
};
// (the host picks between a table and its residual-stop twin with ?:, which needs equal types)
static_assert(sizeof(kVariantsStRes) == sizeof(kVariantsSt), "stream-ring twins differ in size");
static_assert(sizeof(kVariantsCluRes) == sizeof(kVariantsClu), "cluster twins differ in size");
constexpr size_t kRingMaxBytes = 128 * 1024;  // per CTA, all groups' stages
const LoopVariant kVariantsRes[] = {
    {1, 32, k_loop<1, 32, true, 0, false>}, {2, 32, k_loop<2, 32, true, 0, false>}, {4, 20, k_loop<4, 20, true, 0, false>},
    {8, 10, k_loop<8, 10, true, 0, false>}, {16, 5, k_loop<16, 5, true, 0, false>},
};
// smallest instantiated RRMAX >= want for this CB (want <= rr_max_for(cb))
const LoopVariant *pick_variant(int cb, int want, bool resmode) {
    const LoopVariant *best = nullptr;
    if (resmode) {
        for (const auto &v : kVariantsRes)
            if (v.cb == cb) best = &v;
        return best;
    }
    for (const auto &v : kVariants)
        if (v.cb == cb && v.rrmax >= want && (!best || v.rrmax < best->rrmax)) best = &v;
    return best;
}

__global__ void k_sumsq_loop(const double *v, int64_t len, double *out) {
    __shared__ double red[32];
    double a = 0.0;
    for (int64_t i = threadIdx.x; i < len; i += blockDim.x) a = __fma_rn(v[i], v[i], a);
    a = lwarp_sum(a);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = red[0];
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) t = t + red[w];
        *out = t;
    }
}

}  // namespace

size_t loop_exchange_bytes(int total_ctas) {
    return kXchBytes + static_cast<size_t>(2) * total_ctas * kSlotWords * 8;
}

csk_status_t run_loop(csk_ctx_t ctx, const double *At, const double *bt, const double *nsq, int64_t d,
                      int64_t n, double *x, const double *x_star, double tol, int64_t max_iters,
                      const csk_solve_opts_t *opts, csk_report_t *report, cudaStream_t stream,
                      const RankSetup *ranks) {
    const bool multi = ranks != nullptr;
    const bool resmode = (x_star == nullptr);
    // group width: the fewest warps per group with n <= 256 WPG (<= 8 columns per thread:
    // fewer copies of x to update than 16 columns, still one warp per group for n <= 256)
    int wpg = 1;
    while (wpg < kLW && 32 * wpg * 8 < n) wpg *= 2;
    if (opts && opts->group_warps > 0) {
        if (opts->group_warps > kLW || (opts->group_warps & (opts->group_warps - 1)))
            return fail(ctx, CSK_E_ARG, "csk_solve: group_warps must be 1, 2, 4 or 8");
        if (opts->group_warps > wpg) wpg = opts->group_warps;
    }
    {  // A/B knob: force the group width (may go below the default: more columns per thread)
        static const int fw = getenv("CSK_LOOP_WPG") ? atoi(getenv("CSK_LOOP_WPG")) : 0;
        if (fw > 0 && fw <= kLW && (fw & (fw - 1)) == 0 && 32 * fw * 16 >= n) wpg = fw;
    }
    if (32 * wpg * 16 < n) return fail(ctx, CSK_E_UNSUPPORTED, "csk_solve: n too large for the register GEMV");
    int cb = 1;
    while (32 * wpg * cb < n) cb *= 2;
    const int flags = opts ? opts->flags : 0;
    const int rg = kLW / wpg;
    // Geometry for G CTAs: row tiers per group -- registers, then TMEM (8 columns per thread
    // only), then shared memory, then re-read from L2/HBM.
    // the ring's TMA copies need 16-B aligned rows: every rank's A~ base aligned, n even
    bool st_aligned = (reinterpret_cast<uintptr_t>(At) & 15) == 0;
    if (multi)
        for (int r = 0; r < ranks->P; ++r) st_aligned = st_aligned && (reinterpret_cast<uintptr_t>(ranks->At_r[r]) & 15) == 0;
    struct Geo {
        int G, rows_max, rb, rr, rt, rs, st_rows, st_stages;
        size_t smem;
        const LoopVariant *var;
    };
    auto geometry = [&](int Gw, bool clu, Geo &g, int rm_fixed = 0) {
        g.G = Gw;
        g.rows_max = rm_fixed > 0 ? rm_fixed : static_cast<int>((d + Gw - 1) / Gw);
        if (!clu && rm_fixed == 0) g.G = static_cast<int>((d + g.rows_max - 1) / g.rows_max);  // every CTA owns >= 1 row
        g.rb = (g.rows_max + rg - 1) / rg;  // max rows per group
        auto reg_rows = [&](int cap) {
            int r = cap;
            if (opts && opts->reg_rows < 0) r = 0;
            else if (opts && opts->reg_rows > 0 && opts->reg_rows < r) r = opts->reg_rows;
            return r < g.rb ? r : g.rb;
        };
        g.st_rows = 0;
        g.st_stages = 0;
        auto smem_fit = [&](int rest) {
            int f = 0;
            while (f < rest && loop_smem(g.rows_max, wpg, cb, n, f + 1, g.st_stages, g.st_rows).total <=
                                   static_cast<size_t>(ctx->max_smem_optin))
                ++f;
            if (opts && opts->smem_rows < 0) f = 0;
            else if (opts && opts->smem_rows > 0 && opts->smem_rows < f) f = opts->smem_rows;
            return f;
        };
        int rcap = rr_max_for(cb);
        if (clu) {  // the single-cluster variants carry <= 10 register rows (see kVariantsClu)
            rcap = 0;
            for (const auto &v : kVariantsClu)
                if (v.cb == cb && !v.tm && v.rrmax > rcap) rcap = v.rrmax;
        }
        g.rr = reg_rows(rcap);
        g.rt = 0;
        g.rs = smem_fit(g.rb - g.rr);
        const bool allow_tm = cb == 8 && !(flags & CSK_SOLVE_NO_TMEM);
        int tmk = 0;  // 1: wide TMEM loads (6 register rows), 2: narrow (8 register rows)
        if (allow_tm && ((flags & CSK_SOLVE_FORCE_TMEM) || g.rb - g.rr > 0)) {
            // narrow when every row past 8 register rows fits in TMEM (no shared-memory tier)
            tmk = (g.rb - kTmRegRowsNarrow <= kTmRows) ? 2 : 1;
            static const int ftmk = getenv("CSK_LOOP_TMK") ? atoi(getenv("CSK_LOOP_TMK")) : 0;  // A/B knob
            if (ftmk == 1 || ftmk == 2) tmk = ftmk;
            g.rr = reg_rows(tmk == 2 ? kTmRegRowsNarrow : kTmRegRowsWide);
            g.rt = (g.rb - g.rr) < kTmRows ? (g.rb - g.rr) : kTmRows;
            g.rs = smem_fit(g.rb - g.rr - g.rt);
            if (g.rt == 0) tmk = 0;
        }
        g.var = nullptr;
        if (clu) {
            const int want_rr = tmk == 2 ? kTmRegRowsNarrow : tmk == 1 ? kTmRegRowsWide : (g.rr > 0 ? g.rr : 1);
            for (const auto &v : (resmode ? kVariantsCluRes : kVariantsClu))
                if (v.cb == cb && v.tm == (tmk != 0) && v.rrmax >= want_rr && (tmk == 0 || v.rrmax == want_rr) &&
                    (!g.var || v.rrmax < g.var->rrmax))
                    g.var = &v;
        } else if (tmk == 1) {
            g.var = resmode ? &kVariantTmRes : &kVariantTm;
        } else if (tmk == 2) {
            g.var = resmode ? &kVariantTmNRes : &kVariantTmN;
        } else {
            g.var = pick_variant(cb, g.rr > 0 ? g.rr : 1, resmode);
        }
        // rows left over for L2/HBM: stream them through a TMA ring (whole rows, 16-B aligned:
        // n even and an aligned A~), taking shared memory from the resident rows
        if (!clu && g.var && g.rr + g.rt + g.rs < g.rb && (n % 2) == 0 && st_aligned &&
            !(flags & CSK_SOLVE_NO_STREAM_RING)) {
            const LoopVariant *sv = nullptr;
            for (const auto &v : (resmode ? kVariantsStRes : kVariantsSt))
                if (v.cb == cb && v.tm == (tmk == 1)) sv = &v;
            // rows per stage: a multiple of 4 (the GEMV passes), >= ~8 KB per stage for short rows
            int R = 4;
            while (R < 64 && static_cast<int64_t>(R + 4) * n * 8 <= 8192) R += 4;
            const size_t fixed = loop_smem(g.rows_max, wpg, cb, n, 0, 0, 0).total + static_cast<size_t>(rg) * 8 * 16;
            const size_t avail = static_cast<size_t>(ctx->max_smem_optin) > fixed ? ctx->max_smem_optin - fixed : 0;
            const size_t budget = avail < kRingMaxBytes ? avail : kRingMaxBytes;
            auto stages = [&](int r) {
                return static_cast<int>(std::min<size_t>(8, budget / (static_cast<size_t>(rg) * st_stage_bytes(n, r))));
            };
            while (R > 4 && stages(R) < 2) R -= 4;  // the largest stage that is still double-buffered
            const int S = stages(R);
            if (sv && tmk != 2 && S >= 2) {
                g.var = sv;
                if (g.rr > sv->rrmax) g.rr = sv->rrmax;
                g.st_rows = R;
                g.st_stages = S;
                g.rs = smem_fit(g.rb - g.rr - g.rt);
            }
        }
        g.smem = loop_smem(g.rows_max, wpg, cb, n, g.rs, g.st_stages, g.st_rows).total;
        return g.var != nullptr && g.smem <= static_cast<size_t>(ctx->max_smem_optin);
    };
    Geo geo{};
    bool clu = false;
    // Single 16-CTA cluster with the DSMEM exchange when the whole system fits on 16 SMs with
    // no streamed rows and is small enough that 16 SMs' GEMV beats the grid-wide exchange
    // (cluster_size: 0 = auto, 16 = prefer the cluster, 1 = never).
    const int want_cs = opts ? opts->cluster_size : 0;
    if (!multi && want_cs != 1 && (want_cs == kCS || (d * n <= kCluMaxElems && !(opts && opts->num_ctas > 0))) &&
        d >= kCS) {
        Geo g{};
        if (geometry(kCS, true, g) && g.rr + g.rt + g.rs >= g.rb) {
            CSK_CHECK(raise_smem(ctx, reinterpret_cast<const void *>(g.var->fn)));
            int ncl = 0;
            CSK_CHECK(max_resident(ctx, reinterpret_cast<const void *>(g.var->fn), kCS, kLT, g.smem, &ncl));
            if (ncl >= 1) {
                geo = g;
                clu = true;
            }
        }
    }
    if (multi) {
        // P ranks x Gr CTAs; the carve-up is sized by the largest rank's rows per CTA
        int64_t rm = 1;
        for (int r = 0; r < ranks->P; ++r) {
            const int64_t sz = ranks->dlo[r + 1] - ranks->dlo[r];
            rm = std::max<int64_t>(rm, (sz + ranks->Gr - 1) / ranks->Gr);
        }
        if (!geometry(ranks->Gr, false, geo, static_cast<int>(rm))) {
            if (!geo.var) return fail(ctx, CSK_E_UNSUPPORTED, "csk_solve: no kernel for this n");
            return fail(ctx, CSK_E_UNSUPPORTED, "csk_solve: too many rows per CTA for shared memory");
        }
    } else if (!clu) {
        int Gw = opts && opts->num_ctas > 0 ? opts->num_ctas : ctx->num_sms;
        if (Gw > d) Gw = static_cast<int>(d);
        if (!geometry(Gw, false, geo)) {
            if (!geo.var) return fail(ctx, CSK_E_UNSUPPORTED, "csk_solve: no kernel for this n");
            return fail(ctx, CSK_E_UNSUPPORTED, "csk_solve: too many rows per CTA for shared memory (use more CTAs)");
        }
    }
    const int G = geo.G, rows_max = geo.rows_max, rr = geo.rr, rt = geo.rt, rs = geo.rs;
    const size_t smem = geo.smem;
    const LoopVariant *var = geo.var;
    LoopFn fn = var->fn;
    if (multi) {  // the SYS twin of the chosen layout (virtual ranks included)
        const int tmk = !var->tm ? 0 : (var->rrmax == kTmRegRowsWide ? 1 : 2);
        const SysVariant *sv = nullptr;
        for (const auto &v : kVariantsSys)
            if (v.cb == var->cb && v.tmk == tmk && v.st == (geo.st_rows > 0) && v.res == resmode &&
                (tmk != 0 ? v.rrmax == var->rrmax : v.rrmax >= rr) && (!sv || v.rrmax < sv->rrmax))
                sv = &v;
        if (!sv) return CSK_E_UNSUPPORTED;  // the caller takes the host-driven NCCL loop
        fn = sv->fn;
    }
    CSK_CHECK(raise_smem(ctx, reinterpret_cast<const void *>(fn)));
    int per = 0;
    // CTAs of this launch (virtual ranks: all of them) and of the whole exchange
    const int grid = multi ? (ranks->rank < 0 ? ranks->P * ranks->Gr : ranks->Gr) : G;
    const int gtotal = multi ? ranks->P * ranks->Gr : G;
    if (!clu) {
        CSK_CHECK(max_resident(ctx, reinterpret_cast<const void *>(fn), 1, kLT, smem, &per));
        if (per < grid) return fail(ctx, CSK_E_UNSUPPORTED, "csk_solve: grid cannot be co-resident");
    }
    int kb = 1;
    while ((1ll << kb) < d + 1) ++kb;

    const size_t xch_bytes = kXchBytes;
    // multi-rank launches on this GPU (virtual ranks) need one exchange region per rank
    const int nreg = (multi && ranks->rank < 0) ? ranks->P : 1;
    // (a real rank's buffer holds its own region and its own [2][Gr] slots -- the peers' slots live
    //  in their memory; virtual ranks carve every rank's region and slots from this one buffer)
    const int slot_ctas = (multi && ranks->rank >= 0) ? ranks->Gr : gtotal;
    const size_t ex_bytes = loop_exchange_bytes(slot_ctas) + static_cast<size_t>(nreg - 1) * xch_bytes;
    void *const slots_before = ctx->slots.ptr;
    CSK_CHECK(ensure(ctx, ctx->slots, ex_bytes));
    if (multi && ranks->exchange_zeroed && ctx->slots.ptr != slots_before)
        return fail(ctx, CSK_E_CUDA, "csk_solve_sharded: the exported exchange buffer was reallocated");
    CSK_CHECK(ensure(ctx, ctx->report, 8 * 8));
    CSK_CHECK(ensure(ctx, ctx->scalars, 8 * 8));
    if (!(multi && ranks->exchange_zeroed)) CSK_CUDA(ctx, cudaMemsetAsync(ctx->slots.ptr, 0, ex_bytes, stream));
    const double *bb = static_cast<double *>(ctx->scalars.ptr);
    if (resmode) {
        if (multi && ranks->bb) bb = ranks->bb;
        else k_sumsq_loop<<<1, 1024, 0, stream>>>(bt, d, static_cast<double *>(ctx->scalars.ptr));
    }

    LoopParams prm{};
    prm.At = At; prm.bt = bt; prm.nsq = nsq; prm.d = d; prm.n = n; prm.x = x;
    if (!multi) {  // one GPU: one rank owning every row
        prm.P = 1; prm.rank = 0; prm.Gr = G; prm.sys = 0;
        prm.dlo[0] = 0; prm.dlo[1] = d;
        prm.RMr[0] = rows_max;
        // floor(i / RM) = (i M) >> 40 with M = ceil(2^40 / RM) for every i with i RM < 2^40
        // (the error i (M RM - 2^40) / 2^40 < i RM / 2^40 < 1 stays below the gap to the next multiple)
        const unsigned long long M = ((1ull << 40) + static_cast<unsigned long long>(rows_max) - 1) / static_cast<unsigned long long>(rows_max);
        if (static_cast<double>(d) * rows_max < 1099511627776.0 && static_cast<double>(d) * M < 1.8e19) prm.rm_magic = M;
        prm.At_r[0] = At; prm.bt_r[0] = bt; prm.nsq_r[0] = nsq; prm.x_r[0] = x;
    } else {
        prm.P = ranks->P; prm.rank = ranks->rank; prm.Gr = ranks->Gr; prm.sys = ranks->sys;
        for (int r = 0; r <= ranks->P; ++r) prm.dlo[r] = ranks->dlo[r];
        for (int r = 0; r < ranks->P; ++r)
            prm.RMr[r] = static_cast<int>((ranks->dlo[r + 1] - ranks->dlo[r] + ranks->Gr - 1) / ranks->Gr);
        for (int r = 0; r < ranks->P; ++r) {
            prm.At_r[r] = ranks->At_r[r]; prm.bt_r[r] = ranks->bt_r[r]; prm.nsq_r[r] = ranks->nsq_r[r];
            prm.x_r[r] = ranks->x_r[r];
        }
    }
    prm.x_star = x_star; prm.tol = tol; prm.max_iters = max_iters;
    prm.xch = static_cast<unsigned long long *>(ctx->slots.ptr);
    prm.slots = reinterpret_cast<unsigned long long *>(static_cast<unsigned char *>(ctx->slots.ptr) +
                                                       static_cast<size_t>(nreg) * xch_bytes);
    prm.slots_r[0] = prm.slots;
    if (multi) {
        for (int r = 0; r < ranks->P; ++r) {
            if (ranks->slots_r[r]) {  // real ranks: each rank's buffer is [its region][its slots]
                prm.slots_r[r] = ranks->slots_r[r];
                prm.xch_r[r] = reinterpret_cast<unsigned long long *>(
                    reinterpret_cast<unsigned char *>(ranks->slots_r[r]) - xch_bytes);
            } else {  // virtual ranks: regions and slot slices of this ctx's buffer
                prm.slots_r[r] = prm.slots + static_cast<size_t>(r) * 2 * ranks->Gr * kSlotWords;
                prm.xch_r[r] = reinterpret_cast<unsigned long long *>(static_cast<unsigned char *>(ctx->slots.ptr) +
                                                                      static_cast<size_t>(r) * xch_bytes);
            }
        }
    }
    prm.report = static_cast<int64_t *>(ctx->report.ptr);
    prm.bb = bb;
    prm.wpg = wpg;
    static const int fuse_ts = getenv("CSK_LOOP_FUSE_TS") ? atoi(getenv("CSK_LOOP_FUSE_TS")) : 1;  // A/B knob
    prm.fuse_ts = fuse_ts;
    static const int npoll = getenv("CSK_LOOP_NPOLL") ? atoi(getenv("CSK_LOOP_NPOLL")) : 1;  // A/B knobs
    static const int pdelay = getenv("CSK_LOOP_PDELAY") ? atoi(getenv("CSK_LOOP_PDELAY")) : 150;
    prm.npoll = npoll;
    prm.pdelay = pdelay;
    prm.rr = rr;
    prm.rs = rs;
    prm.rt = rt;
    prm.st_rows = geo.st_rows;
    prm.st_stages = geo.st_stages;
    // L2 residency of the streamed rows: the first CSK_LOOP_L2PIN_MB megabytes of them (split evenly
    // over the row groups, whole ring chunks) are copied with evict_last, the rest with evict_first,
    // so that part of A~ is served from L2 every iteration instead of from HBM.  0: no hints.
    static const int l2pin_mb = getenv("CSK_LOOP_L2PIN_MB") ? atoi(getenv("CSK_LOOP_L2PIN_MB")) : kLoopL2PinMB;
    static const int l2rest = getenv("CSK_LOOP_L2PIN_REST") ? atoi(getenv("CSK_LOOP_L2PIN_REST")) : 1;
    prm.st_rest_first = l2rest;
    prm.st_pin = -1;
    static const int l2minchunk =
        getenv("CSK_LOOP_L2PIN_MINCHUNK") ? atoi(getenv("CSK_LOOP_L2PIN_MINCHUNK")) : kLoopL2PinMinChunk;
    if (geo.st_rows > 0 && l2pin_mb > 0 && static_cast<int64_t>(geo.st_rows) * n * 8 >= l2minchunk) {
        const double chunk = static_cast<double>(geo.st_rows) * static_cast<double>(n) * 8.0;
        const double groups = static_cast<double>(G) * static_cast<double>(rg);
        prm.st_pin = static_cast<int>(static_cast<double>(l2pin_mb) * 1.0e6 / (chunk * groups));
    }
    prm.key_bits = kb;
    prm.rows_max = rows_max;
    prm.trace_cap = opts ? opts->trace_cap : 0;
    prm.idx_trace = opts ? opts->idx_trace : nullptr;
    prm.res_trace = opts ? opts->res_trace : nullptr;
    prm.x_trace = opts ? opts->x_trace : nullptr;
    prm.r_trace = (opts && opts->r_trace_cap > 0) ? opts->r_trace : nullptr;
    prm.r_trace_cap = prm.r_trace ? opts->r_trace_cap : 0;
    prm.d_glob = multi ? ranks->dlo[ranks->P] : d;
    prm.phase_cycles = opts ? opts->phase_cycles : nullptr;
    static const double tmo_s = getenv("CSK_EXCHANGE_TIMEOUT_S") ? atof(getenv("CSK_EXCHANGE_TIMEOUT_S")) : 30.0;
    prm.timeout_ns = static_cast<unsigned long long>(tmo_s * 1e9);
    prm.skew = (opts && opts->phase_cycles) ? reinterpret_cast<long long *>(opts->phase_cycles) + 32 : nullptr;
    if (prm.trace_cap <= 0) { prm.idx_trace = nullptr; prm.res_trace = nullptr; prm.x_trace = nullptr; prm.trace_cap = 0; }

    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    if (clu) {  // one 16-CTA cluster: co-scheduled by construction, no cooperative launch needed
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = kCS;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
    } else {
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
    }
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kLT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    // Profiling only (ncu cannot replay cooperative launches): same kernel without the attribute.
    static const bool noncoop = getenv("CSK_PROFILE_NONCOOP") != nullptr;
    if (noncoop && !clu) cfg.numAttrs = 0;
    time_mark(ctx, 1, false, stream);
    CSK_CUDA(ctx, cudaLaunchKernelEx(&cfg, fn, prm));
    time_mark(ctx, 1, true, stream);
    static const bool dbg = getenv("CSK_DEBUG") != nullptr;
    if (dbg)
        fprintf(stderr, "[csk] loop: d=%lld n=%lld G=%d cluster=%d wpg=%d cb=%d rrmax=%d tm=%d rr=%d rt=%d rs=%d ring=%dx%d rows/CTA=%d smem=%zu\n",
                (long long)d, (long long)n, G, clu ? kCS : 0, wpg, cb, var->rrmax, (int)var->tm, rr, rt, rs,
                geo.st_stages, geo.st_rows, rows_max, smem);
    ctx->last_solve_geom[0] = G;
    ctx->last_solve_geom[1] = clu ? kCS : 1;
    ctx->last_solve_geom[2] = rs;
    ctx->last_solve_geom[3] = rr;
    ctx->last_solve_geom[4] = wpg;
    {
        const int t[8] = {G, clu ? kCS : 1, rr, rt, rs, wpg, geo.st_stages, geo.st_rows};
        for (int i = 0; i < 8; ++i) ctx->last_solve_tiers[i] = t[i];
    }
    CSK_CHECK(ensure_host_report(ctx));
    CSK_CUDA(ctx, cudaMemcpyAsync(ctx->report_host, ctx->report.ptr, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
    ctx->pending_stream = stream;
    ctx->pending_resmode = resmode;
    ctx->pending = true;
    if (opts && (opts->flags & CSK_SOLVE_ASYNC)) return CSK_OK;
    return finish_solve(ctx, report);
}

}  // namespace csk
