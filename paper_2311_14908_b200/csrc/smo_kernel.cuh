// smo_kernel.cuh -- the persistent, row-sharded SMO solver kernel for sm_100a.
//
// One launch runs many SMO iterations (§3.2: "a thread per
// independent training data sample ... convergence checks ... for every set of
// iterations").  Design (DESIGN.md §"Kernels"):
//
//   * Rows are sharded over ranks (GPUs, or CTA groups of one GPU) and, inside a
//     rank, over CTAs: CTA c owns a contiguous row block for the whole solve and keeps
//     its solver state -- f (fp64), flags (y, I_up, I_low) and, when it fits, alpha --
//     in shared memory.  Only X is streamed per iteration.
//   * X lives in HBM in a CTA-blocked, feature-major layout ("xblk"): per CTA, tiles of
//     rt rows, each tile [d_pad][rows] fp32.  Warp roles (one CTA per SM):
//       warps 0-7  consumers: one thread per RPT rows; distances, kernel values,
//                  f-update, status, local (f, index) candidates
//       warp 8     scalar warp: candidate record publish, cross-CTA / cross-rank
//                  exchange, combine, pivot gather, pair update (serial fp64), all
//                  overlapped with the consumers' streaming of the next tile
//       warp 9     producer: TMA bulk copies (cp.async.bulk) of X stages into a
//                  shared-memory ring, mbarrier full/empty pipeline
//   * Per iteration (rows a2-a7 of SURVEY.md §8):
//       C  consumers hand their warp candidates to the scalar warp (named barrier 3)
//       scalar warp: CTA record -> every rank's mailbox (peer pointers when the ranks
//          are GPUs) + release atomic on a monotonic arrival counter; wait for all
//          records; lexicographic combine (f, then lowest global index) -> (i_up,
//          i_low), identical in every CTA; convergence test b_low - b_up <= 2 tol
//          (device-latched); gather x_up, x_low from the row-major replica
//       A  consumers start streaming (named barrier 1)
//       scalar warp: eta, clipped step t, snapped alphas, c_u, c_l;
//          owner CTA updates its alpha/flags
//       B  consumers apply f_j = fma(c_l, K_l, fma(c_u, K_u, f_j)) (named barrier 2)
//   * Exact readings: no contraction (--fmad=false), explicit fma where the oracle has
//     one, correctly rounded exp, exact comparisons on alpha.  Results do not depend on
//     the number of ranks / CTAs.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "svm_exp.cuh"

namespace svmk {

constexpr int MAXR = 8;            // max ranks (GPUs or virtual)
constexpr int NT = 256;            // consumer threads per CTA
constexpr int NWC = NT / 32;       // consumer warps
constexpr int SCALAR_WARP = NWC;   // warp 8
constexpr int PRODUCER_WARP = NWC + 1;
constexpr int NTHREADS = NT + 64;  // + scalar warp + producer warp
constexpr int NSYNC = NT + 32;     // participants of the named barriers
constexpr int MAX_STAGES = 16;
constexpr int MIX_MAXSEG = 8;      // mixed rows: at most this many runs of continuous / binary columns
enum { BAR_A = 1, BAR_B = 2, BAR_C = 3, BAR_D = 4, BAR_E = 5 };

enum { ST_RUNNING = 0, ST_CONVERGED = 1, ST_MAXITER = 2, ST_LIMIT = 3, ST_TIMEOUT = -8 };
enum { FL_POS = 1, FL_UP = 2, FL_LOW = 4 };

// One CTA's candidate record: four 16-byte words.  A word carries a 32-bit aux field a and
// a 64-bit payload v in two 8-byte halves, each tagged with the 16-bit sequence number sq
// of the exchange that wrote it (the low 16 bits of the exchange number; the stale
// content of a slot is exchange sq - 2):
//     half 0 = v[31:0] | (a[15:0] << 32) | (sq << 48)
//     half 1 = v[63:32] | (a[31:16] << 32) | (sq << 48)
// Words are written and read as two 64-bit elements (st/ld .v2.u64, relaxed): each
// naturally aligned 64-bit element is single-copy atomic, so a reader that sees sq in
// both halves has read one whole word of exchange sq -- however the 16-byte access is
// split on its way (NVLink, L2) -- and needs no fence, counter or flag ordering.
// Payloads:
//   w0 = (a: i_up, v: f_up)    w1 = (i_low, f_low)
//   w2 = (y_up | y_low << 16, a_up)    w3 = (0, a_low)
// (i = global row, 0xffffffff = empty set).  The mailbox stores the words transposed,
// word[parity][h][g], so one warp load of word h covers 32 consecutive records; the
// selection polls w0/w1 only and fetches w2/w3 of the two winning records afterwards.
struct __align__(128) Mailbox {
    unsigned long long pad[16];
};
__host__ __device__ inline uint4* mbox_words(Mailbox* m, int parity, int h, int g_total) {
    return reinterpret_cast<uint4*>(m + 1) + ((size_t)parity * 4 + h) * g_total;
}
__host__ __device__ inline const uint4* mbox_words(const Mailbox* m, int parity, int h, int g_total) {
    return reinterpret_cast<const uint4*>(m + 1) + ((size_t)parity * 4 + h) * g_total;
}
__host__ __device__ inline size_t mbox_bytes(int cpr, int world) {
    return sizeof(Mailbox) + (size_t)2 * 4 * cpr * world * sizeof(uint4);
}

struct Ctl {                       // per rank solver control, persists across launches
    long long it;                  // SMO updates done
    long long seq;                 // exchanges done
    int state;
    int pad;
    double b_up, b_low;
    long long i_up, i_low;
    long long cache_hits, cache_misses;   // row-cache lookups (a8), accumulated over launches
};

struct Params {
    int kernel;
    double gamma, C, tol;
    long long max_iter, iter_limit;
    int d, d_pad, kc, n_chunks, stages, rt;
    int world, rank_base, ctas_per_rank;
    long long n_global;
    const float* xr;               // row-major replica [n_global][d]
    long long cta_stride;          // floats per CTA block in xblk
    long long row_off[MAXR];
    int n_rows[MAXR];
    const float* xblk[MAXR];
    double* f[MAXR];
    double* alpha[MAXR];
    uint8_t* flags[MAXR];
    Mailbox* mbox[MAXR];
    Ctl* ctl[MAXR];
    long long* trace;
    long long trace_cap;
    double* hist;                  // optional [2 trace_cap]: (c_u, c_l) of every update (shrinking replay)
    unsigned long long* progress;  // host-mapped, may be null
    int check_interval;
    int state_cap;                 // rows per CTA the shared-memory state can hold
    int resident;                  // 1: the CTA's whole X block stays in shared memory (one tile)
    int bin_words;                 // > 0: X is exactly binary (every value 0 or 1) and stored as
                                   // bit rows of bin_words 32-bit words (SURVEY §8(f) compact
                                   // encoding); distances are popcounts -- exact, so identical to
                                   // the fp64 recurrence R13
    const uint32_t* xrbits;        // bit rows [n_global][bin_words] (pivot gather)
    const double* gram;            // full-Gram path (a9): K [n_global][n_global], rows read per
                                   // iteration instead of streaming X (one rank only)
    double* cache[MAXR];           // row cache (a8): [cache_slots][n_rows[r]] per rank, or null
    int cache_slots;
    int cache_hash;                // hash entries (power of two >= 2 cache_slots)
    int independent;               // 1: every rank is its own problem (batched OvO solves): no
                                   // exchange between ranks, per-rank X / max_iter below
    const float* xr_rank[MAXR];    // independent mode: row-major X of problem r
    long long max_iter_rank[MAXR]; // independent mode: max_iter of problem r
    long long timeout_ns;
    int sys_scope;                 // 1 when mailboxes live on other GPUs (system scope)
    int cluster;                   // 1: the ctas_per_rank CTAs of a rank form one thread-block
                                   // cluster and exchange through distributed shared memory
    int crow;                      // cluster mode: 32-bit words of a candidate row carried in
                                   // its record (binary: bin_words, else d), 0 = rows gathered
    int crw;                       // cluster mode: 16-byte words per record (4 + 2 ceil(crow/3))
    unsigned long long* timers;    // optional [8] per-phase cycle totals of CTA 0
    int poll_ns;                   // > 0: back-off between mailbox polls (tuning)
    unsigned long long* dbg_ts;    // diagnostic (SVMB200_SKEW_TS = N): per (iteration < N, CTA) {row-pass start, publish} globaltimer, smid
    int dbg_ts_n;
    int dbg_fast_only;
    int xch_dup;                   // >= 1, test hook (one process): every record also stored in xch_dup - 1 more
                                   // slots, so one GPU polls as many records as xch_dup GPUs would             // diagnostic only (SVMB200_DBG_FAST_ONLY): skip the exp slow phase -- WRONG results, timing probe
    int dp;                        // dense pivot entries in shared memory (>= d; = d_pad unless mixed)
    // Mixed compact rows (SURVEY §8(f) compact encodings): the columns whose values are all
    // exactly 0 or 1 are stored as bits, the others as fp32.  A row of xblk holds mix_nc fp32
    // slots (the continuous columns in order) then mix_nbw bit words (the binary columns in
    // order).  mix_seg lists the runs of the original column order: > 0 = that many
    // continuous columns, < 0 = that many binary columns.  A binary column adds a term of
    // exactly 0 or 1 to the R13 recurrence, so a run adds 1.0 popcount times -- the same
    // roundings as the dense recurrence.  mix_map[i]: original column of continuous slot i
    // (i < mix_nc) / of binary bit i - mix_nc.
    int mix_nseg, mix_nc, mix_nbw;
    int mix_seg[MIX_MAXSEG];
    const int* mix_map;
    const uint32_t* xcomp;         // mixed rows, no row cache: every row of the problem in its
                                   // compact form, row-major [n_global][mix_nc + mix_nbw], so the
                                   // two pivots are gathered compact (one load per word) and
                                   // K(x_u, x_l) is computed from them
    // Dictionary-coded rows (SURVEY §8(f) compact encodings: uint8 pixels): when X holds at
    // most 256 distinct fp32 values, xblk stores one byte per element, the index of its
    // value in dict (the values widened to fp64 exactly); the row pass looks the value up,
    // so the arithmetic is the dense path's.  dict_n = 0: not dictionary-coded.
    int dict_n;
    const double* dict;
    // Working-set selection: 1 = the maximal violating pair (reading
    // R1); 2 = second order (Fan, Chen & Lin 2005, cited at P:L140): u as in R1, then
    // l = argmax over t in I_low with f_t > f_u of (f_t - f_u)^2 / a_t,
    // a_t = K_uu + K_tt - 2 K_ut (<= 1e-12 -> 1e-12), lowest index on ties.  An iteration
    // is then two row passes: a gain pass over K(x_u, .) and its exchange, then the update
    // pass over K(x_u, .), K(x_l, .).
    int wss;
    const double* qself;           // wss 2, linear kernel: x_t . x_t of every global row (R13 order)
    int l2_prefetch;               // streamed X: the producer also prefetches into L2 the stage
                                   // l2_prefetch stages beyond the ring (cp.async.bulk.prefetch.L2),
                                   // so HBM keeps streaming while the ring is full -- during the
                                   // exchange, when the consumers wait (0 = off)
    int l2_keep_chunks;            // streamed X: the first l2_keep_chunks stages (tile-major) of
                                   // every CTA block are copied with an L2 evict_last policy, the
                                   // rest evict_first, so that part of X stays in L2 across
                                   // iterations (0 = no hints)
};

// phase timers (cycles, CTA 0): scalar warp lane 0 ...
enum { PH_S_WAITC = 0, PH_S_PUBLISH, PH_S_POLL, PH_S_READ, PH_S_PIVOT, PH_S_KUL,
       // ... and consumer thread 0
       PH_C_EXCH, PH_C_PIVOT, PH_C_DIST, PH_C_WAITB, PH_C_UPDATE, PH_C_REDUCE,
       PH_S_CAND, PH_S_BUILD, PH_N };

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    return ok != 0;
}
// the same with a suspend-time hint: the thread sleeps until the phase completes (or the
// hint elapses) instead of spinning -- the producer lane and waiting consumers then leave
// the issue slots to the warps doing row work (ncu on W4: the producer's spin loop was ~6%
// of the instructions issued)
__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity), "r"(ns) : "memory");
    return ok != 0;
}
__device__ __forceinline__ long long globaltimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// Pipeline waits are local to the CTA and complete within microseconds; a wait that
// spins for 30 s means a broken pipeline, so it traps (kernel error, not a hang).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    unsigned int spins = 0;
    long long t0 = 0;
    while (!mbar_try_wait_sleep(bar, parity, 2000u)) {
        if ((++spins & 4095u) == 0) {
            const long long now = globaltimer();
            if (t0 == 0) t0 = now;
            else if (now - t0 > 30ll * 1000 * 1000 * 1000) asm volatile("trap;");
        }
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy) : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint64_t l2_policy(bool keep) {
    uint64_t p;
    if (keep) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
template <int NS = NSYNC>
__device__ __forceinline__ void named_sync(int id) {
    asm volatile("bar.sync %0, %1;" :: "r"(id), "n"(NS) : "memory");
}
template <int NS = NSYNC>
__device__ __forceinline__ void named_arrive(int id) {
    asm volatile("bar.arrive %0, %1;" :: "r"(id), "n"(NS) : "memory");
}

// ---- thread-block cluster (distributed shared memory) helpers
__device__ __forceinline__ uint32_t cluster_map(const void* p, int cta) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(cta));
    return r;
}
// record words (see Mailbox) move as two 64-bit elements: {x, y} and {z, w}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, uint4 v) {
    const unsigned long long h0 = (unsigned long long)v.x | ((unsigned long long)v.y << 32);
    const unsigned long long h1 = (unsigned long long)v.z | ((unsigned long long)v.w << 32);
    asm volatile("st.relaxed.cluster.shared::cluster.v2.u64 [%0], {%1, %2};"
                 :: "r"(addr), "l"(h0), "l"(h1) : "memory");
}
__device__ __forceinline__ uint4 ld_volatile_shared_v4(const uint4* p) {
    unsigned long long h0, h1;
    asm volatile("ld.relaxed.cluster.shared::cta.v2.u64 {%0, %1}, [%2];"
                 : "=l"(h0), "=l"(h1) : "r"(smem_u32(p)) : "memory");
    return make_uint4((uint32_t)h0, (uint32_t)(h0 >> 32), (uint32_t)h1, (uint32_t)(h1 >> 32));
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Lexicographic "better" for the two selections: smaller f wins for I_up,
// larger f for I_low, and the lower index wins a tie.  Empty = index INT_MAX.
__device__ __forceinline__ bool better_up(double f1, int i1, double f2, int i2) {
    return f1 < f2 || (f1 == f2 && i1 < i2);
}
__device__ __forceinline__ bool better_low(double f1, int i1, double f2, int i2) {
    return f1 > f2 || (f1 == f2 && i1 < i2);
}

__device__ __forceinline__ uint8_t flags_of(int y, double a, double C) {
    uint8_t fl = (y > 0) ? FL_POS : 0;
    if ((y > 0 && a < C) || (y < 0 && a > 0.0)) fl |= FL_UP;
    if ((y > 0 && a > 0.0) || (y < 0 && a < C)) fl |= FL_LOW;
    return fl;
}

// ------------------------------------------------------------------ shared layout
struct Shared {
    volatile int stop;
    volatile int producer_done;
    volatile unsigned int issued;
    int decision;                  // ST_*, written by the scalar warp before barrier A
    int u, l;                      // global winners of this iteration
    double f_up, f_low;
    double cu, cl;                 // written by the scalar warp before barrier B
    int pass;                      // wss 2: 1 = this row pass is the gain pass of u (barrier A)
    double gain_kuu, gain_fu;      // wss 2 gain pass: K(x_u, x_u) and f_u (barrier B)
    double red_f[2][16];           // per consumer warp candidates (local row index; <= 16 warps)
    double red_a[2][16];           // ... and their alpha when alpha lives in HBM (read by the
                                   // consumer warps, off the scalar warp's critical path)
    int red_i[2][16];
    double wp_f[2][16];            // wide poll: per consumer warp best (f, global row, record)
    int wp_i[2][16], wp_g[2][16];
    int c_hit, c_su, c_sl;         // row cache: both rows cached / their slots
    int c_fill_u, c_fill_l;        // row cache: the slot this iteration fills (miss), else -1
    int lru_head, lru_tail;        // row cache: most / least recently used slot
    int kul_cnt;                   // compacted terms of K(x_u, x_l) (cache mode)
    int timeout;
    // phase timers (diagnostic): consumer thread 0 uses row 0, the scalar warp's lane 0 row 1
    // (in shared memory, not registers: 14 accumulators live across the whole solve loop
    // cost the row pass registers even when timing is off)
    unsigned long long ph_acc[2][PH_N];
    long long ph_t[2];
    unsigned long long bars[2 * MAX_STAGES];
    double exp_tab[svmexp::EXP_TABLE_DOUBLES];
};

template <bool UP>
__device__ __forceinline__ void warp_reduce_fi(double& f, int& i, int width = 32) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        if (o >= width) continue;
        const double f2 = __shfl_xor_sync(0xffffffffu, f, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, i, o);
        const bool take = UP ? better_up(f2, i2, f, i) : better_low(f2, i2, f, i);
        if (take) { f = f2; i = i2; }
    }
}

// Order-preserving 64-bit key of a double (no NaNs; -0 is keyed as +0, since the
// selections compare f values with ==, under which -0 == +0).
__device__ __forceinline__ unsigned long long fkey(double f) {
    unsigned long long b = (unsigned long long)__double_as_longlong(f);
    if (b == 0x8000000000000000ull) b = 0ull;
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double fkey_inv(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}
// Lexicographic minimum of (key, idx) over the lanes of `mask` (every lane of the mask
// calls it with the same mask): three warp reductions on 32-bit halves.  The winner's
// key and index are returned to every lane of the mask.
__device__ __forceinline__ void argmin_redux(unsigned mask, unsigned long long key, unsigned idx,
                                             unsigned long long& kmin, unsigned& imin) {
    const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
    const unsigned mh = __reduce_min_sync(mask, hi);
    const unsigned ml = __reduce_min_sync(mask, hi == mh ? lo : 0xffffffffu);
    imin = __reduce_min_sync(mask, (hi == mh && lo == ml) ? idx : 0xffffffffu);
    kmin = ((unsigned long long)mh << 32) | ml;
}

// (the volatile shared load forces a deferred-blocking bar.sync to resolve before
// the clock is read)
// A (candidate up, candidate low) pair with the alpha and label of each.
struct Cand {
    double fu, fl, au, al;
    int iu, il, yu, yl;
};
__device__ __forceinline__ uint4 rec_pack(uint32_t sq, uint32_t a, unsigned long long v) {
    return make_uint4((uint32_t)v, (sq << 16) | (a & 0xffffu), (uint32_t)(v >> 32), (sq << 16) | (a >> 16));
}
// word h (0..3) of the record of candidate c for exchange sq
__device__ __forceinline__ uint4 rec_word(const Cand& c, int h, uint32_t sq) {
    if (h == 0) return rec_pack(sq, c.iu == INT_MAX ? 0xffffffffu : (uint32_t)c.iu, (unsigned long long)__double_as_longlong(c.fu));
    if (h == 1) return rec_pack(sq, c.il == INT_MAX ? 0xffffffffu : (uint32_t)c.il, (unsigned long long)__double_as_longlong(c.fl));
    if (h == 2) return rec_pack(sq, (uint32_t)((c.yu & 0xffff) | (c.yl << 16)), (unsigned long long)__double_as_longlong(c.au));
    return rec_pack(sq, 0u, (unsigned long long)__double_as_longlong(c.al));
}
// both 8-byte halves were written by exchange sq
__device__ __forceinline__ bool rec_ok(const uint4& v, uint32_t sq) {
    return (((v.y ^ (sq << 16)) | (v.w ^ (sq << 16))) >> 16) == 0u;
}
__device__ __forceinline__ uint32_t rec_aux(const uint4& v) { return (v.y & 0xffffu) | (v.w << 16); }
__device__ __forceinline__ uint32_t rec_lo(const uint4& v) { return v.x; }
__device__ __forceinline__ uint32_t rec_hi(const uint4& v) { return v.z; }
__device__ __forceinline__ unsigned long long rec_payload(const uint4& v) {
    return (unsigned long long)v.x | ((unsigned long long)v.z << 32);
}
__device__ __forceinline__ double rec_f64(const uint4& v) {
    return __longlong_as_double((long long)rec_payload(v));
}
__device__ __forceinline__ int rec_idx(const uint4& v) {
    const uint32_t a = rec_aux(v);
    return a == 0xffffffffu ? INT_MAX : (int)a;
}
__device__ __forceinline__ void rec_store(uint4* p, uint4 v, int sys) {
    const unsigned long long h0 = (unsigned long long)v.x | ((unsigned long long)v.y << 32);
    const unsigned long long h1 = (unsigned long long)v.z | ((unsigned long long)v.w << 32);
    if (sys)
        asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" :: "l"(p), "l"(h0), "l"(h1) : "memory");
    else
        asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" :: "l"(p), "l"(h0), "l"(h1) : "memory");
}
__device__ __forceinline__ uint4 rec_load(const uint4* p, int sys) {
    unsigned long long h0, h1;
    if (sys)
        asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(h0), "=l"(h1) : "l"(p) : "memory");
    else
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(h0), "=l"(h1) : "l"(p) : "memory");
    return make_uint4((uint32_t)h0, (uint32_t)(h0 >> 32), (uint32_t)h1, (uint32_t)(h1 >> 32));
}

#define SVM_PHASE(on, ph)                                                    \
    do {                                                                     \
        if (on) {                                                            \
            (void)*(volatile int*)&sh.decision;                              \
            const long long c_ = clock64();                                  \
            sh.ph_acc[ph_row][ph] += (unsigned long long)(c_ - sh.ph_t[ph_row]); \
            sh.ph_t[ph_row] = c_;                                            \
        }                                                                    \
    } while (0)

// ------------------------------------------------------------------ the kernel
// The scalar warp's record poll: lane L reads words 0 and 1 (the up and low candidates)
// of records L, L + 32, ... (PB records in flight), re-reading the ones not yet written by
// exchange sq, and keeps the lexicographically best up / low candidate it saw with the
// record it came from (gu, gl).  Returns true (warp-uniform) on timeout.
struct Sel {
    double fu, fl;
    int iu, il, gu, gl;
};
template <int PB>
__device__ __forceinline__ bool poll_records(const uint4* w0, const uint4* w1, int g_total, uint32_t sq,
                                             int sys, long long timeout_ns, int lane, Sel& b,
                                             unsigned int& rounds) {
    b.fu = __longlong_as_double(0x7ff0000000000000ll); b.fl = -b.fu;
    b.iu = INT_MAX; b.il = INT_MAX; b.gu = 0; b.gl = 0;
    bool tmo = false;
    long long t0 = 0;
    unsigned int spins = 0;
    for (int g0 = 0; g0 < g_total && !tmo; g0 += 32 * PB) {
        uint4 v[PB][2];
        unsigned pend = 0;
#pragma unroll
        for (int q = 0; q < PB; ++q) if (g0 + 32 * q + lane < g_total) pend |= 1u << q;
        const unsigned mine = pend;
        while (pend) {
            ++rounds;
#pragma unroll
            for (int q = 0; q < PB; ++q)
                if (pend & (1u << q)) {
                    const int g = g0 + 32 * q + lane;
                    v[q][0] = rec_load(w0 + g, sys);
                    v[q][1] = rec_load(w1 + g, sys);
                }
#pragma unroll
            for (int q = 0; q < PB; ++q)
                if ((pend & (1u << q)) && rec_ok(v[q][0], sq) && rec_ok(v[q][1], sq)) pend &= ~(1u << q);
            if (pend && (++spins & 255u) == 0) {
                const long long now = globaltimer();
                if (t0 == 0) t0 = now;
                else if (now - t0 > timeout_ns) { tmo = true; break; }
            }
        }
#pragma unroll
        for (int q = 0; q < PB; ++q)
            if (mine & (1u << q)) {
                const int g = g0 + 32 * q + lane;
                const int iu = rec_idx(v[q][0]), il = rec_idx(v[q][1]);
                const double fu = rec_f64(v[q][0]), fl = rec_f64(v[q][1]);
                if (iu != INT_MAX && better_up(fu, iu, b.fu, b.iu)) { b.fu = fu; b.iu = iu; b.gu = g; }
                if (il != INT_MAX && better_low(fl, il, b.fl, b.il)) { b.fl = fl; b.il = il; b.gl = g; }
            }
        tmo = __any_sync(0xffffffffu, tmo);
    }
    return tmo;
}

// The wide poll (g_total > 160 records, i.e. several GPUs): every consumer thread polls
// records first, first + stride, ... (up to MAXR loads in flight), re-reading the ones not
// yet written by exchange sq, and keeps the best up / low candidate it saw with its record.
// The consumers are idle during the exchange; one warp polling 1,184 records (8 GPUs x 148
// CTAs) would need 8 sequential rounds of loads.  Returns true on timeout (this thread).
template <int MAXR>
__device__ __forceinline__ bool poll_slice(const uint4* w0, const uint4* w1, int g_total, uint32_t sq,
                                           int sys, long long timeout_ns, int first, int stride, Sel& b) {
    b.fu = __longlong_as_double(0x7ff0000000000000ll); b.fl = -b.fu;
    b.iu = INT_MAX; b.il = INT_MAX; b.gu = 0; b.gl = 0;
    bool tmo = false;
    long long t0 = 0;
    unsigned int spins = 0;
    for (int g0 = first; g0 < g_total && !tmo; g0 += MAXR * stride) {
        uint4 v[MAXR][2];
        unsigned pend = 0;
#pragma unroll
        for (int q = 0; q < MAXR; ++q) if (g0 + q * stride < g_total) pend |= 1u << q;
        const unsigned mine = pend;
        while (pend) {
#pragma unroll
            for (int q = 0; q < MAXR; ++q)
                if (pend & (1u << q)) {
                    v[q][0] = rec_load(w0 + g0 + q * stride, sys);
                    v[q][1] = rec_load(w1 + g0 + q * stride, sys);
                }
#pragma unroll
            for (int q = 0; q < MAXR; ++q)
                if ((pend & (1u << q)) && rec_ok(v[q][0], sq) && rec_ok(v[q][1], sq)) pend &= ~(1u << q);
            if (pend && (++spins & 255u) == 0) {
                const long long now = globaltimer();
                if (t0 == 0) t0 = now;
                else if (now - t0 > timeout_ns) { tmo = true; break; }
            }
        }
#pragma unroll
        for (int q = 0; q < MAXR; ++q)
            if (mine & (1u << q)) {
                const int g = g0 + q * stride;
                const int iu = rec_idx(v[q][0]), il = rec_idx(v[q][1]);
                const double fu = rec_f64(v[q][0]), fl = rec_f64(v[q][1]);
                if (iu != INT_MAX && better_up(fu, iu, b.fu, b.iu)) { b.fu = fu; b.iu = iu; b.gu = g; }
                if (il != INT_MAX && better_low(fl, il, b.fl, b.il)) { b.fl = fl; b.il = il; b.gl = g; }
            }
    }
    return tmo;
}

// Word k of local row j in a CTA's resident binary block (row j at words [j Wp, j Wp + Wp)).
__device__ __forceinline__ uint32_t bin_row_word(const float* ring, int j, int k, int W) {
    return reinterpret_cast<const uint32_t*>(ring)[(size_t)j * ((W + 3) & ~3) + k];
}

// Row cache (a8): rank owning global row g (ranks 0..world-1 hold consecutive blocks).
__device__ __forceinline__ int cache_owner(const Params& P, long long g) {
    int r = 0;
    while (r + 1 < P.world && g >= P.row_off[r + 1]) ++r;
    return r;
}
// K_ul can be read from a cached row when the columns it needs live on this GPU.
__device__ __forceinline__ bool kul_cache_ok(const Params& P, int u, int l) {
    if (P.independent) return false;
    return P.cache[cache_owner(P, l)] != nullptr && P.cache[cache_owner(P, u)] != nullptr;
}
// Column g of the cached kernel row in slot s.
__device__ __forceinline__ double kcache_at(const Params& P, int s, long long g) {
    const int r = cache_owner(P, g);
    return __ldcg(P.cache[r] + (long long)s * P.n_rows[r] + (g - P.row_off[r]));
}

// The RPT rows t*RPT .. t*RPT+RPT-1 of slot (feature) i of a stage [slots][rp]
template <int RPT>
__device__ __forceinline__ void load_slot(const float* st, int rp, int i, int t, uint32_t (&v)[RPT]) {
    if (RPT == 4) {
        const uint4 w = reinterpret_cast<const uint4*>(st + (size_t)i * rp)[t];
        v[0] = w.x; v[1 % RPT] = w.y; v[2 % RPT] = w.z; v[3 % RPT] = w.w;
    } else if (RPT == 2) {
        const uint2 w = reinterpret_cast<const uint2*>(st + (size_t)i * rp)[t];
        v[0] = w.x; v[1 % RPT] = w.y;
    } else {
        v[0] = reinterpret_cast<const uint32_t*>(st)[(size_t)i * rp + t];
    }
}
// acc + 1.0, c times (the R13 terms of c binary columns whose term is 1), c >= 0: one add
// when that add is exact and acc >= 0 (then every intermediate sum is exact too: they are
// multiples of ulp(acc + c) no larger than it), else c sequential adds.  (A variant that
// walks the binade crossings instead of the c additions measured slower on W4: the common
// c is 0, 2 or 4.)
__device__ __forceinline__ double add_ones(double acc, int c) {
    if (c <= 4) {
        // the common case (W4's one-hot groups give c = 0, 2 or 4): the four sequential
        // additions, branch-free, and the c-th result (ncu: the data-dependent loop below
        // was the most executed line of the W4 row pass)
        const double a1 = acc + 1.0, a2 = a1 + 1.0, a3 = a2 + 1.0, a4 = a3 + 1.0;
        return c == 0 ? acc : c == 1 ? a1 : c == 2 ? a2 : c == 3 ? a3 : a4;
    }
    const double cd = (double)c;
    const double s = acc + cd;
    const double bb = s - acc;
    const double err = (acc - (s - bb)) + (cd - bb);
    if (err == 0.0 && acc >= 0.0 && s < 9007199254740992.0) return s;
    for (int i = 0; i < c; ++i) acc = acc + 1.0;
    return acc;
}
// Mixed compact rows (Params::mix_*): the R13 recurrence of RPT rows against both pivots,
// run by run in the original column order.
template <int KERNEL, int RPT>
__device__ __forceinline__ void mixed_rows(const Params& P, const float* st, int rp, int t,
                                           const double2* pivm, const uint32_t* pbits,
                                           double (&du)[RPT], double (&dl)[RPT]) {
    if (P.mix_nseg == 2 && P.mix_seg[0] > 0) {
        // the common layout (W4): the continuous columns, then one run of every binary
        // column -- no run bookkeeping, and no bit masks (the padding bits of the last
        // word are 0 in the rows and in the pivots)
        const int nc = P.mix_nc;
#pragma unroll 2
        for (int i = 0; i < nc; ++i) {
            uint32_t v[RPT];
            load_slot<RPT>(st, rp, i, t, v);
            const double2 pv = pivm[i];
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const double x = (double)__uint_as_float(v[q]);
                if (KERNEL == 1) {
                    double e = x - pv.x; du[q] = fma(e, e, du[q]);
                    e = x - pv.y; dl[q] = fma(e, e, dl[q]);
                } else {
                    du[q] = fma(x, pv.x, du[q]); dl[q] = fma(x, pv.y, dl[q]);
                }
            }
        }
        int cu[RPT], cl[RPT];
#pragma unroll
        for (int q = 0; q < RPT; ++q) { cu[q] = 0; cl[q] = 0; }
        for (int w = 0; w < P.mix_nbw; ++w) {
            uint32_t v[RPT];
            load_slot<RPT>(st, rp, nc + w, t, v);
            const uint32_t pu = pbits[w], pl = pbits[P.mix_nbw + w];
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                if (KERNEL == 1) { cu[q] += __popc(v[q] ^ pu); cl[q] += __popc(v[q] ^ pl); }
                else { cu[q] += __popc(v[q] & pu); cl[q] += __popc(v[q] & pl); }
            }
        }
#pragma unroll
        for (int q = 0; q < RPT; ++q) { du[q] = add_ones(du[q], cu[q]); dl[q] = add_ones(dl[q], cl[q]); }
        return;
    }
    int ci = 0, bb = 0;
    for (int sg = 0; sg < P.mix_nseg; ++sg) {
        const int len = P.mix_seg[sg];
        if (len > 0) {
#pragma unroll 2
            for (int i = ci; i < ci + len; ++i) {
                uint32_t v[RPT];
                load_slot<RPT>(st, rp, i, t, v);
                const double2 pv = pivm[i];
#pragma unroll
                for (int q = 0; q < RPT; ++q) {
                    const double x = (double)__uint_as_float(v[q]);
                    if (KERNEL == 1) {
                        double e = x - pv.x; du[q] = fma(e, e, du[q]);
                        e = x - pv.y; dl[q] = fma(e, e, dl[q]);
                    } else {
                        du[q] = fma(x, pv.x, du[q]); dl[q] = fma(x, pv.y, dl[q]);
                    }
                }
            }
            ci += len;
        } else {
            const int nb = -len;
            int cu[RPT], cl[RPT];
#pragma unroll
            for (int q = 0; q < RPT; ++q) { cu[q] = 0; cl[q] = 0; }
            for (int w = bb >> 5; w <= (bb + nb - 1) >> 5; ++w) {
                const int lo = max(bb, 32 * w) - 32 * w, hi = min(bb + nb, 32 * w + 32) - 32 * w;
                const uint32_t m = (hi - lo == 32) ? 0xffffffffu : (((1u << (hi - lo)) - 1u) << lo);
                uint32_t v[RPT];
                load_slot<RPT>(st, rp, P.mix_nc + w, t, v);
                const uint32_t pu = pbits[w], pl = pbits[P.mix_nbw + w];
#pragma unroll
                for (int q = 0; q < RPT; ++q) {
                    if (KERNEL == 1) { cu[q] += __popc((v[q] ^ pu) & m); cl[q] += __popc((v[q] ^ pl) & m); }
                    else { cu[q] += __popc(v[q] & pu & m); cl[q] += __popc(v[q] & pl & m); }
                }
            }
#pragma unroll
            for (int q = 0; q < RPT; ++q) { du[q] = add_ones(du[q], cu[q]); dl[q] = add_ones(dl[q], cl[q]); }
            bb += nb;
        }
    }
}

// Mixed compact rows: the pivots' own sums from their compact forms (pivm: continuous
// pairs (x_u, x_l), pbits: x_u's bit words then x_l's), run by run in the original column
// order -- the R13 recurrence, a binary run adding 1.0 popcount times (add_ones), exactly
// as mixed_rows does for a row.  RBF: D(x_u, x_l); linear: x_u.x_u, x_l.x_l, x_u.x_l.
__device__ __forceinline__ void mixed_pivot_sums(const Params& P, const double2* pivm, const uint32_t* pbits,
                                                 int kernel, double& d_ul, double& s_uu, double& s_ll, double& s_ul) {
    int ci = 0, bb = 0;
    d_ul = 0.0; s_uu = 0.0; s_ll = 0.0; s_ul = 0.0;
    for (int sg = 0; sg < P.mix_nseg; ++sg) {
        const int len = P.mix_seg[sg];
        if (len > 0) {
#pragma unroll 4
            for (int i = ci; i < ci + len; ++i) {
                const double2 pv = pivm[i];
                if (kernel == 1) { const double e = pv.x - pv.y; d_ul = fma(e, e, d_ul); }
                else { s_uu = fma(pv.x, pv.x, s_uu); s_ll = fma(pv.y, pv.y, s_ll); s_ul = fma(pv.x, pv.y, s_ul); }
            }
            ci += len;
        } else {
            const int nb = -len;
            int cx = 0, cuu = 0, cll = 0, cul = 0;
            for (int w = bb >> 5; w <= (bb + nb - 1) >> 5; ++w) {
                const int lo = max(bb, 32 * w) - 32 * w, hi = min(bb + nb, 32 * w + 32) - 32 * w;
                const uint32_t m = (hi - lo == 32) ? 0xffffffffu : (((1u << (hi - lo)) - 1u) << lo);
                const uint32_t pu = pbits[w] & m, pl = pbits[P.mix_nbw + w] & m;
                cx += __popc(pu ^ pl); cuu += __popc(pu); cll += __popc(pl); cul += __popc(pu & pl);
            }
            if (kernel == 1) d_ul = add_ones(d_ul, cx);
            else { s_uu = add_ones(s_uu, cuu); s_ll = add_ones(s_ll, cll); s_ul = add_ones(s_ul, cul); }
            bb += nb;
        }
    }
}

// Dictionary-coded rows (Params::dict_n): the R13 recurrence of RPT rows over the kc
// features of one stage [kc][rp] of byte codes; values from the fp64 dictionary.
template <int KERNEL, int RPT>
__device__ __forceinline__ void dict_rows(int kc, const unsigned char* stb, int rp, int t,
                                          const double2* pv0, const double* dict,
                                          double (&du)[RPT], double (&dl)[RPT]) {
#pragma unroll 4
    for (int kk = 0; kk < kc; ++kk) {
        uint32_t w;
        if (RPT == 4) w = reinterpret_cast<const uint32_t*>(stb + (size_t)kk * rp)[t];
        else if (RPT == 2) w = reinterpret_cast<const uint16_t*>(stb + (size_t)kk * rp)[t];
        else w = stb[(size_t)kk * rp + t];
        const double2 pv = pv0[kk];
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const double x = dict[(w >> (8 * q)) & 0xffu];
            if (KERNEL == 1) {
                double e = x - pv.x; du[q] = fma(e, e, du[q]);
                e = x - pv.y; dl[q] = fma(e, e, dl[q]);
            } else {
                du[q] = fma(x, pv.x, du[q]); dl[q] = fma(x, pv.y, dl[q]);
            }
        }
    }
}

// BINCL: the kernel specialised for binary rows resident in a thread-block cluster (the
// latency-bound small-problem path): the other modes compile out, so the per-iteration code
// is short (instruction-cache resident).
// WIDE: the consumer warps poll the exchange records (several GPUs: > 320 records; a
// separate instantiation, since its registers slow the single-GPU kernels)
// SPEC: 0 every mode; 1 mixed compact rows only, 2 dense streamed fp32 rows only (no cluster
// exchange, Gram, row cache, binary, dictionary or other row format compiled in), 3
// dictionary rows with or without the row cache -- the W4, W5 and W3 kernels, whose row
// passes pay for the registers of modes they never take
template <int KERNEL, int RPT, bool A_SMEM, bool BINCL, int NTC = NT, bool WSS2 = false, bool WIDE = false,
          int SPEC = 0>
__global__ void __launch_bounds__(NTC + 64, 1) smo_persistent(const Params P) {
    // NTC consumer threads (8 or 16 warps), then the scalar and the producer warp
    constexpr int NT_ = NTC, NWC_ = NTC / 32, SCALAR_ = NWC_, PRODUCER_ = NWC_ + 1;
    constexpr int NTHREADS_ = NTC + 64, NSYNC_ = NTC + 32;
    static_assert(NWC_ <= 16, "at most 16 consumer warps");
    // mode switches: compile-time constants in the BINCL specialisation
    const bool m_cluster = BINCL || (SPEC == 0 && P.cluster != 0);
    // (the 16-warp instantiations never hold binary-resident rows or a row cache: the plan
    // takes 8 warps for those, and compiling them out spares the row pass registers)
    const bool m_isbin = BINCL || (SPEC == 0 && NTC == NT && P.bin_words > 0);
    const double* const m_gram = (BINCL || SPEC != 0) ? nullptr : P.gram;
    const int m_cache = (BINCL || NTC != NT || SPEC == 1 || SPEC == 2) ? 0 : P.cache_slots;
    const bool m_resident = BINCL || P.resident != 0;
    constexpr bool m_wss2 = WSS2 && !BINCL;                 // second-order working set (NEXT-2):
                                                            // its own instantiations, so the
                                                            // first-order kernels carry no gain pass
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Shared& sh = *reinterpret_cast<Shared*>(smem_raw);
    size_t off = (sizeof(Shared) + 127) & ~size_t(127);
    // pivots interleaved: piv[k] = (x_up[k], x_low[k]) -> one 16-byte broadcast load per k
    double2* piv = reinterpret_cast<double2*>(smem_raw + off); off += (size_t)P.dp * 16;
    // mixed rows: the pivots in the compact form (continuous pairs, then the bit words of
    // x_up and of x_low)
    const bool m_mixed = SPEC == 1 || (SPEC == 0 && !BINCL && P.mix_nseg > 0);
    double2* pivm = reinterpret_cast<double2*>(smem_raw + off);
    if (m_mixed) off += (size_t)P.mix_nc * 16;
    uint32_t* pbits = reinterpret_cast<uint32_t*>(smem_raw + off);
    if (m_mixed) off += (((size_t)2 * P.mix_nbw * 4) + 15) & ~size_t(15);
    // dictionary-coded rows: the values of the codes (fp64) and the element size of xblk
    const bool m_dict = SPEC == 3 || (!BINCL && SPEC == 0 && P.dict_n > 0);
    const int esz = m_dict ? 1 : 4;
    double* dict_s = reinterpret_cast<double*>(smem_raw + off);
    if (m_dict) off += 256 * 8;
    double* f_s = reinterpret_cast<double*>(smem_raw + off); off += (size_t)P.state_cap * 8;
    double* a_s = reinterpret_cast<double*>(smem_raw + off); if (A_SMEM) off += (size_t)P.state_cap * 8;
    uint8_t* fl_s = smem_raw + off; off += (size_t)P.state_cap;
    off = (off + 7) & ~size_t(7);
    // binary RBF: K for every possible Hamming distance, K_tab[D] = exp_cr(-(gamma D))
    double* ktab = reinterpret_cast<double*>(smem_raw + off);
    if (m_isbin) off += (size_t)(32 * P.bin_words + 1) * 8;
    off = (off + 7) & ~size_t(7);
    // row-cache directory: owner (global row) of every slot + an open-addressing hash
    // row -> slot (cache_hash entries, a power of two >= 2 slots), LRU replacement through a
    // doubly linked recency list of the slots (lru_prev / lru_next)
    int* dir_owner = reinterpret_cast<int*>(smem_raw + off); off += (size_t)m_cache * 4;
    int* lru_prev = reinterpret_cast<int*>(smem_raw + off); off += (size_t)m_cache * 4;
    int* lru_next = reinterpret_cast<int*>(smem_raw + off); off += (size_t)m_cache * 4;
    off = (off + 7) & ~size_t(7);
    int2* dir_hash = reinterpret_cast<int2*>(smem_raw + off); off += (size_t)P.cache_hash * 8;
    // cache mode: the scalar warp compacts the k with a non-zero term of K(x_u, x_l) here
    off = (off + 15) & ~size_t(15);
    double2* kul_t = reinterpret_cast<double2*>(smem_raw + off);
    if (m_cache > 0) off += (size_t)P.dp * 16;
    // cluster mode: records of the rank's CTAs, cmb[parity][cta][crw] (written remotely)
    uint4* cmb = reinterpret_cast<uint4*>(smem_raw + off);
    if (m_cluster) off += (size_t)2 * P.ctas_per_rank * P.crw * 16;
    off = (off + 127) & ~size_t(127);
    float* ring = reinterpret_cast<float*>(smem_raw + off);
    unsigned char* ring_b = smem_raw + off;
    const int stage_floats = P.kc * P.rt;                    // elements per stage
    uint64_t* full = reinterpret_cast<uint64_t*>(sh.bars);
    uint64_t* empty = full + MAX_STAGES;

    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const int rank = P.rank_base + blockIdx.x / P.ctas_per_rank;
    const int cta = blockIdx.x % P.ctas_per_rank;
    const int n_r = P.n_rows[rank];
    const int r0 = (int)(((long long)n_r * cta) / P.ctas_per_rank);
    const int r1 = (int)(((long long)n_r * (cta + 1)) / P.ctas_per_rank);
    const int R = r1 - r0;                                   // rows owned by this CTA
    const long long gbase = P.row_off[rank] + r0;            // global index of local row 0
    const int n_tiles = (R + P.rt - 1) / P.rt;
    const int rt_log2 = __ffs(P.rt) - 1;                     // rt = 256 RPT: a power of two
    const unsigned char* xcta_b = reinterpret_cast<const unsigned char*>(P.xblk[rank]) + (long long)cta * P.cta_stride * esz;
    double* alpha_g = P.alpha[rank] + r0;                    // this CTA's alpha (global)
    const double C = P.C;

    if (t == 0) {
        sh.stop = 0; sh.producer_done = 0; sh.issued = 0; sh.timeout = 0;
        for (int s = 0; s < P.stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NWC_); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int e = t; e < svmexp::EXP_TABLE_DOUBLES; e += NTHREADS_) sh.exp_tab[e] = svmexp::table_entry(e);
    for (int e = t; e < m_cache; e += NTHREADS_) {
        dir_owner[e] = -1;
        lru_prev[e] = e - 1;
        lru_next[e] = e + 1 < m_cache ? e + 1 : -1;
    }
    if (m_dict) for (int e = t; e < 256; e += NTHREADS_) dict_s[e] = e < P.dict_n ? P.dict[e] : 0.0;
    for (int e = t; e < P.cache_hash; e += NTHREADS_) dir_hash[e] = make_int2(-1, -1);
    if (m_cluster)
        for (int e = t; e < 2 * P.ctas_per_rank * P.crw; e += NTHREADS_) cmb[e] = make_uint4(0u, 0u, 0u, 0u);
    if (t == 0) { sh.lru_head = 0; sh.lru_tail = m_cache - 1; }
    for (int j = t; j < R; j += NTHREADS_) {
        f_s[j] = P.f[rank][r0 + j];
        if (A_SMEM) a_s[j] = alpha_g[j];
        fl_s[j] = P.flags[rank][r0 + j];
    }
    __syncthreads();
    const svmexp::PtrTab tab{sh.exp_tab};
    if (KERNEL == 1 && m_isbin) {
        for (int e = t; e <= 32 * P.bin_words; e += NTHREADS_) ktab[e] = svmexp::exp_cr_t(-(P.gamma * (double)e), tab);
        __syncthreads();
    }

    // every CTA of the cluster has zeroed its mailbox before any record is stored into it
    if (m_cluster) cluster_sync_all();

    // ============================================================ producer warp
    if (warp == PRODUCER_) {
        // (cluster mode: the producer waits in the final cluster barrier, so no CTA exits
        // while a peer may still address its shared memory)
        if (m_gram) {
            if (lane == 0) { sh.issued = 0; __threadfence_block(); sh.producer_done = 1; }
            if (m_cluster) cluster_sync_all();
            return;
        }
        if (m_resident) {
            if (lane == 0 && n_tiles > 0) {
                const int rp = (R + 3) & ~3;
                const uint32_t bytes = m_isbin ? (uint32_t)(n_tiles * ((P.bin_words + 3) & ~3) * P.rt * 4)
                                                   : (uint32_t)P.d_pad * rp * (uint32_t)esz;
                mbar_arrive_tx(&full[0], bytes);
                bulk_g2s(ring, xcta_b, bytes, &full[0]);
            }
            if (lane == 0) { sh.issued = 0; __threadfence_block(); sh.producer_done = 1; }
            if (m_cluster) cluster_sync_all();
            return;
        }
        if (lane == 0 && n_tiles > 0) {
            unsigned int s = 0, slot = 0, par = 0;
            bool wrapped = false;
            const uint64_t pol_keep = l2_policy(true), pol_stream = l2_policy(false);
            int tile = 0, chunk = 0;
            // L2 prefetch cursor: l2_prefetch stages beyond the copy cursor plus the ring
            const int pf_ahead = P.l2_prefetch > 0 ? P.l2_prefetch + P.stages : 0;
            int ptile = 0, pchunk = 0;
            for (int q = 0; q < pf_ahead; ++q) {
                if (++pchunk == P.n_chunks) { pchunk = 0; if (++ptile == n_tiles) ptile = 0; }
            }
            for (;;) {
                if (wrapped) {
                    while (!mbar_try_wait_sleep(&empty[slot], par ^ 1u, 2000u)) {
                        if (sh.stop) break;
                    }
                }
                if (sh.stop) break;
                const int rows_t = min(P.rt, R - tile * P.rt);
                const int rp = (rows_t + 3) & ~3;
                const uint32_t bytes = (uint32_t)P.kc * rp * (uint32_t)esz;
                const unsigned char* src = xcta_b + ((long long)tile * P.d_pad * P.rt + (long long)chunk * P.kc * rp) * esz;
                unsigned char* dst = ring_b + (size_t)slot * stage_floats * esz;
                mbar_arrive_tx(&full[slot], bytes);
                if (P.l2_keep_chunks > 0)
                    bulk_g2s_hint(dst, src, bytes, &full[slot],
                                  tile * P.n_chunks + chunk < P.l2_keep_chunks ? pol_keep : pol_stream);
                else
                    bulk_g2s(dst, src, bytes, &full[slot]);
                if (pf_ahead > 0) {
                    const int prows = min(P.rt, R - ptile * P.rt);
                    const int prp = (prows + 3) & ~3;
                    const unsigned char* psrc = xcta_b + ((long long)ptile * P.d_pad * P.rt + (long long)pchunk * P.kc * prp) * esz;
                    bulk_prefetch_l2(psrc, (uint32_t)P.kc * prp * (uint32_t)esz);
                    if (++pchunk == P.n_chunks) { pchunk = 0; if (++ptile == n_tiles) ptile = 0; }
                }
                ++s;
                sh.issued = s;
                if (++slot == (unsigned)P.stages) { slot = 0; par ^= 1u; wrapped = true; }
                if (++chunk == P.n_chunks) { chunk = 0; if (++tile == n_tiles) tile = 0; }
            }
        }
        if (lane == 0) { __threadfence_block(); sh.producer_done = 1; }
        __syncwarp();
        if (m_cluster) cluster_sync_all();
        return;
    }

    const bool is_scalar = (warp == SCALAR_);
    const bool timing = P.timers != nullptr && blockIdx.x == 0 && (t == 0 || (is_scalar && lane == 0));
    const int ph_row = is_scalar ? 1 : 0;
    if (timing) {
        for (int k = 0; k < PH_N; ++k) sh.ph_acc[ph_row][k] = 0;
        sh.ph_t[ph_row] = clock64();
    }
    int final_state = ST_RUNNING;
    Ctl* ctl = P.ctl[rank];
    Mailbox* my_mb = P.mbox[rank];
    const int xworld = P.independent ? 1 : P.world;         // ranks that exchange records
    const int xbase = P.independent ? rank : 0;             // first of them
    const float* xr = P.independent ? P.xr_rank[rank] : P.xr;
    const long long max_iter = P.independent ? P.max_iter_rank[rank] : P.max_iter;
    long long it = ctl->it;                 // written only at kernel end by CTA 0
    long long seq = ctl->seq;
    const long long it_start = it;
    unsigned int cslot = 0, cpar = 0, consumed = 0;
    long long c_hits = 0, c_misses = 0;     // row-cache lookups (scalar lane 0)
    // wss 2 (scalar warp): wphase 0 = the exchange carries first-order candidates (then
    // the gain pass of u follows), 1 = it carries gain candidates (then the update pass);
    // u's index, f, alpha and label are kept from phase 0 for the update
    int wphase = 0, sv_u = 0, sv_l = 0, sv_yu = 0;
    double sv_fu = 0.0, sv_au = 0.0;
    const double INF = __longlong_as_double(0x7ff0000000000000ll);

    if (m_resident && !m_gram && n_tiles > 0 && !is_scalar) mbar_wait(&full[0], 0);
    // ---- initial selection from the current state (no update)
    if (!is_scalar) {
        double fu = INF, fl = -INF;
        int ju = INT_MAX, jl = INT_MAX;
        for (int j = t; j < R; j += NT_) {
            const uint8_t g = fl_s[j];
            const double fj = f_s[j];
            if ((g & FL_UP) && better_up(fj, j, fu, ju)) { fu = fj; ju = j; }
            if ((g & FL_LOW) && better_low(fj, j, fl, jl)) { fl = fj; jl = j; }
        }
        warp_reduce_fi<true>(fu, ju);
        warp_reduce_fi<false>(fl, jl);
        if (lane == 0) {
            sh.red_f[0][warp] = fu; sh.red_i[0][warp] = ju;
            sh.red_f[1][warp] = fl; sh.red_i[1][warp] = jl;
            if (!A_SMEM) {
                sh.red_a[0][warp] = ju == INT_MAX ? 0.0 : alpha_g[ju];
                sh.red_a[1][warp] = jl == INT_MAX ? 0.0 : alpha_g[jl];
            }
        }
    }

    for (;;) {
        named_sync<NSYNC_>(BAR_C);                  // consumer candidates are in sh.red_*
        SVM_PHASE(timing, is_scalar ? PH_S_WAITC : PH_C_REDUCE);
        ++seq;
        if (!is_scalar) {
            // consumers: the scalar warp runs the exchange, the selection, the stopping test,
            // the row-cache directory and the pivot gather, then releases barrier A
            if constexpr (WIDE) {
                // wide poll: the consumers poll the records (the scalar warp publishes this
                // CTA's record meanwhile), each warp hands its best up / low candidate over
                const int g_total = xworld * P.ctas_per_rank * P.xch_dup;
                const int par = (int)(seq & 1);
                Sel b;
                const bool to = poll_slice<4>(mbox_words(my_mb, par, 0, g_total), mbox_words(my_mb, par, 1, g_total),
                                              g_total, (uint32_t)seq & 0xffffu, P.sys_scope, P.timeout_ns, t, NTC, b);
                unsigned long long kwu, kwl;
                unsigned iwu, iwl;
                argmin_redux(0xffffffffu, b.iu == INT_MAX ? ~0ull : fkey(b.fu), b.iu == INT_MAX ? 0xffffffffu : (unsigned)b.iu,
                             kwu, iwu);
                argmin_redux(0xffffffffu, b.il == INT_MAX ? ~0ull : ~fkey(b.fl), b.il == INT_MAX ? 0xffffffffu : (unsigned)b.il,
                             kwl, iwl);
                const unsigned mu = __ballot_sync(0xffffffffu, b.iu != INT_MAX && (unsigned)b.iu == iwu);
                const unsigned ml = __ballot_sync(0xffffffffu, b.il != INT_MAX && (unsigned)b.il == iwl);
                const int gu = __shfl_sync(0xffffffffu, b.gu, mu ? __ffs(mu) - 1 : 0);
                const int gl = __shfl_sync(0xffffffffu, b.gl, ml ? __ffs(ml) - 1 : 0);
                const bool any_to = __any_sync(0xffffffffu, to);
                if (lane == 0) {
                    sh.wp_i[0][warp] = iwu == 0xffffffffu ? INT_MAX : (int)iwu;
                    sh.wp_f[0][warp] = iwu == 0xffffffffu ? INF : fkey_inv(kwu);
                    sh.wp_g[0][warp] = gu;
                    sh.wp_i[1][warp] = iwl == 0xffffffffu ? INT_MAX : (int)iwl;
                    sh.wp_f[1][warp] = iwl == 0xffffffffu ? -INF : fkey_inv(~kwl);
                    sh.wp_g[1][warp] = gl;
                    if (any_to) sh.timeout = 1;
                }
                named_sync<NSYNC_>(BAR_E);
            }
            named_sync<NSYNC_>(BAR_A);
            SVM_PHASE(timing, PH_C_EXCH);
            const int dec = sh.decision;
            if (dec != ST_RUNNING) { final_state = dec; break; }
        } else {
            // ---- exchange seq (a6).  The scalar warp stores this CTA's record (four 16-byte
            // words, each carrying the sequence number and a checksum of its payload) into
            // every rank's mailbox -- peer pointers when the ranks are GPUs -- and polls all
            // g_total records of its own mailbox, every lane keeping up to PB loads in flight.
            // No fences or counters: a record word whose sequence number and checksum match
            // is complete.  Measured against counter- and tree-based exchanges in
            // tools/xch2_bench.cu.
            const int g_total = xworld * P.ctas_per_rank * P.xch_dup;
            const int par = (int)(seq & 1);
            const uint32_t sq = (uint32_t)seq & 0xffffu;
            double fu, fl;
            int iu, il, rec_u, rec_l;
            bool tmo;
            if (m_cluster) {
                // ======== cluster exchange (distributed shared memory).  The two selections
                // run side by side: lanes 0-15 handle I_up, lanes 16-31 I_low.
                const bool lowh = lane >= 16;
                const int hl = lane & 15;
                const int G = P.ctas_per_rank, RW = P.crw, rw = (P.crow + 2) / 3;
                // CTA candidate: reduce the 8 consumer-warp candidates of this half
                // (low half: max f = min of the complemented key)
                const unsigned hmask = lowh ? 0xffff0000u : 0x0000ffffu;
                unsigned long long kv = 0xffffffffffffffffull;
                unsigned jv = 0xffffffffu;
                if (hl < NWC_) {
                    const unsigned long long k = fkey(sh.red_f[lowh ? 1 : 0][hl]);
                    kv = lowh ? ~k : k;
                    jv = (unsigned)sh.red_i[lowh ? 1 : 0][hl];
                }
                unsigned long long kmin;
                unsigned jmin;
                argmin_redux(hmask, kv, jv, kmin, jmin);
                const unsigned long long ku_ = __shfl_sync(0xffffffffu, kmin, 0), kl_ = __shfl_sync(0xffffffffu, kmin, 16);
                const int ju = (int)__shfl_sync(0xffffffffu, jmin, 0), jl = (int)__shfl_sync(0xffffffffu, jmin, 16);
                const double c_fu = ju == INT_MAX ? INF : fkey_inv(ku_);
                const double c_fl = jl == INT_MAX ? -INF : fkey_inv(~kl_);
                SVM_PHASE(timing, PH_S_CAND);
                // lanes h and 16 + h (h < RW) build word h of the record (branch-free)
                if (hl < RW) {
                    uint32_t a;
                    unsigned long long v;
                    if (hl < 4) {
                        const int jj = (hl == 0 || hl == 2) ? ju : jl;
                        const bool empty = jj == INT_MAX;
                        const int jc = empty ? 0 : jj;
                        const double av = A_SMEM ? a_s[jc] : alpha_g[jc];
                        if (hl == 0) { a = empty ? 0xffffffffu : (uint32_t)(gbase + ju); v = __double_as_longlong(c_fu); }
                        else if (hl == 1) { a = empty ? 0xffffffffu : (uint32_t)(gbase + jl); v = __double_as_longlong(c_fl); }
                        else if (hl == 2) {
                            const int yu_ = ju == INT_MAX ? 0 : ((fl_s[ju] & FL_POS) ? 1 : -1);
                            const int yl_ = jl == INT_MAX ? 0 : ((fl_s[jl] & FL_POS) ? 1 : -1);
                            a = (uint32_t)((yu_ & 0xffff) | (yl_ << 16));
                            v = __double_as_longlong(empty ? 0.0 : av);
                        } else { a = 0u; v = __double_as_longlong(empty ? 0.0 : av); }
                    } else {
                        const bool is_u = (hl - 4) < rw;
                        const int k0 = 3 * ((hl - 4) - (is_u ? 0 : rw));
                        const int jr = is_u ? ju : jl;
                        uint32_t e[3] = {0u, 0u, 0u};
                        if (jr != INT_MAX) {
#pragma unroll
                            for (int m = 0; m < 3; ++m)
                                if (k0 + m < P.crow) e[m] = m_isbin ? bin_row_word(ring, jr, k0 + m, P.bin_words)
                                                                        : __float_as_uint(ring[(size_t)(k0 + m) * ((R + 3) & ~3) + jr]);
                        }
                        a = e[0];
                        v = (unsigned long long)e[1] | ((unsigned long long)e[2] << 32);
                    }
                    const uint4 wv = rec_pack(sq, a, v);
                    if (lane == 0) SVM_PHASE(timing, PH_S_BUILD);
                    const uint32_t src = smem_u32(cmb + ((size_t)par * G + cta) * RW + hl);
                    const int half = (G + 1) >> 1;
                    const int j0 = lowh ? half : 0, j1 = lowh ? G : half;
                    for (int j = j0; j < j1; ++j) {
                        uint32_t ra;
                        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(src), "r"(j));
                        st_cluster_v4(ra, wv);
                    }
                }
                SVM_PHASE(timing, PH_S_PUBLISH);
                // lane hl < G polls word 0 (lanes 0-15) or word 1 (lanes 16-31) of CTA hl's record
                double pf = lowh ? -INF : INF;
                int pi = INT_MAX;
                bool to = false;
                if (hl < G) {
                    const uint4* r = cmb + ((size_t)par * G + hl) * RW + (lowh ? 1 : 0);
                    long long t0 = 0;
                    unsigned int spins = 0;
                    uint4 w;
                    for (;;) {
                        w = ld_volatile_shared_v4(r);
                        if (rec_ok(w, sq)) break;
                        if ((++spins & 255u) == 0) {
                            const long long now = globaltimer();
                            if (t0 == 0) t0 = now;
                            else if (now - t0 > P.timeout_ns) { to = true; break; }
                        }
                    }
                    pi = rec_idx(w);
                    if (pi != INT_MAX) pf = rec_f64(w);
                }
                tmo = __any_sync(0xffffffffu, to) || sh.timeout != 0;
                SVM_PHASE(timing, PH_S_POLL);
                {
                    const unsigned long long k0 = fkey(pf);
                    const unsigned long long kk = lowh ? ~k0 : k0;
                    unsigned long long kw;
                    unsigned iw;
                    argmin_redux(hmask, kk, (unsigned)pi, kw, iw);
                    // the record each winner came from: the lane of its half holding it
                    const unsigned hit = __ballot_sync(0xffffffffu, (unsigned)pi == iw && kk == kw);
                    const unsigned hu = hit & 0xffffu, hlw = hit >> 16;
                    iu = (int)__shfl_sync(0xffffffffu, iw, 0);
                    il = (int)__shfl_sync(0xffffffffu, iw, 16);
                    const unsigned long long kwu = __shfl_sync(0xffffffffu, kw, 0), kwl = __shfl_sync(0xffffffffu, kw, 16);
                    fu = iu == INT_MAX ? INF : fkey_inv(kwu);
                    fl = il == INT_MAX ? -INF : fkey_inv(~kwl);
                    rec_u = hu ? __ffs(hu) - 1 : 0;
                    rec_l = hlw ? __ffs(hlw) - 1 : 0;
                }
            } else {
                Cand c;
                int ju, jl;                                   // this CTA's candidates (local rows)
                {
                    // the CTA candidate: lexicographic minimum / maximum of the consumer
                    // warps' candidates (local rows: lower local = lower global index)
                    const int wju = lane < NWC_ ? sh.red_i[0][lane] : INT_MAX;
                    const int wjl = lane < NWC_ ? sh.red_i[1][lane] : INT_MAX;
                    unsigned long long kwu, kwl;
                    unsigned iwu, iwl;
                    argmin_redux(0xffffffffu, wju == INT_MAX ? ~0ull : fkey(sh.red_f[0][min(lane, NWC_ - 1)]),
                                 wju == INT_MAX ? 0xffffffffu : (unsigned)wju, kwu, iwu);
                    argmin_redux(0xffffffffu, wjl == INT_MAX ? ~0ull : ~fkey(sh.red_f[1][min(lane, NWC_ - 1)]),
                                 wjl == INT_MAX ? 0xffffffffu : (unsigned)wjl, kwl, iwl);
                    ju = iwu == 0xffffffffu ? INT_MAX : (int)iwu;
                    jl = iwl == 0xffffffffu ? INT_MAX : (int)iwl;
                    const double fu = ju == INT_MAX ? INF : fkey_inv(kwu);
                    const double fl = jl == INT_MAX ? -INF : fkey_inv(~kwl);
                    c.fu = fu; c.fl = fl;
                    c.iu = (ju == INT_MAX) ? INT_MAX : (int)(gbase + ju);
                    c.il = (jl == INT_MAX) ? INT_MAX : (int)(gbase + jl);
                    if (A_SMEM) {
                        c.au = (ju == INT_MAX) ? 0.0 : a_s[ju];
                        c.al = (jl == INT_MAX) ? 0.0 : a_s[jl];
                    } else {
                        // the winning warps' alpha, read by them (local rows are unique)
                        const unsigned wu = __ballot_sync(0xffffffffu, lane < NWC_ && wju != INT_MAX && wju == ju);
                        const unsigned wl = __ballot_sync(0xffffffffu, lane < NWC_ && wjl != INT_MAX && wjl == jl);
                        c.au = (ju == INT_MAX || !wu) ? 0.0 : sh.red_a[0][__ffs(wu) - 1];
                        c.al = (jl == INT_MAX || !wl) ? 0.0 : sh.red_a[1][__ffs(wl) - 1];
                    }
                    c.yu = (ju == INT_MAX) ? 0 : ((fl_s[ju] & FL_POS) ? 1 : -1);
                    c.yl = (jl == INT_MAX) ? 0 : ((fl_s[jl] & FL_POS) ? 1 : -1);
                    if (m_wss2 && wphase == 1) {
                        // gain candidates: w1 = (t, gain), w2 = (y_t << 16, f_t), w3 = (0, alpha_t)
                        c.au = (jl == INT_MAX) ? 0.0 : f_s[jl];
                        c.yu = 0;
                    }
                }
                Sel best;
                const int gcta = (rank - xbase) * P.ctas_per_rank + cta;
                if (P.xch_dup == 1) {
                    if (lane < 4 * xworld)
                        rec_store(mbox_words(P.mbox[xbase + (lane >> 2)], par, lane & 3, g_total) + gcta,
                                  rec_word(c, lane & 3, sq), P.sys_scope);
                } else {
                    // (test hook) copy k of the record in slot gcta + k * xworld * ctas_per_rank
                    for (int e = lane; e < 4 * xworld * P.xch_dup; e += 32) {
                        const int rr = (e >> 2) % xworld, k = (e >> 2) / xworld;
                        rec_store(mbox_words(P.mbox[xbase + rr], par, e & 3, g_total) + gcta +
                                      k * xworld * P.ctas_per_rank,
                                  rec_word(c, e & 3, sq), P.sys_scope);
                    }
                }
                // warm L2 with this CTA's candidate rows: the two winners' rows are gathered
                // from the row-major replica right after the selection (the critical path)
                if (m_mixed && P.xcomp && m_cache == 0) {
                    const int ncw = P.mix_nc + P.mix_nbw;
                    if (lane < 2) {
                        const int jj = lane == 0 ? ju : jl;
                        if (jj != INT_MAX) asm volatile("prefetch.global.L2 [%0];" :: "l"(P.xcomp + (gbase + jj) * (long long)ncw));
                    }
                } else if (!m_gram && !m_isbin) {
                    const int span = P.d * 4;
                    const int lines = (span + 127) / 128 + 1;
                    for (int q = lane; q < 2 * lines; q += 32) {
                        const int jj = q < lines ? ju : jl;
                        if (jj != INT_MAX) {
                            const char* row = reinterpret_cast<const char*>(xr + (gbase + jj) * (long long)P.d);
                            const int o = min((q % lines) * 128, span - 1);
                            asm volatile("prefetch.global.L2 [%0];" :: "l"(row + o));
                        }
                    }
                }
                if (P.dbg_ts && lane == 0 && it < P.dbg_ts_n)
                    P.dbg_ts[3 * ((long long)it * P.ctas_per_rank * P.world + (long long)rank * P.ctas_per_rank + cta) + 1] =
                        (unsigned long long)globaltimer();
                SVM_PHASE(timing, PH_S_PUBLISH);
                constexpr int PB = 5;                            // records in flight per lane
                unsigned int rounds = 0;
                if constexpr (WIDE) {
                    // the consumer warps polled: lane w takes warp w's candidates
                    named_sync<NSYNC_>(BAR_E);
                    const bool has = lane < NWC_;
                    best.iu = has ? sh.wp_i[0][lane] : INT_MAX;
                    best.fu = has ? sh.wp_f[0][lane] : INF;
                    best.gu = has ? sh.wp_g[0][lane] : 0;
                    best.il = has ? sh.wp_i[1][lane] : INT_MAX;
                    best.fl = has ? sh.wp_f[1][lane] : -INF;
                    best.gl = has ? sh.wp_g[1][lane] : 0;
                    tmo = sh.timeout != 0;
                } else {
                    tmo = poll_records<PB>(mbox_words(my_mb, par, 0, g_total), mbox_words(my_mb, par, 1, g_total),
                                           g_total, sq, P.sys_scope, P.timeout_ns, lane, best, rounds) ||
                          sh.timeout != 0;
                }
                if (timing) sh.ph_acc[ph_row][PH_C_PIVOT] += rounds;     // (timers only) poll rounds of lane 0
                SVM_PHASE(timing, PH_S_POLL);
                // the warp's winners (lexicographic (f, index) minimum / maximum through three
                // redux.sync on the order-preserving key, R22) and the records they came from
                {
                    unsigned long long kwu, kwl;
                    unsigned iwu, iwl;
                    argmin_redux(0xffffffffu, best.iu == INT_MAX ? ~0ull : fkey(best.fu),
                                 best.iu == INT_MAX ? 0xffffffffu : (unsigned)best.iu, kwu, iwu);
                    argmin_redux(0xffffffffu, best.il == INT_MAX ? ~0ull : ~fkey(best.fl),
                                 best.il == INT_MAX ? 0xffffffffu : (unsigned)best.il, kwl, iwl);
                    iu = iwu == 0xffffffffu ? INT_MAX : (int)iwu;
                    il = iwl == 0xffffffffu ? INT_MAX : (int)iwl;
                    fu = iu == INT_MAX ? INF : fkey_inv(kwu);
                    fl = il == INT_MAX ? -INF : fkey_inv(~kwl);
                }
                const unsigned mu = __ballot_sync(0xffffffffu, best.iu == iu);
                const unsigned ml = __ballot_sync(0xffffffffu, best.il == il);
                rec_u = __shfl_sync(0xffffffffu, best.gu, mu ? __ffs(mu) - 1 : 0);
                rec_l = __shfl_sync(0xffffffffu, best.gl, ml ? __ffs(ml) - 1 : 0);
            }
            int dec = ST_RUNNING;
            const bool gainA = m_wss2 && wphase == 0;          // wss 2: the gain pass of u follows
            if (m_wss2 && wphase == 1) {
                // the second-order l (the stopping test was taken on the first-order pair);
                // some t always qualifies (the first-order l has f_l > f_u), else keep it
                if (tmo) dec = ST_TIMEOUT;
                if (il == INT_MAX) il = sv_l;
                iu = sv_u; fu = sv_fu;
            } else {
                if (tmo) dec = ST_TIMEOUT;
                else if (iu == INT_MAX || il == INT_MAX) dec = ST_CONVERGED;
                else if (fl - fu <= 2.0 * P.tol) dec = ST_CONVERGED;
                else if (it == max_iter) dec = ST_MAXITER;
                else if (P.iter_limit > 0 && it - it_start == P.iter_limit) dec = ST_LIMIT;
            }
            if (dec != ST_RUNNING) {
                final_state = dec;
                if (lane == 0) {
                    if (tmo) sh.timeout = 1;
                    sh.decision = dec; sh.u = iu; sh.l = il; sh.f_up = fu; sh.f_low = fl;
                }
                __syncwarp();
                named_arrive<NSYNC_>(BAR_A);
                break;
            }
            if (gainA) { sv_u = iu; sv_l = il; sv_fu = fu; il = iu; }   // the gain pass streams K(x_u, .) only
            // ---- row cache (a8): every CTA runs the same directory operations on the same
            // pair sequence (hash lookup, LRU replacement), so every CTA agrees
            int c_hit = 0, su = -1, sl = -1;
            double kul_pre = 0.0;                   // lane 0: K_ul read early from the row cache
            if (m_cache > 0) {
                if (lane == 0) {
                    const int hm = P.cache_hash - 1;
                    auto hslot = [&](int key) { return (int)(((unsigned)key * 2654435761u) >> 7) & hm; };
                    auto find = [&](int key) {
                        for (int h = hslot(key);; h = (h + 1) & hm) {
                            const int2 e = dir_hash[h];
                            if (e.x == key) return e.y;
                            if (e.x < 0) return -1;
                        }
                    };
                    auto insert = [&](int key, int slot) {
                        int h = hslot(key);
                        while (dir_hash[h].x >= 0) h = (h + 1) & hm;
                        dir_hash[h] = make_int2(key, slot);
                    };
                    auto erase = [&](int key) {                   // linear probing, backward shift
                        int h = hslot(key);
                        while (dir_hash[h].x != key) h = (h + 1) & hm;
                        int j = h;
                        for (;;) {
                            j = (j + 1) & hm;
                            const int2 e = dir_hash[j];
                            if (e.x < 0) break;
                            const int k = hslot(e.x);
                            // move e back to h if its home k is not cyclically in (h, j]
                            const bool in_range = (h <= j) ? (h < k && k <= j) : (h < k || k <= j);
                            if (!in_range) { dir_hash[h] = e; h = j; }
                        }
                        dir_hash[h] = make_int2(-1, -1);
                    };
                    // LRU: the recency list runs from lru_head (most recent) to lru_tail;
                    // a lookup moves its slot to the head, the victim is the tail (or the
                    // slot before it when the tail holds the other row of the pair)
                    auto touch = [&](int sl_) {
                        if (sh.lru_head == sl_) return;
                        const int pv = lru_prev[sl_], nx = lru_next[sl_];
                        lru_next[pv] = nx;                          // pv >= 0: sl_ is not the head
                        if (nx >= 0) lru_prev[nx] = pv; else sh.lru_tail = pv;
                        lru_prev[sl_] = -1; lru_next[sl_] = sh.lru_head;
                        lru_prev[sh.lru_head] = sl_; sh.lru_head = sl_;
                    };
                    auto victim = [&](int avoid) {
                        int v = sh.lru_tail;
                        if (v == avoid) v = lru_prev[v];
                        if (dir_owner[v] >= 0) erase(dir_owner[v]);
                        return v;
                    };
                    int fu_ = -1, fl_ = -1;
                    if (gainA) {
                        // wss 2 gain pass: only u's row (then cached for the update pass)
                        su = find(iu);
                        c_hits += su >= 0; c_misses += su < 0;
                        if (su < 0) { fu_ = victim(-1); dir_owner[fu_] = iu; insert(iu, fu_); }
                        touch(su >= 0 ? su : fu_);
                        sl = su;
                        c_hit = su >= 0 ? 1 : 0;
                    } else {
                    su = find(iu); sl = find(il);
                    c_hit = (su >= 0 && sl >= 0) ? 1 : 0;
                    c_hits += (su >= 0) + (sl >= 0);
                    c_misses += (su < 0) + (sl < 0);
                    if (su < 0) { fu_ = victim(sl); dir_owner[fu_] = iu; insert(iu, fu_); }
                    touch(su >= 0 ? su : fu_);
                    if (sl < 0) { fl_ = victim(su >= 0 ? su : fu_); dir_owner[fl_] = il; insert(il, fl_); }
                    touch(sl >= 0 ? sl : fl_);
                    }
                    sh.c_hit = c_hit; sh.c_su = su; sh.c_sl = sl; sh.c_fill_u = fu_; sh.c_fill_l = fl_;
                    // both rows cached: start the load of K_ul (column l of u's row) now, so its
                    // latency overlaps the winners' words and barrier A
                    if (c_hit && !gainA && kul_cache_ok(P, iu, il)) kul_pre = kcache_at(P, su, il);
                }
                c_hit = __shfl_sync(0xffffffffu, c_hit, 0);
                su = __shfl_sync(0xffffffffu, su, 0);
                sl = __shfl_sync(0xffffffffu, sl, 0);
            }
            SVM_PHASE(timing, PH_S_READ);
            // alpha and label of the two winners: words 2 / 3 of their records, in flight
            // while the pivot rows load (lane 0: w2 of u's record, 1: w2 of l's, 2: w3 of l's)
            // cluster mode: lane 0: word 2 of u's record, 1/2: words 2/3 of l's record,
            // 3.. 3+rw-1: u's row words, 3+rw .. 3+2rw-1: l's row words (validated: they may
            // trail the candidate words)
            const int rwc = (P.crow + 2) / 3;
            const uint4* wp;
            if (m_cluster) {
                int rr, hh;
                if (lane < 3) { rr = lane == 0 ? rec_u : rec_l; hh = lane == 2 ? 3 : 2; }
                else if (lane < 3 + rwc) { rr = rec_u; hh = 4 + (lane - 3); }
                else { rr = rec_l; hh = 4 + rwc + (lane - 3 - rwc); }
                wp = cmb + ((size_t)par * P.ctas_per_rank + rr) * P.crw + (hh < P.crw ? hh : 0);
            } else {
                wp = mbox_words(my_mb, par, lane == 2 ? 3 : 2, g_total) + (lane == 0 ? rec_u : rec_l);
            }
            uint4 wa = make_uint4(0u, 0u, 0u, 0u);
            if (m_cluster) {
                if (lane < 3 + (m_gram || c_hit ? 0 : 2 * rwc)) {
                    wa = ld_volatile_shared_v4(wp);
                    unsigned int spins = 0;
                    while (!rec_ok(wa, sq)) {
                        wa = ld_volatile_shared_v4(wp);
                        if (++spins > (1u << 24)) { sh.timeout = 1; break; }
                    }
                }
            } else if (lane < 3) {
                wa = rec_load(wp, P.sys_scope);
            }
            // ---- pivot rows x_up, x_low into shared memory (fp64, or bit rows)
            if (m_gram || c_hit) {
                // rows of K are read directly (Gram or cached rows; K_ul from the cached row
                // of u); no pivot rows needed
            } else if (m_cluster && P.crow) {
                // the winners' rows travelled in their records (lanes 3.. hold the words)
                const int nu = m_isbin ? P.bin_words : P.d;
                for (int k0 = 0; k0 < (m_isbin ? 32 : P.d_pad); k0 += 32) {
                    const int k = k0 + lane;
                    const int kk = k < nu ? k : 0;
                    const int src_u = 3 + kk / 3, src_l = 3 + rwc + kk / 3, m = kk % 3;
                    // a row word triple travels as (aux, payload lo, payload hi)
                    const uint32_t e0 = rec_aux(wa), e1 = rec_lo(wa), e2 = rec_hi(wa);
                    const uint32_t vu_y = __shfl_sync(0xffffffffu, e0, src_u), vu_z = __shfl_sync(0xffffffffu, e1, src_u),
                                   vu_w = __shfl_sync(0xffffffffu, e2, src_u);
                    const uint32_t vl_y = __shfl_sync(0xffffffffu, e0, src_l), vl_z = __shfl_sync(0xffffffffu, e1, src_l),
                                   vl_w = __shfl_sync(0xffffffffu, e2, src_l);
                    const uint32_t xu = m == 0 ? vu_y : (m == 1 ? vu_z : vu_w);
                    const uint32_t xl = m == 0 ? vl_y : (m == 1 ? vl_z : vl_w);
                    if (m_isbin) {
                        uint32_t* pw = reinterpret_cast<uint32_t*>(piv);
                        const int Wp = (P.bin_words + 3) & ~3;
                        if (k < Wp) { pw[k] = k < nu ? xu : 0u; pw[Wp + k] = k < nu ? xl : 0u; }
                    } else if (k < P.d_pad) {
                        piv[k] = k < nu ? make_double2((double)__uint_as_float(xu), (double)__uint_as_float(xl))
                                        : make_double2(0.0, 0.0);
                    }
                }
            } else if (m_isbin) {
                uint32_t* pw = reinterpret_cast<uint32_t*>(piv);
                const int Wp = (P.bin_words + 3) & ~3;
                if (lane < 2 * Wp) {
                    const int w = lane < Wp ? lane : lane - Wp;
                    pw[lane] = w < P.bin_words ? __ldg(&P.xrbits[(long long)(lane < Wp ? iu : il) * P.bin_words + w]) : 0u;
                }
            } else if (m_mixed && P.xcomp && m_cache == 0) {
                // compact pivots straight from the compact row-major copy: one load per word
                const int nc = P.mix_nc, ncw = nc + P.mix_nbw;
                for (int w0 = 0; w0 < ncw; w0 += 32) {
                    const int w = w0 + lane;
                    const uint32_t uw = w < ncw ? __ldg(&P.xcomp[(long long)iu * ncw + w]) : 0u;
                    const uint32_t lw = w < ncw ? __ldg(&P.xcomp[(long long)il * ncw + w]) : 0u;
                    if (w < nc) pivm[w] = make_double2((double)__uint_as_float(uw), (double)__uint_as_float(lw));
                    else if (w < ncw) { pbits[w - nc] = uw; pbits[P.mix_nbw + w - nc] = lw; }
                }
            } else {
                const float* xu_g = xr + (long long)iu * P.d;
                const float* xl_g = xr + (long long)il * P.d;
                for (int k0 = 0; k0 < P.dp; k0 += 32 * 8) {
                    float vu[8], vl[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int k = k0 + 32 * q + lane;
                        vu[q] = (k < P.d) ? __ldg(&xu_g[k]) : 0.0f;
                        vl[q] = (k < P.d) ? __ldg(&xl_g[k]) : 0.0f;
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int k = k0 + 32 * q + lane;
                        if (k < P.dp) piv[k] = make_double2((double)vu[q], (double)vl[q]);
                    }
                }
                if (m_mixed) {
                    // compact pivots: continuous columns in order, binary columns as bit words
                    __syncwarp();
                    for (int i = lane; i < P.mix_nc; i += 32) pivm[i] = piv[__ldg(&P.mix_map[i])];
                    const int nbin = P.d - P.mix_nc;
                    for (int w = 0; w < P.mix_nbw; ++w) {
                        const int b = 32 * w + lane;
                        const double2 pv = b < nbin ? piv[__ldg(&P.mix_map[P.mix_nc + b])] : make_double2(0.0, 0.0);
                        const unsigned mu = __ballot_sync(0xffffffffu, pv.x != 0.0);
                        const unsigned ml = __ballot_sync(0xffffffffu, pv.y != 0.0);
                        if (lane == 0) { pbits[w] = mu; pbits[P.mix_nbw + w] = ml; }
                    }
                }
            }
            if (lane == 0) { sh.decision = ST_RUNNING; sh.u = iu; sh.l = il; sh.pass = gainA ? 1 : 0; }
            __syncwarp();
            named_arrive<NSYNC_>(BAR_A);
            if (P.dbg_ts && lane == 0 && it < P.dbg_ts_n) {
                unsigned smid;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                unsigned long long* e = P.dbg_ts + 3 * ((long long)it * P.ctas_per_rank * P.world + (long long)rank * P.ctas_per_rank + cta);
                e[0] = (unsigned long long)globaltimer();
                e[2] = smid;
            }
            if (lane < 3 && !m_cluster) {
                unsigned int spins = 0;
                while (!rec_ok(wa, sq)) {            // written with w0/w1: (almost) never taken
                    wa = rec_load(wp, P.sys_scope);
                    if (++spins > (1u << 24)) { sh.timeout = 1; break; }
                }
            }
            const uint32_t wa_aux = rec_aux(wa);
            int yu = (int)(int16_t)(__shfl_sync(0xffffffffu, wa_aux, 0) & 0xffffu);
            double au = __hiloint2double((int)__shfl_sync(0xffffffffu, rec_hi(wa), 0), (int)__shfl_sync(0xffffffffu, rec_lo(wa), 0));
            const int yl = (int)(int16_t)(__shfl_sync(0xffffffffu, wa_aux, 1) >> 16);
            const double al = __hiloint2double((int)__shfl_sync(0xffffffffu, rec_hi(wa), 2), (int)__shfl_sync(0xffffffffu, rec_lo(wa), 2));
            if (m_wss2) {
                // phase 0: keep u's alpha and label for the update; phase 1: word 2 of l's gain
                // record carries f_l (the pair's gap is f_l - f_u, not the first-order gap)
                const double f_rec = __hiloint2double((int)__shfl_sync(0xffffffffu, rec_hi(wa), 1),
                                                      (int)__shfl_sync(0xffffffffu, rec_lo(wa), 1));
                if (gainA) { sv_au = au; sv_yu = yu; }
                else { au = sv_au; yu = sv_yu; fl = f_rec; }
            }
            SVM_PHASE(timing, PH_S_PIVOT);
            const int u = iu, l = il;
            if (m_cache > 0 && !c_hit && !gainA) {
                // compact the non-zero terms of K(x_u, x_l) (RBF: x_u - x_l; linear: pairs
                // with x_u or x_l non-zero) in ascending k
                int cnt = 0;
                for (int k0 = 0; k0 < P.d; k0 += 32) {
                    const int k = k0 + lane;
                    double2 pv = make_double2(0.0, 0.0);
                    bool nz = false;
                    if (k < P.d) {
                        pv = piv[k];
                        if (KERNEL == 1) { pv.x = pv.x - pv.y; nz = pv.x != 0.0; }
                        else nz = (pv.x != 0.0) || (pv.y != 0.0);
                    }
                    const unsigned m = __ballot_sync(0xffffffffu, nz);
                    if (nz) kul_t[cnt + __popc(m & ((1u << lane) - 1u))] = pv;
                    cnt += __popc(m);
                }
                if (lane == 0) sh.kul_cnt = cnt;
                __syncwarp();
            }
        // ---- pair update (a2): eta, clipped step, snapped alphas (lane 0)
            if (gainA) {
                // wss 2 gain pass: K(x_u, x_u) and f_u for the consumers' gains; no update
                if (lane == 0) {
                    sh.gain_kuu = KERNEL == 1 ? 1.0 : __ldg(&P.qself[u]);
                    sh.gain_fu = fu;
                    sh.cu = 0.0; sh.cl = 0.0;
                }
                __syncwarp();
                named_arrive<NSYNC_>(BAR_B);
                wphase = 1;
                continue;
            }
            if (m_wss2) wphase = 0;
            if (lane == 0) {
                double Kuu, Kll, Kul;
                if (m_gram) {
                    const long long n = P.n_global;
                    Kuu = __ldg(&m_gram[(long long)u * n + u]);
                    Kll = __ldg(&m_gram[(long long)l * n + l]);
                    Kul = __ldg(&m_gram[(long long)u * n + l]);
                } else if (m_isbin) {
                    const uint32_t* pw = reinterpret_cast<const uint32_t*>(piv);
                    int cuu = 0, cll = 0, cul = 0, cx = 0;
                    const int Wp = (P.bin_words + 3) & ~3;
                    for (int w = 0; w < P.bin_words; ++w) {
                        const uint32_t a = pw[w], bb = pw[Wp + w];
                        cuu += __popc(a); cll += __popc(bb); cul += __popc(a & bb); cx += __popc(a ^ bb);
                    }
                    if (KERNEL == 1) {
                        Kuu = 1.0; Kll = 1.0;
                        Kul = (u == l) ? 1.0 : ktab[cx];
                    } else {
                        Kuu = (double)cuu; Kll = (double)cll; Kul = (double)cul;
                    }
                } else if (c_hit && kul_cache_ok(P, u, l)) {
                    // both rows cached: K_ul is column l of the cached row of u (computed by
                    // l's owner CTA with the row-pass arithmetic, made visible by its fence);
                    // K(x, x) is column u of u's row / column l of l's row
                    Kul = kul_pre;
                    if (KERNEL == 1) { Kuu = 1.0; Kll = 1.0; }
                    else { Kuu = kcache_at(P, su, u); Kll = kcache_at(P, sl, l); }
                } else if (m_cache > 0) {
                    // only k with a non-zero term change the sums (fma(0, x, acc) == acc), so
                    // the serial chains run over the compacted non-zero terms (ascending k)
                    const int cnt = sh.kul_cnt;
                    if (KERNEL == 1) {
                        double acc = 0.0;
                        for (int i = 0; i < cnt; ++i) { const double dv = kul_t[i].x; acc = fma(dv, dv, acc); }
                        Kuu = 1.0; Kll = 1.0;
                        Kul = (u == l) ? 1.0 : svmexp::exp_cr_t(-(P.gamma * acc), tab);
                    } else {
                        double s_uu = 0.0, s_ll = 0.0, s_ul = 0.0;
                        for (int i = 0; i < cnt; ++i) {
                            const double2 pv = kul_t[i];
                            s_uu = fma(pv.x, pv.x, s_uu); s_ll = fma(pv.y, pv.y, s_ll); s_ul = fma(pv.x, pv.y, s_ul);
                        }
                        Kuu = s_uu; Kll = s_ll; Kul = s_ul;
                    }
                } else if (m_mixed && P.xcomp) {
                    // (the pivots were gathered compact: the same sums from their compact forms)
                    double d_ul, s_uu, s_ll, s_ul;
                    mixed_pivot_sums(P, pivm, pbits, KERNEL, d_ul, s_uu, s_ll, s_ul);
                    if (KERNEL == 1) {
                        Kuu = 1.0; Kll = 1.0;
                        Kul = (u == l) ? 1.0 : svmexp::exp_cr_t(-(P.gamma * d_ul), tab);
                    } else {
                        Kuu = s_uu; Kll = s_ll; Kul = s_ul;
                    }
                } else if (KERNEL == 1) {
                    double acc = 0.0;
#pragma unroll 8
                    for (int k = 0; k < P.d; ++k) { const double2 pv = piv[k]; const double dv = pv.x - pv.y; acc = fma(dv, dv, acc); }
                    Kuu = 1.0; Kll = 1.0;
                    Kul = (u == l) ? 1.0 : svmexp::exp_cr_t(-(P.gamma * acc), tab);
                } else {
                    double s_uu = 0.0, s_ll = 0.0, s_ul = 0.0;
#pragma unroll 8
                    for (int k = 0; k < P.d; ++k) {
                        const double2 pv = piv[k];
                        s_uu = fma(pv.x, pv.x, s_uu);
                        s_ll = fma(pv.y, pv.y, s_ll);
                        s_ul = fma(pv.x, pv.y, s_ul);
                    }
                    Kuu = s_uu; Kll = s_ll; Kul = s_ul;
                }
                const double eta = Kuu + Kll - 2.0 * Kul;
                const double gap = fl - fu;
                const double yu_d = (double)yu, yl_d = (double)yl;
                const double tu = (yu == 1) ? C - au : au;
                const double tl = (yl == 1) ? al : C - al;
                double tt = gap / (eta > 1e-12 ? eta : 1e-12);
                if (tu < tt) tt = tu;
                if (tl < tt) tt = tl;
                const double au2 = (tt == tu) ? (yu == 1 ? C : 0.0) : au + yu_d * tt;
                const double al2 = (tt == tl) ? (yl == 1 ? 0.0 : C) : al - yl_d * tt;
                sh.cu = yu_d * (au2 - au);
                sh.cl = yl_d * (al2 - al);
                // owner CTA: alpha and flags of the two rows
                const long long lu = (long long)u - gbase, ll = (long long)l - gbase;
                if (lu >= 0 && lu < R) {
                    if (A_SMEM) a_s[lu] = au2; else alpha_g[lu] = au2;
                    fl_s[lu] = flags_of(yu, au2, C);
                }
                if (ll >= 0 && ll < R) {
                    if (A_SMEM) a_s[ll] = al2; else alpha_g[ll] = al2;
                    fl_s[ll] = flags_of(yl, al2, C);
                }
                if (P.trace && rank == 0 && cta == 0 && it < P.trace_cap) {
                    P.trace[2 * it] = u; P.trace[2 * it + 1] = l;
                    if (P.hist) { P.hist[2 * it] = sh.cu; P.hist[2 * it + 1] = sh.cl; }
                }
                if (P.progress && rank == 0 && cta == 0 && (it % P.check_interval) == 0)
                    *(volatile unsigned long long*)P.progress = (unsigned long long)it;
            }
            __syncwarp();
            SVM_PHASE(timing, PH_S_KUL);
            named_arrive<NSYNC_>(BAR_B);
            ++it;
            continue;
        }
        // ================= consumers: row pass (a3-a5)
        const int u = sh.u, l = sh.l;
        const bool gain = m_wss2 && sh.pass != 0;      // wss 2: gain pass over K(x_u, .)
        const bool c_hit = m_cache > 0 && sh.c_hit;
        const int su = sh.c_su, sl = sh.c_sl;
        bool rows_ready = m_gram != nullptr;
        const double* krow_u = nullptr;
        const double* krow_l = nullptr;
        double* fill_u = nullptr;
        double* fill_l = nullptr;
        if (m_gram) {
            krow_u = m_gram + (long long)u * P.n_global + gbase;
            krow_l = m_gram + (long long)l * P.n_global + gbase;
        } else if (m_cache > 0) {
            double* cb = P.cache[rank] + r0;                  // this CTA's columns of every slot
            const long long stride = P.n_rows[rank];
            if (c_hit) {
                rows_ready = true;
                krow_u = cb + su * stride;
                krow_l = cb + sl * stride;
            }
        }
        double cu = 0.0, cl = 0.0;
        double bfu = INF, bfl = -INF;
        int bju = INT_MAX, bjl = INT_MAX;
        if (n_tiles == 0) named_sync<NSYNC_>(BAR_B);
        if (m_isbin && !rows_ready && n_tiles > 0) {
            // binary bit rows resident (row j at words [j Wp, j Wp + Wp), Wp = W rounded up to 4);
            // thread t owns row t of every tile.  The popcounts of BT tiles are independent
            // chains computed together (16-byte loads), then the rows are updated after
            // barrier B.
            constexpr int BT = 8;
            const uint32_t* pw = reinterpret_cast<const uint32_t*>(piv);
            const int W = P.bin_words;
            const int Wq = (W + 3) >> 2;                  // 16-byte groups per row
            const uint4* x4 = reinterpret_cast<const uint4*>(ring);
            const uint4* p4 = reinterpret_cast<const uint4*>(pw);
            for (int tb = 0; tb < n_tiles; tb += BT) {
                // all loads of a batch are unconditional (clamped to a valid row), so they
                // issue back to back; rows past the end are computed and discarded
                int jq[BT];
#pragma unroll
                for (int q = 0; q < BT; ++q) jq[q] = min((tb + q) * P.rt + t, R - 1);
                int cu_[BT], cl_[BT];
#pragma unroll
                for (int q = 0; q < BT; ++q) { cu_[q] = 0; cl_[q] = 0; }
                for (int w4 = 0; w4 < Wq; ++w4) {
                    const uint4 pu = p4[w4], pl = p4[Wq + w4];
                    uint4 xv[BT];
#pragma unroll
                    for (int q = 0; q < BT; ++q) xv[q] = x4[jq[q] * Wq + w4];
#pragma unroll
                    for (int q = 0; q < BT; ++q) {
                        if (KERNEL == 1) {
                            cu_[q] += __popc(xv[q].x ^ pu.x) + __popc(xv[q].y ^ pu.y) + __popc(xv[q].z ^ pu.z) + __popc(xv[q].w ^ pu.w);
                            cl_[q] += __popc(xv[q].x ^ pl.x) + __popc(xv[q].y ^ pl.y) + __popc(xv[q].z ^ pl.z) + __popc(xv[q].w ^ pl.w);
                        } else {
                            cu_[q] += __popc(xv[q].x & pu.x) + __popc(xv[q].y & pu.y) + __popc(xv[q].z & pu.z) + __popc(xv[q].w & pu.w);
                            cl_[q] += __popc(xv[q].x & pl.x) + __popc(xv[q].y & pl.y) + __popc(xv[q].z & pl.z) + __popc(xv[q].w & pl.w);
                        }
                    }
                }
                if (tb == 0) {
                    SVM_PHASE(timing, PH_C_DIST);
                    named_sync<NSYNC_>(BAR_B);          // c_u, c_l and the owner's flags are ready
                    SVM_PHASE(timing, PH_C_WAITB);
                    cu = sh.cu; cl = sh.cl;
                }
                double ku[BT], kl[BT], fo[BT];
                uint8_t gq[BT];
#pragma unroll
                for (int q = 0; q < BT; ++q) {
                    const int j = min((tb + q) * P.rt + t, R - 1);
                    if (KERNEL == 1) {
                        ku[q] = ktab[cu_[q]];
                        kl[q] = ktab[cl_[q]];
                    } else {
                        ku[q] = (double)cu_[q]; kl[q] = (double)cl_[q];
                    }
                    fo[q] = f_s[j];
                    gq[q] = fl_s[j];
                }
                // (RBF: K(x_j, x_j) = ktab[0] = 1 already, R16)
                double cfu[BT], cfl[BT];
                int cju[BT], cjl[BT];
#pragma unroll
                for (int q = 0; q < BT; ++q) {
                    const int j = (tb + q) * P.rt + t;
                    cfu[q] = INF; cfl[q] = -INF; cju[q] = j; cjl[q] = j;
                    if (tb + q < n_tiles && j < R) {
                        const double fj = fma(cl, kl[q], fma(cu, ku[q], fo[q]));
                        f_s[j] = fj;
                        if (gq[q] & FL_UP) cfu[q] = fj;
                        if (gq[q] & FL_LOW) cfl[q] = fj;
                    }
                }
                // tree over the batch (rows increase with q: on equal f the lower q wins),
                // then against the running best (earlier rows: a tie keeps it)
#pragma unroll
                for (int s2 = 1; s2 < BT; s2 <<= 1)
#pragma unroll
                    for (int q = 0; q + s2 < BT; q += 2 * s2) {
                        if (cfu[q + s2] < cfu[q]) { cfu[q] = cfu[q + s2]; cju[q] = cju[q + s2]; }
                        if (cfl[q + s2] > cfl[q]) { cfl[q] = cfl[q + s2]; cjl[q] = cjl[q + s2]; }
                    }
                if (cfu[0] < bfu) { bfu = cfu[0]; bju = cju[0]; }
                if (cfl[0] > bfl) { bfl = cfl[0]; bjl = cjl[0]; }
            }
        } else
        for (int tile = 0; tile < n_tiles; ++tile) {
            const int rows_t = min(P.rt, R - tile * P.rt);
            const int rp = (rows_t + 3) & ~3;
            const bool active = t * RPT < rows_t;
            double du[RPT], dl[RPT];
#pragma unroll
            for (int q = 0; q < RPT; ++q) { du[q] = 0.0; dl[q] = 0.0; }
            if (rows_ready) {
                if (active) {
                    // kernel values already computed: rows of K (Gram) or cached rows
                    const double* ku_row = krow_u + tile * P.rt + t * RPT;
                    const double* kl_row = krow_l + tile * P.rt + t * RPT;
#pragma unroll
                    for (int q = 0; q < RPT; ++q) {
                        if (tile * P.rt + t * RPT + q < R) { du[q] = __ldcg(&ku_row[q]); dl[q] = __ldcg(&kl_row[q]); }
                    }
                }
            }
            for (int ch = 0; ch < ((m_isbin || rows_ready) ? 0 : P.n_chunks); ++ch) {
                if (!m_resident) mbar_wait(&full[cslot], cpar);
                const float* st = m_resident ? ring + (size_t)ch * P.kc * rp : ring + (size_t)cslot * stage_floats;
                const unsigned char* stb = ring_b + (m_resident ? (size_t)ch * P.kc * rp : (size_t)cslot * stage_floats) * esz;
                const int k0 = ch * P.kc;
                if (active && m_mixed) {
                    mixed_rows<KERNEL, RPT>(P, st, rp, t, pivm, pbits, du, dl);
                } else if (active && m_dict) {
                    dict_rows<KERNEL, RPT>(P.kc, stb, rp, t, piv + k0, dict_s, du, dl);
                } else if (active) {
                    if (RPT == 4) {
                        const float4* sp = reinterpret_cast<const float4*>(st) + t;
                        const int ld4 = rp >> 2;
#pragma unroll 4
                        for (int kk = 0; kk < P.kc; ++kk) {
                            const float4 v = sp[kk * ld4];
                            const double2 pv = piv[k0 + kk]; const double xu = pv.x, xl = pv.y;
                            const double x0 = v.x, x1 = v.y, x2 = v.z, x3 = v.w;
                            if (KERNEL == 1) {
                                double e;
                                e = x0 - xu; du[0] = fma(e, e, du[0]); e = x0 - xl; dl[0] = fma(e, e, dl[0]);
                                e = x1 - xu; du[1] = fma(e, e, du[1]); e = x1 - xl; dl[1] = fma(e, e, dl[1]);
                                e = x2 - xu; du[2] = fma(e, e, du[2]); e = x2 - xl; dl[2] = fma(e, e, dl[2]);
                                e = x3 - xu; du[3] = fma(e, e, du[3]); e = x3 - xl; dl[3] = fma(e, e, dl[3]);
                            } else {
                                du[0] = fma(x0, xu, du[0]); dl[0] = fma(x0, xl, dl[0]);
                                du[1] = fma(x1, xu, du[1]); dl[1] = fma(x1, xl, dl[1]);
                                du[2] = fma(x2, xu, du[2]); dl[2] = fma(x2, xl, dl[2]);
                                du[3] = fma(x3, xu, du[3]); dl[3] = fma(x3, xl, dl[3]);
                            }
                        }
                    } else if (RPT == 2) {
                        const float2* sp = reinterpret_cast<const float2*>(st) + t;
                        const int ld2 = rp >> 1;
#pragma unroll 4
                        for (int kk = 0; kk < P.kc; ++kk) {
                            const float2 v = sp[kk * ld2];
                            const double2 pv = piv[k0 + kk]; const double xu = pv.x, xl = pv.y;
                            const double x0 = v.x, x1 = v.y;
                            if (KERNEL == 1) {
                                double e;
                                e = x0 - xu; du[0] = fma(e, e, du[0]); e = x0 - xl; dl[0] = fma(e, e, dl[0]);
                                e = x1 - xu; du[1] = fma(e, e, du[1]); e = x1 - xl; dl[1] = fma(e, e, dl[1]);
                            } else {
                                du[0] = fma(x0, xu, du[0]); dl[0] = fma(x0, xl, dl[0]);
                                du[1] = fma(x1, xu, du[1]); dl[1] = fma(x1, xl, dl[1]);
                            }
                        }
                    } else {
                        const float* sp = st + t;
#pragma unroll 8
                        for (int kk = 0; kk < P.kc; ++kk) {
                            const double x0 = sp[kk * rp];
                            const double2 pv = piv[k0 + kk]; const double xu = pv.x, xl = pv.y;
                            if (KERNEL == 1) {
                                double e;
                                e = x0 - xu; du[0] = fma(e, e, du[0]);
                                e = x0 - xl; dl[0] = fma(e, e, dl[0]);
                            } else {
                                du[0] = fma(x0, xu, du[0]); dl[0] = fma(x0, xl, dl[0]);
                            }
                        }
                    }
                }
                __syncwarp();
                if (!m_resident) {
                    if (lane == 0) mbar_arrive(&empty[cslot]);
                    ++consumed;
                    if (++cslot == (unsigned)P.stages) { cslot = 0; cpar ^= 1u; }
                }
            }
            if (tile == 0) {
                SVM_PHASE(timing, PH_C_DIST);
                named_sync<NSYNC_>(BAR_B);          // c_u, c_l, the owner's flags and the fill slots are ready
                SVM_PHASE(timing, PH_C_WAITB);
                cu = sh.cu; cl = sh.cl;
                if (m_cache > 0 && !c_hit) {
                    double* cb = P.cache[rank] + r0;
                    const long long stride = P.n_rows[rank];
                    if (sh.c_fill_u >= 0) fill_u = cb + sh.c_fill_u * stride;
                    if (sh.c_fill_l >= 0) fill_l = cb + sh.c_fill_l * stride;
                }
            }
            if (active) {
                // kernel values of the thread's RPT rows: all fast exps first (independent,
                // branch-free chains), then the rare slow phases, then the f updates
                double ku[RPT], kl[RPT];
                if (rows_ready || KERNEL == 0) {
#pragma unroll
                    for (int q = 0; q < RPT; ++q) { ku[q] = du[q]; kl[q] = dl[q]; }
                } else {
                    bool su[RPT], sl[RPT];
                    bool all_safe = true;
#pragma unroll
                    for (int q = 0; q < RPT; ++q) {
                        ku[q] = svmexp::exp_cr_fast(-(P.gamma * du[q]), tab, su[q]);
                        if (gain) { kl[q] = ku[q]; sl[q] = true; }
                        else kl[q] = svmexp::exp_cr_fast(-(P.gamma * dl[q]), tab, sl[q]);
                        all_safe = all_safe && su[q] && sl[q];
                    }
                    if (!all_safe && !P.dbg_fast_only) {
#pragma unroll
                        for (int q = 0; q < RPT; ++q) {
                            if (!su[q]) ku[q] = svmexp::exp_cr_slow(-(P.gamma * du[q]), tab);
                            if (!sl[q]) kl[q] = svmexp::exp_cr_slow(-(P.gamma * dl[q]), tab);
                        }
                    }
#pragma unroll
                    for (int q = 0; q < RPT; ++q) {
                        const long long jg = gbase + tile * P.rt + t * RPT + q;
                        if (jg == u) ku[q] = 1.0;                // R16
                        if (jg == l) kl[q] = 1.0;
                    }
                }
                if (gain) {
                    // wss 2 gain pass: candidates t in I_low with f_t > f_u, gain
                    // (f_t - f_u)^2 / a_t, a_t = K_uu + K_tt - 2 K_ut (<= 1e-12 -> 1e-12); the
                    // maximum with the lowest index (rows in increasing j, strict >)
                    const double gfu = sh.gain_fu, gkuu = sh.gain_kuu;
#pragma unroll
                    for (int q = 0; q < RPT; ++q) {
                        const int j = tile * P.rt + t * RPT + q;
                        if (j < R) {
                            if (fill_u) fill_u[j] = ku[q];
                            const double fj = f_s[j];
                            if ((fl_s[j] & FL_LOW) && fj > gfu) {
                                const double bb = fj - gfu;
                                const double ktt = KERNEL == 1 ? 1.0 : __ldg(&P.qself[gbase + j]);
                                double aa = gkuu + ktt - 2.0 * ku[q];
                                if (!(aa > 1e-12)) aa = 1e-12;
                                const double gg = (bb * bb) / aa;
                                if (gg > bfl) { bfl = gg; bjl = j; }
                            }
                        }
                    }
                } else
#pragma unroll
                for (int q = 0; q < RPT; ++q) {
                    const int j = tile * P.rt + t * RPT + q;
                    if (j < R) {
                        if (fill_u) fill_u[j] = ku[q];          // row cache: store the computed
                        if (fill_l) fill_l[j] = kl[q];          // kernel values of a missed row
                        const double fj = fma(cl, kl[q], fma(cu, ku[q], f_s[j]));
                        f_s[j] = fj;
                        const uint8_t g = fl_s[j];
                        // rows are visited in increasing j: a tie keeps the earlier row
                        if ((g & FL_UP) && fj < bfu) { bfu = fj; bju = j; }
                        if ((g & FL_LOW) && fj > bfl) { bfl = fj; bjl = j; }
                    }
                }
            }
        }
        // filled cache columns are read by other CTAs' scalar warps (K_ul) in later
        // iterations: order them before this CTA's next record
        if (fill_u || fill_l) __threadfence();
        SVM_PHASE(timing, PH_C_UPDATE);
        {
            unsigned long long kw;
            unsigned iw;
            argmin_redux(0xffffffffu, fkey(bfu), (unsigned)bju, kw, iw);
            bju = (int)iw;
            bfu = bju == INT_MAX ? INF : fkey_inv(kw);
            argmin_redux(0xffffffffu, ~fkey(bfl), (unsigned)bjl, kw, iw);
            bjl = (int)iw;
            bfl = bjl == INT_MAX ? -INF : fkey_inv(~kw);
        }
        if (lane == 0) {
            sh.red_f[0][warp] = bfu; sh.red_i[0][warp] = bju;
            sh.red_f[1][warp] = bfl; sh.red_i[1][warp] = bjl;
            if (!A_SMEM) {
                sh.red_a[0][warp] = bju == INT_MAX ? 0.0 : alpha_g[bju];
                sh.red_a[1][warp] = bjl == INT_MAX ? 0.0 : alpha_g[bjl];
            }
        }
        ++it;
    }
    // ---- shutdown: stop the producer and drain the stages it issued
    if (t == 0) {
        sh.stop = 1;
        __threadfence_block();
        for (;;) {
            const int done = sh.producer_done;
            const unsigned int iss = sh.issued;
            if (consumed < iss) {
                mbar_wait(&full[cslot], cpar);
                for (int w = 0; w < NWC_; ++w) mbar_arrive(&empty[cslot]);
                ++consumed;
                if (++cslot == (unsigned)P.stages) { cslot = 0; cpar ^= 1u; }
            } else if (done) {
                break;
            }
        }
    }
    if (timing)
        for (int k = 0; k < PH_N; ++k) atomicAdd(&P.timers[k], sh.ph_acc[ph_row][k]);
    named_sync<NSYNC_>(BAR_D);
    // ---- write the CTA's state back (consumers) and the rank control (scalar warp)
    if (warp < NWC_) {
        for (int j = t; j < R; j += NT_) {
            P.f[rank][r0 + j] = f_s[j];
            if (A_SMEM) alpha_g[j] = a_s[j];
            P.flags[rank][r0 + j] = fl_s[j];
        }
    } else if (lane == 0 && cta == 0) {
        Ctl* ctl = P.ctl[rank];
        ctl->it = it;
        ctl->seq = seq;
        ctl->state = final_state;
        ctl->b_up = sh.f_up;
        ctl->b_low = sh.f_low;
        ctl->i_up = sh.u == INT_MAX ? -1 : sh.u;
        ctl->i_low = sh.l == INT_MAX ? -1 : sh.l;
        ctl->cache_hits += c_hits;
        ctl->cache_misses += c_misses;
    }
    __syncwarp();
    if (m_cluster) cluster_sync_all();
}

}  // namespace svmk
