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
enum { BAR_A = 1, BAR_B = 2, BAR_C = 3, BAR_D = 4, BAR_E = 5, BAR_F = 6 };

enum { ST_RUNNING = 0, ST_CONVERGED = 1, ST_MAXITER = 2, ST_LIMIT = 3, ST_TIMEOUT = -8 };
enum { FL_POS = 1, FL_UP = 2, FL_LOW = 4 };

// One CTA's candidate record in "LL" form: twelve 8-byte words, each = (32-bit flag << 32)
// | 32-bit payload, flag = exchange sequence number.  Aligned 8-byte stores are single-copy
// atomic, so a record whose twelve flags all read `seq` is complete: no release fence is
// needed on the writer's side.  Payload words: 0-1 f_up, 2-3 f_low, 4-5 a_up, 6-7 a_low
// (lo, hi halves), 8 i_up, 9 i_low (global row, -1 = empty set), 10 y_up | y_low << 16.
constexpr int REC_ROW_WORDS = 8;   // binary rows up to 256 features travel in the record
constexpr int NREP = 8;            // max replicas of every record (spreads the all-to-all reads)
struct __align__(16) Record {
    unsigned long long w[12 + 2 * REC_ROW_WORDS];   // base words, then the two candidate bit rows
};

struct __align__(128) Mailbox {
    unsigned long long count;      // monotonic arrivals (relaxed: a hint that all records landed)
    unsigned long long pad[15];
};
// records follow the header: Record recs[NREP][2][g_total] (replica, exchange parity)
__host__ __device__ inline Record* mbox_parts(Mailbox* m, int rep, int parity, int g_total) {
    return reinterpret_cast<Record*>(m + 1) + ((size_t)rep * 2 + parity) * g_total;
}
__host__ __device__ inline size_t mbox_bytes(int cpr, int world) {
    return sizeof(Mailbox) + (size_t)NREP * 2 * cpr * world * sizeof(Record);
}

struct Ctl {                       // per rank solver control, persists across launches
    long long it;                  // SMO updates done
    long long seq;                 // exchanges done
    int state;
    int pad;
    double b_up, b_low;
    long long i_up, i_low;
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
    unsigned long long* progress;  // host-mapped, may be null
    int check_interval;
    int state_cap;                 // rows per CTA the shared-memory state can hold
    int resident;                  // 1: the CTA's whole X block stays in shared memory (one tile)
    int bin_words;                 // > 0: X is exactly binary (every value 0 or 1) and stored as
                                   // bit rows of bin_words 32-bit words (SURVEY §8(f) compact
                                   // encoding); distances are popcounts -- exact, so identical to
                                   // the fp64 recurrence R13
    const uint32_t* xrbits;        // bit rows [n_global][bin_words] (pivot gather)
    int rec_rows;                  // 1: candidate bit rows travel in the records (bin_words <= 8)
    int nrep;                      // record replicas written (1..NREP); readers pick cta % nrep
    int direct_poll_ns;            // >= 0: skip the counter, poll the records directly with this backoff
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
    unsigned long long* timers;    // optional [8] per-phase cycle totals of CTA 0
};

// phase timers (cycles, CTA 0): scalar warp lane 0 ...
enum { PH_S_WAITC = 0, PH_S_PUBLISH, PH_S_POLL, PH_S_READ, PH_S_PIVOT, PH_S_KUL,
       // ... and consumer thread 0
       PH_C_EXCH, PH_C_PIVOT, PH_C_DIST, PH_C_WAITB, PH_C_UPDATE, PH_C_REDUCE, PH_N };

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
    while (!mbar_try_wait(bar, parity)) {
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
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_v2(unsigned long long* p, unsigned long long a,
                                               unsigned long long b) {
    asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" :: "l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_volatile_v2(const unsigned long long* p, unsigned long long& a,
                                               unsigned long long& b) {
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ unsigned long long ll_word(uint32_t flag, uint32_t payload) {
    return ((unsigned long long)flag << 32) | payload;
}
__device__ __forceinline__ void red_release_gpu(unsigned long long* p) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" :: "l"(p) : "memory");
}
__device__ __forceinline__ void red_release_sys(unsigned long long* p) {
    asm volatile("red.release.sys.global.add.u64 [%0], 1;" :: "l"(p) : "memory");
}
__device__ __forceinline__ void named_sync(int id) {
    asm volatile("bar.sync %0, %1;" :: "r"(id), "n"(NSYNC) : "memory");
}
__device__ __forceinline__ void named_arrive(int id) {
    asm volatile("bar.arrive %0, %1;" :: "r"(id), "n"(NSYNC) : "memory");
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
    double red_f[2][NWC];          // per consumer warp candidates (local row index)
    int red_i[2][NWC];
    double wf[2], wa[2];           // the global winner of this iteration
    int wi[2], wy[2];
    int c_slot_u, c_slot_l;        // row cache: slot holding K(u,.) / K(l,.) (hit) ...
    int c_fill_u, c_fill_l;        // ... or the slot this iteration fills (miss), else -1
    int c_stream;                  // 1: X must be streamed this iteration
    int c_fifo;                    // next FIFO victim slot
    int kul_cnt;                   // compacted terms of K(x_u, x_l) (cache mode)
    double cf[2][NWC + 1];         // per warp combine results (global row index)
    int ci[2][NWC + 1];
    double ca[2][NWC + 1];
    int cy[2][NWC + 1];
    int timeout;
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

// (the volatile shared load forces a deferred-blocking bar.sync to resolve before
// the clock is read)
// A (candidate up, candidate low) pair with the alpha and label of each.
struct Cand {
    double fu, fl, au, al;
    int iu, il, yu, yl;
};
__device__ __forceinline__ void cand_init(Cand& c) {
    c.fu = __longlong_as_double(0x7ff0000000000000ll); c.fl = -c.fu;
    c.au = 0.0; c.al = 0.0; c.iu = INT_MAX; c.il = INT_MAX; c.yu = 0; c.yl = 0;
}
__device__ __forceinline__ void cand_merge(Cand& a, const Cand& b) {
    if (b.iu != INT_MAX && better_up(b.fu, b.iu, a.fu, a.iu)) { a.fu = b.fu; a.iu = b.iu; a.au = b.au; a.yu = b.yu; }
    if (b.il != INT_MAX && better_low(b.fl, b.il, a.fl, a.il)) { a.fl = b.fl; a.il = b.il; a.al = b.al; a.yl = b.yl; }
}
__device__ __forceinline__ void cand_warp_merge(Cand& c) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        Cand b;
        b.fu = __shfl_xor_sync(0xffffffffu, c.fu, o); b.iu = __shfl_xor_sync(0xffffffffu, c.iu, o);
        b.au = __shfl_xor_sync(0xffffffffu, c.au, o); b.yu = __shfl_xor_sync(0xffffffffu, c.yu, o);
        b.fl = __shfl_xor_sync(0xffffffffu, c.fl, o); b.il = __shfl_xor_sync(0xffffffffu, c.il, o);
        b.al = __shfl_xor_sync(0xffffffffu, c.al, o); b.yl = __shfl_xor_sync(0xffffffffu, c.yl, o);
        cand_merge(c, b);
    }
}
__device__ __forceinline__ void ll_store(Record* rec, uint32_t fg, const Cand& c) {
    unsigned long long* w = rec->w;
    const unsigned long long bu = (unsigned long long)__double_as_longlong(c.fu);
    const unsigned long long bl = (unsigned long long)__double_as_longlong(c.fl);
    const unsigned long long au = (unsigned long long)__double_as_longlong(c.au);
    const unsigned long long al = (unsigned long long)__double_as_longlong(c.al);
    const uint32_t iu = c.iu == INT_MAX ? 0xffffffffu : (uint32_t)c.iu;
    const uint32_t il = c.il == INT_MAX ? 0xffffffffu : (uint32_t)c.il;
    const uint32_t yy = (uint32_t)((c.yu & 0xffff) | (c.yl << 16));
    st_volatile_v2(w + 0, ll_word(fg, (uint32_t)bu), ll_word(fg, (uint32_t)(bu >> 32)));
    st_volatile_v2(w + 2, ll_word(fg, (uint32_t)bl), ll_word(fg, (uint32_t)(bl >> 32)));
    st_volatile_v2(w + 4, ll_word(fg, (uint32_t)au), ll_word(fg, (uint32_t)(au >> 32)));
    st_volatile_v2(w + 6, ll_word(fg, (uint32_t)al), ll_word(fg, (uint32_t)(al >> 32)));
    st_volatile_v2(w + 8, ll_word(fg, iu), ll_word(fg, il));
    st_volatile_v2(w + 10, ll_word(fg, yy), ll_word(fg, 0u));
}
// the two candidate bit rows (W words each) after the 12 base words
__device__ __forceinline__ void ll_store_rows(Record* rec, uint32_t fg, const uint32_t* ru, const uint32_t* rl, int W) {
    unsigned long long* w = rec->w + 12;
    for (int h = 0; h < W; h += 2) {
        st_volatile_v2(w + h, ll_word(fg, ru[h]), ll_word(fg, h + 1 < W ? ru[h + 1] : 0u));
        st_volatile_v2(w + REC_ROW_WORDS + h, ll_word(fg, rl[h]), ll_word(fg, h + 1 < W ? rl[h + 1] : 0u));
    }
}
// One attempt: true (and c filled) when every word carries flag fg.
__device__ __forceinline__ bool ll_try_load(const Record* rec, uint32_t fg, Cand& c) {
    unsigned long long v[12];
#pragma unroll
    for (int h = 0; h < 6; ++h) ld_volatile_v2(rec->w + 2 * h, v[2 * h], v[2 * h + 1]);
    bool ok = true;
#pragma unroll
    for (int h = 0; h < 12; ++h) ok = ok && (uint32_t)(v[h] >> 32) == fg;
    if (!ok) return false;
    c.fu = __longlong_as_double((long long)((v[0] & 0xffffffffull) | (v[1] << 32)));
    c.fl = __longlong_as_double((long long)((v[2] & 0xffffffffull) | (v[3] << 32)));
    c.au = __longlong_as_double((long long)((v[4] & 0xffffffffull) | (v[5] << 32)));
    c.al = __longlong_as_double((long long)((v[6] & 0xffffffffull) | (v[7] << 32)));
    const int iu = (int)(uint32_t)v[8], il = (int)(uint32_t)v[9];
    c.iu = iu < 0 ? INT_MAX : iu;
    c.il = il < 0 ? INT_MAX : il;
    const uint32_t py = (uint32_t)v[10];
    c.yu = (int)(int16_t)(py & 0xffff);
    c.yl = (int)(int16_t)(py >> 16);
    return true;
}
__device__ __forceinline__ void red_relaxed_gpu(unsigned long long* p) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" :: "l"(p) : "memory");
}
__device__ __forceinline__ void red_relaxed_sys(unsigned long long* p) {
    asm volatile("red.relaxed.sys.global.add.u64 [%0], 1;" :: "l"(p) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_gpu(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

#define SVM_PHASE(on, ph)                                                    \
    do {                                                                     \
        if (on) {                                                            \
            (void)*(volatile int*)&sh.decision;                              \
            const long long c_ = clock64();                                  \
            ph_acc[ph] += (unsigned long long)(c_ - ph_t);                   \
            ph_t = c_;                                                       \
        }                                                                    \
    } while (0)

// ------------------------------------------------------------------ the kernel
template <int KERNEL, int RPT, bool A_SMEM>
__global__ void __launch_bounds__(NTHREADS, 1) smo_persistent(const Params P) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Shared& sh = *reinterpret_cast<Shared*>(smem_raw);
    size_t off = (sizeof(Shared) + 127) & ~size_t(127);
    // pivots interleaved: piv[k] = (x_up[k], x_low[k]) -> one 16-byte broadcast load per k
    double2* piv = reinterpret_cast<double2*>(smem_raw + off); off += (size_t)P.d_pad * 16;
    double* f_s = reinterpret_cast<double*>(smem_raw + off); off += (size_t)P.state_cap * 8;
    double* a_s = reinterpret_cast<double*>(smem_raw + off); if (A_SMEM) off += (size_t)P.state_cap * 8;
    uint8_t* fl_s = smem_raw + off; off += (size_t)P.state_cap;
    off = (off + 7) & ~size_t(7);
    // binary RBF: K for every possible Hamming distance, K_tab[D] = exp_cr(-(gamma D))
    double* ktab = reinterpret_cast<double*>(smem_raw + off);
    if (P.bin_words) off += (size_t)(32 * P.bin_words + 1) * 8;
    off = (off + 7) & ~size_t(7);
    // row-cache directory: owner (global row) of every slot + an open-addressing hash
    // row -> slot (cache_hash entries, a power of two >= 2 slots), FIFO replacement
    int* dir_owner = reinterpret_cast<int*>(smem_raw + off); off += (size_t)P.cache_slots * 4;
    off = (off + 7) & ~size_t(7);
    int2* dir_hash = reinterpret_cast<int2*>(smem_raw + off); off += (size_t)P.cache_hash * 8;
    // cache mode: the scalar warp compacts the k with a non-zero term of K(x_u, x_l) here
    off = (off + 15) & ~size_t(15);
    double2* kul_t = reinterpret_cast<double2*>(smem_raw + off);
    if (P.cache_slots > 0) off += (size_t)P.d_pad * 16;
    off = (off + 127) & ~size_t(127);
    float* ring = reinterpret_cast<float*>(smem_raw + off);
    const int stage_floats = P.kc * P.rt;
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
    const float* xcta = P.xblk[rank] + (long long)cta * P.cta_stride;
    double* alpha_g = P.alpha[rank] + r0;                    // this CTA's alpha (global)
    const double C = P.C;

    if (t == 0) {
        sh.stop = 0; sh.producer_done = 0; sh.issued = 0; sh.timeout = 0;
        for (int s = 0; s < P.stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NWC); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int e = t; e < svmexp::EXP_TABLE_DOUBLES; e += NTHREADS) sh.exp_tab[e] = svmexp::table_entry(e);
    for (int e = t; e < P.cache_slots; e += NTHREADS) dir_owner[e] = -1;
    for (int e = t; e < P.cache_hash; e += NTHREADS) dir_hash[e] = make_int2(-1, -1);
    if (t == 0) sh.c_fifo = 0;
    for (int j = t; j < R; j += NTHREADS) {
        f_s[j] = P.f[rank][r0 + j];
        if (A_SMEM) a_s[j] = alpha_g[j];
        fl_s[j] = P.flags[rank][r0 + j];
    }
    __syncthreads();
    const svmexp::PtrTab tab{sh.exp_tab};
    if (KERNEL == 1 && P.bin_words) {
        for (int e = t; e <= 32 * P.bin_words; e += NTHREADS) ktab[e] = svmexp::exp_cr_t(-(P.gamma * (double)e), tab);
        __syncthreads();
    }

    // ============================================================ producer warp
    if (warp == PRODUCER_WARP) {
        if (P.gram) {
            if (lane == 0) { sh.issued = 0; __threadfence_block(); sh.producer_done = 1; }
            return;
        }
        if (P.resident) {
            if (lane == 0 && n_tiles > 0) {
                const int rp = (R + 3) & ~3;
                const uint32_t bytes = P.bin_words ? (uint32_t)(n_tiles * P.bin_words * P.rt * 4)
                                                   : (uint32_t)P.d_pad * rp * 4u;
                mbar_arrive_tx(&full[0], bytes);
                bulk_g2s(ring, xcta, bytes, &full[0]);
            }
            if (lane == 0) { sh.issued = 0; __threadfence_block(); sh.producer_done = 1; }
            return;
        }
        if (lane == 0 && n_tiles > 0) {
            unsigned int s = 0, slot = 0, par = 0;
            bool wrapped = false;
            int tile = 0, chunk = 0;
            for (;;) {
                if (wrapped) {
                    while (!mbar_try_wait(&empty[slot], par ^ 1u)) {
                        if (sh.stop) break;
                    }
                }
                if (sh.stop) break;
                const int rows_t = min(P.rt, R - tile * P.rt);
                const int rp = (rows_t + 3) & ~3;
                const uint32_t bytes = (uint32_t)P.kc * rp * 4u;
                const float* src = xcta + (long long)tile * P.d_pad * P.rt + (long long)chunk * P.kc * rp;
                mbar_arrive_tx(&full[slot], bytes);
                bulk_g2s(ring + (size_t)slot * stage_floats, src, bytes, &full[slot]);
                ++s;
                sh.issued = s;
                if (++slot == (unsigned)P.stages) { slot = 0; par ^= 1u; wrapped = true; }
                if (++chunk == P.n_chunks) { chunk = 0; if (++tile == n_tiles) tile = 0; }
            }
        }
        if (lane == 0) { __threadfence_block(); sh.producer_done = 1; }
        return;
    }

    unsigned long long ph_acc[PH_N] = {};
    long long ph_t = clock64();
    const bool is_scalar = (warp == SCALAR_WARP);
    const bool timing = P.timers != nullptr && blockIdx.x == 0 && (t == 0 || (is_scalar && lane == 0));
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
    const double INF = __longlong_as_double(0x7ff0000000000000ll);

    if (P.resident && !P.gram && n_tiles > 0 && !is_scalar) mbar_wait(&full[0], 0);
    // ---- initial selection from the current state (no update)
    if (!is_scalar) {
        double fu = INF, fl = -INF;
        int ju = INT_MAX, jl = INT_MAX;
        for (int j = t; j < R; j += NT) {
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
        }
    }

    for (;;) {
        named_sync(BAR_C);                  // consumer candidates are in sh.red_*
        SVM_PHASE(timing, is_scalar ? PH_S_WAITC : PH_C_REDUCE);
        // ---- exchange seq + 1 (a6).  The scalar warp stores the CTA record (LL form)
        // into every rank's mailbox -- peer pointers when the ranks are GPUs -- and bumps
        // each rank's arrival counter with a relaxed reduction (no fence: the records
        // validate themselves).  One thread polls the local counter; then every thread of
        // the CTA reads its share of the records (re-reading any whose flags are not yet
        // current) and the CTA reduces them lexicographically -- identical in every CTA of
        // every rank.  Chosen by measurement (tools/exchange_bench.cu).
        ++seq;
        const int g_total = xworld * P.ctas_per_rank;
        const int par = (int)(seq & 1);
        const uint32_t fg = (uint32_t)seq;
        if (is_scalar) {
            double fu = lane < NWC ? sh.red_f[0][lane] : INF;
            int ju = lane < NWC ? sh.red_i[0][lane] : INT_MAX;
            double fl = lane < NWC ? sh.red_f[1][lane] : -INF;
            int jl = lane < NWC ? sh.red_i[1][lane] : INT_MAX;
            warp_reduce_fi<true>(fu, ju, NWC);
            warp_reduce_fi<false>(fl, jl, NWC);
            // lanes 0-7 hold the CTA result; every lane writes some replica -> broadcast
            fu = __shfl_sync(0xffffffffu, fu, 0); ju = __shfl_sync(0xffffffffu, ju, 0);
            fl = __shfl_sync(0xffffffffu, fl, 0); jl = __shfl_sync(0xffffffffu, jl, 0);
            {
                Cand c;
                c.fu = fu; c.fl = fl;
                c.iu = (ju == INT_MAX) ? INT_MAX : (int)(gbase + ju);
                c.il = (jl == INT_MAX) ? INT_MAX : (int)(gbase + jl);
                c.au = (ju == INT_MAX) ? 0.0 : (A_SMEM ? a_s[ju] : alpha_g[ju]);
                c.al = (jl == INT_MAX) ? 0.0 : (A_SMEM ? a_s[jl] : alpha_g[jl]);
                c.yu = (ju == INT_MAX) ? 0 : ((fl_s[ju] & FL_POS) ? 1 : -1);
                c.yl = (jl == INT_MAX) ? 0 : ((fl_s[jl] & FL_POS) ? 1 : -1);
                uint32_t ru[REC_ROW_WORDS], rl[REC_ROW_WORDS];
                if (P.rec_rows) {
                    // the candidates' bit rows, from the resident block [tile][word][row]
                    const uint32_t* xbits = reinterpret_cast<const uint32_t*>(ring);
                    const int W = P.bin_words;
#pragma unroll
                    for (int h = 0; h < REC_ROW_WORDS; ++h) {
                        ru[h] = 0u; rl[h] = 0u;
                        if (h < W && ju != INT_MAX) {
                            const int tl = ju / P.rt, rin = ju - tl * P.rt, rows_t = min(P.rt, R - tl * P.rt);
                            ru[h] = xbits[(size_t)tl * W * P.rt + (size_t)h * ((rows_t + 3) & ~3) + rin];
                        }
                        if (h < W && jl != INT_MAX) {
                            const int tl = jl / P.rt, rin = jl - tl * P.rt, rows_t = min(P.rt, R - tl * P.rt);
                            rl[h] = xbits[(size_t)tl * W * P.rt + (size_t)h * ((rows_t + 3) & ~3) + rin];
                        }
                    }
                }
                const int gcta = (rank - xbase) * P.ctas_per_rank + cta;
                for (int q = lane; q < xworld * P.nrep; q += 32) {
                    Record* rec = mbox_parts(P.mbox[xbase + q / P.nrep], q % P.nrep, par, g_total) + gcta;
                    ll_store(rec, fg, c);
                    if (P.rec_rows) ll_store_rows(rec, fg, ru, rl, P.bin_words);
                }
                __syncwarp();
                if (lane < xworld && P.direct_poll_ns < 0) {
                    if (P.sys_scope) red_relaxed_sys(&P.mbox[xbase + lane]->count);
                    else red_relaxed_gpu(&P.mbox[xbase + lane]->count);
                }
            }
            SVM_PHASE(timing, PH_S_PUBLISH);
            if (lane == 0 && P.direct_poll_ns < 0) {
                const unsigned long long target = (unsigned long long)seq * g_total;
                long long t0 = 0;
                unsigned int spins = 0;
                while ((P.sys_scope ? ld_relaxed_sys(&my_mb->count) : ld_relaxed_gpu(&my_mb->count)) < target) {
                    if ((++spins & 1023u) == 0) {
                        const long long now = globaltimer();
                        if (t0 == 0) t0 = now;
                        else if (now - t0 > P.timeout_ns) { sh.timeout = 1; break; }
                    }
                }
            }
            SVM_PHASE(timing, PH_S_POLL);
        }
        named_sync(BAR_E);                  // records published (direct mode) / landed (counter mode)
        uint32_t myrow_u[REC_ROW_WORDS], myrow_l[REC_ROW_WORDS];  // bit rows of my best candidates
        int my_iu = INT_MAX, my_il = INT_MAX;
        {
            Cand c;
            cand_init(c);
            if (!sh.timeout) {
                const Record* recs = mbox_parts(my_mb, cta % P.nrep, par, g_total);
                long long t0 = 0;
                unsigned int spins = 0;
                for (int g = t; g < g_total; g += NSYNC) {
                    Cand r;
                    bool ok;
                    uint32_t wu[REC_ROW_WORDS], wl[REC_ROW_WORDS];
                    for (;;) {
                        ok = ll_try_load(recs + g, fg, r);
                        if (ok && P.rec_rows) {
                            const unsigned long long* w = recs[g].w + 12;
#pragma unroll
                            for (int h = 0; h < REC_ROW_WORDS; h += 2) {
                                unsigned long long a0, a1, b0, b1;
                                if (h < P.bin_words) {
                                    ld_volatile_v2(w + h, a0, a1);
                                    ld_volatile_v2(w + REC_ROW_WORDS + h, b0, b1);
                                    ok = ok && (uint32_t)(a0 >> 32) == fg && (uint32_t)(a1 >> 32) == fg &&
                                         (uint32_t)(b0 >> 32) == fg && (uint32_t)(b1 >> 32) == fg;
                                    wu[h] = (uint32_t)a0; wu[h + 1] = (uint32_t)a1;
                                    wl[h] = (uint32_t)b0; wl[h + 1] = (uint32_t)b1;
                                } else {
                                    wu[h] = wu[h + 1] = wl[h] = wl[h + 1] = 0u;
                                }
                            }
                        }
                        if (ok) break;
                        if (P.direct_poll_ns > 0) __nanosleep(P.direct_poll_ns);
                        if ((++spins & 255u) == 0) {
                            const long long now = globaltimer();
                            if (t0 == 0) t0 = now;
                            else if (now - t0 > P.timeout_ns) { sh.timeout = 1; break; }
                        }
                    }
                    if (!ok) break;
                    if (r.iu != INT_MAX && better_up(r.fu, r.iu, c.fu, c.iu)) {
                        c.fu = r.fu; c.iu = r.iu; c.au = r.au; c.yu = r.yu;
                        my_iu = r.iu;
#pragma unroll
                        for (int h = 0; h < REC_ROW_WORDS; ++h) myrow_u[h] = wu[h];
                    }
                    if (r.il != INT_MAX && better_low(r.fl, r.il, c.fl, c.il)) {
                        c.fl = r.fl; c.il = r.il; c.al = r.al; c.yl = r.yl;
                        my_il = r.il;
#pragma unroll
                        for (int h = 0; h < REC_ROW_WORDS; ++h) myrow_l[h] = wl[h];
                    }
                }
            }
            cand_warp_merge(c);
            if (lane == 0 && P.bin_words && !P.rec_rows && c.iu != INT_MAX && c.il != INT_MAX) {
                // the winner is one of the 9 warp results: pull their bit rows into this
                // SM's L1 now, so the pivot gather after barrier F hits L1
                asm volatile("prefetch.global.L1 [%0];" :: "l"(P.xrbits + (long long)c.iu * P.bin_words));
                asm volatile("prefetch.global.L1 [%0];" :: "l"(P.xrbits + (long long)c.il * P.bin_words));
            }
            if (lane == 0) {
                sh.cf[0][warp] = c.fu; sh.ci[0][warp] = c.iu; sh.ca[0][warp] = c.au; sh.cy[0][warp] = c.yu;
                sh.cf[1][warp] = c.fl; sh.ci[1][warp] = c.il; sh.ca[1][warp] = c.al; sh.cy[1][warp] = c.yl;
            }
        }
        named_sync(BAR_F);
        SVM_PHASE(timing, is_scalar ? PH_S_READ : PH_C_EXCH);
        // every thread reduces the 9 warp results in the same order -> same winners
        double fu = sh.cf[0][0], fl = sh.cf[1][0], au = sh.ca[0][0], al = sh.ca[1][0];
        int iu = sh.ci[0][0], il = sh.ci[1][0], yu = sh.cy[0][0], yl = sh.cy[1][0];
#pragma unroll
        for (int w = 1; w < NWC + 1; ++w) {
            if (better_up(sh.cf[0][w], sh.ci[0][w], fu, iu)) { fu = sh.cf[0][w]; iu = sh.ci[0][w]; au = sh.ca[0][w]; yu = sh.cy[0][w]; }
            if (better_low(sh.cf[1][w], sh.ci[1][w], fl, il)) { fl = sh.cf[1][w]; il = sh.ci[1][w]; al = sh.ca[1][w]; yl = sh.cy[1][w]; }
        }
        int dec = ST_RUNNING;
        if (sh.timeout) dec = ST_TIMEOUT;
        else if (iu == INT_MAX || il == INT_MAX) dec = ST_CONVERGED;
        else if (fl - fu <= 2.0 * P.tol) dec = ST_CONVERGED;
        else if (it == max_iter) dec = ST_MAXITER;
        else if (P.iter_limit > 0 && it - it_start == P.iter_limit) dec = ST_LIMIT;
        if (dec != ST_RUNNING) {
            final_state = dec;
            if (t == 0) { sh.u = iu; sh.l = il; sh.f_up = fu; sh.f_low = fl; }
            break;
        }
        // ---- row cache (a8): thread 0 of every CTA runs the same directory operations on
        // the same pair sequence (hash lookup, FIFO replacement), so every CTA agrees
        if (P.cache_slots > 0 && t == 0) {
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
            const int su = find(iu), sl = find(il);
            int fu_ = -1, fl_ = -1;
            auto victim = [&](int avoid) {
                int v = sh.c_fifo;
                if (v == avoid) v = (v + 1) % P.cache_slots;
                sh.c_fifo = (v + 1) % P.cache_slots;
                if (dir_owner[v] >= 0) erase(dir_owner[v]);
                return v;
            };
            if (su < 0) { fu_ = victim(sl); dir_owner[fu_] = iu; insert(iu, fu_); }
            if (sl < 0) { fl_ = victim(su >= 0 ? su : fu_); dir_owner[fl_] = il; insert(il, fl_); }
            sh.c_slot_u = su; sh.c_slot_l = sl; sh.c_fill_u = fu_; sh.c_fill_l = fl_;
            sh.c_stream = (su < 0 || sl < 0) ? 1 : 0;
        }
        // ---- pivot rows x_up, x_low (fp64 in shared memory, or bit rows), all threads
        if (P.gram) {
            // rows of K are read directly; no pivot rows needed
        } else if (P.rec_rows) {
            uint32_t* pw = reinterpret_cast<uint32_t*>(piv);
            if (my_iu == iu)
                for (int h = 0; h < P.bin_words; ++h) pw[h] = myrow_u[h];
            if (my_il == il)
                for (int h = 0; h < P.bin_words; ++h) pw[P.bin_words + h] = myrow_l[h];
        } else if (P.bin_words) {
            uint32_t* pw = reinterpret_cast<uint32_t*>(piv);
            if (t < 2 * P.bin_words) {
                const int w = t % P.bin_words;
                pw[t] = __ldg(&P.xrbits[(long long)(t < P.bin_words ? iu : il) * P.bin_words + w]);
            }
        } else {
            const float* xu_g = xr + (long long)iu * P.d;
            const float* xl_g = xr + (long long)il * P.d;
            for (int k0 = 0; k0 < P.d_pad; k0 += NSYNC * 4) {
                float vu[4], vl[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int k = k0 + q * NSYNC + t;
                    vu[q] = (k < P.d) ? __ldg(&xu_g[k]) : 0.0f;
                    vl[q] = (k < P.d) ? __ldg(&xl_g[k]) : 0.0f;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int k = k0 + q * NSYNC + t;
                    if (k < P.d_pad) piv[k] = make_double2((double)vu[q], (double)vl[q]);
                }
            }
        }
        named_sync(BAR_A);
        SVM_PHASE(timing, is_scalar ? PH_S_PIVOT : PH_C_PIVOT);
        const int u = iu, l = il;
        if (is_scalar) {
            if (P.cache_slots > 0) {
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
            if (lane == 0) {
                double Kuu, Kll, Kul;
                if (P.gram) {
                    const long long n = P.n_global;
                    Kuu = __ldg(&P.gram[(long long)u * n + u]);
                    Kll = __ldg(&P.gram[(long long)l * n + l]);
                    Kul = __ldg(&P.gram[(long long)u * n + l]);
                } else if (P.bin_words) {
                    const uint32_t* pw = reinterpret_cast<const uint32_t*>(piv);
                    int cuu = 0, cll = 0, cul = 0, cx = 0;
                    for (int w = 0; w < P.bin_words; ++w) {
                        const uint32_t a = pw[w], bb = pw[P.bin_words + w];
                        cuu += __popc(a); cll += __popc(bb); cul += __popc(a & bb); cx += __popc(a ^ bb);
                    }
                    if (KERNEL == 1) {
                        Kuu = 1.0; Kll = 1.0;
                        Kul = (u == l) ? 1.0 : ktab[cx];
                    } else {
                        Kuu = (double)cuu; Kll = (double)cll; Kul = (double)cul;
                    }
                } else if (P.cache_slots > 0) {
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
                }
                if (P.progress && rank == 0 && cta == 0 && (it % P.check_interval) == 0)
                    *(volatile unsigned long long*)P.progress = (unsigned long long)it;
            }
            __syncwarp();
            SVM_PHASE(timing, PH_S_KUL);
            named_arrive(BAR_B);
            ++it;
            continue;
        }
        // ================= consumers: row pass (a3-a5)
        bool rows_ready = P.gram != nullptr;
        const double* krow_u = nullptr;
        const double* krow_l = nullptr;
        double* fill_u = nullptr;
        double* fill_l = nullptr;
        if (P.gram) {
            krow_u = P.gram + (long long)u * P.n_global + gbase;
            krow_l = P.gram + (long long)l * P.n_global + gbase;
        } else if (P.cache_slots > 0) {
            double* cb = P.cache[rank] + r0;                  // this CTA's columns of every slot
            const long long stride = P.n_rows[rank];
            if (!sh.c_stream) {
                rows_ready = true;
                krow_u = cb + sh.c_slot_u * stride;
                krow_l = cb + sh.c_slot_l * stride;
            } else {
                if (sh.c_fill_u >= 0) fill_u = cb + sh.c_fill_u * stride;
                if (sh.c_fill_l >= 0) fill_l = cb + sh.c_fill_l * stride;
            }
        }
        double cu = 0.0, cl = 0.0;
        double bfu = INF, bfl = -INF;
        int bju = INT_MAX, bjl = INT_MAX;
        if (n_tiles == 0) named_sync(BAR_B);
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
            } else if (P.bin_words) {
                if (active) {
                    // bit rows resident in shared memory: [tile][word][row], popcounts
                    const uint32_t* xb = reinterpret_cast<const uint32_t*>(ring) + (size_t)tile * P.bin_words * P.rt + t;
                    const uint32_t* pw = reinterpret_cast<const uint32_t*>(piv);
                    int cu_ = 0, cl_ = 0;
                    for (int w = 0; w < P.bin_words; ++w) {
                        const uint32_t xv = xb[(size_t)w * rp];
                        if (KERNEL == 1) { cu_ += __popc(xv ^ pw[w]); cl_ += __popc(xv ^ pw[P.bin_words + w]); }
                        else { cu_ += __popc(xv & pw[w]); cl_ += __popc(xv & pw[P.bin_words + w]); }
                    }
                    du[0] = (double)cu_; dl[0] = (double)cl_;
                }
            }
            for (int ch = 0; ch < ((P.bin_words || rows_ready) ? 0 : P.n_chunks); ++ch) {
                if (!P.resident) mbar_wait(&full[cslot], cpar);
                const float* st = P.resident ? ring + (size_t)ch * P.kc * rp : ring + (size_t)cslot * stage_floats;
                const int k0 = ch * P.kc;
                if (active) {
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
                if (!P.resident) {
                    if (lane == 0) mbar_arrive(&empty[cslot]);
                    ++consumed;
                    if (++cslot == (unsigned)P.stages) { cslot = 0; cpar ^= 1u; }
                }
            }
            if (tile == 0) {
                SVM_PHASE(timing, PH_C_DIST);
                named_sync(BAR_B);          // c_u, c_l and the owner's flags are ready
                SVM_PHASE(timing, PH_C_WAITB);
                cu = sh.cu; cl = sh.cl;
            }
            if (active) {
#pragma unroll
                for (int q = 0; q < RPT; ++q) {
                    const int j = tile * P.rt + t * RPT + q;
                    if (j < R) {
                        const long long jg = gbase + j;
                        double ku, kl;
                        if (rows_ready) {
                            ku = du[q]; kl = dl[q];
                        } else if (KERNEL == 1 && P.bin_words) {
                            ku = (jg == u) ? 1.0 : ktab[(int)du[q]];
                            kl = (jg == l) ? 1.0 : ktab[(int)dl[q]];
                        } else if (KERNEL == 1) {
                            ku = (jg == u) ? 1.0 : svmexp::exp_cr_t(-(P.gamma * du[q]), tab);
                            kl = (jg == l) ? 1.0 : svmexp::exp_cr_t(-(P.gamma * dl[q]), tab);
                        } else {
                            ku = du[q]; kl = dl[q];
                        }
                        if (fill_u) fill_u[j] = ku;          // row cache: store the computed
                        if (fill_l) fill_l[j] = kl;          // kernel values of a missed row
                        const double fj = fma(cl, kl, fma(cu, ku, f_s[j]));
                        f_s[j] = fj;
                        const uint8_t g = fl_s[j];
                        if ((g & FL_UP) && better_up(fj, j, bfu, bju)) { bfu = fj; bju = j; }
                        if ((g & FL_LOW) && better_low(fj, j, bfl, bjl)) { bfl = fj; bjl = j; }
                    }
                }
            }
        }
        SVM_PHASE(timing, PH_C_UPDATE);
        warp_reduce_fi<true>(bfu, bju);
        warp_reduce_fi<false>(bfl, bjl);
        if (lane == 0) {
            sh.red_f[0][warp] = bfu; sh.red_i[0][warp] = bju;
            sh.red_f[1][warp] = bfl; sh.red_i[1][warp] = bjl;
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
                for (int w = 0; w < NWC; ++w) mbar_arrive(&empty[cslot]);
                ++consumed;
                if (++cslot == (unsigned)P.stages) { cslot = 0; cpar ^= 1u; }
            } else if (done) {
                break;
            }
        }
    }
    if (timing)
        for (int k = 0; k < PH_N; ++k) atomicAdd(&P.timers[k], ph_acc[k]);
    named_sync(BAR_D);
    // ---- write the CTA's state back (consumers) and the rank control (scalar warp)
    if (warp < NWC) {
        for (int j = t; j < R; j += NT) {
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
    }
}

}  // namespace svmk
