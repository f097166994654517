// smo_kernel.cuh -- the persistent, row-sharded SMO solver kernel for sm_100a.
//
// One launch runs many SMO iterations (§3.2: "a thread per
// independent training data sample ... convergence checks ... for every set of
// iterations").  Design (DESIGN.md §"Kernels"):
//
//   * Rows are sharded over ranks (GPUs, or CTA groups of one GPU) and, inside a
//     rank, over CTAs: CTA c owns a contiguous row block for the whole solve and keeps
//     its solver state -- f (fp64), alpha (fp64), flags (y, I_up, I_low) -- in shared
//     memory.  Only X is streamed per iteration.
//   * X lives in HBM in a CTA-blocked, feature-major layout ("xblk"): per CTA, tiles of
//     rt rows, each tile [d_pad][rows] fp32.  A producer warp streams it through a ring
//     of shared-memory stages with cp.async.bulk (TMA bulk copies) + mbarriers; 8
//     consumer warps compute, one thread per row (RPT rows per thread).
//   * Per iteration (a2-a7 of SURVEY.md §8):
//       combine   every CTA reads the 48-byte candidate records of all CTAs of all
//                 ranks from its rank-local mailbox, reduces them lexicographically
//                 (f, then lowest global index) -> (i_up, i_low), identical everywhere
//       test      b_low - b_up <= 2 tol -> converged (device-latched, same decision
//                 in every CTA)
//       update    thread 0 of every CTA gathers x_up, x_low from the row-major replica,
//                 computes eta, the clipped step t and the snapped alphas (fp64,
//                 SPEC.md L203-211); the owner CTA stores its alphas/flags
//       row pass  for each owned row j: D_u = sum_k (x_jk - x_uk)^2, D_l likewise
//                 (ascending k, one fma per term), K = exp_cr(-gamma D) (RBF) or the dot
//                 product (linear); f_j = fma(c_l, K_l, fma(c_u, K_u, f_j)); status;
//                 local (f, index) candidates -> warp shuffle -> CTA record
//       exchange  the record is stored into every rank's mailbox (peer pointers when
//                 the ranks are GPUs), then a release fence + one atomic add per rank
//                 on a monotonic arrival counter.
//   * Exact readings: no contraction (--fmad=false), explicit fma where the oracle has
//     one, correctly rounded exp, exact comparisons on alpha.  Results do not depend on
//     the number of ranks / CTAs.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "svm_exp.cuh"

namespace svmk {

constexpr int MAXR = 8;          // max ranks (GPUs or virtual)
constexpr int NT = 256;          // consumer threads per CTA
constexpr int NWC = NT / 32;     // consumer warps
constexpr int NTHREADS = NT + 32;  // + one producer warp
constexpr int MAX_STAGES = 8;

enum { ST_RUNNING = 0, ST_CONVERGED = 1, ST_MAXITER = 2, ST_LIMIT = 3, ST_TIMEOUT = -8 };
enum { FL_POS = 1, FL_UP = 2, FL_LOW = 4 };

struct __align__(16) Partial {   // one CTA's candidate record (48 B)
    double f_up, f_low, a_up, a_low;
    int32_t i_up, i_low;         // global row index, -1 if the set is empty
    int32_t y_up, y_low;
};

struct __align__(128) Mailbox {
    unsigned long long count;    // monotonic number of records received
    unsigned long long pad[15];
};
// partials follow the header: Partial parts[2][g_total]
__host__ __device__ inline Partial* mbox_parts(Mailbox* m, int parity, int g_total) {
    return reinterpret_cast<Partial*>(m + 1) + (size_t)parity * g_total;
}

struct Ctl {                     // per rank solver control, persists across launches
    long long it;                // SMO updates done
    long long seq;               // exchanges done
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
    const float* xr;             // row-major replica [n_global][d]
    long long cta_stride;        // floats per CTA block in xblk
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
    int state_cap;               // rows per CTA the shared-memory state can hold
    long long timeout_ns;
};

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
__device__ __forceinline__ long long globaltimer_ns() {
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
            const long long now = globaltimer_ns();
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
__device__ __forceinline__ long long globaltimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void bar_consumers() {
    asm volatile("bar.sync 1, %0;" :: "n"(NT) : "memory");
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
    // pipeline control
    volatile int stop;
    volatile int producer_done;
    volatile unsigned int issued;
    int timeout;
    // iteration scalars (written by consumer thread 0 after the combine)
    int decision;                // ST_*
    int u, l;                    // global winners
    double f_up, f_low, a_up, a_low;
    int y_up, y_low;
    double cu, cl, au_new, al_new;
    // reduction scratch
    double red_f[2][NWC];
    int red_i[2][NWC];
    double red_a[2][NWC];
    int red_y[2][NWC];
    unsigned long long bars[2 * MAX_STAGES];
};

__device__ __forceinline__ void warp_reduce_rec(double& f, int& i, double& a, int& y, bool up) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double f2 = __shfl_xor_sync(0xffffffffu, f, o);
        int i2 = __shfl_xor_sync(0xffffffffu, i, o);
        double a2 = __shfl_xor_sync(0xffffffffu, a, o);
        int y2 = __shfl_xor_sync(0xffffffffu, y, o);
        bool take = up ? better_up(f2, i2, f, i) : better_low(f2, i2, f, i);
        if (take) { f = f2; i = i2; a = a2; y = y2; }
    }
}

// Reduce per-thread (f, i, a, y) records of both selections over the NT consumer
// threads; every consumer thread returns with the CTA-wide result in sh.
__device__ __forceinline__ void cta_reduce(Shared& sh, double fu, int iu, double au, int yu,
                                           double fl, int il, double al, int yl) {
    const int t = threadIdx.x, w = t >> 5, lane = t & 31;
    warp_reduce_rec(fu, iu, au, yu, true);
    warp_reduce_rec(fl, il, al, yl, false);
    if (lane == 0) {
        sh.red_f[0][w] = fu; sh.red_i[0][w] = iu; sh.red_a[0][w] = au; sh.red_y[0][w] = yu;
        sh.red_f[1][w] = fl; sh.red_i[1][w] = il; sh.red_a[1][w] = al; sh.red_y[1][w] = yl;
    }
    bar_consumers();
    if (t == 0) {
        for (int k = 1; k < NWC; ++k) {
            if (better_up(sh.red_f[0][k], sh.red_i[0][k], sh.red_f[0][0], sh.red_i[0][0])) {
                sh.red_f[0][0] = sh.red_f[0][k]; sh.red_i[0][0] = sh.red_i[0][k];
                sh.red_a[0][0] = sh.red_a[0][k]; sh.red_y[0][0] = sh.red_y[0][k];
            }
            if (better_low(sh.red_f[1][k], sh.red_i[1][k], sh.red_f[1][0], sh.red_i[1][0])) {
                sh.red_f[1][0] = sh.red_f[1][k]; sh.red_i[1][0] = sh.red_i[1][k];
                sh.red_a[1][0] = sh.red_a[1][k]; sh.red_y[1][0] = sh.red_y[1][k];
            }
        }
    }
    bar_consumers();
}

// ------------------------------------------------------------------ the kernel
template <int KERNEL, int RPT>
__global__ void __launch_bounds__(NTHREADS, 1) smo_persistent(const Params P) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Shared& sh = *reinterpret_cast<Shared*>(smem_raw);
    size_t off = (sizeof(Shared) + 127) & ~size_t(127);
    double* piv_u = reinterpret_cast<double*>(smem_raw + off); off += (size_t)P.d_pad * 8;
    double* piv_l = reinterpret_cast<double*>(smem_raw + off); off += (size_t)P.d_pad * 8;
    double* f_s = reinterpret_cast<double*>(smem_raw + off); off += (size_t)P.state_cap * 8;
    double* a_s = reinterpret_cast<double*>(smem_raw + off); off += (size_t)P.state_cap * 8;
    uint8_t* fl_s = smem_raw + off; off += (size_t)P.state_cap;
    off = (off + 127) & ~size_t(127);
    float* ring = reinterpret_cast<float*>(smem_raw + off);
    const int stage_floats = P.kc * P.rt;
    uint64_t* full = reinterpret_cast<uint64_t*>(sh.bars);
    uint64_t* empty = full + MAX_STAGES;

    const int t = threadIdx.x;
    const int rank = P.rank_base + blockIdx.x / P.ctas_per_rank;
    const int cta = blockIdx.x % P.ctas_per_rank;
    const int g_total = P.world * P.ctas_per_rank;
    const int gcta = rank * P.ctas_per_rank + cta;
    const int n_r = P.n_rows[rank];
    const int r0 = (int)(((long long)n_r * cta) / P.ctas_per_rank);
    const int r1 = (int)(((long long)n_r * (cta + 1)) / P.ctas_per_rank);
    const int R = r1 - r0;                                   // rows owned by this CTA
    const long long gbase = P.row_off[rank] + r0;            // global index of local row 0
    const int n_tiles = (R + P.rt - 1) / P.rt;
    const float* xcta = P.xblk[rank] + (long long)cta * P.cta_stride;
    Mailbox* my_mb = P.mbox[rank];
    Ctl* ctl = P.ctl[rank];

    if (t == 0) {
        sh.stop = 0; sh.producer_done = 0; sh.issued = 0; sh.timeout = 0;
        for (int s = 0; s < P.stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NWC); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // load the CTA's state into shared memory
    for (int j = t; j < R; j += NTHREADS) {
        f_s[j] = P.f[rank][r0 + j];
        a_s[j] = P.alpha[rank][r0 + j];
        fl_s[j] = P.flags[rank][r0 + j];
    }
    __syncthreads();

    // ================================================================ producer warp
    if (t >= NT) {
        if (t == NT && n_tiles > 0) {
            unsigned int s = 0;
            int tile = 0, chunk = 0;
            for (;;) {
                const int slot = s % P.stages;
                const unsigned int round = s / P.stages;
                if (s >= (unsigned)P.stages) {
                    while (!mbar_try_wait(&empty[slot], (round - 1) & 1)) {
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
                if (++chunk == P.n_chunks) { chunk = 0; if (++tile == n_tiles) tile = 0; }
            }
        }
        if (t == NT) { __threadfence_block(); sh.producer_done = 1; }
        return;
    }

    // ================================================================ consumers
    long long it = ctl->it;            // read by every CTA; written only at kernel end
    long long seq = ctl->seq;
    const long long it_start = it;
    unsigned int consumed = 0;
    const double C = P.C;

    // ---- publish this CTA's candidate record for exchange `seq + 1`
    auto publish = [&](double fu, int ju, double fl, int jl) {
        // (ju, jl are local row indices or INT_MAX)
        cta_reduce(sh, fu, ju, 0.0, 0, fl, jl, 0.0, 0);
        if (t == 0) {
            Partial p;
            const int lu = sh.red_i[0][0], ll = sh.red_i[1][0];
            p.f_up = sh.red_f[0][0];
            p.f_low = sh.red_f[1][0];
            p.i_up = (lu == INT_MAX) ? -1 : (int)(gbase + lu);
            p.i_low = (ll == INT_MAX) ? -1 : (int)(gbase + ll);
            p.a_up = (lu == INT_MAX) ? 0.0 : a_s[lu];
            p.a_low = (ll == INT_MAX) ? 0.0 : a_s[ll];
            p.y_up = (lu == INT_MAX) ? 0 : ((fl_s[lu] & FL_POS) ? 1 : -1);
            p.y_low = (ll == INT_MAX) ? 0 : ((fl_s[ll] & FL_POS) ? 1 : -1);
            const int parity = (int)((seq + 1) & 1);
            for (int r = 0; r < P.world; ++r) mbox_parts(P.mbox[r], parity, g_total)[gcta] = p;
            __threadfence_system();
            for (int r = 0; r < P.world; ++r) atomicAdd_system(&P.mbox[r]->count, 1ull);
        }
        ++seq;
    };

    // ---- initial selection from the current state (no update)
    {
        double fu = __longlong_as_double(0x7ff0000000000000ll), fl = -fu;
        int ju = INT_MAX, jl = INT_MAX;
        for (int j = t; j < R; j += NT) {
            const uint8_t g = fl_s[j];
            const double fj = f_s[j];
            if ((g & FL_UP) && better_up(fj, j, fu, ju)) { fu = fj; ju = j; }
            if ((g & FL_LOW) && better_low(fj, j, fl, jl)) { fl = fj; jl = j; }
        }
        publish(fu, ju, fl, jl);
    }

    int final_state = ST_RUNNING;
    for (;;) {
        // ================= wait for exchange `seq`, then combine
        if (t == 0) {
            const unsigned long long target = (unsigned long long)seq * g_total;
            long long t0 = 0;
            unsigned int spins = 0;
            while (ld_acquire_sys(&my_mb->count) < target) {
                if ((++spins & 1023u) == 0) {
                    const long long now = globaltimer();
                    if (t0 == 0) t0 = now;
                    else if (now - t0 > P.timeout_ns) { sh.timeout = 1; break; }
                }
            }
            __threadfence();
        }
        bar_consumers();
        {
            const Partial* parts = mbox_parts(my_mb, (int)(seq & 1), g_total);
            double fu = __longlong_as_double(0x7ff0000000000000ll), fl = -fu, au = 0.0, al = 0.0;
            int iu = INT_MAX, il = INT_MAX, yu = 0, yl = 0;
            if (!sh.timeout) {
                for (int g = t; g < g_total; g += NT) {
                    const double pfu = __ldcg(&parts[g].f_up), pfl = __ldcg(&parts[g].f_low);
                    const int piu = __ldcg(&parts[g].i_up), pil = __ldcg(&parts[g].i_low);
                    if (piu >= 0 && better_up(pfu, piu, fu, iu)) {
                        fu = pfu; iu = piu; au = __ldcg(&parts[g].a_up); yu = __ldcg(&parts[g].y_up);
                    }
                    if (pil >= 0 && better_low(pfl, pil, fl, il)) {
                        fl = pfl; il = pil; al = __ldcg(&parts[g].a_low); yl = __ldcg(&parts[g].y_low);
                    }
                }
            }
            cta_reduce(sh, fu, iu, au, yu, fl, il, al, yl);
        }
        if (t == 0) {
            int dec = ST_RUNNING;
            const int u = sh.red_i[0][0], l = sh.red_i[1][0];
            if (sh.timeout) dec = ST_TIMEOUT;
            else if (u == INT_MAX || l == INT_MAX) dec = ST_CONVERGED;
            else if (sh.red_f[1][0] - sh.red_f[0][0] <= 2.0 * P.tol) dec = ST_CONVERGED;
            else if (it == P.max_iter) dec = ST_MAXITER;
            else if (P.iter_limit > 0 && it - it_start == P.iter_limit) dec = ST_LIMIT;
            sh.decision = dec;
            sh.u = u; sh.l = l;
            sh.f_up = sh.red_f[0][0]; sh.f_low = sh.red_f[1][0];
            sh.a_up = sh.red_a[0][0]; sh.a_low = sh.red_a[1][0];
            sh.y_up = sh.red_y[0][0]; sh.y_low = sh.red_y[1][0];
        }
        bar_consumers();
        if (sh.decision != ST_RUNNING) { final_state = sh.decision; break; }

        // ================= pair update (a2): gather x_up, x_low; eta; clipped step
        const int u = sh.u, l = sh.l;
        for (int k = t; k < P.d_pad; k += NT) {
            piv_u[k] = (k < P.d) ? (double)P.xr[(long long)u * P.d + k] : 0.0;
            piv_l[k] = (k < P.d) ? (double)P.xr[(long long)l * P.d + k] : 0.0;
        }
        bar_consumers();
        if (t == 0) {
            double Kuu, Kll, Kul;
            if (KERNEL == 1) {
                double acc = 0.0;
                for (int k = 0; k < P.d; ++k) { const double dv = piv_u[k] - piv_l[k]; acc = fma(dv, dv, acc); }
                Kuu = 1.0; Kll = 1.0;
                Kul = (u == l) ? 1.0 : svmexp::exp_cr(-(P.gamma * acc));
            } else {
                double s_uu = 0.0, s_ll = 0.0, s_ul = 0.0;
                for (int k = 0; k < P.d; ++k) {
                    s_uu = fma(piv_u[k], piv_u[k], s_uu);
                    s_ll = fma(piv_l[k], piv_l[k], s_ll);
                    s_ul = fma(piv_u[k], piv_l[k], s_ul);
                }
                Kuu = s_uu; Kll = s_ll; Kul = s_ul;
            }
            const double eta = Kuu + Kll - 2.0 * Kul;
            const double gap = sh.f_low - sh.f_up;
            const double yu = (double)sh.y_up, yl = (double)sh.y_low;
            const double au = sh.a_up, al = sh.a_low;
            const double tu = (sh.y_up == 1) ? C - au : au;
            const double tl = (sh.y_low == 1) ? al : C - al;
            double tt = gap / (eta > 1e-12 ? eta : 1e-12);
            if (tu < tt) tt = tu;
            if (tl < tt) tt = tl;
            const double au2 = (tt == tu) ? (sh.y_up == 1 ? C : 0.0) : au + yu * tt;
            const double al2 = (tt == tl) ? (sh.y_low == 1 ? 0.0 : C) : al - yl * tt;
            sh.cu = yu * (au2 - au);
            sh.cl = yl * (al2 - al);
            sh.au_new = au2; sh.al_new = al2;
            // owner CTA updates its shared-memory state for the two rows
            const long long lu = (long long)u - gbase, ll = (long long)l - gbase;
            if (lu >= 0 && lu < R) { a_s[lu] = au2; fl_s[lu] = flags_of(sh.y_up, au2, C); }
            if (ll >= 0 && ll < R) { a_s[ll] = al2; fl_s[ll] = flags_of(sh.y_low, al2, C); }
            if (P.trace && rank == 0 && cta == 0 && it < P.trace_cap) {
                P.trace[2 * it] = u; P.trace[2 * it + 1] = l;
            }
            if (P.progress && rank == 0 && cta == 0 && P.check_interval > 0 &&
                (it % P.check_interval) == 0) {
                *(volatile unsigned long long*)P.progress = (unsigned long long)it;
            }
        }
        bar_consumers();
        const double cu = sh.cu, cl = sh.cl;

        // ================= row pass (a3-a5)
        double bfu = __longlong_as_double(0x7ff0000000000000ll), bfl = -bfu;
        int bju = INT_MAX, bjl = INT_MAX;
        for (int tile = 0; tile < n_tiles; ++tile) {
            const int rows_t = min(P.rt, R - tile * P.rt);
            const int rp = (rows_t + 3) & ~3;
            const bool active = t * RPT < rows_t;
            double du[RPT], dl[RPT];
#pragma unroll
            for (int q = 0; q < RPT; ++q) { du[q] = 0.0; dl[q] = 0.0; }
            for (int ch = 0; ch < P.n_chunks; ++ch) {
                const int slot = consumed % P.stages;
                mbar_wait(&full[slot], (consumed / P.stages) & 1);
                const float* st = ring + (size_t)slot * stage_floats;
                const int k0 = ch * P.kc;
                if (active) {
                    if (RPT == 4) {
                        const float4* sp = reinterpret_cast<const float4*>(st) + t;
                        const int ld4 = rp >> 2;
#pragma unroll 4
                        for (int kk = 0; kk < P.kc; ++kk) {
                            const float4 v = sp[kk * ld4];
                            const double xu = piv_u[k0 + kk], xl = piv_l[k0 + kk];
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
                    } else {
                        const float* sp = st + t;
#pragma unroll 8
                        for (int kk = 0; kk < P.kc; ++kk) {
                            const double x0 = sp[kk * rp];
                            const double xu = piv_u[k0 + kk], xl = piv_l[k0 + kk];
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
                if ((t & 31) == 0) mbar_arrive(&empty[slot]);
                ++consumed;
            }
            if (active) {
#pragma unroll
                for (int q = 0; q < RPT; ++q) {
                    const int j = tile * P.rt + t * RPT + q;
                    if (j < R) {
                        const long long jg = gbase + j;
                        double ku, kl;
                        if (KERNEL == 1) {
                            ku = (jg == u) ? 1.0 : svmexp::exp_cr(-(P.gamma * du[q]));
                            kl = (jg == l) ? 1.0 : svmexp::exp_cr(-(P.gamma * dl[q]));
                        } else {
                            ku = du[q]; kl = dl[q];
                        }
                        const double fj = fma(cl, kl, fma(cu, ku, f_s[j]));
                        f_s[j] = fj;
                        const uint8_t g = fl_s[j];
                        if ((g & FL_UP) && better_up(fj, j, bfu, bju)) { bfu = fj; bju = j; }
                        if ((g & FL_LOW) && better_low(fj, j, bfl, bjl)) { bfl = fj; bjl = j; }
                    }
                }
            }
        }
        ++it;
        publish(bfu, bju, bfl, bjl);
    }

    // ================= shutdown: stop the producer, drain issued stages
    if (t == 0) {
        sh.stop = 1;
        __threadfence_block();
        for (;;) {
            const int done = sh.producer_done;
            const unsigned int iss = sh.issued;
            if (consumed < iss) {
                const int slot = consumed % P.stages;
                mbar_wait(&full[slot], (consumed / P.stages) & 1);
                for (int w = 0; w < NWC; ++w) mbar_arrive(&empty[slot]);
                ++consumed;
            } else if (done) {
                break;
            }
        }
    }
    bar_consumers();
    for (int j = t; j < R; j += NT) {
        P.f[rank][r0 + j] = f_s[j];
        P.alpha[rank][r0 + j] = a_s[j];
        P.flags[rank][r0 + j] = fl_s[j];
    }
    if (t == 0 && cta == 0) {
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
