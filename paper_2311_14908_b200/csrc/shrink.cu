// shrink.cu -- window shrinking around the persistent solver (
// DESIGN.md reading R29, svm_params.shrink_window).
//
// The solve runs in windows of H updates.  At a window start (every row active):
//   k_sel_all        the pair and its gap over all rows (the oracle's selection, ties to
//                    the lowest index) -> the stopping test on the host
//   k_shrink_mark    rows that cannot form a violating pair are set aside for the window:
//                    i in I_up only with f_i > b_low, i in I_low only with f_i < b_up
//   k_compact_*      the active rows, in ascending order, gathered into a sub-problem
//                    (row-major X, y, alpha, f)
// then the persistent solver runs on the sub-problem (warm start, at most H updates,
// ends early when the active rows' gap reaches 2 tol), its alpha and f are scattered back,
// and k_replay applies the window's updates to the rows set aside:
//   f_i <- fma(c_l, K(x_l, x_i), fma(c_u, K(x_u, x_i), f_i))   for every update, in order,
// with the row pass's arithmetic (R13 recurrence, correctly rounded exp) -- so every f is
// the exact incremental value, as if no row had been set aside; only the selection inside
// a window differs from the plain solve.  The rows set aside are read once per window
// (compute-bound replay) instead of streamed from HBM every iteration.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "svm_internal.h"

using namespace svmk;

namespace svmint {

constexpr int SEL_BLOCKS = 296;
constexpr int SEL_THREADS = 256;

__device__ __forceinline__ bool in_up(int8_t y, double a, double C) { return (y > 0 && a < C) || (y < 0 && a > 0.0); }
__device__ __forceinline__ bool in_low(int8_t y, double a, double C) { return (y > 0 && a > 0.0) || (y < 0 && a < C); }

// per block: the lexicographic (f, index) minimum over I_up and maximum over I_low (as the
// minimum of the complemented order-preserving key), then one block reduces the blocks
struct SelPart { unsigned long long ku, kl; long long iu, il; };

__global__ void k_sel_part(const double* __restrict__ f, const int8_t* __restrict__ y,
                           const double* __restrict__ alpha, long long n, double C, SelPart* __restrict__ part) {
    __shared__ SelPart sp[SEL_THREADS / 32];
    unsigned long long ku = ~0ull, kl = ~0ull;
    long long iu = LLONG_MAX, il = LLONG_MAX;
    for (long long j = (long long)blockIdx.x * SEL_THREADS + threadIdx.x; j < n; j += (long long)gridDim.x * SEL_THREADS) {
        const double a = alpha[j];
        const int8_t yy = y[j];
        const unsigned long long k = fkey(f[j]);
        if (in_up(yy, a, C) && (k < ku || (k == ku && j < iu))) { ku = k; iu = j; }
        if (in_low(yy, a, C) && (~k < kl || (~k == kl && j < il))) { kl = ~k; il = j; }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long ku2 = __shfl_xor_sync(0xffffffffu, ku, o), kl2 = __shfl_xor_sync(0xffffffffu, kl, o);
        const long long iu2 = __shfl_xor_sync(0xffffffffu, iu, o), il2 = __shfl_xor_sync(0xffffffffu, il, o);
        if (ku2 < ku || (ku2 == ku && iu2 < iu)) { ku = ku2; iu = iu2; }
        if (kl2 < kl || (kl2 == kl && il2 < il)) { kl = kl2; il = il2; }
    }
    if ((threadIdx.x & 31) == 0) sp[threadIdx.x >> 5] = SelPart{ku, kl, iu, il};
    __syncthreads();
    if (threadIdx.x == 0) {
        SelPart b = sp[0];
        for (int w = 1; w < SEL_THREADS / 32; ++w) {
            const SelPart& c = sp[w];
            if (c.ku < b.ku || (c.ku == b.ku && c.iu < b.iu)) { b.ku = c.ku; b.iu = c.iu; }
            if (c.kl < b.kl || (c.kl == b.kl && c.il < b.il)) { b.kl = c.kl; b.il = c.il; }
        }
        part[blockIdx.x] = b;
    }
}

// out: {i_up, i_low} (-1 = empty) and {f_up, f_low}
struct SelOut { long long iu, il; double fu, fl; };

__global__ void k_sel_final(const SelPart* __restrict__ part, int nb, const double* __restrict__ f, SelOut* out) {
    if (threadIdx.x != 0) return;
    SelPart b = part[0];
    for (int k = 1; k < nb; ++k) {
        const SelPart& c = part[k];
        if (c.ku < b.ku || (c.ku == b.ku && c.iu < b.iu)) { b.ku = c.ku; b.iu = c.iu; }
        if (c.kl < b.kl || (c.kl == b.kl && c.il < b.il)) { b.kl = c.kl; b.il = c.il; }
    }
    SelOut o;
    o.iu = b.iu == LLONG_MAX ? -1 : b.iu;
    o.il = b.il == LLONG_MAX ? -1 : b.il;
    o.fu = o.iu >= 0 ? f[o.iu] : 0.0;
    o.fl = o.il >= 0 ? f[o.il] : 0.0;
    *out = o;
}

// active flags + per-block counts (blocks of CH rows, for the stable compaction)
constexpr int CM_TILE = 256;

__global__ void k_shrink_mark(const double* __restrict__ f, const int8_t* __restrict__ y,
                              const double* __restrict__ alpha, long long n, double C, double b_up,
                              double b_low, long long chunk, uint8_t* __restrict__ act,
                              unsigned long long* __restrict__ cnt) {
    __shared__ unsigned int wc[CM_TILE / 32];
    const long long lo = (long long)blockIdx.x * chunk;
    const long long hi = lo + chunk < n ? lo + chunk : n;
    unsigned int c = 0;
    for (long long j = lo + threadIdx.x; j < hi; j += CM_TILE) {
        const double a = alpha[j];
        const int8_t yy = y[j];
        const bool up = in_up(yy, a, C), low = in_low(yy, a, C);
        const double fj = f[j];
        const bool out = (up && !low && fj > b_low) || (low && !up && fj < b_up);
        act[j] = out ? 0 : 1;
        c += out ? 0u : 1u;
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) wc[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < CM_TILE / 32; ++w) s += wc[w];
        cnt[blockIdx.x] = s;
    }
}

// exclusive scans of the active counts (cnt) and of the inactive counts (chunk sizes -
// cnt) in one block; totals at [nb]
__global__ void k_shrink_scan(unsigned long long* __restrict__ cnt, unsigned long long* __restrict__ icnt,
                              int nb, long long n, long long chunk) {
    if (threadIdx.x != 0) return;
    unsigned long long s = 0, si = 0;
    for (int b = 0; b < nb; ++b) {
        const long long lo = (long long)b * chunk;
        const long long sz = (lo + chunk < n ? lo + chunk : n) - lo;
        const unsigned long long c = cnt[b];
        cnt[b] = s; s += c;
        icnt[b] = si; si += (unsigned long long)sz - c;
    }
    cnt[nb] = s;
    icnt[nb] = si;
}

// stable compaction: the active rows' global indices (idx) and the rows set aside (oidx)
__global__ void k_shrink_lists(const uint8_t* __restrict__ act, long long n, long long chunk,
                               const unsigned long long* __restrict__ cnt, const unsigned long long* __restrict__ icnt,
                               long long* __restrict__ idx, long long* __restrict__ oidx) {
    __shared__ unsigned int wc[CM_TILE / 32];
    const long long lo = (long long)blockIdx.x * chunk;
    const long long hi = lo + chunk < n ? lo + chunk : n;
    long long pos = (long long)cnt[blockIdx.x], ipos = (long long)icnt[blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (long long t0 = lo; t0 < hi; t0 += CM_TILE) {
        const long long j = t0 + threadIdx.x;
        const bool valid = j < hi;
        const bool a = valid && act[j];
        const unsigned m = __ballot_sync(0xffffffffu, a);
        if (lane == 0) wc[warp] = __popc(m);
        __syncthreads();
        unsigned int before = 0, total = 0;
        for (int w = 0; w < CM_TILE / 32; ++w) { if (w < warp) before += wc[w]; total += wc[w]; }
        const unsigned int r = before + __popc(m & ((1u << lane) - 1u));
        const long long nvalid = (hi - t0) < CM_TILE ? (hi - t0) : CM_TILE;
        if (a) idx[pos + r] = j;
        else if (valid) oidx[ipos + (threadIdx.x - r)] = j;     // threadIdx.x - r inactive before j in the tile
        pos += total;
        ipos += nvalid - total;
        __syncthreads();
    }
}

// gather the sub-problem (rows idx) and scatter its state back
__global__ void k_gather_rows(const float* __restrict__ X, long long d, const long long* __restrict__ idx,
                              long long na, float* __restrict__ Xa) {
    const int lane = threadIdx.x & 31;
    for (long long r = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < na;
         r += ((long long)gridDim.x * blockDim.x) >> 5) {
        const float* src = X + idx[r] * d;
        float* dst = Xa + r * d;
        for (long long k = lane; k < d; k += 32) dst[k] = src[k];
    }
}
__global__ void k_gather_state(const long long* __restrict__ idx, long long na, const int8_t* __restrict__ y,
                               const double* __restrict__ alpha, const double* __restrict__ f,
                               int8_t* __restrict__ ya, double* __restrict__ aa, double* __restrict__ fa) {
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < na; r += (long long)gridDim.x * blockDim.x) {
        const long long j = idx[r];
        ya[r] = y[j]; aa[r] = alpha[j]; fa[r] = f[j];
    }
}
__global__ void k_scatter_state(const long long* __restrict__ idx, long long na, const double* __restrict__ aa,
                                const double* __restrict__ fa, double* __restrict__ alpha, double* __restrict__ f) {
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < na; r += (long long)gridDim.x * blockDim.x) {
        const long long j = idx[r];
        alpha[j] = aa[r]; f[j] = fa[r];
    }
}
// the window's pair trace in global indices (and the caller's host trace)
__global__ void k_map_trace(const long long* __restrict__ tr, long long k, const long long* __restrict__ idx,
                            long long* __restrict__ tg) {
    for (long long h = (long long)blockIdx.x * blockDim.x + threadIdx.x; h < 2 * k; h += (long long)gridDim.x * blockDim.x)
        tg[h] = idx[tr[h]];
}

// ---- replay of the window's updates on the rows set aside.  A CTA owns RB rows; the
// window's steps are taken RS at a time (2 RS pivot rows: u_h, l_h); the features in
// chunks of DC.  Thread (warp w, lane): rows lane + 32 q (q < 4), pivots 4 w + p (p < 4),
// so a warp's pivot loads are broadcasts and its row loads consecutive.  The distance of
// every (row, pivot) pair is the R13 recurrence in ascending k (chunks in order), K by the
// correctly rounded exp; then RB threads apply the RS steps to their row's f in order.
constexpr int RB = 128, RS = 16, RP = 2 * RS, DC = 64, RT = 256;
constexpr size_t REPLAY_SMEM = sizeof(double) * ((size_t)DC * RB + DC * RP + RP * (RB + 1) + 96);

template <int KERNEL>
__global__ void __launch_bounds__(RT, 1)
k_replay(const float* __restrict__ X, int d, const long long* __restrict__ rows, long long nr,
         const long long* __restrict__ tg, const double* __restrict__ hist, long long k,
         double gamma, double* __restrict__ f) {
    extern __shared__ __align__(16) double rsm[];
    double (*xs)[RB] = reinterpret_cast<double (*)[RB]>(rsm);                        // [DC][RB] 64 KB
    double (*ps)[RP] = reinterpret_cast<double (*)[RP]>(rsm + DC * RB);              // [DC][RP] 16 KB
    double (*kv)[RB + 1] = reinterpret_cast<double (*)[RB + 1]>(rsm + DC * RB + DC * RP);  // [RP][RB+1] 33 KB
    double* tab = rsm + DC * RB + DC * RP + RP * (RB + 1);
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int e = t; e < svmexp::EXP_TABLE_DOUBLES; e += RT) tab[e] = svmexp::table_entry(e);
    const svmexp::PtrTab T{tab};
    const long long r0 = (long long)blockIdx.x * RB;
    const int nrows = (int)((nr - r0) < RB ? (nr - r0) : RB);
    double fr = 0.0;
    if (t < nrows) fr = f[rows[r0 + t]];
    for (long long h0 = 0; h0 < k; h0 += RS) {
        const int ns = (int)((k - h0) < RS ? (k - h0) : RS);
        double acc[4][4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int p = 0; p < 4; ++p) acc[q][p] = 0.0;
        for (int k0 = 0; k0 < d; k0 += DC) {
            __syncthreads();
            // stage the rows and the pivots (fp64, feature-major), zero padded
            for (int e = t; e < DC * RB; e += RT) {
                const int rr = e / DC, kk = e - rr * DC;
                float v = 0.0f;
                if (rr < nrows && k0 + kk < d) v = X[rows[r0 + rr] * (long long)d + k0 + kk];
                xs[kk][rr] = (double)v;
            }
            for (int e = t; e < DC * RP; e += RT) {
                const int pp = e / DC, kk = e - pp * DC;
                float v = 0.0f;
                if ((pp >> 1) < ns && k0 + kk < d) v = X[tg[2 * (h0 + (pp >> 1)) + (pp & 1)] * (long long)d + k0 + kk];
                ps[kk][pp] = (double)v;
            }
            __syncthreads();
#pragma unroll 4
            for (int kk = 0; kk < DC; ++kk) {
                double xv[4], pv[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) xv[q] = xs[kk][lane + 32 * q];
#pragma unroll
                for (int p = 0; p < 4; ++p) pv[p] = ps[kk][4 * warp + p];
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        if (KERNEL == 1) { const double e = xv[q] - pv[p]; acc[q][p] = fma(e, e, acc[q][p]); }
                        else acc[q][p] = fma(xv[q], pv[p], acc[q][p]);
                    }
            }
        }
        // kernel values (a row set aside is never a pivot: K_ii does not occur)
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                double kvv = acc[q][p];
                if (KERNEL == 1) kvv = svmexp::exp_cr_t(-(gamma * acc[q][p]), T);
                kv[4 * warp + p][lane + 32 * q] = kvv;
            }
        __syncthreads();
        if (t < nrows) {
            for (int s = 0; s < ns; ++s) {
                const double cu = hist[2 * (h0 + s)], cl = hist[2 * (h0 + s) + 1];
                fr = fma(cl, kv[2 * s + 1][t], fma(cu, kv[2 * s][t], fr));
            }
        }
    }
    if (t < nrows) f[rows[r0 + t]] = fr;
}

// Replay, rows resident (d_pad <= 256, the HBM-bound configs): a CTA owns R2 = 64 rows,
// held in shared memory as fp64 for the whole window; the window's steps are taken 32 at a
// time (64 pivot rows, staged per feature chunk).  Thread (warp w, lane): rows lane and
// lane + 32, pivots 8 w .. 8 w + 7 -- 16 independent R13 chains, 2 row loads and 4
// broadcast pivot loads per feature.  Same arithmetic as k_replay.
constexpr int R2 = 64, S2 = 32, P2 = 2 * S2, D2 = 64, D2MAX = 256;
constexpr size_t REPLAY2_SMEM = sizeof(double) * ((size_t)D2MAX * R2 + (size_t)D2 * P2 + (size_t)P2 * (R2 + 1) + 96);

template <int KERNEL>
__global__ void __launch_bounds__(RT, 1)
k_replay_res(const float* __restrict__ X, int d, const long long* __restrict__ rows, long long nr,
             const long long* __restrict__ tg, const double* __restrict__ hist, long long k,
             double gamma, double* __restrict__ f) {
    extern __shared__ __align__(16) double rsm[];
    const int dpad = (d + D2 - 1) / D2 * D2;
    double (*xs)[R2] = reinterpret_cast<double (*)[R2]>(rsm);                                 // [dpad][R2]
    double (*ps)[P2] = reinterpret_cast<double (*)[P2]>(rsm + (size_t)D2MAX * R2);             // [D2][P2]
    double (*kv)[R2 + 1] = reinterpret_cast<double (*)[R2 + 1]>(rsm + (size_t)D2MAX * R2 + D2 * P2);  // [P2][R2+1]
    double* tab = rsm + (size_t)D2MAX * R2 + D2 * P2 + P2 * (R2 + 1);
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int e = t; e < svmexp::EXP_TABLE_DOUBLES; e += RT) tab[e] = svmexp::table_entry(e);
    const svmexp::PtrTab T{tab};
    const long long r0 = (long long)blockIdx.x * R2;
    const int nrows = (int)((nr - r0) < R2 ? (nr - r0) : R2);
    // the CTA's rows, once: fp32 -> fp64, feature-major, zero padded
    for (int e = t; e < dpad * R2; e += RT) {
        const int rr = e / dpad, kk = e - rr * dpad;
        float v = 0.0f;
        if (rr < nrows && kk < d) v = X[rows[r0 + rr] * (long long)d + kk];
        xs[kk][rr] = (double)v;
    }
    double fr = 0.0;
    if (t < nrows) fr = f[rows[r0 + t]];
    for (long long h0 = 0; h0 < k; h0 += S2) {
        const int ns = (int)((k - h0) < S2 ? (k - h0) : S2);
        double acc[2][8];
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int p = 0; p < 8; ++p) acc[q][p] = 0.0;
        for (int k0 = 0; k0 < dpad; k0 += D2) {
            __syncthreads();
            for (int e = t; e < D2 * P2; e += RT) {
                const int pp = e / D2, kk = e - pp * D2;
                float v = 0.0f;
                if ((pp >> 1) < ns && k0 + kk < d) v = X[tg[2 * (h0 + (pp >> 1)) + (pp & 1)] * (long long)d + k0 + kk];
                ps[kk][pp] = (double)v;
            }
            __syncthreads();
#pragma unroll 2
            for (int kk = 0; kk < D2; ++kk) {
                const double x0 = xs[k0 + kk][lane], x1 = xs[k0 + kk][lane + 32];
                const double2* pr = reinterpret_cast<const double2*>(&ps[kk][8 * warp]);
                double pv[8];
#pragma unroll
                for (int p = 0; p < 4; ++p) { const double2 v2 = pr[p]; pv[2 * p] = v2.x; pv[2 * p + 1] = v2.y; }
#pragma unroll
                for (int p = 0; p < 8; ++p) {
                    if (KERNEL == 1) {
                        const double e0 = x0 - pv[p]; acc[0][p] = fma(e0, e0, acc[0][p]);
                        const double e1 = x1 - pv[p]; acc[1][p] = fma(e1, e1, acc[1][p]);
                    } else {
                        acc[0][p] = fma(x0, pv[p], acc[0][p]);
                        acc[1][p] = fma(x1, pv[p], acc[1][p]);
                    }
                }
            }
        }
        // kernel values: all fast phases first (independent), the rare slow ones after
        bool safe[2][8];
        bool all_safe = true;
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int p = 0; p < 8; ++p) {
                double kvv = acc[q][p];
                safe[q][p] = true;
                if (KERNEL == 1) { kvv = svmexp::exp_cr_fast(-(gamma * acc[q][p]), T, safe[q][p]); all_safe = all_safe && safe[q][p]; }
                kv[8 * warp + p][lane + 32 * q] = kvv;
            }
        if (KERNEL == 1 && !all_safe) {
#pragma unroll
            for (int q = 0; q < 2; ++q)
#pragma unroll
                for (int p = 0; p < 8; ++p)
                    if (!safe[q][p]) kv[8 * warp + p][lane + 32 * q] = svmexp::exp_cr_slow(-(gamma * acc[q][p]), T);
        }
        __syncthreads();
        if (t < nrows) {
            for (int s2 = 0; s2 < ns; ++s2) {
                const double cu = hist[2 * (h0 + s2)], cl = hist[2 * (h0 + s2) + 1];
                fr = fma(cl, kv[2 * s2 + 1][t], fma(cu, kv[2 * s2][t], fr));
            }
        }
    }
    if (t < nrows) f[rows[r0 + t]] = fr;
}

}  // namespace svmint

using namespace svmint;

namespace svmint {

// alpha0 / f0 or alpha = 0, f = -y
__global__ void k_shrink_init(const int8_t* __restrict__ y, long long n, const double* __restrict__ alpha0,
                              const double* __restrict__ f0, double* __restrict__ alpha, double* __restrict__ f) {
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
        alpha[j] = alpha0 ? alpha0[j] : 0.0;
        f[j] = f0 ? f0[j] : -(double)y[j];
    }
}

// the shrinking driver (svm_train_ex / svm_train_dev with shrink_window > 0, one rank):
// X, y, alpha (out) device; alpha0 / f0 device (nullable); f_out device (nullable); trace
// host (nullable).
int train_shrink(const float* X, const int8_t* y, long long n, long long d, const svm_params& p,
                 double* alpha, const double* alpha0, const double* f0, double* f_out,
                 long long* trace, long long trace_cap, cudaStream_t st, SolveOut& out) {
    const long long H = p.shrink_window;
    std::vector<void*> owned;
    auto dalloc = [&](void** ptr, size_t bytes) -> int {
        if (cudaMallocAsync(ptr, bytes > 0 ? bytes : 16, st) != cudaSuccess) {
            cudaGetLastError();
            return fail(SVM_ENOMEM, "shrinking: device allocation failed");
        }
        owned.push_back(*ptr);
        return SVM_OK;
    };
    auto release = [&]() { for (void* q : owned) cudaFreeAsync(q, st); owned.clear(); };
    int rc = SVM_OK;
    // every window allocates the sub-problem's blocked copy of X (up to |X|) from the pool:
    // keep all of it cached for the solve (a release at the 2 GiB default threshold would
    // re-map GBs per window -- measured 0.3-0.9 s spikes), restore the threshold after
    cudaMemPool_t pool = nullptr;
    unsigned long long thr_old = 0;
    {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr_old);
            unsigned long long keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        } else {
            pool = nullptr;
        }
        cudaGetLastError();
    }
    struct PoolRestore {
        cudaMemPool_t p; unsigned long long t;
        ~PoolRestore() { if (p) cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &t); }
    } pool_restore{pool, thr_old};
    double* f; double* aa; double* fa; float* Xa; int8_t* ya; uint8_t* act;
    long long *idx, *oidx, *trs, *tg; double* hist; SelPart* part; SelOut* so;
    unsigned long long *cnt, *icnt;
    long long chunk = ((n + 1023) / 1024 + CM_TILE - 1) / CM_TILE * CM_TILE;
    if (chunk < CM_TILE) chunk = CM_TILE;
    const int nb = (int)((n + chunk - 1) / chunk);
    if ((rc = dalloc((void**)&f, (size_t)n * 8)) || (rc = dalloc((void**)&aa, (size_t)n * 8)) ||
        (rc = dalloc((void**)&fa, (size_t)n * 8)) || (rc = dalloc((void**)&Xa, (size_t)n * d * 4)) ||
        (rc = dalloc((void**)&ya, (size_t)n)) || (rc = dalloc((void**)&act, (size_t)n)) ||
        (rc = dalloc((void**)&idx, (size_t)n * 8)) || (rc = dalloc((void**)&oidx, (size_t)n * 8)) ||
        (rc = dalloc((void**)&trs, (size_t)H * 16)) || (rc = dalloc((void**)&tg, (size_t)H * 16)) ||
        (rc = dalloc((void**)&hist, (size_t)H * 16)) || (rc = dalloc((void**)&part, SEL_BLOCKS * sizeof(SelPart))) ||
        (rc = dalloc((void**)&so, sizeof(SelOut))) || (rc = dalloc((void**)&cnt, (size_t)(nb + 1) * 8)) ||
        (rc = dalloc((void**)&icnt, (size_t)(nb + 1) * 8))) { release(); return rc; }
    // state: alpha0 / f0 or alpha = 0, f = -y
    k_shrink_init<<<592, 256, 0, st>>>(y, n, alpha0, f0, alpha, f);
    counted();
    cudaEvent_t e0, e1;
    CKR(cudaEventCreate(&e0));
    CKR(cudaEventCreate(&e1));
    CKR(cudaEventRecord(e0, st));
    long long it = 0;
    long long launches = 0;
    double solve_s = 0.0;
    int state = ST_RUNNING;
    double b_up = 0.0, b_low = 0.0;
    SolveOut so_last;
    long long hits = 0, misses = 0;
    bool plain_rows = false;
    const bool slog = getenv("SVMB200_SHRINK_LOG") != nullptr;     // per-window timing (diagnostic)
    for (;;) {
        // ---- window start: the selection over every row and the stopping test
        k_sel_part<<<SEL_BLOCKS, SEL_THREADS, 0, st>>>(f, y, alpha, n, p.C, part);
        k_sel_final<<<1, 32, 0, st>>>(part, SEL_BLOCKS, f, so);
        counted(2);
        SelOut hs;
        CKR(cudaMemcpyAsync(&hs, so, sizeof(hs), cudaMemcpyDeviceToHost, st));
        CKR(cudaStreamSynchronize(st));
        b_up = hs.fu; b_low = hs.fl;
        if (hs.iu < 0 || hs.il < 0) { state = ST_CONVERGED; break; }
        if (hs.fl - hs.fu <= 2.0 * p.tol) { state = ST_CONVERGED; break; }
        if (it == p.max_iter) { state = ST_MAXITER; break; }
        // ---- the rows set aside for this window, the sub-problem of the active rows
        k_shrink_mark<<<nb, CM_TILE, 0, st>>>(f, y, alpha, n, p.C, hs.fu, hs.fl, chunk, act, cnt);
        k_shrink_scan<<<1, 32, 0, st>>>(cnt, icnt, nb, n, chunk);
        k_shrink_lists<<<nb, CM_TILE, 0, st>>>(act, n, chunk, cnt, icnt, idx, oidx);
        counted(3);
        unsigned long long tot[2];
        CKR(cudaMemcpyAsync(&tot[0], cnt + nb, 8, cudaMemcpyDeviceToHost, st));
        CKR(cudaMemcpyAsync(&tot[1], icnt + nb, 8, cudaMemcpyDeviceToHost, st));
        CKR(cudaStreamSynchronize(st));
        const long long na = (long long)tot[0], ni = (long long)tot[1];
        k_gather_rows<<<1184, 256, 0, st>>>(X, d, idx, na, Xa);
        k_gather_state<<<592, 256, 0, st>>>(idx, na, y, alpha, f, ya, aa, fa);
        counted(2);
        // ---- the window: the persistent solver on the active rows (warm start)
        svm_params q = p;
        const long long remaining = p.max_iter - it;
        q.max_iter = remaining < H ? remaining : H;
        q.iters_per_launch = 0;
        q.cluster = -1;
        q.shrink_window = 0;
        if (q.cache_rows == 0) q.cache_rows = -1;     // (auto cache: decided for the whole problem, off here)
        SolveOut o;
        cudaEvent_t w0 = nullptr, w1 = nullptr, w2 = nullptr;
        if (slog) { cudaEventCreate(&w0); cudaEventCreate(&w1); cudaEventCreate(&w2); cudaEventRecord(w0, st); }
        rc = train_device(Xa, ya, na, d, q, aa, aa, fa, fa, cudaMemcpyDeviceToDevice, nullptr, 0, st, o,
                          trs, hist, H, plain_rows);
        plain_rows = plain_rows || o.plain_rows;      // an fp32-row problem stays one: skip the probes
        if (slog) cudaEventRecord(w1, st);
        if (rc) { release(); return rc; }
        launches += o.launches;
        solve_s += o.seconds_solve;
        hits += o.cache_hits; misses += o.cache_misses;
        const long long kk = o.iterations;
        k_scatter_state<<<592, 256, 0, st>>>(idx, na, aa, fa, alpha, f);
        counted();
        if (kk > 0) {
            k_map_trace<<<64, 256, 0, st>>>(trs, kk, idx, tg);
            counted();
            if (ni > 0) {
                const unsigned grid = (unsigned)((ni + RB - 1) / RB);
                static_assert(svmexp::EXP_TABLE_DOUBLES == 96, "replay table size");
                if (d <= D2MAX && getenv("SVMB200_REPLAY_V1") == nullptr) {
                    const unsigned g2 = (unsigned)((ni + R2 - 1) / R2);
                    if (p.kernel == SVM_RBF) {
                        CKR(cudaFuncSetAttribute((const void*)k_replay_res<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)REPLAY2_SMEM));
                        k_replay_res<1><<<g2, RT, REPLAY2_SMEM, st>>>(X, (int)d, oidx, ni, tg, hist, kk, p.gamma, f);
                    } else {
                        CKR(cudaFuncSetAttribute((const void*)k_replay_res<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)REPLAY2_SMEM));
                        k_replay_res<0><<<g2, RT, REPLAY2_SMEM, st>>>(X, (int)d, oidx, ni, tg, hist, kk, p.gamma, f);
                    }
                } else if (p.kernel == SVM_RBF) {
                    CKR(cudaFuncSetAttribute((const void*)k_replay<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)REPLAY_SMEM));
                    k_replay<1><<<grid, RT, REPLAY_SMEM, st>>>(X, (int)d, oidx, ni, tg, hist, kk, p.gamma, f);
                } else {
                    CKR(cudaFuncSetAttribute((const void*)k_replay<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)REPLAY_SMEM));
                    k_replay<0><<<grid, RT, REPLAY_SMEM, st>>>(X, (int)d, oidx, ni, tg, hist, kk, p.gamma, f);
                }
                counted();
            }
            if (trace && it < trace_cap) {
                const long long nt = (it + kk <= trace_cap ? kk : trace_cap - it);
                CKR(cudaMemcpyAsync(trace + 2 * it, tg, (size_t)nt * 16, cudaMemcpyDeviceToHost, st));
            }
        }
        CKR(cudaGetLastError());
        if (slog) {
            cudaEventRecord(w2, st);
            cudaEventSynchronize(w2);
            float ms_s = 0.f, ms_r = 0.f;
            cudaEventElapsedTime(&ms_s, w0, w1);
            cudaEventElapsedTime(&ms_r, w1, w2);
            fprintf(stderr, "[svmb200 shrink] it=%lld window=%lld active=%lld aside=%lld solve_ms=%.2f replay_ms=%.2f\n",
                    it, kk, na, ni, ms_s, ms_r);
            cudaEventDestroy(w0); cudaEventDestroy(w1); cudaEventDestroy(w2);
        }
        it += kk;
        if (o.state == ST_MAXITER && kk == remaining && remaining < H) {
            // the run's max_iter inside the window: the active rows' selection stands
            state = ST_MAXITER; b_up = o.b_up; b_low = o.b_low;
            break;
        }
        if (o.state != ST_CONVERGED && o.state != ST_MAXITER) { release(); return fail(SVM_ECUDA, "shrinking: window ended in state " + std::to_string(o.state)); }
    }
    if (f_out) CKR(cudaMemcpyAsync(f_out, f, (size_t)n * 8, cudaMemcpyDeviceToDevice, st));
    CKR(cudaEventRecord(e1, st));
    CKR(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    solve_s = ms * 1e-3;                  // the whole windowed solve: selections, compaction, replay
    release();
    CKR(cudaStreamSynchronize(st));
    out = SolveOut();
    out.iterations = it; out.state = state; out.b_up = b_up; out.b_low = b_low;
    out.seconds_solve = solve_s; out.launches = launches;
    out.cache_hits = hits; out.cache_misses = misses;
    return SVM_OK;
}

}  // namespace svmint
