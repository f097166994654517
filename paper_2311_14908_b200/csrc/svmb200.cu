// svmb200.cu -- C ABI (include/svmb200.h) and host driver of the B200 SMO solver.
//
// Stages:
//   a1  stage + shard + init: validate, H2D (host entry points), build the CTA-blocked
//       feature-major copy of each rank's rows (k_build_xblk), init alpha/f/flags
//   a2-a7  the persistent kernel (smo_kernel.cuh), one cooperative launch per
//       `iters_per_launch` iterations (default: the whole solve)
//   a10 finalize: b = -(b_up + b_low)/2, D2H alpha, info
//   a11 predict: predict.cu
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <algorithm>

#include "../../include/svmb200.h"
#include "smo_kernel.cuh"
#include "smo_bincl.cuh"
#include "svm_internal.h"

using namespace svmk;

namespace svmint {
static_assert(sizeof(svm_params) == 88, "svm_params layout (binding and tests assume 88 bytes)");

thread_local std::string g_err;
thread_local long long g_launches = 0;
thread_local std::string g_plan;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

// ------------------------------------------------------------------ prep kernels
// Blocked feature-major copy of one rank's rows: CTA c, tile t, feature k, row r ->
// xblk[c * cta_stride + t * d_pad * rt + k * rows_pad4(t) + r]  (zero padded).
__global__ void k_build_xblk(const float* __restrict__ X, long long n_r, int d, int d_pad,
                             int G, int rt, long long cta_stride, float* __restrict__ xblk) {
    const int c = blockIdx.y;
    const long long r0 = (n_r * c) / G, r1 = (n_r * (c + 1)) / G;
    const long long R = r1 - r0;
    const long long total = R * d_pad;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long k = e / R;
        const long long j = e - k * R;
        const long long tile = j / rt, rin = j - tile * rt;
        const long long rows_t = (R - tile * rt) < rt ? (R - tile * rt) : rt;
        const long long rp = (rows_t + 3) & ~3ll;
        const float v = (k < d) ? X[(r0 + j) * d + k] : 0.0f;
        xblk[(long long)c * cta_stride + tile * (long long)d_pad * rt + k * rp + rin] = v;
    }
}

// x_t . x_t of every row, ascending k, one fma per term (R13; wss 2 gains, linear kernel)
__global__ void k_self_dot(const float* __restrict__ X, long long n, int d, double* __restrict__ q) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    double acc = 0.0;
    for (int k = 0; k < d; ++k) { const double x = X[t * d + k]; acc = fma(x, x, acc); }
    q[t] = acc;
}

// counts values of X that are not exactly 0 or 1
__global__ void k_count_nonbinary(const float* __restrict__ X, long long nx, unsigned long long* out) {
    unsigned long long c = 0;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nx; e += (long long)gridDim.x * blockDim.x) {
        const float v = X[e];
        c += (v != 0.0f && v != 1.0f);
    }
    if (c) atomicAdd(out, c);
}

// per column: 1 if some value is not exactly 0 or 1 (racy stores of the same value)
__global__ void k_col_nonbinary(const float* __restrict__ X, long long n, int d, int* __restrict__ nb) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n * d; e += (long long)gridDim.x * blockDim.x) {
        const float v = X[e];
        if (v != 0.0f && v != 1.0f) nb[e % d] = 1;
    }
}

// Mixed compact rows (Params::mix_*): the CTA-blocked layout of k_build_xblk over d_pad
// 32-bit slots per row -- slot i < nc: X[row][map[i]] (fp32), slot nc + w: bit b of word w
// = X[row][map[nc + 32 w + b]] != 0 -- zero padded.
__global__ void k_build_xblk_mixed(const float* __restrict__ X, long long n_r, int d, const int* __restrict__ map,
                                   int nc, int nbw, int d_pad, int G, int rt, long long cta_stride,
                                   float* __restrict__ xblk) {
    const int c = blockIdx.y;
    const long long r0 = (n_r * c) / G, r1 = (n_r * (c + 1)) / G;
    const long long R = r1 - r0;
    const long long total = R * d_pad;
    const int nbin = d - nc;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long k = e / R;
        const long long j = e - k * R;
        const long long tile = j / rt, rin = j - tile * rt;
        const long long rows_t = (R - tile * rt) < rt ? (R - tile * rt) : rt;
        const long long rp = (rows_t + 3) & ~3ll;
        const float* row = X + (r0 + j) * d;
        uint32_t v = 0u;
        if (k < nc) {
            v = __float_as_uint(row[map[k]]);
        } else if (k < nc + nbw) {
            const int w = (int)(k - nc);
            for (int b = 0; b < 32; ++b) {
                const int i = 32 * w + b;
                if (i < nbin && row[map[nc + i]] != 0.0f) v |= 1u << b;
            }
        }
        xblk[(long long)c * cta_stride + tile * (long long)d_pad * rt + k * rp + rin] = __uint_as_float(v);
    }
}

// Mixed compact rows, row-major: row r = the nc continuous columns (fp32 bits, map order)
// then nbw bit words of the binary columns -- the pivots' compact forms (Params::xcomp).
__global__ void k_build_compact_rows(const float* __restrict__ X, long long n, int d, const int* __restrict__ map,
                                     int nc, int nbw, uint32_t* __restrict__ out) {
    const int ncw = nc + nbw, nbin = d - nc;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n * ncw;
         e += (long long)gridDim.x * blockDim.x) {
        const long long r = e / ncw;
        const int k = (int)(e - r * ncw);
        const float* row = X + r * d;
        uint32_t v = 0u;
        if (k < nc) {
            v = __float_as_uint(row[map[k]]);
        } else {
            const int w = k - nc;
            for (int b = 0; b < 32; ++b) {
                const int i = 32 * w + b;
                if (i < nbin && row[map[nc + i]] != 0.0f) v |= 1u << b;
            }
        }
        out[e] = v;
    }
}

// Dictionary of X's distinct fp32 values (bit patterns): an open-addressing set of 1024
// slots; per-block sets in shared memory merged into the global one.  *count ends > 256 if
// X has more than 256 distinct values (then the build stops early).
constexpr int DICT_SLOTS = 1024;
constexpr unsigned DICT_EMPTY = 0xffffffffu;                // a NaN pattern: never in X
__device__ __forceinline__ unsigned dict_hash(unsigned u) { return (u * 2654435761u) >> 22; }
__global__ void k_dict_insert(const float* __restrict__ X, long long nx, unsigned* __restrict__ keys,
                              int* __restrict__ count) {
    __shared__ unsigned sk[DICT_SLOTS];
    __shared__ int scount;
    for (int i = threadIdx.x; i < DICT_SLOTS; i += blockDim.x) sk[i] = DICT_EMPTY;
    if (threadIdx.x == 0) scount = 0;
    __syncthreads();
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nx; e += (long long)gridDim.x * blockDim.x) {
        if (*(volatile int*)&scount > 256 || *(volatile int*)count > 256) break;
        const unsigned u = __float_as_uint(X[e]);
        unsigned h = dict_hash(u);
        for (int probe = 0;; ++probe) {
            if (probe == DICT_SLOTS) { atomicAdd(&scount, 1000); break; }
            const unsigned prev = atomicCAS(&sk[h], DICT_EMPTY, u);
            if (prev == DICT_EMPTY) { atomicAdd(&scount, 1); break; }
            if (prev == u) break;
            h = (h + 1) & (DICT_SLOTS - 1);
        }
    }
    __syncthreads();
    if (scount > 256) {
        if (threadIdx.x == 0) atomicAdd(count, 1000);
        return;
    }
    for (int i = threadIdx.x; i < DICT_SLOTS; i += blockDim.x) {
        const unsigned u = sk[i];
        if (u == DICT_EMPTY) continue;
        unsigned h = dict_hash(u);
        for (int probe = 0; probe < DICT_SLOTS; ++probe) {
            const unsigned prev = atomicCAS(&keys[h], DICT_EMPTY, u);
            if (prev == DICT_EMPTY) { atomicAdd(count, 1); break; }
            if (prev == u) break;
            h = (h + 1) & (DICT_SLOTS - 1);
        }
    }
}
__device__ __forceinline__ unsigned dict_code(const unsigned* keys, const unsigned char* code, unsigned u) {
    unsigned h = dict_hash(u);
    while (keys[h] != u) h = (h + 1) & (DICT_SLOTS - 1);
    return code[h];
}
// The CTA-blocked layout of k_build_xblk with one byte per element: the dictionary code.
__global__ void k_build_xblk_dict(const float* __restrict__ X, long long n_r, int d, int d_pad, int G, int rt,
                                  long long cta_stride, const unsigned* __restrict__ keys,
                                  const unsigned char* __restrict__ code, unsigned char* __restrict__ xblk) {
    const int c = blockIdx.y;
    const long long r0 = (n_r * c) / G, r1 = (n_r * (c + 1)) / G;
    const long long R = r1 - r0;
    const long long total = R * d_pad;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long k = e / R;
        const long long j = e - k * R;
        const long long tile = j / rt, rin = j - tile * rt;
        const long long rows_t = (R - tile * rt) < rt ? (R - tile * rt) : rt;
        const long long rp = (rows_t + 3) & ~3ll;
        const unsigned char v = (k < d) ? (unsigned char)dict_code(keys, code, __float_as_uint(X[(r0 + j) * d + k])) : 0;
        xblk[(long long)c * cta_stride + tile * (long long)d_pad * rt + k * rp + rin] = v;
    }
}

// bit rows: bit k of word k/32 of row r = X[r][k]
__global__ void k_pack_bits(const float* __restrict__ X, long long n, int d, int W, uint32_t* __restrict__ out) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n * W; e += (long long)gridDim.x * blockDim.x) {
        const long long r = e / W;
        const int w = (int)(e - r * W);
        uint32_t v = 0;
        for (int b = 0; b < 32; ++b) {
            const int k = w * 32 + b;
            if (k < d && X[r * d + k] != 0.0f) v |= 1u << b;
        }
        out[e] = v;
    }
}

// CTA-blocked bit layout of one rank's rows: row j of CTA c at xb[c*cta_stride + j*Wp ..],
// Wp = W rounded up to 4 (zero padded), so a consumer thread reads a row with 16-byte loads
__global__ void k_build_xbits(const uint32_t* __restrict__ bits, long long n_r, int W, int Wp, int G,
                              long long cta_stride, uint32_t* __restrict__ xb) {
    const int c = blockIdx.y;
    const long long r0 = (n_r * c) / G, r1 = (n_r * (c + 1)) / G;
    const long long R = r1 - r0;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < R * Wp; e += (long long)gridDim.x * blockDim.x) {
        const long long j = e / Wp;
        const int w = (int)(e - j * Wp);
        xb[(long long)c * cta_stride + e] = w < W ? bits[(r0 + j) * W + w] : 0u;
    }
}

__global__ void k_init_state(const int8_t* __restrict__ y, long long n, double C,
                             const double* __restrict__ alpha0, const double* __restrict__ f0,
                             double* __restrict__ f, double* __restrict__ alpha,
                             uint8_t* __restrict__ flags) {
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (long long)gridDim.x * blockDim.x) {
        const int yj = y[j];
        const double a = alpha0 ? alpha0[j] : 0.0;
        alpha[j] = a;
        f[j] = f0 ? f0[j] : -(double)yj;                       // f = -y at alpha = 0
        flags[j] = flags_of(yj, a, C);
    }
}

// counts[0] non-finite X, [1] labels outside {+1,-1}, [2] positives, [3] negatives
__global__ void k_validate(const float* __restrict__ X, long long nx, const int8_t* __restrict__ y,
                           long long n, unsigned long long* counts) {
    unsigned long long bad = 0, lab = 0, pos = 0, neg = 0;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nx;
         e += (long long)gridDim.x * blockDim.x)
        bad += !isfinite(X[e]);
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (long long)gridDim.x * blockDim.x) {
        const int v = y[j];
        pos += v == 1; neg += v == -1; lab += (v != 1 && v != -1);
    }
    if (bad) atomicAdd(&counts[0], bad);
    if (lab) atomicAdd(&counts[1], lab);
    if (pos) atomicAdd(&counts[2], pos);
    if (neg) atomicAdd(&counts[3], neg);
}

// The library allocates its scratch with cudaMallocAsync and frees it before returning.
// With the default pool's release threshold (0) every stream synchronisation hands the
// memory back to the driver, so every call would map it again; keep up to 2 GiB cached
// in the current device's default pool (a caching allocator's behaviour).
void pool_setup() {
    static thread_local int done_mask = 0;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 31 || (done_mask >> dev) & 1) { cudaGetLastError(); return; }
    cudaMemPool_t pool;
    unsigned long long thr = 2ull << 30;
    if (const char* e = getenv("SVMB200_POOL_KEEP_MB")) thr = (unsigned long long)atoll(e) << 20;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    done_mask |= 1 << dev;
}

int validate_device(const float* X, const int8_t* y, long long n, long long d, cudaStream_t st,
                    int* n_pos) {
    pool_setup();
    unsigned long long* dc = nullptr;
    CKR(cudaMallocAsync(&dc, 4 * sizeof(unsigned long long), st));
    CKR(cudaMemsetAsync(dc, 0, 4 * sizeof(unsigned long long), st));
    k_validate<<<1024, 256, 0, st>>>(X, n * d, y, n, dc);
    counted();
    unsigned long long hc[4];
    CKR(cudaMemcpyAsync(hc, dc, sizeof(hc), cudaMemcpyDeviceToHost, st));
    CKR(cudaFreeAsync(dc, st));
    CKR(cudaStreamSynchronize(st));
    if (hc[0]) return fail(SVM_ENONFINITE, "X contains " + std::to_string(hc[0]) + " non-finite values");
    if (hc[1]) return fail(SVM_ELABEL, std::to_string(hc[1]) + " labels are not +1/-1");
    if (hc[2] == 0 || hc[3] == 0) return fail(SVM_ESINGLECLASS, "single-class problem");
    if (n_pos) *n_pos = (int)hc[2];
    return SVM_OK;
}

int check_params(long long n, long long d, const svm_params* p, svm_params* q) {
    if (!p) return fail(SVM_EINVAL, "null params");
    *q = *p;
    if (n < 2) return fail(SVM_EINVAL, "n < 2");
    if (d < 1) return fail(SVM_EINVAL, "d < 1");
    if (n > 0x7fffffffll) return fail(SVM_EINVAL, "n >= 2^31");
    if (!(q->C > 0.0) || !std::isfinite(q->C)) return fail(SVM_EINVAL, "C must be finite and > 0");
    if (q->kernel != SVM_LINEAR && q->kernel != SVM_RBF) return fail(SVM_EINVAL, "unknown kernel");
    if (q->kernel == SVM_RBF && (!(q->gamma > 0.0) || !std::isfinite(q->gamma)))
        return fail(SVM_EINVAL, "RBF gamma must be finite and > 0");
    if (q->tol <= 0.0) q->tol = 1e-3;
    if (!std::isfinite(q->tol)) return fail(SVM_EINVAL, "tol must be finite");
    if (q->max_iter <= 0) q->max_iter = (10 * n > 10000) ? 10 * n : 10000;
    if (q->check_interval <= 0) q->check_interval = 64;
    if (q->sv_epsilon <= 0.0) q->sv_epsilon = 1e-8;
    if (q->virtual_ranks <= 1) q->virtual_ranks = 1;
    if (q->virtual_ranks > MAXR) return fail(SVM_EINVAL, "virtual_ranks > 8");
    if (q->wss <= 0) q->wss = 1;
    if (q->shrink_window < 0) return fail(SVM_EINVAL, "shrink_window must be >= 0");
    if (q->wss > 2) return fail(SVM_EINVAL, "wss must be 1 (first order) or 2 (second order)");
    return SVM_OK;
}

// ------------------------------------------------------------------ planning
struct Plan {
    int G = 0;        // CTAs per rank
    int rpt = 1, rt = 256, kc = 16, d_pad = 0, n_chunks = 0, stages = 0, state_cap = 0;
    bool alpha_smem = true;
    bool resident = false;
    int bin_words = 0;
    int cache_slots = 0;
    int cache_hash = 0;
    int cluster = 0;  // > 0: cluster mode with G CTAs per cluster (one cluster per rank)
    bool bincl = false;  // cluster mode on binary rows: the smo_bincl kernel (NTB threads)
    int crow = 0, crw = 0;
    int dp = 0;          // dense pivot entries (shared memory)
    int mix_nc = 0, mix_nbw = 0, mix_nseg = 0;   // mixed compact rows (mix_nseg > 0)
    int mix_seg[MIX_MAXSEG] = {};
    int esz = 4;         // bytes per xblk element (1: dictionary codes)
    int ntc = NT;        // consumer threads per CTA (256, or 512 for the streamed modes)
    long long cta_stride = 0;
    size_t smem = 0;
};

// the solve being planned uses the second-order rule (its kernels have 256 consumer threads)
static thread_local bool t_plan_wss2 = false;

int make_plan(long long n_r_max, int d, int G, int max_smem, Plan& pl, bool binary = false,
              bool gram = false, int cache_slots = 0, int cl_words = 0, const Plan* mix = nullptr) {
    pl.G = G;
    pl.dp = 0;
    if (mix) {
        pl.mix_nc = mix->mix_nc; pl.mix_nbw = mix->mix_nbw; pl.mix_nseg = mix->mix_nseg;
        for (int i = 0; i < MIX_MAXSEG; ++i) pl.mix_seg[i] = mix->mix_seg[i];
        pl.esz = mix->esz;
    }
    // cluster mode: the shared-memory mailbox cmb[2][G][cl_words] of 16-byte words
    const size_t cl_bytes = cl_words > 0 ? (size_t)2 * G * cl_words * 16 + 16 : 0;
    if (gram) {
        // rows of K are read from HBM: state and control only, no X stages
        pl.state_cap = (int)((n_r_max + G - 1) / G);
        if (pl.state_cap < 1) pl.state_cap = 1;
        pl.rpt = pl.state_cap <= NT ? 1 : (pl.state_cap <= 2 * NT ? 2 : 4);
        pl.rt = NT * pl.rpt; pl.kc = 1; pl.d_pad = 1; pl.n_chunks = 0;
        pl.cta_stride = 0;
        pl.alpha_smem = pl.state_cap <= 2048;
        size_t fixed = (sizeof(Shared) + 127) & ~size_t(127);
        fixed += 2 * (size_t)8 * 8 + (size_t)pl.state_cap * (pl.alpha_smem ? 17 : 9);
        fixed = (fixed + 127) & ~size_t(127);
        if (fixed > (size_t)max_smem) return fail(SVM_ENOMEM, "shard too large for the shared-memory state");
        pl.stages = 1; pl.resident = false; pl.smem = fixed;
        return SVM_OK;
    }
    if (binary) {
        // bit rows, resident in shared memory, one row per consumer thread
        pl.state_cap = (int)((n_r_max + G - 1) / G);
        if (pl.state_cap < 1) pl.state_cap = 1;
        pl.rpt = 1; pl.rt = NT; pl.kc = 32;
        pl.bin_words = (d + 31) / 32;
        pl.d_pad = pl.bin_words * 32;                      // pivot region sizing only
        pl.n_chunks = 0;
        const int n_tiles = (pl.state_cap + pl.rt - 1) / pl.rt;
        pl.cta_stride = (long long)n_tiles * ((pl.bin_words + 3) & ~3) * pl.rt;
        pl.alpha_smem = pl.state_cap <= 2048;
        size_t fixed = (sizeof(Shared) + 127) & ~size_t(127);
        fixed += 2 * (size_t)pl.d_pad * 8 + (size_t)pl.state_cap * (pl.alpha_smem ? 17 : 9);
        fixed = ((fixed + 7) & ~size_t(7)) + (size_t)(32 * pl.bin_words + 1) * 8;   // K table
        fixed += cl_bytes;
        fixed = (fixed + 127) & ~size_t(127);
        const size_t bytes = (size_t)pl.cta_stride * 4;
        pl.resident = true;
        pl.stages = 1;
        pl.smem = fixed + bytes;
        if (pl.smem > (size_t)max_smem) return fail(SVM_ENOMEM, "binary block does not fit");
        return SVM_OK;
    }
    pl.state_cap = (int)((n_r_max + G - 1) / G);
    if (pl.state_cap < 1) pl.state_cap = 1;
    // rows per consumer thread: as few tiles per CTA as possible, at most 4 rows
    // consumer threads: 16 warps (more latency hiding for the exp- and fp64-bound row pass)
    // when each thread then still has <= 2 rows per tile, else 8 warps
    // (measured: W4's mixed rows, 12 slots and 2 exps per row, 28.6 -> 24.9 us/iteration;
    // W5's 256 features and W3's row cache are slower with 16 warps: fp64 / HBM bound with
    // RPT 2 and register spills)
    const int slots = pl.mix_nseg > 0 ? pl.mix_nc + pl.mix_nbw : d;
    pl.ntc = (cl_words == 0 && cache_slots == 0 && slots <= 64) ? 512 : NT;
    if (const char* e = getenv("SVMB200_NT")) {                  // tuning override: 256 or 512
        const int v = atoi(e);
        if (v == 256 || (v == 512 && cl_words == 0)) pl.ntc = v;
        // (448: 14 consumer warps + 2 = 16 warps, 4 per SM sub-partition -> 128 registers per
        // thread instead of 96; mixed rows only, tuning)
        if (v == 448 && cl_words == 0 && pl.mix_nseg > 0) pl.ntc = v;
    }
    if (t_plan_wss2) pl.ntc = NT;
    if (pl.bin_words > 0 || cache_slots > 0) pl.ntc = NT;   // (not compiled into the 16-warp kernels)
    pl.rpt = pl.state_cap <= pl.ntc ? 1 : (pl.state_cap <= 2 * pl.ntc ? 2 : 4);
    if (const char* e = getenv("SVMB200_RPT")) {          // tuning override: 1, 2 or 4
        const int r = atoi(e);
        if (r == 1 || r == 2 || r == 4) pl.rpt = r;
    }
    if (pl.ntc > NT && pl.rpt == 4) pl.rpt = 2;           // register budget of 576 threads
    pl.rt = pl.ntc * pl.rpt;
    // Stage size: the largest kc (features per stage) whose zero padding of d stays small and
    // for which two stages fit next to the state -- fewer, larger bulk copies amortise the
    // per-stage mbarrier hand-off (measured on W5: 32 KB x 5 stages 188.9 us/iteration,
    // 48 KB x 3 181.4, 64 KB x 2 177.5, 80 KB x 2 174.4; 125k-row shard 30.1 -> 25.6 us).
    // Mixed rows use one stage per tile (all slots of a row); SVMB200_KC overrides.
    const int kc_min = 8192 * (4 / pl.esz) / pl.rt;        // 32 KB stages
    int kc_env = 0;
    if (const char* e = getenv("SVMB200_KC")) {            // tuning override (features per stage)
        const int v = atoi(e);
        if (v >= 1 && v <= 256) kc_env = v;
    }
    // (first choice: >= 3 stages of >= 64 KB -- a 125k-row W5 shard: 3 x 64 KB 25.6 us,
    // 2 x 104 KB 27.7 us; else the largest two stages)
    const int kc_max = pl.mix_nseg > 0 ? kc_min : (kc_env > 0 ? kc_env : (pl.esz == 1 ? 256 : 64));
    for (int pass = 0; pass < 2; ++pass)
    for (int kc_try = kc_max; kc_try >= 1; --kc_try) {
    const bool want3 = pass == 0 && kc_env == 0 && pl.mix_nseg == 0;
    if (want3 && (size_t)kc_try * pl.rt * pl.esz < 65536) break;
    const bool last_try = !want3 && (kc_try <= kc_min || kc_env > 0 || pl.mix_nseg > 0);
    pl.kc = kc_env > 0 ? kc_env : kc_try;
    if (pl.esz == 1 && (pl.kc & 3)) continue;              // byte stages: 16-byte multiples
    if (!last_try) {
        const int dpad_try = (d + pl.kc - 1) / pl.kc * pl.kc;
        if (dpad_try - d > (d / 50 > 4 ? d / 50 : 4)) continue;   // <= 2% (or 4 features) padding
    }
    pl.d_pad = (d + pl.kc - 1) / pl.kc * pl.kc;
    pl.n_chunks = pl.d_pad / pl.kc;
    pl.dp = pl.d_pad;
    size_t mix_bytes = 0;
    if (pl.mix_nseg > 0) {
        // one stage holds whole compact rows: nc fp32 slots + nbw bit words
        pl.kc = (pl.mix_nc + pl.mix_nbw + 3) & ~3;
        pl.d_pad = pl.kc;
        pl.n_chunks = 1;
        pl.dp = (d + 3) & ~3;
        mix_bytes = (size_t)pl.mix_nc * 16 + (((size_t)2 * pl.mix_nbw * 4 + 15) & ~size_t(15));
    }
    if (pl.esz == 1) {
        pl.kc = (pl.kc + 3) & ~3;                          // byte stages: 16-byte multiples
        pl.d_pad = (d + pl.kc - 1) / pl.kc * pl.kc;
        pl.n_chunks = pl.d_pad / pl.kc;
        pl.dp = pl.d_pad;
        mix_bytes = 256 * 8;                               // the dictionary values
    }
    const int n_tiles = (pl.state_cap + pl.rt - 1) / pl.rt;
    pl.cta_stride = (long long)n_tiles * pl.d_pad * pl.rt;
    pl.alpha_smem = pl.state_cap <= 2048;                  // else alpha stays in HBM
    size_t fixed = (sizeof(Shared) + 127) & ~size_t(127);
    fixed += 2 * (size_t)pl.dp * 8 + mix_bytes + (size_t)pl.state_cap * (pl.alpha_smem ? 17 : 9);  // pivots + state
    int hash = 0;
    if (cache_slots > 0) { hash = 1; while (hash < 2 * cache_slots) hash <<= 1; }
    fixed = ((fixed + 7) & ~size_t(7)) + (size_t)cache_slots * 12;                      // cache directory + LRU list
    fixed = ((fixed + 7) & ~size_t(7)) + (size_t)hash * 8 + (cache_slots > 0 ? (size_t)pl.dp * 16 + 8 : 0);
    pl.cache_hash = hash;
    fixed += cl_bytes;
    fixed = (fixed + 127) & ~size_t(127);
    const size_t stage_bytes = (size_t)pl.kc * pl.rt * pl.esz;
    // resident mode: the whole (single-tile) X block of a CTA fits next to the state
    const size_t resident_bytes = (size_t)pl.d_pad * ((pl.state_cap + 3) & ~3) * pl.esz;
    pl.resident = n_tiles == 1 && fixed + resident_bytes <= (size_t)max_smem && getenv("SVMB200_NO_RESIDENT") == nullptr;
    if (pl.resident) {
        pl.stages = 1;
        pl.smem = fixed + resident_bytes;
        return SVM_OK;
    }
    if ((size_t)max_smem <= fixed + (want3 ? 3 : 2) * stage_bytes) {
        if (!last_try) continue;
        return fail(SVM_ENOMEM, "rows per CTA (" + std::to_string(pl.state_cap) +
                                    ") exceed the shared-memory state capacity; shard over more GPUs");
    }
    pl.stages = (int)((max_smem - fixed) / stage_bytes);
    if (pl.stages > MAX_STAGES) pl.stages = MAX_STAGES;
    pl.smem = fixed + (size_t)pl.stages * stage_bytes;
    return SVM_OK;
    }
    return fail(SVM_ENOMEM, "no stage size fits");
}

typedef void (*KernelFn)(const Params);

// The solver's instantiations live in four translation units compiled in parallel
// (smo_pick.cuh; smo_{gen,spec}_{rbf,lin}.cu): the general ones (every mode, the second-order
// rule, the wide poll) and the specialised ones (mixed-, dense- or dictionary-rows only;
// binary rows in a cluster).
KernelFn pick_general_rbf(int rpt, bool a_smem, int ntc, bool wss2, bool wide);
KernelFn pick_general_lin(int rpt, bool a_smem, int ntc, bool wss2, bool wide);
KernelFn pick_spec_rbf(int rpt, bool a_smem, int ntc, bool wide, bool mix, bool dense, bool dict);
KernelFn pick_spec_lin(int rpt, bool a_smem, int ntc, bool wide, bool mix, bool dense, bool dict);
KernelFn pick_bincl_spec_rbf(bool a_smem);
KernelFn pick_bincl_spec_lin(bool a_smem);

KernelFn pick_bincl(int kernel) { return kernel == SVM_RBF ? smo_bincl<1> : smo_bincl<0>; }

// bincl: binary rows resident in a cluster (the specialised kernel; rpt is 1 there)
KernelFn pick_kernel(int kernel, int rpt, bool a_smem, bool bincl = false, int ntc = NT, bool wss2 = false,
                     bool wide = false, bool mix = false, bool dense = false, bool dict = false) {
    const bool rbf = kernel == SVM_RBF;
    if (bincl && getenv("SVMB200_NO_SPECIALISE") == nullptr)
        return rbf ? pick_bincl_spec_rbf(a_smem) : pick_bincl_spec_lin(a_smem);
    if (!wss2 && (mix || dense || dict)) {
        KernelFn f = rbf ? pick_spec_rbf(rpt, a_smem, ntc, wide, mix, dense, dict)
                         : pick_spec_lin(rpt, a_smem, ntc, wide, mix, dense, dict);
        if (f) return f;
    }
    return rbf ? pick_general_rbf(rpt, a_smem, ntc, wss2, wide) : pick_general_lin(rpt, a_smem, ntc, wss2, wide);
}

int device_limits(int* n_sm, int* max_smem) {
    pool_setup();
    int dev;
    CKR(cudaGetDevice(&dev));
    CKR(cudaDeviceGetAttribute(n_sm, cudaDevAttrMultiProcessorCount, dev));
    CKR(cudaDeviceGetAttribute(max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    return SVM_OK;
}

// ------------------------------------------------------------------ the solve
// Runs the solver for `nranks_here` ranks served by this process/launch.  Every rank r
// of the problem (0..world-1) owns rows [row_off[r], row_off[r] + n_rows[r]).  For a
// single-process solve (world == nranks_here) all pointers are local.
int solve(SolveArgs& a) {
    const svm_params& p = a.p;
    t_plan_wss2 = (p.wss == 2);
    Plan pl;
    int rc = SVM_OK;
    bool binary = false;
    // (wss 2 runs on fp32 / dictionary / mixed rows: the resident bit-row loop has no gain pass)
    if (!a.independent && !a.skip_detect && p.wss != 2 && getenv("SVMB200_NO_BINARY") == nullptr && a.d <= 1024) {
        unsigned long long* dc = nullptr;
        CKR(cudaMallocAsync(&dc, 8, a.stream));
        CKR(cudaMemsetAsync(dc, 0, 8, a.stream));
        k_count_nonbinary<<<1024, 256, 0, a.stream>>>(a.xr, a.n_global * a.d, dc);
        counted();
        unsigned long long nb = 1;
        CKR(cudaMemcpyAsync(&nb, dc, 8, cudaMemcpyDeviceToHost, a.stream));
        CKR(cudaFreeAsync(dc, a.stream));
        CKR(cudaStreamSynchronize(a.stream));
        binary = (nb == 0);
    }
    if (binary && make_plan(a.n_rows_max, (int)a.d, a.ctas_per_rank, a.max_smem, pl, true) != SVM_OK)
        binary = false;
    // full-Gram path (a9): one rank only; forced, or auto for mid-size problems
    double* gram = nullptr;
    cudaEvent_t ev_gram = nullptr;
    const bool single = (a.world == 1 && a.nranks_here == 1 && !a.independent);
    // (measured: building K costs more than the LRU row cache saves for W3, so the Gram
    // path is used only on request)
    const bool want_gram = single && a.p.gram == 1;
    if (a.p.gram == 1 && !single) return fail(SVM_EINVAL, "the Gram path needs a single rank");
    if (want_gram) {
        if (cudaMallocAsync(&gram, (size_t)a.n_global * a.n_global * 8, a.stream) != cudaSuccess) {
            cudaGetLastError();
            gram = nullptr;
            if (a.p.gram == 1) return fail(SVM_ENOMEM, "Gram matrix allocation failed");
        }
    }
    if (gram) {
        binary = false;
        pl = Plan();
        if ((rc = make_plan(a.n_rows_max, (int)a.d, a.ctas_per_rank, a.max_smem, pl, false, true))) {
            cudaFreeAsync(gram, a.stream);
            return rc;
        }
        CKR(cudaEventCreate(&ev_gram));
        CKR(cudaEventRecord(ev_gram, a.stream));          // the solve time includes building K
        if ((rc = gram_device(a.xr, a.n_global, a.d, p.kernel, p.gamma, gram, a.stream))) {
            cudaFreeAsync(gram, a.stream);
            return rc;
        }
    } else if (!binary) {
        // mixed compact rows: binary columns as bits when that shrinks the rows (>= 32 of
        // them, at most MIX_MAXSEG runs of the column order)
        Plan mix;
        std::vector<int> mix_map;
        if (!a.independent && !a.skip_detect && getenv("SVMB200_NO_MIXED") == nullptr && a.d >= 32) {
            int* dnb = nullptr;
            CKR(cudaMallocAsync(&dnb, (size_t)a.d * 4, a.stream));
            CKR(cudaMemsetAsync(dnb, 0, (size_t)a.d * 4, a.stream));
            k_col_nonbinary<<<1024, 256, 0, a.stream>>>(a.xr, a.n_global, (int)a.d, dnb);
            counted();
            std::vector<int> nb((size_t)a.d);
            CKR(cudaMemcpyAsync(nb.data(), dnb, (size_t)a.d * 4, cudaMemcpyDeviceToHost, a.stream));
            CKR(cudaFreeAsync(dnb, a.stream));
            CKR(cudaStreamSynchronize(a.stream));
            int nbin = 0, nseg = 0, prev = -1;
            for (long long k = 0; k < a.d; ++k) {
                const int isbin = nb[k] == 0;
                nbin += isbin;
                if (isbin != prev) { ++nseg; prev = isbin; }
            }
            const int nc = (int)a.d - nbin, nbw = (nbin + 31) / 32;
            if (nbin >= 32 && nseg <= MIX_MAXSEG && 4 * (nc + nbw) <= 3 * a.d) {
                mix.mix_nc = nc; mix.mix_nbw = nbw; mix.mix_nseg = nseg;
                int sg = -1;
                prev = -1;
                for (long long k = 0; k < a.d; ++k) {
                    const int isbin = nb[k] == 0;
                    if (isbin != prev) { ++sg; prev = isbin; }
                    mix.mix_seg[sg] += isbin ? -1 : 1;
                }
                for (long long k = 0; k < a.d; ++k) if (nb[k]) mix_map.push_back((int)k);
                for (long long k = 0; k < a.d; ++k) if (!nb[k]) mix_map.push_back((int)k);
            }
        }
        // dictionary-coded rows: <= 256 distinct fp32 values in X (uint8 pixels, SURVEY
        // §8(f)); preferred when smaller than the mixed rows
        std::vector<double> dict_vals;
        std::vector<unsigned char> dict_code((size_t)DICT_SLOTS, 0);
        std::vector<unsigned> dict_keys((size_t)DICT_SLOTS, DICT_EMPTY);
        if (!a.independent && !a.skip_detect && getenv("SVMB200_NO_DICT") == nullptr && a.d >= 8 &&
            (mix.mix_nseg == 0 || a.d < 4 * (mix.mix_nc + mix.mix_nbw))) {
            unsigned* dk = nullptr;
            int* dcnt = nullptr;
            CKR(cudaMallocAsync(&dk, DICT_SLOTS * 4, a.stream));
            CKR(cudaMallocAsync(&dcnt, 4, a.stream));
            CKR(cudaMemsetAsync(dk, 0xff, DICT_SLOTS * 4, a.stream));
            CKR(cudaMemsetAsync(dcnt, 0, 4, a.stream));
            k_dict_insert<<<592, 256, 0, a.stream>>>(a.xr, a.n_global * a.d, dk, dcnt);
            counted();
            int cnt = 0;
            CKR(cudaMemcpyAsync(&cnt, dcnt, 4, cudaMemcpyDeviceToHost, a.stream));
            CKR(cudaMemcpyAsync(dict_keys.data(), dk, DICT_SLOTS * 4, cudaMemcpyDeviceToHost, a.stream));
            CKR(cudaFreeAsync(dk, a.stream));
            CKR(cudaFreeAsync(dcnt, a.stream));
            CKR(cudaStreamSynchronize(a.stream));
            if (cnt >= 1 && cnt <= 256) {
                for (int h = 0; h < DICT_SLOTS; ++h) {
                    if (dict_keys[h] == DICT_EMPTY) continue;
                    float f;
                    memcpy(&f, &dict_keys[h], 4);
                    dict_code[h] = (unsigned char)dict_vals.size();
                    dict_vals.push_back((double)f);
                }
            }
        }
        pl = Plan();
        if (!dict_vals.empty()) {
            Plan dp_;
            dp_.esz = 1;
            if (make_plan(a.n_rows_max, (int)a.d, a.ctas_per_rank, a.max_smem, pl, false, false, 0, 0, &dp_) == SVM_OK) {
                mix = Plan();
                mix_map.clear();
                a.dict_vals = dict_vals;
                a.dict_keys = dict_keys;
                a.dict_code = dict_code;
            } else {
                pl = Plan();
                dict_vals.clear();
            }
        }
        if (dict_vals.empty() && mix.mix_nseg > 0) {
            if (make_plan(a.n_rows_max, (int)a.d, a.ctas_per_rank, a.max_smem, pl, false, false, 0, 0, &mix) != SVM_OK) {
                mix = Plan();
                mix_map.clear();
                pl = Plan();
            }
        }
        if (mix.mix_nseg == 0 && pl.esz != 1) {
            rc = make_plan(a.n_rows_max, (int)a.d, a.ctas_per_rank, a.max_smem, pl);
            if (rc) return rc;
        }
        a.mix_map = mix_map;
        // kernel-row LRU cache (a8) for streamed X
        int slots = a.p.cache_rows;
        if (slots == 0 && !pl.resident && !a.independent && a.n_global <= 200000) {
            slots = (int)(a.n_global / 25);
            slots = slots < 64 ? 64 : (slots > 2048 ? 2048 : slots);
            size_t fr = 0, tot = 0;
            if (cudaMemGetInfo(&fr, &tot) != cudaSuccess ||
                (double)slots * a.n_global * 8.0 > (double)fr / 3.0)
                slots = 0;
        }
        if (slots > 0 && !pl.resident) {
            if (slots < 4) slots = 4;
            Plan pc;
            if (make_plan(a.n_rows_max, (int)a.d, a.ctas_per_rank, a.max_smem, pc, false, false, slots, 0,
                          (pl.mix_nseg > 0 || pl.esz != 4) ? &pl : nullptr) == SVM_OK &&
                !pc.resident) {
                pl = pc;
                pl.cache_slots = slots;
            }
        }
    }
    // ---- cluster mode: when a rank's rows fit resident in the shared memory of <= 16 CTAs,
    // those CTAs form one thread-block cluster and exchange candidates through distributed
    // shared memory (~0.2 us) instead of global-memory mailboxes (~2.5 us); the candidates'
    // rows travel in the records.  Auto: the smallest power-of-two cluster with <= 2048 rows
    // per CTA (else 16 CTAs if <= 8192 rows each), when it is resident.
    const bool cl_allowed = gram == nullptr && pl.cache_slots == 0 && pl.mix_nseg == 0 && pl.esz == 4 && a.p.cluster != -1 &&
                            p.wss != 2 &&
                            a.world == a.nranks_here && (a.world == 1 || a.independent) &&
                            (a.p.ctas <= 0 || a.p.cluster > 0) && getenv("SVMB200_NO_CLUSTER") == nullptr;
    if (a.p.cluster > 16 || a.p.cluster < -1) return fail(SVM_EINVAL, "cluster must be -1, 0 or 1..16");
    if (a.p.cluster > 0 && !cl_allowed)
        return fail(SVM_EINVAL, "cluster mode needs one rank (or batched problems) and no Gram/cache path");
    if (cl_allowed) {
        const int crow = binary ? (pl.bin_words <= 12 ? pl.bin_words : 0) : (a.d <= 12 ? (int)a.d : 0);
        const int crw = 4 + 2 * ((crow + 2) / 3);
        for (int gc = 1; gc <= 16; gc *= 2) {
            if (a.p.cluster > 0 && gc != a.p.cluster) continue;
            const long long rows = (a.n_rows_max + gc - 1) / gc;
            if (a.p.cluster == 0) {
                if (rows > 8192) continue;
                if (rows > 2048 && gc < 16) continue;
            }
            if ((long long)gc * a.nranks_here > a.n_sm) break;
            Plan pc;
            if (make_plan(a.n_rows_max, (int)a.d, gc, a.max_smem, pc, binary, false, 0, crw) != SVM_OK) {
                cudaGetLastError();
                continue;
            }
            if (!pc.resident) continue;
            // binary rows of <= 256 features: the dedicated latency-path kernel
            if (binary && pc.bin_words <= BINCL_MAXW && getenv("SVMB200_NO_BINCL") == nullptr) {
                pc.bincl = true;
                pc.smem = bincl_smem_bytes(pc.state_cap, pc.bin_words, gc, crw);
                if (pc.smem > (size_t)a.max_smem) continue;
            }
            KernelFn f2 = pc.bincl ? pick_bincl(p.kernel) : pick_kernel(p.kernel, pc.rpt, pc.alpha_smem, binary);
            CKR(cudaFuncSetAttribute((const void*)f2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pc.smem));
            if (gc > 8) CKR(cudaFuncSetAttribute((const void*)f2, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = gc; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.gridDim = dim3(gc * a.nranks_here); cfg.blockDim = dim3(pc.bincl ? NTB : NTHREADS);
            cfg.dynamicSmemBytes = pc.smem; cfg.attrs = at; cfg.numAttrs = 1;
            int ncl = 0;
            if (cudaOccupancyMaxActiveClusters(&ncl, (const void*)f2, &cfg) != cudaSuccess || ncl < 1) {
                cudaGetLastError();
                continue;
            }
            pl = pc;
            pl.cluster = gc; pl.crow = crow; pl.crw = crw;
            a.ctas_per_rank = gc;
            break;
        }
        if (a.p.cluster > 0 && pl.cluster == 0)
            return fail(SVM_EINVAL, "cluster mode needs every rank's rows resident in the cluster's shared memory");
    }
    // (test hook SVMB200_XCH_DUP = k, one process: every record also lands in k - 1 more slots,
    // so one GPU polls as many records as k GPUs would)
    int xch_dup = 1;
    if (const char* e = getenv("SVMB200_XCH_DUP")) xch_dup = std::max(1, std::min(16, atoi(e)));
    if (!a.mbox_local_alloc) xch_dup = 1;
    // the record poll: one warp (<= 320 records: one GPU, or two) or every consumer warp (more
    // GPUs; measured with SVMB200_XCH_DUP = 8, 1,184 records: a 125k-row W5 shard 42.5 -> 38.1
    // us/iteration, W4 31.8 -> 25.4; at 148 records one warp is faster).  SVMB200_WIDE_POLL =
    // 1 / 0 forces it on / off (not with wss 2 or the cluster exchange).
    const long long n_records = (long long)(a.independent ? 1 : a.world) * a.ctas_per_rank * xch_dup;
    bool wide = n_records > 320;
    if (const char* e = getenv("SVMB200_WIDE_POLL")) wide = atoi(e) != 0;
    wide = wide && p.wss != 2 && pl.cluster == 0 && !pl.bincl;
    // the mixed-rows-only 16-warp instantiation (W4): no other mode compiled in
    const bool mix_only = pl.ntc > NT && pl.mix_nseg > 0 && pl.cluster == 0 && !pl.bincl && gram == nullptr &&
                          pl.cache_slots == 0 && pl.bin_words == 0 && p.wss != 2 && pl.esz == 4 &&
                          getenv("SVMB200_NO_SPECIALISE") == nullptr;
    if (pl.ntc == 448 && !mix_only) return fail(SVM_EINVAL, "SVMB200_NT=448 is for the mixed-rows kernel only");
    // the dense-streamed-only 8-warp instantiation (W5 and its shards)
    const bool dense_only = pl.ntc == NT && pl.mix_nseg == 0 && pl.esz == 4 && pl.cluster == 0 && !pl.bincl &&
                            gram == nullptr && pl.cache_slots == 0 && pl.bin_words == 0 && p.wss != 2 &&
                            pl.rpt >= 2 && getenv("SVMB200_NO_SPECIALISE") == nullptr;
    // the dictionary-rows-only 8-warp instantiation (W3; with or without the row cache)
    const bool dict_only = pl.ntc == NT && pl.esz == 1 && pl.mix_nseg == 0 && pl.cluster == 0 && !pl.bincl &&
                           gram == nullptr && pl.bin_words == 0 && p.wss != 2 && !wide && pl.rpt >= 2 &&
                           getenv("SVMB200_NO_SPECIALISE") == nullptr;
    KernelFn fn = pl.bincl ? pick_bincl(p.kernel)
                           : pick_kernel(p.kernel, pl.rpt, pl.alpha_smem, pl.cluster > 0 && pl.bin_words > 0, pl.ntc,
                                         p.wss == 2, wide, mix_only, dense_only, dict_only);
    const int nthreads = pl.bincl ? NTB : pl.ntc + 64;
    {
        const char* mode = gram ? "gram" : pl.bin_words ? "binary-resident"
                         : pl.mix_nseg ? (pl.resident ? "mixed-resident" : pl.cache_slots ? "mixed+row-cache" : "mixed-streamed")
                         : pl.esz == 1 ? (pl.resident ? "dict-resident" : pl.cache_slots ? "dict+row-cache" : "dict-streamed")
                         : pl.resident ? "float-resident" : pl.cache_slots ? "streamed+row-cache" : "streamed";
        char buf[400];
        snprintf(buf, sizeof buf,
                 "{\"kernel\": \"%s<%d%s>\", \"ctas_per_rank\": %d, \"ranks\": %d, \"cluster\": %d, "
                 "\"mode\": \"%s\", \"threads\": %d, \"smem\": %zu, \"rows_per_cta\": %d, \"cache_slots\": %d, "
                 "\"poll\": \"%s\"}",
                 pl.bincl ? "smo_bincl" : "smo_persistent", p.kernel,
                 pl.bincl ? "" : (std::string(",") + std::to_string(pl.rpt) + (pl.alpha_smem ? ",1" : ",0") +
                                  ((pl.cluster > 0 && pl.bin_words > 0) ? ",1" : ",0") + (mix_only ? ",mix" : dense_only ? ",dense" : dict_only ? ",dict" : "")).c_str(),
                 a.ctas_per_rank, a.nranks_here, pl.cluster, mode, nthreads, pl.smem, pl.state_cap, pl.cache_slots,
                 pl.cluster > 0 || pl.bincl ? "cluster" : wide ? "wide" : "warp");
        g_plan = buf;
    }
    CKR(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
    if (pl.cluster > 8) CKR(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    int per_sm = 0;
    CKR(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)fn, nthreads, pl.smem));
    const int grid = a.ctas_per_rank * a.nranks_here;
    if (per_sm < 1 || grid > per_sm * a.n_sm)
        return fail(SVM_ECUDA, "persistent grid of " + std::to_string(grid) + " CTAs is not co-resident");

    cudaStream_t st = a.stream;
    const int world = a.world;
    const size_t mbox_bytes = svmk::mbox_bytes(a.ctas_per_rank * xch_dup, world);

    // ---- per-rank device state (a1)
    std::vector<void*> owned;
    if (gram) owned.push_back(gram);                       // freed with the other scratch
    auto dalloc = [&](void** ptr, size_t bytes) -> int {
        cudaError_t e = cudaMallocAsync(ptr, bytes, st);
        if (e != cudaSuccess) return fail(SVM_ENOMEM, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
        owned.push_back(*ptr);
        return SVM_OK;
    };
    auto release = [&]() {
        for (void* q : owned) cudaFreeAsync(q, st);
        owned.clear();
    };
    Params P;
    memset(&P, 0, sizeof(P));
    P.kernel = p.kernel; P.gamma = p.gamma; P.C = p.C; P.tol = p.tol;
    P.max_iter = p.max_iter; P.iter_limit = p.iters_per_launch > 0 ? p.iters_per_launch : 0;
    P.d = (int)a.d; P.d_pad = pl.d_pad; P.kc = pl.kc; P.n_chunks = pl.n_chunks;
    P.stages = pl.stages; P.rt = pl.rt;
    P.world = world; P.rank_base = a.rank_base; P.ctas_per_rank = a.ctas_per_rank;
    P.n_global = a.n_global; P.xr = a.xr; P.cta_stride = pl.cta_stride;
    P.check_interval = p.check_interval; P.state_cap = pl.state_cap; P.resident = pl.resident ? 1 : 0;
    P.bin_words = pl.bin_words;
    P.dp = pl.dp > 0 ? pl.dp : pl.d_pad;
    P.mix_nseg = pl.mix_nseg; P.mix_nc = pl.mix_nc; P.mix_nbw = pl.mix_nbw;
    for (int i = 0; i < MIX_MAXSEG; ++i) P.mix_seg[i] = pl.mix_seg[i];
    P.gram = gram;
    P.cache_slots = pl.cache_slots;
    P.cache_hash = pl.cache_hash;
    P.cluster = pl.cluster > 0 ? 1 : 0;
    P.crow = pl.crow;
    P.crw = pl.crw;
    P.independent = a.independent ? 1 : 0;
    for (int r = 0; r < world; ++r) {
        P.xr_rank[r] = a.independent ? a.xr_rank[r] : a.xr;
        P.max_iter_rank[r] = a.independent ? a.max_iter_rank[r] : p.max_iter;
    }
    P.timeout_ns = a.timeout_ns;
    P.wss = p.wss;
    if (const char* e = getenv("SVMB200_POLL_NS")) P.poll_ns = atoi(e);
    if (const char* e = getenv("SVMB200_DBG_FAST_ONLY")) P.dbg_fast_only = atoi(e);
    P.xch_dup = xch_dup;
    // L2 residency of streamed X: keep the first tiles of every CTA block in L2
    // (SVMB200_L2_KEEP_MB, per GPU; tuning)
    if (!pl.resident && pl.bin_words == 0 && !gram && pl.mix_nseg == 0 && pl.esz == 4) {
        // (measured on W5 shards: 48 MB kept per GPU -> 125k rows 31.4 -> 30.1 us/iteration,
        // 1M rows 187 -> 184; more is not better, profiles/r1h/l2_keep_W5_shards.txt)
        long long keep_mb = pl.cache_slots == 0 ? 48 : 0;
        if (const char* e = getenv("SVMB200_L2_KEEP_MB")) keep_mb = atoll(e);
        const long long stage_bytes = (long long)pl.kc * pl.rt * 4;
        const long long ctas_here = (long long)a.ctas_per_rank * a.nranks_here;
        if (keep_mb > 0 && stage_bytes > 0) P.l2_keep_chunks = (int)((keep_mb << 20) / (stage_bytes * ctas_here));
        // L2 prefetch beyond the ring (tuning switch SVMB200_L2_PF, stages; default 0)
        if (const char* e = getenv("SVMB200_L2_PF")) P.l2_prefetch = atoi(e);
    }
    P.sys_scope = a.mbox_local_alloc ? 0 : 1;
    const bool want_timers = getenv("SVMB200_PHASE_TIMERS") != nullptr;
    for (int r = 0; r < world; ++r) { P.row_off[r] = a.row_off[r]; P.n_rows[r] = (int)a.n_rows[r]; P.mbox[r] = a.mbox[r]; }

    unsigned* d_keys = nullptr;
    unsigned char* d_code = nullptr;
    if (pl.esz == 1) {
        double* dv;
        if ((rc = dalloc((void**)&dv, 256 * 8))) { release(); return rc; }
        if ((rc = dalloc((void**)&d_keys, DICT_SLOTS * 4))) { release(); return rc; }
        if ((rc = dalloc((void**)&d_code, DICT_SLOTS))) { release(); return rc; }
        CKR(cudaMemcpyAsync(dv, a.dict_vals.data(), a.dict_vals.size() * 8, cudaMemcpyHostToDevice, st));
        CKR(cudaMemcpyAsync(d_keys, a.dict_keys.data(), DICT_SLOTS * 4, cudaMemcpyHostToDevice, st));
        CKR(cudaMemcpyAsync(d_code, a.dict_code.data(), DICT_SLOTS, cudaMemcpyHostToDevice, st));
        P.dict = dv;
        P.dict_n = (int)a.dict_vals.size();
    }
    if (pl.mix_nseg > 0) {
        int* dm;
        if ((rc = dalloc((void**)&dm, a.mix_map.size() * 4))) { release(); return rc; }
        CKR(cudaMemcpyAsync(dm, a.mix_map.data(), a.mix_map.size() * 4, cudaMemcpyHostToDevice, st));
        P.mix_map = dm;
        if (pl.cache_slots == 0 && getenv("SVMB200_NO_COMPACT_PIVOTS") == nullptr) {
            // the compact form of every row (pivot gathers; 4 (nc + nbw) bytes per row)
            uint32_t* xc;
            const long long ncw = pl.mix_nc + pl.mix_nbw;
            if ((rc = dalloc((void**)&xc, (size_t)a.n_global * ncw * 4))) { release(); return rc; }
            k_build_compact_rows<<<1184, 256, 0, st>>>(a.xr, a.n_global, (int)a.d, dm, pl.mix_nc, pl.mix_nbw, xc);
            counted();
            P.xcomp = xc;
        }
    }
    for (int r = a.rank_base; r < a.rank_base + a.nranks_here; ++r) {
        const long long nr = a.n_rows[r];
        float* xb; double* f; double* al; uint8_t* fl; Ctl* ctl;
        if ((rc = dalloc((void**)&xb, (size_t)pl.cta_stride * pl.G * pl.esz + 16))) { release(); return rc; }
        if ((rc = dalloc((void**)&f, (size_t)nr * 8 + 8))) { release(); return rc; }
        if ((rc = dalloc((void**)&fl, (size_t)nr + 8))) { release(); return rc; }
        if ((rc = dalloc((void**)&ctl, sizeof(Ctl)))) { release(); return rc; }
        if (pl.cache_slots > 0) {
            double* cache;
            if ((rc = dalloc((void**)&cache, (size_t)pl.cache_slots * (nr > 0 ? nr : 1) * 8))) { release(); return rc; }
            P.cache[r] = cache;
        }
        al = a.alpha_out[r];
        CKR(cudaMemsetAsync(xb, 0, (size_t)pl.cta_stride * pl.G * pl.esz, st));
        CKR(cudaMemsetAsync(ctl, 0, sizeof(Ctl), st));
        dim3 bg(256, pl.G);
        if (gram) {
            counted(1);   // init_state below
        } else if (pl.bin_words) {
            if (!P.xrbits) {
                uint32_t* xrb;
                if ((rc = dalloc((void**)&xrb, (size_t)a.n_global * pl.bin_words * 4))) { release(); return rc; }
                k_pack_bits<<<1024, 256, 0, st>>>(a.xr, a.n_global, (int)a.d, pl.bin_words, xrb);
                counted();
                P.xrbits = xrb;
            }
            counted(2);   // build + init_state below
            k_build_xbits<<<bg, 256, 0, st>>>(P.xrbits + a.row_off[r] * pl.bin_words, nr, pl.bin_words,
                                               (pl.bin_words + 3) & ~3, pl.G, pl.cta_stride,
                                               reinterpret_cast<uint32_t*>(xb));
        } else if (pl.esz == 1) {
            counted(2);   // build + init_state below
            k_build_xblk_dict<<<bg, 256, 0, st>>>(a.x_rank[r], nr, (int)a.d, pl.d_pad, pl.G, pl.rt, pl.cta_stride,
                                                  d_keys, d_code, reinterpret_cast<unsigned char*>(xb));
        } else if (pl.mix_nseg > 0) {
            counted(2);   // build + init_state below
            k_build_xblk_mixed<<<bg, 256, 0, st>>>(a.x_rank[r], nr, (int)a.d, P.mix_map, pl.mix_nc, pl.mix_nbw,
                                                   pl.d_pad, pl.G, pl.rt, pl.cta_stride, xb);
        } else {
            counted(2);   // build + init_state below
            k_build_xblk<<<bg, 256, 0, st>>>(a.x_rank[r], nr, (int)a.d, pl.d_pad, pl.G, pl.rt, pl.cta_stride, xb);
        }
        const long long woff = a.warm_global ? a.row_off[r] : 0;
        k_init_state<<<256, 256, 0, st>>>(a.y_rank[r], nr, p.C, a.alpha0 ? a.alpha0 + woff : nullptr,
                                          a.f0 ? a.f0 + woff : nullptr, f, al, fl);
        CKR(cudaGetLastError());
        P.xblk[r] = xb; P.f[r] = f; P.alpha[r] = al; P.flags[r] = fl; P.ctl[r] = ctl;
        if (a.mbox_local_alloc) {
            Mailbox* mb;
            if ((rc = dalloc((void**)&mb, mbox_bytes))) { release(); return rc; }
            CKR(cudaMemsetAsync(mb, 0, mbox_bytes, st));
            P.mbox[r] = mb;
        }
    }
    if (p.wss == 2 && p.kernel == SVM_LINEAR) {
        // K(x_t, x_t) of every row for the second-order gains (R13 order, as the oracle's dot)
        double* qs;
        if ((rc = dalloc((void**)&qs, (size_t)a.n_global * 8))) { release(); return rc; }
        k_self_dot<<<(unsigned)((a.n_global + 255) / 256), 256, 0, st>>>(a.xr, a.n_global, (int)a.d, qs);
        counted();
        P.qself = qs;
    }
    long long* dtrace = nullptr;
    if (a.trace && a.trace_cap > 0) {
        if ((rc = dalloc((void**)&dtrace, (size_t)a.trace_cap * 16))) { release(); return rc; }
        CKR(cudaMemsetAsync(dtrace, 0xff, (size_t)a.trace_cap * 16, st));
        P.trace = dtrace; P.trace_cap = a.trace_cap;
    } else if (a.trace_dev && a.dev_cap > 0) {
        P.trace = a.trace_dev; P.hist = a.hist_dev; P.trace_cap = a.dev_cap;
    }
    unsigned long long* skew_ts = nullptr;
    if (const char* e = getenv("SVMB200_SKEW_TS")) {
        const int n_it = atoi(e);
        const size_t bytes = (size_t)n_it * a.ctas_per_rank * world * 3 * 8;
        if (n_it > 0 && (rc = dalloc((void**)&skew_ts, bytes)) == SVM_OK) {
            CKR(cudaMemsetAsync(skew_ts, 0, bytes, st));
            P.dbg_ts = skew_ts; P.dbg_ts_n = n_it;
        } else if (n_it > 0) { release(); return rc; }
    }
    if (want_timers) {
        unsigned long long* tm;
        if ((rc = dalloc((void**)&tm, PH_N * sizeof(unsigned long long)))) { release(); return rc; }
        CKR(cudaMemsetAsync(tm, 0, PH_N * sizeof(unsigned long long), st));
        P.timers = tm;
    }
    unsigned long long* progress_h = nullptr;
    if (cudaHostAlloc(&progress_h, 64, cudaHostAllocMapped) == cudaSuccess) {
        *progress_h = 0;
        unsigned long long* pd = nullptr;
        if (cudaHostGetDevicePointer(&pd, progress_h, 0) == cudaSuccess) P.progress = pd;
    } else {
        progress_h = nullptr;
        cudaGetLastError();
    }
    if (a.pre_launch) {
        rc = a.pre_launch(a, P);
        if (rc) { release(); return rc; }
    }

    // ---- a2-a7: persistent launches
    cudaEvent_t e0, e1;
    CKR(cudaEventCreate(&e0));
    CKR(cudaEventCreate(&e1));
    CKR(cudaEventRecord(e0, st));
    if (ev_gram) { cudaEventDestroy(e0); e0 = ev_gram; }
    Ctl hc;
    memset(&hc, 0, sizeof(hc));
    Ctl hcr[MAXR];
    long long launches = 0;
    for (;;) {
        void* args[] = {(void*)&P};
        cudaError_t e;
        if (pl.cluster) {
            // clusters are independent (no exchange between them): a plain cluster launch
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = pl.cluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.gridDim = dim3(grid); cfg.blockDim = dim3(nthreads);
            cfg.dynamicSmemBytes = pl.smem; cfg.stream = st; cfg.attrs = at; cfg.numAttrs = 1;
            e = cudaLaunchKernelExC(&cfg, (const void*)fn, args);
        } else {
            e = cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(nthreads), args, pl.smem, st);
        }
        if (e != cudaSuccess) { release(); return fail(SVM_ECUDA, std::string("cooperative launch: ") + cudaGetErrorString(e)); }
        ++launches;
        counted();
        bool again = false;
        for (int r = a.rank_base; r < a.rank_base + a.nranks_here; ++r) {
            CKR(cudaMemcpyAsync(&hcr[r], P.ctl[r], sizeof(Ctl), cudaMemcpyDeviceToHost, st));
        }
        CKR(cudaStreamSynchronize(st));
        for (int r = a.rank_base; r < a.rank_base + a.nranks_here; ++r) again = again || hcr[r].state == ST_LIMIT;
        hc = hcr[a.rank_base];
        if (!again) break;
    }
    CKR(cudaEventRecord(e1, st));
    CKR(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (int r = a.rank_base; r < a.rank_base + a.nranks_here; ++r) {
        SolveOut& o = a.out_rank[r];
        o.seconds_solve = ms * 1e-3; o.launches = launches; o.iterations = hcr[r].it;
        o.state = hcr[r].state; o.b_up = hcr[r].b_up; o.b_low = hcr[r].b_low;
        o.cache_hits = hcr[r].cache_hits; o.cache_misses = hcr[r].cache_misses;
    }
    a.out.seconds_solve = ms * 1e-3;
    a.out.launches = launches;
    a.out.iterations = hc.it;
    a.out.state = hc.state;
    a.out.b_up = hc.b_up;
    a.out.b_low = hc.b_low;
    a.out.cache_hits = hc.cache_hits;
    a.out.cache_misses = hc.cache_misses;
    if (a.f_out) {
        for (int r = a.rank_base; r < a.rank_base + a.nranks_here; ++r)
            CKR(cudaMemcpyAsync(a.f_out + (a.f_out_global ? a.row_off[r] : 0), P.f[r],
                                (size_t)a.n_rows[r] * 8, a.f_out_kind, st));
    }
    if (skew_ts) {
        // diagnostic: how far apart the CTAs start their row passes and publish their records
        const int G = a.ctas_per_rank * world;
        const long long n_it = hc.it < P.dbg_ts_n ? hc.it : P.dbg_ts_n;
        std::vector<unsigned long long> h((size_t)P.dbg_ts_n * G * 3);
        CKR(cudaMemcpyAsync(h.data(), skew_ts, h.size() * 8, cudaMemcpyDeviceToHost, st));
        CKR(cudaStreamSynchronize(st));
        std::vector<double> late(G, 0.0), pass(G, 0.0), slate(G, 0.0);
        double spread_pub = 0, spread_start = 0;
        long long used = 0;
        for (long long it = 1; it < n_it; ++it) {           // (iteration 0 starts cold)
            const unsigned long long* e = h.data() + (size_t)it * G * 3;
            unsigned long long p0 = ~0ull, p1 = 0, s0 = ~0ull, s1 = 0;
            bool ok = true;
            for (int c = 0; c < G; ++c) {
                if (!e[3 * c] || !e[3 * c + 1]) { ok = false; break; }
                p0 = std::min(p0, e[3 * c + 1]); p1 = std::max(p1, e[3 * c + 1]);
                s0 = std::min(s0, e[3 * c]); s1 = std::max(s1, e[3 * c]);
            }
            if (!ok) continue;
            ++used;
            spread_pub += (double)(p1 - p0); spread_start += (double)(s1 - s0);
            for (int c = 0; c < G; ++c) {
                late[c] += (double)(e[3 * c + 1] - p0);
                slate[c] += (double)(e[3 * c] - s0);
                pass[c] += (double)(e[3 * c + 1] - e[3 * c]);
            }
        }
        if (used > 0) {
            std::vector<int> ord(G);
            for (int c = 0; c < G; ++c) { ord[c] = c; late[c] /= used; pass[c] /= used; slate[c] /= used; }
            std::sort(ord.begin(), ord.end(), [&](int x, int y) { return late[x] > late[y]; });
            std::vector<double> ps(pass);
            std::sort(ps.begin(), ps.end());
            fprintf(stderr, "[svmb200] skew over %lld iterations (ns): publish spread %.0f, row-pass start spread %.0f, "
                    "row pass min/median/max %.0f/%.0f/%.0f; latest publishers (cta smid late start_late pass):",
                    used, spread_pub / used, spread_start / used, ps[0], ps[G / 2], ps[G - 1]);
            const unsigned long long* e0 = h.data() + (size_t)1 * G * 3;
            for (int q = 0; q < std::min(G, 12); ++q) {
                const int c = ord[q];
                fprintf(stderr, " [%d %llu %.0f %.0f %.0f]", c, e0[3 * c + 2], late[c], slate[c], pass[c]);
            }
            fprintf(stderr, " earliest:");
            for (int q = G - 1; q >= std::max(0, G - 4); --q) {
                const int c = ord[q];
                fprintf(stderr, " [%d %llu %.0f %.0f %.0f]", c, e0[3 * c + 2], late[c], slate[c], pass[c]);
            }
            fprintf(stderr, "\n");
        }
    }
    if (P.timers) {
        unsigned long long tm[PH_N];
        CKR(cudaMemcpyAsync(tm, P.timers, sizeof(tm), cudaMemcpyDeviceToHost, st));
        CKR(cudaStreamSynchronize(st));
        const char* nm[PH_N] = {"S.waitC", "S.publish", "S.poll", "S.select", "S.pivot", "S.kul",
                                "C.waitA", "S.pollrounds", "C.dist", "C.waitB", "C.update", "C.reduce",
                                "S.cand", "S.build"};
        fprintf(stderr, "[svmb200] cycles/iter of CTA 0 over %lld iters (rpt=%d kc=%d stages=%d smem=%zu a_smem=%d resident=%d bin_words=%d cache=%d gram=%d cluster=%d l2keep=%d):",
                hc.it, pl.rpt, pl.kc, pl.stages, pl.smem, (int)pl.alpha_smem, (int)pl.resident, pl.bin_words,
                pl.cache_slots, gram ? 1 : 0, pl.cluster, P.l2_keep_chunks);
        for (int k = 0; k < PH_N; ++k)
            fprintf(stderr, " %s=%.0f", nm[k], hc.it ? (double)tm[k] / hc.it : 0.0);
        fprintf(stderr, "\n");
    }
    if (dtrace) {
        const long long nt = hc.it < a.trace_cap ? hc.it : a.trace_cap;
        CKR(cudaMemcpyAsync(a.trace, dtrace, (size_t)nt * 16, cudaMemcpyDeviceToHost, st));
    }
    release();
    CKR(cudaStreamSynchronize(st));
    if (progress_h) cudaFreeHost(progress_h);
    a.out.gram = gram != nullptr;
    a.out.plain_rows = !gram && pl.bin_words == 0 && pl.mix_nseg == 0 && pl.esz == 4;
    for (int r = a.rank_base; r < a.rank_base + a.nranks_here; ++r) {
        if (hcr[r].state == ST_TIMEOUT) return fail(SVM_ETIMEOUT, "device wait for the candidate exchange timed out");
        if (hcr[r].state != ST_CONVERGED && hcr[r].state != ST_MAXITER)
            return fail(SVM_ECUDA, "solver ended in state " + std::to_string(hcr[r].state));
    }
    return SVM_OK;
}

// Single-process solve over p.virtual_ranks ranks of the current device.  X, y, alpha
// are device pointers; alpha0/f0 (optional) device pointers; f_out any pointer of kind
// f_kind; trace host.
int train_device(const float* X, const int8_t* y, long long n, long long d, const svm_params& p,
                 double* alpha, const double* alpha0, const double* f0, double* f_out,
                 cudaMemcpyKind f_kind, long long* trace, long long trace_cap, cudaStream_t st,
                 SolveOut& out, long long* trace_dev, double* hist_dev, long long dev_cap, bool skip_detect) {
    if (p.shrink_window > 0 && !trace_dev) {
        if (p.virtual_ranks > 1) return fail(SVM_EINVAL, "shrinking runs on one rank (virtual_ranks = 1)");
        return train_shrink(X, y, n, d, p, alpha, alpha0, f0, f_kind == cudaMemcpyDeviceToDevice ? f_out : nullptr,
                            trace, trace_cap, st, out);
    }
    int n_sm = 0, max_smem = 0;
    int rc = device_limits(&n_sm, &max_smem);
    if (rc) return rc;
    const int vr = p.virtual_ranks;
    if (p.shrink_window > 0 && vr > 1) return fail(SVM_EINVAL, "shrinking runs on one rank (virtual_ranks = 1)");
    int ctas = p.ctas > 0 ? p.ctas : n_sm;
    if (ctas > n_sm) ctas = n_sm;
    const int cpr = ctas / vr;
    if (cpr < 1) return fail(SVM_EINVAL, "more virtual ranks than CTAs");
    SolveArgs a;
    a.p = p;
    a.n_global = n; a.d = d; a.xr = X;
    a.world = vr; a.rank_base = 0; a.nranks_here = vr; a.ctas_per_rank = cpr;
    a.n_sm = n_sm; a.max_smem = max_smem;
    const long long per = (n + vr - 1) / vr;           // rank r owns [r per, min(n, (r+1) per))
    for (int r = 0; r < vr; ++r) {
        const long long lo = r * per < n ? r * per : n;
        const long long hi = (r + 1) * per < n ? (r + 1) * per : n;
        a.row_off[r] = lo; a.n_rows[r] = hi - lo;
        if (a.n_rows[r] > a.n_rows_max) a.n_rows_max = a.n_rows[r];
        a.x_rank[r] = X + lo * d;
        a.y_rank[r] = y + lo;
        a.alpha_out[r] = alpha + lo;
    }
    a.mbox_local_alloc = true;
    a.stream = st;
    a.alpha0 = alpha0; a.f0 = f0;
    a.f_out = f_out; a.f_out_kind = f_kind; a.f_out_global = true;
    a.trace = trace; a.trace_cap = trace ? trace_cap : 0;
    a.trace_dev = trace_dev; a.hist_dev = hist_dev; a.dev_cap = dev_cap;
    a.skip_detect = skip_detect;
    rc = solve(a);
    out = a.out;
    return rc;
}

}  // namespace svmint

using namespace svmint;

namespace {

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// info (a10): iterations, state, b_up / b_low from the solve; n_sv and the dual objective
// W = 1/2 sum alpha_i (1 - y_i f_i) reduced on the device (finalize.cu) from device alpha, f, y
int fill_info(svm_info* info, const SolveOut& o, const svm_params& p, const double* alpha_dev,
              const double* f_dev, const int8_t* y_dev, long long n, cudaStream_t st, double t0,
              double h2d_s = 0.0) {
    if (!info) return SVM_OK;
    memset(info, 0, sizeof(*info));
    info->iterations = o.iterations;
    info->converged = (o.state == ST_CONVERGED);
    info->b_up = o.b_up;
    info->b_low = o.b_low;
    info->gap = o.b_low - o.b_up;
    info->seconds_solve = o.seconds_solve;
    info->launches = o.launches;
    info->cache_hits = o.cache_hits;
    info->cache_misses = o.cache_misses;
    info->seconds_h2d = h2d_s;
    double s[2];
    int rc = info_device(alpha_dev, f_dev, y_dev, n, p.sv_epsilon, st, s);
    if (rc) return rc;
    info->n_sv = (int)s[1];
    info->dual_objective = 0.5 * s[0];
    info->seconds_total = now_s() - t0;
    return SVM_OK;
}

}  // namespace

extern "C" int svm_train_ex(const float* X, const int8_t* y, int64_t n, int64_t d,
                            const svm_params* p_in, double* alpha, double* b, svm_info* info,
                            const svm_debug* dbg) {
    const double t0 = now_s();
    if (!X || !y || !alpha || !b) return fail(SVM_EINVAL, "null pointer");
    svm_params p;
    int rc = check_params(n, d, p_in, &p);
    if (rc) return rc;
    if (dbg && ((dbg->alpha0 == nullptr) != (dbg->f0 == nullptr)))
        return fail(SVM_EINVAL, "warm start needs both alpha0 and f0");
    cudaStream_t st;
    CKR(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    float* dX = nullptr; int8_t* dy = nullptr; double* dA = nullptr; double* dA0 = nullptr; double* dF0 = nullptr;
    double* dF = nullptr;
    cudaEvent_t h0 = nullptr, h1 = nullptr;
    float h2d_ms = 0.f;
    SolveOut o;
    do {
        if (cudaMallocAsync(&dX, (size_t)n * d * 4, st) != cudaSuccess ||
            cudaMallocAsync(&dy, (size_t)n, st) != cudaSuccess ||
            cudaMallocAsync(&dA, (size_t)n * 8, st) != cudaSuccess ||
            cudaMallocAsync(&dF, (size_t)n * 8, st) != cudaSuccess) {
            rc = fail(SVM_ENOMEM, "device allocation of the training set failed");
            break;
        }
        if (cudaEventCreate(&h0) != cudaSuccess || cudaEventCreate(&h1) != cudaSuccess) {
            rc = fail(SVM_ECUDA, "event creation failed");
            break;
        }
        cudaEventRecord(h0, st);
        if (cudaMemcpyAsync(dX, X, (size_t)n * d * 4, cudaMemcpyHostToDevice, st) != cudaSuccess ||
            cudaMemcpyAsync(dy, y, (size_t)n, cudaMemcpyHostToDevice, st) != cudaSuccess) {
            rc = fail(SVM_ECUDA, "H2D copy failed");
            break;
        }
        cudaEventRecord(h1, st);
        if (dbg && dbg->alpha0) {
            if (cudaMallocAsync(&dA0, (size_t)n * 8, st) != cudaSuccess ||
                cudaMallocAsync(&dF0, (size_t)n * 8, st) != cudaSuccess) {
                rc = fail(SVM_ENOMEM, "warm start allocation failed");
                break;
            }
            cudaMemcpyAsync(dA0, dbg->alpha0, (size_t)n * 8, cudaMemcpyHostToDevice, st);
            cudaMemcpyAsync(dF0, dbg->f0, (size_t)n * 8, cudaMemcpyHostToDevice, st);
        }
        if ((rc = validate_device(dX, dy, n, d, st, nullptr))) break;
        cudaEventElapsedTime(&h2d_ms, h0, h1);
        rc = train_device(dX, dy, n, d, p, dA, dA0, dF0, dF, cudaMemcpyDeviceToDevice,
                          dbg ? (long long*)dbg->pair_trace : nullptr, dbg ? dbg->pair_trace_cap : 0, st, o);
        if (rc) break;
        if ((rc = fill_info(info, o, p, dA, dF, dy, n, st, t0, h2d_ms * 1e-3))) break;
        if (cudaMemcpyAsync(alpha, dA, (size_t)n * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            (dbg && dbg->f_out && cudaMemcpyAsync(dbg->f_out, dF, (size_t)n * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess)) {
            rc = fail(SVM_ECUDA, "D2H copy failed");
            break;
        }
    } while (0);
    if (dX) cudaFreeAsync(dX, st);
    if (dy) cudaFreeAsync(dy, st);
    if (dA) cudaFreeAsync(dA, st);
    if (dF) cudaFreeAsync(dF, st);
    if (dA0) cudaFreeAsync(dA0, st);
    if (dF0) cudaFreeAsync(dF0, st);
    cudaError_t se = cudaStreamSynchronize(st);
    if (h0) cudaEventDestroy(h0);
    if (h1) cudaEventDestroy(h1);
    cudaStreamDestroy(st);
    if (rc) return rc;
    if (se != cudaSuccess) return fail(SVM_ECUDA, cudaGetErrorString(se));
    *b = -(o.b_up + o.b_low) / 2.0;
    if (info) info->seconds_total = now_s() - t0;
    return SVM_OK;
}

extern "C" int svm_train(const float* X, const int8_t* y, int64_t n, int64_t d, double C,
                         int kernel, double gamma, double tol, double* alpha, double* b) {
    svm_params p;
    memset(&p, 0, sizeof(p));
    p.C = C; p.kernel = kernel; p.gamma = gamma; p.tol = tol;
    return svm_train_ex(X, y, n, d, &p, alpha, b, nullptr, nullptr);
}

extern "C" int svm_train_dev(const float* X, const int8_t* y, int64_t n, int64_t d,
                             const svm_params* p_in, double* alpha, double* b, svm_info* info,
                             const svm_debug* dbg, void* cuda_stream) {
    const double t0 = now_s();
    if (!X || !y || !alpha || !b) return fail(SVM_EINVAL, "null pointer");
    svm_params p;
    int rc = check_params(n, d, p_in, &p);
    if (rc) return rc;
    if (dbg && ((dbg->alpha0 == nullptr) != (dbg->f0 == nullptr)))
        return fail(SVM_EINVAL, "warm start needs both alpha0 and f0");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    if ((rc = validate_device(X, y, n, d, st, nullptr))) return rc;
    SolveOut o;
    double* f_dev = (dbg && dbg->f_out) ? dbg->f_out : nullptr;
    double* f_tmp = nullptr;
    if (!f_dev) {
        CKR(cudaMallocAsync(&f_tmp, (size_t)n * 8, st));
        f_dev = f_tmp;
    }
    rc = train_device(X, y, n, d, p, alpha, dbg ? dbg->alpha0 : nullptr, dbg ? dbg->f0 : nullptr, f_dev,
                      cudaMemcpyDeviceToDevice, dbg ? (long long*)dbg->pair_trace : nullptr,
                      dbg ? dbg->pair_trace_cap : 0, st, o);
    if (!rc) rc = fill_info(info, o, p, alpha, f_dev, y, n, st, t0);
    if (f_tmp) cudaFreeAsync(f_tmp, st);
    if (rc) return rc;
    *b = -(o.b_up + o.b_low) / 2.0;
    return SVM_OK;
}

extern "C" int svm_train_batch_dev(int B, const float* const* X, const int8_t* const* y,
                                   const int64_t* n, int64_t d, const svm_params* p_in,
                                   double* const* alpha, double* b_out, svm_info* info,
                                   void* cuda_stream) {
    const double t0 = now_s();
    if (B < 1 || !X || !y || !n || !alpha || !b_out) return fail(SVM_EINVAL, "null pointer or B < 1");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    int n_sm = 0, max_smem = 0;
    int rc = device_limits(&n_sm, &max_smem);
    if (rc) return rc;
    for (int b0 = 0; b0 < B; b0 += MAXR) {
        const int nb = (B - b0) < MAXR ? (B - b0) : MAXR;
        SolveArgs a;
        svm_params p;
        long long n_max = 0;
        for (int k = 0; k < nb; ++k) {
            if (!X[b0 + k] || !y[b0 + k] || !alpha[b0 + k]) return fail(SVM_EINVAL, "null problem pointer");
            if ((rc = check_params(n[b0 + k], d, p_in, &p))) return rc;
            if (p.wss == 2) return fail(SVM_EINVAL, "wss = 2 is not supported by svm_train_batch_dev");
            if ((rc = validate_device(X[b0 + k], y[b0 + k], n[b0 + k], d, st, nullptr))) return rc;
            a.max_iter_rank[k] = p.max_iter;
            if (p_in->max_iter <= 0) a.max_iter_rank[k] = (10 * n[b0 + k] > 10000) ? 10 * n[b0 + k] : 10000;
            n_max = n[b0 + k] > n_max ? n[b0 + k] : n_max;
        }
        a.p = p;
        a.n_global = n_max; a.d = d; a.xr = X[b0];
        a.world = nb; a.rank_base = 0; a.nranks_here = nb;
        int ctas = p.ctas > 0 ? p.ctas : n_sm;
        if (ctas > n_sm) ctas = n_sm;
        a.ctas_per_rank = ctas / nb;
        if (a.ctas_per_rank < 1)
            return fail(SVM_EINVAL, "fewer CTAs (" + std::to_string(ctas) + ") than problems in a launch (" +
                                        std::to_string(nb) + ")");
        a.n_sm = n_sm; a.max_smem = max_smem;
        a.independent = true;
        for (int k = 0; k < nb; ++k) {
            a.row_off[k] = 0; a.n_rows[k] = n[b0 + k];
            a.x_rank[k] = X[b0 + k]; a.y_rank[k] = y[b0 + k]; a.alpha_out[k] = alpha[b0 + k];
            a.xr_rank[k] = X[b0 + k];
        }
        a.n_rows_max = n_max;
        a.mbox_local_alloc = true;
        a.stream = st;
        a.f_out = nullptr;
        if ((rc = solve(a))) return rc;
        for (int k = 0; k < nb; ++k) {
            const SolveOut& o = a.out_rank[k];
            b_out[b0 + k] = -(o.b_up + o.b_low) / 2.0;
            if (info) {
                svm_info& in = info[b0 + k];
                memset(&in, 0, sizeof(in));
                in.iterations = o.iterations; in.converged = o.state == ST_CONVERGED;
                in.b_up = o.b_up; in.b_low = o.b_low; in.gap = o.b_low - o.b_up;
                in.seconds_solve = o.seconds_solve; in.launches = o.launches;
                in.cache_hits = o.cache_hits; in.cache_misses = o.cache_misses;
                in.seconds_total = now_s() - t0;
            }
        }
    }
    return SVM_OK;
}

extern "C" int svm_predict_dev_ex(const float* X_sv, const double* coef, int64_t n_sv, int64_t d,
                                  double b, int kernel, double gamma, const float* X_test, int64_t m,
                                  double* dec, int mode, void* cuda_stream) {
    if (d < 1 || m < 0 || n_sv < 0) return fail(SVM_EINVAL, "bad sizes");
    if (m == 0) return SVM_OK;
    if (!dec || !X_test || (n_sv > 0 && (!X_sv || !coef))) return fail(SVM_EINVAL, "null pointer");
    if (kernel != SVM_LINEAR && kernel != SVM_RBF) return fail(SVM_EINVAL, "unknown kernel");
    if (kernel == SVM_RBF && !(gamma > 0.0)) return fail(SVM_EINVAL, "RBF gamma must be > 0");
    if (mode != SVM_PREDICT_EXACT && mode != SVM_PREDICT_TENSOR) return fail(SVM_EINVAL, "unknown predict mode");
    return predict_device(X_sv, coef, n_sv, d, b, kernel, gamma, X_test, m, dec,
                          (cudaStream_t)cuda_stream, mode);
}

extern "C" int svm_predict_dev(const float* X_sv, const double* coef, int64_t n_sv, int64_t d,
                               double b, int kernel, double gamma, const float* X_test, int64_t m,
                               double* dec, void* cuda_stream) {
    return svm_predict_dev_ex(X_sv, coef, n_sv, d, b, kernel, gamma, X_test, m, dec,
                              SVM_PREDICT_EXACT, cuda_stream);
}

extern "C" int svm_predict_ex(const float* X_sv, const double* coef, int64_t n_sv, int64_t d,
                              double b, int kernel, double gamma, const float* X_test, int64_t m,
                              double* dec, int mode) {
    if (d < 1 || m < 0 || n_sv < 0) return fail(SVM_EINVAL, "bad sizes");
    if (m == 0) return SVM_OK;
    if (!dec || !X_test || (n_sv > 0 && (!X_sv || !coef))) return fail(SVM_EINVAL, "null pointer");
    cudaStream_t st;
    CKR(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    float *dS = nullptr, *dT = nullptr;
    double *dC = nullptr, *dD = nullptr;
    int rc = SVM_OK;
    do {
        if ((n_sv > 0 && (cudaMallocAsync(&dS, (size_t)n_sv * d * 4, st) != cudaSuccess ||
                          cudaMallocAsync(&dC, (size_t)n_sv * 8, st) != cudaSuccess)) ||
            cudaMallocAsync(&dT, (size_t)m * d * 4, st) != cudaSuccess ||
            cudaMallocAsync(&dD, (size_t)m * 8, st) != cudaSuccess) {
            rc = fail(SVM_ENOMEM, "device allocation for predict failed");
            break;
        }
        if (n_sv > 0) {
            cudaMemcpyAsync(dS, X_sv, (size_t)n_sv * d * 4, cudaMemcpyHostToDevice, st);
            cudaMemcpyAsync(dC, coef, (size_t)n_sv * 8, cudaMemcpyHostToDevice, st);
        }
        cudaMemcpyAsync(dT, X_test, (size_t)m * d * 4, cudaMemcpyHostToDevice, st);
        rc = svm_predict_dev_ex(dS, dC, n_sv, d, b, kernel, gamma, dT, m, dD, mode, st);
        if (rc) break;
        if (cudaMemcpyAsync(dec, dD, (size_t)m * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess)
            rc = fail(SVM_ECUDA, "D2H copy failed");
    } while (0);
    if (dS) cudaFreeAsync(dS, st);
    if (dC) cudaFreeAsync(dC, st);
    if (dT) cudaFreeAsync(dT, st);
    if (dD) cudaFreeAsync(dD, st);
    cudaError_t se = cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    if (rc) return rc;
    if (se != cudaSuccess) return fail(SVM_ECUDA, cudaGetErrorString(se));
    return SVM_OK;
}

extern "C" int svm_predict(const float* X_sv, const double* coef, int64_t n_sv, int64_t d,
                           double b, int kernel, double gamma, const float* X_test, int64_t m,
                           double* dec) {
    return svm_predict_ex(X_sv, coef, n_sv, d, b, kernel, gamma, X_test, m, dec, SVM_PREDICT_EXACT);
}

extern "C" const char* svm_last_error(void) { return g_err.c_str(); }
extern "C" int64_t svm_kernel_launches(void) { return g_launches; }
extern "C" const char* svm_last_plan(void) { return g_plan.c_str(); }
extern "C" const char* svm_version(void) { return "svmb200 0.1 sm_100a"; }
