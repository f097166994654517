// finalize.cu -- row a10 on the device: the solve's summary numbers and the model's
// support vectors, so no caller has to copy alpha / f to the host or run tensor
// arithmetic to build a predictor.
//
//   info_device            n_sv = |{alpha_i > sv_epsilon}| and
//                          W = 1/2 sum_i alpha_i (1 - y_i f_i)   (the dual objective in its f
//                          form, identity from S:L176), reduced in a fixed order
//   svm_support_vectors_dev  the support set {i : alpha_i > sv_epsilon} in ascending i:
//                          X_sv rows, coef_i = alpha_i y_i (exact: y = +-1), indices
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "svm_internal.h"

namespace svmint {

constexpr int FIN_BLOCKS = 148;
constexpr int FIN_THREADS = 256;

// per block: partial W sum (thread-strided, then a fixed tree) and SV count
__global__ void k_info_partial(const double* __restrict__ alpha, const double* __restrict__ f,
                               const int8_t* __restrict__ y, long long n, double eps,
                               double* __restrict__ part_w, unsigned long long* __restrict__ part_n) {
    __shared__ double sw[FIN_THREADS];
    __shared__ unsigned long long sn[FIN_THREADS];
    double w = 0.0;
    unsigned long long c = 0;
    for (long long j = (long long)blockIdx.x * FIN_THREADS + threadIdx.x; j < n; j += (long long)gridDim.x * FIN_THREADS) {
        const double a = alpha[j];
        c += a > eps;
        if (a != 0.0) w += a * (1.0 - (double)y[j] * f[j]);
    }
    sw[threadIdx.x] = w;
    sn[threadIdx.x] = c;
    __syncthreads();
    for (int s = FIN_THREADS / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) { sw[threadIdx.x] += sw[threadIdx.x + s]; sn[threadIdx.x] += sn[threadIdx.x + s]; }
        __syncthreads();
    }
    if (threadIdx.x == 0) { part_w[blockIdx.x] = sw[0]; part_n[blockIdx.x] = sn[0]; }
}

__global__ void k_info_final(const double* __restrict__ part_w, const unsigned long long* __restrict__ part_n,
                             int nb, double* __restrict__ out) {
    if (threadIdx.x == 0) {
        double w = 0.0;
        unsigned long long c = 0;
        for (int b = 0; b < nb; ++b) { w += part_w[b]; c += part_n[b]; }
        out[0] = w;                     // sum alpha_i (1 - y_i f_i) (the caller halves it)
        out[1] = (double)c;
    }
}

// Summary of one rank's rows: out_host[0] = sum alpha (1 - y f), out_host[1] = n_sv.
int info_device(const double* alpha, const double* f, const int8_t* y, long long n, double eps,
                cudaStream_t st, double out_host[2]) {
    out_host[0] = 0.0; out_host[1] = 0.0;
    if (n <= 0) return SVM_OK;
    double* pw;
    CKR(cudaMallocAsync(&pw, FIN_BLOCKS * (8 + 8) + 16, st));
    unsigned long long* pn = reinterpret_cast<unsigned long long*>(pw + FIN_BLOCKS);
    double* o = pw + 2 * FIN_BLOCKS;
    k_info_partial<<<FIN_BLOCKS, FIN_THREADS, 0, st>>>(alpha, f, y, n, eps, pw, pn);
    k_info_final<<<1, 32, 0, st>>>(pw, pn, FIN_BLOCKS, o);
    counted(2);
    CKR(cudaMemcpyAsync(out_host, o, 16, cudaMemcpyDeviceToHost, st));
    CKR(cudaFreeAsync(pw, st));
    CKR(cudaStreamSynchronize(st));
    return SVM_OK;
}

// ---- support-vector compaction (stable: ascending row index)
constexpr int SV_TILE = 256;

__global__ void k_sv_count(const double* __restrict__ alpha, long long n, long long chunk, double eps,
                           unsigned long long* __restrict__ cnt) {
    __shared__ unsigned int wc[SV_TILE / 32];
    const long long lo = (long long)blockIdx.x * chunk;
    const long long hi = lo + chunk < n ? lo + chunk : n;
    unsigned int c = 0;
    for (long long j = lo + threadIdx.x; j < hi; j += SV_TILE) c += alpha[j] > eps;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) wc[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < SV_TILE / 32; ++w) s += wc[w];
        cnt[blockIdx.x] = s;
    }
}

// exclusive scan of the block counts (one block; nb <= 4096), total in cnt[nb]
__global__ void k_sv_scan(unsigned long long* __restrict__ cnt, int nb) {
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int b = 0; b < nb; ++b) { const unsigned long long c = cnt[b]; cnt[b] = s; s += c; }
        cnt[nb] = s;
    }
}

__global__ void k_sv_scatter(const float* __restrict__ X, const int8_t* __restrict__ y,
                             const double* __restrict__ alpha, long long n, int d, long long chunk, double eps,
                             const unsigned long long* __restrict__ base, float* __restrict__ Xsv,
                             double* __restrict__ coef, long long* __restrict__ index) {
    __shared__ unsigned int wc[SV_TILE / 32];
    __shared__ long long rows[SV_TILE];
    const long long lo = (long long)blockIdx.x * chunk;
    const long long hi = lo + chunk < n ? lo + chunk : n;
    long long pos = (long long)base[blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (long long t0 = lo; t0 < hi; t0 += SV_TILE) {
        const long long j = t0 + threadIdx.x;
        const bool sv = j < hi && alpha[j] > eps;
        const unsigned m = __ballot_sync(0xffffffffu, sv);
        if (lane == 0) wc[warp] = __popc(m);
        __syncthreads();
        unsigned int before = 0, total = 0;
        for (int w = 0; w < SV_TILE / 32; ++w) { if (w < warp) before += wc[w]; total += wc[w]; }
        const unsigned int r = before + __popc(m & ((1u << lane) - 1u));
        if (sv) {
            const long long p = pos + r;
            coef[p] = y[j] > 0 ? alpha[j] : -alpha[j];
            if (index) index[p] = j;
            rows[r] = j;
        }
        __syncthreads();
        if (Xsv) {
            // copy the tile's SV rows: one warp per row, coalesced over the features
            for (unsigned int q = warp; q < total; q += SV_TILE / 32) {
                const float* src = X + rows[q] * (long long)d;
                float* dst = Xsv + (pos + q) * (long long)d;
                for (int k = lane; k < d; k += 32) dst[k] = src[k];
            }
        }
        pos += total;
        __syncthreads();
    }
}

}  // namespace svmint

using namespace svmint;

extern "C" int svm_support_vectors_dev(const float* X, const int8_t* y, const double* alpha, int64_t n,
                                       int64_t d, double sv_epsilon, float* X_sv, double* coef,
                                       int64_t* sv_index, int64_t* n_sv, void* cuda_stream) {
    if (!alpha || !n_sv || n < 0 || d < 1) return fail(SVM_EINVAL, "null pointer or bad sizes");
    if ((X_sv || coef || sv_index) && (!coef || !y || (X_sv && !X)))
        return fail(SVM_EINVAL, "coef (and y, and X with X_sv) are required when writing the support set");
    if (!(sv_epsilon > 0.0)) sv_epsilon = 1e-8;
    *n_sv = 0;
    if (n == 0) return SVM_OK;
    cudaStream_t st = (cudaStream_t)cuda_stream;
    long long chunk = ((n + 1023) / 1024 + SV_TILE - 1) / SV_TILE * SV_TILE;
    if (chunk < SV_TILE) chunk = SV_TILE;
    const int nb = (int)((n + chunk - 1) / chunk);
    unsigned long long* cnt;
    CKR(cudaMallocAsync(&cnt, (size_t)(nb + 1) * 8, st));
    k_sv_count<<<nb, SV_TILE, 0, st>>>(alpha, n, chunk, sv_epsilon, cnt);
    k_sv_scan<<<1, 32, 0, st>>>(cnt, nb);
    counted(2);
    if (coef) {
        k_sv_scatter<<<nb, SV_TILE, 0, st>>>(X, y, alpha, n, (int)d, chunk, sv_epsilon, cnt, X_sv, coef,
                                            (long long*)sv_index);
        counted();
    }
    unsigned long long tot = 0;
    CKR(cudaMemcpyAsync(&tot, cnt + nb, 8, cudaMemcpyDeviceToHost, st));
    CKR(cudaFreeAsync(cnt, st));
    CKR(cudaStreamSynchronize(st));
    CKR(cudaGetLastError());
    *n_sv = (int64_t)tot;
    return SVM_OK;
}
