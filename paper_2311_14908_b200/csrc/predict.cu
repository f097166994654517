// predict.cu -- batched decision values:
//   dec_i = sum_s coef_s K(sv_s, x_i) + b,   coef_s = alpha_s y_s.
//
// Exact path (this file, k_predict_exact): fp64 SIMT, one test row per thread, support
// vectors consumed in blocks of SB with their feature chunks staged in shared memory;
// each (i, s) distance accumulates in ascending k with one fma per term, the kernel
// value is the correctly rounded exp, and the SB terms are added to the running sum in
// ascending s -- the oracle's order, so decision values match it bit for bit.
#include <cuda_runtime.h>

#include <cstdlib>

#include "predict_tc.cuh"
#include "svm_exp.cuh"
#include "svm_internal.h"

namespace svmint {

namespace {
constexpr int TI = 256;   // test rows per CTA (one per thread)
constexpr int SB = 8;     // support vectors per block
constexpr int KC = 32;    // features per shared-memory chunk
}

template <int KERNEL>
__global__ void __launch_bounds__(TI) k_predict_exact(const float* __restrict__ Xsv,
                                                      const double* __restrict__ coef, long long nsv,
                                                      int d, double b, double gamma,
                                                      const float* __restrict__ Xt, long long m,
                                                      double* __restrict__ dec) {
    __shared__ float tt[KC][TI + 1];
    __shared__ double sv[SB][KC];
    const int tid = threadIdx.x;
    const long long i0 = (long long)blockIdx.x * TI;
    const long long i = i0 + tid;
    double acc = 0.0;
    for (long long s0 = 0; s0 < nsv; s0 += SB) {
        const int nb = (int)((nsv - s0) < SB ? (nsv - s0) : SB);
        double dist[SB];
#pragma unroll
        for (int s = 0; s < SB; ++s) dist[s] = 0.0;
        for (int k0 = 0; k0 < d; k0 += KC) {
            const int kc = (d - k0) < KC ? (d - k0) : KC;
            __syncthreads();
            for (int e = tid; e < TI * KC; e += TI) {
                const int row = e / KC, kk = e % KC;
                tt[kk][row] = (i0 + row < m && kk < kc) ? Xt[(i0 + row) * d + k0 + kk] : 0.0f;
            }
            for (int e = tid; e < SB * KC; e += TI) {
                const int s = e / KC, kk = e % KC;
                sv[s][kk] = (s < nb && kk < kc) ? (double)Xsv[(s0 + s) * d + k0 + kk] : 0.0;
            }
            __syncthreads();
            for (int kk = 0; kk < kc; ++kk) {
                const double x = tt[kk][tid];
#pragma unroll
                for (int s = 0; s < SB; ++s) {
                    if (KERNEL == 1) {
                        const double e = sv[s][kk] - x;
                        dist[s] = fma(e, e, dist[s]);
                    } else {
                        dist[s] = fma(sv[s][kk], x, dist[s]);
                    }
                }
            }
        }
        for (int s = 0; s < nb; ++s) {
            const double K = (KERNEL == 1) ? svmexp::exp_cr(-(gamma * dist[s])) : dist[s];
            acc = acc + coef[s0 + s] * K;
        }
    }
    if (i < m) dec[i] = acc + b;
}

__global__ void k_scale_norms(double* __restrict__ q, long long n, double s) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        q[i] = s * q[i];
}

__global__ void k_pad_coef(const double* __restrict__ coef, long long n, long long n_pad, double* __restrict__ out) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n_pad; i += (long long)gridDim.x * blockDim.x)
        out[i] = i < n ? coef[i] : 0.0;
}

__global__ void k_interleave(const double* __restrict__ a, const double* __restrict__ b, long long n,
                             double2* __restrict__ out) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = make_double2(a[i], b[i]);
}

// Tensor-core path (predict_tc.cuh): pack both operands to 3xTF32 core-matrix blocks,
// then one CTA per 128 test rows.  Tuning switches: SVMB200_PREDICT_EXP (the epilogue's exp,
// 0-4, see k_predict_tc), SVMB200_PREDICT_BN (128 or 256 support vectors per tile).
template <int BN_>
static int predict_tc_launch(const float* X_sv, const double* coef, long long n_sv, long long d, double b,
                             int kernel, double gamma, const float* X_test, long long m, double* dec,
                             cudaStream_t st, int expv) {
    using namespace svmtc;
    using Cf = TcCfg<BN_>;
    const long long m_pad = (m + BM - 1) / BM * BM;
    const long long n_pad = (n_sv + Cf::BN - 1) / Cf::BN * Cf::BN;
    const int k_chunks = (int)((d + Cf::BK - 1) / Cf::BK);
    float *pa = nullptr, *pb = nullptr;
    double *qt = nullptr, *qs = nullptr, *cf = nullptr;
    double2* qc = nullptr;
    const size_t a_floats = (size_t)m_pad * k_chunks * Cf::BK * 2, b_floats = (size_t)n_pad * k_chunks * Cf::BK * 2;
    if (cudaMallocAsync(&pa, a_floats * 4, st) != cudaSuccess || cudaMallocAsync(&pb, b_floats * 4, st) != cudaSuccess ||
        cudaMallocAsync(&qt, m_pad * 8, st) != cudaSuccess || cudaMallocAsync(&qs, n_pad * 8, st) != cudaSuccess ||
        cudaMallocAsync(&cf, n_pad * 8, st) != cudaSuccess || cudaMallocAsync(&qc, n_pad * 16, st) != cudaSuccess) {
        if (pa) cudaFreeAsync(pa, st); if (pb) cudaFreeAsync(pb, st);
        if (qt) cudaFreeAsync(qt, st); if (qs) cudaFreeAsync(qs, st); if (cf) cudaFreeAsync(cf, st);
        if (qc) cudaFreeAsync(qc, st);
        return fail(SVM_ENOMEM, "predict workspace allocation failed");
    }
    k_pack_3xtf32<<<1184, 256, 0, st>>>(X_test, m, (int)d, k_chunks, m_pad, BM, Cf::BK, pa, qt);
    k_pack_3xtf32<<<1184, 256, 0, st>>>(X_sv, n_sv, (int)d, k_chunks, n_pad, Cf::BN, Cf::BK, pb, qs);
    k_pad_coef<<<256, 256, 0, st>>>(coef, n_sv, n_pad, cf);
    counted(3);
    if (kernel == SVM_RBF) {                       // the epilogue takes -gamma |s|^2 per SV
        k_scale_norms<<<256, 256, 0, st>>>(qs, n_pad, -gamma);
        counted();
    }
    k_interleave<<<256, 256, 0, st>>>(qs, cf, n_pad, qc);
    counted();
    const size_t smem = (size_t)Cf::STAGES * Cf::STAGE_BYTES;
    auto fn = kernel != SVM_RBF ? k_predict_tc<0, 0, BN_>
            : expv == 0 ? k_predict_tc<1, 0, BN_> : expv == 1 ? k_predict_tc<1, 1, BN_>
            : expv == 2 ? k_predict_tc<1, 2, BN_> : expv == 3 ? k_predict_tc<1, 3, BN_>
            : expv == 4 ? k_predict_tc<1, 4, BN_> : k_predict_tc<1, 5, BN_>;
    CKR(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    fn<<<(unsigned)(m_pad / BM), NTHREADS, smem, st>>>(pa, pb, qt, qc, k_chunks, (int)(n_pad / Cf::BN), m, b,
                                                        gamma, dec);
    counted();
    CKR(cudaGetLastError());
    cudaFreeAsync(pa, st); cudaFreeAsync(pb, st); cudaFreeAsync(qt, st); cudaFreeAsync(qs, st); cudaFreeAsync(cf, st);
    cudaFreeAsync(qc, st);
    return SVM_OK;
}

int predict_device_tc(const float* X_sv, const double* coef, long long n_sv, long long d, double b,
                      int kernel, double gamma, const float* X_test, long long m, double* dec,
                      cudaStream_t st) {
    pool_setup();
    int expv = 5;            // measured (1M x 284k x 256): 0 1.01 s, 3 0.90 s, 4 1.11 s (BN = 128);
                             // BN = 256: 3 0.850 s, 5 0.835 s
    if (const char* e = getenv("SVMB200_PREDICT_EXP")) expv = atoi(e);
    int bn = 256;            // measured with expv 3: BN 128 0.91 s, BN 256 0.85 s
    if (const char* e = getenv("SVMB200_PREDICT_BN")) bn = atoi(e);
    if (bn == 256) return predict_tc_launch<256>(X_sv, coef, n_sv, d, b, kernel, gamma, X_test, m, dec, st, expv);
    return predict_tc_launch<128>(X_sv, coef, n_sv, d, b, kernel, gamma, X_test, m, dec, st, expv);
}

int predict_device(const float* X_sv, const double* coef, long long n_sv, long long d, double b,
                   int kernel, double gamma, const float* X_test, long long m, double* dec,
                   cudaStream_t st, int mode) {
    if (mode == SVM_PREDICT_TENSOR && n_sv > 0)
        return predict_device_tc(X_sv, coef, n_sv, d, b, kernel, gamma, X_test, m, dec, st);
    const long long grid = (m + TI - 1) / TI;
    if (grid > 0x7fffffffll) return fail(SVM_EINVAL, "too many test rows");
    if (kernel == SVM_RBF)
        k_predict_exact<1><<<(unsigned)grid, TI, 0, st>>>(X_sv, coef, n_sv, (int)d, b, gamma, X_test, m, dec);
    else
        k_predict_exact<0><<<(unsigned)grid, TI, 0, st>>>(X_sv, coef, n_sv, (int)d, b, gamma, X_test, m, dec);
    counted();
    CKR(cudaGetLastError());
    return SVM_OK;
}

}  // namespace svmint
