// gram.cu -- the full kernel matrix for the Gram path.
//
// K[i][j] = K(x_i, x_j) for all i, j < n, fp64, row-major [n][ld] (or column-blocked for the
// GD trainer, see gd.cu), computed with the same
// arithmetic as the streaming row pass (R13: ascending-k fp64 recurrence, one fma per
// term, from the fp32 inputs; R14: correctly rounded exp; R16: K_ii = 1), so a solve that
// reads rows of K takes exactly the same decisions as one that recomputes them.  The
// recurrence is sequential in k for every (i, j), so this is a SIMT fp64 kernel (no tensor
// cores: tcgen05 has no fp64 kind, and a TF32/3xTF32 Gram would change the values).
//
// Tiles of 64 x 64 outputs, 256 threads, 4 x 4 outputs per thread; 32-feature slabs of
// both row blocks staged in shared memory as fp64 (exact widening); only tiles with
// bi <= bj are computed and mirrored (K is symmetric bit for bit: (a - b)^2 == (b - a)^2).
#include <cuda_runtime.h>

#include "svm_exp.cuh"
#include "svm_internal.h"

namespace svmint {

namespace {
constexpr int GT = 64;    // tile edge
constexpr int GK = 32;    // features per slab
}

template <int KERNEL>
__global__ void __launch_bounds__(256) k_gram(const float* __restrict__ X, long long n, int d,
                                              double gamma, double* __restrict__ K, long long ld, int blk) {
    __shared__ double a[GK][GT + 1];
    __shared__ double b[GK][GT + 1];
    // blockIdx.x enumerates the upper-triangular tile pairs (bi <= bj)
    const long long nt = (n + GT - 1) / GT;
    long long t = blockIdx.x, bi = 0;
    while (t >= nt - bi) { t -= nt - bi; ++bi; }
    const long long bj = bi + t;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;      // 16 x 16 threads
    double acc[4][4];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = 0.0;
    for (int k0 = 0; k0 < d; k0 += GK) {
        const int kc = (d - k0) < GK ? (d - k0) : GK;
        __syncthreads();
        for (int e = threadIdx.x; e < GT * GK; e += 256) {
            const int r = e / GK, kk = e - r * GK;
            const long long ia = bi * GT + r, ib = bj * GT + r;
            a[kk][r] = (ia < n && kk < kc) ? (double)X[ia * d + k0 + kk] : 0.0;
            b[kk][r] = (ib < n && kk < kc) ? (double)X[ib * d + k0 + kk] : 0.0;
        }
        __syncthreads();
        for (int kk = 0; kk < kc; ++kk) {
            double av[4], bv[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) { av[p] = a[kk][ty * 4 + p]; bv[p] = b[kk][tx * 4 + p]; }
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (KERNEL == 1) {
                        const double e = av[p] - bv[q];
                        acc[p][q] = fma(e, e, acc[p][q]);
                    } else {
                        acc[p][q] = fma(av[p], bv[q], acc[p][q]);
                    }
                }
        }
    }
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const long long i = bi * GT + ty * 4 + p, j = bj * GT + tx * 4 + q;
            if (i < n && j < n) {
                double v;
                if (KERNEL == 1) v = (i == j) ? 1.0 : svmexp::exp_cr(-(gamma * acc[p][q]));
                else v = acc[p][q];
                if (blk > 0) {
                    // column-blocked layout (gd.cu): K[r][c] at ((c / blk) n + r) blk + c % blk
                    K[((j / blk) * n + i) * blk + (j % blk)] = v;
                    K[((i / blk) * n + j) * blk + (i % blk)] = v;
                } else {
                    K[i * ld + j] = v;
                    K[j * ld + i] = v;
                }
            }
        }
}

int gram_device(const float* X, long long n, long long d, int kernel, double gamma, double* K,
                cudaStream_t st, long long ld, int blk) {
    if (ld <= 0) ld = n;
    const long long nt = (n + GT - 1) / GT;
    const long long tiles = nt * (nt + 1) / 2;
    if (tiles > 0x7fffffffll) return fail(SVM_EINVAL, "Gram too large");
    if (kernel == SVM_RBF)
        k_gram<1><<<(unsigned)tiles, 256, 0, st>>>(X, n, (int)d, gamma, K, ld, blk);
    else
        k_gram<0><<<(unsigned)tiles, 256, 0, st>>>(X, n, (int)d, gamma, K, ld, blk);
    counted();
    CKR(cudaGetLastError());
    return SVM_OK;
}

}  // namespace svmint
