// gd.cu -- projected-gradient dual trainer on B200.
//
// The paper's second implementation is a TensorFlow graph: "describing the Gaussian RBF
// kernel function ... declaring the gradient descent optimizer algorithm" (P:L174-179,
// §3.3, Fig. 5).  Read as full-batch projected gradient ascent on the SMO dual W
// (R23-R26; include/svmb200.h svm_train_gd_dev):
//     alpha^0 = 0;  each epoch  g = K (alpha o y),  alpha <- clamp(alpha + lr (1 - y o g), 0, C)
//
// B200 design:
//   * K is built once in HBM as fp64 with the row pass's arithmetic (gram.cu, R13/R14/R16;
//     symmetric bit for bit) in a column-blocked layout: block b holds columns
//     [b bc, b bc + bc) of every row, row-major within the block, so the J-row slab one CTA
//     consumes per stage is one contiguous bulk copy (J bc 8 bytes).
//   * k_gd_epoch: one epoch is one pass over K -- a GEMV bound by HBM bandwidth (8 n^2
//     bytes per epoch, 2 flops per 8 bytes).  Thread i of a CTA owns output i0 + i and sums
//     g_i = sum_j K_ij v_j sequentially in ascending j (R24) -- the exact order of the
//     oracle, so the result is bit-identical -- reading K by columns: since K is symmetric,
//     K_ij = K[j][i], and at step j the CTA's threads read the contiguous segment
//     K[j][i0 .. i0 + bc) (coalesced).  A producer warp streams J-row slabs of the CTA's
//     column block (one cp.async.bulk of J bc 8 bytes, plus one of the matching J entries
//     of v = alpha o y) through a ring of shared-memory stages (mbarrier full/empty), so the
//     consumers' fma chains never wait on HBM latency; the projected update is fused into
//     the same pass (alpha, v and g of the next epoch written once).
//   * The grid is one wave: bc = 32 * ceil(n / (32 * SMs)) columns per CTA (<= 256).
//   * k_gd_finalize: bias and objective of the final alpha, one thread, ascending i (the
//     oracle's order).
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "svm_internal.h"

namespace svmint {

namespace {
constexpr int GD_MAXBC = 256;   // columns (consumer threads) per CTA
constexpr int GD_MAXSTAGES = 8;

__device__ __forceinline__ uint32_t gd_smem(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void gd_mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(gd_smem(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void gd_mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(gd_smem(bar)) : "memory");
}
__device__ __forceinline__ void gd_mbar_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(gd_smem(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void gd_mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(gd_smem(bar)), "r"(parity) : "memory");
    }
}
__device__ __forceinline__ void gd_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(gd_smem(dst)), "l"(src), "r"(bytes), "r"(gd_smem(bar)) : "memory");
}
}  // namespace

// One epoch.  CTA c owns columns [c bc, c bc + bc); threads 0..bc-1 consume, the last warp
// produces.  Shared memory: stages x {K slab [J][bc] fp64, v [J] fp64}, then the barriers.
__global__ void __launch_bounds__(GD_MAXBC + 32) k_gd_epoch(
    const double* __restrict__ K, long long n, int bc, int J, int stages,
    const double* __restrict__ v_in, const double* __restrict__ a_in, const int8_t* __restrict__ y,
    double C, double lr, double* __restrict__ a_out, double* __restrict__ v_out,
    double* __restrict__ g_out) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int stage_doubles = J * bc + J;
    double* ring = reinterpret_cast<double*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * stage_doubles * 8);
    uint64_t* empty = full + GD_MAXSTAGES;
    const long long i0 = (long long)blockIdx.x * bc;
    const int nwc = bc / 32;
    const int t = threadIdx.x;
    if (t == 0) {
        for (int s = 0; s < stages; ++s) { gd_mbar_init(&full[s], 1); gd_mbar_init(&empty[s], nwc); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long nchunks = (n + J - 1) / J;
    if (t >= bc) {
        // ---- producer: lane 0 streams the column block, J rows of K per stage
        if (t == bc) {
            const double* Kb = K + (long long)blockIdx.x * n * bc;     // this CTA's column block
            for (long long c = 0; c < nchunks; ++c) {
                const int s = (int)(c % stages);
                if (c >= stages) gd_mbar_wait(&empty[s], (uint32_t)(((c / stages) - 1) & 1));
                const long long j0 = c * J;
                const int rows = (int)((n - j0) < J ? (n - j0) : J);
                const uint32_t vbytes = (uint32_t)(((rows + 1) & ~1) * 8);
                double* st = ring + (size_t)s * stage_doubles;
                const uint32_t kbytes = (uint32_t)rows * bc * 8;
                gd_mbar_expect(&full[s], kbytes + vbytes);
                gd_bulk(st + (size_t)J * bc, v_in + j0, vbytes, &full[s]);
                gd_bulk(st, Kb + j0 * bc, kbytes, &full[s]);
            }
        }
        return;
    }
    // ---- consumers: g_i = sum_j K[j][i] v_j, ascending j, one fma per term (R24)
    double acc = 0.0;
    for (long long c = 0; c < nchunks; ++c) {
        const int s = (int)(c % stages);
        gd_mbar_wait(&full[s], (uint32_t)((c / stages) & 1));
        const double* st = ring + (size_t)s * stage_doubles;
        const double* vs = st + (size_t)J * bc;
        const long long j0 = c * J;
        const int rows = (int)((n - j0) < J ? (n - j0) : J);
        if (rows == J) {
#pragma unroll 8
            for (int r = 0; r < J; ++r) acc = fma(st[r * bc + t], vs[r], acc);
        } else {
            for (int r = 0; r < rows; ++r) acc = fma(st[r * bc + t], vs[r], acc);
        }
        __syncwarp();
        if ((t & 31) == 0) gd_mbar_arrive(&empty[s]);
    }
    const long long i = i0 + t;
    if (i < n) {
        // projected ascent step (R23): grad = dW/dalpha_i = 1 - y_i g_i (y_i g_i is exact)
        const bool pos = y[i] > 0;
        const double grad = 1.0 - (pos ? acc : -acc);
        double a = fma(lr, grad, a_in[i]);
        a = a < 0.0 ? 0.0 : a;
        a = a > C ? C : a;
        a_out[i] = a;
        v_out[i] = pos ? a : -a;
        g_out[i] = acc;
    }
}

// Bias (R25) and W of the final alpha, in the oracle's order (one thread, ascending i).
__global__ void k_gd_finalize(const double* __restrict__ a, const double* __restrict__ v,
                              const double* __restrict__ g, const int8_t* __restrict__ y, long long n,
                              double C, double* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double eps = 1e-8;
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    double sum = 0.0, lin = 0.0, quad = 0.0;
    double mx_sv = -INF, mn_sv = INF, mx_all = -INF, mn_all = INF;
    long long cnt = 0, nsv = 0;
    for (long long i = 0; i < n; ++i) {
        const double ai = a[i], gi = g[i];
        if (ai > eps && ai < C - eps) { sum += (double)y[i] - gi; ++cnt; }
        if (ai > eps) { ++nsv; if (gi > mx_sv) mx_sv = gi; if (gi < mn_sv) mn_sv = gi; }
        if (gi > mx_all) mx_all = gi;
        if (gi < mn_all) mn_all = gi;
        lin += ai;
        quad += v[i] * gi;
    }
    double b;
    if (cnt > 0) b = sum / (double)cnt;
    else if (nsv > 0) b = -(mx_sv + mn_sv) / 2.0;
    else b = -(mx_all + mn_all) / 2.0;
    out[0] = b;
    out[1] = lin - 0.5 * quad;
}

}  // namespace svmint

using namespace svmint;

extern "C" int svm_train_gd_dev(const float* X, const int8_t* y, int64_t n, int64_t d, double C,
                                int kernel, double gamma, double lr, int64_t epochs, double* alpha,
                                double* b, svm_gd_info* info, void* cuda_stream) {
    if (!X || !y || !alpha || !b) return fail(SVM_EINVAL, "null pointer");
    if (n < 2) return fail(SVM_EINVAL, "n < 2");
    if (d < 1) return fail(SVM_EINVAL, "d < 1");
    if (n > 0x7fffffffll) return fail(SVM_EINVAL, "n >= 2^31");
    if (!(C > 0.0) || !std::isfinite(C)) return fail(SVM_EINVAL, "C must be finite and > 0");
    if (kernel != SVM_LINEAR && kernel != SVM_RBF) return fail(SVM_EINVAL, "unknown kernel");
    if (kernel == SVM_RBF && (!(gamma > 0.0) || !std::isfinite(gamma)))
        return fail(SVM_EINVAL, "RBF gamma must be finite and > 0");
    if (!(lr > 0.0) || !std::isfinite(lr)) return fail(SVM_EINVAL, "lr must be finite and > 0");
    if (epochs < 0) return fail(SVM_EINVAL, "epochs < 0");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    int rc = validate_device(X, y, n, d, st, nullptr);
    if (rc) return rc;
    int n_sm = 0, max_smem = 0;
    if ((rc = device_limits(&n_sm, &max_smem))) return rc;

    // ---- launch shape: one wave of CTAs, bc columns each, J rows of K per stage
    long long per = (n + n_sm - 1) / n_sm;
    int bc = (int)(((per + 31) / 32) * 32);
    if (bc > GD_MAXBC) bc = GD_MAXBC;
    if (bc < 32) bc = 32;
    const int ctas = (int)((n + bc - 1) / bc);
    // ---- K in HBM, column-blocked: ctas blocks of [n][bc] (pad columns zero)
    const long long ld = (long long)ctas * bc;
    const size_t kbytes = (size_t)n * (size_t)ld * 8;
    double* K = nullptr;
    if (cudaMallocAsync(&K, kbytes, st) != cudaSuccess) {
        cudaGetLastError();
        return fail(SVM_ENOMEM, "the Gram matrix (" + std::to_string(kbytes) + " bytes) does not fit in HBM");
    }
    double *a0 = nullptr, *a1 = nullptr, *v0 = nullptr, *v1 = nullptr, *g = nullptr, *out = nullptr;
    auto release = [&]() {
        for (double* q : {K, a0, a1, v0, v1, g, out}) if (q) cudaFreeAsync(q, st);
    };
    const size_t vb = (size_t)(ld + 2) * 8;               // ld >= n: room for the even-rounded v copy
    if (cudaMallocAsync(&a0, vb, st) != cudaSuccess || cudaMallocAsync(&a1, vb, st) != cudaSuccess ||
        cudaMallocAsync(&v0, vb, st) != cudaSuccess || cudaMallocAsync(&v1, vb, st) != cudaSuccess ||
        cudaMallocAsync(&g, vb, st) != cudaSuccess || cudaMallocAsync(&out, 16, st) != cudaSuccess) {
        cudaGetLastError();
        release();
        return fail(SVM_ENOMEM, "GD state allocation failed");
    }
    for (double* q : {a0, a1, v0, v1, g}) CKR(cudaMemsetAsync(q, 0, vb, st));
    if (ld != n) CKR(cudaMemsetAsync(K, 0, kbytes, st));     // pad columns are streamed too
    cudaEvent_t e0, e1, e2;
    CKR(cudaEventCreate(&e0)); CKR(cudaEventCreate(&e1)); CKR(cudaEventCreate(&e2));
    CKR(cudaEventRecord(e0, st));
    if ((rc = gram_device(X, n, d, kernel, gamma, K, st, 0, bc))) { release(); return rc; }
    CKR(cudaEventRecord(e1, st));
    int J = 32, stages = 4;
    auto smem_of = [&](int j, int s) { return (size_t)s * ((size_t)j * bc + j) * 8 + 2 * GD_MAXSTAGES * 8; };
    while (smem_of(J, stages) > (size_t)max_smem && stages > 2) --stages;
    while (smem_of(J, stages) > (size_t)max_smem && J > 4) J /= 2;
    const size_t smem = smem_of(J, stages);
    CKR(cudaFuncSetAttribute((const void*)k_gd_epoch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    double *ain = a0, *aout = a1, *vin = v0, *vout = v1;
    for (int64_t e = 0; e <= epochs; ++e) {
        // the last pass (e == epochs) only evaluates g for the final alpha (lr = 0 keeps
        // alpha: fma(0, grad, a) == a)
        const double lre = e < epochs ? lr : 0.0;
        k_gd_epoch<<<ctas, bc + 32, smem, st>>>(K, n, bc, J, stages, vin, ain, y, C, lre, aout, vout, g);
        counted();
        CKR(cudaGetLastError());
        std::swap(ain, aout);
        std::swap(vin, vout);
    }
    k_gd_finalize<<<1, 32, 0, st>>>(ain, vin, g, y, n, C, out);
    counted();
    CKR(cudaGetLastError());
    CKR(cudaEventRecord(e2, st));
    CKR(cudaMemcpyAsync(alpha, ain, (size_t)n * 8, cudaMemcpyDeviceToDevice, st));
    double ho[2];
    CKR(cudaMemcpyAsync(ho, out, 16, cudaMemcpyDeviceToHost, st));
    CKR(cudaStreamSynchronize(st));
    float ms_gram = 0.f, ms_ep = 0.f;
    cudaEventElapsedTime(&ms_gram, e0, e1);
    cudaEventElapsedTime(&ms_ep, e1, e2);
    cudaEventDestroy(e0); cudaEventDestroy(e1); cudaEventDestroy(e2);
    release();
    CKR(cudaStreamSynchronize(st));
    *b = ho[0];
    if (info) {
        memset(info, 0, sizeof(*info));
        info->objective = ho[1];
        info->seconds_gram = ms_gram * 1e-3;
        info->seconds_epochs = ms_ep * 1e-3;
        info->epochs = epochs;
        info->gram_bytes = (int64_t)kbytes;
    }
    char buf[256];
    snprintf(buf, sizeof buf, "{\"kernel\": \"k_gd_epoch\", \"ctas\": %d, \"threads\": %d, \"rows_per_stage\": %d, "
             "\"stages\": %d, \"smem\": %zu, \"mode\": \"gd-gram\"}", ctas, bc + 32, J, stages, smem);
    g_plan = buf;
    return SVM_OK;
}
