// exp_bench.cu -- throughput of the solver's correctly rounded exp fast phase on one B200
// (exps / clk / SM), for several independent exps per thread (ILP) and threads per CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o tools/xb_exp tools/exp_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2311_14908_b200/csrc/svm_exp.cuh"

template <int ILP>
__global__ void k_exp(const double* gin, double* out, int iters, int* slow) {
    __shared__ double tabs[svmexp::EXP_TABLE_DOUBLES];
    __shared__ double xs[1024];
    for (int e = threadIdx.x; e < svmexp::EXP_TABLE_DOUBLES; e += blockDim.x) tabs[e] = svmexp::table_entry(e);
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) xs[i] = gin[i];
    __syncthreads();
    const svmexp::PtrTab tab{tabs};
    double acc = 0.0;
    int ns = 0;
    for (int it = 0; it < iters; ++it) {
        double v[ILP];
        bool s[ILP];
#pragma unroll
        for (int q = 0; q < ILP; ++q) v[q] = svmexp::exp_cr_fast(xs[(threadIdx.x + 37 * q + it) & 1023], tab, s[q]);
#pragma unroll
        for (int q = 0; q < ILP; ++q) { acc += v[q]; ns += !s[q]; }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (ns) atomicAdd(slow, ns);
}

template <int ILP>
void run(int threads, const double* din, double* dout, int* dslow, int nsm) {
    const int iters = 2000;
    k_exp<ILP><<<nsm, threads>>>(din, dout, 10, dslow);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k_exp<ILP><<<nsm, threads>>>(din, dout, iters, dslow);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double exps = (double)nsm * threads * iters * ILP;
    printf("threads %4d ILP %d: %.3f ms  %.3f exps/clk/SM (@%d MHz)\n", threads, ILP, ms,
           exps / nsm / (ms * 1e-3 * clk * 1e3), clk / 1000);
}

int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double h[1024];
    for (int i = 0; i < 1024; ++i) h[i] = -0.001 - 9.0 * (i * 0.6180339887 - (int)(i * 0.6180339887));
    double *din, *dout; int* dslow;
    cudaMalloc(&din, sizeof h); cudaMalloc(&dout, 1 << 20); cudaMalloc(&dslow, 4);
    cudaMemcpy(din, h, sizeof h, cudaMemcpyHostToDevice);
    for (int th : {256, 512}) { run<1>(th, din, dout, dslow, nsm); run<2>(th, din, dout, dslow, nsm); run<4>(th, din, dout, dslow, nsm); run<8>(th, din, dout, dslow, nsm); }
    return 0;
}
