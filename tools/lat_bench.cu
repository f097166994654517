// lat_bench.cu -- dependent-chain latency of the warp primitives the SMO scalar path uses
// (profiling aid): one warp, 1024-long chains, cycles per operation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lb tools/lat_bench.cu && ./lb
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(unsigned* out, long long* cyc, double* dout) {
    unsigned v = threadIdx.x * 2654435761u;
    double d = threadIdx.x * 0.5;
    long long t0, t1;
    // 0: REDUX min
    t0 = clock64();
    for (int i = 0; i < 1024; ++i) v = __reduce_min_sync(0xffffffffu, v) + threadIdx.x;
    t1 = clock64(); cyc[0] = t1 - t0;
    // 1: SHFL xor
    t0 = clock64();
    for (int i = 0; i < 1024; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1u;
    t1 = clock64(); cyc[1] = t1 - t0;
    // 2: DSETP-based select
    t0 = clock64();
    for (int i = 0; i < 1024; ++i) { const double e = d * 0.999; d = (e < d) ? e + 1.0 : d - 1.0; }
    t1 = clock64(); cyc[2] = t1 - t0;
    // 3: IMAD chain
    t0 = clock64();
    for (int i = 0; i < 1024; ++i) v = v * 2654435761u + 12345u;
    t1 = clock64(); cyc[3] = t1 - t0;
    // 4: LDS chain
    __shared__ unsigned sm[1024];
    for (int i = threadIdx.x; i < 1024; i += 32) sm[i] = (i * 7 + 1) & 1023;
    __syncwarp();
    unsigned p = threadIdx.x;
    t0 = clock64();
    for (int i = 0; i < 1024; ++i) p = sm[p];
    t1 = clock64(); cyc[4] = t1 - t0;
    // 5: DFMA chain
    t0 = clock64();
    for (int i = 0; i < 1024; ++i) d = fma(d, 0.999, 0.5);
    t1 = clock64(); cyc[5] = t1 - t0;
    // 6: ballot + ffs chain
    t0 = clock64();
    for (int i = 0; i < 1024; ++i) v = __ffs(__ballot_sync(0xffffffffu, (v & 1) == (threadIdx.x & 1))) + v;
    t1 = clock64(); cyc[6] = t1 - t0;
    // 7: double shfl (2 x 32-bit)
    t0 = clock64();
    for (int i = 0; i < 1024; ++i) d = __shfl_xor_sync(0xffffffffu, d, 1) * 1.0001;
    t1 = clock64(); cyc[7] = t1 - t0;
    out[threadIdx.x] = v + p; dout[threadIdx.x] = d;
}

int main() {
    unsigned* o; long long* c; double* dd;
    cudaMalloc(&o, 128); cudaMalloc(&c, 64); cudaMalloc(&dd, 256);
    k<<<1, 32>>>(o, c, dd); cudaDeviceSynchronize();
    k<<<1, 32>>>(o, c, dd);
    long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    const char* nm[8] = {"redux.min (+iadd)", "shfl.xor (+iadd)", "dsetp+dadd select", "imad", "lds (pointer chase)", "dfma", "ballot+ffs+iadd", "shfl f64 + dmul"};
    for (int i = 0; i < 8; ++i) printf("%-22s %6.1f cycles/op\n", nm[i], h[i] / 1024.0);
    return 0;
}
