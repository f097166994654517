// microbench.cu -- B200 pipe rates that decide the row-pass design: fp32->fp64
// widening (F2F.F64.F32 vs integer bit assembly), DADD/DFMA throughput, DFMA latency.
// Inputs come from shared memory each iteration so nothing can be hoisted.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o tools/mb tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double widen_int(float x) {
    const uint32_t u = __float_as_uint(x);
    const uint32_t a = u & 0x7fffffffu;
    uint32_t hi = (a >> 3) + 0x38000000u + (u & 0x80000000u);
    hi = a ? hi : (u & 0x80000000u);
    return __hiloint2double((int)hi, (int)(u << 29));
}

template <int MODE>
__global__ void k_row(const float* gin, double* out, int iters) {
    __shared__ float xs[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) xs[i] = gin[i];
    __syncthreads();
    double du0 = 0, dl0 = 0, du1 = 0, dl1 = 0;
    const double pu = 0.25, pl = 0.75;
    float facc = 0.f;
    for (int i = 0; i < iters; ++i) {
        const float* p = xs + ((i * 64) & 4095) + (threadIdx.x & 31);
#pragma unroll
        for (int k = 0; k < 16; k += 2) {
            const float a = p[k * 2], b = p[k * 2 + 1];
            if (MODE == 0) {          // the row pass: F2F + 2 DADD + 2 DFMA per element
                const double x = a, y = b;
                double e;
                e = x - pu; du0 = fma(e, e, du0); e = x - pl; dl0 = fma(e, e, dl0);
                e = y - pu; du1 = fma(e, e, du1); e = y - pl; dl1 = fma(e, e, dl1);
            } else if (MODE == 1) {   // same with integer widening
                const double x = widen_int(a), y = widen_int(b);
                double e;
                e = x - pu; du0 = fma(e, e, du0); e = x - pl; dl0 = fma(e, e, dl0);
                e = y - pu; du1 = fma(e, e, du1); e = y - pl; dl1 = fma(e, e, dl1);
            } else if (MODE == 2) {   // F2F only
                du0 += (double)a; du1 += (double)b;
            } else if (MODE == 3) {   // fp64 math only (no conversion)
                const double x = __int_as_float(__float_as_int(a)) * 0 + pu * (double)(k + 1), y = pl * (double)(k + 2);
                double e;
                e = x - pu; du0 = fma(e, e, du0); e = x - pl; dl0 = fma(e, e, dl0);
                e = y - pu; du1 = fma(e, e, du1); e = y - pl; dl1 = fma(e, e, dl1);
            } else {                  // mixed: one F2F, one integer widening
                const double x = a, y = widen_int(b);
                double e;
                e = x - pu; du0 = fma(e, e, du0); e = x - pl; dl0 = fma(e, e, dl0);
                e = y - pu; du1 = fma(e, e, du1); e = y - pl; dl1 = fma(e, e, dl1);
            }
            facc += a;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = du0 + dl0 + du1 + dl1 + facc;
}

__global__ void k_dfma_lat(double* out, int iters, long long* cyc) {
    double a = threadIdx.x * 1e-3;
    const double b = 1.0000001, c = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) a = fma(a, b, c);
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    float* in; double* out; long long* cyc;
    cudaMalloc(&in, 4096 * 4); cudaMalloc(&out, 148 * 4 * 1024 * 8); cudaMalloc(&cyc, 8);
    float h[4096];
    for (int i = 0; i < 4096; ++i) h[i] = (float)((i * 2654435761u) % 1000) / 999.0f;
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 2048;
    const char* names[5] = {"row: F2F+2DADD+2DFMA /elem", "row: intwiden+2DADD+2DFMA", "F2F (+DADD) only",
                            "2DADD+2DFMA, no conversion", "mixed F2F/intwiden"};
    for (int threads : {256, 512, 1024}) {
        const int blocks = nsm * (1024 / threads);
        const double elems = (double)blocks * threads * iters * 16;
        for (int m = 0; m < 5; ++m) {
            auto launch = [&] {
                if (m == 0) k_row<0><<<blocks, threads>>>(in, out, iters);
                if (m == 1) k_row<1><<<blocks, threads>>>(in, out, iters);
                if (m == 2) k_row<2><<<blocks, threads>>>(in, out, iters);
                if (m == 3) k_row<3><<<blocks, threads>>>(in, out, iters);
                if (m == 4) k_row<4><<<blocks, threads>>>(in, out, iters);
            };
            launch(); cudaDeviceSynchronize();
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("threads/blk %4d  %-30s %8.3f ms  %7.2f elem/clk/SM (@1965 MHz)\n", threads, names[m], ms,
                   elems / (ms * 1e-3) / nsm / 1.965e9);
        }
    }
    k_dfma_lat<<<1, 32>>>(out, 100000, cyc); cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cycles\n", c / 100000.0);
    return 0;
}
