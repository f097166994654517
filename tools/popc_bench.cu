// popc_bench.cu -- POPC (+LOP) vs IMAD (+LOP) throughput per SM (profiling aid).
#include <cstdio>
__global__ void k(const unsigned* in, unsigned* out, long long* cyc, int mode) {
    unsigned a[8]; for (int i = 0; i < 8; ++i) a[i] = in[threadIdx.x * 8 + i];
    unsigned acc[8] = {0,0,0,0,0,0,0,0};
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < 256; ++r) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (mode == 0) acc[i] += __popc(a[i] ^ acc[(i + 1) & 7]);
            else acc[i] += (a[i] ^ acc[(i + 1) & 7]) * 3u;
        }
    }
    __syncthreads();
    long long t1 = clock64();
    unsigned s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    unsigned *in, *out; long long* c; cudaMalloc(&in, 1 << 20); cudaMalloc(&out, 1 << 20); cudaMalloc(&c, 8 * 148);
    cudaMemset(in, 0x5a, 1 << 20);
    for (int mode = 0; mode < 2; ++mode) for (int th : {256, 512, 1024}) {
        k<<<1, th>>>(in, out, c, mode); cudaDeviceSynchronize();
        long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        double ops = 256.0 * 8 * th;   // popc (or imad) ops per SM
        printf("%s threads %4d: %.1f ops/clk/SM\n", mode ? "imad+lop" : "popc+lop", th, ops / h);
    }
}
