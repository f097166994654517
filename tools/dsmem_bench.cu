// dsmem_bench.cu -- cost of pushing a record into every CTA of a 16-CTA cluster through
// distributed shared memory (profiling aid): cycles per round for st.shared::cluster.v4
// stores (one lane per (word, target)), measured by CTA 0, with a cluster barrier per round.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o db tools/dsmem_bench.cu && ./db
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __cluster_dims__(16, 1, 1) k(int rounds, int words, long long* cyc) {
    __shared__ __align__(16) uint4 mb[16 * 16];
    const int t = threadIdx.x, lane = t & 31;
    const unsigned cta = blockIdx.x % 16;
    for (int i = t; i < 256; i += blockDim.x) mb[i] = make_uint4(0, 0, 0, 0);
    csync();
    long long acc = 0, acc2 = 0;
    for (int r = 0; r < rounds; ++r) {
        csync();
        long long t0 = clock64();
        if (t < 32) {
            const uint4 w = make_uint4(r, cta, lane, 7);
            if (MODE == 0) {             // lane h < words stores word h to all 16 CTAs
                if (lane < words) {
                    const uint32_t src = s32(&mb[cta * 16 + lane]);
                    for (int j = 0; j < 16; ++j) {
                        uint32_t ra;
                        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(src), "r"(j));
                        asm volatile("st.shared::cluster.v4.u32 [%0], {%1,%2,%3,%4};" :: "r"(ra), "r"(w.x), "r"(w.y), "r"(w.z), "r"(w.w) : "memory");
                    }
                }
            } else if (MODE == 1) {      // all 32 lanes: (word, target) pairs spread
                for (int q = lane; q < words * 16; q += 32) {
                    const int j = q / words, h = q % words;
                    uint32_t ra;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(s32(&mb[cta * 16 + h])), "r"(j));
                    asm volatile("st.shared::cluster.v4.u32 [%0], {%1,%2,%3,%4};" :: "r"(ra), "r"(w.x), "r"(w.y), "r"(w.z), "r"(w.w) : "memory");
                }
            } else {                     // local stores only (baseline)
                if (lane < words) mb[cta * 16 + lane] = w;
            }
            __syncwarp();
        }
        long long t1 = clock64();
        // a dependent local load after the stores (does it wait for them?)
        if (t == 0) { volatile uint4* v = mb; (void)v[0].x; }
        long long t2 = clock64();
        acc += t1 - t0; acc2 += t2 - t1;
    }
    if (blockIdx.x == 0 && t == 0) { cyc[0] = acc; cyc[1] = acc2; }
}

int main() {
    long long* c; cudaMalloc(&c, 16);
    const int rounds = 2000;
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int mode = 0; mode < 3; ++mode)
        for (int words : {4, 8, 12}) {
            if (mode == 0) k<0><<<16, 256>>>(rounds, words, c);
            if (mode == 1) k<1><<<16, 256>>>(rounds, words, c);
            if (mode == 2) k<2><<<16, 256>>>(rounds, words, c);
            long long h[2]; cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
            printf("mode %d words %2d: issue %7.1f cycles, then local LDS %6.1f cycles (%s)\n", mode, words,
                   (double)h[0] / rounds, (double)h[1] / rounds, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
