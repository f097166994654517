// xch3_bench.cu -- the SMO kernel's exchange step in isolation, with the kernel's warp
// roles and barriers (profiling aid).  8 "consumer" warps spin for WORK cycles (the row
// pass) and post per-warp candidates; the scalar warp reduces them, publishes the CTA
// record (4 x 16-byte words {seq|chk, payload[3]}), polls words 0/1 of every record (PB
// per lane), selects, fetches words 2/3 of the winners and releases the consumers.
// Layouts: 0 = transposed word[h][g] (16 B per CTA per array), 1 = record-contiguous
// rec[g][h] (64 B per CTA), 2 = pair-contiguous: (w0,w1) at [g][0..1], (w2,w3) at [g][2..3]
// of a second array.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xb3 tools/xch3_bench.cu && ./xb3
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NTH = 320;

__device__ __forceinline__ uint32_t chk(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t h = a * 0x9E3779B1u ^ (b + 0x7F4A7C15u) * 0x85EBCA77u ^ (c + 0x165667B1u) * 0xC2B2AE3Du;
    h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 13;
    return (h ^ (h >> 16)) & 0xffffu;
}
__device__ int g_kind;
template <int K>
__device__ __forceinline__ uint4 ld16k(const uint4* p) {
    uint4 v;
    if (K == 0) asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    if (K == 1) asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    if (K == 2) asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    if (K == 3) asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    if (K == 4) asm volatile("ld.relaxed.gpu.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    if (K == 5) asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
#define ld16 ld16k<KIND>
__device__ __forceinline__ void st16(uint4* p, uint4 v) {
    asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void bsync(int id) { asm volatile("bar.sync %0, 288;" :: "r"(id) : "memory"); }
__device__ __forceinline__ void barrive(int id) { asm volatile("bar.arrive %0, 288;" :: "r"(id) : "memory"); }

__device__ __forceinline__ uint4* wptr(uint4* base, int layout, int par, int h, int g, int G) {
    if (layout == 0) return base + ((size_t)par * 4 + h) * G + g;
    if (layout == 1) return base + ((size_t)par * G + g) * 4 + h;
    return base + ((size_t)(par * 2 + (h >> 1)) * G + g) * 2 + (h & 1);
}

template <int KIND, int PB>
__global__ void xch(uint4* mb, int iters, int layout, int work, unsigned long long* cyc, double* out) {
    __shared__ double rf[2][8]; __shared__ int ri[2][8];
    __shared__ int su, sl;
    const int t = threadIdx.x, G = gridDim.x, lane = t & 31, warp = t >> 5;
    if (warp == 9) return;
    double acc = 0;
    unsigned long long c_pub = 0, c_poll = 0, c_sel = 0, c_fetch = 0;
    for (int it = 0; it < iters; ++it) {
        const int par = it & 1;
        const uint32_t sq = (uint32_t)(it + 1) & 0xffffu;
        if (warp < 8) {
            const long long t0 = clock64();
            while (clock64() - t0 < work) {}
            if (lane == 0) {
                rf[0][warp] = (double)((blockIdx.x * 7919 + it * 104729 + warp * 31) % 1000003);
                ri[0][warp] = blockIdx.x * 8 + warp;
                rf[1][warp] = (double)((blockIdx.x * 104729 + it * 7919 + warp * 17) % 1000003);
                ri[1][warp] = blockIdx.x * 8 + warp;
            }
            bsync(1);
            bsync(2);
            acc += su + sl;
            continue;
        }
        // scalar warp
        bsync(1);
        long long c0 = clock64();
        double fu = lane < 8 ? rf[0][lane] : 1e300; int iu = lane < 8 ? ri[0][lane] : (1 << 30);
        double fl = lane < 8 ? rf[1][lane] : -1e300; int il = lane < 8 ? ri[1][lane] : (1 << 30);
        for (int o = 4; o; o >>= 1) {
            double f2 = __shfl_xor_sync(~0u, fu, o); int i2 = __shfl_xor_sync(~0u, iu, o);
            if (f2 < fu || (f2 == fu && i2 < iu)) { fu = f2; iu = i2; }
            f2 = __shfl_xor_sync(~0u, fl, o); i2 = __shfl_xor_sync(~0u, il, o);
            if (f2 > fl || (f2 == fl && i2 < il)) { fl = f2; il = i2; }
        }
        fu = __shfl_sync(~0u, fu, 0); iu = __shfl_sync(~0u, iu, 0);
        fl = __shfl_sync(~0u, fl, 0); il = __shfl_sync(~0u, il, 0);
        if (lane < 4) {
            const double f = lane == 0 ? fu : lane == 1 ? fl : 0.5 * lane;
            const uint32_t a = lane == 0 ? iu : lane == 1 ? il : 0x10001u;
            const unsigned long long b = __double_as_longlong(f);
            st16(wptr(mb, layout, par, lane, blockIdx.x, G), make_uint4((sq << 16) | chk(a, (uint32_t)b, (uint32_t)(b >> 32)), a, (uint32_t)b, (uint32_t)(b >> 32)));
        }
        long long c1 = clock64(); c_pub += c1 - c0; c0 = c1;
        double bu = 1e300, bl = -1e300; int bi = 1 << 30, bj = 1 << 30, gu = 0, gl = 0;
        {
            uint4 v[PB][2];
            unsigned pend = 0;
            for (int q = 0; q < PB; ++q) if (32 * q + lane < G) pend |= 1u << q;
            for (int g0 = 0; g0 < G; g0 += 32 * PB) {
            pend = 0;
            for (int q = 0; q < PB; ++q) if (g0 + 32 * q + lane < G) pend |= 1u << q;
            const unsigned mine = pend;
            while (pend) {
#pragma unroll
                for (int q = 0; q < PB; ++q) if (pend & (1u << q)) {
                    v[q][0] = ld16(wptr(mb, layout, par, 0, g0 + 32 * q + lane, G));
                    v[q][1] = ld16(wptr(mb, layout, par, 1, g0 + 32 * q + lane, G));
                }
#pragma unroll
                for (int q = 0; q < PB; ++q)
                    if ((pend & (1u << q)) && v[q][0].x == ((sq << 16) | chk(v[q][0].y, v[q][0].z, v[q][0].w)) &&
                        v[q][1].x == ((sq << 16) | chk(v[q][1].y, v[q][1].z, v[q][1].w)))
                        pend &= ~(1u << q);
            }
#pragma unroll
            for (int q = 0; q < PB; ++q) if (mine & (1u << q)) {
                const double f0 = __longlong_as_double(((unsigned long long)v[q][0].w << 32) | v[q][0].z);
                const double f1 = __longlong_as_double(((unsigned long long)v[q][1].w << 32) | v[q][1].z);
                if (f0 < bu || (f0 == bu && (int)v[q][0].y < bi)) { bu = f0; bi = v[q][0].y; gu = g0 + 32 * q + lane; }
                if (f1 > bl || (f1 == bl && (int)v[q][1].y < bj)) { bl = f1; bj = v[q][1].y; gl = g0 + 32 * q + lane; }
            }
            }
        }
        c1 = clock64(); c_poll += c1 - c0; c0 = c1;
        double wu = bu, wl = bl; int wi = bi, wj = bj;
        for (int o = 16; o; o >>= 1) {
            double f2 = __shfl_xor_sync(~0u, wu, o); int i2 = __shfl_xor_sync(~0u, wi, o);
            if (f2 < wu || (f2 == wu && i2 < wi)) { wu = f2; wi = i2; }
            f2 = __shfl_xor_sync(~0u, wl, o); i2 = __shfl_xor_sync(~0u, wj, o);
            if (f2 > wl || (f2 == wl && i2 < wj)) { wl = f2; wj = i2; }
        }
        const unsigned mu = __ballot_sync(~0u, bi == wi), ml = __ballot_sync(~0u, bj == wj);
        const int ru = __shfl_sync(~0u, gu, __ffs(mu) - 1), rl = __shfl_sync(~0u, gl, __ffs(ml) - 1);
        c1 = clock64(); c_sel += c1 - c0; c0 = c1;
        uint4 wa = make_uint4(0, 0, 0, 0);
        const uint4* wp = wptr(mb, layout, par, lane == 2 ? 3 : 2, lane == 0 ? ru : rl, G);
        if (lane < 3) {
            wa = ld16(wp);
            while (wa.x != ((sq << 16) | chk(wa.y, wa.z, wa.w))) wa = ld16(wp);
        }
        __syncwarp();
        const int yy = __shfl_sync(~0u, (int)wa.y, 0);
        if (lane == 0) { su = wi + yy; sl = wj; }
        c1 = clock64(); c_fetch += c1 - c0;
        barrive(2);
    }
    if (t == 256 && blockIdx.x == 0) { cyc[0] = c_pub; cyc[1] = c_poll; cyc[2] = c_sel; cyc[3] = c_fetch; }
    if (t == 0) out[blockIdx.x] = acc;
}

int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    uint4* mb; double* out; unsigned long long* cyc;
    const size_t bytes = (size_t)2 * 4 * nsm * 16 * 2;
    cudaMalloc(&mb, bytes); cudaMalloc(&out, nsm * 8); cudaMalloc(&cyc, 64);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000;
    for (int grid : {16, 74, 148})
        for (int pb : {1, 5}) {
            const int layout = 1, work = 0;
            cudaMemset(mb, 0, bytes); cudaDeviceSynchronize();
            cudaEventRecord(e0);
            if (pb == 1) xch<0, 1><<<grid, NTH>>>(mb, iters, layout, work, cyc, out);
            else xch<0, 5><<<grid, NTH>>>(mb, iters, layout, work, cyc, out);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            unsigned long long c[4]; cudaMemcpy(c, cyc, 32, cudaMemcpyDeviceToHost);
            printf("grid=%3d PB=%d: %6.3f us/iter  cycles/iter publish=%5llu poll=%5llu select=%4llu fetch=%5llu (%s)\n",
                   grid, pb, 1e3 * ms / iters, c[0] / iters, c[1] / iters, c[2] / iters, c[3] / iters,
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
