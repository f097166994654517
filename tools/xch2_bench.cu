// xch2_bench.cu -- finer microbenchmarks of the grid-wide candidate exchange (profiling aid).
// One persistent CTA per SM, 288 threads; every iteration each CTA publishes a record and
// learns the lexicographic (min f, min index) winner over all CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xb2 tools/xch2_bench.cu && ./xb2
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NTH = 288;

__device__ __forceinline__ double my_f(int cta, int it) { return (double)((cta * 7919 + it * 104729) % 1000003); }

template <int KIND>   // 0 volatile, 1 relaxed.gpu, 2 acquire.gpu, 3 cg
__device__ __forceinline__ uint4 ld16(const uint4* p) {
    uint4 v;
    if (KIND == 0)
        asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    else if (KIND == 1)
        asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    else if (KIND == 2)
        asm volatile("ld.acquire.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    else
        asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st16(uint4* p, uint4 v) {
    asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ unsigned ld32(const unsigned* p) {
    unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void st32(unsigned* p, unsigned v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// ---- P0: ping-pong between CTA 0 and CTA 1 (one-way hop latency = half the round trip)
__global__ void pingpong(unsigned* flags, int iters, long long* cyc) {
    if (threadIdx.x != 0 || blockIdx.x > 1) return;
    const long long t0 = clock64();
    for (int it = 1; it <= iters; ++it) {
        if (blockIdx.x == 0) {
            st32(flags, it);
            while (ld32(flags + 64) != (unsigned)it) {}
        } else {
            while (ld32(flags) != (unsigned)it) {}
            st32(flags + 64, it);
        }
    }
    if (blockIdx.x == 0) *cyc = clock64() - t0;
}

// ---- A: all-to-all LL records of REC 16-byte words {seq, idx, f}; POLL=0: threads t < G
// poll record t; POLL=1: the last warp polls all records (ceil(G/32) per lane, all loads in
// flight), then broadcasts through shared memory.  NREP replicas (readers use cta % NREP).
template <int KIND, int POLL>
__global__ void a2a(uint4* recs, int iters, int nrep, int rec, int backoff, double* out) {
    __shared__ double wf[10]; __shared__ int wi[10];
    const int t = threadIdx.x, G = gridDim.x, lane = t & 31, warp = t >> 5;
    double acc = 0;
    for (int it = 0; it < iters; ++it) {
        const int par = it & 1;
        const unsigned fg = it + 1;
        if (warp == 8) {
            const double f = my_f(blockIdx.x, it);
            const unsigned long long b = __double_as_longlong(f);
            for (int q = lane; q < nrep * rec; q += 32) {
                const int rp = q / rec, w = q % rec;
                st16(recs + ((size_t)(rp * 2 + par) * G + blockIdx.x) * rec + w,
                     make_uint4(fg, blockIdx.x, (unsigned)b, (unsigned)(b >> 32)));
            }
        }
        double bf = 1e300; int bi = 1 << 30;
        const uint4* base = recs + (size_t)((blockIdx.x % nrep) * 2 + par) * G * rec;
        if (POLL == 0) {
            if (t < G) {
                uint4 v;
                for (;;) {
                    bool ok = true;
                    v = ld16<KIND>(base + (size_t)t * rec);
                    ok = v.x == fg;
                    for (int w = 1; w < rec; ++w) ok = ok && ld16<KIND>(base + (size_t)t * rec + w).x == fg;
                    if (ok) break;
                    if (backoff) __nanosleep(backoff);
                }
                bf = __longlong_as_double(((unsigned long long)v.w << 32) | v.z); bi = v.y;
            }
            for (int o = 16; o; o >>= 1) {
                const double f2 = __shfl_xor_sync(~0u, bf, o); const int i2 = __shfl_xor_sync(~0u, bi, o);
                if (f2 < bf || (f2 == bf && i2 < bi)) { bf = f2; bi = i2; }
            }
            if (lane == 0) { wf[warp] = bf; wi[warp] = bi; }
            __syncthreads();
            bf = wf[0]; bi = wi[0];
            for (int w = 1; w < NTH / 32; ++w)
                if (wf[w] < bf || (wf[w] == bf && wi[w] < bi)) { bf = wf[w]; bi = wi[w]; }
        } else {
            if (warp == 8) {
                uint4 v[5];
                unsigned pend = 0;
                for (int q = 0; q < 5; ++q) if (lane + 32 * q < G) pend |= 1u << q;
                while (pend) {
#pragma unroll
                    for (int q = 0; q < 5; ++q) if (pend & (1u << q)) v[q] = ld16<KIND>(base + (size_t)(lane + 32 * q) * rec);
#pragma unroll
                    for (int q = 0; q < 5; ++q) if ((pend & (1u << q)) && v[q].x == fg) pend &= ~(1u << q);
                    if (pend && backoff) __nanosleep(backoff);
                }
#pragma unroll
                for (int q = 0; q < 5; ++q) if (lane + 32 * q < G) {
                    const double f = __longlong_as_double(((unsigned long long)v[q].w << 32) | v[q].z);
                    const int i = v[q].y;
                    if (f < bf || (f == bf && i < bi)) { bf = f; bi = i; }
                }
                for (int o = 16; o; o >>= 1) {
                    const double f2 = __shfl_xor_sync(~0u, bf, o); const int i2 = __shfl_xor_sync(~0u, bi, o);
                    if (f2 < bf || (f2 == bf && i2 < bi)) { bf = f2; bi = i2; }
                }
                if (lane == 0) { wf[0] = bf; wi[0] = bi; }
            }
            __syncthreads();
            bf = wf[0]; bi = wi[0];
        }
        acc += bf + bi;
        __syncthreads();
    }
    if (t == 0) out[blockIdx.x] = acc;
}

// ---- C: counter barrier (NC counters, CTA c bumps counter c % NC) + one warp reads the
// plain records.  REL: red.release (orders the record store) vs fence + red.relaxed.
__global__ void ctr(uint4* recs, unsigned long long* cnt, int iters, int nc, int rel, double* out) {
    __shared__ double sf; __shared__ int si;
    const int t = threadIdx.x, G = gridDim.x, lane = t & 31, warp = t >> 5;
    double acc = 0;
    for (int it = 0; it < iters; ++it) {
        const int par = it & 1;
        if (warp == 8) {
            if (lane == 0) {
                const unsigned long long b = __double_as_longlong(my_f(blockIdx.x, it));
                st16(recs + (size_t)par * G + blockIdx.x, make_uint4(0, blockIdx.x, (unsigned)b, (unsigned)(b >> 32)));
                unsigned long long* c = cnt + 32 * (blockIdx.x % nc);
                if (rel) asm volatile("red.release.gpu.global.add.u64 [%0], 1;" :: "l"(c) : "memory");
                else { __threadfence(); asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" :: "l"(c) : "memory"); }
            }
            if (lane < nc) {
                const unsigned long long tgt = (unsigned long long)(it + 1) * (G / nc + (lane < G % nc ? 1 : 0));
                unsigned long long v;
                do { asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(cnt + 32 * lane) : "memory"); } while (v < tgt);
            }
            __syncwarp();
            double bf = 1e300; int bi = 1 << 30;
            uint4 v[5];
#pragma unroll
            for (int q = 0; q < 5; ++q) if (lane + 32 * q < G) v[q] = ld16<3>(recs + (size_t)par * G + lane + 32 * q);
#pragma unroll
            for (int q = 0; q < 5; ++q) if (lane + 32 * q < G) {
                const double f = __longlong_as_double(((unsigned long long)v[q].w << 32) | v[q].z);
                const int i = v[q].y;
                if (f < bf || (f == bf && i < bi)) { bf = f; bi = i; }
            }
            for (int o = 16; o; o >>= 1) {
                const double f2 = __shfl_xor_sync(~0u, bf, o); const int i2 = __shfl_xor_sync(~0u, bi, o);
                if (f2 < bf || (f2 == bf && i2 < bi)) { bf = f2; bi = i2; }
            }
            if (lane == 0) { sf = bf; si = bi; }
        }
        __syncthreads();
        acc += sf + si;
        __syncthreads();
    }
    if (t == 0) out[blockIdx.x] = acc;
}

// ---- H: two-level LL tree.  Level 1: CTA c writes its record into group g = c / GS's
// slot; the group leader (CTA g*GS) polls its GS records (one lane each) and writes the
// group winner into the level-2 array; level 2: every CTA's last warp polls the NG group
// records (<= 32, one lane each).
__global__ void tree(uint4* l1, uint4* l2, int iters, int gs, int nrep, double* out) {
    __shared__ double sf; __shared__ int si;
    const int t = threadIdx.x, G = gridDim.x, lane = t & 31, warp = t >> 5;
    const int ng = (G + gs - 1) / gs, grp = blockIdx.x / gs;
    double acc = 0;
    for (int it = 0; it < iters; ++it) {
        const int par = it & 1;
        const unsigned fg = it + 1;
        if (warp == 8) {
            if (lane == 0) {
                const unsigned long long b = __double_as_longlong(my_f(blockIdx.x, it));
                st16(l1 + (size_t)par * G + blockIdx.x, make_uint4(fg, blockIdx.x, (unsigned)b, (unsigned)(b >> 32)));
            }
            double bf = 1e300; int bi = 1 << 30;
            if (blockIdx.x == grp * gs) {
                const int n = min(gs, G - grp * gs);
                if (lane < n) {
                    uint4 v;
                    do { v = ld16<1>(l1 + (size_t)par * G + grp * gs + lane); } while (v.x != fg);
                    bf = __longlong_as_double(((unsigned long long)v.w << 32) | v.z); bi = v.y;
                }
                for (int o = 16; o; o >>= 1) {
                    const double f2 = __shfl_xor_sync(~0u, bf, o); const int i2 = __shfl_xor_sync(~0u, bi, o);
                    if (f2 < bf || (f2 == bf && i2 < bi)) { bf = f2; bi = i2; }
                }
                const unsigned long long b = __double_as_longlong(bf);
                if (lane < nrep) st16(l2 + ((size_t)(lane * 2 + par) * ng + grp), make_uint4(fg, bi, (unsigned)b, (unsigned)(b >> 32)));
                bf = 1e300; bi = 1 << 30;
            }
            if (lane < ng) {
                uint4 v;
                do { v = ld16<1>(l2 + ((size_t)((blockIdx.x % nrep) * 2 + par) * ng + lane)); } while (v.x != fg);
                bf = __longlong_as_double(((unsigned long long)v.w << 32) | v.z); bi = v.y;
            }
            for (int o = 16; o; o >>= 1) {
                const double f2 = __shfl_xor_sync(~0u, bf, o); const int i2 = __shfl_xor_sync(~0u, bi, o);
                if (f2 < bf || (f2 == bf && i2 < bi)) { bf = f2; bi = i2; }
            }
            if (lane == 0) { sf = bf; si = bi; }
        }
        __syncthreads();
        acc += sf + si;
        __syncthreads();
    }
    if (t == 0) out[blockIdx.x] = acc;
}

int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    uint4* recs; uint4* l2; unsigned long long* cnt; double* out; unsigned* flags; long long* cyc;
    const size_t rb = (size_t)2 * 16 * nsm * 6 * 16;
    cudaMalloc(&recs, rb); cudaMalloc(&l2, 1 << 16); cudaMalloc(&cnt, 32 * 8 * 64); cudaMalloc(&out, nsm * 8);
    cudaMalloc(&flags, 4096); cudaMalloc(&cyc, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000;
    auto zero = [&] { cudaMemset(recs, 0, rb); cudaMemset(l2, 0, 1 << 16); cudaMemset(cnt, 0, 32 * 8 * 64); cudaMemset(flags, 0, 4096); cudaDeviceSynchronize(); };
    auto time = [&](const char* name, auto fn) {
        zero();
        cudaEventRecord(e0); fn(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%-58s %7.3f us/iter  (%s)\n", name, 1e3 * ms / iters, cudaGetErrorString(cudaGetLastError()));
    };
    {
        zero();
        pingpong<<<2, 32>>>(flags, iters, cyc);
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("P0 ping-pong one-way hop: %.0f cycles\n", (double)c / iters / 2);
        time("P0 ping-pong round trip", [&] { pingpong<<<2, 32>>>(flags, iters, cyc); });
    }
    char nm[128];
    for (int rec : {1, 2, 6})
        for (int nrep : {1, 4}) {
            snprintf(nm, sizeof nm, "A all-thread poll volatile rec=%dx16B nrep=%d", rec, nrep);
            time(nm, [&] { a2a<0, 0><<<nsm, NTH>>>(recs, iters, nrep, rec, 0, out); });
            snprintf(nm, sizeof nm, "A all-thread poll relaxed  rec=%dx16B nrep=%d", rec, nrep);
            time(nm, [&] { a2a<1, 0><<<nsm, NTH>>>(recs, iters, nrep, rec, 0, out); });
            snprintf(nm, sizeof nm, "A warp poll relaxed        rec=%dx16B nrep=%d", rec, nrep);
            time(nm, [&] { a2a<1, 1><<<nsm, NTH>>>(recs, iters, nrep, rec, 0, out); });
        }
    for (int bo : {20, 50, 100, 200}) {
        snprintf(nm, sizeof nm, "A all-thread poll relaxed rec=1 nrep=4 backoff=%dns", bo);
        time(nm, [&] { a2a<1, 0><<<nsm, NTH>>>(recs, iters, 4, 1, bo, out); });
        snprintf(nm, sizeof nm, "A warp poll relaxed rec=1 nrep=4 backoff=%dns", bo);
        time(nm, [&] { a2a<1, 1><<<nsm, NTH>>>(recs, iters, 4, 1, bo, out); });
    }
    time("A warp poll acquire rec=1 nrep=4", [&] { a2a<2, 1><<<nsm, NTH>>>(recs, iters, 4, 1, 0, out); });
    time("A warp poll cg rec=1 nrep=4", [&] { a2a<3, 1><<<nsm, NTH>>>(recs, iters, 4, 1, 0, out); });
    for (int nc : {1, 4, 8, 16})
        for (int rel : {1, 0}) {
            snprintf(nm, sizeof nm, "C counters=%d %s", nc, rel ? "red.release" : "fence+red.relaxed");
            time(nm, [&] { ctr<<<nsm, NTH>>>(recs, cnt, iters, nc, rel, out); });
        }
    for (int gs : {8, 12, 16, 24, 32})
        for (int nrep : {1, 4}) {
            snprintf(nm, sizeof nm, "H tree group=%d nrep=%d", gs, nrep);
            time(nm, [&] { tree<<<nsm, NTH>>>(recs, l2, iters, gs, nrep, out); });
        }
    return 0;
}
