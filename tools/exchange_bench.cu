// exchange_bench.cu -- latency of one grid-wide "all CTAs publish a record, all CTAs
// learn the lexicographic winner" exchange on B200, for the strategies the SMO kernel
// can use.  One persistent CTA per SM, 10 warps; each iteration every CTA publishes a
// 48-byte (f, index) record and must obtain the global winner.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xb tools/exchange_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int NTH = 288;

struct __align__(16) Rec { double f; int i; int pad; double a; double b; double c; double d; };  // 48 B
struct __align__(16) LL { unsigned long long w[6]; };   // 3 doubles-ish payload with flags

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
    unsigned long long v; asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void red_rel(unsigned long long* p) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" :: "l"(p) : "memory");
}
__device__ __forceinline__ void stv2(unsigned long long* p, unsigned long long a, unsigned long long b) {
    asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" :: "l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ldv2(const unsigned long long* p, unsigned long long& a, unsigned long long& b) {
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ unsigned long long W(uint32_t f, uint32_t p) { return ((unsigned long long)f << 32) | p; }

__device__ double my_f(int cta, int it) { return (double)((cta * 7919 + it * 104729) % 1000003); }

// S1: counter + fence; one poller; records read by the scalar warp (5 per lane)
__global__ void s1(Rec* recs, unsigned long long* cnt, int iters, double* out) {
    __shared__ double sf; __shared__ int si;
    const int t = threadIdx.x, G = gridDim.x;
    double acc = 0;
    for (int it = 0; it < iters; ++it) {
        const int par = it & 1;
        if (t == 256) {
            Rec r; r.f = my_f(blockIdx.x, it); r.i = blockIdx.x;
            recs[par * G + blockIdx.x] = r;
            __threadfence();
            atomicAdd(cnt, 1ull);
            const unsigned long long tgt = (unsigned long long)(it + 1) * G;
            while (ld_acq(cnt) < tgt) {}
        }
        __syncthreads();
        if (t >= 256) {
            const int lane = t - 256;
            double bf = 1e300; int bi = 1 << 30;
            for (int g = lane; g < G; g += 32) {
                const double f = __ldcg(&recs[par * G + g].f); const int i = __ldcg(&recs[par * G + g].i);
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
    }
    if (t == 0) out[blockIdx.x] = acc;
}

// S2: LL all-to-all; scalar warp polls every record (unrolled in groups of 2 per lane)
__global__ void s2(LL* recs, int iters, double* out) {
    __shared__ double sf; __shared__ int si;
    const int t = threadIdx.x, G = gridDim.x;
    double acc = 0;
    for (int it = 0; it < iters; ++it) {
        const int par = it & 1;
        const uint32_t fg = it + 1;
        if (t >= 256) {
            const int lane = t - 256;
            if (lane == 0) {
                const unsigned long long b = __double_as_longlong(my_f(blockIdx.x, it));
                unsigned long long* w = recs[par * G + blockIdx.x].w;
                stv2(w, W(fg, (uint32_t)b), W(fg, (uint32_t)(b >> 32)));
                stv2(w + 2, W(fg, blockIdx.x), W(fg, 0));
                stv2(w + 4, W(fg, 0), W(fg, 0));
            }
            double bf = 1e300; int bi = 1 << 30;
            for (int g0 = lane; g0 < G; g0 += 64) {
                unsigned long long v[2][6]; unsigned pend = 0;
                for (int q = 0; q < 2; ++q) if (g0 + 32 * q < G) pend |= 1u << q;
                while (pend) {
                    for (int q = 0; q < 2; ++q) if (pend & (1u << q)) {
                        const unsigned long long* w = recs[par * G + g0 + 32 * q].w;
                        ldv2(w, v[q][0], v[q][1]); ldv2(w + 2, v[q][2], v[q][3]); ldv2(w + 4, v[q][4], v[q][5]);
                    }
                    for (int q = 0; q < 2; ++q) if (pend & (1u << q)) {
                        bool ok = true; for (int h = 0; h < 6; ++h) ok = ok && (uint32_t)(v[q][h] >> 32) == fg;
                        if (ok) pend &= ~(1u << q);
                    }
                }
                for (int q = 0; q < 2; ++q) if (g0 + 32 * q < G) {
                    const double f = __longlong_as_double((v[q][0] & 0xffffffffull) | (v[q][1] << 32));
                    const int i = (int)(uint32_t)v[q][2];
                    if (f < bf || (f == bf && i < bi)) { bf = f; bi = i; }
                }
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

// S3: LL, aggregator CTA 0 (one thread per record) + 8 broadcast replicas
__global__ void s3(LL* recs, LL* bc, int iters, double* out) {
    __shared__ double wf[9]; __shared__ int wi[9];
    __shared__ double sf; __shared__ int si;
    const int t = threadIdx.x, G = gridDim.x, lane = t & 31, warp = t >> 5;
    double acc = 0;
    for (int it = 0; it < iters; ++it) {
        const int par = it & 1;
        const uint32_t fg = it + 1;
        if (t == 256) {
            const unsigned long long b = __double_as_longlong(my_f(blockIdx.x, it));
            unsigned long long* w = recs[par * G + blockIdx.x].w;
            stv2(w, W(fg, (uint32_t)b), W(fg, (uint32_t)(b >> 32)));
            stv2(w + 2, W(fg, blockIdx.x), W(fg, 0));
            stv2(w + 4, W(fg, 0), W(fg, 0));
        }
        if (blockIdx.x == 0) {
            double bf = 1e300; int bi = 1 << 30;
            for (int g = t; g < G; g += NTH) {
                unsigned long long v[6];
                const unsigned long long* w = recs[par * G + g].w;
                for (;;) {
                    ldv2(w, v[0], v[1]); ldv2(w + 2, v[2], v[3]); ldv2(w + 4, v[4], v[5]);
                    bool ok = true; for (int h = 0; h < 6; ++h) ok = ok && (uint32_t)(v[h] >> 32) == fg;
                    if (ok) break;
                }
                const double f = __longlong_as_double((v[0] & 0xffffffffull) | (v[1] << 32));
                const int i = (int)(uint32_t)v[2];
                if (f < bf || (f == bf && i < bi)) { bf = f; bi = i; }
            }
            for (int o = 16; o; o >>= 1) {
                const double f2 = __shfl_xor_sync(~0u, bf, o); const int i2 = __shfl_xor_sync(~0u, bi, o);
                if (f2 < bf || (f2 == bf && i2 < bi)) { bf = f2; bi = i2; }
            }
            if (lane == 0) { wf[warp] = bf; wi[warp] = bi; }
            __syncthreads();
            if (warp == 0) {
                bf = lane < 9 ? wf[lane] : 1e300; bi = lane < 9 ? wi[lane] : (1 << 30);
                for (int o = 16; o; o >>= 1) {
                    const double f2 = __shfl_xor_sync(~0u, bf, o); const int i2 = __shfl_xor_sync(~0u, bi, o);
                    if (f2 < bf || (f2 == bf && i2 < bi)) { bf = f2; bi = i2; }
                }
                if (lane < 8) {
                    const unsigned long long b = __double_as_longlong(bf);
                    unsigned long long* w = bc[par * 8 + lane].w;
                    stv2(w, W(fg, (uint32_t)b), W(fg, (uint32_t)(b >> 32)));
                    stv2(w + 2, W(fg, bi), W(fg, 0));
                    stv2(w + 4, W(fg, 0), W(fg, 0));
                }
                if (lane == 0) { sf = bf; si = bi; }
            }
        } else if (t == 0) {
            unsigned long long v[6];
            const unsigned long long* w = bc[par * 8 + (blockIdx.x & 7)].w;
            for (;;) {
                ldv2(w, v[0], v[1]); ldv2(w + 2, v[2], v[3]); ldv2(w + 4, v[4], v[5]);
                bool ok = true; for (int h = 0; h < 6; ++h) ok = ok && (uint32_t)(v[h] >> 32) == fg;
                if (ok) break;
            }
            sf = __longlong_as_double((v[0] & 0xffffffffull) | (v[1] << 32)); si = (int)(uint32_t)v[2];
        }
        __syncthreads();
        acc += sf + si;
        __syncthreads();
    }
    if (t == 0) out[blockIdx.x] = acc;
}

// S4: counter with red.release (no separate fence), poller spins, then one lane/record reads
__global__ void s4(Rec* recs, unsigned long long* cnt, int iters, double* out) {
    __shared__ double sf; __shared__ int si;
    const int t = threadIdx.x, G = gridDim.x;
    double acc = 0;
    for (int it = 0; it < iters; ++it) {
        const int par = it & 1;
        if (t >= 256) {
            const int lane = t - 256;
            if (lane == 0) {
                Rec r; r.f = my_f(blockIdx.x, it); r.i = blockIdx.x;
                recs[par * G + blockIdx.x] = r;
                red_rel(cnt);
                const unsigned long long tgt = (unsigned long long)(it + 1) * G;
                while (ld_acq(cnt) < tgt) {}
            }
            __syncwarp();
            double bf = 1e300; int bi = 1 << 30;
            double fv[5]; int iv[5];
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                const int g = lane + 32 * q;
                fv[q] = g < G ? __ldcg(&recs[par * G + g].f) : 1e300;
                iv[q] = g < G ? __ldcg(&recs[par * G + g].i) : (1 << 30);
            }
#pragma unroll
            for (int q = 0; q < 5; ++q) if (fv[q] < bf || (fv[q] == bf && iv[q] < bi)) { bf = fv[q]; bi = iv[q]; }
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


// Shared helpers for S5/S6: every thread t < G polls record t (direct polling, as the SMO
// kernel does when X is resident), then warp shuffles + one barrier + a 9-way reduce.
__device__ __forceinline__ void ldv4(const void* p, unsigned& s, unsigned& i, unsigned long long& f) {
    unsigned a, b, c, d;
    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p) : "memory");
    s = a; i = b; f = ((unsigned long long)d << 32) | c;
}
__device__ __forceinline__ void stv4(void* p, unsigned s, unsigned i, unsigned long long f) {
    asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" :: "l"(p), "r"(s), "r"(i), "r"((unsigned)f), "r"((unsigned)(f >> 32)) : "memory");
}
template <int NREP>
__global__ void s5(uint4* recs, int iters, double* out, int rec16) {
    // rec16 = 16-byte words per record: 2 (compact: up + low) or 6 (96-byte LL-style size)
    __shared__ double wf[2][10]; __shared__ int wi[2][10];
    const int t = threadIdx.x, G = gridDim.x, lane = t & 31, warp = t >> 5;
    double acc = 0;
    for (int it = 0; it < iters; ++it) {
        const int par = it & 1;
        const unsigned fg = it + 1;
        if (warp == 8) {
            const double f = my_f(blockIdx.x, it);
            for (int q = lane; q < NREP * rec16; q += 32) {
                const int rep = q / rec16, w = q % rec16;
                uint4* r = recs + ((size_t)(rep * 2 + par) * G + blockIdx.x) * rec16 + w;
                stv4(r, fg, blockIdx.x, __double_as_longlong(f + w));
            }
        }
        __syncthreads();
        double bu = 1e300, bl = -1e300; int iu = 1 << 30, il = 1 << 30;
        if (t < G) {
            const uint4* r = recs + ((size_t)((blockIdx.x % NREP) * 2 + par) * G + t) * rec16;
            unsigned s0, i0; unsigned long long f0;
            unsigned s1, i1; unsigned long long f1;
            for (;;) {
                bool ok = true;
                ldv4(r, s0, i0, f0); ok = s0 == fg;
                ldv4(r + 1, s1, i1, f1); ok = ok && s1 == fg;
                for (int w = 2; w < rec16; ++w) { unsigned sx, ix; unsigned long long fx; ldv4(r + w, sx, ix, fx); ok = ok && sx == fg; }
                if (ok) break;
            }
            bu = __longlong_as_double(f0); iu = i0; bl = __longlong_as_double(f1); il = i1;
        }
        for (int o = 16; o; o >>= 1) {
            const double f2 = __shfl_xor_sync(~0u, bu, o); const int i2 = __shfl_xor_sync(~0u, iu, o);
            if (f2 < bu || (f2 == bu && i2 < iu)) { bu = f2; iu = i2; }
            const double f3 = __shfl_xor_sync(~0u, bl, o); const int i3 = __shfl_xor_sync(~0u, il, o);
            if (f3 > bl || (f3 == bl && i3 < il)) { bl = f3; il = i3; }
        }
        if (lane == 0) { wf[0][warp] = bu; wi[0][warp] = iu; wf[1][warp] = bl; wi[1][warp] = il; }
        __syncthreads();
        bu = wf[0][0]; iu = wi[0][0]; bl = wf[1][0]; il = wi[1][0];
        for (int w = 1; w < NTH / 32; ++w) {
            if (wf[0][w] < bu || (wf[0][w] == bu && wi[0][w] < iu)) { bu = wf[0][w]; iu = wi[0][w]; }
            if (wf[1][w] > bl || (wf[1][w] == bl && wi[1][w] < il)) { bl = wf[1][w]; il = wi[1][w]; }
        }
        acc += bu + iu + bl + il;
        __syncthreads();
    }
    if (t == 0) out[blockIdx.x] = acc;
}

int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    Rec* recs; LL* ll; LL* bc; unsigned long long* cnt; double* out;
    cudaMalloc(&recs, 2 * nsm * sizeof(Rec)); cudaMalloc(&ll, 2 * nsm * sizeof(LL));
    cudaMalloc(&bc, 16 * sizeof(LL)); cudaMalloc(&cnt, 8); cudaMalloc(&out, nsm * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000;
    auto time = [&](const char* name, auto fn) {
        cudaMemset(cnt, 0, 8); cudaMemset(ll, 0, 2 * nsm * sizeof(LL)); cudaMemset(bc, 0, 16 * sizeof(LL));
        cudaDeviceSynchronize();
        cudaEventRecord(e0); fn(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%-44s %7.3f us/exchange  (%s)\n", name, 1e3 * ms / iters, cudaGetErrorString(cudaGetLastError()));
    };
    time("S1 counter+threadfence, 1 poller, warp reads", [&] { s1<<<nsm, NTH>>>(recs, cnt, iters, out); });
    time("S2 LL all-to-all, warp polls all records", [&] { s2<<<nsm, NTH>>>(ll, iters, out); });
    time("S3 LL aggregator + 8 broadcast replicas", [&] { s3<<<nsm, NTH>>>(ll, bc, iters, out); });
    time("S4 counter red.release, warp reads unrolled", [&] { s4<<<nsm, NTH>>>(recs, cnt, iters, out); });
    uint4* r5; cudaMalloc(&r5, (size_t)16 * nsm * 6 * 16);
    auto z5 = [&] { cudaMemset(r5, 0, (size_t)16 * nsm * 6 * 16); cudaDeviceSynchronize(); };
    z5(); time("S5 compact 32B, direct, NREP=1", [&] { s5<1><<<nsm, NTH>>>(r5, iters, out, 2); });
    z5(); time("S5 compact 32B, direct, NREP=4", [&] { s5<4><<<nsm, NTH>>>(r5, iters, out, 2); });
    z5(); time("S5 compact 32B, direct, NREP=8", [&] { s5<8><<<nsm, NTH>>>(r5, iters, out, 2); });
    z5(); time("S6 96B (6x16B), direct, NREP=1", [&] { s5<1><<<nsm, NTH>>>(r5, iters, out, 6); });
    z5(); time("S6 96B (6x16B), direct, NREP=4", [&] { s5<4><<<nsm, NTH>>>(r5, iters, out, 6); });
    return 0;
}
