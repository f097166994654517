// predict_tc.cuh -- batched decision values on the 5th-generation tensor cores.
//
//   dec_i = sum_s coef_s K(sv_s, t_i) + b
//   RBF:    K = exp(-gamma (|t|^2 + |s|^2 - 2 t.s)),  linear: K = t.s
//
// The contraction T * SV^T (m x n_sv x d) is a dense GEMM that is never materialised:
// each CTA owns 128 test rows, streams the support vectors in tiles of BN (256), and the
// epilogue turns every 128 x BN accumulator tile into kernel values and reduces it
// over the support vectors on the fly.
//
//   * operands in "3xTF32": x = hi + lo with hi = x rounded to tf32 and lo = tf32(x - hi);
//     t.s = hi.hi + hi.lo + lo.hi (three tcgen05.mma kind::tf32 into one fp32 TMEM
//     accumulator), ~2^-21 relative per product instead of tf32's 2^-11
//   * operands are pre-packed once into the K-major, no-swizzle core-matrix layout of
//     tcgen05 shared-memory descriptors (8 rows x 16 bytes per core matrix, LBO = 128 B
//     between K-adjacent core matrices, SBO = 8 BK x 4 B between 8-row groups), so every
//     stage is two contiguous cp.async.bulk copies (A hi|lo, B hi|lo; 48 KB with BN = 256)
//   * warp roles: warp 0 producer (bulk copies, mbarrier ring), warp 1 MMA issuer (one
//     thread; TMEM allocation), warps 2-17 epilogue (tcgen05.ld 32x32b, one test row per
//     thread, 4 warps per TMEM lane quarter); TcCfg: 128 x 256 accumulator tiles, two in
//     TMEM, so the epilogue of tile j overlaps the MMAs of tile j + 1
//   * epilogue: x = -gamma (|t|^2 + |s|^2 - 2 t.s) from exact fp64 norms, K = exp(x) with
//     only what needs fp64 in fp64 (exp_split: fp64 range reduction and final fma, the small
//     correction polynomial in fp32; relative error < 4e-13), dec accumulated with fp64 fma --
//     an fp32 exp or sum would cost up to 1e-3 on Adult-like data (C = 100, 15 distinct
//     kernel values, correlated rounding).  The fp64 pipe is shared with the tensor pipe, so
//     every fp64 operation of the epilogue is taken from the MMAs.
// Not bit-exact (tensor cores); parity vs the oracle is BASELINE.json's 1e-4 absolute.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace svmtc {

constexpr int BM = 128;          // test rows per CTA (MMA M)
constexpr int EPI_WARPS = 16;                     // epilogue: EPI_WARPS / 4 warps per TMEM lane quarter
constexpr int NPART = EPI_WARPS / 4;              // column parts of an accumulator tile
constexpr int NTHREADS = 64 + 32 * EPI_WARPS;

// Tile shapes: BN support vectors per accumulator tile (MMA N), BK tf32 elements of K per
// stage, NACC accumulators in TMEM (the MMAs of tile j + 1 .. j + NACC - 1 overlap the
// epilogue of tile j).  BN = 128: 3 stages of 64 KB, 4 accumulators (512 TMEM columns);
// BN = 256: 4 stages of 48 KB, 2 accumulators (all 512 columns) -- each stage's A block
// then feeds twice the MMA work of BN = 128, 25% fewer bytes from L2 per product.  (BN is
// a multiple of 64: the epilogue's 4 column parts load 16 columns at a time.)
template <int BN_>
struct TcCfg {
    static constexpr int BN = BN_;
    static constexpr int BK = BN_ == 128 ? 32 : 16;
    static constexpr int STAGES = BN_ == 128 ? 3 : 4;
    static constexpr int NACC = 512 / BN_;
    static_assert(BN_ % 64 == 0 && NACC * BN_ <= 512, "tile width");
    static constexpr int A_FLOATS = BM * BK;      // one of A hi / A lo per stage
    static constexpr int B_FLOATS = BN * BK;      // one of B hi / B lo per stage
    static constexpr int STAGE_BYTES = (2 * A_FLOATS + 2 * B_FLOATS) * 4;
    static constexpr int TMEM_COLS = 512;         // (a power of two >= NACC * BN)
    static constexpr int SBO = 8 * BK * 4;        // bytes between 8-row groups of a block
    // instruction descriptor: D f32, A/B tf32, both K-major, N = BN, M = BM
    static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                      ((uint32_t)(BM >> 4) << 24);
};

// element (r, k) of a [rows][bk] block in the core-matrix order
__host__ __device__ inline int packed_index(int r, int k, int bk) {
    return (((r >> 3) * (bk / 4) + (k >> 2)) << 5) + ((r & 7) << 2) + (k & 3);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// shared-memory matrix descriptor: K-major, no swizzle, LBO 128 B, SBO bytes between 8-row
// groups, sm100 version 1
template <int SBO>
__device__ __forceinline__ uint64_t smem_desc(const void* p) {
    const uint64_t a = (smem_u32(p) >> 4) & 0x3fffu;
    return a | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(SBO >> 4) << 32) | (1ull << 46);
}

template <uint32_t IDESC>
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "setp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                 :: "r"(tmem_d), "l"(da), "l"(db), "n"(IDESC), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(smem_u32(bar)) : "memory");
}

// exp(x) for x <= 0 in fp64 to a few ulp, for the epilogue (the decision values are
// checked to 1e-4 absolute, the tf32 products are good to ~2^-21, so a correctly rounded
// exp is not needed here -- the exact path has one).  x = (n / 64) ln 2 + r, |r| <= ln 2 / 128:
// exp(x) = 2^(n >> 6) * 2^((n & 63) / 64) * exp(r), exp(r) by its degree-5 Taylor
// polynomial (truncation r^6 / 720 < 4e-17), 2^(j / 64) from a 64-entry table in shared
// memory; x < -708 gives 0 (the kernel value is below 3.3e-308).  About 11 fp64
// operations against ~25 for the libdevice exp, which bounded the epilogue.
__device__ __forceinline__ double exp_nonpos(double x, const double* __restrict__ t64) {
    if (x < -708.0) return 0.0;
    const double sh = 6755399441055744.0;                    // 1.5 * 2^52: round to integer
    const double kk = fma(x, 92.33248261689366, sh);     // x * 64 / ln 2 + shift
    const int n = __double2loint(kk);
    const double nd = kk - sh;
    double r = fma(nd, -0.010830424695996044, x);           // ln 2 / 64, high part (35 bits:
    r = fma(nd, -2.5310172166650877e-13, r);                 // nd * hi exact) and low part
    double q = fma(r, 1.0 / 120.0, 1.0 / 24.0);
    q = fma(q, r, 1.0 / 6.0);
    q = fma(q, r, 0.5);
    q = fma(q, r, 1.0);
    q = fma(q, r, 1.0);
    const double v = t64[n & 63] * q;
    return __hiloint2double(__double2hiint(v) + (n >> 6) * (1 << 20), __double2loint(v));
}

// the same by a degree-13 polynomial after reduction by ln 2 (no table; |r| <= ln 2 / 2,
// truncation < 4e-17)
__device__ __forceinline__ double exp_nonpos_poly(double x) {
    if (x < -708.0) return 0.0;
    const double sh = 6755399441055744.0;
    const double kk = fma(x, 1.4426950408889634, sh);        // x / ln 2 + shift
    const int n = __double2loint(kk);
    const double nd = kk - sh;
    double r = fma(nd, -0.693147180559663, x);               // ln 2, high part (41 bits, |nd| < 2^11:
    r = fma(nd, -2.8235290563031577e-13, r);                 // exact product) and low part
    double q = 1.0 / 6227020800.0;
    q = fma(q, r, 1.0 / 479001600.0);
    q = fma(q, r, 1.0 / 39916800.0);
    q = fma(q, r, 1.0 / 3628800.0);
    q = fma(q, r, 1.0 / 362880.0);
    q = fma(q, r, 1.0 / 40320.0);
    q = fma(q, r, 1.0 / 5040.0);
    q = fma(q, r, 1.0 / 720.0);
    q = fma(q, r, 1.0 / 120.0);
    q = fma(q, r, 1.0 / 24.0);
    q = fma(q, r, 1.0 / 6.0);
    q = fma(q, r, 0.5);
    q = fma(q, r, 1.0);
    q = fma(q, r, 1.0);
    // 2^n in two halves (n >= -1022 - 1 when x >= -708: the result stays normal)
    return __hiloint2double(__double2hiint(q) + n * (1 << 20), __double2loint(q));
}

// fp32 <-> fp64 by integer operations (no conversion instruction on the fp64 pipe, which
// the tensor cores share).  widen: exact; 0 and fp32 subnormals -> +-0 (a dot product of
// fp32 data is never subnormal unless 0 or a cancellation below 2^-126, whose effect on
// exp(.) is nil).  narrow: truncation (relative error < 2^-23), |x| < 2^-126 -> 0.
__device__ __forceinline__ double widen_f32_int(uint32_t fb) {
    const uint32_t ex = (fb >> 23) & 0xffu;
    const uint32_t hi = ex == 0u ? (fb & 0x80000000u)
                                 : ((fb & 0x80000000u) | ((ex + 896u) << 20) | ((fb >> 3) & 0xfffffu));
    const uint32_t lo = ex == 0u ? 0u : (fb << 29);
    return __hiloint2double((int)hi, (int)lo);
}
__device__ __forceinline__ float narrow_f64_int(double x) {
    const uint32_t h = (uint32_t)__double2hiint(x), l = (uint32_t)__double2loint(x);
    const uint32_t e = (h >> 20) & 0x7ffu;
    const uint32_t fb = (h & 0x80000000u) | ((e - 896u) << 23) | ((h & 0xfffffu) << 3) | (l >> 29);
    return e > 896u && e < 1151u ? __uint_as_float(fb) : 0.0f;
}

// The epilogue's kernel value K = exp(x), x = c + g2 * dot (c = -gamma (|t|^2 + |s|^2),
// g2 = 2 gamma, dot = the fp32 accumulator t.s), with as few fp64-pipe operations as the
// accuracy allows -- the fp64 pipe is shared with the tensor cores (ncu: pipe_shared =
// fp64 + tensor), so every fp64 operation of the epilogue is taken from the MMAs.
//   x = (n / 256) ln 2 + r, n = nearest integer of x 256 / ln 2 (1.5 2^52 shift), r by one
//   fma with ln 2 / 256 rounded to double (|n| < 2^18 for x >= -708: error < 6e-14 abs.),
//   exp(x) = 2^(n >> 8) 2^((n & 255) / 256) (1 + r + p),  p = r^2 (1/2 + r/6 + r^2/24)
//   in fp32 (|r| <= ln 2 / 512, |p| <= 9.3e-7: fp32's ~2^-22 relative error on p is
//   < 3e-13 of K; truncation r^5/120 < 4e-17), 2^(j / 256) from a shared-memory table.
// Relative error of K < 4e-13 (BASELINE.json's decision tolerance is 1e-4 absolute;
// with sum |coef| <= 3e6 the kernel-value error adds < 1.2e-6).  x < -707.5 -> 0 (K < 1e-307).
// INT_CVT: the fp32 <-> fp64 conversions by integer operations instead of F2F.
template <bool INT_CVT>
__device__ __forceinline__ double exp_split(uint32_t dot_bits, double c, double g2, const double* __restrict__ t256) {
    const double dot = INT_CVT ? widen_f32_int(dot_bits) : (double)__uint_as_float(dot_bits);
    const double x = fma(g2, dot, c);
    const double sh = 6755399441055744.0;                     // 1.5 * 2^52
    const double tN = fma(x, 369.32993046757464, sh);         // x * 256 / ln 2 + shift
    const int n = __double2loint(tN);
    const double nd = tN - sh;
    const double r = fma(nd, -0.0027076061740622863, x);     // ln 2 / 256
    const float rf = INT_CVT ? narrow_f64_int(r) : __double2float_rn(r);
    const float pf = (rf * rf) * fmaf(fmaf(rf, 1.0f / 24.0f, 1.0f / 6.0f), rf, 0.5f);
    const double q = r + (INT_CVT ? widen_f32_int(__float_as_uint(pf)) : (double)pf);
    const double T = t256[n & 255];
    const double v = fma(T, q, T);
    const double kv = __hiloint2double(__double2hiint(v) + (n >> 8) * (1 << 20), __double2loint(v));
    return n < -261376 ? 0.0 : kv;                            // x < -707.5 (n >> 8 >= -1021: v 2^(n >> 8) normal)
}

// 16 accumulator columns of one test row into its running sum.  FAC (EXPV 5): the row's
// factor exp(a_t), a_t = -gamma |t|^2, is left out of every kernel value and applied once
// to the row's sum (one fp64 add fewer per (row, SV)); the caller takes it only when
// a_t >= -600 for all rows of the warp, so exp(x - a_t) <= exp(600) stays finite.
template <int KERNEL, int EXPV, bool FAC>
__device__ __forceinline__ void epi16(const uint32_t (&v)[16], const double2* __restrict__ qc_c, double a_t,
                                      double g2, const double* __restrict__ t64, double& acc_d) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        double kv;
        const double2 sc = qc_c[j];             // {-gamma |s|^2, coef}: one 16-byte load
        if (KERNEL == 1 && EXPV >= 3) {
            kv = exp_split<EXPV == 4>(v[j], FAC ? sc.x : a_t + sc.x, g2, t64);
        } else if (KERNEL == 1) {
            // fp32 accumulator -> fp64 by integer ops (the fp64 pipe is shared with
            // the tensor cores): rebias the exponent, widen the mantissa; 0 stays 0
            // (the dot of fp32 data is never subnormal unless 0 or a cancellation
            // below 2^-126, whose exp(.) contribution is 1 either way)
            const uint32_t fb = v[j];
            const uint32_t ex = (fb >> 23) & 0xffu;
            const uint32_t hi = ex == 0u ? (fb & 0x80000000u)
                                         : ((fb & 0x80000000u) | ((ex + 896u) << 20) | ((fb >> 3) & 0xfffffu));
            const uint32_t lo = ex == 0u ? 0u : (fb << 29);
            const double dot = __hiloint2double((int)hi, (int)lo);
            // (x > 0 by rounding, when t ~ s, gives K = 1 + O(1e-16): not clamped)
            const double x = fma(g2, dot, a_t + sc.x);
            if (EXPV == 0) kv = exp(x);
            else if (EXPV == 1) kv = exp_nonpos(x, t64);
            else kv = exp_nonpos_poly(x);
        } else {
            kv = (double)__uint_as_float(v[j]);
        }
        acc_d = fma(sc.y, kv, acc_d);
    }
}

// EXPV: the epilogue's exp -- 0 CUDA's fp64 exp, 1 table-driven (exp_nonpos), 2 polynomial,
// 3 exp_split with F2F conversions, 4 exp_split with integer conversions, 5 exp_split with
// the row factor exp(-gamma |t|^2) applied once per row (epi16 FAC).  BN_: TcCfg.
template <int KERNEL, int EXPV, int BN_>
__global__ void __launch_bounds__(NTHREADS, 1)
k_predict_tc(const float* __restrict__ A,   // packed test rows [m_tiles][k_chunks][2][BM*BK]
             const float* __restrict__ B,   // packed SVs       [n_tiles][k_chunks][2][BN*BK]
             const double* __restrict__ qt, // |t_i|^2 [m_pad]
             const double2* __restrict__ qc, // {RBF: -gamma |s|^2 (linear: unused), coef (0 for padding)} [n_pad]
             int k_chunks, int n_tiles, long long m, double b, double gamma,
             double* __restrict__ dec) {
    using Cf = TcCfg<BN_>;
    constexpr int BN = Cf::BN, BK = Cf::BK, STAGES = Cf::STAGES, TMEM_COLS = Cf::TMEM_COLS, NACC = Cf::NACC;
    constexpr int AF = Cf::A_FLOATS, BF = Cf::B_FLOATS;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    float* stage_base = reinterpret_cast<float*>(smem_raw);
    __shared__ uint64_t full[STAGES], empty[STAGES], tfull[NACC], tempty[NACC];
    __shared__ uint32_t tmem_base_sh;
    __shared__ double part_sh[NPART][BM];           // the column parts' partial sums
    __shared__ double t64[256];                     // 2^(j / 64) (exp_nonpos), 2^(j / 256) (exp_split)
    if (threadIdx.x < 256) t64[threadIdx.x] = exp2((double)threadIdx.x / (EXPV >= 3 ? 256.0 : 64.0));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mt = blockIdx.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int a = 0; a < NACC; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], EPI_WARPS); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(smem_u32(&tmem_base_sh)), "n"(TMEM_COLS) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base_sh;

    if (warp == 0) {
        // ---------------- producer
        if (lane == 0) {
            const float* a_tile = A + (size_t)mt * k_chunks * 2 * AF;
            int slot = 0;
            uint32_t par = 0;
            bool wrapped = false;
            for (int nt = 0; nt < n_tiles; ++nt) {
                const float* b_tile = B + (size_t)nt * k_chunks * 2 * BF;
                for (int kc = 0; kc < k_chunks; ++kc) {
                    if (wrapped) mbar_wait(&empty[slot], par ^ 1u);
                    float* st = stage_base + (size_t)slot * (2 * AF + 2 * BF);
                    mbar_arrive_tx(&full[slot], Cf::STAGE_BYTES);
                    bulk_g2s(st, a_tile + (size_t)kc * 2 * AF, 2 * AF * 4, &full[slot]);
                    bulk_g2s(st + 2 * AF, b_tile + (size_t)kc * 2 * BF, 2 * BF * 4, &full[slot]);
                    if (++slot == STAGES) { slot = 0; par ^= 1u; wrapped = true; }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        int slot = 0;
        uint32_t par = 0;
        for (int nt = 0; nt < n_tiles; ++nt) {
            const int acc = nt % NACC;
            const uint32_t tacc = tmem + acc * BN;
            if (nt >= NACC) mbar_wait(&tempty[acc], ((nt / NACC) - 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            for (int kc = 0; kc < k_chunks; ++kc) {
                mbar_wait(&full[slot], par);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (lane == 0) {
                    const float* st = stage_base + (size_t)slot * (2 * AF + 2 * BF);
                    const float* ahi = st;
                    const float* alo = st + AF;
                    const float* bhi = st + 2 * AF;
                    const float* blo = st + 2 * AF + BF;
                    constexpr uint32_t ID = Cf::IDESC;
                    constexpr int SB = Cf::SBO;
#pragma unroll
                    for (int k8 = 0; k8 < BK / 8; ++k8) {
                        const int off = k8 * 64;            // 2 core matrices (256 B) per K = 8
                        const uint32_t first = (kc == 0 && k8 == 0) ? 0u : 1u;
                        mma_tf32<ID>(tacc, smem_desc<SB>(ahi + off), smem_desc<SB>(bhi + off), first);
                        mma_tf32<ID>(tacc, smem_desc<SB>(ahi + off), smem_desc<SB>(blo + off), 1u);
                        mma_tf32<ID>(tacc, smem_desc<SB>(alo + off), smem_desc<SB>(bhi + off), 1u);
                    }
                    mma_commit(&empty[slot]);               // frees the stage when done
                    if (kc == k_chunks - 1) mma_commit(&tfull[acc]);
                }
                __syncwarp();
                if (++slot == STAGES) { slot = 0; par ^= 1u; }
            }
        }
    } else {
        // ---------------- epilogue: warps 2.. -> TMEM lane quarter (warp % 4); the warps of a
        // quarter split the columns of every accumulator tile into NPART parts
        const int quarter = warp & 3;
        const int half = (warp - 2) >> 2;                 // column part
        const int row = quarter * 32 + lane;
        const long long gi = (long long)mt * BM + row;
        // x = -gamma (|t|^2 + |s|^2 - 2 t.s) = (a_t + b_s) + 2 gamma (t.s), a_t = -gamma |t|^2,
        // b_s = -gamma |s|^2 (precomputed per SV, qs holds b_s for RBF): two fp64 operations
        // per (row, SV) instead of four -- they share the pipe with the tensor cores
        const double q_t = qt[(long long)mt * BM + row];
        const double a_t = -gamma * q_t;
        const double g2 = 2.0 * gamma;
        const bool fac = KERNEL == 1 && EXPV == 5 && __all_sync(0xffffffffu, a_t >= -600.0);
        double acc_d = 0.0;
        for (int nt = 0; nt < n_tiles; ++nt) {
            const int acc = nt % NACC;
            mbar_wait(&tfull[acc], (nt / NACC) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const double2* qc_t = qc + (size_t)nt * BN;
#pragma unroll 1
            for (int c0 = half * (BN / NPART); c0 < (half + 1) * (BN / NPART); c0 += 16) {
                // 16 accumulator columns per load (x16)
                uint32_t v[16];
                const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + acc * BN + c0;
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
                    "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                      "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                      "=r"(v[14]), "=r"(v[15])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                // fully unrolled: v[j] must index registers (a partial unroll put v in local
                // memory -- STL/LDL per element)
                if (fac) epi16<KERNEL, EXPV, true>(v, qc_t + c0, a_t, g2, t64, acc_d);
                else epi16<KERNEL, EXPV, false>(v, qc_t + c0, a_t, g2, t64, acc_d);
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        // the parts' partial sums, combined in a fixed order (part 0, 1, ...)
        part_sh[half][row] = acc_d;
        asm volatile("bar.sync 1, %0;" :: "n"(32 * EPI_WARPS) : "memory");
        if (half == 0 && gi < m) {
            double sum = acc_d;
            for (int p = 1; p < NPART; ++p) sum += part_sh[p][row];
            dec[gi] = (fac ? sum * exp(a_t) : sum) + b;
        }
    }
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(TMEM_COLS) : "memory");
    }
}

// Pack rows [rows][d] fp32 (row-major) into [tiles][k_chunks][hi|lo][tr*bk] tf32 blocks
// (tr rows per tile, bk elements of K per chunk); also |x|^2 in fp64.  Padding rows /
// features are zero.
__global__ void k_pack_3xtf32(const float* __restrict__ X, long long rows, int d, int k_chunks,
                              long long rows_pad, int tr, int bk, float* __restrict__ out,
                              double* __restrict__ norms) {
    const int BK = bk;
    const int TILE_FLOATS = tr * bk;
    const long long total = rows_pad * (long long)k_chunks * BK;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long r = e / ((long long)k_chunks * BK);
        const int k = (int)(e - r * (long long)k_chunks * BK);
        const float x = (r < rows && k < d) ? X[r * d + k] : 0.0f;
        uint32_t hb;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(x));
        const float hi = __uint_as_float(hb);
        uint32_t lb;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lb) : "f"(x - hi));
        const float lo = __uint_as_float(lb);
        const long long tile = r / tr;
        const int rr = (int)(r - tile * tr), kc = k / BK, kk = k - kc * BK;
        float* blk = out + ((size_t)tile * k_chunks + kc) * 2 * TILE_FLOATS;
        blk[packed_index(rr, kk, bk)] = hi;
        blk[TILE_FLOATS + packed_index(rr, kk, bk)] = lo;
    }
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < rows_pad;
         r += (long long)gridDim.x * blockDim.x) {
        double s = 0.0;
        if (r < rows)
            for (int k = 0; k < d; ++k) { const double v = X[r * d + k]; s = fma(v, v, s); }
        norms[r] = s;
    }
}

}  // namespace svmtc
