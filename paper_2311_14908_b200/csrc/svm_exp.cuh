// svm_exp.cuh -- correctly rounded fp64 exp for the RBF kernel, sm_100a + host.
//
// The RBF kernel is K(x, z) = exp(-gamma ||x - z||^2) (SPEC.md
// L120).  The CUDA path evaluates exp correctly rounded (reading R14), so
// every kernel value is the unique double nearest the exact exponential of the
// fp64 argument; with identical arguments the trajectory of SMO pair choices is then
// bit-reproducible against any other correctly rounded evaluation.
//
// Method (table-driven, two-phase / Ziv):
//   x = (32 k + j) ln2/32 + r,  |r| <= ln2/64,  r in double-double (3-part ln2/32)
//   exp(x) = 2^k * T_j * exp(r),  T_j = 2^(j/32) as double-double
//   fast phase:  exp(r) - 1 = r + r^2/2 (error-free) + tail (double Horner,
//                degree 3..8), times T in double-double; relative error < 2^-71
//   if the fast result lies within 2^-68 (relative) of a rounding boundary,
//   slow phase:  exp(r) by a degree-13 double-double Horner (~2^-100)
// Arguments below -708 return 0 (reading R15); x = 0 returns 1.
// Domain used by the solver: x <= 0.  Constants: exp_table.inc
// (tools/gen_exp_table.py, decimal arithmetic).
//
// Compiled with --fmad=false: products and sums below are never contracted.
#pragma once

#include <stdint.h>
#include <string.h>
#include <math.h>

#include "exp_table.inc"

#if defined(__CUDACC__)
#define SVM_HD __host__ __device__ __forceinline__
#define SVM_HDM __host__ __device__ __forceinline__
#else
#define SVM_HD static inline
#define SVM_HDM inline
#endif

namespace svmexp {

#if defined(__CUDACC__)
// fast-phase coefficients in the constant bank: DFMA takes them as c[][] operands directly
// (as literals they cost two uniform moves each)
__constant__ double c_IF_hi[16] = {SVM_EXP_IF_HI_INIT};
__constant__ double c_RED[4] = {SVM_EXP_INV_L32, SVM_EXP_L32_1, SVM_EXP_L32_2, SVM_EXP_L32_3};
__device__ const double d_T_hi[32] = {SVM_EXP_T_HI_INIT};
__device__ const double d_T_lo[32] = {SVM_EXP_T_LO_INIT};
__device__ const double d_IF_hi[16] = {SVM_EXP_IF_HI_INIT};
__device__ const double d_IF_lo[16] = {SVM_EXP_IF_LO_INIT};
#endif
static const double h_T_hi[32] = {SVM_EXP_T_HI_INIT};
static const double h_T_lo[32] = {SVM_EXP_T_LO_INIT};
static const double h_IF_hi[16] = {SVM_EXP_IF_HI_INIT};
static const double h_IF_lo[16] = {SVM_EXP_IF_LO_INIT};


struct dd { double hi, lo; };

SVM_HD uint64_t bits_of(double x) {
#if defined(__CUDA_ARCH__)
    return (uint64_t)__double_as_longlong(x);
#else
    uint64_t u; memcpy(&u, &x, 8); return u;
#endif
}
SVM_HD double from_bits(uint64_t u) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double((long long)u);
#else
    double x; memcpy(&x, &u, 8); return x;
#endif
}

SVM_HD dd fast_two_sum(double a, double b) {  // |a| >= |b|
    dd r; r.hi = a + b; r.lo = b - (r.hi - a); return r;
}
SVM_HD dd two_sum(double a, double b) {
    dd r; r.hi = a + b; double bb = r.hi - a; r.lo = (a - (r.hi - bb)) + (b - bb); return r;
}
SVM_HD dd two_prod(double a, double b) {
    dd r; r.hi = a * b; r.lo = fma(a, b, -r.hi); return r;
}
SVM_HD dd dd_mul(dd a, dd b) {
    dd p = two_prod(a.hi, b.hi);
    p.lo = p.lo + (a.hi * b.lo + a.lo * b.hi);
    return fast_two_sum(p.hi, p.lo);
}
SVM_HD dd dd_add(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    dd t = two_sum(a.lo, b.lo);
    s.lo = s.lo + t.hi;
    s = fast_two_sum(s.hi, s.lo);
    s.lo = s.lo + t.lo;
    return fast_two_sum(s.hi, s.lo);
}

// Distance (in units of 2^-68 relative) from the nearest rounding boundary test:
// returns true when (hi + lo) is provably on the same side of every boundary as
// hi, i.e. RN(exact) == hi, given |exact - (hi + lo)| <= hi * 2^-shift.
SVM_HD bool rounding_safe(double hi, double lo, int shift) {
    uint64_t b = bits_of(hi);
    uint64_t E = (b >> 52) & 0x7ffu;                       // hi is normal, in [0.98, 2)
    double hg = from_bits((E - 53u) << 52);                // ulp(hi) / 2
    bool pow2 = (b & 0xfffffffffffffull) == 0;
    double g = (lo < 0.0 && pow2) ? 0.5 * hg : hg;
    double margin = from_bits((E - (uint64_t)shift) << 52);  // 2^(e - shift) >= hi 2^-(shift+1)
    return fabs(fabs(lo) - g) > margin;
}

// The same test for 0.98 <= hi < 2 (the fast phase's R before scaling) in plain fp64
// compares: half an ulp of hi is 2^-53 in [1, 2) and 2^-54 below 1 -- also when hi = 1 and
// lo < 0, the one power of two in range -- and the margin is 2^-67 / 2^-68 (shift 67).
SVM_HD bool rounding_safe_r(double hi, double lo) {
    const bool up = hi >= 1.0;
    const double g = (hi > 1.0 || (hi == 1.0 && lo >= 0.0)) ? 0x1p-53 : 0x1p-54;
    const double margin = up ? 0x1p-67 : 0x1p-68;
    return fabs(fabs(lo) - g) > margin;
}

// Table accessors: host arrays, device global arrays (read-only path), or a caller-
// provided pointer (e.g. a shared-memory copy laid out T_hi[32] T_lo[32] IF_hi[16] IF_lo[16]).
struct HostTab {
    SVM_HDM double T_hi(int j) const { return h_T_hi[j]; }
    SVM_HDM double T_lo(int j) const { return h_T_lo[j]; }
    SVM_HDM double IF_hi(int i) const { return h_IF_hi[i]; }
    SVM_HDM double IF_lo(int i) const { return h_IF_lo[i]; }
};
#if defined(__CUDACC__)
struct GlobalTab {
    __device__ __forceinline__ double T_hi(int j) const { return __ldg(&d_T_hi[j]); }
    __device__ __forceinline__ double T_lo(int j) const { return __ldg(&d_T_lo[j]); }
    __device__ __forceinline__ double IF_hi(int i) const { return __ldg(&d_IF_hi[i]); }
    __device__ __forceinline__ double IF_lo(int i) const { return __ldg(&d_IF_lo[i]); }
};
struct PtrTab {
    const double* p;
    __device__ __forceinline__ double T_hi(int j) const { return p[j]; }
    __device__ __forceinline__ double T_lo(int j) const { return p[32 + j]; }
    __device__ __forceinline__ double IF_hi(int i) const { return p[64 + i]; }
    __device__ __forceinline__ double IF_lo(int i) const { return p[80 + i]; }
};
// copy of the tables in the PtrTab layout (96 doubles)
__device__ __forceinline__ double table_entry(int e) {
    return e < 32 ? d_T_hi[e] : e < 64 ? d_T_lo[e - 32] : e < 80 ? d_IF_hi[e - 64] : d_IF_lo[e - 80];
}
#endif
constexpr int EXP_TABLE_DOUBLES = 96;

// Fast phase: returns the correctly rounded exp(x) and sets safe = true, unless the
// double-double fast result lies too close to a rounding boundary (safe = false; the
// caller then uses exp_cr_slow).  Branch-free apart from that flag, so a caller can
// evaluate several exponentials side by side and take the (rare) slow path afterwards.
//
// Error budget of R = Rh + Rl against exp(x) / 2^k (relative, |r| <= ln2/64 < 2^-6.5):
// argument reduction 2^-80 (three-part ln2/32), truncation after r^8/8! 2^-77, the
// double-evaluated tail r^3 (1/3! + ... + r^5/8!) ~2^-73, the omitted rl r^2/2 ~2^-74,
// table 2^-106: < 2^-71 in all, against the 2^-67 margin of the rounding test.
template <class Tab>
SVM_HDM double exp_cr_fast(double x, const Tab& tab, bool& safe) {
#if defined(__CUDA_ARCH__)
    const double* IFH = c_IF_hi;
    const double INV_L32 = c_RED[0], L32_1 = c_RED[1], L32_2 = c_RED[2], L32_3 = c_RED[3];
#else
    constexpr double IFH[16] = {SVM_EXP_IF_HI_INIT};
    const double INV_L32 = SVM_EXP_INV_L32, L32_1 = SVM_EXP_L32_1, L32_2 = SVM_EXP_L32_2, L32_3 = SVM_EXP_L32_3;
#endif
    const bool special = (x == 0.0) || (x < -708.0);
    const double xc = special ? -1.0 : x;
    // N = nearest integer to x 32/ln2 by the 1.5 2^52 shift (exact: |N| < 2^16); the low
    // word of the shifted value is N as a 32-bit integer
    const double SH = 0x1.8p52;
    const double tN = fma(xc, INV_L32, SH);
    const double N = tN - SH;
    const int Ni = (int)(uint32_t)bits_of(tN);
    const int j = Ni & 31;
    const int k = Ni >> 5;                                 // floor(N / 32)
    // r = x - N ln2/32 = rh + rl
    const double r1 = fma(-N, L32_1, xc);          // exact (Sterbenz, 38-bit L1)
    const double p2h = N * L32_2;
    const double p2l = fma(N, L32_2, -p2h);
    const dd s = two_sum(r1, -p2h);
    const double rh = s.hi;
    const double rl = fma(-N, L32_3, s.lo - p2l);
    // exp(r) - 1 = qh + ql:  rh + rh^2/2 (error-free), + rl (1 + rh) + rh^3 P(rh)
    const double sqh = rh * rh, sql = fma(rh, rh, -sqh);
    const double h = 0.5 * sqh;
    const double qh = rh + h;                              // fast two-sum: |rh| >= |h|
    const double e = h - (qh - rh);
    double P = IFH[8];
    P = fma(P, rh, IFH[7]);
    P = fma(P, rh, IFH[6]);
    P = fma(P, rh, IFH[5]);
    P = fma(P, rh, IFH[4]);
    P = fma(P, rh, IFH[3]);
    const double tail = (sqh * rh) * P;
    const double ql = (e + 0.5 * sql) + (fma(rh, rl, rl) + tail);
    // R = T (1 + q), T = Th + Tl = 2^(j/32)
    const double Th = tab.T_hi(j), Tl = tab.T_lo(j);
    const double ph = Th * qh, pl = fma(Th, qh, -ph);
    const double Rh0 = Th + ph;                            // fast two-sum: Th >= 1 > |ph|
    const double Rl0 = ph - (Rh0 - Th);
    const double Rl1 = Rl0 + (pl + fma(Th, ql, fma(Tl, qh, Tl)));
    const double Rh = Rh0 + Rl1;                           // normalise
    const double Rl = Rl1 - (Rh - Rh0);
#if defined(SVM_EXP_PROBE) && !defined(__CUDA_ARCH__)
    if (!special)
        svm_exp_probe_fast(Rh * from_bits((uint64_t)(k + 1023) << 52),
                           Rl * from_bits((uint64_t)(k + 1023) << 52),
                           !rounding_safe(Rh, Rl, 67));
#endif
    safe = special || rounding_safe_r(Rh, Rl);
    const double scale = from_bits((uint64_t)(k + 1023) << 52);  // k >= -1022: normal
    const double v = Rh * scale;
    return x == 0.0 ? 1.0 : (x < -708.0 ? 0.0 : v);
}

// Slow phase (rare): exp(r) with a degree-13 double-double Horner scheme.
template <class Tab>
SVM_HDM double exp_cr_slow(double x, const Tab& tab) {
    double N = rint(x * SVM_EXP_INV_L32);
    int Ni = (int)N;
    int j = Ni & 31;
    int k = (Ni - j) / 32;
    double r1 = fma(-N, SVM_EXP_L32_1, x);
    dd p2 = two_prod(N, SVM_EXP_L32_2);
    dd s = two_sum(r1, -p2.hi);
    double rlo = (s.lo - p2.lo) - N * SVM_EXP_L32_3;
    dd r = two_sum(s.hi, rlo);
    dd p; p.hi = tab.IF_hi(13); p.lo = tab.IF_lo(13);
    for (int i = 12; i >= 0; --i) {
        dd c; c.hi = tab.IF_hi(i); c.lo = tab.IF_lo(i);
        p = dd_add(dd_mul(p, r), c);
    }
    dd T; T.hi = tab.T_hi(j); T.lo = tab.T_lo(j);
    dd R = dd_mul(p, T);
    double scale = from_bits((uint64_t)(k + 1023) << 52);
    return R.hi * scale;
}

template <class Tab>
SVM_HDM double exp_cr_t(double x, const Tab& tab) {
    bool safe;
    const double v = exp_cr_fast(x, tab, safe);
    return safe ? v : exp_cr_slow(x, tab);
}

SVM_HD double exp_cr(double x) {
#if defined(__CUDA_ARCH__)
    return exp_cr_t(x, GlobalTab());
#else
    return exp_cr_t(x, HostTab());
#endif
}

}  // namespace svmexp
