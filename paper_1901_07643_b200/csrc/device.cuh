// device.cuh -- device helpers shared by the sm_100a kernels: the Givens
// coefficients of a GRC (Eq.4 with reading G1), the fast fp64
// log of the BIC (a9, reading G5), the packed-triangle GRC used by the seed
// derivation (a5), the BIC/tie-break rules (G13, G14) and the table index
// (a10).
#pragma once
#include <cstdint>
#include <cmath>
#include "kernels.h"

namespace bnr {

#define FULLMASK 0xffffffffu

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o);
    return v;
}

// 1/sqrt(x) for a positive normal x: rsqrt.approx.ftz.f64 then one Halley step (see givens)
__device__ __forceinline__ double rsqrt_h(double x)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x, y * y, 1.0);
    return fma(y, e * fma(e, 0.375, 0.5), y);
}

// Givens coefficients for the GRC (Eq.4 read with G1).  h2 == 0 can only
// happen on rank-deficient data (rejected at create); identity then.
__device__ __forceinline__ void givens(double a, double b, double& c, double& s, double& h)
{
    const double h2 = fma(a, a, b * b);
    // 1/sqrt(h2): hardware approximation (relative error <= 9.1e-7, measured) + one
    // third-order (Halley) step y (1 + e/2 + 3e^2/8), e = 1 - h2 y^2: 2.2e-16, measured on
    // 4M values over 1e-87..1e87 (two Newton steps: 2.6e-16 in 3 more FP64 operations);
    // no special-case branches: h2 is a positive normal number unless the data is rank deficient
    const double y = rsqrt_h(h2);
    const bool ok = h2 > 0.0;
    c = ok ? a * y : 1.0;
    s = ok ? b * y : 0.0;
    h = ok ? h2 * y : 0.0;
}

// Givens coefficients without the rank-deficiency guard: in the walk and the
// seed derivation, b is a diagonal entry r_{i+1,i+1}, nonzero for full-rank
// data (checked at create, G26), so h2 > 0.
__device__ __forceinline__ void givens_fr(double a, double b, double& c, double& s, double& h)
{
    const double h2 = fma(a, a, b * b);
    const double y = rsqrt_h(h2);
    c = a * y;
    s = b * y;
    h = h2 * y;
}

// user id of seed-tree level l (plan.h hv_id): top ids first, the gang ids last
__device__ __forceinline__ int hv_of(int l, int m, int gs, int fv0) { return l < gs ? m - 1 - l : fv0 - 1 - (l - gs); }

// Fast natural log for the BIC (a9).  x = 2^e f, f in [1,2); j = top kLnBits bits
// of f's mantissa; tab[j] = (r_j, -ln r_j) with r_j ~ 1/(1 + (j+0.5)/2^kLnBits)
// (host, long double); u = f r_j - 1 (|u| <= 2^-(kLnBits+1));
// ln x = e ln2 + (-ln r_j) + log1p(u), log1p(u) = u q(u):
//   BNREG_LN_DEG 4 (512 entries): q = 1 - u/2 + u^2/3 - u^3/4, truncation u^5/5 < 2e-16;
//   BNREG_LN_DEG 3 (1024 entries): q = 1 + u(-1/2 + u/3), truncation u^4/4 < 1.5e-14
//   (BIC error (n/2) 1.5e-14 <= 7.5e-11 at n = 1e4, against the 1e-6 bar).
// Constants are compile-time literals: the compiler keeps them in its constant bank and
// uses them as DFMA operands directly.
// (BNREG_LN_DEG, kLnBits, kLnEntries: kernels.h)
constexpr double kLn2 = 6.93147180559945309417e-01;   // correctly rounded: e * ln2 in one FMA
                                                        // (error |e| * 2.3e-17 <= 2.4e-14 for |e| <= 1023)

__device__ __forceinline__ double ln_poly(double u, double base)
{
#if BNREG_LN_DEG == 3
    const double t = fma(u, 1.0 / 3.0, -0.5);
    const double q = fma(u, t, 1.0);
    return fma(u, q, base);
#else
    // Horner, not Estrin: one fma with two constants (1/3 in a register) instead of two, no
    // u^2 (measured: 2.7% fewer walk instructions, 1.9% faster at cfg5)
    const double t1 = fma(u, -0.25, 1.0 / 3.0);
    const double t2 = fma(u, t1, -0.5);
    const double q = fma(u, t2, 1.0);
    return fma(u, q, base);
#endif
}

// byte offset of the table entry of x's mantissa (16 B entries)
__device__ __forceinline__ int ln_tab_off(int hi) { return (hi >> (16 - kLnBits)) & ((kLnEntries - 1) << 4); }

__device__ __forceinline__ double fast_ln9(double x, const double2* tab)
{
    const int hi = __double2hiint(x), lo = __double2loint(x);
    const int e = (hi >> 20) - 1023;
    const double f = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);
    const double2 t = *(const double2*)((const char*)tab + ln_tab_off(hi));
    const double base = fma((double)e, kLn2, t.y);
    return ln_poly(fma(f, t.x, -1.0), base);
}

// fast_ln9 with the table addressed in the shared window (tab = shared address).
__device__ __forceinline__ double fast_ln9s(double x, unsigned tab)
{
    const int hi = __double2hiint(x), lo = __double2loint(x);
    const int e = (hi >> 20) - 1023;
    const double f = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);
    double tx, ty;
#ifdef BNREG_FAKE_LN   // timing experiment only (wrong logs): every lane reads entry 0 (one broadcast wavefront)
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(tx), "=d"(ty) : "r"(tab + (ln_tab_off(hi) & 0)));
#else
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(tx), "=d"(ty) : "r"(tab + ln_tab_off(hi)));
#endif
#ifdef BNREG_LN_MAGIC   // the exponent as a double without I2F: (2^52 + E) - (2^52 + 1023) exactly
    const double ed = __hiloint2double(0x43300000, (int)((unsigned)hi >> 20)) - 4503599627371519.0;
    (void)e;
    const double base = fma(ed, kLn2, ty);
#else
    const double base = fma((double)e, kLn2, ty);
#endif
    return ln_poly(fma(f, tx, -1.0), base);
}

// BIC (reading G5): -(n/2) ln(RSS/n) - (n/2)(1 + ln 2pi) - (|S|/2) ln n
//   = mhalf_n * ln RSS + K(|S|);  +inf for RSS <= 1e-300 (G13).
__device__ __forceinline__ double bic_of(double rss, double lnr, double mhalf_n, double Kw)
{
    const double bic = fma(mhalf_n, lnr, Kw);
    return rss > 1e-300 ? bic : __longlong_as_double(0x7ff0000000000000LL);
}

// Argmax tie-break (G14): larger BIC, then smaller |S|, then smaller mask.
__device__ __forceinline__ bool tie_better(double b, uint32_t S, double cb, uint32_t cm)
{
    if (b != cb) return b > cb;
    const int s1 = __popc(S), s2 = __popc(cm);
    return s1 != s2 ? s1 < s2 : S < cm;
}

// Same rule for (BIC, mask) candidates where mask 0xffffffff means "none".
__device__ __forceinline__ bool better(double b1, uint32_t m1, double b2, uint32_t m2)
{
    if (m1 == 0xffffffffu) return false;
    if (m2 == 0xffffffffu) return true;
    return tie_better(b1, m1, b2, m2);
}

// Offset (in entries) of family (v, S) inside child v's block of this rank's
// table, given lm = (1 << v) - 1: compress(S, v) is the bitwise select
// lm ? S : S >> 1 (bit v of S is 0).  World 1: the block is v 2^(m-1).. and
// the offset is the compressed mask; otherwise (plan.h) child v's 2^(m-r)
// entries hold the masks whose top selector bits match this rank's patterns.
template <bool WORLD1>
__device__ __forceinline__ uint32_t block_offset(const TravParams& P, uint32_t S, uint32_t S1, uint32_t lm)
{
    const uint32_t cpr = (S & lm) | (S1 & ~lm);
    if (WORLD1) return cpr;
    const int v = __popc(lm);
    const bool sel = v >= P.m - P.r;
    const int sh = sel ? P.m - P.r : P.m - 1 - P.r;
    return (cpr & ((1u << sh) - 1u)) + ((!sel && (cpr >> sh) != P.patlo) ? (1u << sh) : 0u);
}

}  // namespace bnr
