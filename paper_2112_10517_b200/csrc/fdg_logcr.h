/* fdg_logcr.h -- correctly rounded natural logarithm (double), C11 and CUDA.
 *
 * The reference's log means call libm `log` (fluxes.py:136, 143; CPython's
 * math.log -> glibc).  glibc's log is accurate to 0.52 ulp but not correctly
 * rounded (measured here: 6.4e-4 of inputs misrounded vs 200-bit mpmath), and
 * CUDA's log is a different 1-ulp approximation.  The FAITHFUL kernels use
 * this function instead: a table-driven double-double evaluation
 *
 *     x = 2^k m,  m in [1,2),  c_i = 1 + i/128 nearest to m,
 *     r = m * RN(1/c_i) - 1           (exact, as r_hi + r_lo, |r| <= 2^-8)
 *     ln x = k ln2 + (-ln RN(1/c_i)) + ln(1 + r)
 *
 * with ln2 and the table in double-double (scripts/gen_logtab.py, Python
 * decimal at 60 digits), the leading terms summed with error-free
 * transformations and the series tail r^3(1/3 - r/4 + ... - r^7/10) in
 * double.  Relative error before the final rounding is below 2^-75, so the
 * result equals RN(ln x) except when ln x lies within 2^-75 of a rounding
 * midpoint (tests/test_logcr.py checks it against mpmath).
 *
 * Every operation is an explicit IEEE op or fma(), so the same source gives
 * the same bits on the host (oracle, gcc -ffp-contract=off) and on sm_100a
 * (nvcc --fmad=false or true: fma() calls are explicit, no other products
 * are contracted because every product feeds an explicit error-free step).
 */
#pragma once

#ifdef __CUDACC__
#define FDG_HD __host__ __device__ __forceinline__
#define FDG_LOGTAB_QUAL static __device__ const
#include <cstdint>
#else
#define FDG_HD static inline
#define FDG_LOGTAB_QUAL static const
#include <math.h>
#include <stdint.h>
#include <string.h>
#endif

#include "fdg_logtab.h"

#ifdef __CUDACC__
__device__ __forceinline__ uint64_t fdg_bits(double x) { return (uint64_t)__double_as_longlong(x); }
__device__ __forceinline__ double fdg_from_bits(uint64_t b) { return __longlong_as_double((long long)b); }
#else
static inline uint64_t fdg_bits(double x) { uint64_t b; memcpy(&b, &x, 8); return b; }
static inline double fdg_from_bits(uint64_t b) { double x; memcpy(&x, &b, 8); return x; }
#endif

#ifdef __CUDACC__
__device__ __forceinline__
#else
static inline
#endif
double log_cr(double x)
{
    if (!(x > 0.0)) {
        if (x == 0.0) return fdg_from_bits(0xfff0000000000000ULL); /* -inf */
        if (x != x) return x + x;                                 /* nan */
        return fdg_from_bits(0x7ff8000000000000ULL);              /* negative: nan */
    }
    uint64_t bits = fdg_bits(x);
    int ex = (int)(bits >> 52);
    if (ex == 0x7ff) return x; /* +inf */
    int k;
    if (ex == 0) { /* subnormal: scale into the normal range */
        x = x * 0x1p54;
        bits = fdg_bits(x);
        ex = (int)(bits >> 52);
        k = ex - 1023 - 54;
    } else {
        k = ex - 1023;
    }
    double m = fdg_from_bits((bits & 0x000fffffffffffffULL) | 0x3ff0000000000000ULL);
    int i = ((int)((bits >> 44) & 0xff) + 1) >> 1; /* round((m-1)*128) */
    if (i == 128) {
        k += 1;
        m = m * 0.5;
        i = 0;
    }
#ifdef __CUDACC__
    const double inv_c = __ldg(&fdg_logtab[i][0]);
    const double t_hi = __ldg(&fdg_logtab[i][1]);
    const double t_lo = __ldg(&fdg_logtab[i][2]);
#else
    const double inv_c = fdg_logtab[i][0];
    const double t_hi = fdg_logtab[i][1];
    const double t_lo = fdg_logtab[i][2];
#endif
    /* r = m * inv_c - 1, exactly, as r_hi + r_lo */
    double p_hi = m * inv_c;
    double p_lo = fma(m, inv_c, -p_hi);
    double a = p_hi - 1.0; /* exact (Sterbenz) */
    double r_hi = a + p_lo;
    double bv = r_hi - a;
    double r_lo = (a - (r_hi - bv)) + (p_lo - bv);
    /* r^2 exactly */
    double s_hi = r_hi * r_hi;
    double s_lo = fma(r_hi, r_hi, -s_hi);
    /* tail r^3 (1/3 - r/4 + r^2/5 - ... - r^7/10) */
    double q = -0.1;
    q = fma(q, r_hi, 1.0 / 9.0);
    q = fma(q, r_hi, -0.125);
    q = fma(q, r_hi, 1.0 / 7.0);
    q = fma(q, r_hi, -1.0 / 6.0);
    q = fma(q, r_hi, 0.2);
    q = fma(q, r_hi, -0.25);
    q = fma(q, r_hi, 1.0 / 3.0);
    double tail = (s_hi * r_hi) * q;
    /* leading terms: k ln2_hi (exact) + t_hi + r_hi - s_hi/2 (exact halving),
     * accumulated with two-sums */
    double kd = (double)k;
    double A = kd * FDG_LN2_HI;
    double s1 = A + t_hi;
    double z1 = s1 - A;
    double e1 = (A - (s1 - z1)) + (t_hi - z1);
    double s2 = s1 + r_hi;
    double z2 = s2 - s1;
    double e2 = (s1 - (s2 - z2)) + (r_hi - z2);
    double E = -0.5 * s_hi;
    double s3 = s2 + E;
    double z3 = s3 - s2;
    double e3 = (s2 - (s3 - z3)) + (E - z3);
    /* small terms: first-order r_lo effects and the table / ln2 low parts */
    double lo = r_lo - 0.5 * s_lo;
    lo = lo - r_hi * r_lo;
    lo = lo + r_lo * s_hi;
    lo = lo + tail;
    lo = lo + (t_lo + kd * FDG_LN2_LO);
    lo = lo + ((e1 + e2) + e3);
    return s3 + lo;
}
