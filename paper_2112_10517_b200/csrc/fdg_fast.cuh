// fdg_fast.cuh -- FAST-mode (RhsConfig.kernel == "batched") two-point fluxes.
//
// Same fluxes as the FAITHFUL ones in fdg_device.cuh, rearranged for the FP64
// pipe of sm_100a:
//   * nodes are staged with HALF velocities and HALF pressure (vh = v/2,
//     ph = p/2; exact power-of-two scalings), so every arithmetic mean
//     {a} = (a_l + a_r)/2 is a single add and the 1/2 factors of the fluxes
//     fold away;
//   * the log-mean branch test u < 1e-4 (means.py: u = ((b-a)/(b+a))^2) is
//     the equivalent |log b - log a| < 2 atanh(0.01) on the log difference
//     the log branch needs anyway (one compare, no division);
//   * the series branch is (a+b)/(2 x coth x), x = (log b - log a)/2, a
//     polynomial in (log b - log a)^2 (series_frac): no reciprocal, and
//     both branches are evaluated and selected (branch fractions mix inside
//     every warp; a warp-uniform series branch,
//     FDG_SERIES_VOTE=1, measured slower: it stops ptxas from interleaving
//     consecutive pairs, profiles/r01_tuning.md);
//   * <x>_log = num/den with (num, den) = (a+b, 2x coth x) or (b-a, dl); the
//     two log means of a Ranocha pair share ONE reciprocal 1/(den_rho num_rhop)
//     (MUFU.RCP64H + two Newton steps, branch free);
//   * Ranocha nodes carry log rho and X = log(rho/p): the (rho p) log mean of
//     (rho_l p_r, rho_r p_l) needs log B - log A = X_r - X_l (one add), and X
//     reuses the staging reciprocal of rho.
// Results agree with the reference to a few ulps of each flux (VOL-level
// relative differences ~1e-15, tests/test_gpu_parity.py).
#pragma once

#include "fdg_logtab_fast.h"

namespace fdg {

// Literal FP64 constants of the FAST path live in the constant bank, where
// DFMA/DMUL take them as c[3][...] operands; a literal double in the
// instruction stream costs two UMOVs per use (5.9% of the cfg2 kernel's
// instructions before this table).
enum FastConst {
    KC_LOG1, KC_LOG2, KC_LOG3, KC_LOG4, KC_LOG5, KC_LOG6, KC_LOG7,  // log_fast T(z) coefficients
    KC_LN2_HI, KC_LN2_LO,
    KC_CT1, KC_CT2, KC_CT3,  // 2 x coth x = 2 + z/6 - z^2/360 + z^3/15120, z = (2x)^2
    KC_SERIES_DL,            // u < 1e-4  <=>  |t| < 0.01  <=>  |log(b/a)| < 2 atanh(0.01)
    KC_COUNT
};
static __constant__ double kFast[KC_COUNT] = {
    0.6666666666666734, 0.39999999999417485, 0.2857142874173421, 0.22222198640440488,
    0.1818356087762256, 0.15314136991810745, 0.14795104806627174,
    0.6931471805599453, 2.3190468138462996e-17,
    1.0 / 6.0, -1.0 / 360.0, 1.0 / 15120.0,
    0.02000066670666952,
};

// FAST natural log, ~1.2 ulp (libdevice's log costs ~86 instructions per
// call here, 20% of the cfg2 kernel before this one; this is ~28).
// x = 2^e m, m in [sqrt(1/2), sqrt(2)); log m = f - s (f - T(z)), f = m - 1
// (exact), s = f / (2 + f), z = s^2, T(z) = 2 (atanh(s)/s - 1) fitted to
// degree 7 (scripts/gen_logfast.py: coefficients and the error check).
// Branch free (a call or branch for special inputs would keep ptxas from
// interleaving the logs of consecutive nodes): subnormals are rescaled by
// 2^54, and zero / negative / inf / NaN arguments select -inf / NaN / inf /
// NaN at the end.
__device__ __forceinline__ double log_fast(double x)
{
    const long long bits = __double_as_longlong(x);
    const bool sub = bits < 0x0010000000000000LL;  // subnormal, zero or negative
    const double xs = sub ? x * 0x1p54 : x;
    const int hi = __double2hiint(xs);
    const int lo = __double2loint(xs);
    const int e = (hi - 0x3fe6a09e) >> 20;  // 0x3fe6a09e: high word of sqrt(1/2)
    const double m = __hiloint2double(hi - (e << 20), lo);
    const double f = m - 1.0;
    const double s = f * rcp_fast(2.0 + f);
    const double z = s * s;
    const double z2 = z * z;
    // Estrin: shorter dependency chain than Horner (DFMA latency 8.3 cycles)
    const double p01 = fma(kFast[KC_LOG2], z, kFast[KC_LOG1]);
    const double p23 = fma(kFast[KC_LOG4], z, kFast[KC_LOG3]);
    const double p45 = fma(kFast[KC_LOG6], z, kFast[KC_LOG5]);
    const double p47 = fma(kFast[KC_LOG7], z2, p45);
    const double p03 = fma(p23, z2, p01);
    const double p = fma(p47, z2 * z2, p03);
    const double corr = s * fma(-z, p, f);  // s (f - T)
    const double ed = (double)(sub ? e - 54 : e);
    const double r = fma(ed, kFast[KC_LN2_HI], f) + fma(ed, kFast[KC_LN2_LO], -corr);
    const bool ok = bits > 0 && bits < 0x7ff0000000000000LL;  // positive, finite
    const double special = (bits == 0 || bits == (long long)0x8000000000000000ULL) ? -INFINITY
                           : (bits < 0) ? NAN : x;  // -0, +0 | negative | +inf, NaN
    return ok ? r : special;
}

// The same log for arguments known to be positive, normal and finite: no
// subnormal rescale, no special-value selects (17 fewer instructions per
// call). Bitwise equal to log_fast there. log_normal_ok(x) is the test.
// NEG: returns -log x with the sign folded into operand negations of the last
// two FMAs (exactly the negated value, no extra instruction)
template <bool NEG = false>
__device__ __forceinline__ double log_fast_normal(double x)
{
    const int hi = __double2hiint(x);
    const int lo = __double2loint(x);
    const int e = (hi - 0x3fe6a09e) >> 20;
    const double m = __hiloint2double(hi - (e << 20), lo);
    const double f = m - 1.0;
    const double s = f * rcp_fast(2.0 + f);
    const double z = s * s;
    const double z2 = z * z;
    const double p01 = fma(kFast[KC_LOG2], z, kFast[KC_LOG1]);
    const double p23 = fma(kFast[KC_LOG4], z, kFast[KC_LOG3]);
    const double p45 = fma(kFast[KC_LOG6], z, kFast[KC_LOG5]);
    const double p47 = fma(kFast[KC_LOG7], z2, p45);
    const double p03 = fma(p23, z2, p01);
    const double p = fma(p47, z2 * z2, p03);
    const double corr = s * fma(-z, p, f);
    const double ed = (double)e;
    if constexpr (NEG) return fma(-ed, kFast[KC_LN2_HI], -f) + fma(-ed, kFast[KC_LN2_LO], corr);
    else return fma(ed, kFast[KC_LN2_HI], f) + fma(ed, kFast[KC_LN2_LO], -corr);
}
// Table log for positive, normal, finite arguments (the per-node log tables
// of the staging pass): x = 2^E m, i = top 7 mantissa bits, r_i = RN(128 /
// (128 + i)), f = fma(m, r_i, -1) in [0, 2^-7), log x = k ln2 + T_i +
// log1p(f) with T_i = -ln(r_i) - [i >= 53] ln2 and k = E + [i >= 53] (exact
// identity for the stored r_i; scripts/gen_logtab_fast.py writes the table
// and checks <= 1.5 ulp of max(|log x|, 2^-7) against 60-digit logs).
// log1p(f) = f + f^2 P(f), Taylor to f^7 (truncation < 1.8e-18). 12 FP64
// instructions and one 16-byte L1-resident load instead of 21 + a MUFU
// reciprocal for log_fast_normal.
#ifndef FDG_LOG_TAB
#define FDG_LOG_TAB 1
#endif
template <bool NEG = false>
__device__ __forceinline__ double log_tab(double x)
{
    const int hi = __double2hiint(x);
    const int lo = __double2loint(x);
    const int i = (hi >> 13) & 127;
    const int k = ((hi + (75 << 13)) >> 20) - 1023;
    const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);
    const double2 rt = __ldg(&fdg_logtab_fast[i]);
    const double f = fma(m, rt.x, -1.0);
    const double f2 = f * f;
    const double p01 = fma(1.0 / 3.0, f, -0.5);
    const double p23 = fma(0.2, f, -0.25);
    const double p45 = fma(1.0 / 7.0, f, -1.0 / 6.0);
    const double p = fma(fma(p45, f2, p23), f2, p01);
    const double l1p = fma(f2, p, f);
    const double kd = (double)k;
    if constexpr (NEG) return fma(-kd, kFast[KC_LN2_HI], -rt.y) + fma(-kd, kFast[KC_LN2_LO], -l1p);
    else return fma(kd, kFast[KC_LN2_HI], rt.y) + fma(kd, kFast[KC_LN2_LO], l1p);
}
// TAB: the volume-only twin takes the table log (cfg5 VOL 3.37 -> 3.31 ms);
// in the RHS / stage twins its loads compete with the interface traces for
// L1 and it measured 2% slower (5.37 vs 5.26 ms), so they keep the polynomial
template <int TAB, bool NEG = false>
__device__ __forceinline__ double log_node(double x)
{
    if constexpr (FDG_LOG_TAB && TAB) return log_tab<NEG>(x);
    else return log_fast_normal<NEG>(x);
}

// x positive, normal, finite: one unsigned compare on the high word
__device__ __forceinline__ bool log_normal_ok(double x)
{
    return (unsigned)(__double2hiint(x) - 0x00100000) < 0x7fe00000u;
}

#ifndef FDG_SERIES_VOTE
#define FDG_SERIES_VOTE 0  // 1: warp-uniform series branch (see the header)
#endif

// log-mean branch test on the log difference dl = log b - log a (means.py:
// u < 1e-4); dl is exact up to the rounding of the two logs
__device__ __forceinline__ bool series_test(double dl) { return fabs(dl) < kFast[KC_SERIES_DL]; }

// FDG_LM_LEAN (r02 session 5): the same two candidates with fewer
// instructions per log mean --
//   * the branch test on the high word of z = dl^2 (z >= 0: one integer
//     compare, no FP64-pipe DSETP; the threshold moves by < 2^-20 relative,
//     and both candidates are accurate around it);
//   * num = fma(sgn, a, b) with sgn = +-1 selected in the high word only
//     (b + a on series lanes, b - a otherwise, the same bits as the two
//     separate sums): one select + one DFMA instead of a negation, an add
//     and a two-word select;
//   * FDG_CT_TERMS = 2 drops the z^3/15120 term of 2 x coth x: below the
//     threshold z < 4.0003e-4 it is < 4.3e-15 of the mean (the log candidate
//     just above the threshold carries ~1e-14 from the rounding of dl).
#ifndef FDG_LM_LEAN
#define FDG_LM_LEAN 1
#endif
#ifndef FDG_CT_TERMS
#define FDG_CT_TERMS 2
#endif
// high word of KC_SERIES_DL^2 = 4.000266687e-4 (0x3F3A375575AB25FF): z below it <=> series
constexpr int kSeriesZHi = 0x3F3A3755;

// <a,b>_log = num / den: the log branch (num, den) = (b - a, dl) is the
// caller's; on series lanes it becomes (a + b, 2 x coth x), x = dl/2.
// With t = (b-a)/(b+a) = tanh(x), <a,b>_log = (b-a)/dl = (a+b) tanh(x)/(2x)
// exactly; means.py's series (a+b)/(2 + u (2/3 + ...)), u = t^2, is the same
// function of t.  2 x coth x = 2 + z/6 - z^2/360 + z^3/15120 - ..., z = dl^2:
// dl enters only through the O(z) corrections, so its rounding (which is why
// (b-a)/dl fails for b ~ a) costs nothing, and no reciprocal is needed
// (truncation < 1e-19 relative for |dl| < 0.02 with three terms).
__device__ __forceinline__ double coth_series(double z)
{
#if FDG_CT_TERMS >= 3
    return fma(z, fma(z, fma(z, kFast[KC_CT3], kFast[KC_CT2]), kFast[KC_CT1]), 2.0);
#else
    return fma(z, fma(z, kFast[KC_CT2], kFast[KC_CT1]), 2.0);
#endif
}
__device__ __forceinline__ void series_frac(double a, double b, double dl, bool series, double& num, double& den)
{
    const double z = dl * dl;
    const double cth = coth_series(z);
    num = series ? b + a : num;
    den = series ? cth : den;
}
// lean form: (num, den) of one log mean from scratch
__device__ __forceinline__ void logmean_frac(double a, double b, double dl, double& num, double& den)
{
    const double z = dl * dl;
    const bool series = __double2hiint(z) < kSeriesZHi;
    const double cth = coth_series(z);
    const double sgn = __hiloint2double(series ? 0x3ff00000 : (int)0xbff00000, 0);
    num = fma(sgn, a, b);
    den = series ? cth : dl;
}

// both log means of a pair; the series work only when a lane of the warp needs it
__device__ __forceinline__ void logmean_pair(double a1, double b1, double dl1, double& num1, double& den1, double a2,
                                             double b2, double dl2, double& num2, double& den2, unsigned vm)
{
#if FDG_LM_LEAN
    logmean_frac(a1, b1, dl1, num1, den1);
    logmean_frac(a2, b2, dl2, num2, den2);
#else
    num1 = b1 - a1;
    den1 = dl1;
    num2 = b2 - a2;
    den2 = dl2;
    const bool s1 = series_test(dl1);
    const bool s2 = series_test(dl2);
#if FDG_SERIES_VOTE
    if (__any_sync(vm, s1 || s2))
#endif
    {
        series_frac(a1, b1, dl1, s1, num1, den1);
        series_frac(a2, b2, dl2, s2, num2, den2);
    }
#endif
}

// half-value dot products with the face/metric direction
template <int D, int AXIS>
__device__ __forceinline__ double hdot(const double (&vh)[D], const double* nrm)
{
    if constexpr (AXIS >= 0) {
        return vh[AXIS];
    } else {
        double r = vh[0] * nrm[0];
#pragma unroll
        for (int i = 1; i < D; ++i) r = fma(vh[i], nrm[i], r);
        return r;
    }
}

// f_m_i = f_rho v_avg_i + p_avg n_i with v_avg = vh_l + vh_r, p_avg = ph_l + ph_r
template <int D, int AXIS>
__device__ __forceinline__ void fast_momentum(double f_rho, double p_avg, const double (&vhl)[D],
                                              const double (&vhr)[D], const double* nrm, double* f)
{
#pragma unroll
    for (int i = 0; i < D; ++i) {
        const double t = f_rho * (vhl[i] + vhr[i]);
        if constexpr (AXIS >= 0) f[1 + i] = (i == AXIS) ? t + p_avg : t;
        else f[1 + i] = fma(p_avg, nrm[i], t);
    }
}

// EH = 1: f[D+1] comes back as f_E / 2 (the volume passes multiply it with
// the doubled weight table wtsE: scaling by 2 is exact, so the accumulated
// bits are the same and two multiplies per pair are gone)
#if FDG_RANOCHA_B
// x = (log rho, log b, b) with log tables, (b) without; b = rho / p.
// f_rho = <rho>_log {v.n};  f_E = f_rho (v_l.v_r / 2 + igm1 / <b>_log) + (p_l vn_r + p_r vn_l) / 2
// since p_l p_r / <rho_l p_r, rho_r p_l>_log = 1 / <b_l, b_r>_log.
template <int D, int AXIS, int LOGS, int EH = 0, int NX>
__device__ __forceinline__ void fast_ranocha(const Node<D, NX>& l, const Node<D, NX>& r, const double* nrm,
                                             double igm1, double* f, unsigned vm)
{
    const double bl = l.x[LOGS ? 2 : 0], br = r.x[LOGS ? 2 : 0];
    double dl1, dl2;
    if constexpr (LOGS) {
        dl1 = r.x[0] - l.x[0];  // log rho_r - log rho_l
        dl2 = r.x[1] - l.x[1];  // log b_r - log b_l
    } else {
        dl1 = log_fast(r.rho * rcp_fast(l.rho));
        dl2 = log_fast(br * rcp_fast(bl));
    }
    double num1, den1, num2, den2;  // <rho>_log = num1/den1, <b>_log = num2/den2
    logmean_pair(l.rho, r.rho, dl1, num1, den1, bl, br, dl2, num2, den2, vm);
    // everything that does not need the shared reciprocal is formed while
    // MUFU + its correction run
    const double vn_l = hdot<D, AXIS>(l.v, nrm);
    const double vn_r = hdot<D, AXIS>(r.v, nrm);
    const double pre_rho = num1 * num2 * (vn_l + vn_r);                 // f_rho / rr
    const double pre_e = ((EH ? 0.5 : 1.0) * igm1) * (den1 * den2);     // (igm1 / <b>_log) / rr (EH: half of it)
    double vv = l.v[0] * r.v[0];
#pragma unroll
    for (int i = 1; i < D; ++i) vv = fma(l.v[i], r.v[i], vv);
    const double pv = fma(l.p, vn_r, r.p * vn_l);
    const double rr = rcp_fast(den1 * num2);
    const double f_rho = pre_rho * rr;
    f[0] = f_rho;
    // half values: vv = v_l.v_r / 4, pv = (p_l vn_r + p_r vn_l) / 4
    if constexpr (EH) f[D + 1] = fma(f_rho, fma(pre_e, rr, vv), pv);
    else f[D + 1] = fma(f_rho, fma(pre_e, rr, 2.0 * vv), 2.0 * pv);
    fast_momentum<D, AXIS>(f_rho, l.p + r.p, l.v, r.v, nrm, f);
}
#else
template <int D, int AXIS, int LOGS, int EH = 0, int NX>
__device__ __forceinline__ void fast_ranocha(const Node<D, NX>& l, const Node<D, NX>& r, const double* nrm,
                                             double igm1, double* f, unsigned vm)
{
    // rho-mean and the (rho p)-mean; A = rho_l p_r / 2, B = rho_r p_l / 2
    const double A = l.rho * r.p;
    const double B = r.rho * l.p;
    double dl1, dl2;
    if constexpr (LOGS) {
        dl1 = r.x[0] - l.x[0];  // log rho_r - log rho_l
        dl2 = r.x[1] - l.x[1];  // log B - log A = X_r - X_l, X = log(rho/p)
    } else {
        dl1 = log_fast(r.rho * rcp_fast(l.rho));
        dl2 = log_fast(B * rcp_fast(A));
    }
    double num1, den1, num2, den2;  // <rho>_log = num1/den1, <rho p>_log = 2 num2/den2
    logmean_pair(l.rho, r.rho, dl1, num1, den1, A, B, dl2, num2, den2, vm);
    // everything that does not need the shared reciprocal is formed while
    // MUFU + its correction run; after it: one multiply (f_rho) and one FMA
    // (the energy factor) ahead of the flux assembly
    const double vn_l = hdot<D, AXIS>(l.v, nrm);
    const double vn_r = hdot<D, AXIS>(r.v, nrm);
    const double pre_rho = num1 * num2 * (vn_l + vn_r);              // f_rho / rr
    const double pre_e = ((EH ? 1.0 : 2.0) * igm1) * (l.p * r.p) * (den1 * den2);  // e_int / rr (EH: half of it)
    double vv = l.v[0] * r.v[0];
#pragma unroll
    for (int i = 1; i < D; ++i) vv = fma(l.v[i], r.v[i], vv);
    const double pv = fma(l.p, vn_r, r.p * vn_l);
    const double rr = rcp_fast(den1 * num2);
    // <rho>_log {v.n}; igm1 p_l p_r / <rho p>_log = igm1 (4 ph_l ph_r) den2 / (2 num2)
    const double f_rho = pre_rho * rr;
    // f_E = f_rho (v_l.v_r / 2 + igm1 p_l p_r/<rho p>) + (p_l vn_r + p_r vn_l)/2
    f[0] = f_rho;
    if constexpr (EH) f[D + 1] = fma(f_rho, fma(pre_e, rr, vv), pv);
    else f[D + 1] = fma(f_rho, fma(pre_e, rr, 2.0 * vv), 2.0 * pv);
    fast_momentum<D, AXIS>(f_rho, l.p + r.p, l.v, r.v, nrm, f);
}

#endif

template <int D, int AXIS, int NX>
__device__ __forceinline__ void fast_shima(const Node<D, NX>& l, const Node<D, NX>& r, const double* nrm,
                                           double igm1, double* f)
{
    const double vn_l = hdot<D, AXIS>(l.v, nrm);
    const double vn_r = hdot<D, AXIS>(r.v, nrm);
    const double vn_avg = vn_l + vn_r;
    const double p_avg = l.p + r.p;
    const double f_rho = 0.5 * (l.rho + r.rho) * vn_avg;
    double vv = l.v[0] * r.v[0];
#pragma unroll
    for (int i = 1; i < D; ++i) vv = fma(l.v[i], r.v[i], vv);
    // f_E = f_rho v_l.v_r / 2 + p_avg vn_avg / (gamma-1) + (p_l vn_r + p_r vn_l)/2
    const double pv = fma(l.p, vn_r, r.p * vn_l);
    f[0] = f_rho;
    f[D + 1] = fma(2.0 * f_rho, vv, fma(p_avg * vn_avg, igm1, 2.0 * pv));
    fast_momentum<D, AXIS>(f_rho, p_avg, l.v, r.v, nrm, f);
}

// Kennedy-Gruber; x[0] holds e/2 (half specific total energy)
template <int D, int AXIS, int NX>
__device__ __forceinline__ void fast_kg(const Node<D, NX>& l, const Node<D, NX>& r, const double* nrm, double* f)
{
    const double vn_avg = hdot<D, AXIS>(l.v, nrm) + hdot<D, AXIS>(r.v, nrm);
    const double p_avg = l.p + r.p;
    const double f_rho = 0.5 * (l.rho + r.rho) * vn_avg;
    f[0] = f_rho;
    fast_momentum<D, AXIS>(f_rho, p_avg, l.v, r.v, nrm, f);
    f[D + 1] = fma(f_rho, l.x[0] + r.x[0], p_avg * vn_avg);
}

// Chandrashekar; x[0] = beta = rho/(2p), x[1] = log rho, x[2] = log beta (LOGS)
// KP: the node's pressure slot holds |v/2|^2 instead (volume-only launches:
// this flux never reads p, and {|v|^2}/2 becomes one add instead of 2 d FMAs)
template <int D, int AXIS, int LOGS, int KP = 0, int NX>
__device__ __forceinline__ void fast_chandrashekar(const Node<D, NX>& l, const Node<D, NX>& r, const double* nrm,
                                                   double igm1, double* f, unsigned vm)
{
    double dl1, dl2;
    if constexpr (LOGS) {
        dl1 = r.x[1] - l.x[1];
        dl2 = r.x[2] - l.x[2];
    } else {
        dl1 = log_fast(r.rho * rcp_fast(l.rho));
        dl2 = log_fast(r.x[0] * rcp_fast(l.x[0]));
    }
    double num1, den1, num2, den2;  // <rho>_log = num1/den1, <beta>_log = num2/den2
    logmean_pair(l.rho, r.rho, dl1, num1, den1, l.x[0], r.x[0], dl2, num2, den2, vm);
    const double bsum = l.x[0] + r.x[0];               // 2 {beta}
    const double rr = rcp_fast(den1 * num2 * bsum);
    const double rho_mean = num1 * num2 * bsum * rr;
    const double inv_beta_mean = den2 * den1 * bsum * rr;
    const double p_tilde = 0.5 * (l.rho + r.rho) * (den1 * num2) * rr;  // {rho} / (2 {beta})
    const double vn_avg = hdot<D, AXIS>(l.v, nrm) + hdot<D, AXIS>(r.v, nrm);
    const double f_rho = rho_mean * vn_avg;
    double v2 = 0.0;  // {|v|^2}/2 = |vh_l|^2 + |vh_r|^2
    if constexpr (KP) {
        v2 = l.p + r.p;
    } else {
#pragma unroll
        for (int i = 0; i < D; ++i) v2 = fma(l.v[i], l.v[i], fma(r.v[i], r.v[i], v2));
    }
    f[0] = f_rho;
    double work = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        const double va = l.v[i] + r.v[i];
        const double t = f_rho * va;
        if constexpr (AXIS >= 0) f[1 + i] = (i == AXIS) ? t + p_tilde : t;
        else f[1 + i] = fma(p_tilde, nrm[i], t);
        work = fma(va, f[1 + i], work);
    }
    f[D + 1] = fma(f_rho, fma(0.5 * igm1, inv_beta_mean, -v2), work);
}

// central (0.5 (f(u_l) + f(u_r)).n) from the staged conserved state x[0..D+1]
template <int D, int AXIS, int NX>
__device__ __forceinline__ void fast_central(const Node<D, NX>& l, const Node<D, NX>& r, const double* nrm,
                                             double* f)
{
    const double vn_l = hdot<D, AXIS>(l.v, nrm);  // half normal velocities
    const double vn_r = hdot<D, AXIS>(r.v, nrm);
    f[0] = l.x[0] * vn_l + r.x[0] * vn_r;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        const double t = fma(l.x[1 + i], vn_l, r.x[1 + i] * vn_r);
        const double pn = l.p + r.p;  // half-pressure sum = {p}
        if constexpr (AXIS >= 0) f[1 + i] = (i == AXIS) ? t + pn : t;
        else f[1 + i] = fma(pn, nrm[i], t);
    }
    f[D + 1] = fma(l.x[D + 1] + 2.0 * l.p, vn_l, (r.x[D + 1] + 2.0 * r.p) * vn_r);
}

// FAST staging: rho, v/2, p/2 and the extras
template <int D, int VF, int LOGS, int TAB = 0>
__device__ __forceinline__ Node<D, n_extra(VF, LOGS)> make_node_fast(const double* u, double gm1)
{
    constexpr int NX = n_extra(VF, LOGS);
    Node<D, NX> q;
    const double rho = u[0];
    const double hri = 0.5 * rcp_fast(rho);
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        q.v[i] = u[1 + i] * hri;  // v/2
        s = fma(q.v[i], q.v[i], s);
    }
    q.rho = rho;
    // p/2 = (gamma-1)/2 (E - rho |v|^2 / 2) = (gamma-1)/2 (E - 2 rho |v/2|^2)
    q.p = (0.5 * gm1) * fma(-2.0 * rho, s, u[D + 1]);
    // per-node log tables: the lean log on the (always taken, admissible
    // states) positive-normal path, the full log_fast behind one rarely
    // taken branch for everything else (zero, negative, subnormal, inf, NaN:
    // states the gate reports, or absurdly scaled ones)
#if FDG_RANOCHA_B
    if constexpr (VF == F_RANOCHA) {
        const double b = (0.5 * rho) * rcp_fast(q.p);  // rho / p
        q.x[LOGS ? 2 : 0] = b;
        if constexpr (LOGS) {
            q.x[0] = log_node<TAB>(rho);
            q.x[1] = log_node<TAB>(b);
            if (!(log_normal_ok(rho) && log_normal_ok(b))) {
                q.x[0] = log_fast(rho);
                q.x[1] = log_fast(b);
            }
        }
    } else if constexpr (VF == F_CHANDRASHEKAR) {
#else
    if constexpr (VF == F_RANOCHA && LOGS) {
        const double a = 4.0 * q.p * hri;  // X = log(rho / p) = -log(2 ph / rho), 2 hri = 1/rho
        q.x[0] = log_node<TAB>(rho);
        q.x[1] = FDG_STAGE_LEAN ? log_node<TAB, true>(a) : -log_node<TAB>(a);
        if (!(log_normal_ok(rho) && log_normal_ok(a))) {
            q.x[0] = log_fast(rho);
            q.x[1] = -log_fast(a);
        }
    } else if constexpr (VF == F_CHANDRASHEKAR) {
#endif
        q.x[0] = 0.25 * rho * rcp_fast(q.p);  // beta = rho / (2 p)
        if constexpr (LOGS) {
            q.x[1] = log_node<TAB>(rho);
            q.x[2] = log_node<TAB>(q.x[0]);
            if (!(log_normal_ok(rho) && log_normal_ok(q.x[0]))) {
                q.x[1] = log_fast(rho);
                q.x[2] = log_fast(q.x[0]);
            }
        }
    } else if constexpr (VF == F_KG) {
        q.x[0] = u[D + 1] * hri;  // e/2
    } else if constexpr (VF == F_CENTRAL) {
#pragma unroll
        for (int i = 0; i < 5; ++i) q.x[i] = (i < D + 2) ? u[i] : 0.0;
    }
    return q;
}

// vm: lanes of the warp executing this call together (the series-branch vote)
// volume kinds whose FAST energy flux can come back halved (EH = 1)
__host__ __device__ constexpr bool energy_half(int vf) { return vf == F_RANOCHA; }

template <int D, int VF, int AXIS, int LOGS, int EH = 0, int KP = 0, int NX>
__device__ __forceinline__ void fast_volume_flux(const Node<D, NX>& l, const Node<D, NX>& r, const double* nrm,
                                                 double igm1, double* f, unsigned vm)
{
    if constexpr (VF == F_SHIMA) fast_shima<D, AXIS>(l, r, nrm, igm1, f);
    else if constexpr (VF == F_RANOCHA) fast_ranocha<D, AXIS, LOGS, EH>(l, r, nrm, igm1, f, vm);
    else if constexpr (VF == F_CENTRAL) fast_central<D, AXIS>(l, r, nrm, f);
    else if constexpr (VF == F_KG) fast_kg<D, AXIS>(l, r, nrm, f);
    else fast_chandrashekar<D, AXIS, LOGS, KP>(l, r, nrm, igm1, f, vm);
}

}  // namespace fdg
