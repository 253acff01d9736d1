// fdg_device.cuh -- per-node and per-pair FP64 arithmetic of the
// flux-differencing volume integral, sm_100a.
//
// Two arithmetic policies share every kernel template:
//
//   FAITHFUL  (RhsConfig.kernel == "reference")  reproduces the reference's
//             scalar path operation by operation: the TU that instantiates it
//             is compiled with --fmad=false, every expression keeps the
//             association of the Python source (fluxes.py:132-415), division
//             and sqrt are IEEE round-to-nearest, and the per-node
//             accumulation order is the scalar loop's (ascending partner per
//             line, directions in order, discretization.py:288-323).
//   FAST      (RhsConfig.kernel == "batched")  the throughput path: FMA
//             contraction, one reciprocal per two-point flux (both log means
//             share it), approximate reciprocals where the result only feeds a
//             series correction of size <= 1e-4.
//
// Reference formulas (all in /root/reference/pkg/src/fluxdg):
//   log means          fluxes.py:132-157, means.py:68-118 (Algorithms 2-3 of the paper)
//   cons2prim          fluxes.py:107-121, euler.py:47-60
//   shima              fluxes.py:163-218, 516-547
//   ranocha            fluxes.py:224-287, 550-589
//   central            fluxes.py:293-325, 592-616
//   llf / hll          fluxes.py:335-415
//   kennedy-gruber, chandrashekar: not in the reference,
//   restated in the same core style; parity unpinned.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "fdg_logcr.h"

namespace fdg {

enum FluxKind : int {
    F_CENTRAL = 0,
    F_SHIMA = 1,
    F_RANOCHA = 2,
    F_KG = 3,
    F_CHANDRASHEKAR = 4,
    F_LLF = 5,
    F_HLL = 6,
};
enum Mode : int { FAITHFUL = 0, FAST = 1 };
enum Pre : int { PRE_NONE = 0, PRE_PRIMITIVES = 1, PRE_LOGS = 2 };

constexpr double SERIES_EPSILON = 1.0e-4;  // means.py:16

__host__ __device__ constexpr int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }

// FAST Ranocha nodes also carry b = rho / p: the (rho p) log mean becomes the
// log mean of (b_l, b_r) -- <rho_l p_r, rho_r p_l>_log = p_l p_r <b_l, b_r>_log
// by homogeneity -- so a pair forms neither rho_l p_r, rho_r p_l nor p_l p_r
// (4 of 49 FP64 instructions per pair) for one more staged value per node.
// The FAITHFUL kernels keep the reference's arguments and leave the slot unused.
#ifndef FDG_RANOCHA_B
#define FDG_RANOCHA_B 1
#endif
// number of extra per-node values a volume flux stages next to (rho, v, p)
__host__ __device__ constexpr int n_extra(int vf, int logs)
{
    return vf == F_RANOCHA ? (logs ? 2 : 0) + FDG_RANOCHA_B  // FAST: + b = rho / p (fdg_fast.cuh)
         : vf == F_CHANDRASHEKAR ? (logs ? 3 : 1)
         : vf == F_KG ? 1
         : vf == F_CENTRAL ? 5  // conserved state (rho, m1..m3 | E), padded to 5
         : 0;
}

// ------------------------------------------------------------------ helpers

__device__ __forceinline__ double rcp_approx(double x)
{
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    return r;
}

// ~1 ulp reciprocal without the IEEE-division slow path (FAST mode only):
// MUFU.RCP64H (~2^-22 relative) and one cubically convergent correction,
// r (1 + e + e^2), e = 1 - x r (error e^3 ~ 2^-66): three dependent FMAs
// instead of the four of two Newton steps
__device__ __forceinline__ double rcp_fast(double x)
{
    const double r = rcp_approx(x);
    const double e = fma(-x, r, 1.0);
    return fma(r, fma(e, e, e), r);
}

// ~1 ulp 1/sqrt(x), x > 0 normal, branch free (FAST mode only): MUFU.RSQ64H
// and one cubically convergent correction r (1 + e/2 + 3e^2/8), e = 1 - x r^2
__device__ __forceinline__ double rsqrt_fast(double x)
{
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double e = fma(-x * r, r, 1.0);
    return fma(r, e * fma(0.375, e, 0.5), r);
}

template <int MODE>
__device__ __forceinline__ double dlog(double x)
{
    if constexpr (MODE == FAITHFUL) return log_cr(x);  // glibc-equivalent correctly rounded log
    else return log(x);
}

// Python >= 3.12 builtin sum() of floats (start 0): Neumaier compensated.
// Used once by the reference hot path: fluxes.py:603-605.
template <int N>
__device__ __forceinline__ double py_sum(const double (&x)[N])
{
    double s = x[0], c = 0.0;
#pragma unroll
    for (int i = 1; i < N; ++i) {
        double t = s + x[i];
        if (fabs(s) >= fabs(x[i])) c += (s - t) + x[i];
        else c += (x[i] - t) + s;
        s = t;
    }
    if (c != 0.0 && isfinite(c)) s += c;
    return s;
}

// --------------------------------------------------- faithful log means
// fluxes.py:132-157, operation for operation.

__device__ __forceinline__ double lm_u(double a, double b)
{
    return (a * (a - 2.0 * b) + b * b) / (a * (a + 2.0 * b) + b * b);
}

__device__ __forceinline__ double lm_poly(double u)
{
    return 2.0 + u * (2.0 / 3.0 + u * (2.0 / 5.0 + u * (2.0 / 7.0)));
}

__device__ __forceinline__ double logmean_f(double a, double b)
{
    double u = lm_u(a, b);
    if (u < SERIES_EPSILON) return (a + b) / lm_poly(u);
    return (b - a) / log_cr(b / a);
}

__device__ __forceinline__ double inv_logmean_f(double a, double b)
{
    double u = lm_u(a, b);
    if (u < SERIES_EPSILON) return lm_poly(u) / (a + b);
    return log_cr(b / a) / (b - a);
}

__device__ __forceinline__ double logmean_logs_f(double a, double b, double la, double lb)
{
    double u = lm_u(a, b);
    if (u < SERIES_EPSILON) return (a + b) / lm_poly(u);
    return (b - a) / (lb - la);
}

__device__ __forceinline__ double inv_logmean_logs_f(double a, double b, double la, double lb)
{
    double u = lm_u(a, b);
    if (u < SERIES_EPSILON) return lm_poly(u) / (a + b);
    return (lb - la) / (b - a);
}

// ----------------------------------------------------------------- node data

// Primitive (and staged extra) values of one node as the pair loop sees them.
template <int D, int NX>
struct Node {
    double rho, v[D], p;
    double x[NX > 0 ? NX : 1];
};

// fluxes.py:115-121 (_prim3) / euler.py:47-60: same values in both.
template <int D, int MODE>
__device__ __forceinline__ void cons2prim(const double* u, double& rho, double (&v)[D], double& p,
                                          double gm1)
{
    rho = u[0];
    if constexpr (MODE == FAITHFUL) {
#pragma unroll
        for (int i = 0; i < D; ++i) v[i] = u[1 + i] / rho;
        double s = v[0] * v[0] + v[1] * v[1];
        if constexpr (D == 3) s = s + v[2] * v[2];
        p = gm1 * (u[D + 1] - 0.5 * rho * s);
    } else {
        double ri = rcp_fast(rho);
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            v[i] = u[1 + i] * ri;
            s = fma(v[i], v[i], s);
        }
        p = gm1 * fma(-0.5 * rho, s, u[D + 1]);
    }
}

// admissibility predicate with the gate's own pressure formula
// (discretization.py:660-672)
template <int D>
__device__ __forceinline__ bool gate_ok(const double* u, double gm1)
{
    double rho = u[0];
    double mm = u[1] * u[1] + u[2] * u[2];
    if constexpr (D == 3) mm = mm + u[3] * u[3];
    double p = gm1 * (u[D + 1] - 0.5 * mm / rho);
    return (rho > 0.0) && (p > 0.0) && isfinite(rho) && isfinite(p);
}

// Same decision without the division in the common case: the FMA-path
// pressure p_fast and the gate's pressure differ by a few ulps of
// (gamma-1) max(|E|, kinetic); whenever |p_fast| exceeds 1e-10 (gamma-1)|E|
// their signs agree, otherwise the gate's own formula decides.
#ifndef FDG_STAGE_LEAN
#define FDG_STAGE_LEAN 1  // integer finite / sign tests in gate_fast, half pressure in, negated table log
#endif
// p_half: the staged FAST half pressure p/2
template <int D>
__device__ __forceinline__ int gate_fast(const double* u, double p_half, double gm1)
{
    // 1: admissible, 0: not, -1: |p| too close to 0 for the FAST pressure's
    // sign to be trusted -> the caller re-runs gate_ok (reference formula)
    // rho positive, normal and finite in one unsigned compare on its high
    // word (a positive subnormal density goes to the reference test); an
    // infinite or NaN p fails the magnitude comparison's finite side
    const double rho = u[0];
    const bool rho_ok = (unsigned)(__double2hiint(rho) - 0x00100000) < 0x7fe00000u;
#if FDG_STAGE_LEAN
    // |p/2| finite and the sign of p on the high word (integer pipe); one
    // FP64 compare for the magnitude: |p/2| > (1e-10/2) (gamma-1) |E|
    const int hi = __double2hiint(p_half);
    const bool finite = (unsigned)(hi & 0x7fffffff) < 0x7ff00000u;
    const bool clear = rho_ok && finite && fabs(p_half) > (0.5e-10 * gm1) * fabs(u[D + 1]);
    return clear ? (hi >= 0 ? 1 : 0) : -1;
#else
    const double p_fast = 2.0 * p_half;
    const double ap = fabs(p_fast);
    const bool clear = rho_ok && ap <= 1.7976931348623157e308 && ap > 1e-10 * gm1 * fabs(u[D + 1]);
    return clear ? (p_fast > 0.0 ? 1 : 0) : -1;
#endif
}

}  // namespace fdg

#include "fdg_fast.cuh"

namespace fdg {

// Stage one node: primitives + the extras the volume flux needs.
// FAITHFUL: (rho, v, p) exactly as cons2prim computes them;
// FAST: (rho, v/2, p/2) -- see fdg_fast.cuh.
template <int D, int VF, int MODE, int LOGS, int TAB = 0>
__device__ __forceinline__ Node<D, n_extra(VF, LOGS)> make_node(const double* u, double gm1)
{
    constexpr int NX = n_extra(VF, LOGS);
    if constexpr (MODE == FAST) return make_node_fast<D, VF, LOGS, TAB>(u, gm1);
    Node<D, NX> q;
    cons2prim<D, MODE>(u, q.rho, q.v, q.p, gm1);
    if constexpr (VF == F_RANOCHA) {
#pragma unroll
        for (int i = 0; i < (NX > 0 ? NX : 1); ++i) q.x[i] = 0.0;
        if constexpr (LOGS) {
            q.x[0] = dlog<MODE>(q.rho);
            q.x[1] = dlog<MODE>(q.p);
        }
    } else if constexpr (VF == F_CHANDRASHEKAR) {
        q.x[0] = q.rho / (2.0 * q.p);  // beta
        if constexpr (LOGS) {
            q.x[1] = dlog<MODE>(q.rho);
            q.x[2] = dlog<MODE>(q.x[0]);
        }
    } else if constexpr (VF == F_KG) {
        q.x[0] = u[D + 1] / u[0];  // specific total energy
    } else if constexpr (VF == F_CENTRAL) {
#pragma unroll
        for (int i = 0; i < 5; ++i) q.x[i] = (i < D + 2) ? u[i] : 0.0;
    }
    return q;
}

// --------------------------------------------------------- volume fluxes
// AXIS >= 0: Cartesian form along that axis (normal = unit axis vector),
// AXIS <  0: directional form with the given (averaged metric) normal.

template <int D, int AXIS>
__device__ __forceinline__ void vn_pair(const double (&vl)[D], const double (&vr)[D], const double* nrm,
                                        double& vn_l, double& vn_r)
{
    if constexpr (AXIS >= 0) {
        vn_l = vl[AXIS];
        vn_r = vr[AXIS];
    } else {
        // fluxes.py:213-215: vl1*n0 + vl2*n1 + vl3*n2 (left associative)
        vn_l = vl[0] * nrm[0] + vl[1] * nrm[1];
        vn_r = vr[0] * nrm[0] + vr[1] * nrm[1];
        if constexpr (D == 3) {
            vn_l = vn_l + vl[2] * nrm[2];
            vn_r = vn_r + vr[2] * nrm[2];
        }
    }
}

template <int D, int AXIS>
__device__ __forceinline__ double nrm_comp(const double* nrm, int i)
{
    if constexpr (AXIS >= 0) return i == AXIS ? 1.0 : 0.0;
    else return nrm[i];
}

// mom_i = f_rho * 0.5 * (vl_i + vr_i) + p_avg * n_i   (fluxes.py:175-177, 236-238)
template <int D, int AXIS, int MODE>
__device__ __forceinline__ void momentum(double f_rho, double p_avg, const double (&vl)[D],
                                         const double (&vr)[D], const double* nrm, double* f)
{
#pragma unroll
    for (int i = 0; i < D; ++i) {
        double t = f_rho * 0.5 * (vl[i] + vr[i]);
        if constexpr (AXIS >= 0) {
            f[1 + i] = (i == AXIS) ? t + p_avg : t;  // p_avg * 0.0 terms are exact zeros
        } else {
            if constexpr (MODE == FAST) f[1 + i] = fma(p_avg, nrm[i], t);
            else f[1 + i] = t + p_avg * nrm[i];
        }
    }
}

template <int D, int AXIS, int MODE, int NX>
__device__ __forceinline__ void flux_shima(const Node<D, NX>& l, const Node<D, NX>& r, const double* nrm,
                                           double igm1, double* f)
{
    double vn_l, vn_r;
    vn_pair<D, AXIS>(l.v, r.v, nrm, vn_l, vn_r);
    double rho_avg = 0.5 * (l.rho + r.rho);
    double p_avg = 0.5 * (l.p + r.p);
    double vn_avg = 0.5 * (vn_l + vn_r);
    double f_rho = rho_avg * vn_avg;
    double vv = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) vv += l.v[i] * r.v[i];
    f[0] = f_rho;
    f[D + 1] = 0.5 * f_rho * vv + p_avg * vn_avg * igm1 + 0.5 * (l.p * vn_r + r.p * vn_l);
    momentum<D, AXIS, MODE>(f_rho, p_avg, l.v, r.v, nrm, f);
}

template <int D, int AXIS, int MODE, int LOGS, int NX>
__device__ __forceinline__ void flux_ranocha(const Node<D, NX>& l, const Node<D, NX>& r, const double* nrm,
                                             double igm1, double* f)
{
    double vn_l, vn_r;
    vn_pair<D, AXIS>(l.v, r.v, nrm, vn_l, vn_r);
    double rho_mean, inv_rho_p_mean;
    if constexpr (LOGS) {
        rho_mean = logmean_logs_f(l.rho, r.rho, l.x[0], r.x[0]);
        inv_rho_p_mean = l.p * r.p *
            inv_logmean_logs_f(l.rho * r.p, r.rho * l.p, l.x[0] + r.x[1], r.x[0] + l.x[1]);
    } else {
        rho_mean = logmean_f(l.rho, r.rho);
        inv_rho_p_mean = l.p * r.p * inv_logmean_f(l.rho * r.p, r.rho * l.p);
    }
    double p_avg = 0.5 * (l.p + r.p);
    double vn_avg = 0.5 * (vn_l + vn_r);
    double f_rho = rho_mean * vn_avg;
    double vv = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) vv += l.v[i] * r.v[i];
    f[0] = f_rho;
    f[D + 1] = f_rho * (0.5 * vv + igm1 * inv_rho_p_mean) + 0.5 * (l.p * vn_r + r.p * vn_l);
    momentum<D, AXIS, MODE>(f_rho, p_avg, l.v, r.v, nrm, f);
}

// Physical flux contracted with a direction, conserved input (fluxes.py:293-300).
template <int D, int AXIS>
__device__ __forceinline__ void phys_flux_n(const double* u, double rho, const double (&v)[D], double p,
                                            const double* nrm, double* f)
{
    double vn = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) vn += v[i] * nrm_comp<D, AXIS>(nrm, i);
    f[0] = rho * vn;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        if constexpr (AXIS >= 0) f[1 + i] = (i == AXIS) ? u[1 + i] * vn + p : u[1 + i] * vn;
        else f[1 + i] = u[1 + i] * vn + p * nrm[i];
    }
    f[D + 1] = (u[D + 1] + p) * vn;
}

template <int D, int AXIS, int MODE, int NX>
__device__ __forceinline__ void flux_central(const Node<D, NX>& l, const Node<D, NX>& r, const double* nrm,
                                             double igm1, int prim_form, double* f)
{
    double fl[D + 2], fr[D + 2];
    if (MODE == FAST || !prim_form) {
        phys_flux_n<D, AXIS>(l.x, l.rho, l.v, l.p, nrm, fl);
        phys_flux_n<D, AXIS>(r.x, r.rho, r.v, r.p, nrm, fr);
    } else {
        // flux_central_directional_prim (fluxes.py:592-610)
        const Node<D, NX>* qs[2] = {&l, &r};
        double* fs[2] = {fl, fr};
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const Node<D, NX>& q = *qs[s];
            double vn = 0.0;
#pragma unroll
            for (int i = 0; i < D; ++i) vn += q.v[i] * nrm_comp<D, AXIS>(nrm, i);
            double rhovn = q.rho * vn;
            double sq[D];
#pragma unroll
            for (int i = 0; i < D; ++i) sq[i] = q.v[i] * q.v[i];
            double e = q.p * igm1 + 0.5 * q.rho * py_sum<D>(sq);
            fs[s][0] = rhovn;
#pragma unroll
            for (int i = 0; i < D; ++i) {
                if constexpr (AXIS >= 0) fs[s][1 + i] = (i == AXIS) ? rhovn * q.v[i] + q.p : rhovn * q.v[i];
                else fs[s][1 + i] = rhovn * q.v[i] + q.p * nrm[i];
            }
            fs[s][D + 1] = (e + q.p) * vn;
        }
    }
#pragma unroll
    for (int v = 0; v < D + 2; ++v) f[v] = 0.5 * (fl[v] + fr[v]);
}

// Kennedy-Gruber (parity unpinned): f_rho = {rho}{v.n}; f_m = f_rho{v} + {p}n;
// f_E = f_rho {e} + {p}{v.n}, e = rho E / rho.
template <int D, int AXIS, int MODE, int NX>
__device__ __forceinline__ void flux_kg(const Node<D, NX>& l, const Node<D, NX>& r, const double* nrm, double* f)
{
    double vn_l, vn_r;
    vn_pair<D, AXIS>(l.v, r.v, nrm, vn_l, vn_r);
    double rho_avg = 0.5 * (l.rho + r.rho);
    double p_avg = 0.5 * (l.p + r.p);
    double vn_avg = 0.5 * (vn_l + vn_r);
    double e_avg = 0.5 * (l.x[0] + r.x[0]);
    double f_rho = rho_avg * vn_avg;
    f[0] = f_rho;
    momentum<D, AXIS, MODE>(f_rho, p_avg, l.v, r.v, nrm, f);
    f[D + 1] = f_rho * e_avg + p_avg * vn_avg;
}

// Chandrashekar EC (parity unpinned): beta = rho/(2p);
// f_rho = <rho>_log {v.n}; f_m = f_rho {v} + {rho}/(2{beta}) n;
// f_E = f_rho (1/(2(gamma-1)<beta>_log) - 1/2 {|v|^2}) + {v}.f_m
template <int D, int AXIS, int MODE, int LOGS, int NX>
__device__ __forceinline__ void flux_chandrashekar(const Node<D, NX>& l, const Node<D, NX>& r,
                                                   const double* nrm, double igm1, double* f)
{
    double vn_l, vn_r;
    vn_pair<D, AXIS>(l.v, r.v, nrm, vn_l, vn_r);
    double rho_avg = 0.5 * (l.rho + r.rho);
    double beta_avg = 0.5 * (l.x[0] + r.x[0]);
    const double rho_mean = logmean_f(l.rho, r.rho);
    const double inv_beta_mean = inv_logmean_f(l.x[0], r.x[0]);
    const double p_tilde = rho_avg / (2.0 * beta_avg);
    double vn_avg = 0.5 * (vn_l + vn_r);
    double f_rho = rho_mean * vn_avg;
    double v2_l = 0.0, v2_r = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        v2_l += l.v[i] * l.v[i];
        v2_r += r.v[i] * r.v[i];
    }
    double v2_avg = 0.5 * (v2_l + v2_r);
    f[0] = f_rho;
    double work = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        double va = 0.5 * (l.v[i] + r.v[i]);
        double t = f_rho * va;
        if constexpr (AXIS >= 0) f[1 + i] = (i == AXIS) ? t + p_tilde : t;
        else f[1 + i] = t + p_tilde * nrm[i];
        work += va * f[1 + i];
    }
    f[D + 1] = f_rho * (0.5 * igm1 * inv_beta_mean - 0.5 * v2_avg) + work;
}

struct Gas {
    double gamma, gm1, igm1;
};

// Volume two-point flux dispatch (compile-time kind).
template <int D, int VF, int AXIS, int MODE, int LOGS, int EH = 0, int KP = 0, int NX>
__device__ __forceinline__ void volume_flux(const Node<D, NX>& l, const Node<D, NX>& r, const double* nrm,
                                            const Gas& gas, int pre, double* f, unsigned vm)
{
    if constexpr (MODE == FAST) fast_volume_flux<D, VF, AXIS, LOGS, EH, KP>(l, r, nrm, gas.igm1, f, vm);
    else if constexpr (VF == F_SHIMA) flux_shima<D, AXIS, MODE>(l, r, nrm, gas.igm1, f);
    else if constexpr (VF == F_RANOCHA) flux_ranocha<D, AXIS, MODE, LOGS>(l, r, nrm, gas.igm1, f);
    else if constexpr (VF == F_CENTRAL) flux_central<D, AXIS, MODE>(l, r, nrm, gas.igm1, pre != PRE_NONE, f);
    else if constexpr (VF == F_KG) flux_kg<D, AXIS, MODE>(l, r, nrm, f);
    else flux_chandrashekar<D, AXIS, MODE, LOGS>(l, r, nrm, gas.igm1, f);
}

// ------------------------------------------------------------ surface fluxes
// Conserved-input directional kernels, as surface_terms calls them
// (discretization.py:698, 742: flux_function(kind, "directional")).

template <int D, int MODE>
__device__ __forceinline__ void split_normal(const double* nrm, double& norm, double (&unit)[D])
{
    double nn = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) nn += nrm[i] * nrm[i];
    nn = sqrt(nn);
    norm = nn;
#pragma unroll
    for (int i = 0; i < D; ++i) unit[i] = nrm[i] / nn;
}

template <int D, int MODE>
__device__ __forceinline__ void flux_llf(const double* ul, const double* ur, const double* nrm, const Gas& gas,
                                         double* f)
{
    double rho_l, rho_r, vl[D], vr[D], p_l, p_r;
    cons2prim<D, MODE>(ul, rho_l, vl, p_l, gas.gm1);
    cons2prim<D, MODE>(ur, rho_r, vr, p_r, gas.gm1);
    double norm, unit[D];
    split_normal<D, MODE>(nrm, norm, unit);
    double vn_l = 0.0, vn_r = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        vn_l += vl[i] * unit[i];
        vn_r += vr[i] * unit[i];
    }
    double lam_l = fabs(vn_l) + sqrt(gas.gamma * p_l / rho_l);
    double lam_r = fabs(vn_r) + sqrt(gas.gamma * p_r / rho_r);
    double lam = (lam_r > lam_l) ? lam_r : lam_l;  // python max(a, b)
    double fl[D + 2], fr[D + 2];
    phys_flux_n<D, -1>(ul, rho_l, vl, p_l, nrm, fl);
    phys_flux_n<D, -1>(ur, rho_r, vr, p_r, nrm, fr);
    double halfdiss = 0.5 * lam * norm;
#pragma unroll
    for (int v = 0; v < D + 2; ++v) f[v] = 0.5 * (fl[v] + fr[v]) - halfdiss * (ur[v] - ul[v]);
}

template <int D, int MODE>
__device__ __forceinline__ void flux_hll(const double* ul, const double* ur, const double* nrm, const Gas& gas,
                                         double* f)
{
    double rho_l, rho_r, vl[D], vr[D], p_l, p_r;
    cons2prim<D, MODE>(ul, rho_l, vl, p_l, gas.gm1);
    cons2prim<D, MODE>(ur, rho_r, vr, p_r, gas.gm1);
    double norm, unit[D];
    split_normal<D, MODE>(nrm, norm, unit);
    double vn_l = 0.0, vn_r = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        vn_l += vl[i] * unit[i];
        vn_r += vr[i] * unit[i];
    }
    double c_l = sqrt(gas.gamma * p_l / rho_l);
    double c_r = sqrt(gas.gamma * p_r / rho_r);
    double a1 = vn_l - c_l, b1 = vn_r - c_r;
    double s_l = (b1 < a1) ? b1 : a1;  // python min
    double a2 = vn_l + c_l, b2 = vn_r + c_r;
    double s_r = (b2 > a2) ? b2 : a2;  // python max
    double fl[D + 2], fr[D + 2];
    phys_flux_n<D, -1>(ul, rho_l, vl, p_l, unit, fl);
    phys_flux_n<D, -1>(ur, rho_r, vr, p_r, unit, fr);
    if (s_l >= 0.0) {
#pragma unroll
        for (int v = 0; v < D + 2; ++v) f[v] = norm * fl[v];
    } else if (s_r <= 0.0) {
#pragma unroll
        for (int v = 0; v < D + 2; ++v) f[v] = norm * fr[v];
    } else {
        double inv = 1.0 / (s_r - s_l);
#pragma unroll
        for (int v = 0; v < D + 2; ++v)
            f[v] = norm * ((s_r * fl[v] - s_l * fr[v] + s_l * s_r * (ur[v] - ul[v])) * inv);
    }
}

// FAST Rusanov flux: AXIS >= 0 is the Cartesian face (normal = area e_AXIS,
// area = nrm[AXIS] > 0), AXIS < 0 a general scaled normal.
template <int D, int AXIS>
__device__ __forceinline__ void flux_llf_fast(const double* ul, const double* ur, const double* nrm, const Gas& gas,
                                              double* f)
{
    const double ril = rcp_fast(ul[0]), rir = rcp_fast(ur[0]);
    double vl[D], vr[D], kl = 0.0, kr = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        vl[i] = ul[1 + i] * ril;
        vr[i] = ur[1 + i] * rir;
        kl = fma(ul[1 + i], vl[i], kl);
        kr = fma(ur[1 + i], vr[i], kr);
    }
    const double p_l = gas.gm1 * fma(-0.5, kl, ul[D + 1]);
    const double p_r = gas.gm1 * fma(-0.5, kr, ur[D + 1]);
    double norm, vns_l, vns_r, inorm_ = 0.0;  // |n| and v.n with the scaled normal
    double avl = 0.0, avr = 0.0;              // AXIS >= 0: |v.n| / |n| = |v_axis| (area > 0)
    if constexpr (AXIS >= 0) {
        norm = nrm[AXIS];
        vns_l = vl[AXIS] * norm;
        vns_r = vr[AXIS] * norm;
        avl = fabs(vl[AXIS]);
        avr = fabs(vr[AXIS]);
    } else {
        double nn = 0.0;
        vns_l = 0.0;
        vns_r = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            nn = fma(nrm[i], nrm[i], nn);
            vns_l = fma(vl[i], nrm[i], vns_l);
            vns_r = fma(vr[i], nrm[i], vns_r);
        }
        inorm_ = rsqrt_fast(nn);
        norm = nn * inorm_;
    }
    // sound speeds sqrt(gamma p / rho) as x rsqrt(x): no IEEE sqrt slow path
    // (admissible states have p, rho > 0; the gate reports the others)
    const double cl2 = gas.gamma * p_l * ril, cr2 = gas.gamma * p_r * rir;
    double lam_l, lam_r;
    if constexpr (AXIS >= 0) {
        lam_l = fma(cl2, rsqrt_fast(cl2), avl);
        lam_r = fma(cr2, rsqrt_fast(cr2), avr);
    } else {
        lam_l = fma(fabs(vns_l), inorm_, cl2 * rsqrt_fast(cl2));
        lam_r = fma(fabs(vns_r), inorm_, cr2 * rsqrt_fast(cr2));
    }
    const double halfdiss = 0.5 * fmax(lam_l, lam_r) * norm;
    f[0] = 0.5 * (ul[0] * vns_l + ur[0] * vns_r) - halfdiss * (ur[0] - ul[0]);
#pragma unroll
    for (int i = 0; i < D; ++i) {
        const double pn = (AXIS >= 0) ? ((i == AXIS) ? (p_l + p_r) * norm : 0.0) : (p_l + p_r) * nrm[i];
        f[1 + i] = 0.5 * (fma(ul[1 + i], vns_l, ur[1 + i] * vns_r) + pn) - halfdiss * (ur[1 + i] - ul[1 + i]);
    }
    f[D + 1] = 0.5 * fma(ul[D + 1] + p_l, vns_l, (ur[D + 1] + p_r) * vns_r) - halfdiss * (ur[D + 1] - ul[D + 1]);
}

// FAST Rusanov flux of a fused interface term (line_faces): one side is the
// element's own end node, taken from the staged FAST primitives in shared
// memory (rho, v/2, p/2: no reciprocal, no global re-read of the own trace),
// the other side the neighbour's conserved trace from global memory.
// OWN_LEFT: the own node is the left (minus) state. The two elements of an
// interface then evaluate the flux from differently rounded copies of each
// other's state (staged primitives vs conserved), so the two lifted values
// agree to rounding (~1e-16 relative), not to the bit.
#ifndef FDG_LLF_OWN_LEAN
#define FDG_LLF_OWN_LEAN 1
#endif
#if FDG_LLF_OWN_LEAN
// Every 1/2 of the Rusanov flux is taken from the half-staged own values or
// folded into a uniform constant: own momenta as (2 rho) (v/2), the half
// normal mass-flux factors v.n/2 straight from v/2 (own) and from the halved
// normal (neighbour), the half pressures summed for the pressure term --
// 69 instead of 78 FP64 instructions per flux (3D, axis aligned), same value
// up to the rounding of the rearranged products.
template <int D, int AXIS, bool OWN_LEFT>
__device__ __forceinline__ void flux_llf_fast_own(double orho, const double* ovh, double oph, const double* un,
                                                  const double* nrm, const Gas& gas, double* f)
{
    // own side from the staged values
    const double r2 = 2.0 * orho;
    double om[D], s = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        om[i] = r2 * ovh[i];
        s = fma(ovh[i], ovh[i], s);
    }
    const double oE = fma(r2, s, oph * (2.0 * gas.igm1));  // rho |v|^2 / 2 + p / (gamma - 1)
    // neighbour side from its conserved trace
    const double rin = rcp_fast(un[0]);
    double nv[D], kn = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        nv[i] = un[1 + i] * rin;
        kn = fma(un[1 + i], nv[i], kn);
    }
    const double nph = (0.5 * gas.gm1) * fma(-0.5, kn, un[D + 1]);  // p_n / 2
    // ohv, nhv: v.n / 2 with the scaled normal; olam, nlam: |v.n|/|n| + c
    double norm, ohv, nhv, olam, nlam;
    // c = sqrt(gamma p / rho) = gamma p rsqrt(gamma p rho): no reciprocal of the own density
    const double g2 = 2.0 * gas.gamma;
    const double ogp = g2 * oph, ngp = g2 * nph;
    const double oc = ogp * rsqrt_fast(ogp * orho), nc = ngp * rsqrt_fast(ngp * un[0]);
    if constexpr (AXIS >= 0) {
        norm = nrm[AXIS];
        ohv = ovh[AXIS] * norm;
        nhv = nv[AXIS] * (0.5 * norm);
        olam = fma(2.0, fabs(ovh[AXIS]), oc);
        nlam = nc + fabs(nv[AXIS]);
    } else {
        double nn = 0.0, nvn = 0.0;
        ohv = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            nn = fma(nrm[i], nrm[i], nn);
            ohv = fma(ovh[i], nrm[i], ohv);
            nvn = fma(nv[i], nrm[i], nvn);
        }
        const double inorm_ = rsqrt_fast(nn);
        norm = nn * inorm_;
        nhv = 0.5 * nvn;
        olam = fma(fabs(ohv), 2.0 * inorm_, oc);
        nlam = fma(fabs(nvn), inorm_, nc);
    }
    const double hd = 0.5 * fmax(olam, nlam) * norm;
    const double sg = OWN_LEFT ? hd : -hd;  // -halfdiss (u_r - u_l) = sg (own - neighbour)
    const double hp = oph + nph;            // {p}
    f[0] = fma(sg, orho - un[0], fma(orho, ohv, un[0] * nhv));
#pragma unroll
    for (int i = 0; i < D; ++i) {
        const double c = fma(om[i], ohv, un[1 + i] * nhv);
        double cp;
        if constexpr (AXIS >= 0) cp = (i == AXIS) ? fma(hp, norm, c) : c;
        else cp = fma(hp, nrm[i], c);
        f[1 + i] = fma(sg, om[i] - un[1 + i], cp);
    }
    f[D + 1] = fma(sg, oE - un[D + 1], fma(fma(2.0, oph, oE), ohv, fma(2.0, nph, un[D + 1]) * nhv));
}
#else
template <int D, int AXIS, bool OWN_LEFT>
__device__ __forceinline__ void flux_llf_fast_own(double orho, const double* ovh, double oph, const double* un,
                                                  const double* nrm, const Gas& gas, double* f)
{
    // own side from the staged values
    double ov[D], om[D], s = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        ov[i] = 2.0 * ovh[i];
        om[i] = orho * ov[i];
        s = fma(ovh[i], ovh[i], s);
    }
    const double op = 2.0 * oph;
    const double oE = fma(2.0 * orho, s, op * gas.igm1);
    // neighbour side from its conserved trace
    const double rin = rcp_fast(un[0]);
    double nv[D], kn = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        nv[i] = un[1 + i] * rin;
        kn = fma(un[1 + i], nv[i], kn);
    }
    const double np_ = gas.gm1 * fma(-0.5, kn, un[D + 1]);
    double norm, ovns, nvns, inorm_ = 0.0, aov = 0.0, anv = 0.0;
    if constexpr (AXIS >= 0) {
        norm = nrm[AXIS];
        ovns = ov[AXIS] * norm;
        nvns = nv[AXIS] * norm;
        aov = fabs(ov[AXIS]);
        anv = fabs(nv[AXIS]);
    } else {
        double nn = 0.0;
        ovns = 0.0;
        nvns = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            nn = fma(nrm[i], nrm[i], nn);
            ovns = fma(ov[i], nrm[i], ovns);
            nvns = fma(nv[i], nrm[i], nvns);
        }
        inorm_ = rsqrt_fast(nn);
        norm = nn * inorm_;
    }
    // c = sqrt(gamma p / rho) = gamma p rsqrt(gamma p rho): no reciprocal of the own density
    const double ogp = gas.gamma * op, ngp = gas.gamma * np_;
    const double oc = ogp * rsqrt_fast(ogp * orho), nc = ngp * rsqrt_fast(ngp * un[0]);
    double olam, nlam;
    if constexpr (AXIS >= 0) {
        olam = oc + aov;
        nlam = nc + anv;
    } else {
        olam = fma(fabs(ovns), inorm_, oc);
        nlam = fma(fabs(nvns), inorm_, nc);
    }
    const double hd = 0.5 * fmax(olam, nlam) * norm;
    const double sg = OWN_LEFT ? hd : -hd;  // -halfdiss (u_r - u_l) = sg (own - neighbour)
    f[0] = fma(sg, orho - un[0], 0.5 * fma(orho, ovns, un[0] * nvns));
#pragma unroll
    for (int i = 0; i < D; ++i) {
        const double pn = (AXIS >= 0) ? ((i == AXIS) ? (op + np_) * norm : 0.0) : (op + np_) * nrm[i];
        f[1 + i] = fma(sg, om[i] - un[1 + i], 0.5 * (fma(om[i], ovns, un[1 + i] * nvns) + pn));
    }
    f[D + 1] = fma(sg, oE - un[D + 1], 0.5 * fma(oE + op, ovns, (un[D + 1] + np_) * nvns));
}

#endif

// Two-point flux with conserved inputs for the interface (runtime kind).
template <int D, int MODE>
__device__ __noinline__ void surface_flux(int kind, const double* ul, const double* ur, const double* nrm,
                                          const Gas& gas, double* f)
{
    switch (kind) {
    case F_LLF: flux_llf<D, MODE>(ul, ur, nrm, gas, f); return;
    case F_HLL: flux_hll<D, MODE>(ul, ur, nrm, gas, f); return;
    default: break;
    }
    // symmetric volume kinds used as surface fluxes: stage both states
    // exactly as the conserved-input kernels do, no log tables
    // (surface_terms never passes precomputed data, discretization.py:742)
    switch (kind) {
#define FDG_SURF_SYM(K)                                                 \
    case K: {                                                           \
        const auto l = make_node<D, K, MODE, 0>(ul, gas.gm1);           \
        const auto r = make_node<D, K, MODE, 0>(ur, gas.gm1);           \
        volume_flux<D, K, -1, MODE, 0>(l, r, nrm, gas, PRE_NONE, f,     \
                                       __activemask());                 \
        return;                                                         \
    }
        FDG_SURF_SYM(F_SHIMA)
        FDG_SURF_SYM(F_RANOCHA)
        FDG_SURF_SYM(F_CENTRAL)
        FDG_SURF_SYM(F_KG)
        FDG_SURF_SYM(F_CHANDRASHEKAR)
#undef FDG_SURF_SYM
    default:
#pragma unroll
        for (int v = 0; v < D + 2; ++v) f[v] = __longlong_as_double(0x7ff8000000000000ULL);
    }
}

}  // namespace fdg
