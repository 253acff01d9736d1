/*
 * fdg_oracle.c -- CPU ORACLE (test infrastructure, NOT the product).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * the reported CPU baseline.  The product path (paper_2112_10517_b200) never
 * links or calls it.
 *
 * What it is: a plain-C restatement of the reference's *scalar* flux-
 * differencing path (arXiv 2112.10517 artifact `fluxdg`, read-only at
 * /root/reference/pkg/src/fluxdg), written so that every floating-point
 * operation happens in the same order and association as the Python source:
 *
 *   volume term    discretization.py:267-323  (volume_fluxdiff)
 *   surface term   discretization.py:681-760  (surface_terms, LGL branch)
 *   rhs            discretization.py:896-949  (rhs, fluxdiff branch)
 *   gate           discretization.py:660-672  (_admissibility_gate)
 *   log means      fluxes.py:132-157          (_logmean, _inv_logmean, *_from_logs)
 *   shima          fluxes.py:163-218, 516-547
 *   ranocha        fluxes.py:224-287, 550-589
 *   central        fluxes.py:293-325, 592-616
 *   llf / hll      fluxes.py:335-415
 *   cons2prim      euler.py:47-60 / fluxes.py:107-121
 *
 * Pinning: tests/test_oracle.py checks this library against the golden
 * fixtures written by tests/golden/make_golden.py from the reference itself;
 * volume, surface and rhs outputs are required to be BITWISE equal
 * (np.array_equal).  Build with -ffp-contract=off (no FMA contraction) and
 * without -ffast-math; `log` is glibc's, the same libm CPython's math.log uses.
 *
 * Kennedy-Gruber and Chandrashekar (BASELINE cfg 3/4) are not in the
 * reference: their restatement here is "parity unpinned" and is checked by
 * properties only, in tests/test_flux_properties.py: symmetry, consistency
 * f(u,u,n) = sum_j n_j f^j(u), Cartesian-axis == directional, the
 * Chandrashekar entropy-conservation residual against 50-digit entropy
 * variables (Ranocha as the control), and the KEP structure
 * f_rhov - {v} f_rho = p~ n of both.
 *
 * Surface assembly is written per element and per side (each interface flux
 * is evaluated once from each adjacent element with identical arguments), so
 * every node receives at most one contribution per direction in direction
 * order -- the same per-node sequence of roundings as the reference's
 * face loop -- and elements can be processed in parallel (pthreads).  Neighbour indices
 * < 0 refer to ghost face traces (slab decomposition, see parallel tests).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define SERIES_EPSILON 1.0e-4 /* means.py:16 */

/* OR_LOG: glibc log (the reference's math.log) by default; with
 * -DFDG_ORACLE_LOGCR the correctly rounded log_cr that the GPU FAITHFUL mode
 * uses (same source, paper_2112_10517_b200/csrc/fdg_logcr.h, itself checked
 * against mpmath in tests/test_logcr.py).  liboracle_cr.so is therefore the
 * bitwise oracle for the GPU FAITHFUL kernels, and differs from liboracle.so
 * only where glibc's log is misrounded.                                      */
#ifdef FDG_ORACLE_LOGCR
#include "../paper_2112_10517_b200/csrc/fdg_logcr.h"
#define OR_LOG(x) log_cr(x)
#else
#define OR_LOG(x) log(x)
#endif

enum { F_CENTRAL = 0, F_SHIMA = 1, F_RANOCHA = 2, F_KG = 3, F_CHANDRASHEKAR = 4, F_LLF = 5, F_HLL = 6 };
enum { PRE_NONE = 0, PRE_PRIMITIVES = 1, PRE_LOGS = 2 };

typedef struct {
    int d;           /* 2 or 3 */
    int p1;          /* nodes per direction */
    int64_t n_elem;  /* local elements */
    const double *dsplit;  /* (p1, p1) row-major, build_dsplit(op).matrix */
    const double *weights; /* (p1,) LGL weights */
    double gamma;          /* gas.gamma */
    double igm1;           /* gas.inv_gamma_minus_one = 1/(gamma-1) */
    int cartesian;         /* 1: axis fluxes scaled by areas, J constant */
    const double *areas;   /* (d,) Ja^n_n of the Cartesian mesh */
    double jac_const;      /* J of the Cartesian mesh */
    const double *ja;      /* (n_elem, nn, d, d) curved metrics (NULL if cartesian) */
    const double *jac;     /* (n_elem, nn) (NULL -> jac_const) */
    const int64_t *plus;   /* (d, n_elem): +n neighbour, <0 -> ghost slot -(g+1) */
    const int64_t *minus;  /* (d, n_elem): -n neighbour, <0 -> ghost slot */
    const double *ghost_u;   /* (n_ghost, fn, nvar) face states of remote neighbours */
    const double *ghost_nrm; /* (n_ghost, fn, d) face normals of remote minus neighbours */
} or_mesh;

/* ------------------------------------------------------------------ means */

static inline double lm_u(double a, double b)
{
    return (a * (a - 2.0 * b) + b * b) / (a * (a + 2.0 * b) + b * b);
}

static inline double logmean(double a, double b)
{
    double u = lm_u(a, b);
    if (u < SERIES_EPSILON)
        return (a + b) / (2.0 + u * (2.0 / 3.0 + u * (2.0 / 5.0 + u * (2.0 / 7.0))));
    return (b - a) / OR_LOG(b / a);
}

static inline double inv_logmean(double a, double b)
{
    double u = lm_u(a, b);
    if (u < SERIES_EPSILON)
        return (2.0 + u * (2.0 / 3.0 + u * (2.0 / 5.0 + u * (2.0 / 7.0)))) / (a + b);
    return OR_LOG(b / a) / (b - a);
}

static inline double logmean_logs(double a, double b, double la, double lb)
{
    double u = lm_u(a, b);
    if (u < SERIES_EPSILON)
        return (a + b) / (2.0 + u * (2.0 / 3.0 + u * (2.0 / 5.0 + u * (2.0 / 7.0))));
    return (b - a) / (lb - la);
}

static inline double inv_logmean_logs(double a, double b, double la, double lb)
{
    double u = lm_u(a, b);
    if (u < SERIES_EPSILON)
        return (2.0 + u * (2.0 / 3.0 + u * (2.0 / 5.0 + u * (2.0 / 7.0)))) / (a + b);
    return (lb - la) / (b - a);
}

/* ------------------------------------------------------------- node data */

typedef struct {
    double u[5];   /* conserved */
    double rho, v[3], p;
    double x0, x1; /* log rho, log p (ranocha+logs) | beta (chandrashekar) | e (kg) */
} node_t;

static inline void make_node(node_t *q, const double *u, int d, double gm1, int flux, int pre)
{
    for (int v = 0; v < 5; ++v) q->u[v] = (v < d + 2) ? u[v] : 0.0;
    q->rho = u[0];
    q->v[0] = q->v[1] = q->v[2] = 0.0;
    for (int i = 0; i < d; ++i) q->v[i] = u[1 + i] / u[0];
    double s = q->v[0] * q->v[0] + q->v[1] * q->v[1];
    if (d == 3) s = s + q->v[2] * q->v[2];
    q->p = gm1 * (u[d + 1] - 0.5 * u[0] * s);
    q->x0 = q->x1 = 0.0;
    if (flux == F_RANOCHA && pre == PRE_LOGS) {
        q->x0 = OR_LOG(q->rho);
        q->x1 = OR_LOG(q->p);
    } else if (flux == F_CHANDRASHEKAR) {
        q->x0 = q->rho / (2.0 * q->p); /* beta */
    } else if (flux == F_KG) {
        q->x0 = u[d + 1] / u[0]; /* specific total energy */
    }
}

/* vn as the conserved-input directional kernels write it (fluxes.py:207-215) */
static inline double vn_expr(const double *v, const double *n, int d)
{
    double r = v[0] * n[0] + v[1] * n[1];
    if (d == 3) r = r + v[2] * n[2];
    return r;
}

/* vn as the loop kernels write it: 0.0 then += (fluxes.py:295-297, 524-527) */
static inline double vn_loop(const double *v, const double *n, int d)
{
    double r = 0.0;
    for (int i = 0; i < d; ++i) r += v[i] * n[i];
    return r;
}

/* ----------------------------------------------------------- two-point fluxes
 * normal: the direction handed to the kernel (axis unit vector for the
 * Cartesian forms, the averaged metric vector for curved elements).
 * cart_axis >= 0 selects the Cartesian form (vn = v[j]).                     */

static inline void flux_shima(const node_t *l, const node_t *r, const double *nrm, int cart_axis,
                              int d, double igm1, double *f)
{
    double vn_l, vn_r;
    if (cart_axis >= 0) { vn_l = l->v[cart_axis]; vn_r = r->v[cart_axis]; }
    else { vn_l = vn_expr(l->v, nrm, d); vn_r = vn_expr(r->v, nrm, d); }
    double rho_avg = 0.5 * (l->rho + r->rho);
    double p_avg = 0.5 * (l->p + r->p);
    double vn_avg = 0.5 * (vn_l + vn_r);
    double f_rho = rho_avg * vn_avg;
    double vv = 0.0;
    for (int i = 0; i < d; ++i) vv += l->v[i] * r->v[i];
    double f_e = 0.5 * f_rho * vv + p_avg * vn_avg * igm1 + 0.5 * (l->p * vn_r + r->p * vn_l);
    f[0] = f_rho;
    for (int i = 0; i < d; ++i) f[1 + i] = f_rho * 0.5 * (l->v[i] + r->v[i]) + p_avg * nrm[i];
    f[d + 1] = f_e;
}

static inline void flux_ranocha(const node_t *l, const node_t *r, const double *nrm, int cart_axis,
                                int d, double igm1, int logs, double *f)
{
    double vn_l, vn_r;
    if (cart_axis >= 0) { vn_l = l->v[cart_axis]; vn_r = r->v[cart_axis]; }
    else { vn_l = vn_expr(l->v, nrm, d); vn_r = vn_expr(r->v, nrm, d); }
    double rho_mean, inv_rho_p_mean;
    if (logs) {
        rho_mean = logmean_logs(l->rho, r->rho, l->x0, r->x0);
        inv_rho_p_mean = l->p * r->p *
            inv_logmean_logs(l->rho * r->p, r->rho * l->p, l->x0 + r->x1, r->x0 + l->x1);
    } else {
        rho_mean = logmean(l->rho, r->rho);
        inv_rho_p_mean = l->p * r->p * inv_logmean(l->rho * r->p, r->rho * l->p);
    }
    double p_avg = 0.5 * (l->p + r->p);
    double vn_avg = 0.5 * (vn_l + vn_r);
    double f_rho = rho_mean * vn_avg;
    double vv = 0.0;
    for (int i = 0; i < d; ++i) vv += l->v[i] * r->v[i];
    double f_e = f_rho * (0.5 * vv + igm1 * inv_rho_p_mean) + 0.5 * (l->p * vn_r + r->p * vn_l);
    f[0] = f_rho;
    for (int i = 0; i < d; ++i) f[1 + i] = f_rho * 0.5 * (l->v[i] + r->v[i]) + p_avg * nrm[i];
    f[d + 1] = f_e;
}

/* physical flux contracted with a direction, conserved input (fluxes.py:293-300) */
static inline void phys_flux_n(const node_t *q, const double *nrm, int d, double *f)
{
    double vn = vn_loop(q->v, nrm, d);
    f[0] = q->rho * vn;
    for (int i = 0; i < d; ++i) f[1 + i] = q->u[1 + i] * vn + q->p * nrm[i];
    f[d + 1] = (q->u[d + 1] + q->p) * vn;
}

/* Python >= 3.12 builtin sum() over floats (start 0): the first term is taken
 * exactly, the rest are added with Neumaier compensation, and the
 * compensation is folded in at the end if it is nonzero and finite.  The
 * reference uses it once on the hot path: flux_central_directional_prim's
 * kinetic term (fluxes.py:603-605).                                         */
static inline double py_sum(const double *x, int n)
{
    double s = x[0], c = 0.0;
    for (int i = 1; i < n; ++i) {
        double t = s + x[i];
        if (fabs(s) >= fabs(x[i])) c += (s - t) + x[i];
        else c += (x[i] - t) + s;
        s = t;
    }
    if (c != 0.0 && isfinite(c)) s += c;
    return s;
}

static inline void flux_central(const node_t *l, const node_t *r, const double *nrm, int d,
                                double igm1, int prim_form, double *f)
{
    double fl[5], fr[5];
    if (!prim_form) {
        phys_flux_n(l, nrm, d, fl);
        phys_flux_n(r, nrm, d, fr);
    } else { /* flux_central_directional_prim, fluxes.py:592-610 */
        const node_t *qs[2] = {l, r};
        double *fs[2] = {fl, fr};
        for (int s = 0; s < 2; ++s) {
            const node_t *q = qs[s];
            double vn = vn_loop(q->v, nrm, d);
            double rhovn = q->rho * vn;
            double sq[3] = {0.0, 0.0, 0.0};
            for (int i = 0; i < d; ++i) sq[i] = q->v[i] * q->v[i];
            double e = q->p * igm1 + 0.5 * q->rho * py_sum(sq, d);
            fs[s][0] = rhovn;
            for (int i = 0; i < d; ++i) fs[s][1 + i] = rhovn * q->v[i] + q->p * nrm[i];
            fs[s][d + 1] = (e + q->p) * vn;
        }
    }
    for (int v = 0; v < d + 2; ++v) f[v] = 0.5 * (fl[v] + fr[v]);
}

/* Kennedy-Gruber KEP flux -- NOT in the reference (parity unpinned).
 * f_rho = {rho}{v.n}, f_m = f_rho{v} + {p}n, f_E = f_rho{e} + {p}{v.n}       */
static inline void flux_kg(const node_t *l, const node_t *r, const double *nrm, int cart_axis,
                           int d, double *f)
{
    double vn_l, vn_r;
    if (cart_axis >= 0) { vn_l = l->v[cart_axis]; vn_r = r->v[cart_axis]; }
    else { vn_l = vn_expr(l->v, nrm, d); vn_r = vn_expr(r->v, nrm, d); }
    double rho_avg = 0.5 * (l->rho + r->rho);
    double p_avg = 0.5 * (l->p + r->p);
    double vn_avg = 0.5 * (vn_l + vn_r);
    double e_avg = 0.5 * (l->x0 + r->x0);
    double f_rho = rho_avg * vn_avg;
    f[0] = f_rho;
    for (int i = 0; i < d; ++i) f[1 + i] = f_rho * 0.5 * (l->v[i] + r->v[i]) + p_avg * nrm[i];
    f[d + 1] = f_rho * e_avg + p_avg * vn_avg;
}

/* Chandrashekar EC flux -- NOT in the reference (parity unpinned).
 * beta = rho/(2p); f_rho = <rho>_log {v.n}; f_m = f_rho{v} + {rho}/(2{beta}) n;
 * f_E = f_rho (1/(2(gamma-1)<beta>_log) - 1/2 {|v|^2}) + {v}.f_m             */
static inline void flux_chandrashekar(const node_t *l, const node_t *r, const double *nrm,
                                      int cart_axis, int d, double igm1, double *f)
{
    double vn_l, vn_r;
    if (cart_axis >= 0) { vn_l = l->v[cart_axis]; vn_r = r->v[cart_axis]; }
    else { vn_l = vn_expr(l->v, nrm, d); vn_r = vn_expr(r->v, nrm, d); }
    double rho_mean = logmean(l->rho, r->rho);
    double inv_beta_mean = inv_logmean(l->x0, r->x0);
    double rho_avg = 0.5 * (l->rho + r->rho);
    double beta_avg = 0.5 * (l->x0 + r->x0);
    double p_tilde = rho_avg / (2.0 * beta_avg);
    double vn_avg = 0.5 * (vn_l + vn_r);
    double f_rho = rho_mean * vn_avg;
    double v2_l = 0.0, v2_r = 0.0;
    for (int i = 0; i < d; ++i) { v2_l += l->v[i] * l->v[i]; v2_r += r->v[i] * r->v[i]; }
    double v2_avg = 0.5 * (v2_l + v2_r);
    f[0] = f_rho;
    double work = 0.0;
    for (int i = 0; i < d; ++i) {
        double va = 0.5 * (l->v[i] + r->v[i]);
        f[1 + i] = f_rho * va + p_tilde * nrm[i];
        work += va * f[1 + i];
    }
    f[d + 1] = f_rho * (0.5 * igm1 * inv_beta_mean - 0.5 * v2_avg) + work;
}

static inline void split_normal(const double *nrm, int d, double *norm, double *unit)
{
    double nn = 0.0;
    for (int i = 0; i < d; ++i) nn += nrm[i] * nrm[i];
    nn = sqrt(nn);
    *norm = nn;
    for (int i = 0; i < d; ++i) unit[i] = nrm[i] / nn;
}

static inline void flux_llf(const node_t *l, const node_t *r, const double *nrm, int d,
                            double gamma, double *f)
{
    double norm, unit[3];
    split_normal(nrm, d, &norm, unit);
    double vn_l = 0.0, vn_r = 0.0;
    for (int i = 0; i < d; ++i) { vn_l += l->v[i] * unit[i]; vn_r += r->v[i] * unit[i]; }
    double lam_l = fabs(vn_l) + sqrt(gamma * l->p / l->rho);
    double lam_r = fabs(vn_r) + sqrt(gamma * r->p / r->rho);
    double lam = (lam_r > lam_l) ? lam_r : lam_l; /* python max(a, b) */
    double fl[5], fr[5];
    phys_flux_n(l, nrm, d, fl);
    phys_flux_n(r, nrm, d, fr);
    double halfdiss = 0.5 * lam * norm;
    for (int v = 0; v < d + 2; ++v) f[v] = 0.5 * (fl[v] + fr[v]) - halfdiss * (r->u[v] - l->u[v]);
}

static inline void flux_hll(const node_t *l, const node_t *r, const double *nrm, int d,
                            double gamma, double *f)
{
    double norm, unit[3];
    split_normal(nrm, d, &norm, unit);
    double vn_l = 0.0, vn_r = 0.0;
    for (int i = 0; i < d; ++i) { vn_l += l->v[i] * unit[i]; vn_r += r->v[i] * unit[i]; }
    double c_l = sqrt(gamma * l->p / l->rho);
    double c_r = sqrt(gamma * r->p / r->rho);
    double a1 = vn_l - c_l, b1 = vn_r - c_r;
    double s_l = (b1 < a1) ? b1 : a1; /* python min */
    double a2 = vn_l + c_l, b2 = vn_r + c_r;
    double s_r = (b2 > a2) ? b2 : a2; /* python max */
    double fl[5], fr[5], g[5];
    phys_flux_n(l, unit, d, fl);
    phys_flux_n(r, unit, d, fr);
    if (s_l >= 0.0) {
        for (int v = 0; v < d + 2; ++v) g[v] = fl[v];
    } else if (s_r <= 0.0) {
        for (int v = 0; v < d + 2; ++v) g[v] = fr[v];
    } else {
        double inv = 1.0 / (s_r - s_l);
        for (int v = 0; v < d + 2; ++v)
            g[v] = (s_r * fl[v] - s_l * fr[v] + s_l * s_r * (r->u[v] - l->u[v])) * inv;
    }
    for (int v = 0; v < d + 2; ++v) f[v] = norm * g[v];
}

static inline void two_point(int flux, int pre, const node_t *l, const node_t *r,
                             const double *nrm, int cart_axis, int d, double gamma, double igm1,
                             double *f)
{
    switch (flux) {
    case F_SHIMA: flux_shima(l, r, nrm, cart_axis, d, igm1, f); break;
    case F_RANOCHA: flux_ranocha(l, r, nrm, cart_axis, d, igm1, pre == PRE_LOGS, f); break;
    case F_CENTRAL: flux_central(l, r, nrm, d, igm1, pre != PRE_NONE, f); break;
    case F_KG: flux_kg(l, r, nrm, cart_axis, d, f); break;
    case F_CHANDRASHEKAR: flux_chandrashekar(l, r, nrm, cart_axis, d, igm1, f); break;
    case F_LLF: flux_llf(l, r, nrm, d, gamma, f); break;
    case F_HLL: flux_hll(l, r, nrm, d, gamma, f); break;
    default: for (int v = 0; v < d + 2; ++v) f[v] = NAN;
    }
}

/* ------------------------------------------------------------ index helpers */

static inline int ipow(int b, int e)
{
    int r = 1;
    while (e-- > 0) r *= b;
    return r;
}

/* node id of position a on line m of direction n (operators.py:248-259) */
static inline int line_node(int d, int p1, int n, int m, int a)
{
    int stride = ipow(p1, d - 1 - n);
    int hi = m / stride, lo = m % stride; /* m enumerates the other axes in C order */
    return (hi * p1 + a) * stride + lo;
}

static inline double jac_of(const or_mesh *M, int64_t e, int i)
{
    int nn = ipow(M->p1, M->d);
    return M->jac ? M->jac[e * nn + i] : M->jac_const;
}

/* ------------------------------------------------------------- volume term */

static void volume_element(const or_mesh *M, int64_t e, const double *u, double *out, int flux,
                           int pre, node_t *q, double *acc)
{
    const int d = M->d, p1 = M->p1, nvar = d + 2, nn = ipow(p1, d), nl = ipow(p1, d - 1);
    const double gm1 = M->gamma - 1.0;
    for (int i = 0; i < nn; ++i) make_node(&q[i], u + (e * nn + i) * nvar, d, gm1, flux, pre);
    for (int i = 0; i < nn * nvar; ++i) acc[i] = 0.0;
    for (int n = 0; n < d; ++n) {
        for (int m = 0; m < nl; ++m) {
            for (int a = 0; a < p1; ++a) {
                for (int b = a + 1; b < p1; ++b) {
                    double cab = M->dsplit[a * p1 + b], cba = M->dsplit[b * p1 + a];
                    if (cab == 0.0 && cba == 0.0) continue; /* pair_table drops all-zero pairs */
                    int i = line_node(d, p1, n, m, a), k = line_node(d, p1, n, m, b);
                    double f[5], wi, wk;
                    if (M->cartesian) {
                        double axis[3] = {0.0, 0.0, 0.0};
                        axis[n] = 1.0;
                        two_point(flux, pre, &q[i], &q[k], axis, n, d, M->gamma, M->igm1, f);
                        wi = cab * M->areas[n];
                        wk = cba * M->areas[n];
                    } else {
                        const double *ji = M->ja + ((e * nn + i) * d + n) * d;
                        const double *jk = M->ja + ((e * nn + k) * d + n) * d;
                        double alpha[3];
                        for (int j = 0; j < d; ++j) alpha[j] = 0.5 * (ji[j] + jk[j]);
                        two_point(flux, pre, &q[i], &q[k], alpha, -1, d, M->gamma, M->igm1, f);
                        wi = cab;
                        wk = cba;
                    }
                    for (int v = 0; v < nvar; ++v) {
                        acc[i * nvar + v] += wi * f[v];
                        acc[k * nvar + v] += wk * f[v];
                    }
                }
            }
        }
    }
    for (int i = 0; i < nn; ++i) {
        double J = jac_of(M, e, i);
        for (int v = 0; v < nvar; ++v) out[(e * nn + i) * nvar + v] = acc[i * nvar + v] / J;
    }
}

/* ------------------------------------------------------------ surface term */

static void face_normal(const or_mesh *M, int64_t owner, int n, int m, double *nrm)
{
    /* face_ja[n][owner, m] = owner's own Ja^n at its +face node (geometry.py:311-326) */
    const int d = M->d, p1 = M->p1, nn = ipow(p1, d);
    if (M->cartesian) {
        for (int j = 0; j < d; ++j) nrm[j] = (j == n) ? M->areas[n] : 0.0;
    } else if (owner < 0) {
        const double *g = M->ghost_nrm + ((-owner - 1) * ipow(p1, d - 1) + m) * d;
        for (int j = 0; j < d; ++j) nrm[j] = g[j];
    } else {
        int node = line_node(d, p1, n, m, p1 - 1);
        const double *src = M->ja + ((owner * nn + node) * d + n) * d;
        for (int j = 0; j < d; ++j) nrm[j] = src[j];
    }
}

static void face_state(const or_mesh *M, const double *u, int64_t elem, int n, int m, int pos,
                       double *s)
{
    const int d = M->d, p1 = M->p1, nvar = d + 2, nn = ipow(p1, d);
    const double *src;
    if (elem < 0) src = M->ghost_u + ((-elem - 1) * ipow(p1, d - 1) + m) * nvar;
    else src = u + (elem * nn + line_node(d, p1, n, m, pos)) * nvar;
    for (int v = 0; v < nvar; ++v) s[v] = src[v];
}

static void surface_element(const or_mesh *M, int64_t e, const double *u, double *out, int flux)
{
    const int d = M->d, p1 = M->p1, nvar = d + 2, nn = ipow(p1, d), fn = ipow(p1, d - 1);
    const double gm1 = M->gamma - 1.0;
    const double wm = M->weights[p1 - 1], wp = M->weights[0];
    for (int n = 0; n < d; ++n) {
        int64_t nb_p = M->plus[n * M->n_elem + e];
        int64_t nb_m = M->minus[n * M->n_elem + e];
        for (int m = 0; m < fn; ++m) {
            double sl[5], sr[5], nrm[3], f[5];
            node_t ql, qr;
            /* +n face of e: e is the minus element */
            int im = line_node(d, p1, n, m, p1 - 1);
            face_state(M, u, e, n, m, p1 - 1, sl);
            face_state(M, u, nb_p, n, m, 0, sr);
            face_normal(M, e, n, m, nrm);
            make_node(&ql, sl, d, gm1, F_CENTRAL, PRE_NONE);
            make_node(&qr, sr, d, gm1, F_CENTRAL, PRE_NONE);
            two_point(flux, PRE_NONE, &ql, &qr, nrm, -1, d, M->gamma, M->igm1, f);
            double sm = 1.0 / (wm * jac_of(M, e, im));
            for (int v = 0; v < nvar; ++v) out[(e * nn + im) * nvar + v] += sm * f[v];
            /* -n face of e: e is the plus element */
            int ip = line_node(d, p1, n, m, 0);
            face_state(M, u, nb_m, n, m, p1 - 1, sl);
            face_state(M, u, e, n, m, 0, sr);
            face_normal(M, nb_m, n, m, nrm);
            make_node(&ql, sl, d, gm1, F_CENTRAL, PRE_NONE);
            make_node(&qr, sr, d, gm1, F_CENTRAL, PRE_NONE);
            two_point(flux, PRE_NONE, &ql, &qr, nrm, -1, d, M->gamma, M->igm1, f);
            double sp = 1.0 / (wp * jac_of(M, e, ip));
            for (int v = 0; v < nvar; ++v) out[(e * nn + ip) * nvar + v] -= sp * f[v];
        }
    }
}

/* ------------------------------------------------------------- public API */

/* static element partition over pthreads (the reference is single-threaded;
 * elements are independent in both passes, so this changes no bits)        */
typedef struct {
    const or_mesh *M;
    const double *u;
    double *out;
    int flux, pre, what; /* what: 0 volume, 1 surface, 2 negate */
    int64_t lo, hi;
} job_t;

static void *run_job(void *arg)
{
    job_t *j = (job_t *)arg;
    const int nn = ipow(j->M->p1, j->M->d), nvar = j->M->d + 2;
    if (j->what == 0) {
        node_t *q = (node_t *)malloc(sizeof(node_t) * nn);
        double *acc = (double *)malloc(sizeof(double) * nn * nvar);
        for (int64_t e = j->lo; e < j->hi; ++e) volume_element(j->M, e, j->u, j->out, j->flux, j->pre, q, acc);
        free(q);
        free(acc);
    } else if (j->what == 1) {
        for (int64_t e = j->lo; e < j->hi; ++e) surface_element(j->M, e, j->u, j->out, j->flux);
    } else {
        for (int64_t i = j->lo * nn * nvar; i < j->hi * nn * nvar; ++i) j->out[i] = -j->out[i];
    }
    return NULL;
}

int or_max_threads(void)
{
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

static void run_parallel_range(const or_mesh *M, const double *u, double *out, int flux, int pre,
                               int what, int64_t lo, int64_t hi, int nthreads)
{
    const int64_t n = hi - lo;
    if (n <= 0) return;
    if (nthreads <= 0) nthreads = or_max_threads();
    if (nthreads > 256) nthreads = 256;
    if ((int64_t)nthreads > n) nthreads = (int)n;
    job_t jobs[256];
    pthread_t tids[256];
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].M = M; jobs[t].u = u; jobs[t].out = out;
        jobs[t].flux = flux; jobs[t].pre = pre; jobs[t].what = what;
        jobs[t].lo = lo + n * t / nthreads;
        jobs[t].hi = lo + n * (t + 1) / nthreads;
    }
    if (nthreads == 1) { run_job(&jobs[0]); return; }
    for (int t = 0; t < nthreads; ++t) pthread_create(&tids[t], NULL, run_job, &jobs[t]);
    for (int t = 0; t < nthreads; ++t) pthread_join(tids[t], NULL);
}

static void run_parallel(const or_mesh *M, const double *u, double *out, int flux, int pre,
                         int what, int nthreads)
{
    run_parallel_range(M, u, out, flux, pre, what, 0, M->n_elem, nthreads);
}

/* VOL (already / J), discretization.py:267-323 applied to every element */
int or_volume(const or_mesh *M, const double *u, double *vol, int flux, int pre, int nthreads)
{
    run_parallel(M, u, vol, flux, pre, 0, nthreads);
    return 0;
}

/* out += SURF (discretization.py:681-760); out holds VOL or zeros */
int or_surface(const or_mesh *M, const double *u, double *out, int flux, int nthreads)
{
    run_parallel(M, u, out, flux, 0, 1, nthreads);
    return 0;
}

/* first inadmissible node in C order, or -1 (discretization.py:660-672);
 * rho/p of that node are returned with the gate's own pressure formula.    */
int64_t or_gate(const or_mesh *M, const double *u, double *rho_out, double *p_out)
{
    const int d = M->d, nvar = d + 2, nn = ipow(M->p1, d);
    const int64_t total = M->n_elem * nn;
    for (int64_t g = 0; g < total; ++g) {
        const double *s = u + g * nvar;
        double rho = s[0];
        double mm = s[1] * s[1] + s[2] * s[2];
        if (d == 3) mm = mm + s[3] * s[3];
        double p = (M->gamma - 1.0) * (s[d + 1] - 0.5 * mm / rho);
        if (!((rho > 0.0) && (p > 0.0) && isfinite(rho) && isfinite(p))) {
            if (rho_out) *rho_out = rho;
            if (p_out) *p_out = p;
            return g;
        }
    }
    return -1;
}

/* du = -(VOL + SURF) as rhs(kernel="reference") does (discretization.py:932-949).
 * Returns -1 on success or the flat index of the first inadmissible node.  */
int64_t or_rhs(const or_mesh *M, const double *u, double *du, int vflux, int sflux, int pre,
               int nthreads)
{
    int64_t bad = or_gate(M, u, NULL, NULL);
    if (bad >= 0) return bad;
    or_volume(M, u, du, vflux, pre, nthreads);
    or_surface(M, u, du, sflux, nthreads);
    run_parallel(M, u, du, 0, 0, 2, nthreads);
    return -1;
}

/* rows [lo, hi) of or_rhs (no gate): the interior / boundary split of a slab
 * partition -- interior rows never read ghost_u, which may still be NULL    */
int or_rhs_range(const or_mesh *M, const double *u, double *du, int vflux, int sflux, int pre,
                 int64_t lo, int64_t hi, int nthreads)
{
    run_parallel_range(M, u, du, vflux, pre, 0, lo, hi, nthreads);
    run_parallel_range(M, u, du, sflux, 0, 1, lo, hi, nthreads);
    run_parallel_range(M, u, du, 0, 0, 2, lo, hi, nthreads);
    return 0;
}

/* ------------------------------------------------ Gauss-family schemes
 * Restatement of the reference's scalar gauss path (discretization.py:375-443
 * _gauss_line_terms with include_corner=False as rhs uses it, :966-995
 * _scalar_gauss_volume, :839-895 _gauss_surface, :985-995 assembly):
 * zero-corner hybridized volume term on Gauss nodes with entropy-projected
 * face states, then the interface fluxes of the projected states lifted
 * through the dense boundary rows, then -(acc / J). The projection itself
 * (entropy variables, boundary interpolation, entropy2cons) is numpy in
 * oracle.py, as in the reference. Tables (operators.py:300-357):
 *   vv[a*p1+b]   volume pair weight c_ab (pairs a < b, both-zero pairs skipped)
 *   cvol[s*p1+a] volume-row weight of the (a, face s) crossing
 *   cface[s*p1+a] face-row weight of the crossing
 *   lift[s*p1+a] R[s][a] / w[a]  (side 1: lift_m, side 0: lift_p)
 * proj (n_elem, d, 2, fn, nvar) projected face states; nrm (n_elem, d, 2, fn, d)
 * each element's own face metric traces (the volume crossings); fnrm
 * (n_elem, d, fn, d) the interface normals face_ja (NULL: nrm side 1).     */
typedef struct {
    const double *vv, *cvol, *cface, *lift;
} or_gauss_tables;

static void gauss_element(const or_mesh *M, const or_gauss_tables *T, int64_t e, const double *u,
                          const double *proj, const double *nrm, const double *fnrm, double *du, int vflux,
                          int sflux, node_t *q, double *acc)
{
    const int d = M->d, p1 = M->p1, nvar = d + 2, nn = ipow(p1, d), fn = ipow(p1, d - 1);
    const double gm1 = M->gamma - 1.0;
    for (int i = 0; i < nn; ++i) make_node(&q[i], u + (e * nn + i) * nvar, d, gm1, vflux, PRE_NONE);
    for (int i = 0; i < nn * nvar; ++i) acc[i] = 0.0;
    const double *ja = M->ja + e * nn * d * d;
    double f[5], alpha[3];
    for (int n = 0; n < d; ++n) {
        for (int m = 0; m < fn; ++m) {
            for (int a = 0; a < p1; ++a)
                for (int b = a + 1; b < p1; ++b) {
                    const double cab = T->vv[a * p1 + b], cba = T->vv[b * p1 + a];
                    if (cab == 0.0 && cba == 0.0) continue;
                    const int i = line_node(d, p1, n, m, a), k = line_node(d, p1, n, m, b);
                    for (int j = 0; j < d; ++j) alpha[j] = 0.5 * (ja[(i * d + n) * d + j] + ja[(k * d + n) * d + j]);
                    two_point(vflux, PRE_NONE, &q[i], &q[k], alpha, -1, d, M->gamma, M->igm1, f);
                    for (int v = 0; v < nvar; ++v) {
                        acc[i * nvar + v] += cab * f[v];
                        acc[k * nvar + v] += cba * f[v];
                    }
                }
            for (int s = 0; s < 2; ++s) {
                const double *fs = proj + ((((e * d + n) * 2 + s) * fn) + m) * nvar;
                const double *fj = nrm + ((((e * d + n) * 2 + s) * fn) + m) * d;
                node_t fq;
                make_node(&fq, fs, d, gm1, vflux, PRE_NONE);
                double rface[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
                for (int a = 0; a < p1; ++a) {
                    const int i = line_node(d, p1, n, m, a);
                    for (int j = 0; j < d; ++j) alpha[j] = 0.5 * (ja[(i * d + n) * d + j] + fj[j]);
                    two_point(vflux, PRE_NONE, &q[i], &fq, alpha, -1, d, M->gamma, M->igm1, f);
                    const double ca = T->cvol[s * p1 + a], cf = T->cface[s * p1 + a];
                    for (int v = 0; v < nvar; ++v) {
                        acc[i * nvar + v] += ca * f[v];
                        rface[v] += cf * f[v];
                    }
                }
                for (int a = 0; a < p1; ++a) {
                    const double la = T->lift[s * p1 + a];
                    if (la == 0.0) continue;
                    const int i = line_node(d, p1, n, m, a);
                    for (int v = 0; v < nvar; ++v) acc[i * nvar + v] += la * rface[v];
                }
            }
        }
    }
    /* interfaces: as minus element (+= lift_m F) of face (e, +n) and as plus
     * element (-= lift_p F) of face (minus(e), +n), in the reference's face
     * loop order (faces ascending) */
    for (int n = 0; n < d; ++n) {
        const int64_t ep = M->plus[n * M->n_elem + e], em = M->minus[n * M->n_elem + e];
        for (int pass = 0; pass < 2; ++pass) {
            const int as_plus = (em < e) ? (pass == 0) : (pass == 1);
            const int64_t owner = as_plus ? em : e, other = as_plus ? e : ep;
            for (int m = 0; m < fn; ++m) {
                const double *ul = proj + ((((owner * d + n) * 2 + 1) * fn) + m) * nvar;
                const double *ur = proj + ((((other * d + n) * 2 + 0) * fn) + m) * nvar;
                const double *nr = fnrm ? fnrm + (((owner * d + n) * fn) + m) * d
                                        : nrm + ((((owner * d + n) * 2 + 1) * fn) + m) * d;
                node_t l, r;
                make_node(&l, ul, d, gm1, sflux, PRE_NONE);
                make_node(&r, ur, d, gm1, sflux, PRE_NONE);
                two_point(sflux, PRE_NONE, &l, &r, nr, -1, d, M->gamma, M->igm1, f);
                for (int a = 0; a < p1; ++a) {
                    const double la = T->lift[(as_plus ? 0 : 1) * p1 + a];
                    if (la == 0.0) continue;
                    const int i = line_node(d, p1, n, m, a);
                    for (int v = 0; v < nvar; ++v) {
                        if (as_plus) acc[i * nvar + v] -= la * f[v];
                        else acc[i * nvar + v] += la * f[v];
                    }
                }
            }
        }
    }
    for (int i = 0; i < nn; ++i) {
        const double J = M->jac[e * nn + i];
        for (int v = 0; v < nvar; ++v) {
            const double t = acc[i * nvar + v] / J;
            du[(e * nn + i) * nvar + v] = -t;
        }
    }
}

int or_gauss_rhs(const or_mesh *M, const or_gauss_tables *T, const double *u, const double *proj,
                 const double *nrm, const double *fnrm, double *du, int vflux, int sflux)
{
    const int nn = ipow(M->p1, M->d), nvar = M->d + 2;
    node_t *q = (node_t *)malloc(sizeof(node_t) * nn);
    double *acc = (double *)malloc(sizeof(double) * nn * nvar);
    for (int64_t e = 0; e < M->n_elem; ++e) gauss_element(M, T, e, u, proj, nrm, fnrm, du, vflux, sflux, q, acc);
    free(q);
    free(acc);
    return 0;
}

/* single two-point flux evaluation (conserved input), for property tests */
int or_two_point(int d, int flux, int pre, double gamma, double igm1, const double *ul,
                 const double *ur, const double *nrm, int cart_axis, double *f)
{
    node_t l, r;
    make_node(&l, ul, d, gamma - 1.0, flux, pre);
    make_node(&r, ur, d, gamma - 1.0, flux, pre);
    two_point(flux, pre, &l, &r, nrm, cart_axis, d, gamma, igm1, f);
    return 0;
}

/* scalar log means, exposed for the mpmath-free known-answer tests */
double or_logmean(double a, double b) { return logmean(a, b); }
double or_inv_logmean(double a, double b) { return inv_logmean(a, b); }

/* per-node primitive/extra values exactly as the kernels above see them */
int or_node(const double *u, int d, double gamma, int flux, int pre, double *out)
{
    node_t q;
    make_node(&q, u, d, gamma - 1.0, flux, pre);
    out[0] = q.rho;
    for (int i = 0; i < 3; ++i) out[1 + i] = q.v[i];
    out[4] = q.p;
    out[5] = q.x0;
    out[6] = q.x1;
    return 0;
}

/* the log this build uses (glibc log, or log_cr with -DFDG_ORACLE_LOGCR) */
double or_log(double x) { return OR_LOG(x); }
