// fdg_gauss.cu -- the Gauss-node family of the paper: the
// zero-corner hybridized flux-differencing volume term with entropy-projected
// face states and its interface coupling, on device.
//
// Reference (all /root/reference/pkg/src/fluxdg):
//   _project_all            discretization.py:811-837  (entropy variables ->
//                           boundary interpolation per line -> entropy2cons)
//   _gauss_line_terms       discretization.py:375-443  (include_corner=False in rhs)
//   _scalar_gauss_volume    discretization.py:966-995
//   _gauss_surface          discretization.py:839-895  (each face flux once per
//                           adjacent element, lifted through the dense R rows)
//   rhs gauss branch        discretization.py:976-995  (-(acc / J))
//   mesh_gauss_volume / mesh_gauss_surface  batched.py:556-667 (same math, lanes)
//   hybridized_scatter / skew_pair_table    operators.py:300-357 (tables, host)
//
// Two kernels per RHS:
//   gauss_project_kernel  one CTA per element: entropy variables of every node
//                         in shared memory, then one thread per (direction,
//                         side, face node) interpolates them to the face
//                         (R row), converts back (entropy2cons) and writes the
//                         projected state; the element's own face metric
//                         traces (the crossing normals) likewise.
//   gauss_rhs_kernel      one CTA per EPB elements, one thread per 1D line:
//                         volume pairs, the two face crossings and the lift of
//                         the face rows, direction by direction in the scalar
//                         path's per-node order (accumulators carried in shared
//                         memory across directions); then the interface
//                         fluxes of the projected states (plus face and minus
//                         face of each line) lifted into every node of the
//                         line, in the reference's face-loop order; -(acc/J).
// Compiled with --fmad=false and the FAITHFUL flux functions: with the
// projection given, the RHS is bitwise the C oracle's restatement
// (oracle/fdg_oracle.c or_gauss_rhs, itself bitwise the reference's scalar
// path); the projection uses the correctly rounded log and CUDA exp and
// agrees with numpy's to a few ulps.
#include <algorithm>
#include <cstdio>
#include <cstring>

#include "../../include/fdg.h"
#include "fdg_kernels.cuh"

namespace fdg {

struct GParams {
    const double* u;
    double* out;
    const double* proj;  // (n_elem, D, 2, FN, NVAR) projected face states
    double* proj_out;
    const double* nrm;   // (n_elem, D, 2, FN, D) own face metric traces
    double* nrm_out;
    const double* fnrm;  // (n_elem, D, FN, D) interface normals, or null (nrm side 1)
    const double* ja;    // (n_elem, NN, D, D)
    const double* jac;   // (n_elem, NN)
    const int* plus;
    const int* minus;
    Status* status;  // first_bad: gate; bad_stage: first failing (direction * 2 + side) of the projection
    long long n_elem;
    double vv[64];      // pair weights c_ab (row a, column b)
    double cvol[2][8];  // crossing weights into the volume row
    double cface[2][8]; // crossing weights into the face row
    double lift[2][8];  // R[s][a] / w[a]
    double R[2][8];     // boundary interpolation rows
    Gas gas;
    int surface_flux;
};

template <int D, int P1>
struct GGeo {
    static constexpr int NN = ipow(P1, D);
    static constexpr int FN = ipow(P1, D - 1);
    static constexpr int NVAR = D + 2;
    __device__ static __forceinline__ int line_node(int n, int m, int a)
    {
        const int stride = n == D - 1 ? 1 : (n == D - 2 ? P1 : P1 * P1);
        return (m / stride * P1 + a) * stride + m % stride;
    }
};

// ---------------------------------------------------------------- projection

template <int D, int P1>
__global__ void __launch_bounds__(128) gauss_project_kernel(const __grid_constant__ GParams prm)
{
    using G = GGeo<D, P1>;
    constexpr int NN = G::NN, FN = G::FN, NVAR = G::NVAR;
    __shared__ double sw[NN * NVAR];
    const double g = prm.gas.gamma, gm1 = prm.gas.gm1;
    for (long long e = blockIdx.x; e < prm.n_elem; e += gridDim.x) {
        // entropy variables (euler.py:129-146, operation order kept)
        for (int i = threadIdx.x; i < NN; i += blockDim.x) {
            const double* s = prm.u + (e * NN + i) * NVAR;
            const double rho = s[0];
            double v[D], vv = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) v[k] = s[1 + k] / rho;
            vv = v[0] * v[0];
#pragma unroll
            for (int k = 1; k < D; ++k) vv = vv + v[k] * v[k];
            const double p = gm1 * (s[D + 1] - 0.5 * rho * vv);
            const double ent = log_cr(p) - g * log_cr(rho);
            const double rp = rho / p;
            sw[i * NVAR] = (g - ent) * prm.gas.igm1 - 0.5 * rp * vv;
#pragma unroll
            for (int k = 0; k < D; ++k) sw[i * NVAR + 1 + k] = rp * v[k];
            sw[i * NVAR + D + 1] = -rp;
        }
        __syncthreads();
        // face states: one thread per (direction, side, face node)
        for (int it = threadIdx.x; it < D * 2 * FN; it += blockDim.x) {
            const int n = it / (2 * FN), side = (it / FN) % 2, m = it % FN;
            double wf[NVAR];
#pragma unroll
            for (int v = 0; v < NVAR; ++v) wf[v] = 0.0;
            for (int k = 0; k < P1; ++k) {
                const double r = prm.R[side][k];
                const int node = G::line_node(n, m, k);
#pragma unroll
                for (int v = 0; v < NVAR; ++v) wf[v] += r * sw[node * NVAR + v];
            }
            // entropy2cons (euler.py:149-170)
            const double b = -wf[D + 1];
            if (!(b > 0.0)) atomicMin(&prm.status->bad_stage, (unsigned)(n * 2 + side));
            double v[D], vv;
#pragma unroll
            for (int k = 0; k < D; ++k) v[k] = wf[1 + k] / b;
            vv = v[0] * v[0];
#pragma unroll
            for (int k = 1; k < D; ++k) vv = vv + v[k] * v[k];
            const double ent = g - gm1 * (wf[0] + 0.5 * b * vv);
            const double p = exp((ent + g * log_cr(b)) / (1.0 - g));
            const double rho = b * p;
            double* o = prm.proj_out + (((e * D + n) * 2 + side) * FN + m) * NVAR;
            o[0] = rho;
#pragma unroll
            for (int k = 0; k < D; ++k) o[1 + k] = rho * v[k];
            o[D + 1] = p * prm.gas.igm1 + 0.5 * rho * vv;
        }
        // the element's own metric traces at both faces of every line
        for (int it = threadIdx.x; it < D * 2 * FN * D; it += blockDim.x) {
            const int j = it % D, r0 = it / D;
            const int n = r0 / (2 * FN), side = (r0 / FN) % 2, m = r0 % FN;
            double acc = 0.0;
            for (int k = 0; k < P1; ++k) {
                const int node = G::line_node(n, m, k);
                acc += prm.R[side][k] * __ldg(prm.ja + ((e * NN + node) * D + n) * D + j);
            }
            prm.nrm_out[(((e * D + n) * 2 + side) * FN + m) * D + j] = acc;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------- RHS

template <int D, int P1, int VF>
__global__ void __launch_bounds__(64) gauss_rhs_kernel(const __grid_constant__ GParams prm)
{
    using G = GGeo<D, P1>;
    constexpr int NN = G::NN, FN = G::FN, NVAR = G::NVAR;
    constexpr int EPB = FN >= 64 ? 1 : 64 / FN;
    constexpr int NX = n_extra(VF, 0);
    extern __shared__ double gsm[];
    double* su = gsm;                    // (EPB, NN, NVAR) conserved state
    double* sacc = gsm + EPB * NN * NVAR;  // (EPB, NN, NVAR) accumulators
    const int el = threadIdx.x / FN, m = threadIdx.x % FN;
    const double gm1 = prm.gas.gm1;
    const long long nbatch = (prm.n_elem + EPB - 1) / EPB;
    for (long long batch = blockIdx.x; batch < nbatch; batch += gridDim.x) {
        const long long e0 = batch * EPB;
        const int ne = (int)min((long long)EPB, prm.n_elem - e0);
        for (int t = threadIdx.x; t < ne * NN * NVAR; t += blockDim.x) {
            su[t] = __ldg(prm.u + e0 * NN * NVAR + t);
            sacc[t] = 0.0;
        }
        __syncthreads();
        const bool active = el < ne;
        const long long e = e0 + el;
        // ---- volume: pairs, the two face crossings, the lifted face rows
        for (int n = 0; n < D; ++n) {
            if (active) {
                double acc[P1][NVAR];
                int nodes[P1];
#pragma unroll
                for (int a = 0; a < P1; ++a) {
                    nodes[a] = G::line_node(n, m, a);
#pragma unroll
                    for (int v = 0; v < NVAR; ++v) acc[a][v] = sacc[(el * NN + nodes[a]) * NVAR + v];
                }
                double jn[P1][D];
#pragma unroll
                for (int a = 0; a < P1; ++a)
#pragma unroll
                    for (int j = 0; j < D; ++j) jn[a][j] = __ldg(prm.ja + ((e * NN + nodes[a]) * D + n) * D + j);
                double f[NVAR], alpha[D];
#pragma unroll
                for (int a = 0; a < P1; ++a) {
                    const Node<D, NX> qa = make_node<D, VF, FAITHFUL, 0>(su + (el * NN + nodes[a]) * NVAR, gm1);
#pragma unroll
                    for (int b = a + 1; b < P1; ++b) {
                        const double cab = prm.vv[a * P1 + b], cba = prm.vv[b * P1 + a];
                        if (cab == 0.0 && cba == 0.0) continue;
                        const Node<D, NX> qb = make_node<D, VF, FAITHFUL, 0>(su + (el * NN + nodes[b]) * NVAR, gm1);
#pragma unroll
                        for (int j = 0; j < D; ++j) alpha[j] = 0.5 * (jn[a][j] + jn[b][j]);
                        volume_flux<D, VF, -1, FAITHFUL, 0>(qa, qb, alpha, prm.gas, PRE_NONE, f, 0u);
#pragma unroll
                        for (int v = 0; v < NVAR; ++v) {
                            acc[a][v] += cab * f[v];
                            acc[b][v] += cba * f[v];
                        }
                    }
                }
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const double* fs = prm.proj + (((e * D + n) * 2 + s) * FN + m) * NVAR;
                    const double* fj = prm.nrm + (((e * D + n) * 2 + s) * FN + m) * D;
                    double fsv[NVAR], fjv[D];
#pragma unroll
                    for (int v = 0; v < NVAR; ++v) fsv[v] = __ldg(fs + v);
#pragma unroll
                    for (int j = 0; j < D; ++j) fjv[j] = __ldg(fj + j);
                    const Node<D, NX> fq = make_node<D, VF, FAITHFUL, 0>(fsv, gm1);
                    double rface[NVAR];
#pragma unroll
                    for (int v = 0; v < NVAR; ++v) rface[v] = 0.0;
#pragma unroll
                    for (int a = 0; a < P1; ++a) {
                        const Node<D, NX> qa = make_node<D, VF, FAITHFUL, 0>(su + (el * NN + nodes[a]) * NVAR, gm1);
#pragma unroll
                        for (int j = 0; j < D; ++j) alpha[j] = 0.5 * (jn[a][j] + fjv[j]);
                        volume_flux<D, VF, -1, FAITHFUL, 0>(qa, fq, alpha, prm.gas, PRE_NONE, f, 0u);
                        const double ca = prm.cvol[s][a], cf = prm.cface[s][a];
#pragma unroll
                        for (int v = 0; v < NVAR; ++v) {
                            acc[a][v] += ca * f[v];
                            rface[v] += cf * f[v];
                        }
                    }
#pragma unroll
                    for (int a = 0; a < P1; ++a) {
                        const double la = prm.lift[s][a];
                        if (la == 0.0) continue;
#pragma unroll
                        for (int v = 0; v < NVAR; ++v) acc[a][v] += la * rface[v];
                    }
                }
#pragma unroll
                for (int a = 0; a < P1; ++a)
#pragma unroll
                    for (int v = 0; v < NVAR; ++v) sacc[(el * NN + nodes[a]) * NVAR + v] = acc[a][v];
            }
            __syncthreads();
        }
        // ---- interfaces: as minus element of face (e, +n): += lift_m F; as
        // plus element of face (minus(e), +n): -= lift_p F; faces in the
        // reference's loop order (ascending face index)
        for (int n = 0; n < D; ++n) {
            if (active) {
                const long long ep = __ldg(prm.plus + n * prm.n_elem + e);
                const long long em = __ldg(prm.minus + n * prm.n_elem + e);
#pragma unroll 1
                for (int pass = 0; pass < 2; ++pass) {
                    const bool as_plus = (em < e) ? (pass == 0) : (pass == 1);
                    const long long owner = as_plus ? em : e, other = as_plus ? e : ep;
                    double ul[NVAR], ur[NVAR], nr[D], f[NVAR];
                    const double* pl = prm.proj + (((owner * D + n) * 2 + 1) * FN + m) * NVAR;
                    const double* pr = prm.proj + (((other * D + n) * 2 + 0) * FN + m) * NVAR;
#pragma unroll
                    for (int v = 0; v < NVAR; ++v) {
                        ul[v] = __ldg(pl + v);
                        ur[v] = __ldg(pr + v);
                    }
                    const double* pn = prm.fnrm ? prm.fnrm + ((owner * D + n) * FN + m) * D
                                                : prm.nrm + (((owner * D + n) * 2 + 1) * FN + m) * D;
#pragma unroll
                    for (int j = 0; j < D; ++j) nr[j] = __ldg(pn + j);
                    surface_flux<D, FAITHFUL>(prm.surface_flux, ul, ur, nr, prm.gas, f);
                    const int s = as_plus ? 0 : 1;
#pragma unroll
                    for (int a = 0; a < P1; ++a) {
                        const double la = prm.lift[s][a];
                        if (la == 0.0) continue;
                        double* r = sacc + (el * NN + G::line_node(n, m, a)) * NVAR;
#pragma unroll
                        for (int v = 0; v < NVAR; ++v) {
                            if (as_plus) r[v] -= la * f[v];
                            else r[v] += la * f[v];
                        }
                    }
                }
            }
            __syncthreads();
        }
        // ---- du = -(acc / J)
        for (int t = threadIdx.x; t < ne * NN * NVAR; t += blockDim.x) {
            const int node = t / NVAR;  // element-major within the batch
            const double J = __ldg(prm.jac + e0 * NN + node);
            const double q = sacc[t] / J;
            prm.out[e0 * NN * NVAR + t] = -q;
        }
        __syncthreads();
    }
}

template <int D>
__global__ void gauss_gate_kernel(const double* __restrict__ u, long long n_nodes, double gm1, Status* status)
{
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n_nodes;
         t += (long long)gridDim.x * blockDim.x)
        if (!gate_ok<D>(u + t * (D + 2), gm1)) atomicMin(&status->first_bad, (unsigned long long)t);
}

template <int D, int P1>
size_t gauss_rhs_smem()
{
    using G = GGeo<D, P1>;
    constexpr int EPB = G::FN >= 64 ? 1 : 64 / G::FN;
    return sizeof(double) * 2 * EPB * G::NN * G::NVAR;
}

template <int D, int P1, int VF>
cudaError_t launch_gauss_rhs(const GParams& p, cudaStream_t s, int sm_count)
{
    using G = GGeo<D, P1>;
    constexpr int EPB = G::FN >= 64 ? 1 : 64 / G::FN;
    const size_t smem = gauss_rhs_smem<D, P1>();
    auto kern = gauss_rhs_kernel<D, P1, VF>;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    const long long nb = (p.n_elem + EPB - 1) / EPB;
    const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>(nb, (long long)sm_count * 16));
    kern<<<grid, EPB * G::FN, smem, s>>>(p);
    return cudaGetLastError();
}

template <int D, int P1>
cudaError_t launch_gauss(const GParams& p, int vf, bool project, cudaStream_t s, int sm_count)
{
    if (project) {
        const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>(p.n_elem, (long long)sm_count * 8));
        gauss_project_kernel<D, P1><<<grid, 128, 0, s>>>(p);
        return cudaGetLastError();
    }
    switch (vf) {
    case F_CENTRAL: return launch_gauss_rhs<D, P1, F_CENTRAL>(p, s, sm_count);
    case F_SHIMA: return launch_gauss_rhs<D, P1, F_SHIMA>(p, s, sm_count);
    case F_RANOCHA: return launch_gauss_rhs<D, P1, F_RANOCHA>(p, s, sm_count);
    case F_KG: return launch_gauss_rhs<D, P1, F_KG>(p, s, sm_count);
    case F_CHANDRASHEKAR: return launch_gauss_rhs<D, P1, F_CHANDRASHEKAR>(p, s, sm_count);
    default: return cudaErrorInvalidValue;
    }
}

using GaussFn = cudaError_t (*)(const GParams&, int, bool, cudaStream_t, int);

static GaussFn gauss_fn(int d, int p1)
{
    static const GaussFn t2[] = {launch_gauss<2, 2>, launch_gauss<2, 3>, launch_gauss<2, 4>, launch_gauss<2, 5>,
                                 launch_gauss<2, 6>, launch_gauss<2, 7>, launch_gauss<2, 8>};
    static const GaussFn t3[] = {launch_gauss<3, 2>, launch_gauss<3, 3>, launch_gauss<3, 4>, launch_gauss<3, 5>,
                                 launch_gauss<3, 6>};
    if (d == 2 && p1 >= 2 && p1 <= 8) return t2[p1 - 2];
    if (d == 3 && p1 >= 2 && p1 <= 6) return t3[p1 - 2];
    return nullptr;
}

}  // namespace fdg

using namespace fdg;

struct fdg_gauss {
    int d = 0, p1 = 0, sm_count = 148;
    long long n_elem = 0;
    GParams base{};
    Status* status = nullptr;
    Status* status_host = nullptr;
    double* proj = nullptr;  // library-owned projection / trace scratch (allocated at creation)
    double* nrm = nullptr;
};

extern "C" int fdg_internal_fail(int rc, const char* msg);  // fdg_capi.cu: sets fdg_last_error

static int gfail(int rc, const char* what, cudaError_t err = cudaSuccess)
{
    char buf[320];
    if (err != cudaSuccess) snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(err));
    else snprintf(buf, sizeof(buf), "%s", what);
    return fdg_internal_fail(rc, buf);
}

extern "C" {

int fdg_gauss_create(const fdg_gauss_desc_t* desc, fdg_gauss_t** out)
{
    if (!desc || !out) return gfail(FDG_ERR_ARG, "fdg_gauss_create: null argument");
    *out = nullptr;
    const int p1 = desc->degree + 1;
    if (!gauss_fn(desc->d, p1))
        return gfail(FDG_ERR_UNSUPPORTED, "gauss family on the device: d = 2 with p <= 7, d = 3 with p <= 5");
    if (!desc->vv || !desc->cvol || !desc->cface || !desc->lift || !desc->boundary_interp)
        return gfail(FDG_ERR_ARG, "fdg_gauss_create: operator tables are required");
    if (!desc->ja || !desc->jac || !desc->plus || !desc->minus)
        return gfail(FDG_ERR_ARG, "fdg_gauss_create: device metrics and neighbour tables are required");
    fdg_gauss* g = new fdg_gauss();
    g->d = desc->d;
    g->p1 = p1;
    g->n_elem = desc->n_elem;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g->sm_count, cudaDevAttrMultiProcessorCount, dev);
    GParams& k = g->base;
    memset(&k, 0, sizeof(k));
    for (int i = 0; i < p1 * p1; ++i) k.vv[i] = desc->vv[i];
    for (int s = 0; s < 2; ++s)
        for (int a = 0; a < p1; ++a) {
            k.cvol[s][a] = desc->cvol[s * p1 + a];
            k.cface[s][a] = desc->cface[s * p1 + a];
            k.lift[s][a] = desc->lift[s * p1 + a];
            k.R[s][a] = desc->boundary_interp[s * p1 + a];
        }
    k.gas.gamma = desc->gamma;
    k.gas.gm1 = desc->gamma - 1.0;
    k.gas.igm1 = desc->inv_gamma_minus_one;
    k.ja = desc->ja;
    k.jac = desc->jac;
    k.plus = desc->plus;
    k.minus = desc->minus;
    k.n_elem = desc->n_elem;
    long long fn = 1;
    for (int i = 0; i < g->d - 1; ++i) fn *= p1;
    const size_t n_proj = (size_t)desc->n_elem * g->d * 2 * fn * (g->d + 2);
    const size_t n_nrm = (size_t)desc->n_elem * g->d * 2 * fn * g->d;
    cudaError_t err = cudaMalloc(&g->status, sizeof(Status));
    if (err == cudaSuccess) err = cudaMemset(g->status, 0xff, sizeof(Status));
    if (err == cudaSuccess) err = cudaMallocHost(&g->status_host, sizeof(Status));
    if (err == cudaSuccess && n_proj) err = cudaMalloc(&g->proj, n_proj * sizeof(double));
    if (err == cudaSuccess && n_nrm) err = cudaMalloc(&g->nrm, n_nrm * sizeof(double));
    if (err != cudaSuccess) {
        fdg_gauss_destroy(g);
        return gfail(FDG_ERR_CUDA, "fdg_gauss_create", err);
    }
    k.status = g->status;
    *out = g;
    return FDG_OK;
}

void fdg_gauss_destroy(fdg_gauss_t* g)
{
    if (!g) return;
    if (g->status) cudaFree(g->status);
    if (g->status_host) cudaFreeHost(g->status_host);
    if (g->proj) cudaFree(g->proj);
    if (g->nrm) cudaFree(g->nrm);
    delete g;
}

int fdg_gauss_project(fdg_gauss_t* g, const double* u, double* proj, double* nrm, void* stream)
{
    if (!g || !u) return gfail(FDG_ERR_ARG, "fdg_gauss_project: null argument");
    if (g->n_elem == 0) return FDG_OK;
    GParams k = g->base;
    k.u = u;
    k.proj_out = proj ? proj : g->proj;
    k.nrm_out = nrm ? nrm : g->nrm;
    cudaError_t err = gauss_fn(g->d, g->p1)(k, 0, true, (cudaStream_t)stream, g->sm_count);
    if (err != cudaSuccess) return gfail(FDG_ERR_CUDA, "gauss projection kernel launch", err);
    return FDG_OK;
}

int fdg_gauss_rhs(fdg_gauss_t* g, const fdg_scheme_t* s, const double* u, const double* proj, const double* nrm,
                  const double* fnrm, double* du, void* stream)
{
    if (!g || !s || !u || !du) return gfail(FDG_ERR_ARG, "fdg_gauss_rhs: null argument");
    if (u == du) return gfail(FDG_ERR_ARG, "fdg_gauss_rhs: du must not alias u");
    if (s->volume_flux < 0 || s->volume_flux > F_CHANDRASHEKAR)
        return gfail(FDG_ERR_CONFIG, "gauss volume flux must be symmetric");
    if (s->surface_flux < 0 || s->surface_flux > F_HLL) return gfail(FDG_ERR_CONFIG, "surface_flux: unknown kind");
    if (g->n_elem == 0) return FDG_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (!proj || !nrm) {  // the projection into the library's scratch first
        int rc = fdg_gauss_project(g, u, g->proj, g->nrm, stream);
        if (rc) return rc;
        proj = g->proj;
        nrm = g->nrm;
    }
    GParams k = g->base;
    k.u = u;
    k.out = du;
    k.proj = proj;
    k.nrm = nrm;
    k.fnrm = fnrm;
    k.surface_flux = s->surface_flux;
    cudaError_t err = gauss_fn(g->d, g->p1)(k, s->volume_flux, false, st, g->sm_count);
    if (err != cudaSuccess) return gfail(FDG_ERR_CUDA, "gauss rhs kernel launch", err);
    return FDG_OK;
}

int fdg_gauss_gate(fdg_gauss_t* g, const double* u, void* stream)
{
    if (!g || !u) return gfail(FDG_ERR_ARG, "fdg_gauss_gate: null argument");
    long long nn = 1;
    for (int i = 0; i < g->d; ++i) nn *= g->p1;
    const long long n_nodes = g->n_elem * nn;
    if (n_nodes == 0) return FDG_OK;
    const long long blocks = std::min<long long>((n_nodes + 255) / 256, (long long)g->sm_count * 16);
    if (g->d == 2)
        gauss_gate_kernel<2><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(u, n_nodes, g->base.gas.gm1, g->status);
    else
        gauss_gate_kernel<3><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(u, n_nodes, g->base.gas.gm1, g->status);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return gfail(FDG_ERR_CUDA, "gate kernel launch", err);
    return FDG_OK;
}

int fdg_gauss_reset_status(fdg_gauss_t* g, void* stream)
{
    if (!g) return gfail(FDG_ERR_ARG, "fdg_gauss_reset_status: null argument");
    cudaError_t err = cudaMemsetAsync(g->status, 0xff, sizeof(Status), (cudaStream_t)stream);
    if (err != cudaSuccess) return gfail(FDG_ERR_CUDA, "status reset", err);
    return FDG_OK;
}

int fdg_gauss_read_status(fdg_gauss_t* g, fdg_status_t* out, void* stream)
{
    if (!g || !out) return gfail(FDG_ERR_ARG, "fdg_gauss_read_status: null argument");
    cudaError_t err = cudaMemcpyAsync(g->status_host, g->status, sizeof(Status), cudaMemcpyDeviceToHost,
                                      (cudaStream_t)stream);
    if (err == cudaSuccess) err = cudaStreamSynchronize((cudaStream_t)stream);
    if (err != cudaSuccess) return gfail(FDG_ERR_CUDA, "status read", err);
    out->first_bad = g->status_host->first_bad == ~0ull ? -1 : (int64_t)g->status_host->first_bad;
    out->bad_stage = g->status_host->bad_stage == ~0u ? -1 : (int32_t)g->status_host->bad_stage;
    out->pad = 0;
    return FDG_OK;
}

}  // extern "C"
