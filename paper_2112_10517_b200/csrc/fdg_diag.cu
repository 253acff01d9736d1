// fdg_diag.cu -- device diagnostics: one grid-stride pass over the nodes with
// per-thread partials, a fixed-order block tree, per-block partials in HBM and
// a one-block finish. HBM-bound: u (and dudt / u_exact) read once, coalesced
// (a warp reads 32 consecutive nodes' AoS rows); no atomics, so the result is
// the same on every call for a given mesh and grid.
//
// Reference restated (pkg/src/fluxdg):
//   conserved_totals  discretization.py:1027-1031  sum wbar J u
//   entropy_rate      discretization.py:1011-1024  sum wbar J w(u).dudt, sum |wbar J w dudt|
//   error_norm_l2     discretization.py:1033-1037  sum wbar J (u - u_exact)^2 (sqrt on the host)
//   stable_dt         timeint.py:138-146           min J^(1/d) / (lambda (2p+1)) (cfl on the host)
//   entropy_vars      euler.py:129-146, max_signal_speed euler.py:105-112
#include "fdg_diag.h"
#include "../../include/fdg.h"

namespace fdg {

int diag_n_out(int kind, int d)
{
    switch (kind) {
        case FDG_DIAG_CONSERVED:
        case FDG_DIAG_ERROR_SQ: return d + 2;
        case FDG_DIAG_ENTROPY: return 2;
        case FDG_DIAG_DT: return 1;
        default: return 0;
    }
}

template <int KIND>
struct DiagTraits {
    static constexpr bool is_min = (KIND == FDG_DIAG_DT);
};

// wbar[i] = kron(kron(1, w), w)...: (w[i0] * w[i1]) * w[i2] (discretization.py:619-621)
template <int D>
__device__ __forceinline__ double node_weight(const double* w, int p1, int i)
{
    if constexpr (D == 2) {
        return w[i / p1] * w[i % p1];
    } else {
        return (w[i / (p1 * p1)] * w[(i / p1) % p1]) * w[i % p1];
    }
}

template <int D, int KIND>
__global__ void __launch_bounds__(kDiagThreads, kDiagCtasPerSm) diag_partial_kernel(DiagArgs g)
{
    constexpr int NV = D + 2;
    constexpr int NQ = (KIND == FDG_DIAG_ENTROPY) ? 2 : (KIND == FDG_DIAG_DT ? 1 : NV);
    constexpr bool MIN = DiagTraits<KIND>::is_min;
    __shared__ double sh[NQ][kDiagThreads];
    __shared__ double sw[8];
    if (threadIdx.x < 8) sw[threadIdx.x] = g.w[threadIdx.x];
    __syncthreads();
    const int p1 = g.p1;
    const int nn = (D == 2) ? p1 * p1 : p1 * p1 * p1;
    const long long total = g.n_elem * nn;
    double acc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = MIN ? __longlong_as_double(0x7ff0000000000000LL) : 0.0;
    const double gm1 = g.gm1;
    for (long long t = blockIdx.x * (long long)kDiagThreads + threadIdx.x; t < total;
         t += (long long)gridDim.x * kDiagThreads) {
        const int i = (int)(t % nn);
        const double J = g.jac ? g.jac[t] : g.jac_const;
        const double* u = g.a + t * NV;
        double un[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) un[v] = u[v];
        if constexpr (KIND == FDG_DIAG_DT) {
            const double rho = un[0];
            double vv = 0.0, mm = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const double vk = un[1 + k] / rho;
                vv = (k == 0) ? vk * vk : vv + vk * vk;
                mm = (k == 0) ? un[1] * un[1] : mm + un[1 + k] * un[1 + k];
            }
            const double p = gm1 * (un[D + 1] - 0.5 * mm / rho);
            const double lam = sqrt(vv) + sqrt(g.gamma * p / rho);
            const double den = lam * (double)(2 * (p1 - 1) + 1);
            // Cartesian (constant J): min_i s / den_i = s / max_i den_i exactly
            // (rounded multiply and divide are monotone), so reduce -den and
            // divide once in the finish kernel; curved: the per-node quotient.
            // numpy's min propagates NaN: keep it.
            const double val = g.jac ? ((D == 2) ? sqrt(J) : pow(J, 1.0 / 3.0)) / den : -den;
            acc[0] = (val < acc[0] || isnan(val)) && !isnan(acc[0]) ? val : acc[0];
        } else {
            const double wt = node_weight<D>(sw, p1, i) * J;
            if constexpr (KIND == FDG_DIAG_CONSERVED) {
#pragma unroll
                for (int v = 0; v < NV; ++v) acc[v] += wt * un[v];
            } else if constexpr (KIND == FDG_DIAG_ERROR_SQ) {
                const double* ue = g.b + t * NV;
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const double diff = un[v] - ue[v];
                    acc[v] += (wt * diff) * diff;
                }
            } else {  // entropy production
                const double* du = g.b + t * NV;
                const double rho = un[0];
                double vel[D];
                double vv = 0.0;
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    vel[k] = un[1 + k] / rho;
                    vv = (k == 0) ? vel[k] * vel[k] : vv + vel[k] * vel[k];
                }
                const double p = gm1 * (un[D + 1] - 0.5 * rho * vv);
                const double s = log(p) - g.gamma * log(rho);
                const double rho_p = rho / p;
                double w[NV];
                w[0] = (g.gamma - s) * g.igm1 - 0.5 * rho_p * vv;
#pragma unroll
                for (int k = 0; k < D; ++k) w[1 + k] = rho_p * vel[k];
                w[D + 1] = -rho_p;
                double dot = w[0] * du[0];
#pragma unroll
                for (int v = 1; v < NV; ++v) dot = dot + w[v] * du[v];
                acc[0] += wt * dot;
#pragma unroll
                for (int v = 0; v < NV; ++v) acc[1] += fabs((wt * w[v]) * du[v]);
            }
        }
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) sh[q][threadIdx.x] = acc[q];
    __syncthreads();
    for (int s = kDiagThreads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const double x = sh[q][threadIdx.x], y = sh[q][threadIdx.x + s];
                sh[q][threadIdx.x] = MIN ? ((isnan(x) || y >= x) ? x : y) : x + y;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x < NQ) g.part[blockIdx.x * kDiagQ + threadIdx.x] = sh[threadIdx.x][0];
}

// cart_d > 0: Cartesian DT, the partials hold -max den; out = J^(1/d) / max den
__global__ void __launch_bounds__(kDiagThreads) diag_finish_kernel(const double* __restrict__ part, int blocks,
                                                                   int nq, int is_min, int cart_d, double jac_const,
                                                                   double* __restrict__ out)
{
    __shared__ double sh[kDiagThreads];
    for (int q = 0; q < nq; ++q) {
        double acc = is_min ? __longlong_as_double(0x7ff0000000000000LL) : 0.0;
        for (int b = threadIdx.x; b < blocks; b += kDiagThreads) {
            const double x = part[b * kDiagQ + q];
            acc = is_min ? ((isnan(acc) || x >= acc) ? acc : x) : acc + x;
        }
        sh[threadIdx.x] = acc;
        __syncthreads();
        for (int s = kDiagThreads / 2; s > 0; s >>= 1) {
            if (threadIdx.x < s) {
                const double x = sh[threadIdx.x], y = sh[threadIdx.x + s];
                sh[threadIdx.x] = is_min ? ((isnan(x) || y >= x) ? x : y) : x + y;
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            if (cart_d > 0) {
                const double scale = (cart_d == 2) ? sqrt(jac_const) : pow(jac_const, 1.0 / 3.0);
                out[q] = scale / (-sh[0]);
            } else {
                out[q] = sh[0];
            }
        }
        __syncthreads();
    }
}

template <int D>
static void launch_partial(const DiagArgs& g, cudaStream_t st)
{
    switch (g.kind) {
        case FDG_DIAG_CONSERVED:
            diag_partial_kernel<D, FDG_DIAG_CONSERVED><<<g.blocks, kDiagThreads, 0, st>>>(g);
            break;
        case FDG_DIAG_ENTROPY: diag_partial_kernel<D, FDG_DIAG_ENTROPY><<<g.blocks, kDiagThreads, 0, st>>>(g); break;
        case FDG_DIAG_ERROR_SQ:
            diag_partial_kernel<D, FDG_DIAG_ERROR_SQ><<<g.blocks, kDiagThreads, 0, st>>>(g);
            break;
        default: diag_partial_kernel<D, FDG_DIAG_DT><<<g.blocks, kDiagThreads, 0, st>>>(g); break;
    }
}

cudaError_t launch_diagnostic(const DiagArgs& g, cudaStream_t st)
{
    if (g.d == 2)
        launch_partial<2>(g, st);
    else
        launch_partial<3>(g, st);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    diag_finish_kernel<<<1, kDiagThreads, 0, st>>>(g.part, g.blocks, diag_n_out(g.kind, g.d),
                                                   g.kind == FDG_DIAG_DT,
                                                   (g.kind == FDG_DIAG_DT && !g.jac) ? g.d : 0, g.jac_const, g.out);
    return cudaGetLastError();
}

}  // namespace fdg
