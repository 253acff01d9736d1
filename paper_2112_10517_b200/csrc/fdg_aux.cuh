// fdg_aux.cuh -- small non-template kernels (halo packing, standalone gate);
// included by exactly one translation unit (fdg_capi.cu).
#pragma once
#include "fdg_kernels.cuh"

namespace fdg {

// Gather the face traces of `n_list` elements (halo send buffers): out[(i, m, v)]
// = u[list[i], line_node(dir, m, pos), v] for pos = 0 (side 0) or p (side 1).
// direction 0 (the slab halo): a face of an element is one contiguous run
// of fn * nvar doubles (its first / last fn nodes), so the pack is a batched
// contiguous copy, 16-byte vectors when the run allows
__global__ void pack_faces_dir0_kernel(const double* __restrict__ u, const int* __restrict__ list, int n_list,
                                       long long elem_doubles, long long run, long long run_off,
                                       double* __restrict__ out)
{
    const bool vec = (run % 2 == 0) && (elem_doubles % 2 == 0) && (run_off % 2 == 0) &&
                     ((reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    if (vec) {
        const long long r2 = run / 2;
        const long long total = (long long)n_list * r2;
        for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
             t += (long long)gridDim.x * blockDim.x) {
            const long long i = t / r2, k = t - i * r2;
            const double2* src = reinterpret_cast<const double2*>(u + (long long)list[i] * elem_doubles + run_off);
            reinterpret_cast<double2*>(out)[t] = __ldg(src + k);
        }
    } else {
        const long long total = (long long)n_list * run;
        for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
             t += (long long)gridDim.x * blockDim.x) {
            const long long i = t / run, k = t - i * run;
            out[t] = __ldg(u + (long long)list[i] * elem_doubles + run_off + k);
        }
    }
}

__global__ void pack_faces_kernel(const double* __restrict__ u, const int* __restrict__ list, int n_list, int d,
                                  int p1, int dir, int side, double* __restrict__ out)
{
    const int nvar = d + 2;
    int fn = 1;
    for (int i = 0; i < d - 1; ++i) fn *= p1;
    int nn = fn * p1;
    int stride = 1;
    for (int i = 0; i < d - 1 - dir; ++i) stride *= p1;
    const int pos = side ? p1 - 1 : 0;
    const long long total = (long long)n_list * fn * nvar;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int v = (int)(t % nvar);
        const long long im = t / nvar;
        const int mm = (int)(im % fn);
        const long long i = im / fn;
        const int node = (mm / stride * p1 + pos) * stride + mm % stride;
        out[t] = u[((long long)list[i] * nn + node) * nvar + v];
    }
}

// Standalone admissibility gate (discretization.py:660-672).
template <int D>
__global__ void gate_kernel(const double* __restrict__ u, long long n_nodes, double gm1, long long node_base,
                            Status* status)
{
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n_nodes;
         t += (long long)gridDim.x * blockDim.x) {
        if (!gate_ok<D>(u + t * (D + 2), gm1)) atomicMin(&status->first_bad, (unsigned long long)(node_base + t));
    }
}

}  // namespace fdg
