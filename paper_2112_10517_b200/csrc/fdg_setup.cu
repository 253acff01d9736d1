// fdg_setup.cu -- on-device geometry: nodal coordinates of the (optionally
// warped) periodic box and the curl-form metric terms Ja^i_n and Jacobian J,
// written straight into the device arrays the element kernels read. Replaces
// the host setup (22 GB / 43 s at 128^3) for the
// reference's
//   element_coords   geometry.py:142-178  (x = lo + L t, t = (e + (xi+1)/2) / n,
//                                          + amplitude prod_j sin(2 pi t_j))
//   _metrics_2d      geometry.py:200-214  (Ja = [[d2 x2, -d2 x1], [-d1 x2, d1 x1]])
//   _metrics_3d_curl geometry.py:228-250  (Ja^i_n = D_j(x_l d_k x_m) - D_k(x_l d_j x_m),
//                                          coordinates shifted by the element mean)
// One CTA per element, one thread per node, all fields of the element in
// shared memory; compiled --fmad=false (the host's separate roundings).
#include "fdg_setup.h"

namespace fdg {

__device__ __forceinline__ int node_digit(int i, int p1, int d, int dir)
{
    int stride = 1;
    for (int k = d - 1; k > dir; --k) stride *= p1;
    return (i / stride) % p1;
}

// sum_b D[a_dir, b] f[node with digit dir = b]
__device__ __forceinline__ double deriv(const double* __restrict__ f, const double* __restrict__ dm, int i, int p1,
                                        int d, int dir)
{
    int stride = 1;
    for (int k = d - 1; k > dir; --k) stride *= p1;
    const int a = (i / stride) % p1;
    const int base = i - a * stride;
    double s = 0.0;
    for (int b = 0; b < p1; ++b) s += dm[a * p1 + b] * f[base + b * stride];
    return s;
}

template <int D>
__global__ void geometry_kernel(GeomArgs g)
{
    extern __shared__ double sm[];
    const int p1 = g.p1;
    const int nn = (D == 2) ? p1 * p1 : p1 * p1 * p1;
    double* dm = sm;                 // p1 * p1 (<= 64)
    double* x = dm + 64;             // D * nn
    double* dx = x + D * nn;         // D * D * nn: dx[i][m] = d_i x_m
    double* tmp = dx + D * D * nn;   // 2 * nn products (3D)
    const int i = threadIdx.x;
    for (int k = i; k < p1 * p1; k += blockDim.x) dm[k] = g.dmat[k];
    __syncthreads();
    for (long long e = blockIdx.x; e < g.n_elem; e += gridDim.x) {
        // element multi-index, C order over dims (geometry.py:_element_multi_index)
        int eidx[D];
        long long r = e;
        for (int j = D - 1; j >= 0; --j) {
            eidx[j] = (int)(r % g.dims[j]);
            r /= g.dims[j];
        }
        double t[D];
        if (i < nn) {
            for (int j = 0; j < D; ++j) {
                const double half = 0.5 * (g.nodes[node_digit(i, p1, D, j)] + 1.0);
                t[j] = ((double)eidx[j] + half) / (double)g.dims[j];
                x[j * nn + i] = g.lo[j] + (g.hi[j] - g.lo[j]) * t[j];
            }
            if (g.amplitude != 0.0) {
                double bump = 1.0;
                for (int j = 0; j < D; ++j) bump = bump * sin(2.0 * M_PI * t[j]);
                bump = g.amplitude * bump;
                for (int j = 0; j < D; ++j) x[j * nn + i] += bump;
            }
            if (g.coords)
                for (int j = 0; j < D; ++j) g.coords[(e * nn + i) * D + j] = x[j * nn + i];
        }
        __syncthreads();
        if (g.ja) {
            if (i < nn)
                for (int dir = 0; dir < D; ++dir)
                    for (int m = 0; m < D; ++m) dx[(dir * D + m) * nn + i] = deriv(x + m * nn, dm, i, p1, D, dir);
            __syncthreads();
            double* ja = g.ja + (e * nn + i) * D * D;
            double jac;
            if constexpr (D == 2) {
                if (i < nn) {
                    const double d1x1 = dx[0 * nn + i], d1x2 = dx[1 * nn + i];
                    const double d2x1 = dx[2 * nn + i], d2x2 = dx[3 * nn + i];
                    ja[0] = d2x2;
                    ja[1] = -d2x1;
                    ja[2] = -d1x2;
                    ja[3] = d1x1;
                    jac = d1x1 * d2x2 - d2x1 * d1x2;
                    g.jac[e * nn + i] = jac;
                }
            } else {
                // shift-invariant curl: coordinates minus their element mean
                __shared__ double mean[3];
                if (i < 3) {
                    double s = 0.0;
                    for (int k = 0; k < nn; ++k) s += x[i * nn + k];
                    mean[i] = s / (double)nn;
                }
                __syncthreads();
                if (i < nn)
                    for (int m = 0; m < 3; ++m) x[m * nn + i] -= mean[m];
                __syncthreads();
                const int cyc[3][2] = {{1, 2}, {2, 0}, {0, 1}};
                double out[3][3];
                for (int n = 0; n < 3; ++n) {
                    const int l = cyc[n][0], m = cyc[n][1];
                    for (int ii = 0; ii < 3; ++ii) {
                        const int j = cyc[ii][0], k = cyc[ii][1];
                        if (i < nn) {
                            tmp[i] = x[l * nn + i] * dx[(k * 3 + m) * nn + i];
                            tmp[nn + i] = x[l * nn + i] * dx[(j * 3 + m) * nn + i];
                        }
                        __syncthreads();
                        if (i < nn) out[ii][n] = deriv(tmp, dm, i, p1, 3, j) - deriv(tmp + nn, dm, i, p1, 3, k);
                        __syncthreads();
                    }
                }
                if (i < nn) {
                    for (int a = 0; a < 3; ++a)
                        for (int b = 0; b < 3; ++b) ja[a * 3 + b] = out[a][b];
                    const double* q = dx;
                    auto X = [&](int a, int b) { return q[(a * 3 + b) * nn + i]; };
                    jac = X(0, 0) * (X(1, 1) * X(2, 2) - X(1, 2) * X(2, 1)) -
                          X(0, 1) * (X(1, 0) * X(2, 2) - X(1, 2) * X(2, 0)) +
                          X(0, 2) * (X(1, 0) * X(2, 1) - X(1, 1) * X(2, 0));
                    g.jac[e * nn + i] = jac;
                }
            }
        }
        __syncthreads();
    }
}

size_t geometry_smem(int d, int p1)
{
    int nn = 1;
    for (int k = 0; k < d; ++k) nn *= p1;
    return sizeof(double) * (64 + (size_t)d * nn + (size_t)d * d * nn + 2 * (size_t)nn);
}

cudaError_t launch_geometry(const GeomArgs& g, int sm_count, cudaStream_t st)
{
    int nn = 1;
    for (int k = 0; k < g.d; ++k) nn *= g.p1;
    const int threads = (nn + 31) / 32 * 32;
    const size_t smem = geometry_smem(g.d, g.p1);
    const long long blocks = std::min<long long>(g.n_elem, (long long)sm_count * 16);
    if (blocks == 0) return cudaSuccess;
    if (g.d == 2) {
        cudaFuncSetAttribute(geometry_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        geometry_kernel<2><<<(unsigned)blocks, threads, smem, st>>>(g);
    } else {
        cudaFuncSetAttribute(geometry_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        geometry_kernel<3><<<(unsigned)blocks, threads, smem, st>>>(g);
    }
    return cudaGetLastError();
}

}  // namespace fdg
