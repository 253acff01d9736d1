// fdg_setup.h -- on-device geometry (coordinates, curl-form metrics), launched
// by fdg_capi.cu, compiled in its own unit (fdg_setup.cu, --fmad=false).
#pragma once
#include <algorithm>
#include <cmath>
#include <cuda_runtime.h>

namespace fdg {

struct GeomArgs {
    int d = 0, p1 = 0;
    long long n_elem = 0;
    int dims[3] = {1, 1, 1};
    double lo[3] = {}, hi[3] = {};
    double amplitude = 0.0;
    double nodes[16] = {};      // 1D LGL nodes
    double dmat[64] = {};       // op.D, row-major (p+1)^2
    double* coords = nullptr;   // (n_elem, nn, d) or null
    double* ja = nullptr;       // (n_elem, nn, d, d) or null (coordinates only)
    double* jac = nullptr;      // (n_elem, nn), with ja
};

size_t geometry_smem(int d, int p1);
cudaError_t launch_geometry(const GeomArgs& g, int sm_count, cudaStream_t stream);

}  // namespace fdg
