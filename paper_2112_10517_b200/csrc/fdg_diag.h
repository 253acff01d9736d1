// fdg_diag.h -- device diagnostics reductions (conserved totals, entropy
// production, weighted L2 error, CFL time step), launched by fdg_capi.cu and
// compiled in their own unit (fdg_diag.cu, --fmad=false: the per-node
// arithmetic keeps the reference's multiply-then-add roundings).
#pragma once
#include <cuda_runtime.h>

namespace fdg {

constexpr int kDiagThreads = 256;
constexpr int kDiagQ = 5;  // max quantities per reduction (nvar in 3D)
constexpr int kDiagCtasPerSm = 4;  // 32 warps/SM: enough loads in flight for HBM (<= 64 registers)

struct DiagArgs {
    int d = 0, p1 = 0, kind = 0;
    long long n_elem = 0;
    const double* a = nullptr;    // u
    const double* b = nullptr;    // dudt (entropy) | u_exact (error)
    const double* jac = nullptr;  // (n_elem, nn) curved, else null
    double jac_const = 0.0;
    double w[8] = {};             // 1D LGL weights
    double gamma = 0.0, gm1 = 0.0, igm1 = 0.0;
    double* part = nullptr;       // (blocks, kDiagQ) device partials
    double* out = nullptr;        // device result
    int blocks = 0;
};

// number of doubles written to out for `kind` (enum fdg_diag), 0 if unknown
int diag_n_out(int kind, int d);
// partial pass (blocks x kDiagThreads) + a one-block finish, fixed order:
// deterministic for a given grid
cudaError_t launch_diagnostic(const DiagArgs& g, cudaStream_t stream);

}  // namespace fdg
