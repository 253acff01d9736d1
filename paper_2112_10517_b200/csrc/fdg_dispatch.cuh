// fdg_dispatch.cuh -- compile-time instantiation tables of the element kernel.
#pragma once
#include <algorithm>

#include "fdg_kernels.cuh"

namespace fdg {

using LaunchFn = cudaError_t (*)(const KParams&, cudaStream_t, int sm_count);

template <int D, int P1, int VF, bool CURVED, int MODE, int LOGS>
cudaError_t launch_elem(const KParams& p, cudaStream_t s, int sm_count)
{
    using G = Geo<D, P1>;
    constexpr size_t smem = (size_t)smem_doubles<D, P1, VF, LOGS>() * sizeof(double);
    auto kern = elem_kernel<D, P1, VF, CURVED, MODE, LOGS>;
    static int blocks_per_sm = -1;  // one device per process
    if (blocks_per_sm < 0) {
        cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (err != cudaSuccess) return err;
        int b = 0;
        err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, G::NT, smem);
        if (err != cudaSuccess) return err;
        blocks_per_sm = std::max(1, b);
    }
    const long long nb = (p.n_elem + G::EPB - 1) / G::EPB;
    if (nb <= 0) return cudaSuccess;
    const long long grid = std::min(nb, (long long)blocks_per_sm * sm_count);
    kern<<<(unsigned)grid, G::NT, smem, s>>>(p);
    return cudaGetLastError();
}

template <int D, int P1, int VF, bool CURVED, int MODE>
LaunchFn pick_logs(int logs)
{
    if constexpr (VF == F_RANOCHA || VF == F_CHANDRASHEKAR) {
        return logs ? &launch_elem<D, P1, VF, CURVED, MODE, 1> : &launch_elem<D, P1, VF, CURVED, MODE, 0>;
    } else {
        (void)logs;
        return &launch_elem<D, P1, VF, CURVED, MODE, 0>;
    }
}

template <int D, int P1, int VF, int MODE>
LaunchFn pick_curved(bool curved, int logs)
{
    return curved ? pick_logs<D, P1, VF, true, MODE>(logs) : pick_logs<D, P1, VF, false, MODE>(logs);
}

template <int D, int P1, int MODE>
LaunchFn pick_flux(int vf, bool curved, int logs)
{
    switch (vf) {
    case F_CENTRAL: return pick_curved<D, P1, F_CENTRAL, MODE>(curved, logs);
    case F_SHIMA: return pick_curved<D, P1, F_SHIMA, MODE>(curved, logs);
    case F_RANOCHA: return pick_curved<D, P1, F_RANOCHA, MODE>(curved, logs);
    case F_KG: return pick_curved<D, P1, F_KG, MODE>(curved, logs);
    case F_CHANDRASHEKAR: return pick_curved<D, P1, F_CHANDRASHEKAR, MODE>(curved, logs);
    default: return nullptr;
    }
}

}  // namespace fdg

// one translation unit per (mode, d, p+1) under units/; FAITHFUL ones are compiled with --fmad=false
fdg::LaunchFn fdg_pick_faithful_d2_p2(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_faithful_d2_p3(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_faithful_d2_p4(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_faithful_d2_p5(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_faithful_d2_p6(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_faithful_d2_p7(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_faithful_d2_p8(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_faithful_d3_p2(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_faithful_d3_p3(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_faithful_d3_p4(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_faithful_d3_p5(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_faithful_d3_p6(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_faithful_d3_p7(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_faithful_d3_p8(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_fast_d2_p2(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_fast_d2_p3(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_fast_d2_p4(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_fast_d2_p5(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_fast_d2_p6(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_fast_d2_p7(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_fast_d2_p8(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_fast_d3_p2(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_fast_d3_p3(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_fast_d3_p4(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_fast_d3_p5(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_fast_d3_p6(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_fast_d3_p7(int vf, bool curved, int logs);
fdg::LaunchFn fdg_pick_fast_d3_p8(int vf, bool curved, int logs);
