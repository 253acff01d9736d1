// fdg_dispatch.cuh -- compile-time instantiation tables of the element kernel.
#pragma once
#include <algorithm>

#include "fdg_kernels.cuh"

namespace fdg {

using LaunchFn = cudaError_t (*)(const KParams&, cudaStream_t, int sm_count);

// High-occupancy twin: FAST 3D kernels whose default occupancy is below 8
// CTAs (p+1 = 5: 6 CTAs, 168 regs) are also built with an 8-CTA register cap.
// The default is faster per element in steady state, but when a launch fits
// in one wave only at the higher occupancy the twin removes the second,
// mostly empty wave (session 1, p+1 = 4: cfg2 VOL 20.4 -> 18.4 us, RHS
// 51 -> 39 us; p+1 = 4 now runs 8 CTAs by default, profiles/r01_tuning.md).
#ifndef FDG_HIOCC
#define FDG_HIOCC 8
#endif
template <int D, int P1, int MODE, bool CURVED>
constexpr bool has_hiocc()
{
    // (curved kernels spill heavily at 128 registers: no twin)
    // (FDG_HIOCC counts 64-thread CTAs: only for kernels of that size)
    return FDG_HIOCC > 0 && MODE == FAST && D == 3 && P1 <= 5 && !CURVED && FDG_MIN_BLOCKS == 0 &&
           Geo<D, P1>::NT == 64 && min_blocks<D, P1, MODE, CURVED>() < FDG_HIOCC;
}

#ifndef FDG_VOLK_HIOCC
#define FDG_VOLK_HIOCC 1
#endif
// Volume-integral-only twin (EPIK = EPI_VOLUME) of the FAST 3D kernels the
// BASELINE volume workloads run: the image holds no interface / stage code.
#ifndef FDG_VOLK
#define FDG_VOLK 1
#endif
template <int D, int P1, int MODE, bool CURVED>
constexpr bool has_volk()
{
    return FDG_VOLK && MODE == FAST && D == 3 && P1 >= 4;  // N = 3..7 (north-star degrees)
}

// RHS / RK-stage twins with the interface terms fused (Rusanov): no separate
// face phase, no volume-only / surface-only code in the image
#ifndef FDG_RHSK
#define FDG_RHSK 1
#endif
#ifndef FDG_RHSK_MAXP1
#define FDG_RHSK_MAXP1 8  // N = 5..7 RHS: 4.50 / 5.17 / 3.81 -> 3.96 / . / 3.42 ms with the twins
#endif
template <int D, int P1, int VF, int MODE, bool CURVED>
constexpr bool has_rhsk()
{
    return FDG_RHSK && MODE == FAST && D == 3 && P1 >= 4 && P1 <= FDG_RHSK_MAXP1 && VF != F_CENTRAL;
}

template <int D, int P1, int VF, bool CURVED, int MODE, int LOGS, int OCC>
cudaError_t elem_occupancy(int* blocks_per_sm)
{
    using G = Geo<D, P1>;
    constexpr size_t smem = (size_t)smem_doubles<D, P1, VF, LOGS>() * sizeof(double);
    auto kern = elem_kernel<D, P1, VF, CURVED, MODE, LOGS, OCC>;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    int b = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, G::NT, smem);
    *blocks_per_sm = std::max(1, b);
    return err;
}

// Programmatic dependent launch: an element kernel may be scheduled while the
// previous kernel of the stream drains; it runs its prologue and then waits
// (griddepcontrol.wait, before any global memory access) for that kernel's
// completion and memory flush. Hides launch latency and the parameter-bank
// warm-up behind the previous kernel's tail (kernel-to-kernel in a solver
// loop or a CUDA graph); the dependency itself is unchanged.
template <class Kern>
cudaError_t launch_kernel(Kern kern, unsigned grid, unsigned block, size_t smem, cudaStream_t s, const KParams& p)
{
#if FDG_PDL
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
#else
    kern<<<grid, block, smem, s>>>(p);
    return cudaGetLastError();
#endif
}

template <int D, int P1, int VF, bool CURVED, int MODE, int LOGS>
cudaError_t launch_elem(const KParams& p_in, cudaStream_t s, int sm_count)
{
    KParams p = p_in;
    using G = Geo<D, P1>;
    constexpr size_t smem = (size_t)smem_doubles<D, P1, VF, LOGS>() * sizeof(double);
    constexpr bool twin = has_hiocc<D, P1, MODE, CURVED>();
    // resident CTAs per SM, cached per device (a process may drive several)
    constexpr int kMaxDev = 64;
    static int bps_tab[kMaxDev] = {}, bps_hi_tab[kMaxDev] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    int bps = 0, bps_hi = 0;
    if (dev >= 0 && dev < kMaxDev && bps_tab[dev] > 0) {
        bps = bps_tab[dev];
        bps_hi = bps_hi_tab[dev];
    } else {
        cudaError_t err = elem_occupancy<D, P1, VF, CURVED, MODE, LOGS, 0>(&bps);
        if (err != cudaSuccess) return err;
        if constexpr (twin) {
            err = elem_occupancy<D, P1, VF, CURVED, MODE, LOGS, FDG_HIOCC>(&bps_hi);
            if (err != cudaSuccess) return err;
        }
        if (dev >= 0 && dev < kMaxDev) {
            bps_hi_tab[dev] = bps_hi;
            bps_tab[dev] = bps;  // published last: a reader seeing bps > 0 sees bps_hi
        }
    }
    const long long nb = (p.range_hi - p.range_lo + G::EPB - 1) / G::EPB + (p.range2_hi - p.range2_lo + G::EPB - 1) / G::EPB;
    if (nb <= 0) return cudaSuccess;
    const long long slots = (long long)bps * std::max(1, sm_count - std::max(0, p.reserve_sms));
    // dynamic claiming (one batch per claim, fdg_kernels.cuh); a launch of at
    // most one batch per CTA keeps the static assignment
    if (p.claim && nb <= slots) p.claim = nullptr;
    if constexpr (twin) {
        if (nb > slots && nb <= (long long)bps_hi * sm_count) {
            p.claim = nullptr;  // one batch per CTA
            return launch_kernel(elem_kernel<D, P1, VF, CURVED, MODE, LOGS, FDG_HIOCC>, (unsigned)nb, G::NT, smem, s, p);
        }
    }
    // compile-time-epilogue twins: same launch bounds and shared memory as
    // the general kernel, so the same occupancy
    auto launch_twin = [&](auto kern, bool* attr_set) -> cudaError_t {
        if (dev >= 0 && dev < kMaxDev && !attr_set[dev]) {
            cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (err != cudaSuccess) return err;
            attr_set[dev] = true;
        }
        return launch_kernel(kern, (unsigned)std::min(nb, slots), G::NT, smem, s, p);
    };
    if constexpr (has_volk<D, P1, MODE, CURVED>()) {
        if (p.epilogue == EPI_VOLUME) {
            static bool attr_set[kMaxDev] = {};
            if constexpr (twin && FDG_VOLK_HIOCC) {
                // the volume-only twin of this degree (p + 1 = 5, Cartesian) is also the
                // faster one at the high-occupancy register cap in steady state
                // (N=4 VOL: Ranocha 2.27 -> 2.21 ms, Shima 1.63 -> 1.50 ms)
                const long long slots_hi = (long long)bps_hi * std::max(1, sm_count - std::max(0, p.reserve_sms));
                if (p_in.claim && nb > slots_hi) p.claim = p_in.claim;
                else p.claim = nullptr;
                auto kern = elem_kernel<D, P1, VF, CURVED, MODE, LOGS, FDG_HIOCC, EPI_VOLUME>;
                if (dev >= 0 && dev < kMaxDev && !attr_set[dev]) {
                    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    if (err != cudaSuccess) return err;
                    attr_set[dev] = true;
                }
                return launch_kernel(kern, (unsigned)std::min(nb, slots_hi), G::NT, smem, s, p);
            } else {
                return launch_twin(elem_kernel<D, P1, VF, CURVED, MODE, LOGS, 0, EPI_VOLUME>, attr_set);
            }
        }
    }
    if constexpr (has_rhsk<D, P1, VF, MODE, CURVED>()) {
        if (p.fuse_faces && p.surface_flux == F_LLF && p.epilogue == EPI_RHS) {
            static bool attr_set[kMaxDev] = {};
            return launch_twin(elem_kernel<D, P1, VF, CURVED, MODE, LOGS, 0, EPI_RHS>, attr_set);
        }
        if (p.fuse_faces && p.surface_flux == F_LLF && p.epilogue == EPI_STAGE) {
            static bool attr_set[kMaxDev] = {};
            return launch_twin(elem_kernel<D, P1, VF, CURVED, MODE, LOGS, 0, EPI_STAGE>, attr_set);
        }
    }
    return launch_kernel(elem_kernel<D, P1, VF, CURVED, MODE, LOGS, 0>, (unsigned)std::min(nb, slots), G::NT, smem, s,
                         p);
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
