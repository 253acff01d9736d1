// fdg_kernels.cuh -- the element kernel of the flux-differencing DGSEM RHS.
//
// One CTA owns EPB elements at a time (grid-stride over element batches).
//
//   stage   u (AoS, the reference's (n_elem, nn, nvar) layout) is copied
//           coalesced into shared memory, converted once per node into
//           primitives (+ log rho/log p, beta or e) stored structure-of-arrays
//           with one pad slot per innermost row (bank-conflict-free line
//           walks in every direction); the admissibility gate runs here.
//   volume  direction n = 0..d-1: one thread per 1D line; the thread walks
//           the pair table (a < b, reference order, operators.py:267-290),
//           evaluates each symmetric two-point flux ONCE, and scatters
//           D[a,b] f into node a and D[b,a] f into node b in registers.  The
//           per-node partial sums are carried across directions in shared
//           memory (SoA, padded like the primitives), so every node sees the
//           reference's accumulation order (discretization.py:288-320).
//   epilogue VOL / J (mesh_fluxdiff_volume), or the LGL surface terms
//           (both sides of each interface evaluated from identical
//           arguments, lifted with 1/(w J), direction by direction,
//           discretization.py:730-760) and -(VOL+SURF), optionally fused with
//           a Runge-Kutta stage update (timeint.py:155-162 / SSPRK43).
//
// HBM traffic per node for the volume integral: u read once (8 nvar B) and
// VOL written once (8 nvar B) -- the algorithmic minimum.
#pragma once
#include <type_traits>

#include "fdg_device.cuh"

namespace fdg {

enum Epilogue : int { EPI_VOLUME = 0, EPI_RHS = 1, EPI_STAGE = 2, EPI_SURFACE = 3 };

struct Status {
    unsigned long long first_bad;  // min flat (element*nn + node) failing the gate
    unsigned int bad_stage;        // min RK stage index with a non-finite output
    unsigned int pad;
};

struct KParams {
    const double* u;          // (n_elem, nn, nvar) input state
    double* out;              // VOL | du | next stage | accumulated SURF
    const double* ja;         // (n_elem, nn, d, d) curved metrics
    const double* jac;        // (n_elem, nn) curved Jacobian
    const int* plus;          // (d, n_elem) +n neighbour, < 0: ghost slot -(g+1)
    const int* minus;         // (d, n_elem) -n neighbour
    const double* ghost_u;    // (n_ghost, fn, nvar) remote face states
    const double* ghost_nrm;  // (n_ghost, fn, d) remote face normals
    double* reg;              // RK 2N register
    const double* u0;         // Shu-Osher stage base state
    Status* status;
    long long n_elem;         // elements of the mesh handle (neighbour-table stride)
    long long range_lo;       // this launch covers elements [range_lo, range_hi) (interior /
    long long range_hi;       //   boundary split of a partition); [0, n_elem) by default
    long long range2_lo;      // optional second range [range2_lo, range2_hi) in the same launch
    long long range2_hi;      //   (both boundary planes of a slab in one launch); empty by default
    unsigned long long* claim; // dynamic batch claiming: [0] next batch, [1] CTAs done (null: static grid-stride)
    int zero;                 // always 0 (claim_batch: keeps the claim's address from being provably uniform)
    int claim_chunk_max;      // (unused since claims are per batch, one ahead)
    int rt_iface;             // interface epilogues below FDG_RT_DIR_MIN_P1 take the runtime-direction pass
    int reserve_sms;          // launch only on sm_count - reserve_sms SMs' worth of CTAs (room for concurrent
                              // halo kernels: a full-occupancy grid holds every register of every SM)
    long long elem_base;      // added to element indices reported by the gate
    double wts[3][64];        // per direction: Dsplit[a,b] * Ja^n_n (Cartesian) or Dsplit (curved)
    double wtsE[3][64];       // 2 * wts: the energy row of FAST fluxes that return f_E / 2 (energy_half)
    double areas[3];          // Cartesian Ja^n_n
    double jac_const;         // Cartesian J
    double rjac_const;        // 1/J (FAST)
    double w0, wp;            // LGL weights at the -1 / +1 ends
    double inv_w0, inv_wp;    // 1/w0, 1/wp (FAST: interface terms fused into the volume passes)
    int fuse_faces;           // FAST RHS / RK-stage launches with the Rusanov interface flux: line-end fusion on
    int jac_folded;           // FAST Cartesian launches: wts / wtsE / inv_w0 / inv_wp already carry 1/J (fdg_capi.cu)
    Gas gas;
    int epilogue;
    int surface_flux;
    int precompute;
    int stage_kind;           // 0: low-storage 2N, 1: Shu-Osher convex combination
    int face_prefetch;        // interface epilogues: prefetch neighbour face rows (state >> L2)
    const int* row_order;     // traversal: element rows (row_len consecutive elements) in tile order, or null
    long long row_len;
    unsigned int stage_index;
    double sa, sb, sc, dt;    // 2N: a_i, b_i, -, dt ; SO: A, B, C*dt, -
};

// tuning knobs (compile-time; scripts/ab.sh builds alternatives). Defaults
// measured on B200 (scripts/ab.sh + scripts/sweep.py, profiles/r01_tuning.md):
// 64-thread CTAs (one warp for 3D p+1 = 4, Geo::TT) and the register caps of
// min_blocks().
#ifndef FDG_TARGET_THREADS
#define FDG_TARGET_THREADS 64
#endif
#ifndef FDG_MIN_BLOCKS
#define FDG_MIN_BLOCKS 0  // 0: per-degree default below
#endif
#ifndef FDG_CHANDRA_KP
#define FDG_CHANDRA_KP 1  // volume-only Chandrashekar twins: |v/2|^2 staged in the unused pressure slot
#endif
#ifndef FDG_LINE_REGS
#define FDG_LINE_REGS 1  // compile-time passes: the line's node data in registers (r02: cfg5 VOL 3.52 -> 3.49 ms)
#endif
#ifndef FDG_STAGE_UNROLL
#define FDG_STAGE_UNROLL 1
#endif
constexpr int kStageUnroll = FDG_STAGE_UNROLL;
#ifndef FDG_FACE_UNROLL
#define FDG_FACE_UNROLL 2
#endif
constexpr int kFaceUnroll = FDG_FACE_UNROLL;
#ifndef FDG_PAD
#define FDG_PAD 1
#endif
#ifndef FDG_PREFETCH
#define FDG_PREFETCH 1
#endif
#ifndef FDG_FACE_PREFETCH
#define FDG_FACE_PREFETCH 1  // neighbour face rows into L2 at batch start (interface epilogues)
#endif
#ifndef FDG_NB_SMEM
#define FDG_NB_SMEM 1  // interface neighbour indices read into shared memory at batch start (v13: cfg4 RHS +7.7%, cfg5 RHS +3.4%)
#endif
#ifndef FDG_DIR_REV
#define FDG_DIR_REV 0
#endif
#ifndef FDG_PDL
#define FDG_PDL 0  // 1: programmatic dependent launch (fdg_dispatch.cuh); measured no gain in a CUDA graph
#endif
template <int D, int P1>
struct Geo {
    static constexpr int NN = ipow(P1, D);
    static constexpr int LINES = ipow(P1, D - 1);
    static constexpr int NVAR = D + 2;
    // 3D, p + 1 = 4: nodes XOR-swizzled instead of padded (SWZ): with a
    // half-warp on 16 lines at one line position (any direction) every bank
    // pair is hit exactly once, and the element block stays 64 slots
#ifndef FDG_SWIZZLE
#define FDG_SWIZZLE 1
#endif
    // (p + 1 = 8: bank pair (node & 15) ^ ((node >> 3) & 15), the same property
    // for the 32 lines of a warp; profiles/r01_tuning.md)
    static constexpr bool SWZ = FDG_SWIZZLE && D == 3 && (P1 == 4 || P1 == 8);
    // other 3D degrees: plain node order -- the pad slot per innermost row
    // costs more conflicts than it removes there (scripts/bank_model.py:
    // p+1 = 3/5/7: 5.7/3.7/6.5 -> 3.3/2.7/3.0 wavefronts per warp load)
    static constexpr bool PADDED = FDG_PAD && !SWZ && !(FDG_SWIZZLE && D == 3);
    static constexpr int NNP = PADDED ? NN + NN / P1 : NN;  // one pad slot per innermost row
    // threads per CTA target: one warp (2 elements) for 3D p+1 = 4 -- no
    // barrier coupling between warps, cfg2 VOL +1.3%, RHS +3.7% against 2-warp
    // CTAs (profiles/r01_tuning.md) -- else FDG_TARGET_THREADS
#ifndef FDG_P4_TT
#define FDG_P4_TT 32
#endif
    static constexpr int TT = (D == 3 && P1 == 4 && FDG_TARGET_THREADS == 64) ? FDG_P4_TT : FDG_TARGET_THREADS;
    // 3D p + 1 = 5, 6, 7: 25 / 36 / 49 lines per element leave 22-44% of a
    // 64-thread CTA's lanes idle (FP64-bound degrees: lane utilisation is
    // throughput); per-degree batch sizes, measured (profiles/r02_tuning.md).
    // Even EPB * NN * NVAR keeps every batch 16-byte aligned for the bulk copies.
#ifndef FDG_EPB_P5
#define FDG_EPB_P5 0  // 0: TT / LINES (2 elements, 50 of 64 lanes: larger batches measured slower, r02_tuning.md)
#endif
#ifndef FDG_EPB_P6
#define FDG_EPB_P6 3  // 108 of 128 lanes (1 element: 36 of 64)
#endif
#ifndef FDG_EPB_P7
#define FDG_EPB_P7 2  // 98 of 128 lanes, 4-warp CTAs
#endif
    static constexpr int EPB_OVR = D != 3 ? 0 : (P1 == 5 ? FDG_EPB_P5 : (P1 == 6 ? FDG_EPB_P6 : (P1 == 7 ? FDG_EPB_P7 : 0)));
    static constexpr int EPB = EPB_OVR > 0 ? EPB_OVR : (LINES >= TT ? 1 : TT / LINES);
    static constexpr int NT = ((EPB * LINES + 31) / 32) * 32;
    static constexpr int FS = EPB * NNP;      // stride of one primitive field
    static constexpr int FA = EPB * NNP + 1;  // stride of one accumulator variable (odd: spreads banks)
    static constexpr int NF = 2 * D * LINES;  // face nodes per element (2 sides x d directions)

    __host__ __device__ static constexpr int stride(int n) { return ipow(P1, D - 1 - n); }

    // node id of position a on line m of direction n (operators.py:248-259)
    template <int N>
    __device__ static __forceinline__ int line_node(int m, int a)
    {
        constexpr int stride = ipow(P1, D - 1 - N);
        return (m / stride * P1 + a) * stride + m % stride;
    }
    __device__ static __forceinline__ int pad(int node)
    {
        if constexpr (SWZ && P1 == 4) return node ^ (((node >> 4) * 5) & 15);  // bank pair (node & 15) ^ 5 (node >> 4)
        else if constexpr (SWZ) return node ^ ((node >> 3) & 15);
        else return PADDED ? node + node / P1 : node;
    }
    // accumulator slot of (variable v, element el, node)
    __device__ static __forceinline__ int acc(int v, int el, int node) { return v * FA + el * NNP + pad(node); }
};

// resident-CTA hint for __launch_bounds__ (register cap 64K / (NT * MINB)).
// 3D FAST Cartesian p+1 <= 4: 8 CTAs of 64 threads (128 registers, no spills)
// -- 2.7% faster in steady state than 6 CTAs at 168 registers and one wave for
// cfg2 (profiles/r01_tuning.md); curved kernels spill at 128 registers;
// others: 6 (p+1 <= 5) or as many as fit.
#ifndef FDG_WARPS_HI
#define FDG_WARPS_HI 12  // 3D p + 1 = 6, 7: resident warps per SM the register cap aims at (0: no cap).
#endif                   // 168 registers instead of 254 (N=5 Ranocha VOL 3.35 -> 2.46 ms); p + 1 = 8 holds
                         // 4 CTAs per SM by shared memory, so a cap would only cost registers
#ifndef FDG_WARPS_P7_LOG
#define FDG_WARPS_P7_LOG 8  // p + 1 = 7 with a log-mean flux: 251 registers without spills beat 168 with 384 B
#endif                      // of them (N=6 Ranocha VOL 3.93 -> 3.34 ms; Shima the other way, 1.91 vs 2.29 ms)
template <int D, int P1, int MODE, bool CURVED, int VF = -1>
__host__ __device__ constexpr int min_blocks()
{
    // a target of resident warps per SM (16: 128 registers, 12: 168), turned
    // into CTAs of this degree's size
    constexpr bool log_flux = VF == F_RANOCHA || VF == F_CHANDRASHEKAR;
    constexpr int warps = (MODE == FAST && D == 3 && P1 <= 4 && !CURVED) ? 16
                          : (P1 <= 5 ? 12
                             : ((D == 3 && P1 <= 7) ? ((P1 == 7 && log_flux) ? FDG_WARPS_P7_LOG : FDG_WARPS_HI) : 0));
    constexpr int cta_warps = Geo<D, P1>::NT / 32;
    return FDG_MIN_BLOCKS > 0 ? FDG_MIN_BLOCKS : (warps / cta_warps > 0 ? warps / cta_warps : 1);
}

template <int D, int P1, int VF, int LOGS>
__host__ __device__ constexpr int sq_doubles()
{
    using G = Geo<D, P1>;
    constexpr int prims = (2 + D + n_extra(VF, LOGS)) * G::FS;
    constexpr int faces = G::EPB * G::NF * G::NVAR;
    return prims > faces ? prims : faces;
}

// accumulator / AoS-staging block offset (even: 16-byte aligned bulk copies)
template <int D, int P1, int VF, int LOGS>
__host__ __device__ constexpr int sacc_offset()
{
    return (sq_doubles<D, P1, VF, LOGS>() + 1) & ~1;
}

template <int D, int P1, int VF, int LOGS>
__host__ __device__ constexpr int smem_doubles()
{
    using G = Geo<D, P1>;
    // primitive fields (later: the face-flux buffer) + accumulators (the
    // accumulator block doubles as the AoS staging buffer of u, which is
    // smaller) + the bulk-copy mbarrier
    return sacc_offset<D, P1, VF, LOGS>() + G::NVAR * G::FA + 1;
}

// ---- TMA bulk copy of a batch's state into shared memory (one elected
// thread issues it, an mbarrier counts the bytes; SASS UBLKCP + SYNCS)
#ifndef FDG_TMA
#define FDG_TMA 1
#endif
__device__ __forceinline__ void mbar_init(uint64_t* bar)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar)
{
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"(b)
                 : "memory");
}
// shared -> global bulk copy (one bulk group); the smem source may be reused
// after bulk_wait_read(), the data is globally visible after bulk_wait_all()
__device__ __forceinline__ void bulk_store(void* dst, const void* src, unsigned bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"((unsigned)__cvta_generic_to_shared(src)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase)
{
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(b),
        "r"(phase)
        : "memory");
}

// one batch claim by thread 0, result left in flight. nvcc and ptxas turn an
// atomic add on a uniform address into the warp-aggregated form (leader
// election, one ATOMG, SHFL broadcast of the result), and the shuffle waits
// for the atomic right away: 2.7% of the cfg5 VOL stall samples sat on it
// (r02_v6 capture). The address is therefore offset by (laneid & zero) with
// the lane id read through volatile asm and `zero` a kernel parameter that is
// always 0: not provably uniform, so the plain instruction is emitted and
// its result is only waited for at the end of the batch.
__device__ __forceinline__ long long claim_batch(unsigned long long* counter, int zero)
{
    unsigned lane;
    asm volatile("mov.u32 %0, %%laneid;" : "=r"(lane));
    unsigned long long r;
    asm volatile("atom.global.add.u64 %0, [%1], 1;" : "=l"(r) : "l"(counter + (lane & (unsigned)zero)) : "memory");
    return (long long)r;
}

// compile-time for loop: f(integral_constant<int, i>) for i in [B, E)
template <int B, int E, class F>
__device__ __forceinline__ void sfor(F&& f)
{
    if constexpr (B < E) {
        f(std::integral_constant<int, B>{});
        sfor<B + 1, E>(f);
    }
}

template <int D, int NX>
__device__ __forceinline__ void store_node(double* sq, int fs, int idx, const Node<D, NX>& q)
{
    sq[idx] = q.rho;
#pragma unroll
    for (int i = 0; i < D; ++i) sq[(1 + i) * fs + idx] = q.v[i];
    sq[(1 + D) * fs + idx] = q.p;
#pragma unroll
    for (int j = 0; j < NX; ++j) sq[(2 + D + j) * fs + idx] = q.x[j];
}

template <int D, int NX>
__device__ __forceinline__ Node<D, NX> load_node(const double* sq, int fs, int idx)
{
    Node<D, NX> q;
    q.rho = sq[idx];
#pragma unroll
    for (int i = 0; i < D; ++i) q.v[i] = sq[(1 + i) * fs + idx];
    q.p = sq[(1 + D) * fs + idx];
#pragma unroll
    for (int j = 0; j < NX; ++j) q.x[j] = sq[(2 + D + j) * fs + idx];
    if constexpr (NX == 0) q.x[0] = 0.0;
    return q;
}

// FAST interface terms of one LGL line, fused into the line's volume pass
// (RHS and RK-stage launches, Rusanov flux). The thread that owns line m of
// direction n holds the accumulators of the line's two end nodes in
// registers, and those are exactly the element's face nodes of direction n:
// the -n face at line position 0 (the element is the plus side:
// out -= f / (w_0 J), discretization.py:758-760) and the +n face at position
// p (minus side: out += f / (w_p J)). The accumulators are still unscaled
// (the epilogue multiplies by 1/J), so the lifts enter as f / w. All four
// trace loads are issued before the first flux; no shared-memory round trip,
// no barrier, no per-item index arithmetic. Both sides of an interface still
// evaluate the flux from identical conserved arguments in the same order, so
// the two lifted values are the same double (discrete conservation holds to
// the last bit of the flux). The per-node summation order differs from the
// reference's (VOL/J first, then the faces by direction), which is why only
// the FAST kernels do this; FAITHFUL keeps the reference order below.
// vmap: slot -> conserved variable (identity, or the rotated momentum slots
// of the runtime-direction pass; the flux comes back in the same slots).
// the neighbours' facing traces of line m (plus neighbour's first node,
// minus neighbour's last node), slot v = conserved variable vmap[v]
template <int D, int P1>
__device__ __forceinline__ void line_faces_load(const KParams& prm, const int* vmap, int m, int first, int last, int nbm,
                                                int nbp, double* pf, double* ml)
{
    using G = Geo<D, P1>;
    constexpr int NVAR = G::NVAR, FN = G::LINES;
    const double* sp = nbp >= 0 ? prm.u + ((long long)nbp * G::NN + first) * NVAR
                                : prm.ghost_u + ((long long)(-nbp - 1) * FN + m) * NVAR;
    const double* sm = nbm >= 0 ? prm.u + ((long long)nbm * G::NN + last) * NVAR
                                : prm.ghost_u + ((long long)(-nbm - 1) * FN + m) * NVAR;
#pragma unroll
    for (int v = 0; v < NVAR; ++v) {
        pf[v] = __ldg(sp + vmap[v]);
        ml[v] = __ldg(sm + vmap[v]);
    }
}

// the two Rusanov fluxes of the line's end nodes (own side from the staged
// FAST primitives, flux_llf_fast_own) lifted as f / w into the accumulators
template <int D, int P1, bool CURVED, int AXIS>
__device__ __forceinline__ void line_faces_apply(const KParams& prm, long long e, int n, const int* vmap, int m, int last,
                                                 int nbm, const double* pf, const double* ml, double* acc_first,
                                                 double* acc_last, const double* sq, int sq_first, int sq_last)
{
    using G = Geo<D, P1>;
    constexpr int NVAR = G::NVAR, FN = G::LINES;
    double np[D], nm[D];
    if constexpr (CURVED) {
        const double* jm = nbm >= 0 ? prm.ja + (((long long)nbm * G::NN + last) * D + n) * D
                                    : prm.ghost_nrm + ((long long)(-nbm - 1) * FN + m) * D;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            np[j] = __ldg(prm.ja + ((e * G::NN + last) * D + n) * D + j);
            nm[j] = __ldg(jm + j);
        }
    } else {
#pragma unroll
        for (int j = 0; j < D; ++j) np[j] = nm[j] = (j == AXIS) ? prm.areas[n] : 0.0;
    }
    // own end nodes: staged rho, v/2 (slot j = variable vmap[1+j]), p/2
    double lv[D], fv[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
        lv[j] = sq[vmap[1 + j] * G::FS + sq_last];
        fv[j] = sq[vmap[1 + j] * G::FS + sq_first];
    }
    double f[NVAR];
    flux_llf_fast_own<D, AXIS, true>(sq[sq_last], lv, sq[(1 + D) * G::FS + sq_last], pf, np, prm.gas, f);
#pragma unroll
    for (int v = 0; v < NVAR; ++v) acc_last[v] = fma(prm.inv_wp, f[v], acc_last[v]);
    flux_llf_fast_own<D, AXIS, false>(sq[sq_first], fv, sq[(1 + D) * G::FS + sq_first], ml, nm, prm.gas, f);
#pragma unroll
    for (int v = 0; v < NVAR; ++v) acc_first[v] = fma(-prm.inv_w0, f[v], acc_first[v]);
}

#ifndef FDG_FACE_OWN
#define FDG_FACE_OWN 1  // own end-node states from the staged primitives in shared memory (flux_llf_fast_own): cfg5 RHS 6.35 -> 5.52 ms
#endif
// sq_first / sq_last: shared-memory slots of the line's end nodes (FAST primitives: rho, v/2, p/2)
template <int D, int P1, bool CURVED, int AXIS>
__device__ __forceinline__ void line_faces(const KParams& prm, long long e, int n, const int* vmap, int m, int first,
                                           int last, int nbm, int nbp, double* acc_first, double* acc_last,
                                           const double* sq, int sq_first, int sq_last)
{
    using G = Geo<D, P1>;
    constexpr int NVAR = G::NVAR, FN = G::LINES;
    auto load = [&](const double* src, double* s) {
#pragma unroll
        for (int v = 0; v < NVAR; ++v) s[v] = __ldg(src + vmap[v]);
    };
#if FDG_FACE_OWN
    {
        double pf[NVAR], ml[NVAR];
        line_faces_load<D, P1>(prm, vmap, m, first, last, nbm, nbp, pf, ml);
        line_faces_apply<D, P1, CURVED, AXIS>(prm, e, n, vmap, m, last, nbm, pf, ml, acc_first, acc_last, sq, sq_first,
                                               sq_last);
        return;
    }
#endif
    const double* own = prm.u + e * (long long)(G::NN * NVAR);
    double ol[NVAR], pf[NVAR], ml[NVAR], of[NVAR];
    load(own + last * NVAR, ol);   // +n face: (own last | plus neighbour first)
    load(nbp >= 0 ? prm.u + ((long long)nbp * G::NN + first) * NVAR : prm.ghost_u + ((long long)(-nbp - 1) * FN + m) * NVAR,
         pf);
    load(nbm >= 0 ? prm.u + ((long long)nbm * G::NN + last) * NVAR : prm.ghost_u + ((long long)(-nbm - 1) * FN + m) * NVAR,
         ml);                      // -n face: (minus neighbour last | own first)
    load(own + first * NVAR, of);
    double np[D], nm[D];
    if constexpr (CURVED) {
        const double* jm = nbm >= 0 ? prm.ja + (((long long)nbm * G::NN + last) * D + n) * D
                                    : prm.ghost_nrm + ((long long)(-nbm - 1) * FN + m) * D;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            np[j] = __ldg(prm.ja + ((e * G::NN + last) * D + n) * D + j);
            nm[j] = __ldg(jm + j);
        }
    } else {
#pragma unroll
        for (int j = 0; j < D; ++j) np[j] = nm[j] = (j == AXIS) ? prm.areas[n] : 0.0;
    }
    double f[NVAR];
    flux_llf_fast<D, AXIS>(ol, pf, np, prm.gas, f);
#pragma unroll
    for (int v = 0; v < NVAR; ++v) acc_last[v] = fma(prm.inv_wp, f[v], acc_last[v]);
    flux_llf_fast<D, AXIS>(ml, of, nm, prm.gas, f);
#pragma unroll
    for (int v = 0; v < NVAR; ++v) acc_first[v] = fma(-prm.inv_w0, f[v], acc_first[v]);
}

// One direction of the volume integral for the thread's line.
// KP: FAST Chandrashekar nodes of a volume-only launch carry |v/2|^2 in the pressure slot
template <int D, int P1, int VF, int MODE, int EPIK>
__host__ __device__ constexpr int kin_in_p()
{
    return (FDG_CHANDRA_KP && MODE == FAST && VF == F_CHANDRASHEKAR && EPIK == 0 /* EPI_VOLUME */) ? 1 : 0;
}
template <int D, int P1, int VF, bool CURVED, int MODE, int LOGS, int N, bool FIRST = (N == 0), int KP = 0>
__device__ __forceinline__ void volume_direction(const KParams& prm, const double* sq, double* sacc, int el,
                                                 int m, long long e, unsigned vm, bool faces = false, int nbm = 0,
                                                 int nbp = 0, double* aos = nullptr)
{
    using G = Geo<D, P1>;
    constexpr int NVAR = G::NVAR;
    constexpr int NX = n_extra(VF, LOGS);
    double acc[P1][NVAR];
    int nodes[P1];
#pragma unroll
    for (int a = 0; a < P1; ++a) nodes[a] = G::template line_node<N>(m, a);
    if constexpr (FIRST) {
#pragma unroll
        for (int a = 0; a < P1; ++a)
#pragma unroll
            for (int v = 0; v < NVAR; ++v) acc[a][v] = 0.0;
    } else {
#pragma unroll
        for (int a = 0; a < P1; ++a)
#pragma unroll
            for (int v = 0; v < NVAR; ++v) acc[a][v] = sacc[G::acc(v, el, nodes[a])];
    }
    double jl[CURVED ? P1 : 1][D];
    if constexpr (CURVED) {
#pragma unroll
        for (int a = 0; a < P1; ++a)
#pragma unroll
            for (int j = 0; j < D; ++j) jl[a][j] = __ldg(prm.ja + ((e * G::NN + nodes[a]) * D + N) * D + j);
    }
    const int sbase = el * G::NNP;
#if FDG_LINE_REGS
    // the whole line's node data in registers: P1 shared-memory loads per node
    // instead of one per pair it takes part in
    Node<D, NX> qline[P1];
    sfor<0, P1>([&](auto A) {
        constexpr int a = decltype(A)::value;
        qline[a] = load_node<D, NX>(sq, G::FS, sbase + G::pad(nodes[a]));
    });
#endif
    // compile-time pair loops (a < b in pair-table order): keeps acc/jl in registers
    sfor<0, P1>([&](auto A) {
        constexpr int a = decltype(A)::value;
#if FDG_LINE_REGS
        const Node<D, NX>& qa = qline[a];
#else
        const Node<D, NX> qa = load_node<D, NX>(sq, G::FS, sbase + G::pad(nodes[a]));
#endif
        sfor<a + 1, P1>([&](auto B) {
            constexpr int b = decltype(B)::value;
            // every off-diagonal LGL Dsplit entry is nonzero (checked at mesh
            // creation), so the reference's pair table visits every pair
            const double wa = prm.wts[N][a * P1 + b];
            const double wb = prm.wts[N][b * P1 + a];
            constexpr int EH = (MODE == FAST && energy_half(VF)) ? 1 : 0;
#if FDG_LINE_REGS
            const Node<D, NX>& qb = qline[b];
#else
            const Node<D, NX> qb = load_node<D, NX>(sq, G::FS, sbase + G::pad(nodes[b]));
#endif
            double f[NVAR];
            if constexpr (CURVED) {
                double alpha[D];
#pragma unroll
                for (int j = 0; j < D; ++j) alpha[j] = 0.5 * (jl[a][j] + jl[b][j]);
                volume_flux<D, VF, -1, MODE, LOGS, EH, KP>(qa, qb, alpha, prm.gas, prm.precompute, f, vm);
            } else {
                volume_flux<D, VF, N, MODE, LOGS, EH, KP>(qa, qb, nullptr, prm.gas, prm.precompute, f, vm);
            }
#pragma unroll
            for (int v = 0; v < NVAR - EH; ++v) {
                acc[a][v] += wa * f[v];
                acc[b][v] += wb * f[v];
            }
            if constexpr (EH) {  // f[NVAR-1] = f_E / 2, weights doubled: the same product, exactly
                acc[a][NVAR - 1] += prm.wtsE[N][a * P1 + b] * f[NVAR - 1];
                acc[b][NVAR - 1] += prm.wtsE[N][b * P1 + a] * f[NVAR - 1];
            }
        });
    });
    if constexpr (MODE == FAST) {
        if (faces) {
            int ident[NVAR];
#pragma unroll
            for (int v = 0; v < NVAR; ++v) ident[v] = v;
            line_faces<D, P1, CURVED, CURVED ? -1 : N>(prm, e, N, ident, m, nodes[0], nodes[P1 - 1], nbm, nbp, acc[0],
                                                        acc[P1 - 1], sq, sbase + G::pad(nodes[0]),
                                                        sbase + G::pad(nodes[P1 - 1]));
        }
    }
    // FDG_AOS_LAST: the last pass of a volume-only launch (lines of P1
    // consecutive nodes; values final: 1/J is folded into the weights) leaves
    // its results as AoS straight in the primitive region for the bulk store
    // -- once every thread of the CTA is past its pair loop, nothing reads the
    // primitives any more -- instead of SoA accumulators that the epilogue
    // reads back and transposes (40 shared-memory instructions per thread).
    // Called by every thread of the CTA (the barrier).
    if (aos) {
        __syncthreads();
#pragma unroll
        for (int a = 0; a < P1; ++a)
#pragma unroll
            for (int v = 0; v < NVAR; ++v) aos[(el * G::NN + nodes[a]) * NVAR + v] = acc[a][v];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        return;
    }
#pragma unroll
    for (int a = 0; a < P1; ++a)
#pragma unroll
        for (int v = 0; v < NVAR; ++v) sacc[G::acc(v, el, nodes[a])] = acc[a][v];
}

template <int D, int P1>
__device__ __forceinline__ int line_stride(int n)  // P1^(D-1-n) without a runtime power loop
{
    return D == 3 ? (n == 0 ? P1 * P1 : (n == 1 ? P1 : 1)) : (n == 0 ? P1 : 1);
}

// ---------------------------------------------------------------------------
// FAST volume pass with a RUNTIME direction n: one copy of the pair code for
// all d directions (the compile-time passes triple the kernel's SASS: 190 KB
// at p+1 = 8, where ncu showed 10.8% "no instruction" stalls). Cartesian
// meshes load every node's velocity ROTATED, v'_j = v_{(n+j) mod d}, and call
// the axis-0 flux: for an axis-aligned direction the fluxes are rotation
// covariant, so the rotated momentum components come out in the same slots
// and go back to their variables through the same map when the accumulators
// are loaded and stored (addresses only, no selects). Curved meshes use the
// general-normal flux with the direction's metric row. Not for FAITHFUL (the
// rotation reorders dot-product sums) nor the central flux (its staged
// conserved momenta would need the same rotation).
#ifndef FDG_RT_DIR_MIN_P1
#define FDG_RT_DIR_MIN_P1 5  // p+1 = 4: 7% slower; 5: cfg4 RHS +5%; 8: cfg3 +3-16% (profiles/r01_tuning.md)
#endif
#ifndef FDG_RT_DIR_MIN_P1_VOLK
#define FDG_RT_DIR_MIN_P1_VOLK 8  // N=4/5/6 Ranocha VOL: 2.51 -> 2.27, 2.51 -> 2.22, 4.50 -> 3.91 ms
#endif
template <int D, int P1, int VF>
__host__ __device__ constexpr bool runtime_direction()
{
    return P1 >= FDG_RT_DIR_MIN_P1 && VF != F_CENTRAL;
}
// interface epilogues (RHS, RK stage) of the FAST kernels below that degree
// also take the runtime-direction pass: the RHS kernel executes the volume
// passes AND the face / stage code, and with three compile-time volume
// passes its executed footprint overflowed the instruction cache (cfg5 RHS,
// ncu r02: "no instruction" the largest stall reason, 22% of samples)
#ifndef FDG_RT_DIR_IFACE
#define FDG_RT_DIR_IFACE 1
#endif
template <int D, int P1, int VF>
__host__ __device__ constexpr bool runtime_direction_iface()
{
    return FDG_RT_DIR_IFACE && VF != F_CENTRAL && !runtime_direction<D, P1, VF>();
}

template <int D, int P1, int VF, bool CURVED, int LOGS, int KP = 0>
__device__ __forceinline__ void volume_direction_rt(const KParams& prm, const double* sq, double* sacc, int el, int m,
                                                    long long e, int n, bool first, unsigned vm, bool faces = false,
                                                    int nbm = 0, int nbp = 0)
{
    using G = Geo<D, P1>;
    constexpr int NVAR = G::NVAR;
    constexpr int NX = n_extra(VF, LOGS);
    const int stride = line_stride<D, P1>(n);
    // line position 0: (m / stride) P1 stride + m % stride, with the three
    // compile-time strides spelled out (no runtime division)
    const int base = (n == 0) ? m : ((D == 3 && n == 1) ? (m / P1) * P1 * P1 + m % P1 : m * P1);
    // variable / field index of rotated slot j (rho, v'_0..v'_{d-1}, E | p, extras)
    int vmap[NVAR];
    vmap[0] = 0;
    vmap[NVAR - 1] = NVAR - 1;
#pragma unroll
    for (int j = 0; j < D; ++j) vmap[1 + j] = CURVED ? 1 + j : 1 + (n + j >= D ? n + j - D : n + j);
    double acc[P1][NVAR];
#pragma unroll
    for (int a = 0; a < P1; ++a) {
        const int nd = base + a * stride;
#pragma unroll
        for (int v = 0; v < NVAR; ++v) acc[a][v] = first ? 0.0 : sacc[G::acc(vmap[v], el, nd)];
    }
    const int sbase = el * G::NNP;
    auto load = [&](int a) {
        const int idx = sbase + G::pad(base + a * stride);
        Node<D, NX> q;
        q.rho = sq[idx];
#pragma unroll
        for (int j = 0; j < D; ++j) q.v[j] = sq[vmap[1 + j] * G::FS + idx];
        q.p = sq[(1 + D) * G::FS + idx];
#pragma unroll
        for (int k = 0; k < NX; ++k) q.x[k] = sq[(2 + D + k) * G::FS + idx];
        if constexpr (NX == 0) q.x[0] = 0.0;
        return q;
    };
    const double* w = prm.wts[n];
    constexpr int EH = energy_half(VF) ? 1 : 0;
    [[maybe_unused]] const double* wE = prm.wtsE[n];
    // curved meshes: the line's metric rows Ja^n (P1 x D values) are loaded
    // once, all loads in flight together, instead of two rows per pair inside
    // the pair loop (cfg4 RHS, r02 s5 capture: 13.8% of the stall samples sat
    // on those loads)
#ifndef FDG_RT_JL_MAXP1
#define FDG_RT_JL_MAXP1 5  // with the line's node data in registers too (FDG_RT_LINE_REGS_MAXP1): the pair loop
                           // runs on registers only, cfg4 RHS 0.925 -> 0.900 ms (either one alone: 0.95 - 0.96 ms)
#endif
    constexpr bool JLR = CURVED && P1 <= FDG_RT_JL_MAXP1;
    [[maybe_unused]] double jl[JLR ? P1 : 1][D];
    if constexpr (JLR) {
#pragma unroll
        for (int a = 0; a < P1; ++a)
#pragma unroll
            for (int j = 0; j < D; ++j) jl[a][j] = __ldg(prm.ja + ((e * G::NN + base + a * stride) * D + n) * D + j);
    }
    // FDG_FACE_EARLY: where the neighbour-trace loads of the fused interface
    // terms are issued -- 0: after the pair loop (with the fluxes), 1: before
    // the last pair (one flux evaluation hides the L2 latency), 2: before
    // the pair loop
#ifndef FDG_FACE_EARLY
#define FDG_FACE_EARLY 0
#endif
    constexpr bool EARLY = FDG_FACE_OWN && FDG_FACE_EARLY > 0;
    [[maybe_unused]] double pf[NVAR], ml[NVAR];
    if constexpr (EARLY && FDG_FACE_EARLY == 2) {
        if (faces) line_faces_load<D, P1>(prm, vmap, m, base, base + (P1 - 1) * stride, nbm, nbp, pf, ml);
    }
    // whole line in registers up to this degree (P1 shared-memory node loads
    // per pass instead of P1 + P1 (P1 - 1) / 2)
#ifndef FDG_RT_LINE_REGS_MAXP1
#define FDG_RT_LINE_REGS_MAXP1 5  // (with FDG_RT_JL_MAXP1) cfg4 RHS 0.925 -> 0.900 ms, SSPRK43 step 4.38 -> 4.30 ms
#endif
    // (not below p + 1 = 5: the p + 1 = 4 RHS twin lives at 128 registers, cfg5 RHS 4.95 -> 5.24 ms with it)
    constexpr bool LREG = P1 >= 5 && P1 <= FDG_RT_LINE_REGS_MAXP1;
    [[maybe_unused]] Node<D, NX> qline[LREG ? P1 : 1];
    if constexpr (LREG) {
#pragma unroll
        for (int a = 0; a < P1; ++a) qline[a] = load(a);
    }
    sfor<0, P1>([&](auto A) {
        constexpr int a = decltype(A)::value;
        Node<D, NX> qa;
        if constexpr (LREG) qa = qline[a];
        else qa = load(a);
        sfor<a + 1, P1>([&](auto B) {
            constexpr int b = decltype(B)::value;
            if constexpr (EARLY && FDG_FACE_EARLY == 1 && a == P1 - 2 && b == P1 - 1) {
                if (faces) line_faces_load<D, P1>(prm, vmap, m, base, base + (P1 - 1) * stride, nbm, nbp, pf, ml);
            }
            Node<D, NX> qb;
            if constexpr (LREG) qb = qline[b];
            else qb = load(b);
            const double wa = w[a * P1 + b];
            const double wb = w[b * P1 + a];
            double f[NVAR];
            if constexpr (CURVED) {
                double alpha[D];
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    if constexpr (JLR)
                        alpha[j] = 0.5 * (jl[a][j] + jl[b][j]);
                    else
                        alpha[j] = 0.5 * (__ldg(prm.ja + ((e * G::NN + base + a * stride) * D + n) * D + j) +
                                          __ldg(prm.ja + ((e * G::NN + base + b * stride) * D + n) * D + j));
                }
                fast_volume_flux<D, VF, -1, LOGS, EH, KP>(qa, qb, alpha, prm.gas.igm1, f, vm);
            } else {
                fast_volume_flux<D, VF, 0, LOGS, EH, KP>(qa, qb, nullptr, prm.gas.igm1, f, vm);
            }
#pragma unroll
            for (int v = 0; v < NVAR - EH; ++v) {
                acc[a][v] = fma(wa, f[v], acc[a][v]);
                acc[b][v] = fma(wb, f[v], acc[b][v]);
            }
            if constexpr (EH) {
                acc[a][NVAR - 1] = fma(wE[a * P1 + b], f[NVAR - 1], acc[a][NVAR - 1]);
                acc[b][NVAR - 1] = fma(wE[b * P1 + a], f[NVAR - 1], acc[b][NVAR - 1]);
            }
        });
    });
    if (faces) {
        if constexpr (EARLY)
            line_faces_apply<D, P1, CURVED, CURVED ? -1 : 0>(prm, e, n, vmap, m, base + (P1 - 1) * stride, nbm, pf, ml,
                                                              acc[0], acc[P1 - 1], sq, sbase + G::pad(base),
                                                              sbase + G::pad(base + (P1 - 1) * stride));
        else
            line_faces<D, P1, CURVED, CURVED ? -1 : 0>(prm, e, n, vmap, m, base, base + (P1 - 1) * stride, nbm, nbp,
                                                        acc[0], acc[P1 - 1], sq, sbase + G::pad(base),
                                                        sbase + G::pad(base + (P1 - 1) * stride));
    }
#pragma unroll
    for (int a = 0; a < P1; ++a) {
        const int nd = base + a * stride;
#pragma unroll
        for (int v = 0; v < NVAR; ++v) sacc[G::acc(vmap[v], el, nd)] = acc[a][v];
    }
}

template <int D, int P1, int VF, bool CURVED, int MODE, int LOGS, int N, bool FIRST, int KP = 0>
__device__ __forceinline__ void vdir(const KParams& prm, const double* sq, double* sacc, int el, int m, long long e,
                                     bool active, unsigned vm, bool fuse = false, const int* nb = nullptr,
                                     double* aos = nullptr)
{
    if constexpr (MODE == FAST) {
        if (vm) {
            const bool faces = fuse && active;
            volume_direction<D, P1, VF, CURVED, MODE, LOGS, N, FIRST, KP>(prm, sq, sacc, el, m, active ? e : e - el, vm,
                                                                       faces, faces ? nb[(el * D + N) * 2] : 0,
                                                                       faces ? nb[(el * D + N) * 2 + 1] : 0, aos);
        }
    } else {
        if (active) volume_direction<D, P1, VF, CURVED, MODE, LOGS, N, FIRST, KP>(prm, sq, sacc, el, m, e, 0u);
    }
}

template <int D>
__device__ __forceinline__ void load_state(const double* src, double* s)
{
#pragma unroll
    for (int v = 0; v < D + 2; ++v) s[v] = __ldg(src + v);
}

// Interface flux: Rusanov inline (the common case, registers only), the other
// kinds through the out-of-line dispatcher.
template <int D, bool CURVED, int MODE, int N>
__device__ __forceinline__ void face_flux(const KParams& prm, const double* ul, const double* ur, const double* nrm,
                                          double* f)
{
    if (prm.surface_flux == F_LLF) {
        if constexpr (MODE == FAST) flux_llf_fast<D, CURVED ? -1 : N>(ul, ur, nrm, prm.gas, f);
        else flux_llf<D, MODE>(ul, ur, nrm, prm.gas, f);
    } else {
        // copies: only these arrays have their address taken by the
        // out-of-line call, the caller's stay in registers
        double a[D + 2], b[D + 2], nn[D], g[D + 2];
#pragma unroll
        for (int v = 0; v < D + 2; ++v) {
            a[v] = ul[v];
            b[v] = ur[v];
        }
#pragma unroll
        for (int j = 0; j < D; ++j) nn[j] = nrm[j];
        surface_flux<D, MODE>(prm.surface_flux, a, b, nn, prm.gas, g);
#pragma unroll
        for (int v = 0; v < D + 2; ++v) f[v] = g[v];
    }
}

// Interface flux of one face node of element e: direction n, side 1 = its
// +n face (e is the minus element), side 0 = its -n face (e is the plus
// element); line m of direction n. Same arguments from both adjacent
// elements, so both see identical bits (discretization.py:730-760 evaluates
// each face once and scatters both ways).

template <int D, int P1, bool CURVED, int MODE>
__device__ __forceinline__ void face_flux_item(const KParams& prm, long long e, int n, int side, int m, double* f,
                                               int nb_pre = 0)
{
    using G = Geo<D, P1>;
    constexpr int NVAR = G::NVAR;
    constexpr int FN = G::LINES;
    const int stride = line_stride<D, P1>(n);
    const int hi = m / stride, lo = m - hi * stride;
    const int first = hi * P1 * stride + lo;         // line position 0
    const int last = first + (P1 - 1) * stride;      // line position p
    double ul[NVAR], ur[NVAR], nrm[D];
    if (side) {
        load_state<D>(prm.u + (e * G::NN + last) * NVAR, ul);
        const int nb = FDG_NB_SMEM ? nb_pre : __ldg(prm.plus + n * prm.n_elem + e);
        if (nb >= 0) load_state<D>(prm.u + ((long long)nb * G::NN + first) * NVAR, ur);
        else load_state<D>(prm.ghost_u + ((long long)(-nb - 1) * FN + m) * NVAR, ur);
        if constexpr (CURVED) {
#pragma unroll
            for (int j = 0; j < D; ++j) nrm[j] = __ldg(prm.ja + ((e * G::NN + last) * D + n) * D + j);
        }
    } else {
        const int nb = FDG_NB_SMEM ? nb_pre : __ldg(prm.minus + n * prm.n_elem + e);
        if (nb >= 0) {
            load_state<D>(prm.u + ((long long)nb * G::NN + last) * NVAR, ul);
            if constexpr (CURVED) {
#pragma unroll
                for (int j = 0; j < D; ++j) nrm[j] = __ldg(prm.ja + (((long long)nb * G::NN + last) * D + n) * D + j);
            }
        } else {
            const long long g = -nb - 1;
            load_state<D>(prm.ghost_u + (g * FN + m) * NVAR, ul);
            if constexpr (CURVED) {
#pragma unroll
                for (int j = 0; j < D; ++j) nrm[j] = __ldg(prm.ghost_nrm + (g * FN + m) * D + j);
            }
        }
        load_state<D>(prm.u + (e * G::NN + first) * NVAR, ur);
    }
    if constexpr (!CURVED) {
#pragma unroll
        for (int j = 0; j < D; ++j) nrm[j] = (j == n) ? prm.areas[n] : 0.0;
    }
    // one general-normal code path for every direction (a Cartesian face is
    // the normal area e_n): keeps the RHS kernel inside the instruction cache
    face_flux<D, true, MODE, 0>(prm, ul, ur, nrm, f);
}

#if FDG_PHASE_TIMING
// profiling build only (scripts/ab.sh "pt:.:-DFDG_PHASE_TIMING=1"): SM cycles per phase, summed over CTAs/batches
__device__ unsigned long long fdg_phase_cycles[8];
__device__ unsigned long long fdg_cta_ns[3 * 8192];  // per-CTA globaltimer start/end, SM id
extern "C" int fdg_debug_phase_cycles(unsigned long long* out, int reset)
{
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, fdg_phase_cycles, sizeof(fdg_phase_cycles));
    if (reset) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(fdg_phase_cycles, z, sizeof(z));
    }
    return 0;
}
extern "C" int fdg_debug_cta_ns(unsigned long long* out, int n)
{
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, fdg_cta_ns, sizeof(unsigned long long) * 3 * n);
    return 0;
}
#define FDG_PT(i)                          \
    if (tid == 0) {                        \
        const long long t_ = clock64();    \
        pt_[i] += t_ - pt_last_;           \
        pt_last_ = t_;                     \
    }
#else
#define FDG_PT(i)
#endif

// OCC > 0 overrides the resident-CTA hint (the high-occupancy twin used when a
// launch fits one wave only at that occupancy, fdg_dispatch.cuh)
// EPIK >= 0 fixes the epilogue at compile time (the volume-integral-only
// twin: no interface / stage code in the kernel image, fdg_dispatch.cuh)
template <int D, int P1, int VF, bool CURVED, int MODE, int LOGS, int OCC = 0, int EPIK = -1>
__global__ void __launch_bounds__(Geo<D, P1>::NT, OCC > 0 ? OCC : min_blocks<D, P1, MODE, CURVED, VF>())
    elem_kernel(const __grid_constant__ KParams prm)
{
    using G = Geo<D, P1>;
    constexpr int NN = G::NN, NVAR = G::NVAR, EPB = G::EPB, NT = G::NT;
    constexpr int NX = n_extra(VF, LOGS);
    constexpr int KP = kin_in_p<D, P1, VF, MODE, EPIK>();
    constexpr int KU = (EPB * NN * NVAR + NT - 1) / NT;  // state values per thread
    constexpr int KN = (EPB * NN + NT - 1) / NT;         // nodes per thread
    extern __shared__ double smem[];
    double* sq = smem;                        // (2+D+NX) fields x FS
    double* sacc = smem + sacc_offset<D, P1, VF, LOGS>();  // NVAR x FA (AoS u staging before the volume pass)
    const int tid = threadIdx.x;
    // full batches are 16-byte multiples (so every batch starts 16-byte
    // aligned) and u is 16-byte aligned: a batch arrives by one bulk copy
    // (a ragged last batch of odd size, or a misaligned u: the per-thread
    // copy loop)
    constexpr bool TMA_SHAPE = FDG_TMA && (EPB * NN * NVAR) % 2 == 0;
    const bool tma_u = TMA_SHAPE && (reinterpret_cast<uintptr_t>(prm.u) & 15) == 0;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sacc + G::NVAR * G::FA);
    // VOL leaves as AoS through the (then free) primitive region by a bulk store
    const int epi = EPIK >= 0 ? EPIK : prm.epilogue;
    // FAST: directions in descending order, so the fused interface terms of
    // direction 0 (neighbours farthest away in the element order, their face
    // rows prefetched into L2 at batch start) are read last; the per-node sum
    // order is free in FAST mode (FAITHFUL keeps the reference's 0..d-1)
    constexpr bool REV = FDG_DIR_REV && MODE == FAST;
    const bool tma_out_ok = TMA_SHAPE && epi != EPI_STAGE && (reinterpret_cast<uintptr_t>(prm.out) & 15) == 0;
    bool tma_pending = false;  // a bulk store may still be reading the primitive region
    unsigned phase = 0;
    if (TMA_SHAPE && tid == 0) mbar_init(bar);
    if (TMA_SHAPE) __syncthreads();
#if FDG_PDL
    // launched with programmatic stream serialization (fdg_dispatch.cuh):
    // everything above touches only registers and the parameter bank
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
#if FDG_PHASE_TIMING
    long long pt_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long pt_last_ = clock64();
    unsigned long long ns0_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns0_));
#endif
    const int el = tid / G::LINES;
    const int m = tid % G::LINES;
    // lanes holding a line of the batch: the FAST volume phases run on all of
    // them (lanes of absent elements in a ragged last batch compute on stale
    // shared data that is never stored), so the series-branch vote sees whole
    // warps -- a compile-time full mask when the CTA has no spare threads
    constexpr int USED = EPB * G::LINES;
    const unsigned vmask = (USED == NT) ? 0xffffffffu : __ballot_sync(0xffffffffu, tid < USED) * (tid < USED);
    const long long nb1 = (prm.range_hi - prm.range_lo + EPB - 1) / EPB;
    const long long nbatch = nb1 + (prm.range2_hi - prm.range2_lo + EPB - 1) / EPB;
    auto range_end = [&](long long b) -> long long { return b < nb1 ? prm.range_hi : prm.range2_hi; };
#if FDG_NB_SMEM
    __shared__ int s_nb[EPB * 2 * D];
    // FAST RHS / RK-stage launches with the Rusanov flux: interface terms
    // fused into the volume passes (line_faces), no separate face phase
    // (EPIK = RHS / STAGE twins are only launched when this holds)
    const bool fuse = (EPIK == EPI_RHS || EPIK == EPI_STAGE) ||
                      (MODE == FAST && VF != F_CENTRAL && prm.fuse_faces && (epi == EPI_RHS || epi == EPI_STAGE) &&
                       prm.surface_flux == F_LLF);
#else
    constexpr bool fuse = false;
    const int* s_nb = nullptr;
#endif

    // traversal order: batch b covers elements [first(b), first(b) + EPB).
    // With a row order (fdg_mesh_set_traversal) the rows of the element
    // index space are visited tile by tile, so the +-x / +-y neighbours a
    // batch's interface terms read are staged by CTAs of the same wave (L2
    // hits) instead of 16384 elements away; batches never straddle rows.
    const bool remap = prm.row_order && (prm.row_len % EPB) == 0 && prm.range_lo == 0 && prm.range_hi == prm.n_elem;
    auto first = [&](long long b) -> long long {
        const long long f = b < nb1 ? prm.range_lo + b * EPB : prm.range2_lo + (b - nb1) * EPB;
        if (!remap) return f;
        // (element indices fit 31 bits -- the neighbour tables are int32 --
        // so the row split is one 32-bit division)
        const unsigned rl = (unsigned)prm.row_len;
        const unsigned r = (unsigned)f / rl;
        return (long long)__ldg(prm.row_order + r) * prm.row_len + ((unsigned)f - r * rl);
    };

    // batch assignment: static grid-stride, or dynamic claiming, one batch at
    // a time, from a per-mesh counter (prm.claim): no tail imbalance (r02_v2
    // capture: 3.36 of 4 warps per scheduler active on average with the static
    // order, 3.98 with claiming; cfg5 VOL 3.87 -> 3.57 ms), and a CTA that
    // becomes resident late (SMs held by the halo exchange's NCCL kernels next
    // to an interior launch) takes fewer batches instead of stretching the
    // tail. Claims run ONE BATCH AHEAD: while batch i is processed the CTA
    // already knows batch i+1 (so the L2 prefetch below is exact) and thread
    // 0's atomic for batch i+2 is in flight, its result parked in a register
    // until the end of the iteration (no exposed atomic latency).
    const bool dyn = prm.claim != nullptr;
    __shared__ long long s_claim[2];
    long long batch = blockIdx.x, next = 0;
    [[maybe_unused]] long long pending = 0;
    if (dyn) {
        if (tid == 0) {
            s_claim[0] = claim_batch(prm.claim, prm.zero);
            s_claim[1] = claim_batch(prm.claim, prm.zero);
        }
        __syncthreads();
        batch = s_claim[0];
        next = s_claim[1];
        __syncthreads();
    }
    auto advance = [&]() {
        if (!dyn) {
            batch += gridDim.x;
            return;
        }
        if (tid == 0) s_claim[0] = pending;
        __syncthreads();  // (every iteration has a block barrier between this read and the next write)
        batch = next;
        next = s_claim[0];
    };
    // first element of the current batch; the next batch's is computed once,
    // for the L2 prefetch, and carried into the next iteration
    long long e0_cur = batch < nbatch ? first(batch) : 0, e0_next = 0;
    for (; batch < nbatch; advance(), e0_cur = e0_next) {
        if (dyn && tid == 0) pending = claim_batch(prm.claim, prm.zero);
        const long long e0 = e0_cur;
        const int ne = (int)min((long long)EPB, range_end(batch) - e0);
        const long long base = e0 * NN * NVAR;
        const int count = ne * NN * NVAR;
        const long long e = e0 + el;
        const bool active = (el < ne);
        // (a batch starting at an odd double offset -- odd-size elements in a
        // range launch starting at an odd element -- takes the copy loops)
        const bool tma = tma_u && (count % 2) == 0 && (base % 2) == 0;
        const bool tma_out = tma_out_ok && (count % 2) == 0 && (base % 2) == 0;

        const long long nb_next = !dyn ? batch + gridDim.x : next;
        if (nb_next < nbatch) e0_next = first(nb_next);
#if FDG_PREFETCH
        // warm L2 with the next batch of this CTA (its state, and metrics on
        // curved meshes) while this one computes: the next staging copy then
        // waits on L2, not HBM, latency
        {
            const long long nb = nb_next;
            if (nb < nbatch) {
                const long long f2 = e0_next;
                const long long ne2 = min((long long)EPB, range_end(nb) - f2);
                const char* p0 = reinterpret_cast<const char*>(prm.u + f2 * NN * NVAR);
                const int bytes = (int)(ne2 * NN * NVAR * 8);
                for (int off = tid * 128; off < bytes; off += NT * 128)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(p0 + off));
                if constexpr (CURVED) {
                    const char* p1 = reinterpret_cast<const char*>(prm.ja + f2 * NN * D * D);
                    const int b1 = (int)(ne2 * NN * D * D * 8);
                    for (int off = tid * 128; off < b1; off += NT * 128)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(p1 + off));
                }
            }
        }
#endif
#if FDG_FACE_PREFETCH
        // interface epilogues on states much larger than L2 (prm.face_prefetch,
        // set at mesh creation): warm L2 with the face rows of this batch's
        // neighbours in directions 0 and 1 now, so the face phase (after the
        // volume passes) finds them there. Those neighbours are far ahead /
        // behind in the traversal (128^3: +-16384 and +-128 elements) and
        // their face loads went to DRAM (cfg5 RHS: 12.6 GB read per launch for
        // a 5.4 GB state; the prefetch: 10.45 -> 9.93 ms; on L2-resident
        // meshes it costs 1-3%). Direction-2 neighbours are adjacent elements.
        if (prm.face_prefetch && epi != EPI_VOLUME && D == 3) {
            constexpr int NFP = EPB * 4;  // (element, neighbour) items: -0, +0, -1, +1
            for (int it = tid; it < NFP; it += NT) {
                const int fel = it >> 2, which = it & 3, n = which >> 1, plus = which & 1;
                if (fel < ne) {
                    const int nb = __ldg((plus ? prm.plus : prm.minus) + n * prm.n_elem + e0 + fel);
                    if (nb >= 0) {
                        // the neighbour's face adjacent to e: position 0 (plus
                        // neighbour) or P1-1 (minus neighbour) along direction n
                        constexpr int S0 = P1 * P1;
                        const int stride = n == 0 ? S0 : P1;
                        const int a = plus ? 0 : P1 - 1;
                        const char* blk = reinterpret_cast<const char*>(prm.u + (long long)nb * NN * NVAR);
                        const int runs = n == 0 ? 1 : P1, run_nodes = n == 0 ? S0 : P1;
                        for (int r = 0; r < runs; ++r) {
                            const int node0 = (r * P1 + a) * stride;  // (hi, a, lo = 0)
                            const char* p = blk + (long long)node0 * NVAR * 8;
                            for (int off = 0; off < run_nodes * NVAR * 8; off += 128)
                                asm volatile("prefetch.global.L2 [%0];" ::"l"(p + off));
                        }
                    }
                }
            }
        }
#endif
#if FDG_NB_SMEM
        // the batch's 2D neighbour indices, read now (their latency hides
        // behind the volume passes) for the interface phase; the previous
        // batch's readers passed the face phase's last barrier
        if (epi != EPI_VOLUME)
            for (int it = tid; it < EPB * 2 * D; it += NT) {
                const int fel = it / (2 * D), r = it - fel * 2 * D, n = r >> 1, side = r & 1;
                s_nb[it] = (fel < ne) ? __ldg((side ? prm.plus : prm.minus) + n * prm.n_elem + e0 + fel) : 0;
            }
#endif
        if (epi != EPI_SURFACE) {
            // ---- stage: coalesced copy (AoS), then primitives per node (SoA).
            // Compile-time trip counts: every load of the batch is in flight
            // before the first shared-memory store, and the per-node chains
            // (division, reciprocal, logs) of one thread run side by side.
            FDG_PT(7)
            if (tma) {
                if (tid == 0) {
                    bulk_load(sacc, prm.u + base, (unsigned)count * 8u, bar);
                    if (tma_pending) bulk_wait_read();  // the previous batch's VOL has left the primitive region
                }
                mbar_wait(bar, phase);
                phase ^= 1u;
            } else {
                if (tma_pending && tid == 0) bulk_wait_read();
                constexpr int CH = KU < 24 ? KU : 16;
#pragma unroll
                for (int k0 = 0; k0 < KU; k0 += CH) {
                    double tmp[CH];
#pragma unroll
                    for (int k = 0; k < CH; ++k) {
                        const int t = tid + (k0 + k) * NT;
                        tmp[k] = (k0 + k < KU && t < count) ? __ldg(prm.u + base + t) : 0.0;
                    }
#pragma unroll
                    for (int k = 0; k < CH; ++k) {
                        const int t = tid + (k0 + k) * NT;
                        if (k0 + k < KU && t < count) sacc[t] = tmp[k];
                    }
                }
            }
            __syncthreads();
            FDG_PT(0)
            {
                // the gate's rare paths leave the node loop: its body is
                // straight-line arithmetic that ptxas can interleave
                unsigned slow = 0;                     // FAST: nodes needing the reference pressure test
                unsigned bad = ~0u;                    // first failing flat node of this thread (batch-local index)
#pragma unroll(kStageUnroll)
                for (int k = 0; k < KN; ++k) {
                    const int t = tid + k * NT;
                    if (t < ne * NN) {
                        const int tel = t / NN, node = t - tel * NN;
                        const double* su = sacc + t * NVAR;
                        Node<D, NX> q = make_node<D, VF, MODE, LOGS, EPIK == EPI_VOLUME>(su, prm.gas.gm1);
                        if constexpr (MODE == FAST) {
                            const int g = gate_fast<D>(su, q.p, prm.gas.gm1);  // 1 ok, 0 bad, -1 undecided
                            slow |= (g < 0) ? (1u << k) : 0u;
                            bad = (g == 0 && (unsigned)t < bad) ? (unsigned)t : bad;
                        } else {
                            bad = (!gate_ok<D>(su, prm.gas.gm1) && (unsigned)t < bad) ? (unsigned)t : bad;
                        }
                        if constexpr (KP) {  // (after the gate, which reads the half pressure)
                            double s2 = 0.0;
#pragma unroll
                            for (int i = 0; i < D; ++i) s2 = fma(q.v[i], q.v[i], s2);
                            q.p = s2;
                        }
                        store_node<D, NX>(sq, G::FS, tel * G::NNP + G::pad(node), q);
                    }
                }
                if (slow) {
#pragma unroll 1
                    for (int k = 0; k < KN; ++k) {
                        const int t = tid + k * NT;
                        if (((slow >> k) & 1u) && !gate_ok<D>(sacc + t * NVAR, prm.gas.gm1) && (unsigned)t < bad)
                            bad = (unsigned)t;
                    }
                }
                if (bad != ~0u) atomicMin(&prm.status->first_bad, (unsigned long long)((prm.elem_base + e0) * NN) + bad);
            }
            __syncthreads();
            FDG_PT(1)
            // ---- volume integral, direction by direction (accumulators: SoA)
            // runtime-direction pass (one copy of the pair code): p+1 >= 5, and
            // the fused RHS / RK-stage twins at every degree -- their image
            // (three compile-time passes, each with two inlined Rusanov
            // fluxes) overflowed the 32 KB L1.5 instruction cache: cfg5 RHS
            // 7.83 -> 6.44 ms with one copy (profiles/r02_tuning.md); the
            // volume-only twin keeps the compile-time passes below p+1 = 5
            // (3.87 vs 4.03 ms: there the rotated-load address math costs more)
            // (the volume-only twin's small image keeps the compile-time
            // passes up to p + 1 = 7, FDG_RT_DIR_MIN_P1_VOLK)
            // RHS / stage twins: runtime pass at p + 1 = 4 (cfg5 RHS 7.90 -> 6.44 ms when
            // it went in) and on the curved p + 1 = 5 mesh (cfg4 step 4.30 vs 4.36 ms),
            // compile-time passes from FDG_RHSK_CT_MINP1 on (Cartesian N = 4 / 5 / 6
            // Ranocha RHS 3.58 / 3.96 / 4.93 -> 3.31 / 3.14 / 4.17 ms)
#ifndef FDG_RHSK_CT_MINP1
#define FDG_RHSK_CT_MINP1 5
#endif
#ifndef FDG_RHSK_CT_MAXP1
#define FDG_RHSK_CT_MAXP1 7
#endif
            constexpr bool RHSK_CT = P1 >= FDG_RHSK_CT_MINP1 && P1 <= FDG_RHSK_CT_MAXP1 && !(P1 == 5 && CURVED);
            constexpr bool RT_ONLY = MODE == FAST && VF != F_CENTRAL &&
                                     (EPIK == EPI_VOLUME ? P1 >= FDG_RT_DIR_MIN_P1_VOLK
                                      : (EPIK == EPI_RHS || EPIK == EPI_STAGE) ? !RHSK_CT
                                                                               : runtime_direction<D, P1, VF>());
            bool rt_pass = RT_ONLY;
            if constexpr (!RT_ONLY && MODE == FAST && runtime_direction_iface<D, P1, VF>())
                rt_pass = (epi != EPI_VOLUME) && prm.rt_iface;
#ifndef FDG_AOS_LAST
#define FDG_AOS_LAST 1
#endif
            // results straight to the bulk-store staging from the last compile-time
            // pass (lines of consecutive nodes): the volume-only twin on Cartesian
            // meshes whose CTAs have no idle threads (the barrier inside). In the
            // runtime-direction pass the same measured slower (cfg5 RHS 4.95 ->
            // 5.50 ms, cfg3 VOL 0.877 -> 0.982 ms), so only here.
            constexpr bool AOS_OK = FDG_AOS_LAST && EPIK == EPI_VOLUME && MODE == FAST && !CURVED && !REV && D == 3 &&
                                    USED == NT;
            const bool aos_on = AOS_OK && prm.jac_folded && tma_out;
            if (rt_pass) {
                if constexpr (MODE == FAST && VF != F_CENTRAL) {
#pragma unroll 1
                    for (int i = 0; i < D; ++i) {
                        const int n = REV ? D - 1 - i : i;
                        if (vmask) {
                            const bool faces = fuse && active;
                            volume_direction_rt<D, P1, VF, CURVED, LOGS, KP>(prm, sq, sacc, el, m, active ? e : e - el, n, i == 0,
                                                                         vmask, faces, faces ? s_nb[(el * D + n) * 2] : 0,
                                                                         faces ? s_nb[(el * D + n) * 2 + 1] : 0);
                        }
                        __syncthreads();
                    }
                }
            } else if constexpr (!RT_ONLY) {
                vdir<D, P1, VF, CURVED, MODE, LOGS, REV ? D - 1 : 0, true, KP>(prm, sq, sacc, el, m, e, active, vmask, fuse, s_nb);
                __syncthreads();
                FDG_PT(2)
                vdir<D, P1, VF, CURVED, MODE, LOGS, REV ? D - 2 : 1, false, KP>(prm, sq, sacc, el, m, e, active, vmask, fuse, s_nb);
                __syncthreads();
                FDG_PT(3)
                if constexpr (D == 3) {
                    double* aos = aos_on ? sq : nullptr;
                    vdir<D, P1, VF, CURVED, MODE, LOGS, REV ? 0 : 2, false, KP>(prm, sq, sacc, el, m, e, active, vmask, fuse, s_nb,
                                                                            aos);
                    __syncthreads();
                    if (aos) {
                        if (tid == 0) bulk_store(prm.out + base, sq, (unsigned)count * 8u);
                        tma_pending = true;
                        continue;
                    }
                }
            }
            FDG_PT(4)
            // ---- VOL = acc / J   (FAITHFUL: the reference's division, out /= jac;
            //                       FAST: times 1/J)
            // one thread per node: the Jacobian and index math once per node
#pragma unroll
            for (int k = 0; k < KN; ++k) {
                const int t = tid + k * NT;
                if (t < ne * NN) {
                    const int tel = t / NN, node = t - tel * NN;
                    double scale;
                    // (FAST Cartesian: 1/J is already in the weights, fold_jacobian)
                    if constexpr (MODE == FAST)
                        scale = CURVED ? rcp_fast(__ldg(prm.jac + e0 * NN + t)) : 1.0;
                    else
                        scale = CURVED ? __ldg(prm.jac + e0 * NN + t) : prm.jac_const;
#pragma unroll
                    for (int v = 0; v < NVAR; ++v) {
                        const int s = G::acc(v, tel, node);
                        const double vol = (MODE == FAST) ? (CURVED ? sacc[s] * scale : sacc[s]) : sacc[s] / scale;
                        if (epi == EPI_VOLUME) {
                            if (tma_out) sq[t * NVAR + v] = vol;  // AoS, conflict-free (odd stride)
                            else prm.out[base + t * NVAR + v] = vol;
                        } else {
                            sacc[s] = vol;
                        }
                    }
                }
            }
            if (epi == EPI_VOLUME) {
                // the next batch's bulk copy (async proxy) overwrites what
                // this one wrote and read through the generic proxy
                if (TMA_SHAPE) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncthreads();
                if (tma_out && tid == 0) bulk_store(prm.out + base, sq, (unsigned)count * 8u);
                tma_pending = tma_out;
                FDG_PT(5)
                continue;
            }
        } else {
            // mesh_surface: accumulate into the caller's array
            if (tma_pending && tid == 0) bulk_wait_read();  // the outputs are staged in the primitive region
#pragma unroll
            for (int k = 0; k < KU; ++k) {
                const int t = tid + k * NT;
                if (t < count) {
                    const int tel = t / (NN * NVAR);
                    const int r = t - tel * NN * NVAR;
                    const int node = r / NVAR, v = r - node * NVAR;
                    sacc[G::acc(v, tel, node)] = prm.out[base + t];
                }
            }
        }
        __syncthreads();
        // ---- interface terms, direction by direction: every face node of the
        // batch evaluates its interface flux on its own (both sides of an
        // interface from identical arguments, no inter-CTA traffic) and lifts
        // it straight into its node's accumulator. Within one direction a node
        // lies on at most one face, and the passes keep the reference's
        // per-node order (n ascending; discretization.py:754-760: out +=
        // 1/(w_p J) f on the minus side, out -= 1/(w_0 J) f on the plus side).
        // one copy of the face code (runtime n): three inlined copies spilled
        // registers in the curved p+1 = 5 kernels
#pragma unroll 1
        for (int n = fuse ? D : 0; n < D; ++n) {
            const int stride = line_stride<D, P1>(n);
            constexpr int NI = 2 * G::LINES;  // face nodes per element in direction n
            constexpr int KF = (EPB * NI + NT - 1) / NT;
#pragma unroll(kFaceUnroll)
            for (int k = 0; k < KF; ++k) {
                const int it = tid + k * NT;
                if (it < ne * NI) {
                    const int fel = it / NI, r = it - fel * NI;
                    const int side = r / G::LINES, mm = r - side * G::LINES;
                    double fl[NVAR];
#if FDG_NB_SMEM
                    face_flux_item<D, P1, CURVED, MODE>(prm, e0 + fel, n, side, mm, fl, s_nb[(fel * D + n) * 2 + side]);
#else
                    face_flux_item<D, P1, CURVED, MODE>(prm, e0 + fel, n, side, mm, fl);
#endif
                    const int hi = mm / stride, lo = mm - hi * stride;
                    const int node = (hi * P1 + (side ? P1 - 1 : 0)) * stride + lo;
                    const double J = CURVED ? __ldg(prm.jac + (e0 + fel) * NN + node) : prm.jac_const;
                    if (side) {  // e is the minus element: its +n face
                        const double sm = 1.0 / (prm.wp * J);
#pragma unroll
                        for (int v = 0; v < NVAR; ++v) sacc[G::acc(v, fel, node)] += sm * fl[v];
                    } else {
                        const double sp = 1.0 / (prm.w0 * J);
#pragma unroll
                        for (int v = 0; v < NVAR; ++v) sacc[G::acc(v, fel, node)] -= sp * fl[v];
                    }
                }
            }
            __syncthreads();
        }
        // ---- outputs per node
        bool bad = false;
#pragma unroll
        for (int k = 0; k < KN; ++k) {
            const int t = tid + k * NT;
            if (t >= ne * NN) continue;
            const int tel = t / NN, node = t - tel * NN;
#pragma unroll
            for (int v = 0; v < NVAR; ++v) {
                const double val = sacc[G::acc(v, tel, node)];
                const long long g = base + (long long)t * NVAR + v;
                if (epi == EPI_SURFACE || epi == EPI_RHS) {
                    const double y = (epi == EPI_RHS) ? -val : val;
                    if (tma_out) sq[t * NVAR + v] = y;  // AoS for the bulk store
                    else prm.out[g] = y;
                } else {  // EPI_STAGE
                    const double kv = -val;
                    const double x = __ldg(prm.u + g);
                    double y;
                    if (prm.stage_kind == 0) {
                        // du = a_i du + dt k ; v = v + b_i du     (timeint.py:157-158)
                        // (a_0 == 0: the register starts at zero, nothing to read)
                        double rg;
                        if (prm.sa == 0.0) rg = prm.dt * kv;
                        else if constexpr (MODE == FAST) rg = fma(prm.sa, prm.reg[g], prm.dt * kv);
                        else rg = prm.sa * prm.reg[g] + prm.dt * kv;
                        prm.reg[g] = rg;
                        y = x + prm.sb * rg;
                    } else {
                        // y = (A u0 + B x) + (C dt) k             (Shu-Osher SSPRK43)
                        const double s = (prm.sa != 0.0) ? prm.sa * __ldg(prm.u0 + g) + prm.sb * x : x;
                        y = s + prm.sc * kv;
                    }
                    prm.out[g] = y;
                    bad |= !isfinite(y);
                }
            }
        }
        if (bad) atomicMin(&prm.status->bad_stage, prm.stage_index);
        if (TMA_SHAPE) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tma_out && tid == 0) bulk_store(prm.out + base, sq, (unsigned)count * 8u);
        tma_pending = tma_out;
    }
    if (tma_out_ok && tid == 0) bulk_wait_all();
    if (dyn && tid == 0) {
        // the last CTA out resets the counter for the next launch on this mesh
        // (every CTA has left its loop, so nothing claims after the reset)
        __threadfence();
        if (atomicAdd(prm.claim + 1, 1ull) == (unsigned long long)gridDim.x - 1) {
            atomicExch(prm.claim, 0ull);
            atomicExch(prm.claim + 1, 0ull);
        }
    }
#if FDG_PHASE_TIMING
    if (tid == 0)
        for (int i = 0; i < 8; ++i) atomicAdd(&fdg_phase_cycles[i], (unsigned long long)pt_[i]);
    if (tid == 0 && blockIdx.x < 8192) {
        unsigned long long ns1_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns1_));
        unsigned smid_;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_));
        fdg_cta_ns[3 * blockIdx.x] = ns0_;
        fdg_cta_ns[3 * blockIdx.x + 1] = ns1_;
        fdg_cta_ns[3 * blockIdx.x + 2] = smid_;
    }
#endif
}

}  // namespace fdg
