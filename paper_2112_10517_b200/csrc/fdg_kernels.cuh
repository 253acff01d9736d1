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
    long long n_elem;
    long long elem_base;      // added to element indices reported by the gate
    double wts[3][64];        // per direction: Dsplit[a,b] * Ja^n_n (Cartesian) or Dsplit (curved)
    double areas[3];          // Cartesian Ja^n_n
    double jac_const;         // Cartesian J
    double w0, wp;            // LGL weights at the -1 / +1 ends
    Gas gas;
    int epilogue;
    int surface_flux;
    int precompute;
    int stage_kind;           // 0: low-storage 2N, 1: Shu-Osher convex combination
    unsigned int stage_index;
    double sa, sb, sc, dt;    // 2N: a_i, b_i, -, dt ; SO: A, B, C*dt, -
};

template <int D, int P1>
struct Geo {
    static constexpr int NN = ipow(P1, D);
    static constexpr int LINES = ipow(P1, D - 1);
    static constexpr int NVAR = D + 2;
    static constexpr int NNP = NN + NN / P1;  // one pad slot per innermost row
    static constexpr int EPB = LINES >= 128 ? 1 : 128 / LINES;
    static constexpr int NT = ((EPB * LINES + 31) / 32) * 32;
    static constexpr int FS = EPB * NNP;      // stride of one primitive field
    static constexpr int FA = EPB * NNP + 1;  // stride of one accumulator variable (odd: spreads banks)

    // node id of position a on line m of direction n (operators.py:248-259)
    template <int N>
    __device__ static __forceinline__ int line_node(int m, int a)
    {
        constexpr int stride = ipow(P1, D - 1 - N);
        return (m / stride * P1 + a) * stride + m % stride;
    }
    __device__ static __forceinline__ int pad(int node) { return node + node / P1; }
    // accumulator slot of (variable v, element el, node)
    __device__ static __forceinline__ int acc(int v, int el, int node) { return v * FA + el * NNP + pad(node); }
};

template <int D, int P1, int VF, int LOGS>
__host__ __device__ constexpr int smem_doubles()
{
    using G = Geo<D, P1>;
    // primitive fields + accumulators (the accumulator block doubles as the
    // AoS staging buffer of u, which is smaller)
    return (2 + D + n_extra(VF, LOGS)) * G::FS + G::NVAR * G::FA;
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

// One direction of the volume integral for the thread's line.
template <int D, int P1, int VF, bool CURVED, int MODE, int LOGS, int N>
__device__ __forceinline__ void volume_direction(const KParams& prm, const double* sq, double* sacc, int el,
                                                 int m, long long e)
{
    using G = Geo<D, P1>;
    constexpr int NVAR = G::NVAR;
    constexpr int NX = n_extra(VF, LOGS);
    double acc[P1][NVAR];
    int nodes[P1];
#pragma unroll
    for (int a = 0; a < P1; ++a) nodes[a] = G::template line_node<N>(m, a);
    if constexpr (N == 0) {
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
    // compile-time pair loops (a < b in pair-table order): keeps acc/jl in registers
    sfor<0, P1>([&](auto A) {
        constexpr int a = decltype(A)::value;
        const Node<D, NX> qa = load_node<D, NX>(sq, G::FS, sbase + G::pad(nodes[a]));
        sfor<a + 1, P1>([&](auto B) {
            constexpr int b = decltype(B)::value;
            // every off-diagonal LGL Dsplit entry is nonzero (checked at mesh
            // creation), so the reference's pair table visits every pair
            const double wa = prm.wts[N][a * P1 + b];
            const double wb = prm.wts[N][b * P1 + a];
            const Node<D, NX> qb = load_node<D, NX>(sq, G::FS, sbase + G::pad(nodes[b]));
            double f[NVAR];
            if constexpr (CURVED) {
                double alpha[D];
#pragma unroll
                for (int j = 0; j < D; ++j) alpha[j] = 0.5 * (jl[a][j] + jl[b][j]);
                volume_flux<D, VF, -1, MODE, LOGS>(qa, qb, alpha, prm.gas, prm.precompute, f);
            } else {
                volume_flux<D, VF, N, MODE, LOGS>(qa, qb, nullptr, prm.gas, prm.precompute, f);
            }
#pragma unroll
            for (int v = 0; v < NVAR; ++v) {
                acc[a][v] += wa * f[v];
                acc[b][v] += wb * f[v];
            }
        });
    });
#pragma unroll
    for (int a = 0; a < P1; ++a)
#pragma unroll
        for (int v = 0; v < NVAR; ++v) sacc[G::acc(v, el, nodes[a])] = acc[a][v];
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
        surface_flux<D, MODE>(prm.surface_flux, ul, ur, nrm, prm.gas, f);
    }
}

// Interface terms of direction N for the thread's line (both of its ends).
template <int D, int P1, bool CURVED, int MODE, int N>
__device__ __forceinline__ void surface_direction(const KParams& prm, double* sacc, int el, int m, long long e)
{
    using G = Geo<D, P1>;
    constexpr int NVAR = G::NVAR;
    constexpr int FN = G::LINES;
    double ul[NVAR], ur[NVAR], nrm[D], f[NVAR];
    // +N face of e (e is the minus element): own node at line end, neighbour's line start
    {
        const int im = G::template line_node<N>(m, P1 - 1);
        load_state<D>(prm.u + (e * G::NN + im) * NVAR, ul);
        const int nb = __ldg(prm.plus + N * prm.n_elem + e);
        if (nb >= 0) load_state<D>(prm.u + ((long long)nb * G::NN + G::template line_node<N>(m, 0)) * NVAR, ur);
        else load_state<D>(prm.ghost_u + ((long long)(-nb - 1) * FN + m) * NVAR, ur);
        if constexpr (CURVED) {
#pragma unroll
            for (int j = 0; j < D; ++j) nrm[j] = __ldg(prm.ja + ((e * G::NN + im) * D + N) * D + j);
        } else {
#pragma unroll
            for (int j = 0; j < D; ++j) nrm[j] = (j == N) ? prm.areas[N] : 0.0;
        }
        face_flux<D, CURVED, MODE, N>(prm, ul, ur, nrm, f);
        const double J = CURVED ? __ldg(prm.jac + e * G::NN + im) : prm.jac_const;
        const double sm = 1.0 / (prm.wp * J);
#pragma unroll
        for (int v = 0; v < NVAR; ++v) sacc[G::acc(v, el, im)] += sm * f[v];
    }
    // -N face of e (e is the plus element): neighbour's line end, own line start
    {
        const int ip = G::template line_node<N>(m, 0);
        const int nb = __ldg(prm.minus + N * prm.n_elem + e);
        const int jm = G::template line_node<N>(m, P1 - 1);
        if (nb >= 0) {
            load_state<D>(prm.u + ((long long)nb * G::NN + jm) * NVAR, ul);
            if constexpr (CURVED) {
#pragma unroll
                for (int j = 0; j < D; ++j) nrm[j] = __ldg(prm.ja + (((long long)nb * G::NN + jm) * D + N) * D + j);
            }
        } else {
            const long long g = -nb - 1;
            load_state<D>(prm.ghost_u + (g * FN + m) * NVAR, ul);
            if constexpr (CURVED) {
#pragma unroll
                for (int j = 0; j < D; ++j) nrm[j] = __ldg(prm.ghost_nrm + (g * FN + m) * D + j);
            }
        }
        if constexpr (!CURVED) {
#pragma unroll
            for (int j = 0; j < D; ++j) nrm[j] = (j == N) ? prm.areas[N] : 0.0;
        }
        load_state<D>(prm.u + (e * G::NN + ip) * NVAR, ur);
        face_flux<D, CURVED, MODE, N>(prm, ul, ur, nrm, f);
        const double J = CURVED ? __ldg(prm.jac + e * G::NN + ip) : prm.jac_const;
        const double sp = 1.0 / (prm.w0 * J);
#pragma unroll
        for (int v = 0; v < NVAR; ++v) sacc[G::acc(v, el, ip)] -= sp * f[v];
    }
}

template <int D, int P1, int VF, bool CURVED, int MODE, int LOGS>
__global__ void __launch_bounds__(Geo<D, P1>::NT) elem_kernel(const __grid_constant__ KParams prm)
{
    using G = Geo<D, P1>;
    constexpr int NN = G::NN, NVAR = G::NVAR, EPB = G::EPB, NT = G::NT;
    constexpr int NX = n_extra(VF, LOGS);
    extern __shared__ double smem[];
    double* sq = smem;                        // (2+D+NX) fields x FS
    double* sacc = smem + (2 + D + NX) * G::FS;  // NVAR x FA (AoS u staging before the volume pass)
    const int tid = threadIdx.x;
    const int el = tid / G::LINES;
    const int m = tid % G::LINES;
    const long long nbatch = (prm.n_elem + EPB - 1) / EPB;
    const int epi = prm.epilogue;

    for (long long batch = blockIdx.x; batch < nbatch; batch += gridDim.x) {
        const long long e0 = batch * EPB;
        const int ne = (int)min((long long)EPB, prm.n_elem - e0);
        const long long base = e0 * NN * NVAR;
        const int count = ne * NN * NVAR;
        const long long e = e0 + el;
        const bool active = (el < ne);

        if (epi != EPI_SURFACE) {
            // ---- stage: coalesced copy (AoS), then primitives per node (SoA)
            for (int t = tid; t < count; t += NT) sacc[t] = __ldg(prm.u + base + t);
            __syncthreads();
            for (int t = tid; t < ne * NN; t += NT) {
                const int tel = t / NN, node = t - tel * NN;
                const double* su = sacc + t * NVAR;
                if (!gate_ok<D>(su, prm.gas.gm1))
                    atomicMin(&prm.status->first_bad, (unsigned long long)((prm.elem_base + e0) * NN + t));
                const Node<D, NX> q = make_node<D, VF, MODE, LOGS>(su, prm.gas.gm1);
                store_node<D, NX>(sq, G::FS, tel * G::NNP + G::pad(node), q);
            }
            __syncthreads();
            // ---- volume integral, direction by direction (accumulators: SoA)
            if (active) volume_direction<D, P1, VF, CURVED, MODE, LOGS, 0>(prm, sq, sacc, el, m, e);
            __syncthreads();
            if (active) volume_direction<D, P1, VF, CURVED, MODE, LOGS, 1>(prm, sq, sacc, el, m, e);
            __syncthreads();
            if constexpr (D == 3) {
                if (active) volume_direction<D, P1, VF, CURVED, MODE, LOGS, 2>(prm, sq, sacc, el, m, e);
                __syncthreads();
            }
            // ---- VOL = acc / J
            for (int t = tid; t < count; t += NT) {
                const int tel = t / (NN * NVAR);
                const int r = t - tel * NN * NVAR;
                const int node = r / NVAR, v = r - node * NVAR;
                const double J = CURVED ? __ldg(prm.jac + (e0 + tel) * NN + node) : prm.jac_const;
                const int s = G::acc(v, tel, node);
                const double vol = sacc[s] / J;
                if (epi == EPI_VOLUME) prm.out[base + t] = vol;
                else sacc[s] = vol;
            }
            if (epi == EPI_VOLUME) {
                __syncthreads();
                continue;
            }
        } else {
            // mesh_surface: accumulate into the caller's array
            for (int t = tid; t < count; t += NT) {
                const int tel = t / (NN * NVAR);
                const int r = t - tel * NN * NVAR;
                const int node = r / NVAR, v = r - node * NVAR;
                sacc[G::acc(v, tel, node)] = prm.out[base + t];
            }
        }
        __syncthreads();
        // ---- interface terms, direction by direction
        if (active) surface_direction<D, P1, CURVED, MODE, 0>(prm, sacc, el, m, e);
        __syncthreads();
        if (active) surface_direction<D, P1, CURVED, MODE, 1>(prm, sacc, el, m, e);
        __syncthreads();
        if constexpr (D == 3) {
            if (active) surface_direction<D, P1, CURVED, MODE, 2>(prm, sacc, el, m, e);
            __syncthreads();
        }
        // ---- outputs
        bool bad = false;
        for (int t = tid; t < count; t += NT) {
            const int tel = t / (NN * NVAR);
            const int r = t - tel * NN * NVAR;
            const int node = r / NVAR, v = r - node * NVAR;
            const double val = sacc[G::acc(v, tel, node)];
            if (epi == EPI_SURFACE) {
                prm.out[base + t] = val;
            } else if (epi == EPI_RHS) {
                prm.out[base + t] = -val;
            } else {  // EPI_STAGE
                const double k = -val;
                const double x = __ldg(prm.u + base + t);
                double y;
                if (prm.stage_kind == 0) {
                    // du = a_i du + dt k ; v = v + b_i du     (timeint.py:157-158)
                    // (a_0 == 0: the register starts at zero, nothing to read)
                    double rg;
                    if (prm.sa == 0.0) rg = prm.dt * k;
                    else if constexpr (MODE == FAST) rg = fma(prm.sa, prm.reg[base + t], prm.dt * k);
                    else rg = prm.sa * prm.reg[base + t] + prm.dt * k;
                    prm.reg[base + t] = rg;
                    y = x + prm.sb * rg;
                } else {
                    // y = (A u0 + B x) + (C dt) k             (Shu-Osher SSPRK43)
                    const double s = (prm.sa != 0.0) ? prm.sa * __ldg(prm.u0 + base + t) + prm.sb * x : x;
                    y = s + prm.sc * k;
                }
                prm.out[base + t] = y;
                bad |= !isfinite(y);
            }
        }
        if (bad) atomicMin(&prm.status->bad_stage, prm.stage_index);
        __syncthreads();
    }
}

}  // namespace fdg
