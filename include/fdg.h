/* fdg.h -- C ABI of libfdg.so, the B200 (sm_100a) flux-differencing DGSEM
 * volume integral / RHS for the compressible Euler equations.
 *
 * Drop-in boundary for the reference artifact `fluxdg` (arXiv 2112.10517,
 * /root/reference/pkg/src/fluxdg).  The reference has no FFI; its plugin seam
 * is the kernel string of RhsConfig (discretization.py:73, 932-936) and the
 * module-level functions below.  Each entry point replaces one of them:
 *
 *   fdg_volume    <- batched.mesh_fluxdiff_volume(u, setup, config)      batched.py:450-511
 *                    (and discretization.volume_fluxdiff per element,     discretization.py:267-323)
 *   fdg_surface   <- batched.mesh_surface(u, setup, surface_flux, out)   batched.py:514-544
 *                    / discretization.surface_terms(..., out=out)         discretization.py:681-788
 *   fdg_rhs       <- discretization.rhs(u, setup, config)                discretization.py:896-949
 *   fdg_rk_stage  <- one stage of timeint.rk_step                        timeint.py:149-163
 *                    (and of SSPRK43, which the reference does not ship)
 *   fdg_gate      <- discretization._admissibility_gate                  discretization.py:660-672
 *   fdg_mesh_create <- the device image of build_setup's SpatialSetup    discretization.py:609-657
 *   fdg_build_geometry <- geometry.element_coords + compute_metrics       geometry.py:142-178, 200-250
 *   fdg_diagnostic  <- discretization.conserved_totals                   discretization.py:1027-1031
 *                      discretization.entropy_rate (its two sums)        discretization.py:1011-1024
 *                      discretization.error_norm_l2 (before the sqrt)     discretization.py:1033-1037
 *                      timeint.stable_dt (before the cfl factor)         timeint.py:138-146
 *
 * Conventions: all state pointers are DEVICE pointers owned by the caller
 * (torch allocations in the Python host layer); the library allocates only a
 * 16-byte status record per mesh handle, at creation (and, on the first
 * fdg_diagnostic call, a few KB of per-block partials).  Calls are
 * stream-ordered and asynchronous; only fdg_read_status synchronizes.
 * Layout: the reference's own AoS layout, u[e][i][v] = (n_elem, (p+1)^d, d+2),
 * node index C-ordered over the reference coordinates, variables
 * (rho, rho v_1..rho v_d, rho E).
 * Return codes map 1:1 to the reference's exceptions (errors.py):
 *   FDG_ERR_CONFIG -> ConfigurationError, FDG_ERR_UNSUPPORTED ->
 *   UnsupportedOperatorError; an inadmissible state is reported through the
 *   status record (AdmissibilityError on the host, same message format).
 */
#ifndef FDG_H
#define FDG_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define FDG_ABI_VERSION 1

enum fdg_rc { FDG_OK = 0, FDG_ERR_CONFIG = 1, FDG_ERR_UNSUPPORTED = 2, FDG_ERR_CUDA = 3, FDG_ERR_ARG = 4 };

/* two-point flux kinds (fluxes.py:30-31 plus the BASELINE additions) */
enum fdg_flux {
    FDG_FLUX_CENTRAL = 0,
    FDG_FLUX_SHIMA = 1,
    FDG_FLUX_RANOCHA = 2,
    FDG_FLUX_KENNEDY_GRUBER = 3, /* not in the reference (parity unpinned) */
    FDG_FLUX_CHANDRASHEKAR = 4,  /* not in the reference (parity unpinned) */
    FDG_FLUX_LLF = 5,            /* surface only (Rusanov) */
    FDG_FLUX_HLL = 6             /* surface only */
};
/* RhsConfig.precompute (discretization.py:72) */
enum fdg_precompute { FDG_PRE_NONE = 0, FDG_PRE_PRIMITIVES = 1, FDG_PRE_PRIMITIVES_AND_LOGS = 2 };
/* RhsConfig.kernel: "reference" -> FAITHFUL (scalar path's arithmetic, correctly
 * rounded log), "batched" -> FAST (FMA, shared reciprocals) */
enum fdg_mode { FDG_MODE_FAITHFUL = 0, FDG_MODE_FAST = 1 };

typedef struct fdg_mesh fdg_mesh_t;

typedef struct fdg_mesh_desc {
    int32_t d;             /* 2 or 3 */
    int32_t degree;        /* p, 1..7 */
    int64_t n_elem;        /* elements held by this rank */
    int64_t elem_base;     /* global index of local element 0 (error messages) */
    double gamma;          /* GasParams.gamma */
    double inv_gamma_minus_one; /* GasParams.inv_gamma_minus_one */
    const double *dsplit;  /* HOST (p+1)^2, build_dsplit(op).matrix, row-major */
    const double *weights; /* HOST (p+1), op.weights */
    int32_t cartesian;     /* metrics.cartesian: axis fluxes scaled by areas */
    double areas[3];       /* Cartesian Ja^n_n (diag of metrics.ja[0,0]) */
    double jac_const;      /* Cartesian J */
    const double *ja;      /* DEVICE (n_elem, nn, d, d), curved only */
    const double *jac;     /* DEVICE (n_elem, nn), curved only */
    const int32_t *plus;   /* DEVICE (d, n_elem): +n neighbour, <0 -> ghost slot -(g+1) */
    const int32_t *minus;  /* DEVICE (d, n_elem): -n neighbour, <0 -> ghost slot */
    const double *ghost_nrm; /* DEVICE (n_ghost, fn, d) face normals of remote minus
                                neighbours (curved partitions), or NULL */
} fdg_mesh_desc_t;

typedef struct fdg_scheme {
    int32_t volume_flux;  /* enum fdg_flux, symmetric kinds only */
    int32_t surface_flux; /* enum fdg_flux */
    int32_t precompute;   /* enum fdg_precompute */
    int32_t mode;         /* enum fdg_mode */
} fdg_scheme_t;

typedef struct fdg_stage {
    int32_t kind;     /* 0: low-storage 2N  reg = a reg + dt k; v_out = v_in + b reg
                         1: Shu-Osher      v_out = (A u0 + B v_in) + Cdt k (A == 0: v_in + Cdt k) */
    uint32_t index;   /* stage number reported on a non-finite result */
    double a, b, cdt, dt;
} fdg_stage_t;

typedef struct fdg_status {
    int64_t first_bad;  /* flat (element * nn + node) of the first inadmissible node, or -1 */
    int32_t bad_stage;  /* first RK stage with a non-finite result, or -1 */
    int32_t pad;
} fdg_status_t;

int fdg_abi_version(void);
const char *fdg_last_error(void);
int fdg_supported(int32_t d, int32_t degree);
unsigned long long fdg_launch_count(void);
/* page-locked host buffers for fdg_volume_host (cudaHostAlloc): the copy
 * engines reach ~54 GB/s H2D on them on every B200 host measured, against
 * 14-54 GB/s for caching-allocator pinned blocks (profiles/r01_e2e.md) */
int fdg_host_alloc(size_t bytes, void **out);
int fdg_host_free(void *ptr);

int fdg_mesh_create(const fdg_mesh_desc_t *desc, fdg_mesh_t **out);
void fdg_mesh_destroy(fdg_mesh_t *mesh);

/* VOL = (1/J) sum_n sum_k Dsplit f*_n(u_i, u_k)   (not negated) */
int fdg_volume(fdg_mesh_t *mesh, const fdg_scheme_t *scheme, const double *u, double *vol, void *stream);
/* the same for elements [elem_lo, elem_hi) only (u, vol: the whole arrays);
 * the volume integral is element-local, so host<->device copies of element
 * chunks can be pipelined against it (batched.py:450-511 processes any block
 * of elements independently as well) */
int fdg_volume_range(fdg_mesh_t *mesh, const fdg_scheme_t *scheme, const double *u, double *vol, int64_t elem_lo,
                     int64_t elem_hi, void *stream);
/* fdg_volume on a HOST state into a HOST buffer (the call an FFI user with
 * numpy arrays makes; batched.py:450-511 takes and returns host arrays):
 * element chunks are copied in on one library-owned stream, integrated on
 * `stream`, copied out on another, so both copy directions and the SMs work
 * concurrently.  u_host/vol_host should be pinned (pageable memory works but
 * serializes the copies); u_dev/vol_dev are caller-owned device scratch of the
 * state's size.  n_chunks <= 0 picks >= 4 MB chunks (2..16).  Asynchronous: `stream`
 * is ordered after the last copy-out, so synchronizing it (or
 * fdg_read_status) completes the call. */
int fdg_volume_host(fdg_mesh_t *mesh, const fdg_scheme_t *scheme, const double *u_host, double *vol_host,
                    double *u_dev, double *vol_dev, int32_t n_chunks, void *stream);
/* out += SURF  (LGL interface terms, lifted and /J) */
int fdg_surface(fdg_mesh_t *mesh, const fdg_scheme_t *scheme, const double *u, const double *ghost_u,
                double *out, void *stream);
/* du = -(VOL + SURF) */
int fdg_rhs(fdg_mesh_t *mesh, const fdg_scheme_t *scheme, const double *u, const double *ghost_u, double *du,
            void *stream);
/* one Runge-Kutta stage fused with the RHS: v_out must not alias v_in */
int fdg_rk_stage(fdg_mesh_t *mesh, const fdg_scheme_t *scheme, const fdg_stage_t *stage, const double *v_in,
                 const double *ghost_u, double *v_out, double *reg, const double *u0, void *stream);
/* fdg_rhs / fdg_rk_stage restricted to the local elements [lo, hi) plus an
 * optional second range [lo2, hi2) (empty: lo2 == hi2) in the same launch
 * (u, du, v_in, v_out, reg, u0: the whole arrays; only those rows are
 * written). The overlap split of a slab partition: the interior elements
 * never read ghost_u (NULL is fine) and run while the face-trace exchange is
 * in flight; the two boundary planes run after it, in one launch, with the
 * received ghosts. Results are bitwise those of the whole-slab call (every
 * element's arithmetic is independent of which launch covers it). */
int fdg_rhs_range(fdg_mesh_t *mesh, const fdg_scheme_t *scheme, const double *u, const double *ghost_u, double *du,
                  int64_t lo, int64_t hi, int64_t lo2, int64_t hi2, void *stream);
int fdg_rk_stage_range(fdg_mesh_t *mesh, const fdg_scheme_t *scheme, const fdg_stage_t *stage, const double *v_in,
                       const double *ghost_u, double *v_out, double *reg, const double *u0, int64_t lo, int64_t hi,
                       int64_t lo2, int64_t hi2, void *stream);
/* admissibility of every node (rho > 0, p > 0, finite) into the status record */
int fdg_gate(fdg_mesh_t *mesh, const double *u, void *stream);
int fdg_reset_status(fdg_mesh_t *mesh, void *stream);
/* synchronizes `stream`, copies the status record out */
int fdg_read_status(fdg_mesh_t *mesh, fdg_status_t *out, void *stream);

/* traversal order of the element kernels: row_order (DEVICE, n_rows int32,
 * a permutation of 0..n_rows-1, n_rows = n_elem / row_len) lists the rows of
 * row_len consecutive elements in the order CTAs take them; NULL restores
 * the natural order. Results are unchanged (every element's arithmetic is
 * independent of the order); meant for states much larger than L2, where
 * visiting the mesh tile by tile keeps interface neighbours in L2. The
 * array must outlive the mesh handle or the next call. */
int fdg_mesh_set_traversal(fdg_mesh_t *mesh, const int32_t *row_order, int64_t row_len);

/* interface launches (fdg_rhs*, fdg_rk_stage*, fdg_surface) size their
 * persistent grid for sm_count - n_sms SMs: at full occupancy the element
 * kernel holds every register of every SM, so a concurrent kernel (the halo
 * packer, NCCL's send/recv) cannot start until it ends; the sharded RHS
 * reserves a few SMs so the exchange overlaps the interior launch. Batches
 * are claimed dynamically, so the smaller grid costs no load imbalance. */
int fdg_mesh_set_reserve_sms(fdg_mesh_t *mesh, int32_t n_sms);

/* diagnostics reductions over every node of the mesh (rank-local; sums and
 * the min combine across ranks with an all-reduce).  `a` = u, `b` = dudt
 * (ENTROPY) or u_exact (ERROR_SQ), else NULL; `out` is a DEVICE buffer of
 *   CONSERVED: d+2  sum_e,i wbar_i J u[e,i,v]
 *   ENTROPY:   2    sum wbar J w(u).dudt, sum_e,i,v |wbar J w_v dudt_v|
 *   ERROR_SQ:  d+2  sum wbar J (u - u_exact)^2
 *   DT:        1    min J^(1/d) / ((|v| + c)(2p+1))
 * Deterministic (fixed-order tree, no atomics); no admissibility check
 * (an inadmissible node gives NaN, as the reference's log/sqrt would). */
enum fdg_diag { FDG_DIAG_CONSERVED = 0, FDG_DIAG_ENTROPY = 1, FDG_DIAG_ERROR_SQ = 2, FDG_DIAG_DT = 3 };
int fdg_diagnostic(fdg_mesh_t *mesh, int32_t kind, const double *a, const double *b, double *out, void *stream);

/* on-device geometry of the periodic box [lo, hi]^d split into dims
 * elements, warped by amplitude prod_j sin(2 pi t_j) (build_mesh/element_coords),
 * with the curl-form metrics (compute_metrics). Writes DEVICE arrays:
 * coords (n_elem, nn, d) and/or ja (n_elem, nn, d, d) + jac (n_elem, nn);
 * any may be NULL (ja and jac together). n_elem = prod dims. */
typedef struct fdg_geometry_desc {
    int32_t d;
    int32_t degree;        /* p, 1..7 */
    int32_t dims[3];
    double lo[3], hi[3];
    double amplitude;
    const double *nodes;   /* HOST (p+1) op.nodes */
    const double *dmat;    /* HOST (p+1)^2 op.D, row-major */
} fdg_geometry_desc_t;
int fdg_build_geometry(const fdg_geometry_desc_t *desc, double *coords, double *ja, double *jac, void *stream);

/* ---- Gauss-node family (the paper's second scheme family):
 * volume_scheme "gauss_fluxdiff" / "gauss_surface_correction" of the
 * reference's rhs (discretization.py:966-995), i.e. the zero-corner
 * hybridized flux-differencing volume term with entropy-projected face
 * states (_project_all, :811-837) plus the interface fluxes of the projected
 * states lifted through the dense boundary rows (_gauss_surface, :839-895).
 * The two schemes differ only in the volume pair weights the host passes
 * (hybridized Q_h entries vs the split-derivative matrix, operators.py:300-357). */
typedef struct fdg_gauss fdg_gauss_t;
typedef struct fdg_gauss_desc {
    int32_t d;             /* 2 (p <= 7) or 3 (p <= 5) */
    int32_t degree;
    int64_t n_elem;
    double gamma, inv_gamma_minus_one;
    const double *boundary_interp; /* HOST (2, p+1): R rows at -1 / +1 */
    const double *vv;      /* HOST (p+1, p+1): volume pair weights c_ab, a != b */
    const double *cvol;    /* HOST (2, p+1): crossing weight into the volume row */
    const double *cface;   /* HOST (2, p+1): crossing weight into the face row */
    const double *lift;    /* HOST (2, p+1): R[s][a] / w[a] */
    const double *ja;      /* DEVICE (n_elem, nn, d, d) metric terms at the Gauss nodes */
    const double *jac;     /* DEVICE (n_elem, nn) */
    const int32_t *plus;   /* DEVICE (d, n_elem) periodic neighbours */
    const int32_t *minus;  /* DEVICE (d, n_elem) */
} fdg_gauss_desc_t;
int fdg_gauss_create(const fdg_gauss_desc_t *desc, fdg_gauss_t **out);
void fdg_gauss_destroy(fdg_gauss_t *g);
/* entropy-projected face states proj (n_elem, d, 2, fn, d+2) and each
 * element's own face metric traces nrm (n_elem, d, 2, fn, d); NULL outputs go
 * to library-owned scratch (allocated at creation) */
int fdg_gauss_project(fdg_gauss_t *g, const double *u, double *proj, double *nrm, void *stream);
/* du = -(VOL + SURF) / J of the Gauss schemes; proj/nrm NULL: projected first
 * (fdg_gauss_project into the scratch); fnrm (n_elem, d, fn, d) interface
 * normals or NULL (the minus element's side-1 traces) */
int fdg_gauss_rhs(fdg_gauss_t *g, const fdg_scheme_t *scheme, const double *u, const double *proj, const double *nrm,
                  const double *fnrm, double *du, void *stream);
/* status: first_bad = first inadmissible node (gate), bad_stage = first
 * direction*2+side whose projected state is inadmissible (entropy2cons) */
int fdg_gauss_gate(fdg_gauss_t *g, const double *u, void *stream);
int fdg_gauss_reset_status(fdg_gauss_t *g, void *stream);
int fdg_gauss_read_status(fdg_gauss_t *g, fdg_status_t *out, void *stream);

/* halo helper: out[i][m][v] = u[elems[i]][line node m of direction dir at end `side`][v] */
int fdg_pack_faces(const double *u, const int32_t *elems, int32_t n, int32_t d, int32_t degree, int32_t dir,
                   int32_t side, double *out, void *stream);

/* sustained FP64 FMA throughput of this device (TFLOP/s, 2 flop per DFMA) */
int fdg_fp64_probe(double *tflops, void *stream);

#ifdef __cplusplus
}
#endif
#endif
