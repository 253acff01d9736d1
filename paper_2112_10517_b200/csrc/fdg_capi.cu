// fdg_capi.cu -- the extern "C" boundary of libfdg.so (declared in include/fdg.h).
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/fdg.h"
#include "fdg_aux.cuh"
#include "fdg_diag.h"
#include "fdg_setup.h"
#include "fdg_dispatch.cuh"

using namespace fdg;

static constexpr int kMaxChunks = 32;

struct fdg_mesh {
    int d = 0, p1 = 0;
    long long n_elem = 0;
    bool curved = false;
    int sm_count = 148;
    int dyn_claim = 1;
    int reserve_sms = 0;  // fdg_mesh_set_reserve_sms: interface launches leave these SMs' slots free
    KParams base{};
    Status* status = nullptr;       // device
    unsigned long long* claim = nullptr;  // device: dynamic batch-claiming counter + done count (interface launches)
    Status* status_host = nullptr;  // page-locked read-back slot (a pageable D2H target is a slow, bounced copy)
    double w1d[8] = {};             // 1D LGL weights (diagnostics)
    double* diag_part = nullptr;    // (diag_blocks, kDiagQ) partials, allocated on first use
    int diag_blocks = 0;
    // host-buffer pipeline (fdg_volume_host): two copy streams + events, made on first use
    cudaStream_t s_in = nullptr, s_out = nullptr;
    cudaEvent_t ev_start = nullptr, ev_done = nullptr;
    cudaEvent_t ev_in[kMaxChunks] = {}, ev_k[kMaxChunks] = {};
};

static thread_local std::string g_last_error;
static std::atomic<unsigned long long> g_launches{0};

static int fail(int rc, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
static int fail(int rc, const char* fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return rc;
}

static int cuda_fail(cudaError_t err, const char* what)
{
    return fail(FDG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(err));
}

static const char* flux_name(int k)
{
    static const char* names[] = {"central", "shima", "ranocha", "kennedy_gruber", "chandrashekar", "llf", "hll"};
    return (k >= 0 && k < 7) ? names[k] : "?";
}

extern "C" {

// error reporting for the other translation units (fdg_gauss.cu)
int fdg_internal_fail(int rc, const char* msg) { return fail(rc, "%s", msg); }

int fdg_abi_version(void) { return FDG_ABI_VERSION; }

const char* fdg_last_error(void) { return g_last_error.c_str(); }

int fdg_supported(int32_t d, int32_t degree) { return (d == 2 || d == 3) && degree >= 1 && degree <= 7; }

unsigned long long fdg_launch_count(void) { return g_launches.load(); }

int fdg_host_alloc(size_t bytes, void** out)
{
    if (!out) return fail(FDG_ERR_ARG, "fdg_host_alloc: null argument");
    *out = nullptr;
    cudaError_t err = cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocDefault);
    if (err != cudaSuccess) return cuda_fail(err, "cudaHostAlloc");
    return FDG_OK;
}

int fdg_host_free(void* ptr)
{
    if (!ptr) return FDG_OK;
    cudaError_t err = cudaFreeHost(ptr);
    if (err != cudaSuccess) return cuda_fail(err, "cudaFreeHost");
    return FDG_OK;
}

int fdg_mesh_create(const fdg_mesh_desc_t* desc, fdg_mesh_t** out)
{
    if (!desc || !out) return fail(FDG_ERR_ARG, "fdg_mesh_create: null argument");
    *out = nullptr;
    if (desc->d != 2 && desc->d != 3)
        return fail(FDG_ERR_UNSUPPORTED, "supported dimensions are 2 and 3, got %d", desc->d);
    if (desc->degree < 1 || desc->degree > 7)
        return fail(FDG_ERR_UNSUPPORTED, "degree %d outside the device-supported range 1..7", desc->degree);
    if (desc->n_elem < 0) return fail(FDG_ERR_ARG, "n_elem must be >= 0");
    if (!desc->dsplit || !desc->weights) return fail(FDG_ERR_ARG, "dsplit and weights are required");
    if (!desc->plus || !desc->minus) return fail(FDG_ERR_ARG, "neighbour tables are required");
    if (!desc->cartesian && (!desc->ja || !desc->jac))
        return fail(FDG_ERR_ARG, "curved meshes need device ja and jac");
    fdg_mesh* m = new fdg_mesh();
    m->d = desc->d;
    m->p1 = desc->degree + 1;
    m->n_elem = desc->n_elem;
    m->curved = !desc->cartesian;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&m->sm_count, cudaDevAttrMultiProcessorCount, dev);
    KParams& k = m->base;
    memset(&k, 0, sizeof(k));
    for (int a = 0; a < m->p1; ++a)
        for (int b = 0; b < m->p1; ++b)
            if (a != b && desc->dsplit[a * m->p1 + b] == 0.0) {
                delete m;
                return fail(FDG_ERR_UNSUPPORTED, "split matrix has a zero off-diagonal entry (%d, %d)", a, b);
            }
    // per-direction pair weights: Dsplit[a,b] * Ja^n_n on Cartesian meshes
    // (the reference's wi = cab * area, discretization.py:297-298), Dsplit on
    // curved ones (discretization.py:318-320)
    for (int n = 0; n < 3; ++n)
        for (int i = 0; i < m->p1 * m->p1; ++i)
        {
            k.wts[n][i] = desc->cartesian ? desc->dsplit[i] * desc->areas[n] : desc->dsplit[i];
            k.wtsE[n][i] = 2.0 * k.wts[n][i];
        }
    for (int i = 0; i < m->p1; ++i) m->w1d[i] = desc->weights[i];
    k.w0 = desc->weights[0];
    k.wp = desc->weights[m->p1 - 1];
    k.inv_w0 = 1.0 / k.w0;
    k.inv_wp = 1.0 / k.wp;
    {
        // tuning override (A/B runs only): FDG_FUSE_FACES=0 keeps the separate face phase in the FAST kernels
        const char* env = getenv("FDG_FUSE_FACES");
        k.fuse_faces = env ? atoi(env) : 1;
    }
    for (int i = 0; i < 3; ++i) k.areas[i] = desc->areas[i];
    k.jac_const = desc->jac_const;
    k.rjac_const = desc->cartesian ? 1.0 / desc->jac_const : 0.0;
    k.ja = desc->ja;
    k.jac = desc->jac;
    k.plus = desc->plus;
    k.minus = desc->minus;
    k.ghost_nrm = desc->ghost_nrm;
    k.n_elem = desc->n_elem;
    k.range_lo = 0;
    k.range_hi = desc->n_elem;
    k.elem_base = desc->elem_base;
    k.gas.gamma = desc->gamma;
    k.gas.gm1 = desc->gamma - 1.0;  // fluxes.py: gm1 = gas.gamma - 1.0
    k.gas.igm1 = desc->inv_gamma_minus_one;
    cudaError_t err = cudaMalloc(&m->status, sizeof(Status));
    if (err != cudaSuccess) {
        delete m;
        return cuda_fail(err, "cudaMalloc(status)");
    }
    err = cudaMemset(m->status, 0xff, sizeof(Status));
    if (err != cudaSuccess) {
        cudaFree(m->status);
        delete m;
        return cuda_fail(err, "cudaMemset(status)");
    }
    k.status = m->status;
    err = cudaMalloc(&m->claim, 2 * sizeof(unsigned long long));
    if (err == cudaSuccess) err = cudaMemset(m->claim, 0, 2 * sizeof(unsigned long long));
    if (err != cudaSuccess) {
        cudaFree(m->status);
        if (m->claim) cudaFree(m->claim);
        delete m;
        return cuda_fail(err, "cudaMalloc(claim counter)");
    }
    // launches deeper than one batch per CTA claim batches dynamically
    // (FDG_DYN_CLAIM=0|1|2 tunes: off | interface epilogues only | all)
    {
        const char* env = getenv("FDG_DYN_CLAIM");
        m->dyn_claim = env ? atoi(env) : 2;
        // (round 2: the volume integral claims dynamically too: cfg5 VOL 3.87 -> 3.57 ms)
        k.claim_chunk_max = 1;
        k.zero = 0;
        // runtime-direction volume pass in the p+1 <= 4 interface kernels:
        // measured slower (cfg5 RHS 9.42 vs 8.92 ms with dynamic claiming,
        // profiles/r02_ab_rt_dc.txt), off by default
        const char* rt = getenv("FDG_RT_IFACE");
        k.rt_iface = rt ? atoi(rt) : 0;
    }
    {
        long long nn = 1;
        for (int i = 0; i < m->d; ++i) nn *= m->p1;
        const double state_bytes = (double)m->n_elem * (double)nn * (m->d + 2) * 8.0;
        // round 2: off by default -- with the interface terms fused into the
        // volume passes it measured 1.2% slower (profiles/r02_tuning.md); the
        // size gate below is what FDG_FACE_PREFETCH=1 meant before
        (void)state_bytes;
        k.face_prefetch = 0;
        // tuning override (A/B runs only): FDG_FACE_PREFETCH=0|1
        if (const char* env = getenv("FDG_FACE_PREFETCH")) k.face_prefetch = atoi(env) != 0;
    }
    *out = m;
    return FDG_OK;
}

void fdg_mesh_destroy(fdg_mesh_t* m)
{
    if (!m) return;
    if (m->status) cudaFree(m->status);
    if (m->claim) cudaFree(m->claim);
    if (m->status_host) cudaFreeHost(m->status_host);
    if (m->diag_part) cudaFree(m->diag_part);
    if (m->s_in) cudaStreamDestroy(m->s_in);
    if (m->s_out) cudaStreamDestroy(m->s_out);
    for (cudaEvent_t e : {m->ev_start, m->ev_done})
        if (e) cudaEventDestroy(e);
    for (int c = 0; c < kMaxChunks; ++c) {
        if (m->ev_in[c]) cudaEventDestroy(m->ev_in[c]);
        if (m->ev_k[c]) cudaEventDestroy(m->ev_k[c]);
    }
    delete m;
}

static int check_scheme(const fdg_scheme_t* s, bool need_volume, bool need_surface)
{
    if (!s) return fail(FDG_ERR_ARG, "scheme is null");
    if (s->mode != FDG_MODE_FAITHFUL && s->mode != FDG_MODE_FAST)
        return fail(FDG_ERR_CONFIG, "kernel: unknown mode %d", s->mode);
    if (s->precompute < 0 || s->precompute > 2)
        return fail(FDG_ERR_CONFIG, "precompute: unknown mode %d", s->precompute);
    if (need_volume && (s->volume_flux < 0 || s->volume_flux > F_CHANDRASHEKAR))
        return fail(FDG_ERR_CONFIG,
                    "volume flux must be symmetric (central, shima, ranocha, kennedy_gruber, chandrashekar), "
                    "got %s",
                    flux_name(s->volume_flux));
    if (need_surface && (s->surface_flux < 0 || s->surface_flux > F_HLL))
        return fail(FDG_ERR_CONFIG, "surface_flux: unknown kind %d", s->surface_flux);
    return FDG_OK;
}

using PickFn = LaunchFn (*)(int, bool, int);

#define FDG_ROW(m, d)                                                                                    \
    {                                                                                                    \
        fdg_pick_##m##_d##d##_p2, fdg_pick_##m##_d##d##_p3, fdg_pick_##m##_d##d##_p4, fdg_pick_##m##_d##d##_p5, \
            fdg_pick_##m##_d##d##_p6, fdg_pick_##m##_d##d##_p7, fdg_pick_##m##_d##d##_p8                   \
    }

static LaunchFn find(const fdg_mesh* m, const fdg_scheme_t* s, int vf)
{
    static const PickFn faithful[2][7] = {FDG_ROW(faithful, 2), FDG_ROW(faithful, 3)};
    static const PickFn fast[2][7] = {FDG_ROW(fast, 2), FDG_ROW(fast, 3)};
    if (m->p1 < 2 || m->p1 > 8 || m->d < 2 || m->d > 3) return nullptr;
    const int logs = (s->precompute == FDG_PRE_PRIMITIVES_AND_LOGS) ? 1 : 0;
    const PickFn fn = (s->mode == FDG_MODE_FAITHFUL ? faithful : fast)[m->d - 2][m->p1 - 2];
    return fn(vf, m->curved, logs);
}

// FAST launches on Cartesian meshes: 1/J folded into the pair weights and the
// lift factors once per launch on the host (196 multiplies), so the
// accumulators already hold VOL (and the fused interface lifts f / (w J)) and
// the kernels' epilogue has no per-node scaling pass. FAITHFUL keeps the
// reference's acc / J division.
static void fold_jacobian(const fdg_mesh* m, const fdg_scheme_t* s, KParams& k)
{
    if (s->mode == FDG_MODE_FAITHFUL || m->curved || k.jac_folded) return;
    for (int n = 0; n < 3; ++n)
        for (int i = 0; i < 64; ++i) {
            k.wts[n][i] *= k.rjac_const;
            k.wtsE[n][i] *= k.rjac_const;
        }
    k.inv_w0 *= k.rjac_const;
    k.inv_wp *= k.rjac_const;
    k.jac_folded = 1;
}

static int run(fdg_mesh* m, const fdg_scheme_t* s, KParams& k, int vf, void* stream)
{
    fold_jacobian(m, s, k);
    k.claim = (m->dyn_claim >= 2 || (m->dyn_claim == 1 && k.epilogue != EPI_VOLUME)) ? m->claim : nullptr;
    k.reserve_sms = (k.epilogue != EPI_VOLUME) ? m->reserve_sms : 0;
    LaunchFn fn = find(m, s, vf);
    if (!fn) return fail(FDG_ERR_UNSUPPORTED, "no kernel for d=%d, p=%d, flux %s", m->d, m->p1 - 1, flux_name(vf));
    if (m->n_elem == 0) return FDG_OK;
    cudaError_t err = fn(k, (cudaStream_t)stream, m->sm_count);
    if (err != cudaSuccess) return cuda_fail(err, "element kernel launch");
    g_launches.fetch_add(1);
    return FDG_OK;
}

int fdg_volume(fdg_mesh_t* m, const fdg_scheme_t* s, const double* u, double* vol, void* stream)
{
    if (!m || !u || !vol) return fail(FDG_ERR_ARG, "fdg_volume: null argument");
    int rc = check_scheme(s, true, false);
    if (rc) return rc;
    KParams k = m->base;
    k.u = u;
    k.out = vol;
    k.epilogue = EPI_VOLUME;
    k.precompute = s->precompute;
    k.surface_flux = F_LLF;
    return run(m, s, k, s->volume_flux, stream);
}

static long long nodes_per_elem(const fdg_mesh* m)
{
    long long nn = 1;
    for (int i = 0; i < m->d; ++i) nn *= m->p1;
    return nn;
}

// volume kernel on elements [lo, hi): pointers shifted, element ids kept global
static int volume_range(fdg_mesh* m, const fdg_scheme_t* s, LaunchFn fn, const double* u, double* vol, long long lo,
                        long long hi, cudaStream_t stream)
{
    if (lo == hi) return FDG_OK;
    const long long nn = nodes_per_elem(m);
    const long long nvar = m->d + 2;
    KParams k = m->base;
    k.u = u + lo * nn * nvar;
    k.out = vol + lo * nn * nvar;
    if (k.ja) k.ja += lo * nn * m->d * m->d;
    if (k.jac) k.jac += lo * nn;
    k.n_elem = hi - lo;
    k.range_lo = 0;
    k.range_hi = hi - lo;
    k.elem_base += lo;
    k.row_order = nullptr;  // the row order indexes the whole mesh
    k.row_len = 0;
    k.epilogue = EPI_VOLUME;
    k.precompute = s->precompute;
    k.surface_flux = F_LLF;
    fold_jacobian(m, s, k);
    cudaError_t err = fn(k, stream, m->sm_count);
    if (err != cudaSuccess) return cuda_fail(err, "element kernel launch");
    g_launches.fetch_add(1);
    return FDG_OK;
}

int fdg_volume_range(fdg_mesh_t* m, const fdg_scheme_t* s, const double* u, double* vol, int64_t lo, int64_t hi,
                     void* stream)
{
    if (!m || !u || !vol) return fail(FDG_ERR_ARG, "fdg_volume_range: null argument");
    if (lo < 0 || hi > m->n_elem || lo > hi) return fail(FDG_ERR_ARG, "fdg_volume_range: bad range [%lld, %lld)",
                                                          (long long)lo, (long long)hi);
    int rc = check_scheme(s, true, false);
    if (rc) return rc;
    LaunchFn fn = find(m, s, s->volume_flux);
    if (!fn) return fail(FDG_ERR_UNSUPPORTED, "no kernel for d=%d, p=%d", m->d, m->p1 - 1);
    return volume_range(m, s, fn, u, vol, lo, hi, (cudaStream_t)stream);
}

static int pipeline_init(fdg_mesh* m)
{
    if (m->s_in) return FDG_OK;
    cudaError_t err = cudaSuccess;
    auto ev = [&](cudaEvent_t* e) {
        if (err == cudaSuccess) err = cudaEventCreateWithFlags(e, cudaEventDisableTiming);
    };
    ev(&m->ev_start);
    ev(&m->ev_done);
    for (int c = 0; c < kMaxChunks; ++c) {
        ev(&m->ev_in[c]);
        ev(&m->ev_k[c]);
    }
    if (err == cudaSuccess) err = cudaStreamCreateWithFlags(&m->s_out, cudaStreamNonBlocking);
    if (err == cudaSuccess) err = cudaStreamCreateWithFlags(&m->s_in, cudaStreamNonBlocking);
    if (err != cudaSuccess) return cuda_fail(err, "pipeline streams/events");
    return FDG_OK;
}

int fdg_volume_host(fdg_mesh_t* m, const fdg_scheme_t* s, const double* u_host, double* vol_host, double* u_dev,
                    double* vol_dev, int32_t n_chunks, void* stream)
{
    if (!m || !u_host || !vol_host || !u_dev || !vol_dev) return fail(FDG_ERR_ARG, "fdg_volume_host: null argument");
    int rc = check_scheme(s, true, false);
    if (rc) return rc;
    LaunchFn fn = find(m, s, s->volume_flux);
    if (!fn) return fail(FDG_ERR_UNSUPPORTED, "no kernel for d=%d, p=%d", m->d, m->p1 - 1);
    if (m->n_elem == 0) return FDG_OK;
    rc = pipeline_init(m);
    if (rc) return rc;
    const long long elem_bytes = nodes_per_elem(m) * (m->d + 2) * (long long)sizeof(double);
    // default: 4 tapered chunks up to 64 MB, then one per 16 MB (<= 16); every
    // chunk costs ~10-20 us of copy setup on B200/PCIe5 (profiles/r01_e2e.md:
    // cfg2's 10.5 MB state, 2 equal chunks 0.361 ms, 4 tapered 0.353, 8: 0.399)
    if (n_chunks <= 0) {
        const long long bytes = m->n_elem * elem_bytes;
        n_chunks = bytes < (4LL << 20) ? 2 : (int32_t)std::max<long long>(4, std::min<long long>(16, bytes >> 24));
    }
    n_chunks = (int32_t)std::min<long long>(std::min<long long>(n_chunks, kMaxChunks), m->n_elem);
    cudaStream_t st = (cudaStream_t)stream;
    // both copy streams start after everything already queued on `stream`
    cudaError_t err = cudaEventRecord(m->ev_start, st);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(m->s_in, m->ev_start, 0);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(m->s_out, m->ev_start, 0);
    // tapered chunks: the first chunk's H2D and the last chunk's D2H are the
    // only copies nothing overlaps, so with 3+ chunks those two are half the
    // size of the others (weights 1/2, 1, ..., 1, 1/2)
    const long long W2 = n_chunks >= 3 ? 2LL * (n_chunks - 1) : 2LL * n_chunks;  // total weight x 2
    auto edge = [&](int c) -> long long {  // element index where chunk c starts
        if (c <= 0) return 0;
        if (c >= n_chunks) return m->n_elem;
        const long long w = n_chunks >= 3 ? 2LL * c - 1 : 2LL * c;
        return m->n_elem * w / W2;
    };
    for (int c = 0; c < n_chunks && err == cudaSuccess; ++c) {
        const long long lo = edge(c), hi = edge(c + 1);
        if (lo == hi) continue;
        const size_t off = (size_t)(lo * elem_bytes / (long long)sizeof(double));
        const size_t bytes = (size_t)((hi - lo) * elem_bytes);
        err = cudaMemcpyAsync(u_dev + off, u_host + off, bytes, cudaMemcpyHostToDevice, m->s_in);
        if (err == cudaSuccess) err = cudaEventRecord(m->ev_in[c], m->s_in);
        if (err == cudaSuccess) err = cudaStreamWaitEvent(st, m->ev_in[c], 0);
        if (err != cudaSuccess) break;
        rc = volume_range(m, s, fn, u_dev, vol_dev, lo, hi, st);
        if (rc) return rc;
        err = cudaEventRecord(m->ev_k[c], st);
        if (err == cudaSuccess) err = cudaStreamWaitEvent(m->s_out, m->ev_k[c], 0);
        if (err == cudaSuccess)
            err = cudaMemcpyAsync(vol_host + off, vol_dev + off, bytes, cudaMemcpyDeviceToHost, m->s_out);
    }
    // `stream` resumes after the last D2H copy
    if (err == cudaSuccess) err = cudaEventRecord(m->ev_done, m->s_out);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(st, m->ev_done, 0);
    if (err != cudaSuccess) return cuda_fail(err, "host pipeline");
    return FDG_OK;
}

int fdg_surface(fdg_mesh_t* m, const fdg_scheme_t* s, const double* u, const double* ghost_u, double* out,
                void* stream)
{
    if (!m || !u || !out) return fail(FDG_ERR_ARG, "fdg_surface: null argument");
    int rc = check_scheme(s, false, true);
    if (rc) return rc;
    KParams k = m->base;
    k.u = u;
    k.out = out;
    k.ghost_u = ghost_u;
    k.epilogue = EPI_SURFACE;
    k.surface_flux = s->surface_flux;
    k.precompute = s->precompute;
    // the surface-only pass does not stage volume data: any instantiation works
    return run(m, s, k, F_SHIMA, stream);
}

static int check_range(const fdg_mesh* m, int64_t lo, int64_t hi, const char* who)
{
    if (lo < 0 || hi > m->n_elem || lo > hi)
        return fail(FDG_ERR_ARG, "%s: bad element range [%lld, %lld) of %lld", who, (long long)lo, (long long)hi,
                    m->n_elem);
    return FDG_OK;
}

static int check_ranges(const fdg_mesh* m, int64_t lo, int64_t hi, int64_t lo2, int64_t hi2, const char* who)
{
    int rc = check_range(m, lo, hi, who);
    if (!rc) rc = check_range(m, lo2, hi2, who);
    if (!rc && lo2 < hi2 && lo < hi && lo2 < hi && lo < hi2)
        return fail(FDG_ERR_ARG, "%s: ranges [%lld, %lld) and [%lld, %lld) overlap", who, (long long)lo, (long long)hi,
                    (long long)lo2, (long long)hi2);
    return rc;
}

int fdg_rhs_range(fdg_mesh_t* m, const fdg_scheme_t* s, const double* u, const double* ghost_u, double* du, int64_t lo,
                  int64_t hi, int64_t lo2, int64_t hi2, void* stream)
{
    if (!m || !u || !du) return fail(FDG_ERR_ARG, "fdg_rhs: null argument");
    if (u == du) return fail(FDG_ERR_ARG, "fdg_rhs: du must not alias u");
    int rc = check_scheme(s, true, true);
    if (!rc) rc = check_ranges(m, lo, hi, lo2, hi2, "fdg_rhs_range");
    if (rc) return rc;
    if (lo == hi && lo2 == hi2) return FDG_OK;
    KParams k = m->base;
    k.u = u;
    k.out = du;
    k.ghost_u = ghost_u;
    k.epilogue = EPI_RHS;
    k.surface_flux = s->surface_flux;
    k.precompute = s->precompute;
    k.range_lo = lo;
    k.range_hi = hi;
    k.range2_lo = lo2;
    k.range2_hi = hi2;
    return run(m, s, k, s->volume_flux, stream);
}

int fdg_rhs(fdg_mesh_t* m, const fdg_scheme_t* s, const double* u, const double* ghost_u, double* du,
            void* stream)
{
    if (!m) return fail(FDG_ERR_ARG, "fdg_rhs: null argument");
    return fdg_rhs_range(m, s, u, ghost_u, du, 0, m->n_elem, 0, 0, stream);
}

int fdg_rk_stage_range(fdg_mesh_t* m, const fdg_scheme_t* s, const fdg_stage_t* st, const double* v_in,
                       const double* ghost_u, double* v_out, double* reg, const double* u0, int64_t lo, int64_t hi,
                       int64_t lo2, int64_t hi2, void* stream)
{
    if (!m || !st || !v_in || !v_out) return fail(FDG_ERR_ARG, "fdg_rk_stage: null argument");
    if (v_in == v_out) return fail(FDG_ERR_ARG, "fdg_rk_stage: v_out must not alias v_in");
    if (st->kind == 0 && !reg) return fail(FDG_ERR_ARG, "fdg_rk_stage: 2N stage needs the register");
    if (st->kind == 1 && st->a != 0.0 && !u0) return fail(FDG_ERR_ARG, "fdg_rk_stage: stage needs u0");
    if (st->kind != 0 && st->kind != 1) return fail(FDG_ERR_CONFIG, "stage kind %d unknown", st->kind);
    int rc = check_scheme(s, true, true);
    if (!rc) rc = check_ranges(m, lo, hi, lo2, hi2, "fdg_rk_stage_range");
    if (rc) return rc;
    if (lo == hi && lo2 == hi2) return FDG_OK;
    KParams k = m->base;
    k.u = v_in;
    k.out = v_out;
    k.ghost_u = ghost_u;
    k.reg = reg;
    k.u0 = u0;
    k.epilogue = EPI_STAGE;
    k.surface_flux = s->surface_flux;
    k.precompute = s->precompute;
    k.stage_kind = st->kind;
    k.stage_index = st->index;
    k.sa = st->a;
    k.sb = st->b;
    k.sc = st->cdt;
    k.dt = st->dt;
    k.range_lo = lo;
    k.range_hi = hi;
    k.range2_lo = lo2;
    k.range2_hi = hi2;
    return run(m, s, k, s->volume_flux, stream);
}

int fdg_rk_stage(fdg_mesh_t* m, const fdg_scheme_t* s, const fdg_stage_t* st, const double* v_in,
                 const double* ghost_u, double* v_out, double* reg, const double* u0, void* stream)
{
    if (!m) return fail(FDG_ERR_ARG, "fdg_rk_stage: null argument");
    return fdg_rk_stage_range(m, s, st, v_in, ghost_u, v_out, reg, u0, 0, m->n_elem, 0, 0, stream);
}

int fdg_gate(fdg_mesh_t* m, const double* u, void* stream)
{
    if (!m || !u) return fail(FDG_ERR_ARG, "fdg_gate: null argument");
    long long nn = 1;
    for (int i = 0; i < m->d; ++i) nn *= m->p1;
    const long long n_nodes = m->n_elem * nn;
    if (n_nodes == 0) return FDG_OK;
    const int threads = 256;
    const long long blocks = std::min<long long>((n_nodes + threads - 1) / threads, (long long)m->sm_count * 16);
    const double gm1 = m->base.gas.gm1;
    const long long node_base = m->base.elem_base * nn;
    if (m->d == 2)
        gate_kernel<2><<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(u, n_nodes, gm1, node_base, m->status);
    else
        gate_kernel<3><<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(u, n_nodes, gm1, node_base, m->status);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return cuda_fail(err, "gate kernel launch");
    g_launches.fetch_add(1);
    return FDG_OK;
}

int fdg_mesh_set_reserve_sms(fdg_mesh_t* m, int32_t n_sms)
{
    if (!m) return fail(FDG_ERR_ARG, "fdg_mesh_set_reserve_sms: null mesh");
    if (n_sms < 0 || n_sms >= m->sm_count)
        return fail(FDG_ERR_ARG, "fdg_mesh_set_reserve_sms: %d of %d SMs", n_sms, m->sm_count);
    m->reserve_sms = n_sms;
    return FDG_OK;
}

int fdg_mesh_set_traversal(fdg_mesh_t* m, const int32_t* row_order, int64_t row_len)
{
    if (!m) return fail(FDG_ERR_ARG, "fdg_mesh_set_traversal: null mesh");
    if (!row_order) {
        m->base.row_order = nullptr;
        m->base.row_len = 0;
        return FDG_OK;
    }
    if (row_len < 1 || m->n_elem % row_len != 0)
        return fail(FDG_ERR_ARG, "fdg_mesh_set_traversal: row_len %lld does not divide n_elem %lld",
                    (long long)row_len, m->n_elem);
    m->base.row_order = row_order;
    m->base.row_len = row_len;
    return FDG_OK;
}

int fdg_diagnostic(fdg_mesh_t* m, int32_t kind, const double* a, const double* b, double* out, void* stream)
{
    if (!m || !a || !out) return fail(FDG_ERR_ARG, "fdg_diagnostic: null argument");
    if (diag_n_out(kind, m->d) == 0) return fail(FDG_ERR_ARG, "fdg_diagnostic: unknown kind %d", kind);
    if ((kind == FDG_DIAG_ENTROPY || kind == FDG_DIAG_ERROR_SQ) && !b)
        return fail(FDG_ERR_ARG, "fdg_diagnostic: kind %d needs a second state", kind);
    if (!m->diag_part) {
        // one resident wave: kDiagCtasPerSm CTAs of 256 threads per SM
        m->diag_blocks = kDiagCtasPerSm * m->sm_count;
        cudaError_t err = cudaMalloc(&m->diag_part, sizeof(double) * kDiagQ * m->diag_blocks);
        if (err != cudaSuccess) {
            m->diag_part = nullptr;
            return cuda_fail(err, "cudaMalloc(diagnostic partials)");
        }
    }
    DiagArgs g;
    g.d = m->d;
    g.p1 = m->p1;
    g.kind = kind;
    g.n_elem = m->n_elem;
    g.a = a;
    g.b = b;
    g.jac = m->curved ? m->base.jac : nullptr;
    g.jac_const = m->base.jac_const;
    for (int i = 0; i < 8; ++i) g.w[i] = m->w1d[i];
    g.gamma = m->base.gas.gamma;
    g.gm1 = m->base.gas.gm1;
    g.igm1 = m->base.gas.igm1;
    g.part = m->diag_part;
    g.out = out;
    g.blocks = m->diag_blocks;
    cudaError_t err = launch_diagnostic(g, (cudaStream_t)stream);
    if (err != cudaSuccess) return cuda_fail(err, "diagnostic kernel launch");
    g_launches.fetch_add(2);
    return FDG_OK;
}

int fdg_build_geometry(const fdg_geometry_desc_t* desc, double* coords, double* ja, double* jac, void* stream)
{
    if (!desc || !desc->nodes || !desc->dmat) return fail(FDG_ERR_ARG, "fdg_build_geometry: null argument");
    if (desc->d != 2 && desc->d != 3)
        return fail(FDG_ERR_UNSUPPORTED, "supported dimensions are 2 and 3, got %d", desc->d);
    if (desc->degree < 1 || desc->degree > 7)
        return fail(FDG_ERR_UNSUPPORTED, "degree %d outside the device-supported range 1..7", desc->degree);
    if ((ja == nullptr) != (jac == nullptr)) return fail(FDG_ERR_ARG, "fdg_build_geometry: ja and jac go together");
    GeomArgs g;
    g.d = desc->d;
    g.p1 = desc->degree + 1;
    g.n_elem = 1;
    for (int j = 0; j < g.d; ++j) {
        if (desc->dims[j] < 1) return fail(FDG_ERR_ARG, "fdg_build_geometry: dims[%d] = %d", j, desc->dims[j]);
        g.dims[j] = desc->dims[j];
        g.lo[j] = desc->lo[j];
        g.hi[j] = desc->hi[j];
        g.n_elem *= desc->dims[j];
    }
    g.amplitude = desc->amplitude;
    for (int k = 0; k < g.p1; ++k) g.nodes[k] = desc->nodes[k];
    for (int k = 0; k < g.p1 * g.p1; ++k) g.dmat[k] = desc->dmat[k];
    g.coords = coords;
    g.ja = ja;
    g.jac = jac;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t err = launch_geometry(g, sms, (cudaStream_t)stream);
    if (err != cudaSuccess) return cuda_fail(err, "geometry kernel launch");
    g_launches.fetch_add(1);
    return FDG_OK;
}

int fdg_reset_status(fdg_mesh_t* m, void* stream)
{
    if (!m) return fail(FDG_ERR_ARG, "fdg_reset_status: null mesh");
    cudaError_t err = cudaMemsetAsync(m->status, 0xff, sizeof(Status), (cudaStream_t)stream);
    if (err != cudaSuccess) return cuda_fail(err, "cudaMemsetAsync(status)");
    return FDG_OK;
}

int fdg_read_status(fdg_mesh_t* m, fdg_status_t* out, void* stream)
{
    if (!m || !out) return fail(FDG_ERR_ARG, "fdg_read_status: null argument");
    cudaError_t err = cudaSuccess;
    if (!m->status_host) err = cudaHostAlloc(&m->status_host, sizeof(Status), cudaHostAllocDefault);
    if (err == cudaSuccess)
        err = cudaMemcpyAsync(m->status_host, m->status, sizeof(Status), cudaMemcpyDeviceToHost, (cudaStream_t)stream);
    if (err == cudaSuccess) err = cudaStreamSynchronize((cudaStream_t)stream);
    if (err != cudaSuccess) return cuda_fail(err, "status read");
    const Status h = *m->status_host;
    out->first_bad = (h.first_bad == ~0ULL) ? -1 : (int64_t)h.first_bad;
    out->bad_stage = (h.bad_stage == ~0U) ? -1 : (int32_t)h.bad_stage;
    out->pad = 0;
    return FDG_OK;
}

int fdg_pack_faces(const double* u, const int32_t* elems, int32_t n, int32_t d, int32_t degree, int32_t dir,
                   int32_t side, double* out, void* stream)
{
    if (!u || !elems || !out) return fail(FDG_ERR_ARG, "fdg_pack_faces: null argument");
    if ((d != 2 && d != 3) || degree < 1 || dir < 0 || dir >= d) return fail(FDG_ERR_ARG, "fdg_pack_faces: bad shape");
    if (n == 0) return FDG_OK;
    const int threads = 256;
    if (dir == 0) {
        const long long p1 = degree + 1, nvar = d + 2;
        long long fn = 1;
        for (int i = 0; i < d - 1; ++i) fn *= p1;
        const long long run = fn * nvar, elem = fn * p1 * nvar;
        const long long off = side ? (p1 - 1) * run : 0;
        const long long work = (long long)n * run / 2;
        const int blocks = (int)std::max<long long>(1, std::min<long long>((work + threads - 1) / threads, 148LL * 8));
        pack_faces_dir0_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(u, elems, n, elem, run, off, out);
    } else {
        const int blocks = 296;
        pack_faces_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(u, elems, n, d, degree + 1, dir, side, out);
    }
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return cuda_fail(err, "pack kernel launch");
    g_launches.fetch_add(1);
    return FDG_OK;
}

}  // extern "C"
