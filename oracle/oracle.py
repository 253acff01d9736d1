"""CPU oracle wrapper -- TEST INFRASTRUCTURE, not the product.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this module, as the checker or as the reported
CPU baseline. The product package ``paper_2112_10517_b200`` never imports it.

It wraps ``liboracle.so`` (fdg_oracle.c, built by ``oracle/Makefile``), a
plain-C restatement of the reference's scalar flux-differencing path that is
pinned BITWISE to the reference's own outputs (tests/golden/*.npz, written by
tests/golden/make_golden.py from /root/reference/pkg/src/fluxdg):

* ``volume(u, setup, flux, precompute)`` == ``volume_fluxdiff`` over all
  elements (reference discretization.py:267-323)
* ``surface(u, setup, flux, out)``       == ``surface_terms`` LGL branch
  (discretization.py:681-760)
* ``rhs(u, setup, vflux, sflux, precompute)`` == ``rhs(kernel="reference")``
  (discretization.py:896-949), including the admissibility gate message
  (discretization.py:660-672)
* ``rk54_step`` == ``rk_step`` with the Carpenter-Kennedy RK54 tableau
  (timeint.py:101-163), same numpy operation sequence
* ``ssprk43_step`` -- the Shu-Osher SSPRK(4,3) step BASELINE cfg 4 asks for;
  NOT in the reference (parity unpinned, checked by order conditions).

``setup`` is duck-typed: anything with ``d``, ``op.weights``,
``dsplit.matrix``, ``metrics.{ja,jac,cartesian}``, ``plus_neighbor`` and
``gas.{gamma,inv_gamma_minus_one}`` -- the reference's SpatialSetup and the
product's SpatialSetup both qualify, and so do plain namespaces.
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATHS = {
    "glibc": os.path.join(HERE, "liboracle.so"),  # reference arithmetic, bit for bit
    "cr": os.path.join(HERE, "liboracle_cr.so"),  # same, with the correctly rounded log_cr
}

FLUX_IDS = {
    "central": 0,
    "shima": 1,
    "ranocha": 2,
    "kennedy_gruber": 3,
    "chandrashekar": 4,
    "llf": 5,
    "hll": 6,
}
PRE_IDS = {"none": 0, "primitives": 1, "primitives_and_logs": 2}


class OrMesh(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int),
        ("p1", ctypes.c_int),
        ("n_elem", ctypes.c_int64),
        ("dsplit", ctypes.c_void_p),
        ("weights", ctypes.c_void_p),
        ("gamma", ctypes.c_double),
        ("igm1", ctypes.c_double),
        ("cartesian", ctypes.c_int),
        ("areas", ctypes.c_void_p),
        ("jac_const", ctypes.c_double),
        ("ja", ctypes.c_void_p),
        ("jac", ctypes.c_void_p),
        ("plus", ctypes.c_void_p),
        ("minus", ctypes.c_void_p),
        ("ghost_u", ctypes.c_void_p),
        ("ghost_nrm", ctypes.c_void_p),
    ]


class OrGaussTables(ctypes.Structure):
    _fields_ = [("vv", ctypes.c_void_p), ("cvol", ctypes.c_void_p), ("cface", ctypes.c_void_p), ("lift", ctypes.c_void_p)]


_libs = {}


def build(force=False):
    """Compile liboracle*.so in place (gcc, strict IEEE flags, see Makefile)."""
    if force or not all(os.path.exists(p) for p in LIB_PATHS.values()):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATHS


def lib(variant="glibc"):
    if variant not in _libs:
        path = LIB_PATHS[variant]
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        P = ctypes.POINTER(OrMesh)
        vp = ctypes.c_void_p
        L.or_volume.argtypes = [P, vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.or_surface.argtypes = [P, vp, vp, ctypes.c_int, ctypes.c_int]
        L.or_rhs.argtypes = [P, vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.or_rhs.restype = ctypes.c_int64
        L.or_rhs_range.argtypes = [P, vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                   ctypes.c_int64, ctypes.c_int]
        L.or_gate.argtypes = [P, vp, vp, vp]
        L.or_gauss_rhs.argtypes = [P, ctypes.POINTER(OrGaussTables), vp, vp, vp, vp, vp, ctypes.c_int, ctypes.c_int]
        L.or_gate.restype = ctypes.c_int64
        L.or_two_point.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
            vp, vp, vp, ctypes.c_int, vp,
        ]
        L.or_logmean.argtypes = [ctypes.c_double, ctypes.c_double]
        L.or_logmean.restype = ctypes.c_double
        L.or_inv_logmean.argtypes = [ctypes.c_double, ctypes.c_double]
        L.or_inv_logmean.restype = ctypes.c_double
        L.or_max_threads.restype = ctypes.c_int
        _libs[variant] = L
    return _libs[variant]


def _ptr(a):
    return None if a is None else a.ctypes.data


class MeshArrays:
    """Contiguous host arrays describing one (possibly partitioned) mesh."""

    def __init__(self, d, p1, n_elem, dsplit, weights, gamma, igm1, cartesian, areas,
                 jac_const, ja, jac, plus, minus, ghost_u=None, ghost_nrm=None):
        c = np.ascontiguousarray
        self.keep = dict(
            dsplit=c(dsplit, dtype=np.float64),
            weights=c(weights, dtype=np.float64),
            areas=c(areas, dtype=np.float64) if areas is not None else None,
            ja=c(ja, dtype=np.float64) if ja is not None else None,
            jac=c(jac, dtype=np.float64) if jac is not None else None,
            plus=c(plus, dtype=np.int64),
            minus=c(minus, dtype=np.int64),
            ghost_u=c(ghost_u, dtype=np.float64) if ghost_u is not None else None,
            ghost_nrm=c(ghost_nrm, dtype=np.float64) if ghost_nrm is not None else None,
        )
        k = self.keep
        self.d, self.p1, self.n_elem = d, p1, n_elem
        self.struct = OrMesh(
            d, p1, n_elem, _ptr(k["dsplit"]), _ptr(k["weights"]), gamma, igm1, int(cartesian),
            _ptr(k["areas"]), jac_const, _ptr(k["ja"]), _ptr(k["jac"]), _ptr(k["plus"]),
            _ptr(k["minus"]), _ptr(k["ghost_u"]), _ptr(k["ghost_nrm"]),
        )


def mesh_from_setup(setup, lo=0, hi=None):
    """MeshArrays for elements [lo, hi) of a full periodic setup (no ghosts)."""
    d = setup.d
    weights = np.asarray(setup.op.weights)
    p1 = weights.shape[0]
    metrics = setup.metrics
    plus = np.stack([np.asarray(setup.plus_neighbor[n]) for n in range(d)])
    n_elem = plus.shape[1]
    minus = np.empty_like(plus)
    for n in range(d):
        minus[n, plus[n]] = np.arange(n_elem)
    cart = bool(metrics.cartesian)
    ja = None if cart else np.asarray(metrics.ja)
    jac = None if cart else np.asarray(metrics.jac)
    if cart:
        if getattr(metrics, "areas", None) is not None and getattr(metrics, "jac_const", None) is not None:
            # scalar Cartesian metrics (no per-node arrays materialised)
            areas = np.asarray(metrics.areas, dtype=np.float64)
            jac_const = float(metrics.jac_const)
        else:
            areas = np.diag(np.asarray(metrics.ja[0, 0])).copy()
            jac_const = float(metrics.jac[0, 0])
        jac = None
    else:
        areas = None
        jac_const = 0.0
    return MeshArrays(
        d, p1, n_elem, np.asarray(setup.dsplit.matrix), weights, setup.gas.gamma,
        setup.gas.inv_gamma_minus_one, cart, areas, jac_const, ja, jac, plus, minus,
    )


def _mesh(m):
    return m if isinstance(m, MeshArrays) else mesh_from_setup(m)


def volume(u, setup, flux="ranocha", precompute="none", nthreads=0, variant="glibc"):
    m = _mesh(setup)
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty_like(u)
    lib(variant).or_volume(ctypes.byref(m.struct), _ptr(u), _ptr(out), FLUX_IDS[flux], PRE_IDS[precompute], nthreads)
    return out


def surface(u, setup, flux="llf", out=None, nthreads=0, variant="glibc"):
    m = _mesh(setup)
    u = np.ascontiguousarray(u, dtype=np.float64)
    if out is None:
        out = np.zeros_like(u)
    assert out.flags.c_contiguous and out.dtype == np.float64
    lib(variant).or_surface(ctypes.byref(m.struct), _ptr(u), _ptr(out), FLUX_IDS[flux], nthreads)
    return out


class OracleAdmissibilityError(RuntimeError):
    pass


def gate(u, setup):
    """(element, node, rho, p) of the first inadmissible node, or None."""
    m = _mesh(setup)
    u = np.ascontiguousarray(u, dtype=np.float64)
    rho = np.zeros(1)
    p = np.zeros(1)
    g = lib().or_gate(ctypes.byref(m.struct), _ptr(u), _ptr(rho), _ptr(p))
    if g < 0:
        return None
    nn = u.shape[1]
    return int(g // nn), int(g % nn), float(rho[0]), float(p[0])


def rhs(u, setup, volume_flux="ranocha", surface_flux="ranocha", precompute="none", nthreads=0,
        variant="glibc"):
    m = _mesh(setup)
    u = np.ascontiguousarray(u, dtype=np.float64)
    bad = gate(u, m)
    if bad is not None:
        e, i, rho, p = bad
        raise OracleAdmissibilityError(
            "inadmissible state at element %d, node %d: rho=%r, p=%r" % (e, i, rho, p)
        )
    du = np.empty_like(u)
    lib(variant).or_rhs(
        ctypes.byref(m.struct), _ptr(u), _ptr(du), FLUX_IDS[volume_flux], FLUX_IDS[surface_flux],
        PRE_IDS[precompute], nthreads,
    )
    return du


def rhs_range(u, mesh, du, lo, hi, volume_flux="ranocha", surface_flux="ranocha", precompute="none", nthreads=0,
              variant="glibc"):
    """Rows [lo, hi) of rhs into ``du`` (no gate): the interior / boundary
    split of a slab partition (interior rows never read ghost traces)."""
    m = _mesh(mesh)
    u = np.ascontiguousarray(u, dtype=np.float64)
    assert du.flags.c_contiguous and du.dtype == np.float64 and du.shape == u.shape
    lib(variant).or_rhs_range(ctypes.byref(m.struct), _ptr(u), _ptr(du), FLUX_IDS[volume_flux], FLUX_IDS[surface_flux],
                              PRE_IDS[precompute], int(lo), int(hi), nthreads)
    return du


def two_point(ul, ur, normal, flux, gamma=1.4, cart_axis=-1, precompute="none", variant="glibc"):
    ul = np.ascontiguousarray(ul, dtype=np.float64)
    ur = np.ascontiguousarray(ur, dtype=np.float64)
    nrm = np.zeros(3)
    nrm[: len(normal)] = normal
    f = np.zeros(5)
    d = ul.shape[0] - 2
    lib(variant).or_two_point(d, FLUX_IDS[flux], PRE_IDS[precompute], gamma, 1.0 / (gamma - 1.0),
                       _ptr(ul), _ptr(ur), _ptr(nrm), cart_axis, _ptr(f))
    return f[: d + 2]


def logmean(a, b):
    return lib().or_logmean(a, b)


def inv_logmean(a, b):
    return lib().or_inv_logmean(a, b)


def max_threads():
    return lib().or_max_threads()


# --- time stepping (numpy, same operation sequence as timeint.py:149-163) ---

RK54_A = (
    0.0,
    -567301805773 / 1357537059087,
    -2404267990393 / 2016746695238,
    -3550918686646 / 2091501179385,
    -1275806237668 / 842570457699,
)
RK54_B = (
    1432997174477 / 9575080441755,
    5161836677717 / 13612068292357,
    1720146321549 / 2090206949498,
    3134564353537 / 4481467310338,
    2277821191437 / 14882151754819,
)


def rk54_step(u, dt, rhs_fn):
    du = np.zeros_like(u)
    v = np.array(u, copy=True)
    for i in range(5):
        k = rhs_fn(v)
        du = RK54_A[i] * du + dt * k
        v = v + RK54_B[i] * du
    return v


def ssprk43_step(u, dt, rhs_fn):
    """Four-stage third-order SSP RK in Shu-Osher form (NOT in the reference)."""
    u1 = u + 0.5 * dt * rhs_fn(u)
    u2 = u1 + 0.5 * dt * rhs_fn(u1)
    u3 = (2.0 / 3.0) * u + (1.0 / 3.0) * u2 + (1.0 / 6.0) * dt * rhs_fn(u2)
    return u3 + 0.5 * dt * rhs_fn(u3)


# ------------------------------------------------------------ diagnostics
# numpy restatement of the reference's diagnostics reductions (test
# infrastructure: checked against tests/golden/diagnostics.npz, written by the
# reference itself).


def _wbar_jac(setup):
    """wbar (discretization.py:619-621) times J, shape (n_elem, nn)."""
    wbar = np.ones(1)
    for _ in range(setup.d):
        wbar = np.kron(wbar, np.asarray(setup.op.weights, dtype=np.float64))
    return wbar[None, :] * np.asarray(setup.metrics.jac)


def _primitives(u, gamma):
    d = u.shape[-1] - 2
    rho = u[..., 0]
    v = u[..., 1 : d + 1] / rho[..., None]
    return d, rho, v


def entropy_vars(u, gamma):
    """euler.py:129-146."""
    d, rho, v = _primitives(u, gamma)
    p = (gamma - 1.0) * (u[..., d + 1] - 0.5 * rho * np.sum(v * v, axis=-1))
    s = np.log(p) - gamma * np.log(rho)
    rho_p = rho / p
    w = np.empty_like(u)
    w[..., 0] = (gamma - s) * (1.0 / (gamma - 1.0)) - 0.5 * rho_p * np.sum(v * v, axis=-1)
    w[..., 1 : d + 1] = rho_p[..., None] * v
    w[..., d + 1] = -rho_p
    return w


def conserved_totals(u, setup):
    """discretization.py:1027-1031."""
    return np.sum(_wbar_jac(setup)[..., None] * u, axis=(0, 1))


def entropy_rate(u, dudt, setup, gamma=1.4):
    """discretization.py:1011-1024: (total, total / scale)."""
    w = entropy_vars(u, gamma)
    wt = _wbar_jac(setup)
    total = float(np.sum(wt * np.sum(w * dudt, axis=-1)))
    scale = np.sum(np.abs(wt[..., None] * w * dudt))
    return (0.0, 0.0) if scale == 0.0 else (total, total / scale)


def error_norm_l2(u, u_exact, setup):
    """discretization.py:1033-1037."""
    diff = u - u_exact
    return np.sqrt(np.sum(_wbar_jac(setup)[..., None] * diff * diff, axis=(0, 1)))


def stable_dt(u, setup, cfl=0.5, gamma=1.4):
    """timeint.py:138-146 with max_signal_speed (euler.py:105-112)."""
    d, rho, v = _primitives(u, gamma)
    mom = u[..., 1 : d + 1]
    p = (gamma - 1.0) * (u[..., d + 1] - 0.5 * np.sum(mom * mom, axis=-1) / rho)
    lam = np.sqrt(np.sum(v * v, axis=-1)) + np.sqrt(gamma * p / rho)
    scale = np.asarray(setup.metrics.jac) ** (1.0 / d)
    return cfl * float(np.min(scale / (lam * (2 * setup.op.degree + 1))))


# ------------------------------------------------------- Gauss-family schemes
# numpy restatement of the reference's entropy projection and scatter tables
# (test infrastructure; pinned against tests/golden/gauss_*.npz written by the
# reference itself, tests/test_oracle.py). The element loop is C (or_gauss_rhs).

_FACE_N = (-1.0, 1.0)


def gauss_tables(op, scheme):
    """(vv, cvol, cface, lift) of operators.py:300-357 in float, from the
    operator's own arrays: the hybridized skew operator
    Q_h = [[skew(M D), R^T N / 2], [-N R / 2, N / 2]] gives the volume pair
    weights 2 Q[a,b] / w_a (gauss_fluxdiff) -- or the split-derivative
    matrix 2D - M^-1 R^T B N R (gauss_surface_correction) -- the crossing
    weights 2 Q[a, face] / w_a and 2 Q[face, a], and the lift R[s] / w."""
    w = np.asarray(op.weights, dtype=np.float64)
    D = np.asarray(op.D, dtype=np.float64)
    R = np.asarray(op.boundary_interp, dtype=np.float64)
    n = w.shape[0]
    nf = np.array(_FACE_N)
    md = w[:, None] * D
    q = np.zeros((n + 2, n + 2))
    q[:n, :n] = 0.5 * (md - md.T)
    q[:n, n:] = 0.5 * (R.T * nf[None, :])
    q[n:, :n] = -0.5 * (nf[:, None] * R)
    q[n:, n:] = 0.5 * np.diag(nf)
    vv = np.zeros((n, n))
    if scheme == "gauss_surface_correction":
        mat = 2.0 * D - (R.T @ (nf[:, None] * R)) / w[:, None]
        for a in range(n):
            for b in range(a + 1, n):
                if mat[a, b] != 0.0 or mat[b, a] != 0.0:
                    vv[a, b], vv[b, a] = float(mat[a, b]), float(mat[b, a])
    else:
        for a in range(n):
            for b in range(a + 1, n):
                if q[a, b] != 0.0 or q[b, a] != 0.0:
                    vv[a, b], vv[b, a] = float(2.0 * q[a, b] / w[a]), float(2.0 * q[b, a] / w[b])
    cvol = np.array([[float(2.0 * q[a, n + s] / w[a]) for a in range(n)] for s in (0, 1)])
    cface = np.array([[float(2.0 * q[n + s, a]) for a in range(n)] for s in (0, 1)])
    lift = np.array([[float(R[s, a] / w[a]) for a in range(n)] for s in (0, 1)])
    return vv, cvol, cface, lift


def gauss_project(u, op, gamma=1.4):
    """Entropy-projected face states (n_elem, d, 2, fn, nvar) as
    discretization._project_all computes them (entropy variables, boundary
    interpolation along each direction, entropy2cons); None entries if a face
    state is inadmissible (the caller raises)."""
    u = np.asarray(u, dtype=np.float64)
    n_elem, nn, nvar = u.shape
    d = nvar - 2
    p1 = round(nn ** (1.0 / d))
    w = entropy_vars(u, gamma)
    w_nd = w.reshape((n_elem,) + (p1,) * d + (nvar,))
    fn = p1 ** (d - 1)
    out = np.empty((n_elem, d, 2, fn, nvar))
    R = np.asarray(op.boundary_interp, dtype=np.float64)
    for n in range(d):
        moved = np.moveaxis(w_nd, n + 1, -2)
        for side in (0, 1):
            wf = np.einsum("...kv,k->...v", moved, R[side]).reshape(n_elem, -1, nvar)
            out[:, n, side] = entropy2cons(wf, gamma)
    return out


def entropy2cons(w, gamma):
    """euler.py:149-170."""
    d = w.shape[-1] - 2
    b = -w[..., d + 1]
    if not np.all(b > 0.0):
        raise OracleAdmissibilityError("entropy2cons: last entropy variable must be negative (min -w=%r)"
                                       % float(np.min(b)))
    v = w[..., 1 : d + 1] / b[..., None]
    s = gamma - (gamma - 1.0) * (w[..., 0] + 0.5 * b * np.sum(v * v, axis=-1))
    p = np.exp((s + gamma * np.log(b)) / (1.0 - gamma))
    rho = b * p
    out = np.empty_like(w)
    out[..., 0] = rho
    out[..., 1 : d + 1] = rho[..., None] * v
    out[..., d + 1] = p * (1.0 / (gamma - 1.0)) + 0.5 * rho * np.sum(v * v, axis=-1)
    return out


def gauss_face_traces(ja, op, d):
    """Each element's own metric traces (n_elem, d, 2, fn, d) as
    discretization._own_face_ja computes them per element (einsum)."""
    ja = np.asarray(ja, dtype=np.float64)
    n_elem, nn = ja.shape[:2]
    p1 = round(nn ** (1.0 / d))
    R = np.asarray(op.boundary_interp, dtype=np.float64)
    out = np.empty((n_elem, d, 2, p1 ** (d - 1), d))
    for e in range(n_elem):
        nd = ja[e].reshape((p1,) * d + (d, d))
        for n in range(d):
            field = np.moveaxis(nd[..., n, :], n, -2)
            for s in (0, 1):
                out[e, n, s] = np.einsum("...kj,k->...j", field, R[s]).reshape(-1, d)
    return out


def gauss_rhs(u, setup, scheme, volume_flux, surface_flux, proj=None, nrm=None, fnrm=None, variant="glibc"):
    """du of rhs(u, setup, RhsConfig(volume_scheme=scheme, ...)) on Gauss
    operators (discretization.py:976-995, the scalar path). ``setup``:
    d, op, gas, metrics.{ja, jac[, face_ja]}, plus_neighbor."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    d = setup.d
    gamma = setup.gas.gamma
    bad = gate(u, _gauss_mesh(setup, u.shape[0]))
    if bad is not None:
        e, i, rho, p = bad
        raise OracleAdmissibilityError("inadmissible state at element %d, node %d: rho=%r, p=%r" % (e, i, rho, p))
    if proj is None:
        proj = gauss_project(u, setup.op, gamma)
    if nrm is None:
        nrm = gauss_face_traces(setup.metrics.ja, setup.op, d)
    if fnrm is None and getattr(setup.metrics, "face_ja", None) is not None:
        fnrm = np.stack([np.asarray(setup.metrics.face_ja[n]) for n in range(d)], axis=1)
    vv, cvol, cface, lift = (np.ascontiguousarray(t) for t in gauss_tables(setup.op, scheme))
    tab = OrGaussTables(vv.ctypes.data, cvol.ctypes.data, cface.ctypes.data, lift.ctypes.data)
    m = _gauss_mesh(setup, u.shape[0])
    proj = np.ascontiguousarray(proj)
    nrm = np.ascontiguousarray(nrm)
    fnrm = None if fnrm is None else np.ascontiguousarray(fnrm)
    du = np.empty_like(u)
    lib(variant).or_gauss_rhs(ctypes.byref(m.struct), ctypes.byref(tab), _ptr(u), _ptr(proj), _ptr(nrm), _ptr(fnrm),
                              _ptr(du), FLUX_IDS[volume_flux], FLUX_IDS[surface_flux])
    return du


def _gauss_mesh(setup, n_elem):
    d = setup.d
    plus = np.stack([np.asarray(setup.plus_neighbor[n]) for n in range(d)])
    minus = np.empty_like(plus)
    for n in range(d):
        minus[n, plus[n]] = np.arange(n_elem)
    w = np.asarray(setup.op.weights)
    return MeshArrays(d, w.shape[0], n_elem, np.zeros((w.shape[0], w.shape[0])), w, setup.gas.gamma,
                      setup.gas.inv_gamma_minus_one, False, None, 0.0, np.asarray(setup.metrics.ja),
                      np.asarray(setup.metrics.jac), plus, minus)
