"""Drop-in RHS / volume-integral entry points (reference discretization.py and
batched.py signatures), executed by the sm_100a kernels of libfdg.so.

    rhs(u, setup, config, counter=None)            discretization.py:896-963
    volume_fluxdiff(u_elem, dop, metrics, vol_flux, gas, pre=None)
                                                   discretization.py:267-323
    mesh_fluxdiff_volume(u, setup, config)         batched.py:450-511
    mesh_surface(u, setup, surface_flux, out)      batched.py:514-544
    surface_terms(u, setup, surface_flux, out=None)  discretization.py:681-788

``RhsConfig.kernel`` keeps the reference's two names with the reference's
meaning: "reference" is the bitwise-reproducible path (the FAITHFUL kernels:
the scalar path's operation order, IEEE division, correctly rounded log) and
"batched" the throughput path (the FAST kernels). Inputs may be numpy arrays
(copied through pinned staging buffers, a new numpy array is returned, as in
the reference) or torch tensors (CUDA tensors stay on the device; CPU tensors
are copied in and the result copied back).

``setup`` may be this package's SpatialSetup or the reference's own.
"""

import os
from dataclasses import dataclass

import numpy as np

from . import fluxes as _fluxes
from .device import device_mesh_for, scheme_struct
from .errors import AdmissibilityError, ConfigurationError, UnsupportedOperatorError
from .geometry import compute_metrics, element_coords, neighbor_table
from .operators import build_dsplit, node_lines, pair_table

VOLUME_SCHEMES = ("fluxdiff", "gauss_fluxdiff", "gauss_surface_correction")
GAUSS_SCHEMES = ("gauss_fluxdiff", "gauss_surface_correction")
PRECOMPUTE_MODES = ("none", "primitives", "primitives_and_logs")
KERNELS = ("reference", "batched")
VOLUME_KINDS = _fluxes.VOLUME_KINDS
SURFACE_KINDS = _fluxes.SURFACE_KINDS
_OUT_OF_SCOPE_SCHEMES = ("strong", "weak", "overintegration")


@dataclass(frozen=True)
class RhsConfig:
    """Scheme selection for one RHS evaluation (reference discretization.py:87-150)."""

    volume_scheme: str = "fluxdiff"
    volume_flux: str = "ranocha"
    surface_flux: str = "ranocha"
    precompute: str = "none"
    overint_degree: int = None
    kernel: str = "reference"

    def validate(self, setup=None):
        if self.volume_scheme not in VOLUME_SCHEMES:
            if self.volume_scheme in _OUT_OF_SCOPE_SCHEMES:
                raise ConfigurationError(
                    "volume_scheme: %r is not on the device path (flux differencing only)" % (self.volume_scheme,)
                )
            raise ConfigurationError(
                "volume_scheme: unknown scheme %r (choose from %s)" % (self.volume_scheme, ", ".join(VOLUME_SCHEMES))
            )
        if self.precompute not in PRECOMPUTE_MODES:
            raise ConfigurationError(
                "precompute: unknown mode %r (choose from %s)" % (self.precompute, ", ".join(PRECOMPUTE_MODES))
            )
        if self.kernel not in KERNELS:
            raise ConfigurationError("kernel: unknown kernel %r (choose from %s)" % (self.kernel, ", ".join(KERNELS)))
        if self.surface_flux not in SURFACE_KINDS:
            raise ConfigurationError(
                "surface_flux: unknown kind %r (choose from %s)" % (self.surface_flux, ", ".join(SURFACE_KINDS))
            )
        _fluxes.require_volume_kind(self.volume_flux)
        if setup is not None:
            family = getattr(setup.op, "family", "lgl")
            if self.volume_scheme.startswith("gauss") and family != "gauss":
                raise ConfigurationError(
                    "volume_scheme: %r requires gauss operators, got family %r" % (self.volume_scheme, family)
                )
            if self.volume_scheme == "fluxdiff" and family != "lgl":
                raise ConfigurationError(
                    "volume_scheme: 'fluxdiff' requires the lgl family (diagonal boundary operator); "
                    "use the gauss schemes on gauss nodes"
                )

    def scheme(self):
        return scheme_struct(self.volume_flux, self.surface_flux, self.precompute, self.kernel)


def as_rhs_config(config):
    """This package's RhsConfig for ``config``, which may be the reference's
    own ``fluxdg.RhsConfig`` (discretization.py:87-150) or any object with
    its fields: the scheme is built from the fields, never from methods the
    reference's class lacks."""
    if isinstance(config, RhsConfig):
        return config
    try:
        fields = {k: getattr(config, k) for k in ("volume_scheme", "volume_flux", "surface_flux", "precompute")}
    except AttributeError as err:
        raise ConfigurationError("config: not an RhsConfig (%s)" % (err,)) from err
    fields["kernel"] = getattr(config, "kernel", "reference")
    fields["overint_degree"] = getattr(config, "overint_degree", None)
    return RhsConfig(**fields)


@dataclass(frozen=True)
class SpatialSetup:
    """Everything precomputable for RHS evaluations on one mesh/operator
    (reference discretization.py:576-606)."""

    mesh: object
    op: object
    gas: object
    metrics: object
    coords: np.ndarray
    lines: tuple
    plus_neighbor: tuple
    dsplit: object

    @property
    def n_elements(self):
        return self.mesh.n_elements

    @property
    def n_nodes(self):
        return self.op.n_nodes**self.mesh.d

    @property
    def d(self):
        return self.mesh.d

    @property
    def dofs(self):
        return self.n_elements * self.n_nodes

    @property
    def wbar(self):
        w = np.ones(1)
        for _ in range(self.d):
            w = np.kron(w, self.op.weights)
        return w


def build_setup(mesh, op, gas, with_coords=True, device=None):
    """Geometry, connectivity and operator tables (reference discretization.py:609-657).
    ``with_coords=False`` skips the nodal coordinates of Cartesian meshes
    (3.2 GB at 128^3, N=3) when no initial condition needs them.
    ``device`` (extension, e.g. "cuda"): coordinates and curved metrics are
    computed on the GPU (geometry.device_geometry) and held as CUDA tensors,
    so no per-node geometry is built on or copied from the host."""
    if op.family == "gauss":
        return _build_gauss_setup(mesh, op, gas, device)
    if op.family != "lgl":
        raise UnsupportedOperatorError("unknown operator family %r" % (op.family,))
    if device is not None:
        from .geometry import MetricData, device_geometry

        coords, ja, jac = device_geometry(mesh, op, device=device, coords=with_coords)
        if mesh.is_cartesian:
            metrics = compute_metrics(mesh, op)  # d areas + J, no per-node arrays
        else:
            metrics = MetricData(mesh.d, op.n_nodes, mesh.n_elements, False, ja=ja, jac=jac)
    else:
        coords = element_coords(mesh, op) if (with_coords or not mesh.is_cartesian) else None
        metrics = compute_metrics(mesh, op, coords)
    return SpatialSetup(
        mesh=mesh,
        op=op,
        gas=gas,
        metrics=metrics,
        coords=coords,
        lines=node_lines(op.n_nodes, mesh.d),
        plus_neighbor=neighbor_table(mesh),
        dsplit=build_dsplit(op),
    )


def _build_gauss_setup(mesh, op, gas, device=None):
    """Setup on Gauss nodes (reference discretization.py:609-657 with a gauss
    operator): coordinates at the Gauss nodes, per-node metric terms (also on
    Cartesian meshes: the gauss kernels always take the directional form,
    as the reference's gauss path does), neighbours; no split matrix."""
    from .geometry import MetricData, device_geometry

    R = op.boundary_interp
    if device is not None:
        coords, ja, jac = device_geometry(mesh, op, device=device, coords=True)
        if mesh.is_cartesian:
            m = compute_metrics(mesh, op)
            ja, jac = m.ja, m.jac
        metrics = MetricData(mesh.d, op.n_nodes, mesh.n_elements, mesh.is_cartesian, ja=ja, jac=jac,
                             boundary_interp=R)
    else:
        coords = element_coords(mesh, op)
        m = compute_metrics(mesh, op, coords)
        metrics = MetricData(mesh.d, op.n_nodes, mesh.n_elements, m.cartesian, areas=m.areas,
                             jac_const=m.jac_const, ja=m.ja, jac=m.jac, boundary_interp=R)
    return SpatialSetup(
        mesh=mesh, op=op, gas=gas, metrics=metrics, coords=coords,
        lines=node_lines(op.n_nodes, mesh.d), plus_neighbor=neighbor_table(mesh), dsplit=None,
    )


# --------------------------------------------------------------- plumbing


def _is_torch(x):
    try:
        import torch

        return isinstance(x, torch.Tensor)
    except ImportError:  # pragma: no cover
        return False


class _Io:
    """Moves a caller's array to the device and the result back in the
    caller's flavour (numpy -> numpy, torch CPU -> torch CPU, CUDA -> CUDA)."""

    def __init__(self, dm, u, key="in"):
        # `key`: the pinned staging slot; two live _Io objects need two slots
        # (the first's H2D copy is asynchronous from its slot)
        torch = dm.torch
        self.dm = dm
        self.kind = "cuda" if (_is_torch(u) and u.is_cuda) else ("torch" if _is_torch(u) else "numpy")
        if self.kind == "cuda":
            self.u = u if (u.dtype == torch.float64 and u.is_contiguous()) else u.double().contiguous()
        elif self.kind == "torch" and u.dtype == torch.float64 and u.is_contiguous() and u.is_pinned():
            # pinned caller buffer: one async H2D copy, no host staging
            self.u = torch.empty(dm.shape, dtype=torch.float64, device=dm.device)
            self.u.copy_(u.view(dm.shape), non_blocking=True)
        else:
            arr = u if _is_torch(u) else torch.from_numpy(np.ascontiguousarray(u, dtype=np.float64))
            if tuple(arr.shape) != dm.shape:
                raise ValueError("state shape %r does not match the mesh %r" % (tuple(arr.shape), dm.shape))
            pinned = dm.staging(key, dm.shape)
            pinned.copy_(arr)
            self.u = torch.empty(dm.shape, dtype=torch.float64, device=dm.device)
            self.u.copy_(pinned, non_blocking=True)
        if tuple(self.u.shape) != dm.shape:
            raise ValueError("state shape %r does not match the mesh %r" % (tuple(self.u.shape), dm.shape))

    def device_out(self, out=None):
        if out is not None and _is_torch(out) and out.is_cuda:
            return out
        return self.dm.empty()

    def finish(self, res, out=None):
        torch = self.dm.torch
        if out is not None and _is_torch(out):
            if out.data_ptr() == res.data_ptr():
                return out
            out.copy_(res.view(out.shape), non_blocking=out.is_pinned() or out.is_cuda)
            if not out.is_cuda:
                torch.cuda.current_stream().synchronize()
            return out
        if self.kind == "cuda":
            return res
        pinned = self.dm.staging("out", self.dm.shape)
        pinned.copy_(res, non_blocking=True)
        self.dm.torch.cuda.current_stream().synchronize()
        if self.kind == "torch":
            if out is not None:
                out.copy_(pinned)
                return out
            return pinned.clone()
        if out is not None:
            out[...] = pinned.numpy()
            return out
        return pinned.numpy().copy()


def _pinned_f64(t, shape):
    return (
        _is_torch(t)
        and not t.is_cuda
        and t.is_pinned()
        and str(t.dtype) == "torch.float64"
        and t.is_contiguous()
        and t.numel() == int(np.prod(shape))
    )


def _count(counter, two_point, logmean):
    _fluxes.bump(counter, two_point=two_point, logmean=logmean)


_PAIR_COUNTS = {}  # id(dsplit matrix) -> (matrix, pair count): the counters need it every call


def _volume_counts(setup, vol_flux):
    d = setup.d
    p1 = setup.op.degree + 1
    mat = setup.dsplit.matrix
    hit = _PAIR_COUNTS.get(id(mat))
    if hit is None or hit[0] is not mat:
        hit = _PAIR_COUNTS[id(mat)] = (mat, len(pair_table(np.asarray(mat))))
    two_point = setup_n_elements(setup) * d * p1 ** (d - 1) * hit[1]
    logmean = 2 * two_point if vol_flux in ("ranocha", "chandrashekar") else 0
    return two_point, logmean


def _surface_logmeans(surface_flux, n_faces):
    """Two log means per Ranocha surface evaluation (fluxes.py:281,
    batched.py:218); Chandrashekar's two (rho and beta) are counted alike."""
    return 2 * n_faces if surface_flux in ("ranocha", "chandrashekar") else 0


def _surface_counts(setup):
    d = setup.d
    p1 = setup.op.degree + 1
    return setup_n_elements(setup) * d * p1 ** (d - 1)


def setup_n_elements(setup):
    n = getattr(setup, "n_elements", None)
    if n is not None:
        return int(n)
    return int(np.asarray(setup.plus_neighbor[0]).shape[0])


def _raise_gate(dm, io, gas):
    first_bad, _ = dm.read_status()
    if first_bad >= 0:
        dm.raise_if_inadmissible(io.u, first_bad, gas.gamma)


# ------------------------------------------------------------ entry points


def _raise_cons2prim(dm, u_dev, gas):
    """The reference's cons2prim error (euler.py:47-60 via _require_admissible)
    for a state the device gate rejected."""
    t = u_dev
    rho = t[..., 0]
    mom = t[..., 1 : dm.d + 1]
    p = (gas.gamma - 1.0) * (t[..., dm.d + 1] - 0.5 * rho * ((mom / rho[..., None]) ** 2).sum(-1))
    raise AdmissibilityError(
        "cons2prim: inadmissible state (min rho=%r, min p=%r)" % (float(rho.min()), float(p.min()))
    )


def mesh_fluxdiff_volume(u, setup, config, out=None):
    """VOL = (1/J) sum_n sum_k Dsplit f*_n  for every element (batched.py:450-511).
    Not negated. Raises AdmissibilityError like the reference's cons2prim.
    ``out`` (extension): a CUDA or pinned CPU tensor to receive VOL."""
    config = as_rhs_config(config)
    config.validate(setup)
    dm = device_mesh_for(setup)
    scheme = config.scheme()
    if _pinned_f64(u, dm.shape) and (out is None or _pinned_f64(out, dm.shape)):
        # host-resident state: chunked H2D / kernel / D2H pipeline
        dm.reset_status()
        dest = out if out is not None else dm.staging("out", dm.shape)
        u_dev, res = dm.volume_host(u, scheme, dest)
        io = None
    elif isinstance(u, np.ndarray) and out is None and u.dtype == np.float64 and u.flags.c_contiguous \
            and tuple(u.shape) == dm.shape and u.nbytes >= _HOST_PIPELINE_MIN_BYTES:
        # numpy in / numpy out (the reference's own call): the state goes
        # through the same chunked pipeline via the pinned staging buffers
        # (one host memcpy in, one out; the H2D / kernel / D2H chunks overlap)
        pin_in = dm.staging("in", dm.shape)
        pin_out = dm.staging("out", dm.shape)
        _host_copy(pin_in.numpy(), u)
        dm.reset_status()
        u_dev, _ = dm.volume_host(pin_in, scheme, pin_out)
        first_bad, _ = dm.read_status()
        if first_bad >= 0:
            _raise_cons2prim(dm, u_dev, setup.gas)
        tp, lm = _volume_counts(setup, config.volume_flux)
        _count(None, tp, lm)
        res = np.empty(dm.shape)
        _host_copy(res, pin_out.numpy())
        return res
    else:
        io = _Io(dm, u)
        dm.reset_status()
        res = dm.volume(io.u, scheme, out=io.device_out(out))
        u_dev = io.u
    first_bad, _ = dm.read_status()
    if first_bad >= 0:
        _raise_cons2prim(dm, u_dev, setup.gas)
    tp, lm = _volume_counts(setup, config.volume_flux)
    _count(None, tp, lm)
    if io is None:
        # read_status synchronized the stream that waited for the last D2H copy
        return res if out is not None else res.clone()
    return io.finish(res, out=out)


# numpy states at least this large take the chunked host pipeline
_HOST_PIPELINE_MIN_BYTES = 4 << 20

_COPY_POOL = None


def _host_copy(dst, src):
    """dst[...] = src for large C-contiguous float64 arrays, split along the
    first axis over the host cores this process may run on (numpy releases the
    GIL inside the copy). One thread moves ~5-10 GB/s and, into a fresh array,
    also takes every first-touch page fault; the 5.4 GB cfg5 state took 0.6 s
    each way on one thread."""
    global _COPY_POOL
    n = dst.shape[0]
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    parts = min(cores, 16, max(1, dst.nbytes >> 24), n)  # >= 16 MB per piece
    if parts <= 1:
        np.copyto(dst, src)
        return
    if _COPY_POOL is None or _COPY_POOL._max_workers < parts:
        from concurrent.futures import ThreadPoolExecutor

        _COPY_POOL = ThreadPoolExecutor(max_workers=parts, thread_name_prefix="fdg-copy")
    cuts = [n * i // parts for i in range(parts + 1)]
    futs = [_COPY_POOL.submit(np.copyto, dst[a:b], src[a:b]) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]
    for f in futs:
        f.result()


def mesh_surface(u, setup, surface_flux, out, kernel="batched"):
    """out += SURF, the LGL interface terms (batched.py:514-544). Raises
    AdmissibilityError like the reference's cons2prim (batched.py:521) on an
    inadmissible state, before ``out`` is touched."""
    if surface_flux not in SURFACE_KINDS:
        raise ConfigurationError("surface_flux: unknown kind %r" % (surface_flux,))
    dm = device_mesh_for(setup)
    io = _Io(dm, u)
    dm.reset_status()
    dm.gate(io.u)
    first_bad, _ = dm.read_status()
    if first_bad >= 0:
        _raise_cons2prim(dm, io.u, setup.gas)
    acc = _Io(dm, out, key="in2")
    dm.surface(io.u, scheme_struct(None, surface_flux, "none", kernel), acc.u)
    sc = _surface_counts(setup)
    _count(None, sc, _surface_logmeans(surface_flux, sc))
    return acc.finish(acc.u, out=out)


def surface_terms(u, setup, surface_flux, subtract_own=False, face_states=None, out=None):
    """SURF added into ``out`` (zeros if None) with the scalar path's
    arithmetic (discretization.py:681-760, LGL branch). The reference's
    strong-form (``subtract_own``) and projected-face (``face_states``)
    variants serve schemes that are not flux differencing on LGL nodes; they
    raise UnsupportedOperatorError here."""
    if subtract_own:
        raise UnsupportedOperatorError("surface_terms: subtract_own (strong-form coupling) is not on the device path")
    if face_states is not None:
        raise UnsupportedOperatorError("surface_terms: face_states overrides are not on the device path")
    if out is None:
        out = np.zeros_like(np.asarray(u, dtype=np.float64)) if not _is_torch(u) else u.new_zeros(u.shape)
    return mesh_surface(u, setup, surface_flux, out, kernel="reference")


def rhs(u, setup, config, counter=None):
    """du/dt = -(VOL + SURF) (discretization.py:896-949), admissibility gate
    included (discretization.py:660-672). The gauss schemes (volume_scheme
    "gauss_fluxdiff" / "gauss_surface_correction" on Gauss operators) run
    fdg_gauss_* (discretization.py:976-995)."""
    config = as_rhs_config(config)
    config.validate(setup)
    if config.volume_scheme in GAUSS_SCHEMES:
        return _gauss_rhs(u, setup, config, counter)
    dm = device_mesh_for(setup)
    io = _Io(dm, u)
    dm.reset_status()
    res = dm.rhs(io.u, config.scheme(), out=io.device_out())
    _raise_gate(dm, io, setup.gas)
    tp, lm = _volume_counts(setup, config.volume_flux)
    sc = _surface_counts(setup)
    _count(counter, tp + sc, lm + _surface_logmeans(config.surface_flux, sc))
    return io.finish(res)


def _gauss_counts(setup, config):
    """The reference's counter totals for the gauss path (measured on it):
    per element line, |pairs| + 2 (p+1) volume evaluations and 2 interface
    evaluations; two log means per Ranocha / Chandrashekar evaluation."""
    from .operators import gauss_scatter_tables

    d = setup.d
    p1 = setup.op.degree + 1
    vv = gauss_scatter_tables(setup.op, config.volume_scheme)[0]
    pairs = sum(1 for a in range(p1) for b in range(a + 1, p1) if vv[a, b] != 0.0 or vv[b, a] != 0.0)
    lines = setup_n_elements(setup) * d * p1 ** (d - 1)
    vol = lines * (pairs + 2 * p1)
    surf = 2 * lines
    logs = ("ranocha", "chandrashekar")
    return vol + surf, (2 * vol if config.volume_flux in logs else 0) + (2 * surf if config.surface_flux in logs else 0)


def _gauss_rhs(u, setup, config, counter):
    from .device import gauss_mesh_for

    gm = gauss_mesh_for(setup, config.volume_scheme)
    io = _Io(gm, u)
    gm.reset_status()
    gm.gate(io.u)
    first_bad, _ = gm.read_status()
    if first_bad >= 0:
        gm.raise_if_inadmissible(io.u, first_bad, setup.gas.gamma)
    proj, nrm = gm.project(io.u)
    res = gm.rhs(io.u, config.scheme(), out=io.device_out(), proj=proj, nrm=nrm)
    _, bad_face = gm.read_status()
    if bad_face >= 0:
        _raise_projection(io.u, setup, bad_face)
    tp, lm = _gauss_counts(setup, config)
    _count(counter, tp, lm)
    return io.finish(res)


def _raise_projection(u_dev, setup, code):
    """The reference's _project_all error (discretization.py:826-836)."""
    from .euler import entropy_vars

    n, side = divmod(int(code), 2)
    u = u_dev.double().cpu().numpy()
    d = u.shape[-1] - 2
    p1 = setup.op.degree + 1
    w = entropy_vars(u, setup.gas).reshape((u.shape[0],) + (p1,) * d + (d + 2,))
    row = np.asarray(setup.op.boundary_interp)[side]
    wf = np.tensordot(np.moveaxis(w, n + 1, -2), row, axes=([-2], [0]))
    b = -wf[..., d + 1]
    raise AdmissibilityError(
        "entropy projection produced an inadmissible face state (direction %d, side %d): "
        "entropy2cons: last entropy variable must be negative (min -w=%r)" % (n, side, float(np.min(b)))
    )


class _ElementSetup:
    """A one-element periodic setup for the per-element entry point. Curved
    metrics live in device buffers that each call overwrites in place (the
    DeviceMesh reads them through its pointers), so one device image serves
    every element of a mesh."""

    def __init__(self, dop, gas, d, cart):
        from types import SimpleNamespace

        self.d = d
        self.op = dop.op
        self.dsplit = dop
        self.gas = gas
        nn = dop.op.n_nodes**d
        self.plus_neighbor = tuple(np.zeros(1, dtype=np.int64) for _ in range(d))
        self.n_elements = 1
        if cart is not None:
            areas, jac_const = cart
            self.metrics = SimpleNamespace(cartesian=True, areas=tuple(areas), jac_const=float(jac_const))
        else:
            import torch

            self.metrics = SimpleNamespace(
                cartesian=False,
                ja=torch.zeros((1, nn, d, d), dtype=torch.float64, device="cuda"),
                jac=torch.ones((1, nn), dtype=torch.float64, device="cuda"),
            )


_ELEM_CACHE = {}  # key -> (dop, _ElementSetup): strong refs, a few entries (LRU)
_ELEM_CACHE_MAX = 8


def _element_setup(dop, gas, d, cart):
    key = (id(dop), d, float(gas.gamma), cart)
    hit = _ELEM_CACHE.pop(key, None)
    if hit is None or hit[0] is not dop:
        hit = (dop, _ElementSetup(dop, gas, d, cart))
    _ELEM_CACHE[key] = hit  # most recent last
    while len(_ELEM_CACHE) > _ELEM_CACHE_MAX:
        _ELEM_CACHE.pop(next(iter(_ELEM_CACHE)))
    return hit[1]


def _axis_aligned_areas(ja):
    """Per-direction areas if the element's metric is constant and diagonal
    (reference geometry.py:200-209), else None."""
    if np.ptp(ja, axis=0).max() != 0.0:
        return None
    a0 = ja[0]
    if np.count_nonzero(a0 - np.diag(np.diag(a0))):
        return None
    return np.diag(a0).tolist()


def volume_fluxdiff(u_elem, dop, metrics, vol_flux, gas, pre=None):
    """One element's VOL with the scalar path's arithmetic
    (discretization.py:267-323). ``pre`` selects the precompute variant like
    the reference's PrecomputedElementData (its ``mode`` is used; the tables
    themselves are recomputed on the device). The device image of the
    one-element mesh is cached per (dop, gas, Cartesian areas), so a loop over
    a mesh's elements builds it once."""
    _fluxes.require_volume_kind(vol_flux)
    u_elem = np.asarray(u_elem, dtype=np.float64)
    d = u_elem.shape[-1] - 2
    mode = "none" if pre is None else getattr(pre, "mode", pre)
    ja = np.asarray(metrics.ja, dtype=np.float64)
    jac = np.asarray(metrics.jac, dtype=np.float64)
    areas = _axis_aligned_areas(ja)
    cart = None
    if areas is not None and np.ptp(jac) == 0.0:
        cart = (tuple(areas), float(jac[0]))
    es = _element_setup(dop, gas, d, cart)
    if cart is None:
        import torch

        dm = device_mesh_for(es)
        dm.ja.copy_(torch.from_numpy(np.ascontiguousarray(ja)).view(dm.ja.shape), non_blocking=False)
        dm.jac.copy_(torch.from_numpy(np.ascontiguousarray(jac)).view(dm.jac.shape), non_blocking=False)
    cfg = RhsConfig(volume_flux=vol_flux, precompute=mode, kernel="reference")
    return mesh_fluxdiff_volume(u_elem[None], es, cfg)[0]


# ------------------------------------------------------------- diagnostics


def _diag(setup, kind, u, b=None, gate=False):
    """One fdg_diagnostic reduction on the device; numpy / CPU inputs are
    copied in. ``gate``: the reference's entropy_vars / max_signal_speed raise
    on an inadmissible node (euler.py:26-41), so run the device gate first."""
    dm = device_mesh_for(setup)
    io = _Io(dm, u)
    iob = None if b is None else _Io(dm, b, key="in2")
    if gate:
        dm.reset_status()
        dm.gate(io.u)
    res = dm.diagnostic(kind, io.u, None if iob is None else iob.u)
    if gate:
        first_bad, _ = dm.read_status()
        if first_bad >= 0:
            dm.raise_if_inadmissible(io.u, first_bad, setup.gas.gamma)
    return res.cpu().numpy()


def entropy_rate(u, dudt, setup):
    """Normalized semidiscrete entropy production (discretization.py:1011-1024):
    (sum wbar J w.dudt, that / sum |wbar J w dudt|), both sums on the device."""
    from .device import DIAG_ENTROPY

    total, scale = (float(x) for x in _diag(setup, DIAG_ENTROPY, u, dudt, gate=True))
    if scale == 0.0:
        return 0.0, 0.0
    return total, total / scale


def conserved_totals(u, setup):
    """sum wbar J u per variable (discretization.py:1027-1031), on the device."""
    from .device import DIAG_CONSERVED

    return _diag(setup, DIAG_CONSERVED, u)


def error_norm_l2(u, u_exact, setup):
    """sqrt(sum wbar J (u - u_exact)^2) per variable (discretization.py:1033-1037);
    the sums on the device."""
    from .device import DIAG_ERROR_SQ

    return np.sqrt(_diag(setup, DIAG_ERROR_SQ, u, u_exact))
