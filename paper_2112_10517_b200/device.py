"""Device image of a SpatialSetup and the stream-ordered calls into libfdg.so.

PyTorch is used only to own device memory and streams; all arithmetic runs in
the sm_100a kernels behind include/fdg.h. A DeviceMesh accepts either this
package's SpatialSetup or the reference's (duck-typed: d, op.weights,
op.degree, dsplit.matrix, metrics.{cartesian, ja, jac}, plus_neighbor, gas).
"""

import ctypes
import os
import weakref

import numpy as np

from . import _native as N
from .errors import AdmissibilityError, ConfigurationError, DivergenceError, UnsupportedOperatorError


def _torch():
    import torch

    if not torch.cuda.is_available():
        from .errors import NativeLibraryError

        raise NativeLibraryError("no CUDA device: the flux-differencing path runs on the GPU only")
    return torch


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream_handle(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def scheme_struct(volume_flux, surface_flux, precompute, kernel):
    try:
        return N.Scheme(
            N.FLUX_IDS[volume_flux] if volume_flux is not None else 1,
            N.FLUX_IDS[surface_flux] if surface_flux is not None else 5,
            N.PRECOMPUTE_IDS[precompute],
            N.MODE_IDS[kernel],
        )
    except KeyError as err:
        raise ConfigurationError("unknown scheme option %s" % err) from err


def _metric_scalars(metrics, d):
    """(areas, J) of a Cartesian mesh from either metrics flavour."""
    areas = getattr(metrics, "areas", None)
    jac_const = getattr(metrics, "jac_const", None)
    if areas is None or jac_const is None:
        ja0 = np.asarray(metrics.ja[0, 0])
        areas = tuple(float(ja0[n, n]) for n in range(d))
        jac_const = float(metrics.jac[0, 0])
    return tuple(areas), float(jac_const)


# enum fdg_diag (include/fdg.h)
DIAG_CONSERVED, DIAG_ENTROPY, DIAG_ERROR_SQ, DIAG_DT = 0, 1, 2, 3


class DeviceMesh:
    """Uploaded tables + the libfdg mesh handle for one (partition of a) mesh.

    ``partition`` (optional) describes a slab of a larger mesh: a dict with
    ``lo``/``hi`` (global element range), ``plus``/``minus`` (d, n_local) int
    neighbour tables where negative entries are ghost slots, and
    ``ghost_nrm`` (n_ghost, fn, d) face normals for curved meshes
    (see parallel.py).
    """

    def __init__(self, setup, device=None, partition=None):
        torch = _torch()
        self.torch = torch
        self.device = torch.device(device if device is not None else "cuda")
        self.d = int(setup.d)
        op = setup.op
        self.degree = int(op.degree)
        self.p1 = self.degree + 1
        self.nn = self.p1**self.d
        self.nvar = self.d + 2
        self.fn = self.p1 ** (self.d - 1)
        if not N.lib().fdg_supported(self.d, self.degree):
            raise UnsupportedOperatorError(
                "degree %d in %dD is outside the device kernels' range (p = 1..7)" % (self.degree, self.d)
            )
        gas = setup.gas
        self.gamma = float(gas.gamma)
        metrics = setup.metrics
        self.cartesian = bool(metrics.cartesian)
        dsplit = np.ascontiguousarray(np.asarray(setup.dsplit.matrix, dtype=np.float64))
        weights = np.ascontiguousarray(np.asarray(op.weights, dtype=np.float64))
        self._host_keep = (dsplit, weights)
        if partition is None:
            plus = np.stack([np.asarray(setup.plus_neighbor[n], dtype=np.int64) for n in range(self.d)])
            n_elem = plus.shape[1]
            minus = np.empty_like(plus)
            for n in range(self.d):
                minus[n, plus[n]] = np.arange(n_elem)
            lo, hi = 0, n_elem
            ghost_nrm = None
        else:
            plus = np.asarray(partition["plus"], dtype=np.int64)
            minus = np.asarray(partition["minus"], dtype=np.int64)
            lo, hi = int(partition["lo"]), int(partition["hi"])
            n_elem = hi - lo
            ghost_nrm = partition.get("ghost_nrm")
        self.n_elem, self.elem_lo = n_elem, lo
        dev = self.device
        self.plus = torch.as_tensor(plus.astype(np.int32), device=dev).contiguous()
        self.minus = torch.as_tensor(minus.astype(np.int32), device=dev).contiguous()
        self.ja = self.jac = self.ghost_nrm = None
        areas, jac_const = (0.0, 0.0, 0.0), 0.0
        if self.cartesian:
            areas, jac_const = _metric_scalars(metrics, self.d)
            areas = tuple(areas) + (0.0,) * (3 - len(areas))
        else:
            if isinstance(metrics.ja, torch.Tensor):  # device-built geometry (build_setup(device=...))
                self.ja = metrics.ja[lo:hi].to(dev).contiguous()
                self.jac = metrics.jac[lo:hi].to(dev).contiguous()
            else:
                self.ja = torch.as_tensor(np.ascontiguousarray(np.asarray(metrics.ja)[lo:hi]), device=dev)
                self.jac = torch.as_tensor(np.ascontiguousarray(np.asarray(metrics.jac)[lo:hi]), device=dev)
            if ghost_nrm is not None:
                self.ghost_nrm = torch.as_tensor(np.ascontiguousarray(ghost_nrm, dtype=np.float64), device=dev)
        desc = N.MeshDesc()
        desc.d, desc.degree, desc.n_elem, desc.elem_base = self.d, self.degree, n_elem, lo
        desc.gamma, desc.inv_gamma_minus_one = float(gas.gamma), float(gas.inv_gamma_minus_one)
        desc.dsplit, desc.weights = dsplit.ctypes.data, weights.ctypes.data
        desc.cartesian = int(self.cartesian)
        desc.areas = (ctypes.c_double * 3)(*areas)
        desc.jac_const = jac_const
        desc.ja = None if self.ja is None else self.ja.data_ptr()
        desc.jac = None if self.jac is None else self.jac.data_ptr()
        desc.plus, desc.minus = self.plus.data_ptr(), self.minus.data_ptr()
        desc.ghost_nrm = None if self.ghost_nrm is None else self.ghost_nrm.data_ptr()
        handle = ctypes.c_void_p()
        N.check(N.lib().fdg_mesh_create(ctypes.byref(desc), ctypes.byref(handle)))
        self.handle = handle
        self._finalizer = weakref.finalize(self, N.lib().fdg_mesh_destroy, handle)
        self.areas, self.jac_const = areas[: self.d], jac_const
        self._staging = {}
        self.row_order = None
        self._set_traversal(setup)

    def _set_traversal(self, setup):
        """Opt-in tile-by-tile traversal (fdg_mesh_set_traversal), env
        FDG_TILE="tx,ty": rows of dims[2] elements visited in tiles of
        tx x ty rows so the +-x / +-y interface neighbours are staged by the
        same wave (FDG_TILE=0: natural order)."""
        mesh = getattr(setup, "mesh", None)
        dims = tuple(getattr(mesh, "dims", ()))
        env = os.environ.get("FDG_TILE")
        if self.d != 3 or len(dims) != 3 or env in ("", "0"):
            return
        _, n1, n2 = dims
        n0 = self.n_elem // (n1 * n2)  # planes held here (slab partitions split direction 0)
        if env is None:
            # default: 8 x 8 rows per tile when the state is much larger than
            # L2 (the +-x neighbours' traces then come from L2 instead of
            # DRAM: cfg5 RHS 6.35 -> 6.25 ms, profiles/r02_tuning.md);
            # L2-sized meshes keep the natural order (cfg4 48^3: 1% slower tiled)
            state_bytes = self.n_elem * self.nn * self.nvar * 8
            if state_bytes <= 8 * 126 * 2**20 or n0 % 8 or n1 % 8:
                return
            tx, ty = 8, 8
        else:
            tx, ty = (int(v) for v in env.split(","))
        if n0 * n1 * n2 != self.n_elem or n0 % tx or n1 % ty:
            return
        r = np.arange(n0 * n1).reshape(n0 // tx, tx, n1 // ty, ty).transpose(0, 2, 1, 3).ravel()
        self.row_order = self.torch.as_tensor(r.astype(np.int32), device=self.device)
        N.check(N.lib().fdg_mesh_set_traversal(self.handle, _ptr(self.row_order), n2))

    def reserve_sms(self, n):
        """Leave ``n`` SMs' worth of CTA slots free in interface launches
        (fdg_mesh_set_reserve_sms): room for the halo kernels to run
        concurrently with the interior elements."""
        N.check(N.lib().fdg_mesh_set_reserve_sms(self.handle, int(n)))

    # ------------------------------------------------------------ shapes
    @property
    def shape(self):
        return (self.n_elem, self.nn, self.nvar)

    def empty(self):
        return self.torch.empty(self.shape, dtype=self.torch.float64, device=self.device)

    def staging(self, key, shape):
        """Pinned host buffer reused across calls (no allocation on the hot path)."""
        buf = self._staging.get(key)
        if buf is None or tuple(buf.shape) != tuple(shape):
            buf = N.pinned_empty(shape)  # cudaHostAlloc: full-rate copies (profiles/r01_e2e.md)
            self._staging[key] = buf
        return buf

    # ------------------------------------------------------------- calls
    def volume(self, u, scheme, out=None, stream=None):
        out = self.empty() if out is None else out
        N.check(N.lib().fdg_volume(self.handle, ctypes.byref(scheme), _ptr(u), _ptr(out), _stream_handle(stream)))
        return out

    def volume_range(self, u, scheme, out, lo, hi, stream=None):
        """VOL of local elements [lo, hi) only; u and out are the whole arrays."""
        N.check(
            N.lib().fdg_volume_range(
                self.handle, ctypes.byref(scheme), _ptr(u), _ptr(out), int(lo), int(hi), _stream_handle(stream)
            )
        )
        return out

    def volume_host(self, u_host, scheme, out_host, n_chunks=0, stream=None):
        """VOL of a pinned host state into a pinned host buffer through
        fdg_volume_host: the H2D copy of chunk c+1, the kernel on chunk c and
        the D2H copy of chunk c-1 overlap. Ordered on ``stream`` (default: the
        current one), which resumes after the last copy-out, so events
        recorded around this call bracket the whole transfer. Returns the
        device copy of the state (for error reports) and ``out_host``."""
        torch = self.torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        u_dev = self._scratch("u_dev")
        v_dev = self._scratch("v_dev")
        last = self._staging.get("_scratch_done")
        if last is not None:
            s.wait_event(last)  # scratch reuse after a call on another stream
        N.check(
            N.lib().fdg_volume_host(
                self.handle, ctypes.byref(scheme), _ptr(u_host), _ptr(out_host), _ptr(u_dev), _ptr(v_dev),
                int(n_chunks), ctypes.c_void_p(s.cuda_stream),
            )
        )
        if last is None:
            last = self._staging["_scratch_done"] = torch.cuda.Event()
        last.record(s)
        return u_dev, out_host

    def _scratch(self, key):
        """Device buffer of the state's size, reused across calls."""
        buf = self._staging.get(key)
        if buf is None:
            buf = self.empty()
            self._staging[key] = buf
        return buf

    def surface(self, u, scheme, out, ghost_u=None, stream=None):
        N.check(
            N.lib().fdg_surface(
                self.handle, ctypes.byref(scheme), _ptr(u), _ptr(ghost_u), _ptr(out), _stream_handle(stream)
            )
        )
        return out

    def _ranges(self, lo, hi, ranges):
        """(lo, hi, lo2, hi2) of a range launch, or None for the whole mesh."""
        if ranges is not None:
            rs = list(ranges)
            if not 1 <= len(rs) <= 2:
                raise ValueError("one or two element ranges, got %d" % len(rs))
            (a, b), (c, d) = rs[0], (rs[1] if len(rs) == 2 else (0, 0))
            return int(a), int(b), int(c), int(d)
        if lo is None and hi is None:
            return None
        return int(0 if lo is None else lo), int(self.n_elem if hi is None else hi), 0, 0

    def rhs(self, u, scheme, out=None, ghost_u=None, stream=None, lo=None, hi=None, ranges=None):
        """du = -(VOL + SURF); with ``lo``/``hi`` (or up to two ``ranges``)
        only those local elements (fdg_rhs_range: the overlap split)."""
        out = self.empty() if out is None else out
        r = self._ranges(lo, hi, ranges)
        if r is None:
            N.check(N.lib().fdg_rhs(self.handle, ctypes.byref(scheme), _ptr(u), _ptr(ghost_u), _ptr(out),
                                    _stream_handle(stream)))
        else:
            N.check(N.lib().fdg_rhs_range(self.handle, ctypes.byref(scheme), _ptr(u), _ptr(ghost_u), _ptr(out), *r,
                                          _stream_handle(stream)))
        return out

    def stage(self, scheme, stage, v_in, v_out, reg=None, u0=None, ghost_u=None, stream=None, lo=None, hi=None,
              ranges=None):
        args = (self.handle, ctypes.byref(scheme), ctypes.byref(stage), _ptr(v_in), _ptr(ghost_u), _ptr(v_out),
                _ptr(reg), _ptr(u0))
        r = self._ranges(lo, hi, ranges)
        if r is None:
            N.check(N.lib().fdg_rk_stage(*args, _stream_handle(stream)))
        else:
            N.check(N.lib().fdg_rk_stage_range(*args, *r, _stream_handle(stream)))
        return v_out

    def gate(self, u, stream=None):
        N.check(N.lib().fdg_gate(self.handle, _ptr(u), _stream_handle(stream)))

    def reset_status(self, stream=None):
        N.check(N.lib().fdg_reset_status(self.handle, _stream_handle(stream)))

    def read_status(self, stream=None):
        rec = N.StatusRec()
        N.check(N.lib().fdg_read_status(self.handle, ctypes.byref(rec), _stream_handle(stream)))
        return int(rec.first_bad), int(rec.bad_stage)

    def diagnostic(self, kind, a, b=None, out=None, stream=None):
        """fdg_diagnostic: the rank-local reduction `kind` (DIAG_*) of device
        state(s) into a small device tensor (see include/fdg.h)."""
        n_out = {DIAG_CONSERVED: self.nvar, DIAG_ENTROPY: 2, DIAG_ERROR_SQ: self.nvar, DIAG_DT: 1}[kind]
        if out is None:
            out = self.torch.empty(n_out, dtype=self.torch.float64, device=self.device)
        N.check(
            N.lib().fdg_diagnostic(
                self.handle, int(kind), _ptr(a), None if b is None else _ptr(b), _ptr(out), _stream_handle(stream)
            )
        )
        return out

    def pack_faces(self, u, elems, direction, side, out, stream=None):
        N.check(
            N.lib().fdg_pack_faces(
                _ptr(u), _ptr(elems), int(elems.numel()), self.d, self.degree, direction, side, _ptr(out),
                _stream_handle(stream),
            )
        )
        return out

    # ------------------------------------------------------------ errors
    def raise_if_inadmissible(self, u, first_bad, gamma):
        """AdmissibilityError with the reference gate's message
        (discretization.py:668-671); indices are global element ids."""
        if first_bad < 0:
            return
        e, i = divmod(first_bad, self.nn)
        row = u[e - self.elem_lo, i].double().cpu().numpy() if hasattr(u, "cpu") else np.asarray(u[e - self.elem_lo, i])
        rho = row[0]
        mom = row[1 : self.d + 1]
        p = (gamma - 1.0) * (row[self.d + 1] - 0.5 * np.sum(mom * mom, axis=-1) / rho)
        raise AdmissibilityError(
            "inadmissible state at element %d, node %d: rho=%r, p=%r" % (int(e), int(i), float(rho), float(p))
        )


class GaussDeviceMesh:
    """Device image of a Gauss-family setup for one scheme (its scatter
    tables, operators.gauss_scatter_tables) and the libfdg gauss handle
    (fdg_gauss_*): metric terms at the Gauss nodes, neighbour tables, and the
    library-owned projection scratch. Duck-typed setup: d, op.{weights, D,
    boundary_interp, degree}, metrics.{ja, jac}, plus_neighbor, gas."""

    def __init__(self, setup, scheme, device=None):
        from .operators import gauss_scatter_tables

        torch = _torch()
        self.torch = torch
        self.device = torch.device(device if device is not None else "cuda")
        self.d = int(setup.d)
        op = setup.op
        self.degree = int(op.degree)
        self.p1 = self.degree + 1
        self.nn = self.p1**self.d
        self.nvar = self.d + 2
        self.fn = self.p1 ** (self.d - 1)
        self.gamma = float(setup.gas.gamma)
        plus = np.stack([np.asarray(setup.plus_neighbor[n], dtype=np.int64) for n in range(self.d)])
        self.n_elem = n_elem = plus.shape[1]
        self.elem_lo = 0
        minus = np.empty_like(plus)
        for n in range(self.d):
            minus[n, plus[n]] = np.arange(n_elem)
        dev = self.device
        self.plus = torch.as_tensor(plus.astype(np.int32), device=dev).contiguous()
        self.minus = torch.as_tensor(minus.astype(np.int32), device=dev).contiguous()
        ja, jac = setup.metrics.ja, setup.metrics.jac
        if isinstance(ja, torch.Tensor):
            self.ja, self.jac = ja.to(dev).contiguous(), jac.to(dev).contiguous()
        else:
            self.ja = torch.as_tensor(np.ascontiguousarray(np.asarray(ja, dtype=np.float64)), device=dev)
            self.jac = torch.as_tensor(np.ascontiguousarray(np.asarray(jac, dtype=np.float64)), device=dev)
        tabs = [np.ascontiguousarray(t, dtype=np.float64) for t in gauss_scatter_tables(op, scheme)]
        R = np.ascontiguousarray(np.asarray(op.boundary_interp, dtype=np.float64))
        self._host_keep = (tabs, R)
        desc = N.GaussDesc()
        desc.d, desc.degree, desc.n_elem = self.d, self.degree, n_elem
        desc.gamma, desc.inv_gamma_minus_one = float(setup.gas.gamma), float(setup.gas.inv_gamma_minus_one)
        desc.boundary_interp = R.ctypes.data
        desc.vv, desc.cvol, desc.cface, desc.lift = (t.ctypes.data for t in tabs)
        desc.ja, desc.jac = self.ja.data_ptr(), self.jac.data_ptr()
        desc.plus, desc.minus = self.plus.data_ptr(), self.minus.data_ptr()
        handle = ctypes.c_void_p()
        N.check(N.lib().fdg_gauss_create(ctypes.byref(desc), ctypes.byref(handle)))
        self.handle = handle
        self._finalizer = weakref.finalize(self, N.lib().fdg_gauss_destroy, handle)
        self._staging = {}

    @property
    def shape(self):
        return (self.n_elem, self.nn, self.nvar)

    def empty(self):
        return self.torch.empty(self.shape, dtype=self.torch.float64, device=self.device)

    def staging(self, key, shape):
        buf = self._staging.get(key)
        if buf is None or tuple(buf.shape) != tuple(shape):
            buf = N.pinned_empty(shape)
            self._staging[key] = buf
        return buf

    def proj_shape(self):
        return (self.n_elem, self.d, 2, self.fn, self.nvar)

    def nrm_shape(self):
        return (self.n_elem, self.d, 2, self.fn, self.d)

    def project(self, u, proj=None, nrm=None, stream=None):
        torch = self.torch
        proj = proj if proj is not None else torch.empty(self.proj_shape(), dtype=torch.float64, device=self.device)
        nrm = nrm if nrm is not None else torch.empty(self.nrm_shape(), dtype=torch.float64, device=self.device)
        N.check(N.lib().fdg_gauss_project(self.handle, _ptr(u), _ptr(proj), _ptr(nrm), _stream_handle(stream)))
        return proj, nrm

    def rhs(self, u, scheme, out=None, proj=None, nrm=None, fnrm=None, stream=None):
        out = self.empty() if out is None else out
        N.check(N.lib().fdg_gauss_rhs(self.handle, ctypes.byref(scheme), _ptr(u), _ptr(proj), _ptr(nrm), _ptr(fnrm),
                                      _ptr(out), _stream_handle(stream)))
        return out

    def gate(self, u, stream=None):
        N.check(N.lib().fdg_gauss_gate(self.handle, _ptr(u), _stream_handle(stream)))

    def reset_status(self, stream=None):
        N.check(N.lib().fdg_gauss_reset_status(self.handle, _stream_handle(stream)))

    def read_status(self, stream=None):
        rec = N.StatusRec()
        N.check(N.lib().fdg_gauss_read_status(self.handle, ctypes.byref(rec), _stream_handle(stream)))
        return int(rec.first_bad), int(rec.bad_stage)

    raise_if_inadmissible = DeviceMesh.raise_if_inadmissible


_GAUSS_CACHE = {}


def gauss_mesh_for(setup, scheme, device=None):
    """GaussDeviceMesh cached per (setup object, scheme); dropped with the setup."""
    key = (id(setup), scheme, str(device))
    hit = _GAUSS_CACHE.get(key)
    if hit is not None and hit[0]() is setup:
        return hit[1]
    gm = GaussDeviceMesh(setup, scheme, device=device)
    try:
        ref = weakref.ref(setup)
        weakref.finalize(setup, lambda k=key, r=ref: _GAUSS_CACHE.pop(k, None) if _GAUSS_CACHE.get(k, (None,))[0] is r
                         else None)
    except TypeError:
        ref = (lambda s: (lambda: s))(setup)
    _GAUSS_CACHE[key] = (ref, gm)
    return gm


_CACHE = {}


def device_mesh_for(setup, device=None):
    """DeviceMesh cached per setup object. The entry is dropped as soon as the
    setup is garbage collected (weakref.finalize), which releases the device
    tables and the libfdg handle with it; objects without weakref support
    keep their entry (and themselves) alive until ``clear_cache()``."""
    key = (id(setup), str(device))
    hit = _CACHE.get(key)
    if hit is not None and hit[0]() is setup:
        return hit[1]
    dm = DeviceMesh(setup, device=device)
    try:
        ref = weakref.ref(setup)
        weakref.finalize(setup, _evict, key, ref)
    except TypeError:  # objects without weakref support: keep them alive with the cache entry
        ref = (lambda s: (lambda: s))(setup)
    _CACHE[key] = (ref, dm)
    return dm


def _evict(key, ref):
    hit = _CACHE.get(key)
    if hit is not None and hit[0] is ref:
        del _CACHE[key]


def clear_cache():
    """Drop every cached DeviceMesh (their device memory is freed once unreferenced)."""
    _CACHE.clear()
    _GAUSS_CACHE.clear()


__all__ = ["DeviceMesh", "GaussDeviceMesh", "device_mesh_for", "gauss_mesh_for", "scheme_struct", "DivergenceError"]
