"""Structured periodic box meshes, nodal coordinates and metric terms.

Host-side setup (the device consumes the results once per mesh handle; for
large meshes ``device_geometry`` computes the same arrays on the GPU).
Conventions of the reference (geometry.py:40-329): element index C-ordered
over dims, x = lo + L (e + (xi+1)/2)/N per direction, optional warp
a * prod_j sin(2 pi t_j) added to every coordinate, metric terms
ja[e, i, n, j] = (J a^n)_j by direct differentiation in 2D and the curl form
in 3D (discrete metric identity to roundoff), face normals taken from the
minus element's own +face nodes. Coordinates use the reference's mapping
arithmetic (bitwise equal for equal nodes); the metric derivatives are
tensor contractions here, equal to the reference's to roundoff
(tests/test_setup.py: <= 1e-13 relative).

Difference by design: a Cartesian mesh stores its metrics as d areas and one
Jacobian (the reference materialises per-node arrays, 22 GB at 128^3 N=3);
``MetricData.ja``/``jac`` are materialised lazily on access for callers that
index them.
"""

from dataclasses import dataclass

import numpy as np

from .errors import MeshError


@dataclass(frozen=True)
class StructuredMesh:
    dims: tuple
    lo: tuple
    hi: tuple
    amplitude: float = 0.0

    def __post_init__(self):
        if len(self.dims) not in (2, 3):
            raise MeshError("supported dimensions are 2 and 3, got %r" % (self.dims,))
        if any(n < 1 for n in self.dims):
            raise MeshError("every direction needs at least one element: %r" % (self.dims,))
        if any(b <= a for a, b in zip(self.lo, self.hi)):
            raise MeshError("empty box: lo=%r hi=%r" % (self.lo, self.hi))

    @property
    def d(self):
        return len(self.dims)

    @property
    def n_elements(self):
        n = 1
        for k in self.dims:
            n *= k
        return n

    @property
    def widths(self):
        return tuple((b - a) / n for a, b, n in zip(self.lo, self.hi, self.dims))

    @property
    def is_cartesian(self):
        return self.amplitude == 0.0


def build_mesh(dims, bounds=(-5.0, 5.0), amplitude=0.0):
    """`bounds` is one (lo, hi) pair for every direction or one pair per direction."""
    dims = tuple(int(n) for n in dims)
    if np.ndim(bounds) == 1:
        bounds = [bounds] * len(dims)
    lo = tuple(float(b[0]) for b in bounds)
    hi = tuple(float(b[1]) for b in bounds)
    return StructuredMesh(dims, lo, hi, float(amplitude))


def _axis_coords(mesh, nodes1d):
    """Per direction j: (x_j, t_j) on the (dims[j], p+1) grid of element
    index x node position, t = (e + (xi+1)/2) / n_j the fraction of the box
    and x = lo_j + L_j t (the mapping of the reference's structured mesh,
    geometry.py:94-136)."""
    half = 0.5 * (np.asarray(nodes1d, dtype=np.float64) + 1.0)
    out = []
    for j, n in enumerate(mesh.dims):
        t = (np.arange(n)[:, None] + half[None, :]) / n
        out.append((mesh.lo[j] + (mesh.hi[j] - mesh.lo[j]) * t, t))
    return out


def _tensor_grid(per_axis, d, j):
    """Broadcast direction j's (n_j, p1) table onto the element/node grid
    (n_0..n_{d-1}, p1, .., p1): axis j is element index, axis d+j node index."""
    shape = [1] * (2 * d)
    shape[j] = per_axis.shape[0]
    shape[d + j] = per_axis.shape[1]
    return per_axis.reshape(shape)


def element_coords(mesh, op):
    """(n_elements, (p+1)^d, d) nodal coordinates: elements C-ordered over
    dims, nodes C-ordered over the reference axes. A warped mesh adds
    a * prod_j sin(2 pi t_j) to every coordinate."""
    d = mesh.d
    p1 = len(op.nodes)
    axes = _axis_coords(mesh, op.nodes)
    full = tuple(mesh.dims) + (p1,) * d
    n_elem, nn = mesh.n_elements, p1**d
    coords = np.empty(full + (d,))
    for j in range(d):
        coords[..., j] = _tensor_grid(axes[j][0], d, j)
    if mesh.amplitude != 0.0:
        bump = _tensor_grid(np.sin(2.0 * np.pi * axes[0][1]), d, 0)
        for j in range(1, d):
            bump = bump * _tensor_grid(np.sin(2.0 * np.pi * axes[j][1]), d, j)
        coords += (mesh.amplitude * bump)[..., None]
    # (e_0..e_{d-1}, a_0..a_{d-1}) is already (element, node) C-order
    return coords.reshape(n_elem, nn, d)


def _ref_derivative(dmat, f, axis):
    """d f / d xi_axis of nodal values f (n_elem, p1, .., p1): the 1D
    differentiation matrix contracted with node axis ``axis`` (0-based over
    the reference directions)."""
    return np.moveaxis(np.tensordot(f, dmat, axes=([axis + 1], [1])), -1, axis + 1)


def _metrics_2d(x_nd, dmat):
    """Ja^n_j by differentiating the mapping: Ja^0 = (y_eta, -x_eta),
    Ja^1 = (-y_xi, x_xi), J = x_xi y_eta - x_eta y_xi."""
    g = [[_ref_derivative(dmat, x_nd[..., m], i) for m in range(2)] for i in range(2)]  # g[i][m] = dx_m/dxi_i
    ja = np.stack(
        [np.stack([g[1][1], -g[1][0]], axis=-1), np.stack([-g[0][1], g[0][0]], axis=-1)], axis=-2
    )
    return ja, g[0][0] * g[1][1] - g[1][0] * g[0][1]


def _metrics_3d_curl(x_nd, dmat):
    """Conservative curl form of the 3D metric terms (Kopriva 2006):
    Ja^i_n = d_j (x_l d_k x_m) - d_k (x_l d_j x_m) with (j, k) the two
    reference directions after i and (l, m) the two physical components
    after n, cyclically. The discrete derivatives commute, so the discrete
    metric identity sum_i d_i Ja^i = 0 holds to roundoff. Coordinates are
    re-centred per element first (the form is invariant under a shift of
    x_l; small products lose less to cancellation)."""
    g = [[_ref_derivative(dmat, x_nd[..., m], i) for m in range(3)] for i in range(3)]  # dx_m/dxi_i
    xc = [x_nd[..., m] - x_nd[..., m].mean(axis=(1, 2, 3), keepdims=True) for m in range(3)]
    nxt = lambda q: ((q + 1) % 3, (q + 2) % 3)  # noqa: E731
    ja = np.empty(x_nd.shape[:-1] + (3, 3))
    for i in range(3):
        j, k = nxt(i)
        for n in range(3):
            l, m = nxt(n)
            ja[..., i, n] = _ref_derivative(dmat, xc[l] * g[k][m], j) - _ref_derivative(dmat, xc[l] * g[j][m], k)
    rows = [np.stack(g[i], axis=-1) for i in range(3)]  # row i = d x / d xi_i
    c = np.cross(rows[1], rows[2])
    jac = rows[0][..., 0] * c[..., 0] + rows[0][..., 1] * c[..., 1] + rows[0][..., 2] * c[..., 2]  # triple product
    return ja, jac


class MetricData:
    """Discrete geometry of one mesh/operator pairing.

    cartesian: ``areas[n]`` = Ja^n_n and ``jac_const`` = J (uniform box);
    curved: ``ja`` (n_elem, nn, d, d) and ``jac`` (n_elem, nn).
    ``face_ja[n]`` (n_elem, fn, d) is the minus element's +face trace of its
    own Ja^n (for LGL a restriction: geometry.py:311-326 of the reference).
    """

    def __init__(self, d, p1, n_elem, cartesian, areas=None, jac_const=None, ja=None, jac=None, boundary_interp=None):
        self.d, self.p1, self.n_elem = d, p1, n_elem
        self.cartesian = bool(cartesian)
        self.areas = None if areas is None else tuple(float(a) for a in areas)
        self.jac_const = None if jac_const is None else float(jac_const)
        self._ja, self._jac = ja, jac
        self._face_ja = None
        self._elem_face_ja = None
        # Gauss nodes have no boundary node: face traces are extrapolations
        # with the boundary rows R (reference geometry.py:253-262, 311-326)
        self.boundary_interp = None if boundary_interp is None else np.asarray(boundary_interp, dtype=np.float64)

    @property
    def nn(self):
        return self.p1**self.d

    @property
    def ja(self):
        if self._ja is None:
            ja = np.zeros((self.n_elem, self.nn, self.d, self.d))
            for n in range(self.d):
                ja[:, :, n, n] = self.areas[n]
            self._ja = ja
        return self._ja

    @property
    def jac(self):
        if self._jac is None:
            self._jac = np.full((self.n_elem, self.nn), self.jac_const)
        return self._jac

    @property
    def elem_face_ja(self):
        """elem_face_ja[n][e, s, m, :]: element e's own trace of its Ja^n on
        side s (0: the -1 face, 1: the +1 face) at face node m."""
        if self._elem_face_ja is None:
            from .operators import node_lines

            lines = node_lines(self.p1, self.d)
            ja = np.asarray(self.ja)
            out = []
            for n in range(self.d):
                vals = ja[:, lines[n], n, :]  # (n_elem, fn, p1, d)
                if self.boundary_interp is None:
                    sides = [vals[:, :, 0, :], vals[:, :, -1, :]]
                else:
                    sides = [np.einsum("efkj,k->efj", vals, self.boundary_interp[s]) for s in (0, 1)]
                out.append(np.ascontiguousarray(np.stack(sides, axis=1)))
            self._elem_face_ja = tuple(out)
        return self._elem_face_ja

    @property
    def face_ja(self):
        if self._face_ja is None and self.boundary_interp is not None:
            self._face_ja = tuple(np.ascontiguousarray(t[:, 1]) for t in self.elem_face_ja)
        if self._face_ja is None:
            from .operators import node_lines

            lines = node_lines(self.p1, self.d)
            self._face_ja = tuple(
                np.ascontiguousarray(self.ja[:, lines[n][:, -1], n, :]) for n in range(self.d)
            )
        return self._face_ja


def compute_metrics(mesh, op, coords=None):
    d = mesh.d
    p1 = op.n_nodes
    n_elem = mesh.n_elements
    if mesh.is_cartesian:
        h = mesh.widths
        jac_val = 1.0
        for w in h:
            jac_val *= 0.5 * w
        areas = [jac_val / (0.5 * h[n]) for n in range(d)]
        return MetricData(d, p1, n_elem, True, areas=areas, jac_const=jac_val)
    if coords is None:
        coords = element_coords(mesh, op)
    x_nd = coords.reshape((n_elem,) + (p1,) * d + (d,))
    ja_nd, jac_nd = (_metrics_2d if d == 2 else _metrics_3d_curl)(x_nd, op.D)
    ja = ja_nd.reshape(n_elem, p1**d, d, d)
    jac = jac_nd.reshape(n_elem, p1**d)
    if not np.all(jac > 0.0):
        e, i = np.unravel_index(np.argmin(jac), jac.shape)
        raise MeshError(
            "non-positive Jacobian %r at element %d, node %d (amplitude too large?)" % (float(jac[e, i]), int(e), int(i))
        )
    return MetricData(d, p1, n_elem, False, ja=ja, jac=jac)


def device_geometry(mesh, op, device="cuda", coords=True, metrics=True):
    """element_coords and compute_metrics's curved arrays computed on the GPU
    (fdg_build_geometry): returns (coords, ja, jac) as CUDA float64 tensors
    (None where not requested; ja/jac None for Cartesian meshes, whose
    metrics are scalars). Same arithmetic as the host path up to summation
    order and the device sin (tests/test_gpu_parity.py pins <= 1e-13)."""
    import ctypes

    import torch

    from . import _native as N

    d = mesh.d
    p1 = op.n_nodes
    nn = p1**d
    n_elem = mesh.n_elements
    dev = torch.device(device)
    want_metrics = metrics and not mesh.is_cartesian
    c = torch.empty((n_elem, nn, d), dtype=torch.float64, device=dev) if coords else None
    ja = torch.empty((n_elem, nn, d, d), dtype=torch.float64, device=dev) if want_metrics else None
    jac = torch.empty((n_elem, nn), dtype=torch.float64, device=dev) if want_metrics else None
    if c is None and ja is None:
        return None, None, None
    nodes = np.ascontiguousarray(op.nodes, dtype=np.float64)
    dmat = np.ascontiguousarray(op.D, dtype=np.float64)
    desc = N.GeometryDesc()
    desc.d, desc.degree = d, p1 - 1
    desc.dims = (ctypes.c_int32 * 3)(*(tuple(mesh.dims) + (1,) * (3 - d)))
    desc.lo = (ctypes.c_double * 3)(*(tuple(mesh.lo) + (0.0,) * (3 - d)))
    desc.hi = (ctypes.c_double * 3)(*(tuple(mesh.hi) + (0.0,) * (3 - d)))
    desc.amplitude = float(mesh.amplitude)
    desc.nodes, desc.dmat = nodes.ctypes.data, dmat.ctypes.data
    ptr = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())  # noqa: E731
    stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    N.check(N.lib().fdg_build_geometry(ctypes.byref(desc), ptr(c), ptr(ja), ptr(jac), stream))
    if jac is not None:
        jmin = float(jac.min())
        if not jmin > 0.0:
            flat = int(torch.argmin(jac))
            raise MeshError(
                "non-positive Jacobian %r at element %d, node %d (amplitude too large?)" % (jmin, flat // nn, flat % nn)
            )
    return c, ja, jac


def neighbor_table(mesh):
    """plus_neighbor[n][e]: the element across the +n face of e, periodic in
    every direction (element multi-index e_n -> (e_n + 1) mod dims[n])."""
    dims = tuple(mesh.dims)
    idx = np.indices(dims).reshape(len(dims), -1)
    out = []
    for n in range(len(dims)):
        shifted = idx.copy()
        shifted[n] = (shifted[n] + 1) % dims[n]
        out.append(np.ravel_multi_index(tuple(shifted), dims))
    return tuple(out)
