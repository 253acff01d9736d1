"""Structured periodic box meshes, nodal coordinates and metric terms.

Host-side setup (the device consumes the results once per mesh handle).
Conventions follow the reference (geometry.py:40-329): element index
C-ordered over dims, x = lo + L (e + (xi+1)/2)/N per direction, optional
warp a * prod_j sin(2 pi t_j) added to every coordinate, metric terms
ja[e, i, n, j] = (J a^n)_j by direct differentiation in 2D and the curl form
in 3D (discrete metric identity to roundoff), face normals taken from the
minus element's own +face nodes. The numpy call sequence is the reference's,
so curved metrics are bit-identical to it on the same BLAS
(tests/test_setup.py).

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


def _element_multi_index(mesh):
    grids = np.meshgrid(*[np.arange(n) for n in mesh.dims], indexing="ij")
    return np.stack([g.ravel() for g in grids], axis=-1)


def _fractions(mesh, nodes1d):
    half = 0.5 * (nodes1d + 1.0)
    return [(np.arange(n)[:, None] + half[None, :]) / n for n in mesh.dims]


def element_coords(mesh, op):
    """(n_elements, (p+1)^d, d) nodal coordinates."""
    d = mesh.d
    tfrac = _fractions(mesh, op.nodes)
    n1d = tfrac[0].shape[1]
    elem_idx = _element_multi_index(mesh)
    n_elem = elem_idx.shape[0]
    shape = (n1d,) * d
    nn = n1d**d
    coords = np.empty((n_elem, nn, d))
    tgrids = []
    for j in range(d):
        t_e = tfrac[j][elem_idx[:, j]]
        expand = [None] * d
        expand[j] = slice(None)
        tgrids.append(np.broadcast_to(t_e[(slice(None),) + tuple(expand)], (n_elem,) + shape))
    lengths = [b - a for a, b in zip(mesh.lo, mesh.hi)]
    for j in range(d):
        coords[:, :, j] = (mesh.lo[j] + lengths[j] * tgrids[j]).reshape(n_elem, nn)
    if mesh.amplitude != 0.0:
        bump = np.ones((n_elem,) + shape)
        for j in range(d):
            bump = bump * np.sin(2.0 * np.pi * tgrids[j])
        bump = mesh.amplitude * bump.reshape(n_elem, nn)
        for j in range(d):
            coords[:, :, j] += bump
    return coords


def apply_along(mat, arr, axis):
    moved = np.moveaxis(arr, axis, -1)
    return np.moveaxis(moved @ mat.T, -1, axis)


def _metrics_2d(x_nd, dmat):
    x1, x2 = x_nd[..., 0], x_nd[..., 1]
    d1x1 = apply_along(dmat, x1, 1)
    d1x2 = apply_along(dmat, x2, 1)
    d2x1 = apply_along(dmat, x1, 2)
    d2x2 = apply_along(dmat, x2, 2)
    ja = np.empty(x1.shape + (2, 2))
    ja[..., 0, 0] = d2x2
    ja[..., 0, 1] = -d2x1
    ja[..., 1, 0] = -d1x2
    ja[..., 1, 1] = d1x1
    return ja, d1x1 * d2x2 - d2x1 * d1x2


def _metrics_3d_curl(x_nd, dmat):
    x = [x_nd[..., m] for m in range(3)]
    dx = [[apply_along(dmat, x[m], i + 1) for m in range(3)] for i in range(3)]
    axes = tuple(range(1, x[0].ndim))
    x = [c - c.mean(axis=axes, keepdims=True) for c in x]  # shift-invariant curl; small products
    cyc = ((1, 2), (2, 0), (0, 1))
    ja = np.empty(x[0].shape + (3, 3))
    for n in range(3):
        l, m = cyc[n]
        for i in range(3):
            j, k = cyc[i]
            ja[..., i, n] = apply_along(dmat, x[l] * dx[k][m], j + 1) - apply_along(dmat, x[l] * dx[j][m], k + 1)
    jac = (
        dx[0][0] * (dx[1][1] * dx[2][2] - dx[1][2] * dx[2][1])
        - dx[0][1] * (dx[1][0] * dx[2][2] - dx[1][2] * dx[2][0])
        + dx[0][2] * (dx[1][0] * dx[2][1] - dx[1][1] * dx[2][0])
    )
    return ja, jac


class MetricData:
    """Discrete geometry of one mesh/operator pairing.

    cartesian: ``areas[n]`` = Ja^n_n and ``jac_const`` = J (uniform box);
    curved: ``ja`` (n_elem, nn, d, d) and ``jac`` (n_elem, nn).
    ``face_ja[n]`` (n_elem, fn, d) is the minus element's +face trace of its
    own Ja^n (for LGL a restriction: geometry.py:311-326 of the reference).
    """

    def __init__(self, d, p1, n_elem, cartesian, areas=None, jac_const=None, ja=None, jac=None):
        self.d, self.p1, self.n_elem = d, p1, n_elem
        self.cartesian = bool(cartesian)
        self.areas = None if areas is None else tuple(float(a) for a in areas)
        self.jac_const = None if jac_const is None else float(jac_const)
        self._ja, self._jac = ja, jac
        self._face_ja = None

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
    def face_ja(self):
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
    """plus_neighbor[n][e]: element across the +n face of e (periodic)."""
    idx = np.arange(mesh.n_elements).reshape(mesh.dims)
    return tuple(np.roll(idx, -1, axis=n).ravel().copy() for n in range(mesh.d))
