"""Legendre-Gauss-Lobatto SBP operators and the split-derivative matrix.

Host-side setup only: the device receives Dsplit and the LGL weights once per
mesh handle. The construction is the textbook one the reference uses
(operators.py:79-217): Lobatto nodes as the roots of P'_p by Newton's method
from Chebyshev-Lobatto guesses, weights 2/(p(p+1)P_p^2), the barycentric
differentiation matrix, and the SBP re-assembly
D = (skew(M D) + R^T B N R / 2) / w, so that M D + D^T M = R^T B N R holds to
a few ulps. The arithmetic sequence is kept identical so the tables are
bit-for-bit those of the reference (tests/test_setup.py pins them against
tests/golden/operators.npz).
"""

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .errors import UnsupportedOperatorError

MAX_DEGREE = 15
DEVICE_MAX_DEGREE = 7

_FACE_SIGNS = np.array([-1.0, 1.0])


@dataclass(frozen=True)
class Operator1D:
    degree: int
    family: str
    nodes: np.ndarray
    weights: np.ndarray
    D: np.ndarray
    boundary_interp: np.ndarray  # rows evaluate at -1 and +1

    @property
    def n_nodes(self):
        return self.degree + 1


@dataclass(frozen=True)
class FluxDiffOperator:
    """2D - M^{-1} R^T B N R (zero diagonal, M-antisymmetric)."""

    matrix: np.ndarray
    op: Operator1D


def _legendre(p, x):
    """P_p(x) and P_p'(x) by the three-term recurrence."""
    x = np.asarray(x, dtype=float)
    prev, cur = np.ones_like(x), x.copy()
    dprev, dcur = np.zeros_like(x), np.ones_like(x)
    if p == 0:
        return prev, dprev
    for n in range(1, p):
        nxt = ((2 * n + 1) * x * cur - n * prev) / (n + 1)
        dnxt = dprev + (2 * n + 1) * cur
        prev, cur = cur, nxt
        dprev, dcur = dcur, dnxt
    return cur, dcur


def _lobatto(p):
    if p == 1:
        return np.array([-1.0, 1.0]), np.array([1.0, 1.0])
    x = -np.cos(np.pi * np.arange(1, p) / p)
    for _ in range(100):
        leg, dleg = _legendre(p, x)
        ddleg = (2.0 * x * dleg - p * (p + 1) * leg) / (1.0 - x * x)
        step = dleg / ddleg
        x -= step
        if np.max(np.abs(step)) < 1.0e-15:
            break
    x = 0.5 * (x - x[::-1])
    nodes = np.concatenate(([-1.0], x, [1.0]))
    leg, _ = _legendre(p, nodes)
    return nodes, 2.0 / (p * (p + 1) * leg * leg)


def _barycentric(nodes):
    diff = nodes[:, None] - nodes[None, :]
    np.fill_diagonal(diff, 1.0)
    return 1.0 / np.prod(diff, axis=1)


def _differentiation(nodes):
    lam = _barycentric(nodes)
    diff = nodes[:, None] - nodes[None, :]
    np.fill_diagonal(diff, 1.0)
    mat = (lam[None, :] / lam[:, None]) / diff
    np.fill_diagonal(mat, 0.0)
    np.fill_diagonal(mat, -np.sum(mat, axis=1))
    return mat


def _interp_row(nodes, lam, y):
    diff = y - nodes
    hit = np.nonzero(diff == 0.0)[0]
    row = np.zeros_like(nodes)
    if hit.size:
        row[hit[0]] = 1.0
        return row
    c = lam / diff
    return c / np.sum(c)


def _check_degree(p):
    if not (1 <= p <= MAX_DEGREE):
        raise UnsupportedOperatorError("degree %r outside supported range 1..%d" % (p, MAX_DEGREE))


@lru_cache(maxsize=None)
def lgl_operator(p):
    _check_degree(p)
    nodes, weights = _lobatto(p)
    mat = _differentiation(nodes)
    lam = _barycentric(nodes)
    boundary = np.vstack([_interp_row(nodes, lam, -1.0), _interp_row(nodes, lam, 1.0)])
    md = weights[:, None] * mat
    rtbnr = boundary.T @ (_FACE_SIGNS[:, None] * boundary)
    mat = (0.5 * (md - md.T) + 0.5 * rtbnr) / weights[:, None]
    for a in (nodes, weights, mat, boundary):
        a.setflags(write=False)
    return Operator1D(p, "lgl", nodes, weights, mat, boundary)


def make_operator(p, family="lgl"):
    if family != "lgl":
        raise UnsupportedOperatorError(
            "node family %r: the flux-differencing path is LGL-only (diagonal boundary operator)" % (family,)
        )
    return lgl_operator(p)


def build_dsplit(op):
    """Split-derivative matrix for two-point volume fluxes (reference
    operators.py:204-217): 2D - M^{-1} R^T B N R."""
    if op.family != "lgl":
        raise UnsupportedOperatorError(
            "split derivative requires a diagonal boundary operator (lgl), got %r" % (op.family,)
        )
    r = op.boundary_interp
    mat = 2.0 * op.D - (r.T @ (_FACE_SIGNS[:, None] * r)) / op.weights[:, None]
    mat.setflags(write=False)
    return FluxDiffOperator(mat, op)


@lru_cache(maxsize=None)
def node_lines(p1, d):
    """Per direction, the (p1^(d-1), p1) node ids of every 1D line (reference
    operators.py:248-259): direction 0 is the slowest axis."""
    idx = np.arange(p1**d).reshape((p1,) * d)
    out = []
    for n in range(d):
        lines = np.ascontiguousarray(np.moveaxis(idx, n, -1).reshape(-1, p1))
        lines.flags.writeable = False
        out.append(lines)
    return tuple(out)


def pair_table(mat):
    """[(a, b, mat[a,b], mat[b,a]) for a < b] without all-zero pairs
    (reference operators.py:267-290)."""
    n = mat.shape[0]
    return tuple(
        (a, b, float(mat[a, b]), float(mat[b, a]))
        for a in range(n)
        for b in range(a + 1, n)
        if mat[a, b] != 0.0 or mat[b, a] != 0.0
    )
