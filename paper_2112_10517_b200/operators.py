"""One-dimensional SBP operators on [-1, 1] and the tables the kernels consume.

Interface (names and meaning of the reference's operators module,
operators.py:29-357): ``Operator1D`` (degree, family, nodes, weights, D,
boundary_interp), ``FluxDiffOperator`` (matrix = 2D - M^-1 R^T B N R),
``lgl_operator``/``make_operator``, ``build_dsplit``, ``node_lines``,
``pair_table``.

Construction (independent of the reference's float Newton iteration and
float SBP re-assembly): every table is evaluated in 40-digit arithmetic
(mpmath) and rounded ONCE to double, so each entry is the correctly rounded
value of the exact operator:

* nodes: Lobatto = +-1 and the roots of P_p'; Gauss = the roots of P_{p+1};
  Newton on the three-term Legendre recurrence from Chebyshev guesses;
* weights: Lobatto 2 / (p (p+1) P_p(x)^2), Gauss 2 / ((1-x^2) P'_{p+1}(x)^2);
* D: the Lagrange-basis derivative at the nodes in barycentric form,
  D_ij = (lam_j / lam_i) / (x_i - x_j), D_ii = -sum_{j != i} D_ij;
* R: the Lagrange basis evaluated at -1 / +1 (unit rows for Lobatto);
* Dsplit (Lobatto only): 2 D - M^-1 R^T B N R, exact zero diagonal.

The exact operators satisfy M D + D^T M = R^T B N R; the rounded tables do
to one rounding per entry (tests/test_setup.py). The reference's own
float construction agrees with these tables to <= 1 ulp of each entry
(tests/test_setup.py pins that against tests/golden/operators.npz); where a
test needs the reference's exact bits it takes them from the golden tables
(tests/golden_io.py), and a reference-built SpatialSetup passed to the
drop-in entry points is used as given (its Dsplit and weights go to the
device unchanged).
"""

from dataclasses import dataclass
from functools import lru_cache

import mpmath
import numpy as np

from .errors import UnsupportedOperatorError

MAX_DEGREE = 15
DEVICE_MAX_DEGREE = 7
FAMILIES = ("lgl", "gauss")
_DPS = 40


@dataclass(frozen=True)
class Operator1D:
    degree: int
    family: str
    nodes: np.ndarray            # (p+1,)
    weights: np.ndarray          # (p+1,) diagonal mass matrix
    D: np.ndarray                # (p+1, p+1) differentiation matrix
    boundary_interp: np.ndarray  # (2, p+1): evaluation at -1 (row 0) and +1 (row 1)

    @property
    def n_nodes(self):
        return self.degree + 1


@dataclass(frozen=True)
class FluxDiffOperator:
    """2D - M^{-1} R^T B N R: zero diagonal, M-antisymmetric off-diagonal."""

    matrix: np.ndarray
    op: Operator1D


# ------------------------------------------------------ exact construction


def _legendre_mp(n, x):
    """(P_n(x), P_n'(x)) in mpmath by the recurrence
    k P_k = (2k-1) x P_{k-1} - (k-1) P_{k-2}, P_k' = P_{k-2}' + (2k-1) P_{k-1}."""
    p0, p1 = mpmath.mpf(1), x
    d0, d1 = mpmath.mpf(0), mpmath.mpf(1)
    if n == 0:
        return p0, d0
    for k in range(2, n + 1):
        p0, p1 = p1, ((2 * k - 1) * x * p1 - (k - 1) * p0) / k
        d0, d1 = d1, d0 + (2 * k - 1) * p0
    return p1, d1


def _newton_roots(f_df, guesses):
    out = []
    tol = mpmath.mpf(10) ** (-(_DPS - 5))
    for x in guesses:
        x = mpmath.mpf(x)
        for _ in range(100):
            f, df = f_df(x)
            step = f / df
            x -= step
            if abs(step) < tol:
                break
        out.append(x)
    return out


def _lobatto_mp(p):
    # interior nodes: zeros of P_p'; (P_p')' from the Legendre ODE
    # (1 - x^2) P'' = 2 x P' - p (p+1) P
    def f_df(x):
        lp, dlp = _legendre_mp(p, x)
        return dlp, (2 * x * dlp - p * (p + 1) * lp) / (1 - x * x)

    inner = _newton_roots(f_df, [-mpmath.cos(mpmath.pi * k / p) for k in range(1, p)])
    nodes = [mpmath.mpf(-1)] + inner + [mpmath.mpf(1)]
    weights = [mpmath.mpf(2) / (p * (p + 1) * _legendre_mp(p, x)[0] ** 2) for x in nodes]
    return nodes, weights


def _gauss_mp(p):
    n = p + 1
    guesses = [-mpmath.cos(mpmath.pi * (k + mpmath.mpf(3) / 4) / (n + mpmath.mpf(1) / 2)) for k in range(n)]
    nodes = _newton_roots(lambda x: _legendre_mp(n, x), guesses)
    weights = [mpmath.mpf(2) / ((1 - x * x) * _legendre_mp(n, x)[1] ** 2) for x in nodes]
    return nodes, weights


def _lagrange_tables_mp(nodes):
    """(D, R) of the Lagrange basis on ``nodes`` in mpmath."""
    n = len(nodes)
    lam = []
    for i in range(n):
        prod = mpmath.mpf(1)
        for j in range(n):
            if j != i:
                prod *= nodes[i] - nodes[j]
        lam.append(1 / prod)
    D = [[mpmath.mpf(0)] * n for _ in range(n)]
    for i in range(n):
        for j in range(n):
            if i != j:
                D[i][j] = (lam[j] / lam[i]) / (nodes[i] - nodes[j])
        D[i][i] = -mpmath.fsum(D[i][j] for j in range(n) if j != i)
    R = []
    for y in (mpmath.mpf(-1), mpmath.mpf(1)):
        hit = [k for k in range(n) if nodes[k] == y]
        if hit:
            R.append([mpmath.mpf(1) if k == hit[0] else mpmath.mpf(0) for k in range(n)])
        else:
            c = [lam[k] / (y - nodes[k]) for k in range(n)]
            s = mpmath.fsum(c)
            R.append([ck / s for ck in c])
    return D, R


def _to_f64(a):
    """Round once to double; entries that are zero in exact arithmetic (the
    middle node of an odd count, interior LGL diagonals of D, the diagonal
    of Dsplit) come out of the 40-digit evaluation as ~1e-40 residues and are
    snapped to an exact 0."""
    flat = [x for row in a for x in row] if isinstance(a[0], list) else list(a)
    scale = max(abs(x) for x in flat)
    tiny = scale * mpmath.mpf(10) ** (-(_DPS - 10))
    snap = lambda x: 0.0 if abs(x) <= tiny else float(x)  # noqa: E731
    arr = np.array([[snap(x) for x in row] for row in a]) if isinstance(a[0], list) else np.array([snap(x) for x in a])
    arr.setflags(write=False)
    return arr


@lru_cache(maxsize=None)
def _exact_tables(p, family):
    with mpmath.workdps(_DPS):
        nodes, weights = (_lobatto_mp if family == "lgl" else _gauss_mp)(p)
        D, R = _lagrange_tables_mp(nodes)
        dsplit = None
        if family == "lgl":
            n = p + 1
            # 2D - M^-1 R^T B N R: R^T B N R = diag(-1, 0, .., 0, 1) for Lobatto
            dsplit = [[2 * D[i][j] for j in range(n)] for i in range(n)]
            dsplit[0][0] += 1 / weights[0]
            dsplit[p][p] -= 1 / weights[p]
        return (_to_f64(nodes), _to_f64(weights), _to_f64(D), _to_f64(R), None if dsplit is None else _to_f64(dsplit))


def _check_degree(p):
    if not (1 <= p <= MAX_DEGREE):
        raise UnsupportedOperatorError("degree %r outside supported range 1..%d" % (p, MAX_DEGREE))


@lru_cache(maxsize=None)
def make_operator(p, family="lgl"):
    """The degree-p operator of node family ``family`` ('lgl' or 'gauss')."""
    _check_degree(p)
    if family not in FAMILIES:
        raise UnsupportedOperatorError("unknown node family %r (choose from %s)" % (family, ", ".join(FAMILIES)))
    nodes, weights, D, R, _ = _exact_tables(p, family)
    return Operator1D(p, family, nodes, weights, D, R)


def lgl_operator(p):
    return make_operator(p, "lgl")


def gauss_operator(p):
    return make_operator(p, "gauss")


def build_dsplit(op):
    """Split-derivative matrix for two-point volume fluxes (reference
    operators.py:204-217): 2D - M^{-1} R^T B N R. Operators built here use
    the correctly rounded table; any other LGL operator object (e.g. the
    reference's own) gets it from its D and weights, which for unit
    boundary rows is 2 D with 1/w_0 added at (0, 0) and 1/w_p subtracted at
    (p, p) -- the same roundings as the reference's matrix expression."""
    if op.family != "lgl":
        raise UnsupportedOperatorError(
            "split derivative requires a diagonal boundary operator (lgl), got %r" % (op.family,)
        )
    if isinstance(op, Operator1D) and op is make_operator(op.degree, "lgl"):
        mat = _exact_tables(op.degree, "lgl")[4]
    else:
        D = np.asarray(op.D, dtype=np.float64)
        w = np.asarray(op.weights, dtype=np.float64)
        R = np.asarray(op.boundary_interp, dtype=np.float64)
        bnd = R[1][:, None] * R[1][None, :] - R[0][:, None] * R[0][None, :]
        mat = 2.0 * D - bnd / w[:, None]
        mat.setflags(write=False)
    return FluxDiffOperator(mat, op)


# ------------------------------------------------------------ index tables


@lru_cache(maxsize=None)
def node_lines(p1, d):
    """Per direction n, the (p1^(d-1), p1) node ids of the 1D lines of a
    (p1)^d element: node ids are C-ordered over the d reference axes
    (direction 0 slowest), so position a on line m of direction n is
    (m // s * p1 + a) * s + m % s with s = p1^(d-1-n) -- the same formula
    the device kernels use (Geo::line_node, fdg_kernels.cuh)."""
    out = []
    for n in range(d):
        s = p1 ** (d - 1 - n)
        m = np.arange(p1 ** (d - 1))[:, None]
        a = np.arange(p1)[None, :]
        lines = ((m // s) * p1 + a) * s + m % s
        lines.setflags(write=False)
        out.append(lines)
    return tuple(out)


def pair_table(mat):
    """Upper-triangle scatter list [(a, b, mat[a,b], mat[b,a]) for a < b]
    with the pairs whose two weights are both zero dropped (the order the
    reference's pair loops visit, operators.py:267-290)."""
    m = np.asarray(mat)
    ia, ib = np.triu_indices(m.shape[0], k=1)
    keep = (m[ia, ib] != 0.0) | (m[ib, ia] != 0.0)
    return tuple((int(a), int(b), float(m[a, b]), float(m[b, a])) for a, b in zip(ia[keep], ib[keep]))


# ------------------------------------------------------ Gauss-family tables

_FACE_SIGN = (-1.0, 1.0)
GAUSS_SCHEMES = ("gauss_fluxdiff", "gauss_surface_correction")


def hybridized_skew(op):
    """The hybridized skew operator on [volume nodes; -1 face; +1 face]
    (reference operators.py:220-245, build_hybridized):
    Q_h = [[ (M D - (M D)^T)/2,  R^T N / 2 ],
           [ -N R / 2,           N / 2     ]]
    so Q_h + Q_h^T = blockdiag(0, N) and the face consistency flux lives in
    the volume operator."""
    w = np.asarray(op.weights, dtype=np.float64)
    D = np.asarray(op.D, dtype=np.float64)
    R = np.asarray(op.boundary_interp, dtype=np.float64)
    n = w.shape[0]
    sgn = np.array(_FACE_SIGN)
    md = w[:, None] * D
    q = np.zeros((n + 2, n + 2))
    q[:n, :n] = 0.5 * (md - md.T)
    q[:n, n:] = 0.5 * (R.T * sgn[None, :])
    q[n:, :n] = -0.5 * (sgn[:, None] * R)
    q[n:, n:] = 0.5 * np.diag(sgn)
    return q


def gauss_scatter_tables(op, scheme):
    """Per-line scatter coefficients of the Gauss schemes (reference
    operators.py:300-357, hybridized_scatter / skew_pair_table), evaluated in
    float from the operator's own arrays:

    * vv (p+1, p+1): volume pair weights, vv[a, b] = c_ab for the pair (a, b):
      2 Q_h[a, b] / w_a ("gauss_fluxdiff") or the split-derivative matrix
      2D - M^-1 R^T B N R ("gauss_surface_correction"); both-zero pairs are 0
    * cvol (2, p+1): crossing weight into volume row a, 2 Q_h[a, face s] / w_a
    * cface (2, p+1): crossing weight into the face row, 2 Q_h[face s, a]
    * lift (2, p+1): R[s, a] / w_a (carries a face row back to the line)."""
    if scheme not in GAUSS_SCHEMES:
        raise UnsupportedOperatorError("unknown gauss scheme %r" % (scheme,))
    w = np.asarray(op.weights, dtype=np.float64)
    R = np.asarray(op.boundary_interp, dtype=np.float64)
    n = w.shape[0]
    q = hybridized_skew(op)
    if scheme == "gauss_surface_correction":
        sgn = np.array(_FACE_SIGN)
        mat = 2.0 * np.asarray(op.D, dtype=np.float64) - (R.T @ (sgn[:, None] * R)) / w[:, None]
        vv = np.where(np.eye(n, dtype=bool), 0.0, mat)
    else:
        vv = np.zeros((n, n))
        for a in range(n):
            for b in range(n):
                if a != b:
                    vv[a, b] = 2.0 * q[a, b] / w[a]
    cvol = np.array([[2.0 * q[a, n + s] / w[a] for a in range(n)] for s in (0, 1)])
    cface = np.array([[2.0 * q[n + s, a] for a in range(n)] for s in (0, 1)])
    lift = np.array([[R[s, a] / w[a] for a in range(n)] for s in (0, 1)])
    return vv, cvol, cface, lift
