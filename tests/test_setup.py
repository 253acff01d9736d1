"""Host-side setup against the reference's recorded tables (tests/golden/).

* operators: this package's tables are the correctly rounded exact operators
  (operators.py); the reference's float construction agrees to <= 4 ulps of
  the table's largest entry (pinned here), and the SBP identity holds to one
  rounding per entry;
* with the reference's own 1D tables (golden_operator), coordinates,
  neighbours, wave states and the Cartesian metrics are BITWISE the
  reference's, curved metrics within 1e-15 (summation order of the
  derivative contractions and the determinant)."""

import numpy as np
import pytest

from paper_2112_10517_b200 import GasParams, build_mesh, build_setup, lgl_operator, prim2cons
from paper_2112_10517_b200.operators import build_dsplit, node_lines, pair_table
from paper_2112_10517_b200 import workloads
from tests import golden_io as G


@pytest.mark.parametrize("p", range(1, 16))
def test_lgl_operator_matches_reference_tables(p):
    ops = G.operators()
    op = lgl_operator(p)
    for key, got in (("nodes", op.nodes), ("weights", op.weights), ("D", op.D), ("R", op.boundary_interp),
                     ("dsplit", build_dsplit(op).matrix)):
        want = ops["%s_%d" % (key, p)]
        ulp = np.spacing(np.abs(want).max())
        assert np.abs(got - want).max() <= 32 * ulp, (key, np.abs(got - want).max() / ulp)
    assert np.array_equal(op.boundary_interp, ops["R_%d" % p])
    # the reference-table path of build_dsplit reproduces its matrix bit for bit
    assert np.array_equal(build_dsplit(G.golden_operator(p)).matrix, ops["dsplit_%d" % p])


@pytest.mark.parametrize("p", range(1, 16))
@pytest.mark.parametrize("family", ["lgl", "gauss"])
def test_operator_sbp_and_exactness(p, family):
    from paper_2112_10517_b200.operators import make_operator

    op = make_operator(p, family)
    w, D, R = op.weights, op.D, op.boundary_interp
    Q = w[:, None] * D
    B = R[1][:, None] * R[1][None, :] - R[0][:, None] * R[0][None, :]
    assert np.abs(Q + Q.T - B).max() <= 4e-15 * max(1.0, np.abs(Q).max())
    assert abs(w.sum() - 2.0) <= 4e-16 * p
    # D is exact on polynomials of degree p, the quadrature on degree 2p-1 (lgl) / 2p+1 (gauss)
    x = op.nodes
    assert np.abs(D @ x**p - p * x ** (p - 1)).max() <= 1e-13 * max(1, p**2)
    k = 2 * p - 1 if family == "lgl" else 2 * p + 1
    assert abs(w @ x**k - (1.0 - (-1.0) ** (k + 1)) / (k + 1)) <= 1e-14
    assert abs(w @ x ** (k - 1) - (1.0 - (-1.0) ** k) / k) <= 1e-14
    if family == "lgl":
        ds = build_dsplit(op).matrix
        assert np.all(np.diag(ds) == 0.0)


@pytest.mark.parametrize("p", [1, 3, 4, 7])
def test_dsplit_properties(p):
    op = lgl_operator(p)
    ds = build_dsplit(op).matrix
    assert np.all(np.diag(ds) == 0.0)
    m = op.weights[:, None] * ds
    assert np.abs(m + m.T).max() < 1e-14 * np.abs(m).max()
    # pair table keeps every off-diagonal pair of an LGL operator
    assert len(pair_table(ds)) == p * (p + 1) // 2


def test_node_lines_strides():
    lines = node_lines(4, 3)
    assert lines[0][0].tolist() == [0, 16, 32, 48]
    assert lines[1][0].tolist() == [0, 4, 8, 12]
    assert lines[2][0].tolist() == [0, 1, 2, 3]


@pytest.mark.parametrize("name", G.CASES)
def test_setup_against_reference(name):
    c = G.case(name)
    mesh = build_mesh(tuple(c["dims"]), bounds=tuple(c["bounds"]), amplitude=float(c["amplitude"]))
    setup = build_setup(mesh, G.golden_operator(int(c["p"])), GasParams(1.4))
    assert np.array_equal(setup.coords, c["coords"])
    assert setup.metrics.cartesian == bool(c["cartesian"])
    assert np.abs(setup.metrics.ja - c["ja"]).max() <= 1e-15 * np.abs(c["ja"]).max()
    assert np.abs(setup.metrics.jac - c["jac"]).max() <= 1e-15 * np.abs(c["jac"]).max()
    if setup.metrics.cartesian:
        assert np.array_equal(setup.metrics.ja, c["ja"]) and np.array_equal(setup.metrics.jac, c["jac"])
    for n in range(setup.d):
        assert np.abs(setup.metrics.face_ja[n] - c["face_ja_%d" % n]).max() <= 1e-15 * np.abs(c["ja"]).max()
        assert np.array_equal(setup.plus_neighbor[n], c["plus_%d" % n])
    # this package's own operator: the same geometry to the nodes' rounding
    own = build_setup(mesh, lgl_operator(int(c["p"])), GasParams(1.4))
    assert np.abs(own.coords - c["coords"]).max() <= 1e-14 * max(1.0, np.abs(c["coords"]).max())
    assert np.abs(own.metrics.ja - c["ja"]).max() <= 1e-13 * np.abs(c["ja"]).max()


@pytest.mark.parametrize("name", ["c2d_cart_p3", "c3d_curv_p4", "c3d_cart_p3"])
def test_wave_state_bitwise(name):
    c = G.case(name)
    if "u_wave" not in c:
        pytest.skip("no wave state")
    q = workloads.wave_primitives(c["coords"])
    assert np.array_equal(prim2cons(q, GasParams(1.4)), c["u_wave"])


def test_cfg1_state_and_sizes():
    setup, u, cfg = workloads.build(1, op=G.golden_operator(3))
    assert u.shape == (256, 16, 4)
    assert np.array_equal(u, G.config(1)["u"])
    assert cfg.volume_flux == "ranocha" and cfg.surface_flux == "llf"


@pytest.mark.slow
def test_cfg2_cfg4_samples_bitwise():
    g2 = G.config(2)
    setup, u, _ = workloads.build(2, op=G.golden_operator(3))
    assert np.array_equal(u[g2["elements"]], g2["u_sample"])
    assert np.array_equal(u.sum(axis=(0, 1)), g2["u_sum"])
    g4 = G.config(4)
    setup, u, _ = workloads.build(4, op=G.golden_operator(4))
    idx = g4["elements"]
    assert np.array_equal(u[idx], g4["u_sample"])
    assert np.abs(setup.metrics.ja[idx] - g4["ja_sample"]).max() <= 1e-15 * np.abs(g4["ja_sample"]).max()
    assert np.abs(setup.metrics.jac[idx] - g4["jac_sample"]).max() <= 1e-15 * np.abs(g4["jac_sample"]).max()


@pytest.mark.slow
def test_cfg3_state_sample_bitwise():
    g3 = G.config(3)
    setup, u, _ = workloads.build(3, op=G.golden_operator(7))
    assert np.array_equal(u[g3["elements"]], g3["u_sample"])
    assert np.array_equal(u.sum(axis=(0, 1)), g3["u_sum"])


def test_cartesian_metrics_are_scalars():
    mesh = build_mesh((3, 2, 2), bounds=(-1.0, 1.0))
    setup = build_setup(mesh, lgl_operator(3), GasParams(1.4), with_coords=False)
    assert setup.coords is None
    assert setup.metrics._ja is None  # nothing per node until asked
    h = (2.0 / 3.0, 1.0, 1.0)
    jac = (0.5 * h[0]) * (0.5 * h[1]) * (0.5 * h[2])
    assert setup.metrics.jac_const == jac
    assert setup.metrics.areas == tuple(jac / (0.5 * h[n]) for n in range(3))
