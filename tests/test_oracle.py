"""Pin the CPU oracle (oracle/fdg_oracle.c) to the reference's own outputs.

Every comparison against the scalar path is BITWISE (np.array_equal): the
oracle restates volume_fluxdiff / surface_terms / rhs(kernel="reference")
operation by operation (reference discretization.py:267-323, 681-760,
896-949). The batched-path fixtures (batched.py:450-544) are compared at the
reference's own equivalence tolerance (tests/test_batched.py: 1e-13 abs).
"""

import numpy as np
import pytest

from oracle import oracle
from tests import golden_io as G


@pytest.mark.parametrize("name", G.CASES)
def test_volume_bitwise(name):
    c = G.case(name)
    setup = G.golden_setup(name)
    checked = 0
    for key in c:
        if not key.startswith("vol_"):
            continue
        _, state, flux, pre = key.split("_", 3)
        got = oracle.volume(c["u_" + state], setup, flux, pre)
        assert np.array_equal(got, c[key]), key
        checked += 1
    assert checked >= 2


@pytest.mark.parametrize("name", G.CASES)
def test_volume_vs_batched_path(name):
    c = G.case(name)
    setup = G.golden_setup(name)
    for key in c:
        if not key.startswith("volb_"):
            continue
        _, state, flux = key.split("_", 2)
        pre = "none"
        if flux == "ranocha_logs":
            flux, pre = "ranocha", "primitives_and_logs"
        got = oracle.volume(c["u_" + state], setup, flux, pre)
        scale = max(1.0, np.abs(c[key]).max())
        assert np.abs(got - c[key]).max() <= 1e-13 * scale, key


@pytest.mark.parametrize("name", G.CASES)
def test_surface_bitwise(name):
    c = G.case(name)
    setup = G.golden_setup(name)
    for key in c:
        if not key.startswith("surf_"):
            continue
        _, state, flux = key.split("_", 2)
        got = oracle.surface(c["u_" + state], setup, flux)
        assert np.array_equal(got, c[key]), key


@pytest.mark.parametrize("name", G.CASES)
def test_rhs_bitwise(name):
    c = G.case(name)
    setup = G.golden_setup(name)
    n = 0
    for key in c:
        if not key.startswith("rhs_"):
            continue
        parts = key.split("_")
        state, vf, sf = parts[1], parts[2], parts[3]
        pre = "primitives_and_logs" if key.endswith("_logs") else "none"
        got = oracle.rhs(c["u_" + state], setup, vf, sf, pre)
        assert np.array_equal(got, c[key]), key
        n += 1
    assert n >= 1


@pytest.mark.parametrize("name", ["c2d_cart_p3", "c3d_curv_p2", "c3d_curv_p4"])
def test_rk54_bitwise(name):
    c = G.case(name)
    setup = G.golden_setup(name)
    dt = float(c["rk54_dt"])
    for state in G.states(name):
        got = oracle.rk54_step(c["u_" + state], dt, lambda v: oracle.rhs(v, setup, "ranocha", "llf"))
        assert np.array_equal(got, c["rk54_" + state])


def test_cfg1_bitwise():
    c = G.config(1)
    from types import SimpleNamespace

    # cfg1 = 2D 16x16 Cartesian on [-1,1]^2, N=3 (BASELINE.json configs[0])
    ops = G.operators()
    n_elem = 256
    idx = np.arange(n_elem).reshape(16, 16)
    plus = tuple(np.roll(idx, -1, axis=n).ravel() for n in range(2))
    jac_val = (0.5 * 2.0 / 16) ** 2
    area = jac_val / (0.5 * 2.0 / 16)
    ja = np.zeros((n_elem, 16, 2, 2))
    ja[:, :, 0, 0] = area
    ja[:, :, 1, 1] = area
    setup = SimpleNamespace(
        d=2,
        op=SimpleNamespace(weights=ops["weights_3"]),
        dsplit=SimpleNamespace(matrix=ops["dsplit_3"]),
        metrics=SimpleNamespace(ja=ja, jac=np.full((n_elem, 16), jac_val), cartesian=True),
        plus_neighbor=plus,
        gas=SimpleNamespace(gamma=1.4, inv_gamma_minus_one=1.0 / (1.4 - 1.0)),
    )
    assert np.array_equal(oracle.volume(c["u"], setup, "ranocha"), c["vol"])
    assert np.array_equal(oracle.surface(c["u"], setup, "llf"), c["surf"])
    assert np.array_equal(oracle.rhs(c["u"], setup, "ranocha", "llf"), c["du"])
    assert np.array_equal(
        oracle.rhs(c["u"], setup, "ranocha", "llf", "primitives_and_logs"), c["du_logs"]
    )


def test_gate_names_first_bad_node():
    setup = G.golden_setup("c2d_cart_p3")
    u = G.case("c2d_cart_p3")["u_rand"].copy()
    u[1, 2, -1] = 0.01
    u[4, 0, 0] = -1.0
    with pytest.raises(oracle.OracleAdmissibilityError, match="element 1, node 2"):
        oracle.rhs(u, setup)


def test_logmean_known_values():
    # equal arguments hit the series branch exactly: L(a, a) = a
    for a in (0.5, 1.0, 3.7, 1e-3, 1e5):
        assert oracle.logmean(a, a) == a
        assert oracle.inv_logmean(a, a) == 1.0 / a
    # well separated: (b - a)/log(b/a)
    assert oracle.logmean(1.0, np.e) == pytest.approx(np.e - 1.0, rel=1e-15)


# ------------------------------------------------------------ diagnostics


def _diag_golden():
    return dict(np.load(G.os.path.join(G.GOLDEN, "diagnostics.npz")))


@pytest.mark.parametrize("name", G.CASES)
def test_diagnostics_oracle_pinned(name):
    """The numpy restatement of conserved_totals / entropy_rate /
    error_norm_l2 / stable_dt against the reference's own outputs
    (tests/golden/make_diagnostics.py). Bar: <= 1e-14 relative (sums),
    entropy total within 1e-14 of its absolute scale."""
    g = _diag_golden()
    c = G.case(name)
    setup = G.golden_setup(name)
    for s in G.states(name):
        u = c["u_" + s]
        want = g["cons_%s_%s" % (name, s)]
        got = oracle.conserved_totals(u, setup)
        assert np.abs(got - want).max() <= 1e-14 * np.abs(want).max(), s
        assert abs(oracle.stable_dt(u, setup) - float(g["dt_%s_%s" % (name, s)])) <= 1e-15 * float(
            g["dt_%s_%s" % (name, s)]
        ), s
        for vf, sf in (("ranocha", "ranocha"), ("ranocha", "llf")):
            key = "ent_%s_%s_%s_%s" % (name, s, vf, sf)
            if key not in g:
                continue
            total, norm = oracle.entropy_rate(u, c["rhs_%s_%s_%s" % (s, vf, sf)], setup)
            t_ref, n_ref = g[key]
            scale = abs(t_ref / n_ref) if n_ref != 0.0 else 0.0
            assert abs(total - t_ref) <= 1e-14 * max(scale, 1e-300), key
    u_exact = c["u_wave"] if "u_wave" in c else 1.01 * c["u_rand"]
    want = g["err_%s" % name]
    got = oracle.error_norm_l2(c["u_rand"], u_exact, setup)
    assert np.abs(got - want).max() <= 1e-14 * np.abs(want).max()


# ---------------------------------------------------- full-size config pins


def test_cfg5_sample_oracle_pinned():
    """The reference's scalar volume_fluxdiff on sampled cfg5 elements
    (tests/golden/cfg5.npz): the glibc oracle is bitwise equal; the host
    sample generator (workloads.cartesian_sample, the CPU baseline's input)
    reproduces the reference's state for element 0 bit for bit."""
    from types import SimpleNamespace

    from paper_2112_10517_b200 import workloads
    from paper_2112_10517_b200.euler import GasParams
    from paper_2112_10517_b200.operators import build_dsplit, lgl_operator

    g = G.config(5)
    u = g["u_sample"]
    n = u.shape[0]
    op = G.golden_operator(3)
    setup = SimpleNamespace(
        d=3, op=op, dsplit=build_dsplit(op), gas=GasParams(1.4),
        metrics=SimpleNamespace(cartesian=True, areas=(float(g["area"]),) * 3, jac_const=float(g["jac"])),
        plus_neighbor=tuple(np.arange(n) for _ in range(3)),
    )
    for flux in ("ranocha", "shima"):
        assert np.array_equal(oracle.volume(u, setup, flux), g["vol_%s" % flux]), flux
    assert np.array_equal(oracle.volume(u, setup, "ranocha", "primitives_and_logs"), g["vol_ranocha_logs"])
    assert int(g["elements"][0]) == 0
    u0, areas, jac = workloads.cartesian_sample(5, 1, op=G.golden_operator(3))
    assert np.array_equal(u0[0], u[0])
    assert jac == float(g["jac"]) and areas[0] == float(g["area"])


# ------------------------------------------------------ Gauss-family oracle


@pytest.mark.parametrize("name", G.GAUSS_CASES)
def test_gauss_oracle_bitwise(name):
    """oracle.gauss_project (numpy, as _project_all) and or_gauss_rhs (C, as
    the scalar gauss path) against the reference's own outputs
    (tests/golden/make_gauss.py): BITWISE for every scheme and flux pair."""
    c = G.gauss_case(name)
    st = G.gauss_setup(name)
    d = st.d
    for sname in ("rand", "wave"):
        u = c["u_" + sname]
        proj = oracle.gauss_project(u, st.op)
        want_proj = np.stack([np.stack([c["proj_%s_%d_%d" % (sname, n, s)] for s in (0, 1)], axis=1)
                              for n in range(d)], axis=1)
        assert np.array_equal(proj, want_proj), sname
        for key in c:
            if not key.startswith("rhs_%s_" % sname):
                continue
            rest = key[len("rhs_%s_" % sname):]
            scheme = "gauss_surface_correction" if rest.startswith("gauss_surface_correction") else "gauss_fluxdiff"
            vf, sf = rest[len(scheme) + 1:].split("_")
            du = oracle.gauss_rhs(u, st, scheme, vf, sf)
            assert np.array_equal(du, c[key]), key


def test_gauss_scatter_tables_match_oracle():
    from paper_2112_10517_b200.operators import gauss_scatter_tables

    for name in G.GAUSS_CASES:
        st = G.gauss_setup(name)
        for scheme in ("gauss_fluxdiff", "gauss_surface_correction"):
            mine = gauss_scatter_tables(st.op, scheme)
            ref = oracle.gauss_tables(st.op, scheme)
            assert all(np.array_equal(a, b) for a, b in zip(mine, ref)), (name, scheme)


def test_gauss_counter_totals_match_reference():
    """Analytic counter totals of the gauss path (discretization._gauss_counts)
    against the reference's FluxCounter on the same call."""
    from types import SimpleNamespace

    from paper_2112_10517_b200.discretization import _gauss_counts

    for name in G.GAUSS_CASES:
        c = G.gauss_case(name)
        st = G.gauss_setup(name)
        for key in c:
            if not key.startswith("counts_rand_"):
                continue
            rest = key[len("counts_rand_"):]
            scheme = "gauss_surface_correction" if rest.startswith("gauss_surface_correction") else "gauss_fluxdiff"
            vf, sf = rest[len(scheme) + 1:].split("_")
            cfg = SimpleNamespace(volume_scheme=scheme, volume_flux=vf, surface_flux=sf)
            tp, lm = _gauss_counts(st, cfg)
            assert (tp, 0, lm) == tuple(int(x) for x in c[key]), key
