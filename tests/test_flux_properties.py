"""Property pins of the two BASELINE volume fluxes the reference does not ship
(Kennedy-Gruber for cfg4, Chandrashekar for cfg3), on the oracle's C
restatement (oracle/fdg_oracle.c). The GPU FAITHFUL kernels are bitwise equal
to that restatement (tests/test_gpu_parity.py::test_faithful_unpinned_fluxes_
match_oracle), so these properties carry over to the device.

Patterns follow the reference's own flux tests:
* symmetry            ref tests/test_fluxes.py:47-57
* consistency         ref tests/test_fluxes.py:60-71  (f(u,u,n) = sum_j n_j f^j(u))
* entropy condition   ref tests/test_acceptance.py:103-139 (Tadmor residual of
                      the EC flux against 50-digit entropy variables, wide
                      random pairs plus near-identical pairs in the log-mean
                      series branch)
* kinetic energy preservation: f_rhov - {v} f_rho = p~ n with the flux's
  own pressure p~ ({p} for KG, {rho}/(2{beta}) for Chandrashekar)
Ranocha (pinned by the reference) runs through the same EC harness as a
control.
"""

import mpmath
import numpy as np
import pytest

from oracle import oracle

GAMMA = 1.4
mpmath.mp.dps = 50


def _prim2cons(q):
    d = q.shape[-1] - 2
    u = np.empty_like(q)
    u[..., 0] = q[..., 0]
    u[..., 1 : d + 1] = q[..., :1] * q[..., 1 : d + 1]
    u[..., d + 1] = q[..., d + 1] / (GAMMA - 1.0) + 0.5 * q[..., 0] * np.sum(q[..., 1 : d + 1] ** 2, axis=-1)
    return u


def _random_states(rng, d, n):
    """Wide admissible states (ref test_acceptance.py:95-100)."""
    q = np.empty((n, d + 2))
    q[:, 0] = 10.0 ** rng.uniform(-1.0, 1.0, n)
    q[:, 1 : d + 1] = rng.uniform(-3.0, 3.0, (n, d))
    q[:, d + 1] = 10.0 ** rng.uniform(-1.0, 1.0, n)
    return _prim2cons(q)


def _physical_flux(u, normal):
    d = len(normal)
    rho = u[0]
    v = u[1 : d + 1] / rho
    p = (GAMMA - 1.0) * (u[d + 1] - 0.5 * rho * np.dot(v, v))
    vn = np.dot(v, normal)
    f = np.empty(d + 2)
    f[0] = rho * vn
    f[1 : d + 1] = u[1 : d + 1] * vn + p * np.asarray(normal)
    f[d + 1] = (u[d + 1] + p) * vn
    return f


def _flux(ul, ur, normal, kind):
    return oracle.two_point(ul, ur, normal, kind, gamma=GAMMA)


def _entropy_vars_mp(u):
    d = len(u) - 2
    g = mpmath.mpf(GAMMA)
    rho = mpmath.mpf(float(u[0]))
    m = [mpmath.mpf(float(x)) for x in u[1 : d + 1]]
    E = mpmath.mpf(float(u[d + 1]))
    v = [x / rho for x in m]
    v2 = sum(x * x for x in v)
    p = (g - 1) * (E - rho * v2 / 2)
    s = mpmath.log(p) - g * mpmath.log(rho)
    rho_p = rho / p
    return [(g - s) / (g - 1) - rho_p * v2 / 2] + [rho_p * x for x in v] + [-rho_p]


@pytest.mark.parametrize("d", [2, 3])
@pytest.mark.parametrize("kind", ["kennedy_gruber", "chandrashekar"])
def test_symmetry(d, kind):
    rng = np.random.default_rng(11 + d)
    ul = _random_states(rng, d, 300)
    ur = _random_states(rng, d, 300)
    for i in range(len(ul)):
        n = rng.standard_normal(d)
        a = _flux(ul[i], ur[i], n, kind)
        b = _flux(ur[i], ul[i], n, kind)
        assert np.abs(a - b).max() <= 1e-13 * max(1.0, np.abs(a).max()), i


@pytest.mark.parametrize("d", [2, 3])
@pytest.mark.parametrize("kind", ["kennedy_gruber", "chandrashekar"])
def test_consistency(d, kind):
    rng = np.random.default_rng(21 + d)
    for u in _random_states(rng, d, 300):
        n = rng.standard_normal(d)
        want = _physical_flux(u, n)
        got = _flux(u, u, n, kind)
        assert np.abs(got - want).max() <= 1e-13 * max(1.0, np.abs(want).max())


@pytest.mark.parametrize("d", [2, 3])
@pytest.mark.parametrize("kind", ["kennedy_gruber", "chandrashekar"])
def test_cartesian_axis_matches_directional(d, kind):
    rng = np.random.default_rng(31 + d)
    ul = _random_states(rng, d, 100)
    ur = _random_states(rng, d, 100)
    for i in range(len(ul)):
        for j in range(d):
            e = np.zeros(d)
            e[j] = 1.0
            a = oracle.two_point(ul[i], ur[i], e, kind, gamma=GAMMA, cart_axis=j)
            b = _flux(ul[i], ur[i], e, kind)
            assert np.abs(a - b).max() <= 1e-13 * max(1.0, np.abs(a).max())


@pytest.mark.parametrize("kind", ["chandrashekar", "ranocha"])
def test_entropy_conservation_mpmath(kind):
    """Tadmor condition (w_r - w_l) . f = psi_r - psi_l, psi = rho v . n, with
    w at 50 digits; residual normalized by the cancelling mass (ref
    test_acceptance.py:103-139)."""
    worst = 0.0
    for d in (2, 3):
        rng = np.random.default_rng(100 + d)
        n_wide, n_close = 1500, 300
        left = _random_states(rng, d, n_wide + n_close)
        right = np.empty_like(left)
        right[:n_wide] = _random_states(rng, d, n_wide)
        right[n_wide:] = left[n_wide:] * (1.0 + 1e-8 * rng.uniform(-1.0, 1.0, (n_close, d + 2)))
        normals = rng.uniform(0.2, 1.2, (n_wide + n_close, d))
        for i in range(n_wide + n_close):
            f = _flux(left[i], right[i], normals[i], kind)
            wl = _entropy_vars_mp(left[i])
            wr = _entropy_vars_mp(right[i])
            terms = [(b - a) * mpmath.mpf(float(c)) for a, b, c in zip(wl, wr, f)]
            dpsi = sum(
                (mpmath.mpf(float(right[i][j + 1])) - mpmath.mpf(float(left[i][j + 1]))) * mpmath.mpf(float(normals[i][j]))
                for j in range(d)
            )
            resid = abs(sum(terms) - dpsi)
            scale = sum(abs(t) for t in terms) + abs(dpsi) + 1
            worst = max(worst, float(resid / scale))
    assert worst < 1e-12, worst


def _logmean(a, b):
    return (b - a) / np.log(b / a) if a != b else a


@pytest.mark.parametrize("d", [2, 3])
@pytest.mark.parametrize("kind", ["kennedy_gruber", "chandrashekar"])
def test_kinetic_energy_preserving_structure(d, kind):
    """f_rhov - {v} f_rho = p~ n: the momentum flux is the mass flux times the
    mean velocity plus a scalar pressure along the normal only."""
    rng = np.random.default_rng(41 + d)
    ul = _random_states(rng, d, 300)
    ur = _random_states(rng, d, 300)
    for i in range(len(ul)):
        n = rng.standard_normal(d)
        f = _flux(ul[i], ur[i], n, kind)
        vl = ul[i][1 : d + 1] / ul[i][0]
        vr = ur[i][1 : d + 1] / ur[i][0]
        pl = (GAMMA - 1.0) * (ul[i][d + 1] - 0.5 * ul[i][0] * vl @ vl)
        pr = (GAMMA - 1.0) * (ur[i][d + 1] - 0.5 * ur[i][0] * vr @ vr)
        if kind == "kennedy_gruber":
            ptil = 0.5 * (pl + pr)
        else:
            bl, br = ul[i][0] / (2 * pl), ur[i][0] / (2 * pr)
            ptil = 0.5 * (ul[i][0] + ur[i][0]) / (bl + br)
        rest = f[1 : d + 1] - 0.5 * (vl + vr) * f[0]
        scale = max(1.0, np.abs(f).max())
        assert np.abs(rest - ptil * n).max() <= 1e-13 * scale, (i, rest, ptil * n)
        # the mass flux: KG {rho}{v.n}, Chandrashekar <rho>_log {v.n}
        vn = 0.5 * (vl + vr) @ n
        rho_m = 0.5 * (ul[i][0] + ur[i][0]) if kind == "kennedy_gruber" else _logmean(ul[i][0], ur[i][0])
        assert abs(f[0] - rho_m * vn) <= 1e-12 * max(1.0, abs(f[0]), abs(rho_m * vn))
