"""GPU tests of the drop-in entry points' contracts (reference signatures and
error behaviour), beyond the numerics of tests/test_gpu_parity.py:

* per-element ``volume_fluxdiff`` (ref discretization.py:267-323) against the
  reference's own per-element outputs recorded in the golden cases
  (``vol_<state>_<flux>_<pre>`` = the scalar path) -- bitwise against the
  correctly-rounded-log oracle, <= 1e-13 relative against the reference;
* a config object that only has the reference RhsConfig's fields
  (discretization.py:87-150) is accepted by every entry point;
* ``surface_terms`` keeps the reference signature (discretization.py:681);
* ``mesh_surface`` raises the reference's cons2prim error (batched.py:521);
* chained device steps ``u = stepper.step(u, dt)`` (stage buffers
  aliasing the input) equal chained oracle steps, RK54 and SSPRK43;
* the DeviceMesh cache drops an entry when its setup dies.
"""

import gc
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import oracle
from tests import golden_io as G

pytestmark = pytest.mark.gpu


def _pkg():
    import paper_2112_10517_b200 as P

    return P


def _rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("name", ["c2d_cart_p3", "c2d_curv_p3", "c3d_cart_p3", "c3d_curv_p4", "c3d_cart_p7"])
def test_volume_fluxdiff_per_element(name):
    P = _pkg()
    c = G.case(name)
    setup = G.golden_setup(name)
    dop = SimpleNamespace(op=setup.op, matrix=setup.dsplit.matrix)
    n_check = min(6, setup.n_elements)
    for key in c:
        if not key.startswith("vol_"):
            continue
        _, state, flux, pre = key.split("_", 3)
        u = c["u_" + state]
        want_cr = oracle.volume(u, setup, flux, pre, variant="cr")
        for e in range(n_check):
            metrics = SimpleNamespace(ja=setup.metrics.ja[e], jac=setup.metrics.jac[e])
            got = P.volume_fluxdiff(u[e], dop, metrics, flux, setup.gas, pre=None if pre == "none" else pre)
            assert got.shape == u[e].shape
            assert np.array_equal(got, want_cr[e]), (key, e)
            assert _rel(got, c[key][e]) <= 1e-13, (key, e)


def test_volume_fluxdiff_reuses_one_device_image():
    P = _pkg()
    from paper_2112_10517_b200 import discretization as D

    setup = G.golden_setup("c3d_curv_p4")
    c = G.case("c3d_curv_p4")
    dop = SimpleNamespace(op=setup.op, matrix=setup.dsplit.matrix)
    D._ELEM_CACHE.clear()
    for e in range(4):
        P.volume_fluxdiff(c["u_rand"][e], dop, SimpleNamespace(ja=setup.metrics.ja[e], jac=setup.metrics.jac[e]),
                          "ranocha", setup.gas)
    assert len(D._ELEM_CACHE) == 1


def _reference_like_config(**kw):
    """Only the fields of the reference's RhsConfig: no scheme() method."""
    base = dict(volume_scheme="fluxdiff", volume_flux="ranocha", surface_flux="ranocha", precompute="none",
                overint_degree=None, kernel="reference")
    base.update(kw)
    return SimpleNamespace(**base)


def test_reference_rhsconfig_fields_accepted():
    import torch

    P = _pkg()
    from paper_2112_10517_b200.device import device_mesh_for

    name = "c3d_curv_p2"
    c = G.case(name)
    setup = G.golden_setup(name)
    u = c["u_rand"]
    cfg = _reference_like_config(surface_flux="llf")
    assert not hasattr(cfg, "scheme")
    got = P.rhs(u, setup, cfg)
    assert np.array_equal(got, oracle.rhs(u, setup, "ranocha", "llf", variant="cr"))
    vol = P.mesh_fluxdiff_volume(u, setup, cfg)
    assert np.array_equal(vol, oracle.volume(u, setup, "ranocha", variant="cr"))
    st = P.DeviceStepper(device_mesh_for(setup), cfg, P.RK54)
    st.step(torch.as_tensor(u, device="cuda"), 1e-4)
    with pytest.raises(P.ConfigurationError):
        P.rhs(u, setup, _reference_like_config(kernel="gpu"))


def test_surface_terms_reference_signature():
    P = _pkg()
    name = "c2d_curv_p3"
    c = G.case(name)
    setup = G.golden_setup(name)
    u = c["u_wave"]
    out = np.zeros_like(u)
    got = P.surface_terms(u, setup, "llf", False, None, out)
    assert got is out
    assert np.array_equal(got, c["surf_wave_llf"])
    got2 = P.surface_terms(u, setup, "llf", out=None)
    assert np.array_equal(got2, c["surf_wave_llf"])
    with pytest.raises(P.UnsupportedOperatorError):
        P.surface_terms(u, setup, "llf", subtract_own=True)
    with pytest.raises(P.UnsupportedOperatorError):
        P.surface_terms(u, setup, "llf", face_states=[(u, u)] * setup.d)


def test_mesh_surface_raises_cons2prim_error():
    P = _pkg()
    name = "c3d_cart_p3"
    c = G.case(name)
    setup = G.golden_setup(name)
    u = c["u_rand"].copy()
    u[1, 5, 0] = -0.5
    out = np.zeros_like(u)
    with pytest.raises(P.AdmissibilityError, match="cons2prim: inadmissible state"):
        P.mesh_surface(u, setup, "llf", out)
    assert not out.any()  # nothing accumulated before the error


@pytest.mark.parametrize("method,vf", [("RK54", "ranocha"), ("SSPRK43", "kennedy_gruber")])
def test_device_stepper_chained_steps(method, vf):
    """u = step(u) four times (the stepper's output fed back as its input)
    equals four chained oracle steps bitwise (FAITHFUL)."""
    import torch

    P = _pkg()
    from paper_2112_10517_b200.device import device_mesh_for

    name = "c3d_curv_p2"
    c = G.case(name)
    setup = G.golden_setup(name)
    m = getattr(P, method)
    cfg = P.RhsConfig(volume_flux=vf, surface_flux="llf", kernel="reference")
    st = P.DeviceStepper(device_mesh_for(setup), cfg, m)
    dt = 2e-4
    u = torch.as_tensor(c["u_wave"], device="cuda")
    want = c["u_wave"]
    f = lambda v: oracle.rhs(v, setup, vf, "llf", variant="cr")  # noqa: E731
    step = oracle.rk54_step if method == "RK54" else oracle.ssprk43_step
    for k in range(4):
        u = st.step(u, dt)
        want = step(want, dt, f)
        assert np.array_equal(u.cpu().numpy(), want), k


def test_device_mesh_cache_evicts_dead_setups():
    P = _pkg()
    from paper_2112_10517_b200 import device as Dv

    gas = P.GasParams(1.4)
    setup = P.build_setup(P.build_mesh((3, 3, 3), bounds=(-1.0, 1.0)), P.lgl_operator(3), gas)
    Dv.device_mesh_for(setup)
    n = len(Dv._CACHE)
    del setup
    gc.collect()
    assert len(Dv._CACHE) == n - 1
