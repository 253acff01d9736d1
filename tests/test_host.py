"""Host logic that needs no GPU: configuration validation, counters, the
Runge-Kutta tableaux (order conditions; SSPRK43 is not in the reference and
is pinned by its order conditions and an observed convergence slope)."""

import numpy as np
import pytest

from paper_2112_10517_b200 import (
    RK54,
    SSPRK43,
    ConfigurationError,
    DivergenceError,
    FluxCounter,
    RhsConfig,
    count_guard,
    integrate,
    rk_step,
)
from paper_2112_10517_b200.timeint import RKMethod, ShuOsherMethod
from tests import golden_io as G


def test_config_rejects_unknown_names():
    setup = G.golden_setup("c2d_cart_p3")
    cases = [
        (RhsConfig(volume_scheme="nope"), "volume_scheme"),
        (RhsConfig(precompute="cached"), "precompute"),
        (RhsConfig(kernel="gpu"), "kernel"),
        (RhsConfig(surface_flux="roe"), "surface_flux"),
        (RhsConfig(volume_flux="llf"), "volume flux"),
        (RhsConfig(volume_scheme="strong"), "volume_scheme"),
    ]
    for cfg, field in cases:
        with pytest.raises(ConfigurationError, match=field):
            cfg.validate(setup)
    RhsConfig(volume_flux="kennedy_gruber", surface_flux="llf", kernel="batched").validate(setup)


def test_rk54_tableau_tamper_fails():
    a = list(RK54.a)
    a[2] *= 1.0 + 1e-9
    with pytest.raises(ConfigurationError, match="order conditions"):
        RKMethod("tampered", tuple(a), RK54.b, RK54.c)


def test_ssprk43_tableau_tamper_fails():
    with pytest.raises(ConfigurationError):
        ShuOsherMethod("bad", SSPRK43.A, SSPRK43.B, (0.5, 0.5, 1.0 / 6.0, 0.6), SSPRK43.c)


@pytest.mark.parametrize("method,order", [(RK54, 4), (SSPRK43, 3)])
def test_convergence_order_linear_oscillator(method, order):
    # y' = A y, rotation; global error slope of the method
    A = np.array([[0.0, 1.0], [-1.0, 0.0]])

    def f(v, t):
        return v @ A.T

    errs = []
    for n in (20, 40, 80):
        dt = 2.0 / n
        y, _ = integrate(np.array([1.0, 0.0]), f, n_steps=n, dt=dt, method=method)
        exact = np.array([np.cos(2.0), -np.sin(2.0)])
        errs.append(np.abs(y - exact).max())
    slopes = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(np.abs(slopes - order) < 0.2), slopes


def test_divergence_is_reported_with_stage():
    def f(v, t):
        return np.full_like(v, np.inf)

    with pytest.raises(DivergenceError, match="after stage 0"):
        rk_step(np.ones(3), 0.0, 0.1, f)
    with pytest.raises(DivergenceError, match="diverged in step 0") as info:
        integrate(np.ones(3), f, n_steps=2, dt=0.1)
    assert np.array_equal(info.value.last_fields, np.ones(3))


def test_counter_guard_nesting():
    from paper_2112_10517_b200.fluxes import bump

    outer, inner, extra = FluxCounter(), FluxCounter(), FluxCounter()
    with count_guard(outer):
        with count_guard(inner):
            bump(extra, two_point=3, logmean=6)
        bump(None, two_point=1)
    assert (outer.two_point_evals, inner.two_point_evals, extra.two_point_evals) == (4, 3, 3)
    assert outer.logmean_evals == 6
