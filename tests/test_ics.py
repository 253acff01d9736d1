"""Benchmark initial conditions and the PID protocol's host side against the
reference's own outputs (tests/golden/ics.npz, written by
tests/golden/make_ics.py from the reference harness)."""

import os

import numpy as np
import pytest

from tests import golden_io as G


def _g():
    return dict(np.load(os.path.join(G.GOLDEN, "ics.npz")))


@pytest.mark.parametrize("d", [2, 3])
def test_initial_conditions_bitwise(d):
    from paper_2112_10517_b200 import ics

    g = _g()
    x = g["coords_%dd" % d]
    assert np.array_equal(ics.vortex_primitives(x, 0.0, 20.0, 1.4), g["vortex_%dd" % d])
    assert np.array_equal(ics.vortex_primitives(x, 0.7, 20.0, 1.4), g["vortex_t_%dd" % d])
    assert np.array_equal(ics.sinusoidal_primitives(x, 1.4), g["sinus_%dd" % d])
    assert np.array_equal(ics.free_stream_primitives(x), g["free_%dd" % d])
    assert np.array_equal(ics.random_primitives(x, 3), g["random_%dd" % d])


@pytest.mark.parametrize("d", [2, 3])
def test_pid_run_setup_matches_reference(d):
    """build_pid_run reproduces the reference harness's coordinates and
    initial state (isentropic vortex on [-5, 5]^d) bit for bit, and the host
    stable_dt its step size."""
    from paper_2112_10517_b200 import StepController, stable_dt
    from paper_2112_10517_b200.pid import build_pid_run

    g = _g()
    setup, u0, cfg = build_pid_run(d=d, p=3, elements=8 if d == 2 else 4, kernel="reference")
    assert np.array_equal(setup.coords, g["coords_%dd" % d])
    assert np.array_equal(u0, g["u0_%dd" % d])
    dt = stable_dt(u0, setup.mesh, setup.metrics, setup.gas, 3, StepController(0.5))
    assert abs(dt - float(g["dt0_%dd" % d])) <= 1e-15 * float(g["dt0_%dd" % d])
