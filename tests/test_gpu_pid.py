"""The paper's PID protocol on the device (paper_2112_10517_b200.pid) against
the reference harness's run_simulation (tests/golden/ics.npz): the isentropic
vortex, RK54, CFL step size recomputed every step, 3 steps -- FAITHFUL device
stepping within 1e-12 of the reference's fields (the correctly rounded log
vs glibc's), and a finite PID from the graph-captured 90-step protocol."""

import os

import numpy as np
import pytest

from tests import golden_io as G

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d", [2, 3])
def test_vortex_run_matches_reference_harness(d):
    import torch

    from paper_2112_10517_b200 import RK54, DeviceStepper, StepController, stable_dt
    from paper_2112_10517_b200.device import device_mesh_for
    from paper_2112_10517_b200.pid import build_pid_run

    g = dict(np.load(os.path.join(G.GOLDEN, "ics.npz")))
    setup, u0, cfg = build_pid_run(d=d, p=3, elements=8 if d == 2 else 4, kernel="reference")
    st = DeviceStepper(device_mesh_for(setup), cfg, RK54)
    u = torch.as_tensor(u0, device="cuda")
    t = 0.0
    for _ in range(3):
        dt = stable_dt(u, None, setup.metrics, setup.gas, 3, StepController(0.5), setup=setup)
        u = st.step(u, dt)
        t += dt
    want = g["final_%dd" % d]
    got = u.cpu().numpy()
    assert abs(t - float(g["t_%dd" % d])) <= 1e-14 * float(g["t_%dd" % d])
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()


@pytest.mark.parametrize("d,kernel", [(2, "batched"), (3, "batched"), (3, "reference")])
def test_pid_protocol_runs(d, kernel):
    from paper_2112_10517_b200.pid import build_pid_run, measure_pid_device

    setup, u0, cfg = build_pid_run(d=d, p=3, kernel=kernel)
    res = measure_pid_device(setup, u0, cfg, n_steps=90, repeats=2)
    assert res["n_rhs"] == 450 and res["dofs"] == 8**d * 4**d
    assert 0.0 < res["mean_pid"] < 1e-6
    assert np.all(np.isfinite(res["final"]))
