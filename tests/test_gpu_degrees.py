"""GPU parity at EVERY 3D degree N = 1..7 (p + 1 = 2..8): the per-degree launch
shapes (elements per batch, CTA size, register cap, volume-only / RHS / stage
twins, compile-time vs runtime direction passes) are all chosen
per p + 1, and the golden fixtures only hold N = 2, 3, 4, 6, 7 in 3D, so this
file runs each degree against the C oracle on small meshes whose element
counts leave ragged last batches for the batch sizes in use (2, 3 and 7).

Bars: FAITHFUL rhs BITWISE equal to the correctly-rounded-log oracle; FAST
volume integral <= 1e-12 max|VOL_ref|, FAST rhs <= 1e-12 max(max|VOL_ref|,
max|SURF_ref|) (the cancellation-aware bar of test_gpu_parity.py); one RK
stage (the stage twins) through DeviceStepper against the RHS path.
"""

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu

# (BASELINE state generator, dims): Cartesian 45 elements (ragged for batches
# of 2 and 7), curved 20 elements (ragged for batches of 3)
MESHES = [(2, (5, 3, 3)), (4, (5, 2, 2))]


def _build(cfg, dims, p):
    from paper_2112_10517_b200 import workloads
    from paper_2112_10517_b200.operators import lgl_operator

    setup, u, _ = workloads.build(cfg, dims=dims, op=lgl_operator(p))
    return setup, u


@pytest.mark.parametrize("cfg, dims", MESHES)
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7])
def test_faithful_rhs_bitwise_every_degree(p, cfg, dims):
    import paper_2112_10517_b200 as P

    setup, u = _build(cfg, dims, p)
    for vf in ("ranocha", "shima"):
        want = oracle.rhs(u, setup, vf, "llf", variant="cr")
        got = P.rhs(u, setup, P.RhsConfig(volume_flux=vf, surface_flux="llf", kernel="reference"))
        assert np.array_equal(got, want), (p, vf)


@pytest.mark.parametrize("cfg, dims", MESHES)
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7])
def test_fast_volume_and_rhs_every_degree(p, cfg, dims):
    import paper_2112_10517_b200 as P

    setup, u = _build(cfg, dims, p)
    surf = oracle.surface(u, setup, "llf", variant="cr")
    for vf, pre in (("ranocha", "primitives_and_logs"), ("ranocha", "none"), ("shima", "none"),
                    ("kennedy_gruber", "none"), ("chandrashekar", "primitives_and_logs")):
        c = P.RhsConfig(volume_flux=vf, surface_flux="llf", precompute=pre, kernel="batched")
        vref = oracle.volume(u, setup, vf, pre, variant="cr")
        vol = P.mesh_fluxdiff_volume(u, setup, c)
        assert np.abs(vol - vref).max() <= 1e-12 * np.abs(vref).max(), (p, vf, pre)
        dref = oracle.rhs(u, setup, vf, "llf", pre, variant="cr")
        du = P.rhs(u, setup, c)
        scale = max(np.abs(vref).max(), np.abs(surf).max())
        assert np.abs(du - dref).max() <= 1e-12 * scale, (p, vf, pre)


@pytest.mark.parametrize("p", [3, 4, 5, 6, 7])
def test_fast_stage_twin_matches_rhs_path(p):
    """One SSPRK43 step through the fused stage kernels against the same step
    assembled on the host from the FAST RHS (same kernels' arithmetic up to
    the stage update's rounding): <= 1e-13 of max|u|."""
    import torch

    import paper_2112_10517_b200 as P
    from paper_2112_10517_b200.device import device_mesh_for

    setup, u = _build(2, (5, 3, 3), p)
    c = P.RhsConfig(volume_flux="ranocha", surface_flux="llf", precompute="primitives_and_logs", kernel="batched")
    dt = 1e-4
    st = P.DeviceStepper(device_mesh_for(setup), c, P.SSPRK43)
    got = st.step(torch.as_tensor(u, device="cuda"), dt).cpu().numpy()
    want = oracle.ssprk43_step(u, dt, lambda y: P.rhs(y, setup, c))
    assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max(), p
