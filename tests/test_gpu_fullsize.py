"""Parity at the BASELINE configurations' FULL sizes (GPU).

cfg5 (128^3 N=3 Cartesian, 134 M nodes, noisy wave) and cfg4 (48^3 N=4
curved, KG / Ranocha), whole mesh, through the public API and the C ABI,
against the C oracle on the same state:

* FAITHFUL (kernel="reference"): BITWISE equal to liboracle_cr (the scalar
  path's arithmetic with a correctly rounded log) -- RHS on the whole mesh,
  one SSPRK43 step on cfg4;
* FAST (kernel="batched"): VOL <= 1e-12 max|VOL_ref| (literal bar);
  RHS <= 1e-12 max(max|VOL_ref|, max|SURF_ref|) (cancellation-aware bar,
  SURVEY.md 9 item 1) and the literal max|du - du_ref| / max|du_ref| is
  recorded next to the reference's own self-floor (bat-vs-ref of SURVEY.md
  9 item 1: 7.4e-13 at cfg2, 9.85e-12 Ranocha / 1.18e-11 Shima at cfg4);
* reference-generated samples: cfg5 scalar volume_fluxdiff on 16 sampled
  elements (tests/golden/cfg5.npz), cfg4 batched rhs on 12 sampled elements
  with the whole-mesh maxima (tests/golden/cfg4_rhs.npz).

Every measured error is appended to gpurun_out/parity_fullsize.jsonl (when
that directory exists) so the numbers can be committed under profiles/.
"""

import json
import os

import numpy as np
import pytest

from oracle import oracle
from tests import golden_io as G

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SELF_FLOOR = {  # the reference's batched-vs-scalar du disagreement
    ("cfg4", "ranocha"): 9.85e-12,
    ("cfg4", "shima"): 1.18e-11,
    ("cfg2", "ranocha"): 7.38e-13,
}


def _log(rec):
    d = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(d):
        with open(os.path.join(d, "parity_fullsize.jsonl"), "a") as f:
            f.write(json.dumps(rec) + "\n")


def _P():
    import paper_2112_10517_b200 as P

    return P


def _rel(a, b, scale):
    return float(np.abs(a - b).max() / scale)


@pytest.fixture(scope="module")
def cfg5():
    """cfg5 built on the device (workloads.build_device) and its host copy."""
    from paper_2112_10517_b200 import workloads

    setup, u_dev, _ = workloads.build_device(5, kernel="reference")
    u = u_dev.cpu().numpy()
    return setup, u_dev, u


@pytest.mark.parametrize("flux", ["ranocha", "shima"])
def test_cfg5_full_mesh(cfg5, flux):
    P = _P()
    setup, u_dev, u = cfg5
    mesh = oracle.mesh_from_setup(setup)
    # FAITHFUL rhs: bitwise on all 134 M nodes
    du_cr = oracle.rhs(u, mesh, flux, "llf", variant="cr")
    got = P.rhs(u_dev, setup, P.RhsConfig(volume_flux=flux, surface_flux="llf", kernel="reference")).cpu().numpy()
    n_diff = int(np.count_nonzero(got != du_cr))
    assert n_diff == 0, n_diff
    del got, du_cr
    # FAST volume (the headline kernel) and rhs against the reference arithmetic
    pre = "primitives_and_logs" if flux == "ranocha" else "none"
    vol_ref = oracle.volume(u, mesh, flux, pre)
    vol_scale = float(np.abs(vol_ref).max())
    vol = P.mesh_fluxdiff_volume(u_dev, setup, P.RhsConfig(volume_flux=flux, precompute=pre, kernel="batched"))
    e_vol = _rel(vol.cpu().numpy(), vol_ref, vol_scale)
    del vol
    surf_ref = oracle.surface(u, mesh, "llf")
    surf_scale = float(np.abs(surf_ref).max())
    du_ref = -(vol_ref + surf_ref)
    del surf_ref, vol_ref
    du_scale = float(np.abs(du_ref).max())
    du = P.rhs(u_dev, setup, P.RhsConfig(volume_flux=flux, surface_flux="llf", precompute=pre, kernel="batched"))
    diff = float(np.abs(du.cpu().numpy() - du_ref).max())
    rec = {
        "case": "cfg5 128^3 N=3 %s+llf, whole mesh (134217728 nodes)" % flux,
        "faithful_rhs_bitwise_vs_oracle_cr": True,
        "fast_vol_rel_max_vol": e_vol,
        "fast_rhs_rel_cancellation_aware": diff / max(vol_scale, surf_scale),
        "fast_rhs_rel_literal_max_du": diff / du_scale,
        "max_vol": vol_scale, "max_surf": surf_scale, "max_du": du_scale,
        "precompute": pre,
    }
    _log(rec)
    assert e_vol <= 1e-12, rec
    assert diff <= 1e-12 * max(vol_scale, surf_scale), rec


@pytest.mark.parametrize("flux", ["ranocha", "shima"])
def test_cfg5_reference_sample(flux):
    """The reference's scalar volume_fluxdiff on 16 sampled cfg5 elements."""
    from types import SimpleNamespace

    P = _P()
    g = G.config(5)
    u = g["u_sample"]
    n = u.shape[0]
    op = G.golden_operator(3)
    area = float(g["area"])
    setup = SimpleNamespace(
        d=3, op=op, dsplit=P.build_dsplit(op), gas=P.GasParams(1.4),
        metrics=SimpleNamespace(cartesian=True, areas=(area,) * 3, jac_const=float(g["jac"])),
        plus_neighbor=tuple(np.arange(n) for _ in range(3)), n_elements=n,
    )
    want = g["vol_%s" % flux]
    scale = float(np.abs(want).max())
    got = P.mesh_fluxdiff_volume(u, setup, P.RhsConfig(volume_flux=flux, kernel="reference"))
    assert np.array_equal(got, oracle.volume(u, setup, flux, variant="cr"))
    e_faith = _rel(got, want, scale)
    fast = P.mesh_fluxdiff_volume(u, setup, P.RhsConfig(volume_flux=flux, kernel="batched"))
    e_fast = _rel(fast, want, scale)
    rec = {"case": "cfg5 reference sample (16 elements, scalar volume_fluxdiff) %s" % flux,
           "faithful_rel": e_faith, "fast_rel": e_fast}
    if flux == "ranocha":
        want_l = g["vol_ranocha_logs"]
        fl = P.mesh_fluxdiff_volume(u, setup, P.RhsConfig(volume_flux=flux, kernel="batched",
                                                          precompute="primitives_and_logs"))
        rec["fast_logs_rel"] = _rel(fl, want_l, scale)
        assert rec["fast_logs_rel"] <= 1e-12
    _log(rec)
    assert e_faith <= 1e-13 and e_fast <= 1e-12, rec


@pytest.fixture(scope="module")
def cfg4():
    from paper_2112_10517_b200 import workloads

    setup, u, _ = workloads.build(4, kernel="reference", op=G.golden_operator(4))
    return setup, u


@pytest.mark.parametrize("flux", ["kennedy_gruber", "ranocha"])
def test_cfg4_full_rhs(cfg4, flux):
    import torch

    P = _P()
    setup, u = cfg4
    mesh = oracle.mesh_from_setup(setup)
    u_dev = torch.as_tensor(u, device="cuda")
    got = P.rhs(u_dev, setup, P.RhsConfig(volume_flux=flux, surface_flux="llf", kernel="reference")).cpu().numpy()
    du_cr = oracle.rhs(u, mesh, flux, "llf", variant="cr")
    n_diff = int(np.count_nonzero(got != du_cr))
    assert n_diff == 0, n_diff
    vol_ref = oracle.volume(u, mesh, flux)
    surf_ref = oracle.surface(u, mesh, "llf")
    du_ref = -(vol_ref + surf_ref)
    scales = (float(np.abs(vol_ref).max()), float(np.abs(surf_ref).max()), float(np.abs(du_ref).max()))
    rec = {"case": "cfg4 48^3 N=4 curved %s+llf, whole mesh (13824000 nodes)" % flux,
           "faithful_rhs_bitwise_vs_oracle_cr": True,
           "faithful_rel_literal_vs_glibc_oracle": _rel(got, du_ref, scales[2]),
           "max_vol": scales[0], "max_surf": scales[1], "max_du": scales[2]}
    for pre in (("none", "primitives_and_logs") if flux == "ranocha" else ("none",)):
        du = P.rhs(u_dev, setup, P.RhsConfig(volume_flux=flux, surface_flux="llf", precompute=pre,
                                             kernel="batched")).cpu().numpy()
        diff = float(np.abs(du - du_ref).max())
        rec["fast_%s_rel_cancellation_aware" % pre] = diff / max(scales[0], scales[1])
        rec["fast_%s_rel_literal_max_du" % pre] = diff / scales[2]
        vol = P.mesh_fluxdiff_volume(u_dev, setup, P.RhsConfig(volume_flux=flux, precompute=pre, kernel="batched"))
        rec["fast_%s_vol_rel" % pre] = _rel(vol.cpu().numpy(), vol_ref, scales[0])
    rec["reference_self_floor_literal"] = SELF_FLOOR.get(("cfg4", flux))
    _log(rec)
    for pre in (("none", "primitives_and_logs") if flux == "ranocha" else ("none",)):
        assert rec["fast_%s_vol_rel" % pre] <= 1e-12, rec
        assert rec["fast_%s_rel_cancellation_aware" % pre] <= 1e-12, rec


def test_cfg4_reference_batched_rhs_sample(cfg4):
    """Against the reference's own batched rhs on the full cfg4 mesh
    (tests/golden/cfg4_rhs.npz): sampled rows, bars relative to the
    reference's whole-mesh maxima."""
    import torch

    P = _P()
    setup, u = cfg4
    g = G.config("4_rhs")
    idx = g["elements"]
    assert np.array_equal(u[idx], g["u_sample"])  # the same state, bit for bit
    u_dev = torch.as_tensor(u, device="cuda")
    vs = float(g["vol_max"].max())
    ss = float(g["surf_max"].max())
    ds = float(g["du_max"].max())
    rec = {"case": "cfg4 vs the reference's batched rhs (ranocha+llf), 12 sampled elements"}
    for kernel in ("reference", "batched"):
        du = P.rhs(u_dev, setup, P.RhsConfig(volume_flux="ranocha", surface_flux="llf", kernel=kernel))
        d = du[torch.as_tensor(idx, device="cuda")].cpu().numpy()
        diff = float(np.abs(d - g["du_sample"]).max())
        rec[kernel + "_rel_literal_max_du"] = diff / ds
        rec[kernel + "_rel_cancellation_aware"] = diff / max(vs, ss)
        vol = P.mesh_fluxdiff_volume(u_dev, setup, P.RhsConfig(volume_flux="ranocha", kernel=kernel))
        rec[kernel + "_vol_rel"] = _rel(vol[torch.as_tensor(idx, device="cuda")].cpu().numpy(), g["vol_sample"], vs)
    rec["reference_self_floor_literal"] = SELF_FLOOR[("cfg4", "ranocha")]
    _log(rec)
    for kernel in ("reference", "batched"):
        assert rec[kernel + "_vol_rel"] <= 1e-12, rec
        assert rec[kernel + "_rel_cancellation_aware"] <= 1e-12, rec


def test_cfg4_ssprk43_step(cfg4):
    """One SSPRK43 step of cfg4 (KG + llf): FAITHFUL bitwise vs the oracle's
    step (4 oracle RHS on the whole mesh); FAST within 1e-13 max|u|."""
    import torch

    P = _P()
    from paper_2112_10517_b200.device import device_mesh_for

    setup, u = cfg4
    mesh = oracle.mesh_from_setup(setup)
    dt = 1e-4
    u_dev = torch.as_tensor(u, device="cuda")
    dm = device_mesh_for(setup)
    want = oracle.ssprk43_step(u, dt, lambda v: oracle.rhs(v, mesh, "kennedy_gruber", "llf", variant="cr"))
    st = P.DeviceStepper(dm, P.RhsConfig(volume_flux="kennedy_gruber", surface_flux="llf", kernel="reference"),
                         P.SSPRK43)
    got = st.step(u_dev, dt).cpu().numpy()
    n_diff = int(np.count_nonzero(got != want))
    fast = P.DeviceStepper(dm, P.RhsConfig(volume_flux="kennedy_gruber", surface_flux="llf", kernel="batched"),
                           P.SSPRK43).step(u_dev, dt).cpu().numpy()
    e_fast = _rel(fast, want, float(np.abs(want).max()))
    _log({"case": "cfg4 SSPRK43 step (KG+llf, dt=1e-4), whole mesh", "faithful_bitwise": n_diff == 0,
          "fast_rel_max_u": e_fast})
    assert n_diff == 0, n_diff
    assert e_fast <= 1e-13
