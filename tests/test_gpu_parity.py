"""GPU parity: the sm_100a kernels (through the C ABI) against the oracle and
the reference's golden outputs.

Bars (written in each test):
* kernel="reference" (FAITHFUL) is BITWISE equal to the oracle built with the
  correctly rounded log (liboracle_cr.so), which is itself bitwise equal to
  the reference except where glibc's log misrounds; against the reference's
  own outputs du must agree to <= 1e-12 relative in max norm (literal
  north-star bar).
* kernel="batched" (FAST) volume integral: max|VOL - VOL_ref| <= 1e-12 max|VOL_ref|;
  full RHS: max|du - du_ref| <= 1e-12 max(max|VOL_ref|, max|SURF_ref|)
  (cancellation-aware bar).
"""

import numpy as np
import pytest

from oracle import oracle
from tests import golden_io as G

pytestmark = pytest.mark.gpu


def _pkg():
    import paper_2112_10517_b200 as P

    return P


def _rel(a, b, scale=None):
    scale = np.abs(b).max() if scale is None else scale
    return np.abs(a - b).max() / max(scale, 1e-300)


# ---------------------------------------------------------------- FAITHFUL


@pytest.mark.parametrize("name", G.CASES)
def test_faithful_volume_bitwise(name):
    P = _pkg()
    c = G.case(name)
    setup = G.golden_setup(name)
    for key in c:
        if not key.startswith("vol_"):
            continue
        _, state, flux, pre = key.split("_", 3)
        u = c["u_" + state]
        got = P.mesh_fluxdiff_volume(u, setup, P.RhsConfig(volume_flux=flux, precompute=pre, kernel="reference"))
        want = oracle.volume(u, setup, flux, pre, variant="cr")
        assert np.array_equal(got, want), key
        assert _rel(got, c[key]) <= 1e-13, key  # vs the reference's own bits


@pytest.mark.parametrize("name", G.CASES)
def test_faithful_surface_bitwise(name):
    P = _pkg()
    c = G.case(name)
    setup = G.golden_setup(name)
    for key in c:
        if not key.startswith("surf_"):
            continue
        _, state, flux = key.split("_", 2)
        u = c["u_" + state]
        got = P.surface_terms(u, setup, flux)
        want = oracle.surface(u, setup, flux, variant="cr")
        assert np.array_equal(got, want), key
        if flux != "ranocha":  # no log in the other surface fluxes: reference bits
            assert np.array_equal(got, c[key]), key


@pytest.mark.parametrize("name", G.CASES)
def test_faithful_rhs_bitwise(name):
    P = _pkg()
    c = G.case(name)
    setup = G.golden_setup(name)
    for key in c:
        if not key.startswith("rhs_"):
            continue
        parts = key.split("_")
        state, vf, sf = parts[1], parts[2], parts[3]
        pre = "primitives_and_logs" if key.endswith("_logs") else "none"
        u = c["u_" + state]
        got = P.rhs(u, setup, P.RhsConfig(volume_flux=vf, surface_flux=sf, precompute=pre, kernel="reference"))
        assert np.array_equal(got, oracle.rhs(u, setup, vf, sf, pre, variant="cr")), key
        assert _rel(got, c[key]) <= 1e-12, key  # literal du bar vs the reference


@pytest.mark.parametrize("vf", ["kennedy_gruber", "chandrashekar"])
@pytest.mark.parametrize("name", ["c2d_curv_p3", "c3d_cart_p3", "c3d_curv_p4"])
def test_faithful_unpinned_fluxes_match_oracle(name, vf):
    P = _pkg()
    c = G.case(name)
    setup = G.golden_setup(name)
    u = c["u_rand"]
    got = P.rhs(u, setup, P.RhsConfig(volume_flux=vf, surface_flux="llf", kernel="reference"))
    assert np.array_equal(got, oracle.rhs(u, setup, vf, "llf", variant="cr"))


def test_cfg1_faithful_bitwise_and_literal_du():
    P = _pkg()
    from paper_2112_10517_b200 import workloads

    g = G.config(1)
    setup, u, _ = workloads.build(1, op=G.golden_operator(3))
    du = P.rhs(u, setup, P.RhsConfig(volume_flux="ranocha", surface_flux="llf", kernel="reference"))
    assert np.array_equal(du, oracle.rhs(u, setup, "ranocha", "llf", variant="cr"))
    assert _rel(du, g["du"]) <= 1e-12


# -------------------------------------------------------------------- FAST


@pytest.mark.parametrize("name", G.CASES)
def test_fast_volume_within_tolerance(name):
    P = _pkg()
    c = G.case(name)
    setup = G.golden_setup(name)
    for key in c:
        if not key.startswith("vol_") or not key.endswith("_none"):
            continue
        _, state, flux, _ = key.split("_", 3)
        u = c["u_" + state]
        for pre in ("none", "primitives_and_logs"):
            got = P.mesh_fluxdiff_volume(u, setup, P.RhsConfig(volume_flux=flux, precompute=pre, kernel="batched"))
            assert _rel(got, c[key]) <= 1e-12, (key, pre)


@pytest.mark.parametrize("name", G.CASES)
def test_fast_rhs_within_tolerance(name):
    P = _pkg()
    c = G.case(name)
    setup = G.golden_setup(name)
    for key in c:
        if not key.startswith("rhs_") or key.endswith("_logs"):
            continue
        parts = key.split("_")
        state, vf, sf = parts[1], parts[2], parts[3]
        u = c["u_" + state]
        vol = c.get("vol_%s_%s_none" % (state, vf))
        surf = c.get("surf_%s_%s" % (state, sf))
        scale = max(np.abs(vol).max(), np.abs(surf).max())
        for pre in ("none", "primitives_and_logs"):
            got = P.rhs(u, setup, P.RhsConfig(volume_flux=vf, surface_flux=sf, precompute=pre, kernel="batched"))
            assert _rel(got, c[key], scale) <= 1e-12, (key, pre)


# ----------------------------------------------------------- full-size cfgs


def test_cfg2_samples_and_checksum():
    """BASELINE cfg2 (16^3, N=3, Ranocha) at full size: sampled elements
    against the reference's scalar volume_fluxdiff, plus the whole-mesh
    checksum of the reference's batched VOL."""
    P = _pkg()
    from paper_2112_10517_b200 import workloads

    g = G.config(2)
    setup, u, _ = workloads.build(2, op=G.golden_operator(3))
    idx = g["elements"]
    for kernel, pre, key, tol in (
        ("reference", "none", "vol_ranocha", 1e-13),
        ("reference", "primitives_and_logs", "vol_ranocha_logs", 1e-13),
        ("batched", "primitives_and_logs", "vol_ranocha", 1e-12),
        ("batched", "none", "vol_ranocha", 1e-12),
    ):
        vol = P.mesh_fluxdiff_volume(u, setup, P.RhsConfig(volume_flux="ranocha", precompute=pre, kernel=kernel))
        assert _rel(vol[idx], g[key]) <= tol, (kernel, pre)
        s = np.abs(vol).sum(axis=(0, 1))
        assert np.all(np.abs(s - g["volb_ranocha_abs_sum"]) <= 1e-12 * g["volb_ranocha_abs_sum"]), (kernel, pre)


def test_cfg4_samples_curved():
    P = _pkg()
    from paper_2112_10517_b200 import workloads

    g = G.config(4)
    setup, u, _ = workloads.build(4, op=G.golden_operator(4))
    idx = g["elements"]
    for flux in ("ranocha", "shima"):
        ref = P.mesh_fluxdiff_volume(u, setup, P.RhsConfig(volume_flux=flux, kernel="reference"))
        assert _rel(ref[idx], g["vol_" + flux]) <= 1e-13
        fast = P.mesh_fluxdiff_volume(u, setup, P.RhsConfig(volume_flux=flux, kernel="batched"))
        assert _rel(fast[idx], g["vol_" + flux]) <= 1e-12


def test_cfg3_samples_n7():
    P = _pkg()
    from paper_2112_10517_b200 import workloads

    g = G.config(3)
    setup, u, _ = workloads.build(3, op=G.golden_operator(7))
    idx = g["elements"]
    ref = P.mesh_fluxdiff_volume(u, setup, P.RhsConfig(volume_flux="ranocha", kernel="reference"))
    assert _rel(ref[idx], g["vol_ranocha"]) <= 1e-13
    fast = P.mesh_fluxdiff_volume(u, setup, P.RhsConfig(volume_flux="ranocha", kernel="batched",
                                                        precompute="primitives_and_logs"))
    assert _rel(fast[idx], g["vol_ranocha"]) <= 1e-12
    # Chandrashekar (cfg3's named flux, unpinned): FAST vs FAITHFUL on the full mesh
    a = P.mesh_fluxdiff_volume(u, setup, P.RhsConfig(volume_flux="chandrashekar", kernel="reference"))
    b = P.mesh_fluxdiff_volume(u, setup, P.RhsConfig(volume_flux="chandrashekar", kernel="batched",
                                                     precompute="primitives_and_logs"))
    assert _rel(b, a) <= 1e-12


# ------------------------------------------------------------- properties


@pytest.mark.parametrize("vf", ["ranocha", "shima", "kennedy_gruber", "chandrashekar", "central"])
@pytest.mark.parametrize("kernel", ["reference", "batched"])
def test_free_stream_on_curved_mesh(vf, kernel):
    """A constant state stays constant on the warped mesh (metric identity)."""
    P = _pkg()
    from paper_2112_10517_b200 import workloads

    setup, _, _ = workloads.build(4, dims=(6, 6, 6))
    q = np.zeros((setup.n_elements, setup.n_nodes, 5))
    q[..., 0] = 1.3
    q[..., 1:4] = (0.1, -0.2, 0.3)
    q[..., 4] = 2.0
    u = P.prim2cons(q, setup.gas)
    cfg = P.RhsConfig(volume_flux=vf, surface_flux="llf", kernel=kernel)
    du = P.rhs(u, setup, cfg)
    vol = P.mesh_fluxdiff_volume(u, setup, cfg)
    # VOL and SURF are each O(max|VOL|) and cancel to roundoff of that size
    assert np.abs(du).max() <= 1e-13 * np.abs(vol).max()


@pytest.mark.parametrize("kernel", ["reference", "batched"])
def test_conservation_and_entropy_conservation(kernel):
    P = _pkg()
    setup = G.golden_setup("c3d_curv_p4")
    from paper_2112_10517_b200 import workloads

    setup, u, _ = workloads.build(4, dims=(4, 4, 4))
    wbar = np.ones(1)
    for _ in range(3):
        wbar = np.kron(wbar, setup.op.weights)
    du = P.rhs(u, setup, P.RhsConfig(volume_flux="ranocha", surface_flux="ranocha", kernel=kernel))
    weights = wbar[None, :] * setup.metrics.jac
    totals = np.sum(weights[..., None] * du, axis=(0, 1))
    scale = np.sum(np.abs(weights[..., None] * du), axis=(0, 1))
    assert np.all(np.abs(totals) <= 1e-12 * scale)
    _, normalized = P.entropy_rate(u, du, setup)
    assert abs(normalized) < 1e-12


def test_counters_match_reference_contract():
    P = _pkg()
    c = G.case("c3d_curv_p2")
    setup = G.golden_setup("c3d_curv_p2")
    cnt = P.FluxCounter()
    P.rhs(c["u_rand"], setup, P.RhsConfig(volume_flux="ranocha", surface_flux="llf", kernel="batched"), counter=cnt)
    assert (cnt.two_point_evals, cnt.one_point_evals, cnt.logmean_evals) == tuple(c["counts_rand_ranocha_llf"])


def test_gate_names_first_bad_node():
    P = _pkg()
    c = G.case("c2d_cart_p3")
    setup = G.golden_setup("c2d_cart_p3")
    u = c["u_rand"].copy()
    u[1, 2, -1] = 0.01
    u[4, 0, 0] = -1.0
    with pytest.raises(P.AdmissibilityError, match="element 1, node 2"):
        P.rhs(u, setup, P.RhsConfig(kernel="batched"))
    with pytest.raises(P.AdmissibilityError, match="cons2prim"):
        P.mesh_fluxdiff_volume(u, setup, P.RhsConfig(kernel="batched"))


@pytest.mark.parametrize("pre", ["none", "primitives_and_logs"])
@pytest.mark.parametrize("vf", ["ranocha", "chandrashekar"])
def test_fast_log_means_over_wide_ranges(vf, pre):
    """FAST log means (branch-free log_fast, log-difference series test, the
    2x coth x series) on states spanning 120 decades between elements and up
    to 1e3 contrast inside an element,
    against the FAITHFUL arithmetic of the oracle: per-element relative
    max-norm difference <= 1e-12."""
    P = _pkg()
    from paper_2112_10517_b200 import workloads

    setup, u, _ = workloads.build(2, dims=(4, 4, 4))
    rng = np.random.default_rng(11)
    ne, nn = u.shape[:2]
    scale = 10.0 ** rng.uniform(-60, 60, size=(ne, 1))
    contrast = np.where(rng.random((ne, 1)) < 0.5, 10.0 ** rng.uniform(-1.5, 1.5, size=(ne, nn)),
                        rng.uniform(0.9999, 1.0001, size=(ne, nn)))  # also the series branch
    c = scale * contrast
    u = u * c[..., None]  # velocity unchanged, rho, p scaled
    got = P.mesh_fluxdiff_volume(u, setup, P.RhsConfig(volume_flux=vf, precompute=pre, kernel="batched"))
    want = oracle.volume(u, setup, vf, pre, variant="cr")
    err = np.abs(got - want).max(axis=(1, 2)) / np.abs(want).max(axis=(1, 2))
    assert err.max() <= 1e-12, err.max()


@pytest.mark.parametrize("kernel", ["reference", "batched"])
def test_pinned_pipeline_matches_device_path(kernel):
    """Pinned host state -> chunked H2D / fdg_volume_range / D2H pipeline:
    bitwise equal to one whole-mesh launch (the volume integral is element-local)."""
    P = _pkg()
    import torch
    from paper_2112_10517_b200 import workloads

    setup, u, _ = workloads.build(2, dims=(16, 16, 12))  # 7.9 MB: several 2 MB chunks
    cfg = P.RhsConfig(volume_flux="ranocha", precompute="primitives_and_logs", kernel=kernel)
    want = P.mesh_fluxdiff_volume(torch.as_tensor(u, device="cuda"), setup, cfg).cpu().numpy()
    u_pin = torch.from_numpy(u).pin_memory()
    out_pin = torch.full(u.shape, np.nan, dtype=torch.float64).pin_memory()
    dm = P.device.device_mesh_for(setup)
    before = P._native.launch_count()
    got = P.mesh_fluxdiff_volume(u_pin, setup, cfg, out=out_pin)
    assert got.data_ptr() == out_pin.data_ptr()
    assert P._native.launch_count() - before > 1  # several element chunks
    assert np.array_equal(out_pin.numpy(), want)
    got2 = P.mesh_fluxdiff_volume(u_pin, setup, cfg)  # no out: fresh host tensor
    assert np.array_equal(got2.numpy(), want)
    # explicit ranges tile the mesh
    ud = torch.as_tensor(u, device="cuda")
    vd = torch.full_like(ud, np.nan)
    for lo, hi in ((0, 1), (1, 100), (100, 100), (100, dm.n_elem)):
        dm.volume_range(ud, cfg.scheme(), vd, lo, hi)
    assert np.array_equal(vd.cpu().numpy(), want)
    with pytest.raises(Exception, match="bad range"):
        dm.volume_range(ud, cfg.scheme(), vd, 5, dm.n_elem + 1)
    bad = u.copy()
    bad[300, 3, 0] = -1.0
    with pytest.raises(P.AdmissibilityError, match="cons2prim"):
        P.mesh_fluxdiff_volume(torch.from_numpy(bad).pin_memory(), setup, cfg, out=out_pin)


@pytest.mark.parametrize("cfgno, dims, vf", [(2, (5, 3, 3), "ranocha"), (4, (3, 3, 5), "kennedy_gruber")])
@pytest.mark.parametrize("kernel", ["reference", "batched"])
def test_bulk_copy_and_fallback_paths_agree(cfgno, dims, vf, kernel):
    """The element kernel stages each batch by one TMA bulk copy and writes VOL /
    du by one bulk store when the device buffers are 16-byte aligned, and falls
    back to per-thread copies otherwise (and for ragged batches of odd size):
    both give bitwise identical volume integrals and RHS."""
    P = _pkg()
    import torch
    from paper_2112_10517_b200 import workloads

    setup, u, _ = workloads.build(cfgno, dims=dims)  # odd element counts: ragged last batches
    cfg = P.RhsConfig(volume_flux=vf, surface_flux="llf", kernel=kernel)
    scheme = cfg.scheme()
    dm = P.device.device_mesh_for(setup)
    n = u.size
    ua = torch.as_tensor(u, device="cuda")
    raw_u = torch.empty(n + 1, dtype=torch.float64, device="cuda")
    raw_o = torch.empty(n + 1, dtype=torch.float64, device="cuda")
    um = raw_u[1:].view(u.shape)  # 8-byte aligned only: the per-thread paths
    um.copy_(ua)
    om = raw_o[1:].view(u.shape)
    assert um.data_ptr() % 16 == 8 and om.data_ptr() % 16 == 8
    for call in (dm.volume, dm.rhs):
        oa = torch.full_like(ua, np.nan)
        om.fill_(np.nan)
        call(ua, scheme, out=oa)
        call(um, scheme, out=om)
        torch.cuda.synchronize()
        assert torch.equal(oa, om), call.__name__


# ------------------------------------------------------------ time stepping


@pytest.mark.parametrize("name", ["c2d_cart_p3", "c3d_curv_p2", "c3d_curv_p4"])
def test_device_rk54_faithful_bitwise(name):
    import torch

    P = _pkg()
    from paper_2112_10517_b200.device import device_mesh_for

    c = G.case(name)
    setup = G.golden_setup(name)
    cfg = P.RhsConfig(volume_flux="ranocha", surface_flux="llf", kernel="reference")
    dm = device_mesh_for(setup)
    stepper = P.DeviceStepper(dm, cfg, P.RK54)
    dt = float(c["rk54_dt"])
    for state in G.states(name):
        u = c["u_" + state]
        got = stepper.step(torch.as_tensor(u, device="cuda"), dt).cpu().numpy()
        want = oracle.rk54_step(u, dt, lambda v: oracle.rhs(v, setup, "ranocha", "llf", variant="cr"))
        assert np.array_equal(got, want)
        assert _rel(got, c["rk54_" + state]) <= 1e-14


def test_device_ssprk43_faithful_bitwise():
    import torch

    P = _pkg()
    from paper_2112_10517_b200.device import device_mesh_for

    c = G.case("c3d_curv_p4")
    setup = G.golden_setup("c3d_curv_p4")
    cfg = P.RhsConfig(volume_flux="kennedy_gruber", surface_flux="llf", kernel="reference")
    stepper = P.DeviceStepper(device_mesh_for(setup), cfg, P.SSPRK43)
    u = c["u_wave"]
    dt = 1e-3
    got = stepper.step(torch.as_tensor(u, device="cuda"), dt).cpu().numpy()
    want = oracle.ssprk43_step(u, dt, lambda v: oracle.rhs(v, setup, "kennedy_gruber", "llf", variant="cr"))
    assert np.array_equal(got, want)


def test_device_stepper_graph_and_divergence():
    import torch

    P = _pkg()
    from paper_2112_10517_b200.device import device_mesh_for

    c = G.case("c2d_cart_p3")
    setup = G.golden_setup("c2d_cart_p3")
    cfg = P.RhsConfig(volume_flux="ranocha", surface_flux="llf", kernel="batched")
    st = P.DeviceStepper(device_mesh_for(setup), cfg, P.RK54)
    u = torch.as_tensor(c["u_rand"], device="cuda")
    plain = st.step(u, 1e-3).clone()
    out = st.capture(u, 1e-3)
    st.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, plain)
    bad = u.clone()
    bad[2, 3, 0] = -1.0
    with pytest.raises(P.AdmissibilityError, match="element 2, node 3"):
        st.step(bad, 1e-3)


# --------------------------------------------------- partitioned device path


@pytest.mark.parametrize("world,dims,p,amp", [(2, (4, 2, 3), 3, 0.0), (3, (6, 2, 2), 4, -0.1), (2, (4, 5), 3, 0.1),
                                          (2, (8, 3, 5), 4, -0.1), (3, (9, 4, 3), 3, 0.0)])
@pytest.mark.parametrize("kernel", ["reference", "batched"])
def test_slab_partition_on_device_bitwise(world, dims, p, amp, kernel):
    """The ghost-slot path of the element kernel: W slabs on one GPU, face
    traces packed with fdg_pack_faces and handed over by device copies (the
    NCCL exchange moves exactly these buffers), RHS of every slab bitwise equal
    to the single-domain RHS."""
    import torch

    P = _pkg()
    from paper_2112_10517_b200.device import DeviceMesh
    from paper_2112_10517_b200.parallel import slab_partition

    gas = P.GasParams(1.4)
    setup = P.build_setup(P.build_mesh(dims, bounds=(-1.0, 1.0), amplitude=amp), P.lgl_operator(p), gas)
    rng = np.random.default_rng(3)
    q = np.empty((setup.n_elements, setup.n_nodes, setup.d + 2))
    q[..., 0] = 1.0 + 0.3 * rng.random(q.shape[:2])
    q[..., 1 : setup.d + 1] = 0.3 * (rng.random(q.shape[:2] + (setup.d,)) - 0.5)
    q[..., -1] = 1.0 + 0.3 * rng.random(q.shape[:2])
    u = P.prim2cons(q, gas)
    cfg = P.RhsConfig(volume_flux="ranocha", surface_flux="llf", kernel=kernel)
    want = P.rhs(u, setup, cfg)
    parts = [slab_partition(setup, r, world) for r in range(world)]
    dms = [DeviceMesh(setup, partition=pt) for pt in parts]
    us = [torch.as_tensor(np.ascontiguousarray(u[pt["lo"] : pt["hi"]]), device="cuda") for pt in parts]
    fn = (p + 1) ** (setup.d - 1)
    first, last = [], []
    for dm, pt, ul in zip(dms, parts, us):
        F = pt["plane"]
        a = torch.empty((F, fn, setup.d + 2), dtype=torch.float64, device="cuda")
        b = torch.empty_like(a)
        dm.pack_faces(ul, torch.as_tensor(pt["send_first"], device="cuda"), 0, 0, a)
        dm.pack_faces(ul, torch.as_tensor(pt["send_last"], device="cuda"), 0, 1, b)
        first.append(a)
        last.append(b)
    for r, (dm, pt, ul) in enumerate(zip(dms, parts, us)):
        ghost = torch.cat([first[(r + 1) % world], last[(r - 1) % world]])
        got = dm.rhs(ul, cfg.scheme(), ghost_u=ghost).cpu().numpy()
        assert np.array_equal(got, want[pt["lo"] : pt["hi"]]), r
        # the overlap split: interior range WITHOUT ghosts, then the boundary planes
        F, n = pt["plane"], pt["hi"] - pt["lo"]
        out = torch.full_like(ul, float("nan"))
        if n > 2 * F:
            dm.rhs(ul, cfg.scheme(), out=out, ghost_u=None, lo=F, hi=n - F)
            dm.rhs(ul, cfg.scheme(), out=out, ghost_u=ghost, ranges=[(0, F), (n - F, n)])
        else:
            dm.rhs(ul, cfg.scheme(), out=out, ghost_u=ghost, lo=0, hi=n)
        assert np.array_equal(out.cpu().numpy(), want[pt["lo"] : pt["hi"]]), ("split", r)


# ---------------------------------------------------------------- diagnostics


def _diag_golden():
    return dict(np.load(G.os.path.join(G.GOLDEN, "diagnostics.npz")))


@pytest.mark.parametrize("name", G.CASES)
def test_device_diagnostics_match_reference(name):
    """fdg_diagnostic (through the public conserved_totals / entropy_rate /
    error_norm_l2 / stable_dt) against the reference's own outputs. Bars:
    sums <= 1e-13 relative to the largest component; the entropy total
    within 1e-13 of its absolute scale; dt <= 1e-14 relative (different
    summation order, same per-node arithmetic)."""
    P = _pkg()
    g = _diag_golden()
    c = G.case(name)
    setup = G.golden_setup(name)
    for s in G.states(name):
        u = c["u_" + s]
        want = g["cons_%s_%s" % (name, s)]
        got = P.conserved_totals(u, setup)
        assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max(), s
        dt_ref = float(g["dt_%s_%s" % (name, s)])
        dt = P.stable_dt(u, None, setup.metrics, setup.gas, setup.op.degree, P.StepController(0.5), setup=setup)
        assert abs(dt - dt_ref) <= 1e-14 * dt_ref, (s, dt, dt_ref)
        for vf, sf in (("ranocha", "ranocha"), ("ranocha", "llf")):
            key = "ent_%s_%s_%s_%s" % (name, s, vf, sf)
            if key not in g:
                continue
            total, norm = P.entropy_rate(u, c["rhs_%s_%s_%s" % (s, vf, sf)], setup)
            t_ref, n_ref = g[key]
            scale = abs(t_ref / n_ref) if n_ref != 0.0 else 0.0
            assert abs(total - t_ref) <= 1e-13 * max(scale, 1e-300), key
    u_exact = c["u_wave"] if "u_wave" in c else 1.01 * c["u_rand"]
    want = g["err_%s" % name]
    got = P.error_norm_l2(c["u_rand"], u_exact, setup)
    assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max()


@pytest.mark.parametrize("k,dims", [(2, None), (4, (16, 16, 16))])
def test_device_diagnostics_full_size(k, dims):
    """BASELINE cfg2 (16^3 Cartesian, full size) and cfg4's curved map (16^3) on the device:
    totals vs a correctly rounded sum (<= 1e-14 of the absolute sum), dt vs
    the numpy oracle (<= 1e-14), bitwise-repeatable calls, and the
    size-independent properties: the RHS conserves every variable and the
    entropy-conservative flux pair produces no entropy (both <= 1e-12 of
    their absolute scales)."""
    import torch

    P = _pkg()
    from paper_2112_10517_b200 import workloads
    from paper_2112_10517_b200.device import DIAG_CONSERVED, DIAG_ENTROPY, device_mesh_for

    import math

    setup, u, _ = workloads.build(k, dims=dims)
    # the reference sums over the node axes sequentially (numpy reduces a
    # non-contiguous axis without pairwise blocking): its error grows like
    # n eps. Pin the device to a correctly rounded sum (math.fsum, <= 1e-14)
    # and the oracle to it within n eps.
    terms = oracle._wbar_jac(setup)[..., None] * u
    exact = np.array([math.fsum(terms[..., v].ravel()) for v in range(u.shape[-1])])
    absum = np.abs(terms).sum(axis=(0, 1))
    got = P.conserved_totals(u, setup)
    assert np.all(np.abs(got - exact) <= 1e-14 * absum)
    want = oracle.conserved_totals(u, setup)
    assert np.all(np.abs(want - exact) <= terms.shape[0] * terms.shape[1] * 2.3e-16 * absum)
    dt = P.stable_dt(u, None, setup.metrics, setup.gas, setup.op.degree, P.StepController(0.5), setup=setup)
    assert abs(dt - oracle.stable_dt(u, setup)) <= 1e-14 * dt
    ud = torch.as_tensor(u, device="cuda")
    cfg = P.RhsConfig(volume_flux="ranocha", surface_flux="ranocha", kernel="batched")
    du = P.rhs(ud, setup, cfg)
    dm = device_mesh_for(setup)
    a = dm.diagnostic(DIAG_CONSERVED, du)
    b = dm.diagnostic(DIAG_CONSERVED, du)
    assert torch.equal(a, b)
    wbar_j = oracle._wbar_jac(setup)
    du_h = du.cpu().numpy()
    scale = np.sum(np.abs(wbar_j[..., None] * du_h), axis=(0, 1))
    assert np.all(np.abs(a.cpu().numpy()) <= 1e-12 * scale)
    total, scale = (float(x) for x in dm.diagnostic(DIAG_ENTROPY, ud, du).cpu())  # raw sums
    assert abs(total) < 1e-12 * scale
    assert abs(total - oracle.entropy_rate(u, du_h, setup)[0]) <= 1e-13 * scale


def test_surface_accumulates_into_numpy_out():
    """mesh_surface with a numpy state AND a non-zero numpy accumulator: both
    are staged through distinct pinned slots (a shared slot let the second
    host copy overwrite the first before its H2D copy ran). FAITHFUL bits."""
    P = _pkg()
    c = G.case("c3d_curv_p4")
    setup = G.golden_setup("c3d_curv_p4")
    u = c["u_rand"]
    acc0 = np.random.default_rng(3).standard_normal(u.shape)
    got = P.mesh_surface(u, setup, "llf", acc0.copy(), kernel="reference")
    want = oracle.surface(u, setup, "llf", out=acc0.copy(), variant="cr")
    assert np.array_equal(got, want)


# ---------------------------------------------------------------- device geometry


@pytest.mark.parametrize("name", G.CASES)
def test_device_geometry_matches_reference(name):
    """fdg_build_geometry (build_setup(device="cuda")) against the reference's
    recorded coordinates and curl-form metrics. Bars: coords <= 1e-15 of
    max|x|; Ja and J <= 1e-13 of their max norms (summation order of the
    derivative sums and the device sin differ from numpy's)."""
    import torch

    P = _pkg()
    c = G.case(name)
    dims = tuple(int(x) for x in c["dims"])
    bounds = tuple(float(x) for x in c["bounds"])
    mesh = P.build_mesh(dims, bounds=bounds, amplitude=float(c["amplitude"]))
    op = G.golden_operator(int(c["p"]))
    setup = P.build_setup(mesh, op, P.GasParams(1.4), device="cuda")
    x = setup.coords.cpu().numpy()
    assert np.abs(x - c["coords"]).max() <= 1e-15 * np.abs(c["coords"]).max()
    if bool(c["cartesian"]):
        assert setup.metrics.cartesian
        return
    assert isinstance(setup.metrics.ja, torch.Tensor) and setup.metrics.ja.is_cuda
    ja = setup.metrics.ja.cpu().numpy()
    jac = setup.metrics.jac.cpu().numpy()
    assert np.abs(ja - c["ja"]).max() <= 1e-13 * np.abs(c["ja"]).max()
    assert np.abs(jac - c["jac"]).max() <= 1e-13 * np.abs(c["jac"]).max()


def test_device_geometry_rhs_cfg4():
    """BASELINE cfg4's warped map (24^3 here, N=4, Kennedy-Gruber + Rusanov):
    the metrics agree to 1e-12 of max|Ja| (curl-form rounding noise), the
    RHS on the device-built geometry equals the RHS on the host-built one
    within the RHS bar (1e-12 of max(|VOL|, |du|)), and the device DT /
    totals agree (1e-13)."""
    import torch

    P = _pkg()
    from paper_2112_10517_b200 import workloads

    setup_h, u, cfg = workloads.build(4, dims=(24, 24, 24))
    setup_d = P.build_setup(setup_h.mesh, setup_h.op, setup_h.gas, device="cuda")
    assert np.abs(setup_d.coords.cpu().numpy() - setup_h.coords).max() <= 1e-15
    ja_h = np.asarray(setup_h.metrics.ja)
    # curl form: each entry is a difference of derivatives of products
    # (x_l - mean) d x_m, whose rounding noise (~eps per term, both paths)
    # is ~1e-15 absolute here against entries of 1.7e-3 -> bar 1e-12
    assert np.abs(setup_d.metrics.ja.cpu().numpy() - ja_h).max() <= 1e-12 * np.abs(ja_h).max()
    ud = torch.as_tensor(u, device="cuda")
    du_h = P.rhs(ud, setup_h, cfg).cpu().numpy()
    du_d = P.rhs(ud, setup_d, cfg).cpu().numpy()
    vol = P.mesh_fluxdiff_volume(ud, setup_h, cfg).cpu().numpy()
    assert np.abs(du_d - du_h).max() <= 1e-12 * max(np.abs(vol).max(), np.abs(du_h).max())
    t_h = P.conserved_totals(ud, setup_h)
    t_d = P.conserved_totals(ud, setup_d)
    assert np.all(np.abs(t_d - t_h) <= 1e-13 * np.abs(t_h).max())
    sc = P.StepController(0.5)
    dt_h = P.stable_dt(ud, None, None, setup_h.gas, 4, sc, setup=setup_h)
    dt_d = P.stable_dt(ud, None, None, setup_d.gas, 4, sc, setup=setup_d)
    assert abs(dt_d - dt_h) <= 1e-13 * dt_h


@pytest.mark.parametrize("k,dims,tile", [(5, (8, 8, 8), "2,2"), (4, (8, 4, 6), "4,2"), (2, (4, 8, 8), "2,4")])
def test_tiled_traversal_is_bitwise(monkeypatch, k, dims, tile):
    """fdg_mesh_set_traversal only reorders which CTA takes which element
    rows: VOL, RHS and a fused RK stage are BITWISE those of the natural
    order (Cartesian and curved meshes)."""
    import torch

    P = _pkg()
    from paper_2112_10517_b200 import workloads
    from paper_2112_10517_b200.device import device_mesh_for

    outs = []
    for env in ("0", tile):
        monkeypatch.setenv("FDG_TILE", env)
        setup, u, cfg = workloads.build(k, dims=dims)
        dm = device_mesh_for(setup)
        assert (dm.row_order is None) == (env == "0")
        ud = torch.as_tensor(u, device="cuda")
        vol = P.mesh_fluxdiff_volume(ud, setup, cfg)
        du = P.rhs(ud, setup, cfg)
        outs.append((vol.cpu(), du.cpu()))
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])


def test_device_stepper_stable_dt():
    """DeviceStepper.stable_dt (device DT reduction) equals the oracle's
    stable_dt (<= 1e-14 relative) on a curved cfg4-map mesh, and a step with
    it stays finite."""
    import torch

    P = _pkg()
    from paper_2112_10517_b200 import workloads
    from paper_2112_10517_b200.device import device_mesh_for

    setup, u, cfg = workloads.build(4, dims=(8, 8, 8))
    dm = device_mesh_for(setup)
    st = P.DeviceStepper(dm, cfg, P.SSPRK43)
    ud = torch.as_tensor(u, device="cuda")
    dt = st.stable_dt(ud, P.StepController(0.5))
    want = oracle.stable_dt(u, setup)
    assert abs(dt - want) <= 1e-14 * want
    out = st.step(ud, dt)
    assert bool(torch.isfinite(out).all())
