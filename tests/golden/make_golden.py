"""Generate the golden fixtures under tests/golden/ from the REFERENCE package.

This script is the only place that imports the reference (`fluxdg`, read-only
at /root/reference/pkg/src). It runs in the build container, never on the GPU
box; its outputs (small .npz files) are committed so the GPU-side tests and the
oracle pins can run without /root/reference.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--big]

What is recorded (all float64, bitwise as the reference produced them):

* operators.npz   -- lgl_operator(p) nodes/weights/D/boundary_interp and
                     build_dsplit(op).matrix for p = 1..15
                     (reference operators.py:169-217)
* case_<name>.npz -- small meshes: coords, ja, jac, face_ja, neighbours
                     (geometry.py:142-329), seeded states, and the outputs of
                     - volume_fluxdiff per element        (discretization.py:267-323)
                     - surface_terms from zeros           (discretization.py:681-788)
                     - rhs(kernel="reference"/"batched")  (discretization.py:896-949)
                     - batched.mesh_fluxdiff_volume / mesh_surface (batched.py:450-544)
                     - rk_step (RK54)                     (timeint.py:149-163)
                     - FluxCounter totals                 (fluxes.py:37-101)
* cfg<k>.npz      -- BASELINE.json configs at full size: sampled-element
                     scalar VOL + state/geometry of those elements, and
                     full-mesh checksums of the batched VOL (with --big).
* cfg4_rhs.npz    -- (--only cfg4rhs) the reference's batched rhs / VOL /
                     SURF on the full 48^3 curved cfg4 mesh: sampled rows
                     plus whole-mesh maxima
* cfg5.npz        -- (--only cfg5) 128^3 noisy-wave elements and their
                     scalar volume_fluxdiff (Ranocha, Shima)
"""

import argparse
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

import fluxdg  # noqa: E402
from fluxdg import (  # noqa: E402
    FluxCounter,
    GasParams,
    RhsConfig,
    build_mesh,
    build_setup,
    count_guard,
    lgl_operator,
    prim2cons,
    rhs,
)
from fluxdg import batched as B  # noqa: E402
from fluxdg.discretization import (  # noqa: E402
    precompute_element_data,
    surface_terms,
    volume_fluxdiff,
)
from fluxdg.geometry import element_metrics  # noqa: E402
from fluxdg.operators import build_dsplit  # noqa: E402
from fluxdg.timeint import rk_step  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
GAS = GasParams(1.4)


def random_field(setup, seed, amp):
    """Same recipe as the reference's tests/conftest.py random_field."""
    rng = np.random.default_rng(seed)
    d = setup.d
    n = setup.n_elements * setup.n_nodes
    q = np.empty((n, d + 2))
    q[:, 0] = 1.0 + amp * rng.random(n)
    q[:, 1 : d + 1] = amp * (rng.random((n, d)) - 0.5)
    q[:, d + 1] = 1.0 + amp * rng.random(n)
    u = prim2cons(q, GAS)
    return np.ascontiguousarray(u.reshape(setup.n_elements, setup.n_nodes, d + 2))


def wave_field(setup):
    """BASELINE cfg1/cfg2/cfg4 density wave: rho = 1 + 0.98 sin(pi * sum x),
    v = (0.1, 0.2[, 0.3]), p = 20."""
    x = setup.coords
    d = setup.d
    q = np.empty(x.shape[:-1] + (d + 2,))
    q[..., 0] = 1.0 + 0.98 * np.sin(np.pi * x.sum(-1))
    for i in range(d):
        q[..., 1 + i] = (0.1, 0.2, 0.3)[i]
    q[..., d + 1] = 20.0
    return prim2cons(q, GAS)


def scalar_volume(u, setup, flux, pre_mode):
    out = np.empty_like(u)
    for e in range(setup.n_elements):
        terms = element_metrics(setup.metrics, e)
        pre = precompute_element_data(u[e], GAS, pre_mode) if pre_mode != "none" else None
        out[e] = volume_fluxdiff(u[e], setup.dsplit, terms, flux, GAS, pre)
    return out


def counts(u, setup, cfg):
    c = FluxCounter()
    with count_guard(c):
        rhs(u, setup, cfg)
    return np.array([c.two_point_evals, c.one_point_evals, c.logmean_evals], dtype=np.int64)


CASES = {
    # name: (dims, p, amplitude, bounds)
    "c2d_cart_p3": ((3, 3), 3, 0.0, (-1.0, 1.0)),
    "c2d_curv_p3": ((3, 3), 3, 0.12, (-5.0, 5.0)),
    "c2d_curv_p5": ((2, 3), 5, 0.12, (-5.0, 5.0)),
    "c2d_cart_p1": ((4, 3), 1, 0.0, (-1.0, 1.0)),
    "c2d_dim1_p3": ((1, 4), 3, 0.0, (-1.0, 1.0)),
    "c3d_cart_p3": ((2, 2, 3), 3, 0.0, (-1.0, 1.0)),
    "c3d_curv_p4": ((3, 2, 2), 4, -0.1, (-1.0, 1.0)),
    "c3d_curv_p2": ((2, 2, 2), 2, 0.08, (-5.0, 5.0)),
    "c3d_cart_p7": ((2, 1, 2), 7, 0.0, (-1.0, 1.0)),
    "c3d_curv_p6": ((1, 2, 2), 6, 0.05, (-1.0, 1.0)),
}

# (volume flux, surface flux) pairs recorded through rhs(kernel="reference")
RHS_PAIRS = [
    ("ranocha", "llf"),
    ("ranocha", "ranocha"),
    ("shima", "llf"),
    ("shima", "hll"),
    ("central", "central"),
    ("ranocha", "shima"),
]


def make_operators():
    out = {}
    for p in range(1, 16):
        op = lgl_operator(p)
        out["nodes_%d" % p] = op.nodes
        out["weights_%d" % p] = op.weights
        out["D_%d" % p] = op.D
        out["R_%d" % p] = op.boundary_interp
        out["dsplit_%d" % p] = build_dsplit(op).matrix
    np.savez_compressed(os.path.join(HERE, "operators.npz"), **out)


def make_case(name, dims, p, amp, bounds):
    t0 = time.time()
    mesh = build_mesh(dims, bounds=bounds, amplitude=amp)
    setup = build_setup(mesh, lgl_operator(p), GAS)
    d = setup.d
    rec = {
        "dims": np.array(dims),
        "p": np.array(p),
        "amplitude": np.array(amp),
        "bounds": np.array(bounds),
        "coords": setup.coords,
        "ja": setup.metrics.ja,
        "jac": setup.metrics.jac,
        "cartesian": np.array(setup.metrics.cartesian),
    }
    for n in range(d):
        rec["face_ja_%d" % n] = setup.metrics.face_ja[n]
        rec["plus_%d" % n] = setup.plus_neighbor[n]
    big = p >= 6
    states = {"rand": random_field(setup, seed=5, amp=0.5)}
    if not big:
        states["wave"] = wave_field(setup)
    for sname, u in states.items():
        rec["u_%s" % sname] = u
        fluxes = ("shima", "ranocha", "central") if not big else ("ranocha", "shima")
        for flux in fluxes:
            rec["vol_%s_%s_none" % (sname, flux)] = scalar_volume(u, setup, flux, "none")
            rec["volb_%s_%s" % (sname, flux)] = B.mesh_fluxdiff_volume(
                u, setup, RhsConfig(volume_flux=flux)
            )
        if not big:
            rec["vol_%s_ranocha_primitives_and_logs" % sname] = scalar_volume(
                u, setup, "ranocha", "primitives_and_logs"
            )
            rec["vol_%s_central_primitives" % sname] = scalar_volume(
                u, setup, "central", "primitives"
            )
            rec["volb_%s_ranocha_logs" % sname] = B.mesh_fluxdiff_volume(
                u, setup, RhsConfig(volume_flux="ranocha", precompute="primitives_and_logs")
            )
        surfs = ("llf", "ranocha", "shima", "hll", "central") if not big else ("llf",)
        for sf in surfs:
            rec["surf_%s_%s" % (sname, sf)] = surface_terms(u, setup, sf, out=np.zeros_like(u))
            rec["surfb_%s_%s" % (sname, sf)] = B.mesh_surface(u, setup, sf, np.zeros_like(u))
        pairs = RHS_PAIRS if not big else [("ranocha", "llf")]
        for vf, sf in pairs:
            rec["rhs_%s_%s_%s" % (sname, vf, sf)] = rhs(
                u, setup, RhsConfig(volume_flux=vf, surface_flux=sf)
            )
            rec["rhsb_%s_%s_%s" % (sname, vf, sf)] = rhs(
                u, setup, RhsConfig(volume_flux=vf, surface_flux=sf, kernel="batched")
            )
        if not big:
            rec["rhs_%s_ranocha_llf_logs" % sname] = rhs(
                u,
                setup,
                RhsConfig(volume_flux="ranocha", surface_flux="llf", precompute="primitives_and_logs"),
            )
        rec["counts_%s_ranocha_llf" % sname] = counts(
            u, setup, RhsConfig(volume_flux="ranocha", surface_flux="llf")
        )
        rec["counts_%s_shima_llf" % sname] = counts(
            u, setup, RhsConfig(volume_flux="shima", surface_flux="llf")
        )
        # one RK54 step through the scalar RHS
        dt = 1.0e-3
        cfg = RhsConfig(volume_flux="ranocha", surface_flux="llf")
        rec["rk54_dt"] = np.array(dt)
        rec["rk54_%s" % sname] = rk_step(u, 0.0, dt, lambda v, t: rhs(v, setup, cfg))
    np.savez_compressed(os.path.join(HERE, "case_%s.npz" % name), **rec)
    print("case %-14s %6.1fs" % (name, time.time() - t0), flush=True)


def sample_elements(n_elem, k, seed):
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(n_elem, size=k, replace=False))
    # always include the first and last element (periodic wrap on every side)
    idx[0] = 0
    idx[-1] = n_elem - 1
    return np.unique(idx)


def elem_volume(u, setup, e, flux, pre_mode="none"):
    terms = element_metrics(setup.metrics, e)
    pre = precompute_element_data(u[e], GAS, pre_mode) if pre_mode != "none" else None
    return volume_fluxdiff(u[e], setup.dsplit, terms, flux, GAS, pre)


def make_cfg1():
    mesh = build_mesh((16, 16), bounds=(-1.0, 1.0))
    setup = build_setup(mesh, lgl_operator(3), GAS)
    u = wave_field(setup)
    cfg = RhsConfig(volume_flux="ranocha", surface_flux="llf")
    rec = {
        "u": u,
        "vol": scalar_volume(u, setup, "ranocha", "none"),
        "surf": surface_terms(u, setup, "llf", out=np.zeros_like(u)),
        "du": rhs(u, setup, cfg),
        "du_batched": rhs(u, setup, RhsConfig(volume_flux="ranocha", surface_flux="llf", kernel="batched")),
        "du_logs": rhs(u, setup, RhsConfig(volume_flux="ranocha", surface_flux="llf", precompute="primitives_and_logs")),
    }
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), **rec)
    print("cfg1 done", flush=True)


def make_cfg2():
    mesh = build_mesh((16, 16, 16), bounds=(-1.0, 1.0))
    setup = build_setup(mesh, lgl_operator(3), GAS)
    u = wave_field(setup)
    idx = sample_elements(setup.n_elements, 32, 2)
    rec = {"elements": idx, "u_sample": u[idx]}
    for flux in ("ranocha", "shima"):
        rec["vol_%s" % flux] = np.stack([elem_volume(u, setup, e, flux) for e in idx])
    rec["vol_ranocha_logs"] = np.stack(
        [elem_volume(u, setup, e, "ranocha", "primitives_and_logs") for e in idx]
    )
    volb = B.mesh_fluxdiff_volume(u, setup, RhsConfig(volume_flux="ranocha"))
    rec["volb_ranocha_sample"] = volb[idx]
    rec["volb_ranocha_abs_sum"] = np.abs(volb).sum(axis=(0, 1))
    rec["volb_ranocha_max"] = np.abs(volb).max(axis=(0, 1))
    rec["u_sum"] = u.sum(axis=(0, 1))
    np.savez_compressed(os.path.join(HERE, "cfg2.npz"), **rec)
    print("cfg2 done", flush=True)


def make_cfg3():
    mesh = build_mesh((32, 32, 32), bounds=(-1.0, 1.0))
    setup = build_setup(mesh, lgl_operator(7), GAS)
    n_elem, nn = setup.n_elements, setup.n_nodes
    rng = np.random.default_rng(0)
    q = np.empty((n_elem, nn, 5))
    q[..., 0] = 1.0 + 0.1 * rng.uniform(-1.0, 1.0, size=(n_elem, nn))
    for i in range(3):
        q[..., 1 + i] = rng.normal(0.0, 0.1, size=(n_elem, nn))
    q[..., 4] = 1.0 + 0.1 * rng.uniform(-1.0, 1.0, size=(n_elem, nn))
    u = prim2cons(q, GAS)
    idx = sample_elements(n_elem, 6, 3)
    rec = {"elements": idx, "u_sample": u[idx], "u_sum": u.sum(axis=(0, 1))}
    rec["vol_ranocha"] = np.stack([elem_volume(u, setup, e, "ranocha") for e in idx])
    np.savez_compressed(os.path.join(HERE, "cfg3.npz"), **rec)
    print("cfg3 done", flush=True)


def make_cfg4():
    mesh = build_mesh((48, 48, 48), bounds=(-1.0, 1.0), amplitude=-0.1)
    setup = build_setup(mesh, lgl_operator(4), GAS)
    u = wave_field(setup)
    idx = sample_elements(setup.n_elements, 12, 4)
    rec = {
        "elements": idx,
        "u_sample": u[idx],
        "ja_sample": setup.metrics.ja[idx],
        "jac_sample": setup.metrics.jac[idx],
        "coords_sample": setup.coords[idx],
        "u_sum": u.sum(axis=(0, 1)),
        "jac_sum": setup.metrics.jac.sum(),
    }
    for flux in ("ranocha", "shima"):
        rec["vol_%s" % flux] = np.stack([elem_volume(u, setup, e, flux) for e in idx])
    np.savez_compressed(os.path.join(HERE, "cfg4.npz"), **rec)
    print("cfg4 done", flush=True)


def make_cfg4_rhs():
    """cfg4 at full size through the reference's batched rhs (ranocha + llf):
    du, VOL and SURF on the cfg4 sample elements plus whole-mesh maxima (the
    scales of the cancellation-aware bar) and checksums. ~35 s, ~20 GB."""
    mesh = build_mesh((48, 48, 48), bounds=(-1.0, 1.0), amplitude=-0.1)
    setup = build_setup(mesh, lgl_operator(4), GAS)
    u = wave_field(setup)
    idx = sample_elements(setup.n_elements, 12, 4)
    cfg = RhsConfig(volume_flux="ranocha", surface_flux="llf", kernel="batched")
    t0 = time.time()
    du = rhs(u, setup, cfg)
    vol = B.mesh_fluxdiff_volume(u, setup, cfg)
    surf = B.mesh_surface(u, setup, "llf", np.zeros_like(u))
    rec = {
        "elements": idx,
        "u_sample": u[idx],
        "du_sample": du[idx],
        "vol_sample": vol[idx],
        "surf_sample": surf[idx],
        "du_max": np.abs(du).max(axis=(0, 1)),
        "vol_max": np.abs(vol).max(axis=(0, 1)),
        "surf_max": np.abs(surf).max(axis=(0, 1)),
        "du_abs_sum": np.abs(du).sum(axis=(0, 1)),
        "u_sum": u.sum(axis=(0, 1)),
    }
    np.savez_compressed(os.path.join(HERE, "cfg4_rhs.npz"), **rec)
    print("cfg4_rhs done (%.1fs)" % (time.time() - t0), flush=True)


def make_cfg5():
    """cfg5 (128^3, N=3): the BASELINE noisy wave with N(0,1) noise clipped
    to [-1, 1], coordinates from the reference's
    element_coords, scalar volume_fluxdiff (Ranocha, Shima) on 16 sampled
    elements. The full setup (22 GB) is never built: VOL is element-local
    and the Cartesian metrics are two scalars."""
    from fluxdg.geometry import MetricTerms, element_coords

    mesh = build_mesh((128, 128, 128), bounds=(-1.0, 1.0))
    op = lgl_operator(3)
    coords = element_coords(mesh, op)
    n_elem, nn = coords.shape[0], coords.shape[1]
    rng = np.random.default_rng(0)
    z = np.clip(rng.normal(size=(n_elem, nn)), -1.0, 1.0)
    idx = sample_elements(n_elem, 16, 5)
    x = coords[idx]
    q = np.empty(x.shape[:-1] + (5,))
    q[..., 0] = 1.0 + 0.98 * np.sin(np.pi * x.sum(-1)) + 0.01 * z[idx]
    q[..., 1:4] = (0.1, 0.2, 0.3)
    q[..., 4] = 20.0
    u = prim2cons(q, GAS)
    h = 2.0 / 128
    jac = (0.5 * h) ** 3
    area = jac / (0.5 * h)
    ja = np.zeros((nn, 3, 3))
    for n in range(3):
        ja[:, n, n] = area
    terms = MetricTerms(ja, np.full(nn, jac))
    dop = build_dsplit(op)
    rec = {"elements": idx, "u_sample": u, "coords_sample": x, "z_sample": z[idx], "jac": np.array(jac),
           "area": np.array(area)}
    for flux in ("ranocha", "shima"):
        rec["vol_%s" % flux] = np.stack([volume_fluxdiff(u[k], dop, terms, flux, GAS, None) for k in range(len(idx))])
    rec["vol_ranocha_logs"] = np.stack([
        volume_fluxdiff(u[k], dop, terms, "ranocha", GAS, precompute_element_data(u[k], GAS, "primitives_and_logs"))
        for k in range(len(idx))])
    np.savez_compressed(os.path.join(HERE, "cfg5.npz"), **rec)
    print("cfg5 done", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also write cfg2/cfg3/cfg4 fixtures")
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    print("reference fluxdg", fluxdg.__version__, "numpy", np.__version__)
    if args.only is None or args.only == "operators":
        make_operators()
    for name, (dims, p, amp, bounds) in CASES.items():
        if args.only is None or args.only == name:
            make_case(name, dims, p, amp, bounds)
    if args.only in (None, "cfg1"):
        make_cfg1()
    if args.big or args.only in ("cfg2", "cfg3", "cfg4"):
        if args.only in (None, "cfg2"):
            make_cfg2()
        if args.only in (None, "cfg3"):
            make_cfg3()
        if args.only in (None, "cfg4"):
            make_cfg4()
    if args.only == "cfg4rhs":
        make_cfg4_rhs()
    if args.only == "cfg5":
        make_cfg5()


if __name__ == "__main__":
    main()
