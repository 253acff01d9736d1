"""Golden fixtures of the reference's Gauss-family schemes:
the zero-corner hybridized volume term on Gauss nodes with entropy-projected
face states, in both arrangements ("gauss_fluxdiff", "gauss_surface_correction"),
and its interface coupling (reference batched.py:558-667,
discretization.py:811-895, 932-995, operators.py:300-357).

Runs only in the build container (imports /root/reference); the outputs are
committed as tests/golden/gauss_<case>.npz.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_gauss.py

Per case: the Gauss operator tables, geometry (coords, ja, jac, elem_face_ja,
face_ja, neighbours), two seeded states, their entropy projections
(_project_all), and for each (scheme, volume flux, surface flux):
rhs(kernel="reference") (the scalar path), rhs(kernel="batched"), the scalar
volume term alone (_scalar_gauss_volume / J) and the batched one
(mesh_gauss_volume).
"""

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from fluxdg import (  # noqa: E402
    FluxCounter,
    GasParams,
    RhsConfig,
    build_mesh,
    build_setup,
    count_guard,
    make_operator,
    prim2cons,
    rhs,
)
from fluxdg import batched as B  # noqa: E402
from fluxdg.discretization import _project_all, _scalar_gauss_volume  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
GAS = GasParams(1.4)

CASES = {
    # name: (dims, p, amplitude, bounds)
    "g2d_cart_p3": ((3, 3), 3, 0.0, (-1.0, 1.0)),
    "g2d_curv_p3": ((3, 2), 3, 0.1, (-1.0, 1.0)),
    "g3d_cart_p2": ((2, 2, 3), 2, 0.0, (-1.0, 1.0)),
    "g3d_curv_p3": ((2, 3, 2), 3, -0.1, (-1.0, 1.0)),
}
COMBOS = [
    ("gauss_fluxdiff", "ranocha", "llf"),
    ("gauss_fluxdiff", "ranocha", "ranocha"),
    ("gauss_fluxdiff", "shima", "llf"),
    ("gauss_fluxdiff", "central", "central"),
    ("gauss_surface_correction", "ranocha", "llf"),
    ("gauss_surface_correction", "shima", "hll"),
]


def random_field(setup, seed, amp):
    rng = np.random.default_rng(seed)
    d = setup.d
    n = setup.n_elements * setup.n_nodes
    q = np.empty((n, d + 2))
    q[:, 0] = 1.0 + amp * rng.random(n)
    q[:, 1 : d + 1] = amp * (rng.random((n, d)) - 0.5)
    q[:, d + 1] = 1.0 + amp * rng.random(n)
    return np.ascontiguousarray(prim2cons(q, GAS).reshape(setup.n_elements, setup.n_nodes, d + 2))


def wave_field(setup):
    x = setup.coords
    d = setup.d
    q = np.empty(x.shape[:-1] + (d + 2,))
    q[..., 0] = 1.0 + 0.5 * np.sin(np.pi * x.sum(-1))
    for i in range(d):
        q[..., 1 + i] = (0.1, 0.2, 0.3)[i]
    q[..., d + 1] = 2.0
    return prim2cons(q, GAS)


def make_case(name, dims, p, amp, bounds):
    t0 = time.time()
    op = make_operator(p, "gauss")
    mesh = build_mesh(dims, bounds=bounds, amplitude=amp)
    setup = build_setup(mesh, op, GAS)
    d = setup.d
    rec = {
        "dims": np.array(dims), "p": np.array(p), "amplitude": np.array(amp), "bounds": np.array(bounds),
        "nodes": op.nodes, "weights": op.weights, "D": op.D, "R": op.boundary_interp,
        "coords": setup.coords, "ja": setup.metrics.ja, "jac": setup.metrics.jac,
        "cartesian": np.array(setup.metrics.cartesian),
    }
    for n in range(d):
        rec["face_ja_%d" % n] = setup.metrics.face_ja[n]
        rec["elem_face_ja_%d" % n] = setup.metrics.elem_face_ja[n]
        rec["plus_%d" % n] = setup.plus_neighbor[n]
    states = {"rand": random_field(setup, 7, 0.4), "wave": wave_field(setup)}
    for sname, u in states.items():
        rec["u_%s" % sname] = u
        proj = _project_all(u, setup)
        for n in range(d):
            for s in (0, 1):
                rec["proj_%s_%d_%d" % (sname, n, s)] = proj[n][s]
        for scheme, vf, sf in COMBOS:
            key = "%s_%s_%s_%s" % (sname, scheme, vf, sf)
            cfg = RhsConfig(volume_scheme=scheme, volume_flux=vf, surface_flux=sf)
            cnt = FluxCounter()
            with count_guard(cnt):
                rec["rhs_" + key] = rhs(u, setup, cfg)
            rec["counts_" + key] = np.array([cnt.two_point_evals, cnt.one_point_evals, cnt.logmean_evals])
            rec["rhsb_" + key] = rhs(u, setup, RhsConfig(volume_scheme=scheme, volume_flux=vf, surface_flux=sf,
                                                         kernel="batched"))
            if sf == "llf" or vf == "central":
                acc = [[[0.0] * (d + 2) for _ in range(setup.n_nodes)] for _ in range(setup.n_elements)]
                _scalar_gauss_volume(u, setup, scheme, vf, proj, acc)
                rec["vol_" + key] = np.asarray(acc) / setup.metrics.jac[:, :, None]
                rec["volb_" + key] = B.mesh_gauss_volume(u, setup, cfg, proj)
    np.savez_compressed(os.path.join(HERE, "gauss_%s.npz" % name), **rec)
    print("gauss case %-12s %6.1fs" % (name, time.time() - t0), flush=True)


def main():
    only = sys.argv[1] if len(sys.argv) > 1 else None
    for name, args in CASES.items():
        if only is None or only == name:
            make_case(name, *args)


if __name__ == "__main__":
    main()
