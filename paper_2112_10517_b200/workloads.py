"""BASELINE.json configurations as concrete seeded inputs.

The reference measures on its own ICs (no public dataset); these synthetic
states stand in for BASELINE's five configs. Each builder returns
``(setup, u, config)`` with ``u`` the conserved state (n_elem, nn, d+2)
built with prim2cons (bit-identical to the reference's for the same inputs,
tests/test_setup.py).

  cfg1  2D N=3 16^2 Cartesian [-1,1]^2, Ranocha + Rusanov (llf), density wave
  cfg2  3D N=3 16^3 Cartesian, Ranocha, density wave (volume integral)
  cfg3  3D N=7 32^3 Cartesian, Chandrashekar, seeded random state
  cfg4  3D N=4 48^3 curved (amplitude -0.1 in the reference's convention),
        Kennedy-Gruber + llf, density wave, SSPRK43
  cfg5  3D N=3 128^3 Cartesian, Ranocha / Shima + llf, perturbed wave with
        the N(0,1) noise clipped to [-1, 1] (the literal state has rho <= 0
        at 76,163 nodes)
"""

import numpy as np

from .discretization import RhsConfig, build_setup
from .euler import GasParams, prim2cons
from .geometry import build_mesh
from .operators import lgl_operator

GAS = GasParams(1.4)

CONFIGS = {
    1: dict(dims=(16, 16), p=3, amplitude=0.0, volume_flux="ranocha", surface_flux="llf", state="wave"),
    2: dict(dims=(16, 16, 16), p=3, amplitude=0.0, volume_flux="ranocha", surface_flux="llf", state="wave"),
    3: dict(dims=(32, 32, 32), p=7, amplitude=0.0, volume_flux="chandrashekar", surface_flux="llf", state="random"),
    4: dict(dims=(48, 48, 48), p=4, amplitude=-0.1, volume_flux="kennedy_gruber", surface_flux="llf", state="wave"),
    5: dict(dims=(128, 128, 128), p=3, amplitude=0.0, volume_flux="ranocha", surface_flux="llf", state="noisy_wave"),
}


def wave_primitives(coords):
    """rho = 1 + 0.98 sin(pi sum x), v = (0.1, 0.2[, 0.3]), p = 20."""
    d = coords.shape[-1]
    q = np.empty(coords.shape[:-1] + (d + 2,))
    q[..., 0] = 1.0 + 0.98 * np.sin(np.pi * coords.sum(-1))
    for i in range(d):
        q[..., 1 + i] = (0.1, 0.2, 0.3)[i]
    q[..., d + 1] = 20.0
    return q


def random_primitives(shape, d, seed=0):
    """cfg3: rho = 1 + 0.1 U(-1,1); v_i ~ N(0, 0.1^2); p = 1 + 0.1 U(-1,1),
    drawn from default_rng(seed) in this order over (n_elem, nn)."""
    rng = np.random.default_rng(seed)
    q = np.empty(shape + (d + 2,))
    q[..., 0] = 1.0 + 0.1 * rng.uniform(-1.0, 1.0, size=shape)
    for i in range(d):
        q[..., 1 + i] = rng.normal(0.0, 0.1, size=shape)
    q[..., d + 1] = 1.0 + 0.1 * rng.uniform(-1.0, 1.0, size=shape)
    return q


def noisy_wave_primitives(coords, seed=0):
    """cfg5: the wave + 0.01 clip(N(0,1), -1, 1) on rho."""
    q = wave_primitives(coords)
    rng = np.random.default_rng(seed)
    z = np.clip(rng.normal(size=coords.shape[:-1]), -1.0, 1.0)
    q[..., 0] = q[..., 0] + 0.01 * z
    return q


def build(k, dims=None, kernel="batched", volume_flux=None, precompute=None, op=None):
    """(setup, u, config) for BASELINE config ``k`` (optionally resized).
    ``op``: the 1D operator (default lgl_operator(p); tests pass the
    reference's recorded tables to reproduce its states bit for bit)."""
    c = CONFIGS[k]
    dims = tuple(dims) if dims is not None else c["dims"]
    mesh = build_mesh(dims, bounds=(-1.0, 1.0), amplitude=c["amplitude"])
    setup = build_setup(mesh, op if op is not None else lgl_operator(c["p"]), GAS)
    if c["state"] == "wave":
        q = wave_primitives(setup.coords)
    elif c["state"] == "random":
        q = random_primitives((setup.n_elements, setup.n_nodes), setup.d)
    else:
        q = noisy_wave_primitives(setup.coords)
    u = np.ascontiguousarray(prim2cons(q, GAS))
    vf = volume_flux or c["volume_flux"]
    if precompute is None:
        precompute = "primitives_and_logs" if (kernel == "batched" and vf in ("ranocha", "chandrashekar")) else "none"
    config = RhsConfig(volume_flux=vf, surface_flux=c["surface_flux"], precompute=precompute, kernel=kernel)
    return setup, u, config


# ------------------------------------------------------------- device builds


def _prim2cons_torch(q, igm1):
    """prim2cons (euler.py:63-75 operation order) on a CUDA tensor."""
    d = q.shape[-1] - 2
    rho = q[..., 0]
    v = q[..., 1 : d + 1]
    u = q.new_empty(q.shape)
    u[..., 0] = rho
    u[..., 1 : d + 1] = rho[..., None] * v
    u[..., d + 1] = q[..., d + 1] * igm1 + 0.5 * rho * (v * v).sum(-1)
    return u


def build_device(k, dims=None, kernel="batched", volume_flux=None, precompute=None, device="cuda", op=None):
    """(setup, u, config) for BASELINE config ``k`` with the geometry built
    on the GPU (build_setup(device=...): fdg_build_geometry) and the state
    computed there from the device coordinates: no per-node host arrays, so
    the 128^3 cfg5 mesh (5.4 GB state) is ready in seconds instead of the
    host setup's 22 GB / 43 s. ``u`` is a CUDA tensor. The seeded draws
    (cfg3 uniform/normal, cfg5 noise) come from numpy's default_rng(0) in
    the host builder's order, so they are the same numbers; the sin of the
    density wave is the device's (within an ulp of numpy's)."""
    import dataclasses

    import torch

    c = CONFIGS[k]
    dims = tuple(dims) if dims is not None else c["dims"]
    mesh = build_mesh(dims, bounds=(-1.0, 1.0), amplitude=c["amplitude"])
    op = op if op is not None else lgl_operator(c["p"])
    need_coords = c["state"] != "random"
    setup = build_setup(mesh, op, GAS, with_coords=need_coords, device=device)
    n_elem, nn, d = setup.n_elements, setup.n_nodes, setup.d
    dev = torch.device(device)
    if c["state"] == "random":
        q = torch.as_tensor(random_primitives((n_elem, nn), d), device=dev)
    else:
        x = setup.coords
        q = torch.empty((n_elem, nn, d + 2), dtype=torch.float64, device=dev)
        q[..., 0] = 1.0 + 0.98 * torch.sin(torch.pi * x.sum(-1))
        for i in range(d):
            q[..., 1 + i] = (0.1, 0.2, 0.3)[i]
        q[..., d + 1] = 20.0
        del x
        if c["state"] == "noisy_wave":
            rng = np.random.default_rng(0)
            z = np.clip(rng.normal(size=(n_elem, nn)), -1.0, 1.0)
            q[..., 0] += 0.01 * torch.as_tensor(z, device=dev)
            del z
        setup = dataclasses.replace(setup, coords=None)  # frees the device coordinates
    u = _prim2cons_torch(q, GAS.inv_gamma_minus_one)
    del q
    vf = volume_flux or c["volume_flux"]
    if precompute is None:
        precompute = "primitives_and_logs" if (kernel == "batched" and vf in ("ranocha", "chandrashekar")) else "none"
    config = RhsConfig(volume_flux=vf, surface_flux=c["surface_flux"], precompute=precompute, kernel=kernel)
    return setup, u, config


def cartesian_sample(k, n_elem_sample, gas=GAS, op=None):
    """Host state of the first ``n_elem_sample`` elements of Cartesian config
    ``k`` (C-ordered element index), built with the reference's coordinate
    formula (geometry.py:94-136: x = lo + L (e + (xi+1)/2)/n) and the config's
    seeded draws -- the bounded CPU-baseline sample of a mesh too large to
    build on the host. Returns (u, areas, jac_const)."""
    c = CONFIGS[k]
    if c["amplitude"] != 0.0:
        raise ValueError("cartesian_sample: config %d is curved" % k)
    dims = c["dims"]
    d = len(dims)
    op = op if op is not None else lgl_operator(c["p"])
    p1 = op.n_nodes
    nn = p1**d
    half = 0.5 * (op.nodes + 1.0)
    eidx = np.stack(np.unravel_index(np.arange(n_elem_sample), dims), axis=-1)
    x = np.empty((n_elem_sample,) + (p1,) * d + (d,))
    for j in range(d):
        t = (eidx[:, j][:, None] + half[None, :]) / dims[j]  # (n, p1)
        shape = [n_elem_sample] + [1] * d
        shape[1 + j] = p1
        x[..., j] = -1.0 + 2.0 * t.reshape(shape)
    x = x.reshape(n_elem_sample, nn, d)
    if c["state"] == "random":
        q = random_primitives((int(np.prod(dims)), nn), d)[:n_elem_sample]
    else:
        q = wave_primitives(x)
        if c["state"] == "noisy_wave":
            rng = np.random.default_rng(0)
            z = np.clip(rng.normal(size=n_elem_sample * nn), -1.0, 1.0).reshape(n_elem_sample, nn)
            q[..., 0] = q[..., 0] + 0.01 * z
    u = np.ascontiguousarray(prim2cons(q, gas))
    h = [2.0 / n for n in dims]
    jac = 1.0
    for w in h:
        jac *= 0.5 * w
    areas = [jac / (0.5 * h[n]) for n in range(d)]
    return u, areas, jac
