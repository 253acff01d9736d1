"""Slab decomposition + face-trace halo, multi-process on the CPU (gloo).

Each rank computes the RHS of its slab with the oracle, fed only with its own
elements and the ghost face traces received through HaloExchange; the result
must be BITWISE the corresponding slice of the single-domain RHS. This pins
the partition, the ghost-slot layout, the packer and the exchange plumbing
that the GPU path (NCCL + fdg_pack_faces + the element kernel's ghost reads)
uses unchanged.
"""

import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, dims, p, amp, vf, sf, results):
    import torch
    import torch.distributed as dist

    from oracle import oracle
    from paper_2112_10517_b200 import GasParams, build_mesh, build_setup, lgl_operator, prim2cons
    from paper_2112_10517_b200.parallel import HaloExchange, slab_partition

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gas = GasParams(1.4)
        setup = build_setup(build_mesh(dims, bounds=(-1.0, 1.0), amplitude=amp), lgl_operator(p), gas)
        rng = np.random.default_rng(11)
        q = np.empty((setup.n_elements, setup.n_nodes, setup.d + 2))
        q[..., 0] = 1.0 + 0.3 * rng.random(q.shape[:2])
        q[..., 1 : setup.d + 1] = 0.3 * (rng.random(q.shape[:2] + (setup.d,)) - 0.5)
        q[..., -1] = 1.0 + 0.3 * rng.random(q.shape[:2])
        u = prim2cons(q, gas)
        part = slab_partition(setup, rank, world)
        lo, hi = part["lo"], part["hi"]
        u_loc = np.ascontiguousarray(u[lo:hi])
        halo = HaloExchange(part, setup.d, p + 1, torch, dist)
        ghost = halo(torch.from_numpy(u_loc))
        cart = setup.metrics.cartesian
        mesh = oracle.MeshArrays(
            setup.d, p + 1, hi - lo, setup.dsplit.matrix, setup.op.weights, gas.gamma, gas.inv_gamma_minus_one,
            cart, setup.metrics.areas if cart else None, setup.metrics.jac_const if cart else 0.0,
            None if cart else setup.metrics.ja[lo:hi], None if cart else setup.metrics.jac[lo:hi],
            part["plus"], part["minus"],
            ghost_u=None if ghost is None else ghost.numpy(), ghost_nrm=part["ghost_nrm"],
        )
        du_loc = oracle.rhs(u_loc, mesh, vf, sf)
        du_all = oracle.rhs(u, setup, vf, sf)
        results[rank] = bool(np.array_equal(du_loc, du_all[lo:hi]))
    finally:
        dist.destroy_process_group()


def _split_worker(rank, world, port, dims, p, amp, results):
    """The overlap split (parallel.split_launch): interior rows computed
    while the exchange is in flight with NO ghost buffer, boundary planes
    after finish() with the ghosts -- bitwise the single-domain rows."""
    import torch
    import torch.distributed as dist

    from oracle import oracle
    from paper_2112_10517_b200 import GasParams, build_mesh, build_setup, lgl_operator, prim2cons
    from paper_2112_10517_b200 import parallel as PL
    from paper_2112_10517_b200.parallel import HaloExchange, slab_partition, split_launch

    PL.SPLIT_MIN_PLANES = 3  # these tiny slabs take the split path
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gas = GasParams(1.4)
        setup = build_setup(build_mesh(dims, bounds=(-1.0, 1.0), amplitude=amp), lgl_operator(p), gas)
        rng = np.random.default_rng(12)
        q = np.empty((setup.n_elements, setup.n_nodes, setup.d + 2))
        q[..., 0] = 1.0 + 0.3 * rng.random(q.shape[:2])
        q[..., 1 : setup.d + 1] = 0.3 * (rng.random(q.shape[:2] + (setup.d,)) - 0.5)
        q[..., -1] = 1.0 + 0.3 * rng.random(q.shape[:2])
        u = prim2cons(q, gas)
        part = slab_partition(setup, rank, world)
        lo, hi = part["lo"], part["hi"]
        u_loc = np.ascontiguousarray(u[lo:hi])
        halo = HaloExchange(part, setup.d, p + 1, torch, dist)
        cart = setup.metrics.cartesian

        def mesh(ghost):
            return oracle.MeshArrays(
                setup.d, p + 1, hi - lo, setup.dsplit.matrix, setup.op.weights, gas.gamma, gas.inv_gamma_minus_one,
                cart, setup.metrics.areas if cart else None, setup.metrics.jac_const if cart else 0.0,
                None if cart else setup.metrics.ja[lo:hi], None if cart else setup.metrics.jac[lo:hi],
                part["plus"], part["minus"],
                ghost_u=None if ghost is None else ghost.numpy(), ghost_nrm=part["ghost_nrm"],
            )

        du_loc = np.full_like(u_loc, np.nan)
        calls = []

        def launch(ranges, ghost):
            for a, b in (ranges if ranges is not None else [(0, hi - lo)]):
                calls.append((a, b, ghost is not None))
                oracle.rhs_range(u_loc, mesh(ghost), du_loc, a, b, "ranocha", "llf")

        split_launch(halo, torch.from_numpy(u_loc), hi - lo, launch)
        du_all = oracle.rhs(u, setup, "ranocha", "llf")
        interior_no_ghost = all(not g for a, b, g in calls if a > 0 and b < hi - lo)
        results[rank] = (bool(np.array_equal(du_loc, du_all[lo:hi])), interior_no_ghost, len(calls))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dims,p,amp", [(2, (6, 2, 3), 3, 0.0), (3, (9, 2, 2), 4, -0.1), (2, (6, 3), 3, 0.1)])
def test_overlap_split_bitwise(world, dims, p, amp):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    manager = ctx.Manager()
    results = manager.dict()
    port = _free_port()
    procs = [ctx.Process(target=_split_worker, args=(r, world, port, dims, p, amp, results)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=180)
        assert pr.exitcode == 0
    for r in range(world):
        ok, interior_no_ghost, n_calls = results[r]
        assert ok and interior_no_ghost and n_calls == 3, (r, results[r])


@pytest.mark.parametrize(
    "world,dims,p,amp",
    [(2, (4, 2, 3), 3, 0.0), (2, (2, 3, 2), 2, 0.08), (3, (6, 2, 2), 4, -0.1), (2, (4, 5), 3, 0.1)],
)
def test_slab_rhs_bitwise(world, dims, p, amp):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    manager = ctx.Manager()
    results = manager.dict()
    port = _free_port()
    procs = [
        ctx.Process(target=_worker, args=(r, world, port, dims, p, amp, "ranocha", "llf", results))
        for r in range(world)
    ]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=180)
        assert pr.exitcode == 0
    assert dict(results) == {r: True for r in range(world)}


def test_partition_tables():
    from paper_2112_10517_b200 import GasParams, build_mesh, build_setup, lgl_operator
    from paper_2112_10517_b200.errors import ConfigurationError
    from paper_2112_10517_b200.parallel import slab_partition

    setup = build_setup(build_mesh((4, 2, 2), bounds=(-1.0, 1.0)), lgl_operator(3), GasParams(1.4))
    part = slab_partition(setup, 1, 2)
    assert (part["lo"], part["hi"], part["plane"]) == (8, 16, 4)
    assert part["plus"][0, 4:].tolist() == [-1, -2, -3, -4]  # last plane -> plus ghosts
    assert part["minus"][0, :4].tolist() == [-5, -6, -7, -8]  # first plane -> minus ghosts
    assert np.all(part["plus"][1:] >= 0) and np.all(part["minus"][1:] >= 0)
    single = slab_partition(setup, 0, 1)
    assert single["n_ghost"] == 0 and np.all(single["plus"] >= 0)
    with pytest.raises(ConfigurationError):
        slab_partition(setup, 0, 5)


def _diag_worker(rank, world, port, results):
    import torch
    import torch.distributed as dist

    from oracle import oracle
    from paper_2112_10517_b200 import workloads
    from paper_2112_10517_b200.device import DIAG_CONSERVED, DIAG_DT
    from paper_2112_10517_b200.parallel import combine_diagnostic, slab_partition

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        setup, u, _ = workloads.build(4, dims=(6, 4, 4))
        part = slab_partition(setup, rank, world)
        lo, hi = part["lo"], part["hi"]
        wj = oracle._wbar_jac(setup)[lo:hi]
        local = torch.as_tensor(np.sum(wj[..., None] * u[lo:hi], axis=(0, 1)))
        combine_diagnostic(DIAG_CONSERVED, local, dist)
        # DT stand-in: this slab's own min of the per-node quotient
        sub = type("S", (), {})()
        sub.metrics = type("M", (), {"jac": np.asarray(setup.metrics.jac)[lo:hi]})()
        sub.op = setup.op
        dt_local = torch.tensor([oracle.stable_dt(u[lo:hi], sub, cfl=1.0)], dtype=torch.float64)
        combine_diagnostic(DIAG_DT, dt_local, dist)
        results[rank] = (local.numpy().copy(), float(dt_local[0]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_combine_diagnostic(world):
    """Sharded diagnostics: per-slab partial sums and mins all-reduced with
    gloo equal the single-domain values (sums within the sequential-sum bound
    n eps of the absolute sum, the dt min exactly)."""
    import torch.multiprocessing as mp

    from oracle import oracle
    from paper_2112_10517_b200 import workloads

    results = mp.Manager().dict()
    mp.spawn(_diag_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    setup, u, _ = workloads.build(4, dims=(6, 4, 4))
    terms = oracle._wbar_jac(setup)[..., None] * u
    want = terms.sum(axis=(0, 1))
    dt = oracle.stable_dt(u, setup, cfl=1.0)
    for r in range(world):
        got, got_dt = results[r]
        n = terms.shape[0] * terms.shape[1]
        assert np.all(np.abs(got - want) <= n * 2.3e-16 * np.abs(terms).sum(axis=(0, 1)))
        assert got_dt == dt
