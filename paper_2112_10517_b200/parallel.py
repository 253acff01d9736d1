"""Slab domain decomposition of the periodic mesh and the face-trace halo.

One process per GPU. Rank r owns the contiguous element range of planes
[P r / W, P (r+1) / W) of reference direction 0 (the slowest index of the
reference's C-ordered element numbering, geometry.py:87-90), so the only data
crossing a partition are the conserved states on the two x-faces of the slab
(p+1)^(d-1) (d+2) doubles per face. Each side then evaluates the shared face
flux from identical inputs (the element kernel evaluates every interface
from both sides anyway), so the partitioned RHS is bit-identical to the
single-domain one (tests/test_parallel.py checks it with gloo on the CPU
oracle; the GPU path uses the same partition and buffers with NCCL).

Ghost slots (negative neighbour entries -(g+1) in the local tables):
  g in [0, F)      plus ghosts: face traces (line position 0) of the next
                   rank's first plane, for the +x faces of my last plane
  g in [F, 2F)     minus ghosts: face traces (line position p) of the previous
                   rank's last plane, for the -x faces of my first plane
with F elements per plane; ``ghost_nrm`` holds the minus neighbours' own +x
face metrics for curved meshes (static, computed from the global setup).
"""

import numpy as np

from .errors import ConfigurationError
from .operators import node_lines


def _plane(setup):
    dims = setup.mesh.dims
    n_elem = int(np.prod(dims))
    return dims[0], n_elem // dims[0], n_elem


def slab_partition(setup, rank, world):
    """Local neighbour tables, ghost-slot layout and send lists of one rank."""
    planes, F, n_elem = _plane(setup)
    if world > planes:
        raise ConfigurationError("cannot split %d element planes over %d ranks" % (planes, world))
    d = setup.d
    p1 = setup.op.degree + 1
    p_lo, p_hi = planes * rank // world, planes * (rank + 1) // world
    lo, hi = p_lo * F, p_hi * F
    n_loc = hi - lo
    plus_g = np.stack([np.asarray(setup.plus_neighbor[n], dtype=np.int64) for n in range(d)])
    minus_g = np.empty_like(plus_g)
    for n in range(d):
        minus_g[n, plus_g[n]] = np.arange(n_elem)
    plus = plus_g[:, lo:hi] - lo
    minus = minus_g[:, lo:hi] - lo
    if world > 1:
        last = np.arange(hi - F, hi) - lo  # local ids of my last plane
        first = np.arange(lo, lo + F) - lo  # local ids of my first plane
        plus[0, last] = -(np.arange(F) + 1)
        minus[0, first] = -(F + np.arange(F) + 1)
    assert np.all((plus >= -2 * F) & (plus < n_loc)) and np.all((minus >= -2 * F) & (minus < n_loc))
    ghost_nrm = None
    if world > 1 and not setup.metrics.cartesian:
        fn = p1 ** (d - 1)
        ends = node_lines(p1, d)[0][:, -1]  # +x face nodes, line order
        remote_minus = minus_g[0, lo : lo + F]  # previous rank's last plane
        ghost_nrm = np.zeros((2 * F, fn, d))
        ja = setup.metrics.ja
        if hasattr(ja, "is_cuda"):  # device-built geometry: gather on the device, copy the small result
            import torch

            sel = ja[torch.as_tensor(remote_minus, device=ja.device)][:, torch.as_tensor(ends, device=ja.device), 0, :]
            ghost_nrm[F:] = sel.cpu().numpy()
        else:
            ghost_nrm[F:] = np.asarray(ja)[remote_minus][:, ends, 0, :]
    return {
        "rank": rank,
        "world": world,
        "lo": lo,
        "hi": hi,
        "plane": F,
        "plus": plus,
        "minus": minus,
        "ghost_nrm": ghost_nrm,
        "n_ghost": 2 * F if world > 1 else 0,
        # what I send: my first plane's line-start traces to rank-1 (its plus
        # ghosts) and my last plane's line-end traces to rank+1 (its minus ghosts)
        "send_first": np.arange(0, F, dtype=np.int32),
        "send_last": np.arange(n_loc - F, n_loc, dtype=np.int32),
    }


def pack_faces_host(u, elems, d, p1, direction, side):
    """Host twin of fdg_pack_faces: (len(elems), fn, nvar) face traces."""
    lines = node_lines(p1, d)[direction]
    pos = p1 - 1 if side else 0
    return np.ascontiguousarray(u[np.asarray(elems)][:, lines[:, pos], :])


class HaloExchange:
    """Face-trace exchange of one slab per RHS evaluation.

    Works on CPU tensors with gloo (tests) and on CUDA tensors with NCCL;
    ``pack`` is the device packer (DeviceMesh.pack_faces) or None for the
    host packer. Grouped send/recv to both ring neighbours. ``start`` /
    ``finish`` split it so the interior elements run while it is in flight
    (``split_launch``); calling the object does both (blocking).
    """

    def __init__(self, part, d, p1, torch, dist, device="cpu", pack=None, group=None):
        self.part, self.d, self.p1 = part, d, p1
        self.torch, self.dist, self.group = torch, dist, group
        self.device = device
        self.pack = pack
        F = part["plane"]
        fn = p1 ** (d - 1)
        nvar = d + 2
        self.world, self.rank = part["world"], part["rank"]
        mk = lambda *s: torch.empty(s, dtype=torch.float64, device=device)  # noqa: E731
        self.send_first = mk(F, fn, nvar)
        self.send_last = mk(F, fn, nvar)
        self.ghost = mk(2 * F, fn, nvar)
        self.first_idx = torch.as_tensor(part["send_first"], device=device)
        self.last_idx = torch.as_tensor(part["send_last"], device=device)

    # ---- split API: start the exchange, run the interior, finish, run the boundary
    def start(self, u):
        """Pack this slab's two x-face planes of ``u`` and post the grouped
        send/recv (asynchronous: NCCL queues it on its own stream behind the
        packing kernels); ``finish`` waits for it and returns the ghosts."""
        self._reqs = []
        if self.world == 1:
            return
        torch, dist = self.torch, self.dist
        if self.pack is not None:
            self.pack(u, self.first_idx, 0, 0, self.send_first)
            self.pack(u, self.last_idx, 0, 1, self.send_last)
        else:
            un = u.numpy() if hasattr(u, "numpy") else u
            self.send_first.copy_(torch.from_numpy(pack_faces_host(un, self.part["send_first"], self.d, self.p1, 0, 0)))
            self.send_last.copy_(torch.from_numpy(pack_faces_host(un, self.part["send_last"], self.d, self.p1, 0, 1)))
        F = self.part["plane"]
        nxt, prv = (self.rank + 1) % self.world, (self.rank - 1) % self.world
        # tags disambiguate the two messages when both neighbours are one rank
        # (W = 2, gloo); NCCL matches them in posting order, which is the same
        ops = [
            dist.P2POp(dist.isend, self.send_first, prv, group=self.group, tag=1),
            dist.P2POp(dist.isend, self.send_last, nxt, group=self.group, tag=2),
            dist.P2POp(dist.irecv, self.ghost[:F], nxt, group=self.group, tag=1),
            dist.P2POp(dist.irecv, self.ghost[F:], prv, group=self.group, tag=2),
        ]
        self._reqs = dist.batch_isend_irecv(ops)

    def finish(self):
        """Wait for the exchange posted by ``start`` (NCCL: the current CUDA
        stream waits for it, the host does not) and return the ghost traces
        (None on one rank)."""
        for req in self._reqs:
            req.wait()
        self._reqs = []
        return self.ghost if self.world > 1 else None

    def __call__(self, u):
        """Blocking exchange: ghosts of ``u`` for a whole-slab launch."""
        self.start(u)
        return self.finish()

    def ranges(self, n_loc):
        """(interior, boundary) element ranges of the split: the interior
        elements read no ghost slot; the boundary is the first and last
        planes (one range when they touch), run as ONE launch."""
        F = self.part["plane"]
        if self.world == 1:
            return (0, n_loc), []
        if n_loc <= 2 * F:
            return None, [(0, n_loc)]
        return (F, n_loc - F), [(0, F), (n_loc - F, n_loc)]


HALO_RESERVE_SMS = 8  # SMs left to the packer / NCCL while the interior runs (DeviceMesh.reserve_sms)
# the split pays one extra launch (its ramp and tail, ~20-90 us measured on
# B200, profiles/r02_overlap_c.jsonl) to hide the exchange; below this many
# planes per slab, or this many nodes, the blocking exchange + one launch wins
SPLIT_MIN_PLANES = 8
SPLIT_MIN_NODES = 1 << 22


def split_launch(halo, u, n_loc, launch, nodes_per_elem=None):
    """One RHS-type evaluation with the face-trace exchange overlapped:
    ``launch(ranges, ghost)`` runs the kernel on the element ``ranges``
    (None: the whole slab). Order: pack + post the exchange, the interior (no
    ghosts) while it is in flight, wait, then both boundary planes in one
    launch with the received ghosts. Bitwise equal to one whole-slab launch
    after a blocking exchange. Small slabs (fewer than SPLIT_MIN_PLANES
    planes or SPLIT_MIN_NODES nodes) take that blocking path."""
    if halo is None or halo.world == 1:
        launch(None, None)
        return
    F = halo.part["plane"]
    big = n_loc >= SPLIT_MIN_PLANES * F and (nodes_per_elem is None or n_loc * nodes_per_elem >= SPLIT_MIN_NODES)
    if not big:
        launch(None, halo(u))
        return
    interior, boundary = halo.ranges(n_loc)
    halo.start(u)
    if interior is not None:
        launch([interior], None)
    ghost = halo.finish()
    launch(boundary, ghost)


def combine_diagnostic(kind, local, dist, group=None):
    """Rank-local fdg_diagnostic results -> the global value, in place: an
    all-reduce SUM for the sums (CONSERVED, ENTROPY, ERROR_SQ) and MIN for DT,
    the only global collectives of a sharded run besides the halo
    (SURVEY.md 8e). ``local`` is the (small) tensor DeviceMesh.diagnostic
    returned on this rank's slab."""
    from .device import DIAG_DT

    op = dist.ReduceOp.MIN if kind == DIAG_DT else dist.ReduceOp.SUM
    dist.all_reduce(local, op=op, group=group)
    return local
