"""Explicit Runge-Kutta time integration, host API and device-resident steppers.

Host API (the reference's timeint module, timeint.py:23-220: same names,
arguments, semantics and error messages): ``RKMethod`` (2N-storage
coefficients a, b, c), ``RK54`` (Carpenter-Kennedy five-stage fourth order),
``StepController``, ``stable_dt``, ``rk_step(u, t, dt, rhs_fn, method)``,
``integrate(...)``.

Added (BASELINE config 4; not in the reference, parity unpinned):
``ShuOsherMethod`` and ``SSPRK43`` -- the four-stage third-order
strong-stability-preserving method

    u1 = u  + dt/2 L(u);   u2 = u1 + dt/2 L(u1)
    u3 = 2/3 u + 1/3 u2 + dt/6 L(u2);   u_new = u3 + dt/2 L(u3)

Validation at construction: every method is reduced to its Butcher tableau
by running the scheme's update rules on symbolic stage-derivative
coefficients (a linear simulation), and the tableau is checked against the
order conditions b . Psi(t) = 1/gamma(t) of every rooted tree t up to the
method's order (generated recursively), plus c = A 1. A mistyped
coefficient fails loudly at import.

Device path: ``DeviceStepper`` runs every stage as ONE fused kernel
(fdg_rk_stage: volume + surface + RHS + stage update), optionally captured in
a CUDA graph, and checks the admissibility / finiteness status once per step.
On a failure it replays the step stage by stage to raise exactly the error
the reference's rk_step would raise.
"""

from dataclasses import dataclass
from fractions import Fraction
from functools import lru_cache

import numpy as np

from . import _native as N
from .errors import AdmissibilityError, ConfigurationError, DivergenceError
from .euler import max_signal_speed

# ----------------------------------------------------------- order theory


@lru_cache(maxsize=None)
def _rooted_trees(order):
    """All rooted trees with ``order`` nodes as sorted tuples of subtrees
    (the one-node tree is ())."""
    if order == 1:
        return ((),)
    out = set()

    def forests(n, max_tree):
        # multisets of trees with n nodes in total, trees in non-increasing order
        if n == 0:
            yield ()
            return
        for k in range(n, 0, -1):
            for t in _rooted_trees(k):
                if max_tree is not None and (k, t) > max_tree:
                    continue
                for rest in forests(n - k, (k, t)):
                    yield ((k, t),) + rest

    for f in forests(order - 1, None):
        out.add(tuple(sorted(t for _, t in f)))
    return tuple(sorted(out))


def _size(tree):
    return 1 + sum(_size(t) for t in tree)


def _density(tree):
    g = _size(tree)
    for t in tree:
        g *= _density(t)
    return g


def _stage_weights(tree, amat):
    """Psi(t): the per-stage elementary weight vector, Psi(()) = 1 and
    Psi([t_1..t_m]) = prod_k A Psi(t_k)."""
    psi = np.ones(amat.shape[0])
    for t in tree:
        psi = psi * (amat @ _stage_weights(t, amat))
    return psi


def _validate_tableau(name, amat, bvec, cvec, order, tol=1e-14):
    residuals = {"stage times": float(np.max(np.abs(amat.sum(axis=1) - cvec)))}
    for k in range(1, order + 1):
        for tree in _rooted_trees(k):
            got = float(bvec @ _stage_weights(tree, amat))
            residuals["tree %s (order %d)" % (tree, k)] = abs(got - 1.0 / _density(tree))
    worst = max(residuals, key=residuals.get)
    if residuals[worst] > tol:
        raise ConfigurationError("order conditions violated for %r: %s residual %.3e" % (name, worst, residuals[worst]))


def _simulate_2n(a, b):
    """Butcher (A, b) of the 2N scheme du <- a_i du + dt k_i, v <- v + b_i du,
    by carrying du and v as coefficient vectors over (dt k_0 .. dt k_{s-1})."""
    s = len(b)
    amat = np.zeros((s, s))
    du = np.zeros(s)
    v = np.zeros(s)
    for i in range(s):
        amat[i] = v  # stage i is evaluated at the current v
        du = a[i] * du
        du[i] += 1.0
        v = v + b[i] * du
    return amat, v


def _simulate_shu_osher(A, B, C):
    """Butcher (A, b) of y_i = A_i u + B_i y_{i-1} + C_i dt L(y_{i-1})."""
    s = len(C)
    amat = np.zeros((s, s))
    y = np.zeros(s)  # y_0 = u: no stage derivative yet
    for i in range(s):
        if abs(A[i] + B[i] - 1.0) > 1e-15:
            raise ConfigurationError("stage %d: A + B must be 1" % (i + 1))
        amat[i] = y
        y = B[i] * y  # the A_i u part contributes no stage derivative
        y[i] += C[i]
    return amat, y


# ------------------------------------------------------------------ methods


@dataclass(frozen=True)
class RKMethod:
    """2N-storage explicit Runge-Kutta coefficients: per stage
    du <- a_i du + dt f(v, t + c_i dt); v <- v + b_i du."""

    name: str
    a: tuple
    b: tuple
    c: tuple
    order: int = 4

    def __post_init__(self):
        if not (len(self.a) == len(self.b) == len(self.c)):
            raise ConfigurationError(
                "stage coefficient lists must have equal length, got %d/%d/%d" % (len(self.a), len(self.b), len(self.c))
            )
        if self.a[0] != 0.0:
            raise ConfigurationError("a[0] must be 0 (nothing to carry into the first stage)")
        amat, bvec = _simulate_2n(self.a, self.b)
        _validate_tableau(self.name, amat, bvec, np.asarray(self.c, dtype=float), self.order)

    @property
    def n_stages(self):
        return len(self.b)

    def advance(self, u, t, dt, rhs_fn):
        du = u * 0.0
        v = u.copy() if hasattr(u, "copy") else u.clone()
        for i, (ai, bi, ci) in enumerate(zip(self.a, self.b, self.c)):
            du = ai * du + dt * rhs_fn(v, t + ci * dt)
            v = v + bi * du
            _require_finite(v, i, t, dt)
        return v


@dataclass(frozen=True)
class ShuOsherMethod:
    """Convex-combination stages y_i = A_i u_n + B_i y_{i-1} + C_i dt L(y_{i-1}),
    y_0 = u_n (SSP form: A_i, B_i >= 0, A_i + B_i = 1)."""

    name: str
    A: tuple
    B: tuple
    C: tuple
    c: tuple
    order: int = 3

    def __post_init__(self):
        amat, bvec = _simulate_shu_osher(self.A, self.B, self.C)
        _validate_tableau(self.name, amat, bvec, np.asarray(self.c, dtype=float), self.order)

    @property
    def n_stages(self):
        return len(self.C)

    def advance(self, u, t, dt, rhs_fn):
        y = u
        for i in range(self.n_stages):
            k = rhs_fn(y, t + self.c[i] * dt)
            base = y if self.A[i] == 0.0 else self.A[i] * u + self.B[i] * y
            y = base + (self.C[i] * dt) * k
            _require_finite(y, i, t, dt)
        return y


def _require_finite(v, stage, t, dt):
    ok = bool(v.isfinite().all()) if hasattr(v, "isfinite") else bool(np.all(np.isfinite(v)))
    if not ok:
        raise DivergenceError("non-finite state after stage %d (t=%.6g, dt=%.3e)" % (stage, t, dt))


# Carpenter & Kennedy (1994), five-stage fourth-order 2N-storage scheme
RK54 = RKMethod(
    "carpenter-kennedy 5/4",
    a=(
        0.0,
        -567301805773 / 1357537059087,
        -2404267990393 / 2016746695238,
        -3550918686646 / 2091501179385,
        -1275806237668 / 842570457699,
    ),
    b=(
        1432997174477 / 9575080441755,
        5161836677717 / 13612068292357,
        1720146321549 / 2090206949498,
        3134564353537 / 4481467310338,
        2277821191437 / 14882151754819,
    ),
    c=(
        0.0,
        1432997174477 / 9575080441755,
        2526269341429 / 6820363962896,
        2006345519317 / 3224310063776,
        2802321613138 / 2924317926251,
    ),
)

SSPRK43 = ShuOsherMethod(
    "ssprk(4,3)",
    A=(0.0, 0.0, float(Fraction(2, 3)), 0.0),
    B=(1.0, 1.0, float(Fraction(1, 3)), 1.0),
    C=(0.5, 0.5, float(Fraction(1, 6)), 0.5),
    c=(0.0, 0.5, 1.0, 0.5),
    order=3,
)


@dataclass(frozen=True)
class StepController:
    """CFL number of the step-size rule in stable_dt."""

    cfl: float = 0.5

    def __post_init__(self):
        if not self.cfl > 0.0:
            raise ConfigurationError("cfl: must be positive, got %r" % (self.cfl,))


def stable_dt(u, mesh, metrics, gas, p, controller, setup=None):
    """dt = cfl min_nodes J^(1/d) / (lambda_max (2p+1)) (reference
    timeint.py:138-146): J^(1/d) the local mesh size, (2p+1) the degree
    scaling of the explicit limit.

    ``setup`` (extension): the SpatialSetup ``u`` lives on; with it (required
    for a CUDA tensor ``u``) the min runs on the device (fdg_diagnostic DT)."""
    if setup is not None or (hasattr(u, "is_cuda") and u.is_cuda):
        if setup is None:
            raise ConfigurationError("stable_dt: a CUDA state needs setup= (the device mesh)")
        from .device import DIAG_DT
        from .discretization import _diag

        return controller.cfl * float(_diag(setup, DIAG_DT, u, gate=True)[0])
    d = len(mesh.dims)
    h = np.asarray(metrics.jac) ** (1.0 / d)
    return controller.cfl * float(np.min(h / (max_signal_speed(u, gas) * (2 * p + 1))))


def rk_step(u, t, dt, rhs_fn, method=RK54):
    """One step of ``method`` with exactly one rhs_fn(v, t) call per stage;
    raises DivergenceError on a non-finite stage (reference timeint.py:149-163)."""
    if not dt > 0.0:
        raise ConfigurationError("dt: must be positive, got %r" % (dt,))
    return method.advance(u, t, dt, rhs_fn)


def integrate(u0, rhs_fn, *, n_steps=None, t_end=None, dt=None, dt_fn=None, t0=0.0, method=RK54, callbacks=()):
    """March rhs_fn from u0 for ``n_steps`` steps or up to ``t_end`` (the last
    step clipped to land on it), with a fixed ``dt`` or ``dt_fn(u, t)``;
    callbacks run as cb(step, t, dt, u) after every step. A stage
    DivergenceError is re-raised with the last good state attached
    (.last_fields, .step, .t). Returns (u, {"steps", "t", "rhs_evals"})
    (reference timeint.py:166-220)."""
    if (n_steps is None) == (t_end is None):
        raise ConfigurationError("exactly one of n_steps and t_end must be given")
    if (dt is None) == (dt_fn is None):
        raise ConfigurationError("exactly one of dt and dt_fn must be given")
    slack = 0.0 if t_end is None else 1e-12 * max(1.0, abs(t_end))

    def finished(step, t):
        return step >= n_steps if n_steps is not None else t >= t_end - slack

    u = u0.copy() if hasattr(u0, "copy") else u0.clone()
    t, step = t0, 0
    while not finished(step, t):
        h = dt if dt is not None else dt_fn(u, t)
        if t_end is not None and t + h > t_end:
            h = t_end - t
        try:
            u_new = rk_step(u, t, h, rhs_fn, method)
        except DivergenceError as err:
            wrapped = DivergenceError("diverged in step %d at t=%.6g: %s" % (step, t, err))
            wrapped.last_fields, wrapped.step, wrapped.t = u, step, t
            raise wrapped from err
        u, t, step = u_new, t + h, step + 1
        for cb in callbacks:
            cb(step, t, h, u)
    return u, {"steps": step, "t": t, "rhs_evals": method.n_stages * step}


# ---------------------------------------------------------------- device


class DeviceStepper:
    """Device-resident time stepping: one fused kernel per stage.

    ``dm`` is a DeviceMesh, ``config`` an RhsConfig. ``exchange`` (optional)
    is called as ``exchange(v_in) -> ghost_u`` before every stage (halo
    exchange of a slab partition, parallel.py). The state passed to ``step``
    is never written; the result lives in one of the internal stage buffers.
    Chained stepping (``u = st.step(u, dt)``) is supported: when ``u`` is one
    of the stage buffers, the stages ping-pong between the two others (a
    third buffer is allocated on first need), so no stage overwrites its own
    input or the Shu-Osher base state u_n.
    """

    def __init__(self, dm, config, method=RK54, exchange=None):
        from .discretization import as_rhs_config

        config = as_rhs_config(config)
        config.validate()
        self.dm = dm
        self.torch = dm.torch
        self.scheme = config.scheme()
        self.method = method
        self.exchange = exchange
        self.buf = [dm.empty(), dm.empty()]
        self.reg = dm.empty() if isinstance(method, RKMethod) else None
        self.graph = None
        self._graph_key = None

    def _stages(self, u, dt):
        """(stage struct, v_in, v_out, u0) for every stage of one step."""
        out = []
        m = self.method
        src = u
        pool = self._pool(u)
        for i in range(m.n_stages):
            dst = pool[i % 2]
            st = N.Stage()
            st.index = i
            st.dt = dt
            if isinstance(m, RKMethod):
                st.kind, st.a, st.b, st.cdt = 0, m.a[i], m.b[i], 0.0
                out.append((st, src, dst, None))
            else:
                st.kind, st.a, st.b, st.cdt = 1, m.A[i], m.B[i], m.C[i] * dt
                out.append((st, src, dst, u if m.A[i] != 0.0 else None))
            src = dst
        return out

    def _pool(self, u):
        """The two stage buffers of a step from ``u``: never ``u``'s own."""
        ptr = u.data_ptr() if hasattr(u, "data_ptr") else None
        free = [b for b in self.buf if b.data_ptr() != ptr]
        if len(free) < 2:
            self.buf.append(self.dm.empty())
            free.append(self.buf[-1])
        return free[:2]

    def _launch(self, stages):
        for st, v_in, v_out, u0 in stages:
            self._stage(st, v_in, v_out, u0)

    def _stage(self, st, v_in, v_out, u0):
        """One fused stage; with a split-capable exchange (parallel.HaloExchange)
        the interior elements run while the face traces are in flight."""
        ex = self.exchange
        if ex is not None and hasattr(ex, "start"):
            from .parallel import split_launch

            def launch(ranges, ghost):
                self.dm.stage(self.scheme, st, v_in, v_out, reg=self.reg, u0=u0, ghost_u=ghost, ranges=ranges)

            split_launch(ex, v_in, self.dm.n_elem, launch, self.dm.nn)
            return
        ghost = ex(v_in) if ex is not None else None
        self.dm.stage(self.scheme, st, v_in, v_out, reg=self.reg, u0=u0, ghost_u=ghost)

    def step(self, u, dt, check=True, t=0.0):
        if not dt > 0.0:
            raise ConfigurationError("dt: must be positive, got %r" % (dt,))
        stages = self._stages(u, dt)
        if check:
            self.dm.reset_status()
        self._launch(stages)
        if check:
            first_bad, bad_stage = self.dm.read_status()
            if first_bad >= 0 or bad_stage >= 0:
                self._replay(u, dt, t)
        return stages[-1][2]

    def _replay(self, u, dt, t):
        """Re-run the step stage by stage and raise the reference's error."""
        stages = self._stages(u, dt)
        for st, v_in, v_out, u0 in stages:
            self.dm.reset_status()
            self._stage(st, v_in, v_out, u0)
            first_bad, bad_stage = self.dm.read_status()
            if first_bad >= 0:
                self.dm.raise_if_inadmissible(v_in, first_bad, self.dm.gamma)
            if bad_stage >= 0:
                raise DivergenceError("non-finite state after stage %d (t=%.6g, dt=%.3e)" % (st.index, t, dt))

    def stable_dt(self, u, controller, dist=None, group=None):
        """stable_dt (timeint.py:138-146) of the device state ``u`` of this
        rank: fdg_diagnostic DT on the device, all-reduced MIN across ranks
        when ``dist`` is given (parallel.combine_diagnostic); one 8-byte read
        back."""
        from .device import DIAG_DT

        # the reference's max_signal_speed raises on an inadmissible node
        # (euler.py:26-41): gate this rank's slab before anything is reduced,
        # so a NaN never enters the MIN all-reduce
        self.dm.reset_status()
        self.dm.gate(u)
        first_bad, _ = self.dm.read_status()
        if first_bad >= 0:
            self.dm.raise_if_inadmissible(u, first_bad, self.dm.gamma)
        local = self.dm.diagnostic(DIAG_DT, u)
        if dist is not None:
            from .parallel import combine_diagnostic

            combine_diagnostic(DIAG_DT, local, dist, group=group)
        return controller.cfl * float(local[0])

    # ---- CUDA graph of one whole step (no status reads inside)
    def capture(self, u, dt):
        """Capture one step from the fixed input ``u`` into a CUDA graph."""
        torch = self.torch
        stages = self._stages(u, dt)
        self._launch(stages)  # warm-up: kernel attributes, occupancy queries
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._launch(stages)
        self.graph = g
        self._graph_key = (u.data_ptr(), dt)
        return stages[-1][2]

    def replay(self):
        self.graph.replay()
