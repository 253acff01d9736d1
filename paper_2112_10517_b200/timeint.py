"""Explicit Runge-Kutta time integration, host API and device-resident steppers.

Host API (reference timeint.py:23-220, same names and semantics):
``RKMethod``, ``RK54`` (Carpenter-Kennedy 5-stage 4th order, 2N storage),
``rk_step(u, t, dt, rhs_fn, method)``, ``integrate(...)``, ``stable_dt``.

Added (BASELINE config 4; not in the reference, parity unpinned):
``SSPRK43`` -- the four-stage third-order strong-stability-preserving method
in Shu-Osher form

    u1 = u  + dt/2 L(u);   u2 = u1 + dt/2 L(u1)
    u3 = 2/3 u + 1/3 u2 + dt/6 L(u2);   u_new = u3 + dt/2 L(u3)

Device path: ``DeviceStepper`` runs every stage as ONE fused kernel
(fdg_rk_stage: volume + surface + RHS + stage update, ping-pong state
buffers), optionally captured in a CUDA graph, and checks the admissibility /
finiteness status once per step. On a failure it replays the step stage by
stage to raise exactly the error the reference's rk_step would raise.
"""

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import AdmissibilityError, ConfigurationError, DivergenceError
from .euler import max_signal_speed


@dataclass(frozen=True)
class RKMethod:
    """Low-storage (2N) coefficients: du <- a_i du + dt f; v <- v + b_i du."""

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
        _check_order_conditions(*_butcher_2n(self.a, self.b), np.asarray(self.c), self.order, self.name)

    @property
    def n_stages(self):
        return len(self.b)


@dataclass(frozen=True)
class ShuOsherMethod:
    """Stages y_i = A_i u_n + B_i y_{i-1} + C_i dt L(y_{i-1}) (y_0 = u_n)."""

    name: str
    A: tuple
    B: tuple
    C: tuple
    c: tuple
    order: int = 3

    def __post_init__(self):
        _check_order_conditions(*_butcher_shu_osher(self.A, self.B, self.C), np.asarray(self.c), self.order, self.name)

    @property
    def n_stages(self):
        return len(self.C)


def _butcher_2n(a, b):
    """(A, b) of the Butcher tableau implied by a 2N scheme."""
    s = len(b)
    rows = []
    for i in range(1, s + 1):
        row = []
        for m in range(i):
            coef = b[m]
            prod = 1.0
            for n in range(m + 1, i):
                prod *= a[n]
                coef += b[n] * prod
            row.append(coef)
        rows.append(row)
    amat = np.zeros((s, s))
    for i in range(1, s):
        amat[i, : len(rows[i - 1])] = rows[i - 1]
    return amat, np.asarray(rows[-1], dtype=float)


def _butcher_shu_osher(A, B, C):
    """Butcher (A, b) of y_i = A_i u + B_i y_{i-1} + C_i dt L(y_{i-1})."""
    s = len(C)
    # represent each y_i as u + sum_j W[i, j] dt L(y_j)
    W = np.zeros((s + 1, s))
    for i in range(1, s + 1):
        W[i] = B[i - 1] * W[i - 1]
        W[i, i - 1] += C[i - 1]
        # A_i + B_i must be 1 for consistency
        if abs(A[i - 1] + B[i - 1] - 1.0) > 1e-15:
            raise ConfigurationError("stage %d: A + B must be 1" % i)
    return W[:s], W[s]


def _check_order_conditions(amat, bw, c, order, name, tol=1e-14):
    residuals = {"stage times": float(np.max(np.abs(amat.sum(axis=1) - c)))}
    ac = amat @ c
    conds = [("sum b", bw.sum(), 1.0), ("b.c", bw @ c, 0.5), ("b.c^2", bw @ c**2, 1 / 3), ("b.Ac", bw @ ac, 1 / 6)]
    if order >= 4:
        conds += [
            ("b.c^3", bw @ c**3, 0.25),
            ("b.(c*Ac)", bw @ (c * ac), 0.125),
            ("b.Ac^2", bw @ (amat @ c**2), 1 / 12),
            ("b.AAc", bw @ (amat @ ac), 1 / 24),
        ]
    for label, got, want in conds:
        residuals[label] = abs(float(got) - want)
    worst = max(residuals, key=residuals.get)
    if residuals[worst] > tol:
        raise ConfigurationError("order conditions violated for %r: %s residual %.3e" % (name, worst, residuals[worst]))


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
    A=(0.0, 0.0, 2.0 / 3.0, 0.0),
    B=(1.0, 1.0, 1.0 / 3.0, 1.0),
    C=(0.5, 0.5, 1.0 / 6.0, 0.5),
    c=(0.0, 0.5, 1.0, 0.5),
    order=3,
)


@dataclass(frozen=True)
class StepController:
    cfl: float = 0.5

    def __post_init__(self):
        if not self.cfl > 0.0:
            raise ConfigurationError("cfl: must be positive, got %r" % (self.cfl,))


def stable_dt(u, mesh, metrics, gas, p, controller, setup=None):
    """dt = cfl min J^(1/d) / (lambda_max (2p+1))  (reference timeint.py:138-146).

    ``setup`` (extension): the SpatialSetup ``u`` lives on; with it (required
    for a CUDA tensor ``u``) the min runs on the device (fdg_diagnostic DT)."""
    if setup is not None or (hasattr(u, "is_cuda") and u.is_cuda):
        if setup is None:
            raise ConfigurationError("stable_dt: a CUDA state needs setup= (the device mesh)")
        from .device import DIAG_DT
        from .discretization import _diag

        return controller.cfl * float(_diag(setup, DIAG_DT, u, gate=True)[0])
    lam = max_signal_speed(u, gas)
    scale = np.asarray(metrics.jac) ** (1.0 / mesh.d)
    return controller.cfl * float(np.min(scale / (lam * (2 * p + 1))))


def _isfinite_all(v):
    if hasattr(v, "isfinite"):
        return bool(v.isfinite().all())
    return bool(np.all(np.isfinite(v)))


def rk_step(u, t, dt, rhs_fn, method=RK54):
    """One step with any rhs_fn (host API, reference timeint.py:149-163)."""
    if not dt > 0.0:
        raise ConfigurationError("dt: must be positive, got %r" % (dt,))
    if isinstance(method, ShuOsherMethod):
        u0 = u
        y = u
        for i in range(method.n_stages):
            k = rhs_fn(y, t + method.c[i] * dt)
            if method.A[i] != 0.0:
                y = method.A[i] * u0 + method.B[i] * y + (method.C[i] * dt) * k
            else:
                y = y + (method.C[i] * dt) * k
            if not _isfinite_all(y):
                raise DivergenceError("non-finite state after stage %d (t=%.6g, dt=%.3e)" % (i, t, dt))
        return y
    du = u * 0.0
    v = u.copy() if hasattr(u, "copy") else u.clone()
    for i in range(method.n_stages):
        k = rhs_fn(v, t + method.c[i] * dt)
        du = method.a[i] * du + dt * k
        v = v + method.b[i] * du
        if not _isfinite_all(v):
            raise DivergenceError("non-finite state after stage %d (t=%.6g, dt=%.3e)" % (i, t, dt))
    return v


def integrate(u0, rhs_fn, *, n_steps=None, t_end=None, dt=None, dt_fn=None, t0=0.0, method=RK54, callbacks=()):
    """March rhs_fn from u0 (reference timeint.py:166-220)."""
    if (n_steps is None) == (t_end is None):
        raise ConfigurationError("exactly one of n_steps and t_end must be given")
    if (dt is None) == (dt_fn is None):
        raise ConfigurationError("exactly one of dt and dt_fn must be given")
    u = u0.copy() if hasattr(u0, "copy") else u0.clone()
    t = t0
    step = 0
    eps = 1e-12 * max(1.0, abs(t_end)) if t_end is not None else 0.0
    while True:
        if n_steps is not None:
            if step >= n_steps:
                break
        elif t >= t_end - eps:
            break
        h = dt if dt is not None else dt_fn(u, t)
        if t_end is not None and t + h > t_end:
            h = t_end - t
        try:
            u_next = rk_step(u, t, h, rhs_fn, method)
        except DivergenceError as err:
            wrapped = DivergenceError("diverged in step %d at t=%.6g: %s" % (step, t, err))
            wrapped.last_fields = u
            wrapped.step = step
            wrapped.t = t
            raise wrapped from err
        u = u_next
        t += h
        step += 1
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
            ghost = self.exchange(v_in) if self.exchange is not None else None
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
            ghost = self.exchange(v_in) if self.exchange is not None else None
            self.dm.stage(self.scheme, st, v_in, v_out, reg=self.reg, u0=u0, ghost_u=ghost)
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
