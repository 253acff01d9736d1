"""Ideal-gas helpers used on the host (initial conditions, diagnostics).

Same conventions as the reference (euler.py:18-75): conserved states carry
the variable index last, u = (rho, rho v_1..rho v_d, rho E); the arithmetic
below keeps the reference's operation order so states built here are
bit-identical to the reference's prim2cons output.
"""

from dataclasses import dataclass, field

import numpy as np

from .errors import AdmissibilityError


@dataclass(frozen=True)
class GasParams:
    """Ideal gas; 1/(gamma-1) is stored because every energy flux uses it
    (reference euler.py:18-29)."""

    gamma: float = 1.4
    inv_gamma_minus_one: float = field(init=False)

    def __post_init__(self):
        if not self.gamma > 1.0:
            raise AdmissibilityError("gamma must exceed 1, got %r" % (self.gamma,))
        object.__setattr__(self, "inv_gamma_minus_one", 1.0 / (self.gamma - 1.0))


def _dim(u):
    d = u.shape[-1] - 2
    if d not in (1, 2, 3):
        raise AdmissibilityError("state vector length %d is not d+2 for d in 1..3" % u.shape[-1])
    return d


def _require_admissible(rho, p, what):
    if not (np.all(rho > 0.0) and np.all(p > 0.0)):
        raise AdmissibilityError(
            "%s: inadmissible state (min rho=%r, min p=%r)" % (what, float(np.min(rho)), float(np.min(p)))
        )


def prim2cons(q, gas):
    """(rho, v, p) -> conserved, as reference euler.py:63-75."""
    q = np.asarray(q, dtype=float)
    d = _dim(q)
    rho = q[..., 0]
    v = q[..., 1 : d + 1]
    p = q[..., d + 1]
    _require_admissible(rho, p, "prim2cons")
    u = np.empty_like(q)
    u[..., 0] = rho
    u[..., 1 : d + 1] = rho[..., None] * v
    u[..., d + 1] = p * gas.inv_gamma_minus_one + 0.5 * rho * np.sum(v * v, axis=-1)
    return u


def cons2prim(u, gas):
    """conserved -> (rho, v, p), as reference euler.py:47-60."""
    u = np.asarray(u, dtype=float)
    d = _dim(u)
    rho = u[..., 0]
    v = u[..., 1 : d + 1] / rho[..., None]
    kinetic = 0.5 * rho * np.sum(v * v, axis=-1)
    p = (gas.gamma - 1.0) * (u[..., d + 1] - kinetic)
    _require_admissible(rho, p, "cons2prim")
    q = np.empty_like(u)
    q[..., 0] = rho
    q[..., 1 : d + 1] = v
    q[..., d + 1] = p
    return q


def entropy_vars(u, gas):
    """Entropy variables for U = -rho s/(gamma-1), s = log p - gamma log rho
    (reference euler.py:129-146); used by the entropy diagnostics."""
    u = np.asarray(u, dtype=float)
    d = _dim(u)
    rho = u[..., 0]
    v = u[..., 1 : d + 1] / rho[..., None]
    p = (gas.gamma - 1.0) * (u[..., d + 1] - 0.5 * rho * np.sum(v * v, axis=-1))
    _require_admissible(rho, p, "entropy_vars")
    s = np.log(p) - gas.gamma * np.log(rho)
    rho_p = rho / p
    w = np.empty_like(u)
    w[..., 0] = (gas.gamma - s) * gas.inv_gamma_minus_one - 0.5 * rho_p * np.sum(v * v, axis=-1)
    w[..., 1 : d + 1] = rho_p[..., None] * v
    w[..., d + 1] = -rho_p
    return w


def max_signal_speed(u, gas):
    """|v| + c per node (CFL; reference euler.py:105-112)."""
    u = np.asarray(u, dtype=float)
    d = _dim(u)
    rho = u[..., 0]
    v = u[..., 1 : d + 1] / rho[..., None]
    vmag = np.sqrt(np.sum(v * v, axis=-1))
    mom = u[..., 1 : d + 1]
    p = (gas.gamma - 1.0) * (u[..., d + 1] - 0.5 * np.sum(mom * mom, axis=-1) / rho)
    _require_admissible(rho, p, "sound_speed")
    return vmag + np.sqrt(gas.gamma * p / rho)
