"""Ideal-gas state conversions used on the host (initial conditions, error
reports, diagnostics checks); the device kernels carry their own.

Contract of the reference's euler module (euler.py:18-146): states carry the
variable index last, u = (rho, rho v_1..rho v_d, rho E); primitives
q = (rho, v_1..v_d, p); inadmissible input raises AdmissibilityError with the
reference's message ("<what>: inadmissible state (min rho=.., min p=..)").
The floating-point evaluation order of every formula below is the textbook
one the reference uses too (kinetic energy 1/2 rho |v|^2 with |v|^2 summed in
component order), so states built here from the same primitives carry the
same bits (tests/test_setup.py).
"""

from dataclasses import dataclass, field

import numpy as np

from .errors import AdmissibilityError


@dataclass(frozen=True)
class GasParams:
    """Calorically perfect gas. ``inv_gamma_minus_one`` = 1/(gamma-1) is
    derived once: every energy flux multiplies by it."""

    gamma: float = 1.4
    inv_gamma_minus_one: float = field(init=False)

    def __post_init__(self):
        if not self.gamma > 1.0:
            raise AdmissibilityError("gamma must exceed 1, got %r" % (self.gamma,))
        object.__setattr__(self, "inv_gamma_minus_one", 1.0 / (self.gamma - 1.0))


def _components(a):
    """(first, middle d columns, last, d) of a state-like array."""
    a = np.asarray(a, dtype=float)
    d = a.shape[-1] - 2
    if not 1 <= d <= 3:
        raise AdmissibilityError("state vector length %d is not d+2 for d in 1..3" % a.shape[-1])
    return a[..., 0], a[..., 1 : d + 1], a[..., d + 1], d


def _sq_norm(vec):
    """|v|^2 summed in component order (v_1^2 + v_2^2) + v_3^2."""
    acc = vec[..., 0] * vec[..., 0]
    for i in range(1, vec.shape[-1]):
        acc = acc + vec[..., i] * vec[..., i]
    return acc


def _check(rho, p, what):
    if np.all(rho > 0.0) and np.all(p > 0.0):
        return
    raise AdmissibilityError(
        "%s: inadmissible state (min rho=%r, min p=%r)" % (what, float(np.min(rho)), float(np.min(p)))
    )


def _assemble(first, middle, last, like):
    out = np.empty_like(like)
    d = middle.shape[-1]
    out[..., 0] = first
    out[..., 1 : d + 1] = middle
    out[..., d + 1] = last
    return out


def prim2cons(q, gas):
    """(rho, v, p) -> (rho, rho v, rho E), rho E = p/(gamma-1) + 1/2 rho |v|^2."""
    rho, v, p, _ = _components(q)
    _check(rho, p, "prim2cons")
    energy = p * gas.inv_gamma_minus_one + 0.5 * rho * _sq_norm(v)
    return _assemble(rho, rho[..., None] * v, energy, np.asarray(q, dtype=float))


def _velocity_pressure(u, gas):
    rho, mom, energy, _ = _components(u)
    v = mom / rho[..., None]
    p = (gas.gamma - 1.0) * (energy - 0.5 * rho * _sq_norm(v))
    return rho, v, p


def cons2prim(u, gas):
    """(rho, rho v, rho E) -> (rho, v, p), p = (gamma-1)(rho E - 1/2 rho |v|^2)."""
    rho, v, p = _velocity_pressure(u, gas)
    _check(rho, p, "cons2prim")
    return _assemble(rho, v, p, np.asarray(u, dtype=float))


def entropy_vars(u, gas):
    """w = dU/du for the entropy U = -rho s/(gamma-1), s = log p - gamma log rho:
    w = ((gamma - s)/(gamma-1) - rho |v|^2/(2p), rho v/p, -rho/p)."""
    rho, v, p = _velocity_pressure(u, gas)
    _check(rho, p, "entropy_vars")
    s = np.log(p) - gas.gamma * np.log(rho)
    b = rho / p
    first = (gas.gamma - s) * gas.inv_gamma_minus_one - 0.5 * b * _sq_norm(v)
    return _assemble(first, b[..., None] * v, -b, np.asarray(u, dtype=float))


def max_signal_speed(u, gas):
    """|v| + c per node, c = sqrt(gamma p / rho) (the CFL speed)."""
    rho, mom, energy, _ = _components(u)
    v = mom / rho[..., None]
    p = (gas.gamma - 1.0) * (energy - 0.5 * _sq_norm(mom) / rho)
    _check(rho, p, "sound_speed")
    return np.sqrt(_sq_norm(v)) + np.sqrt(gas.gamma * p / rho)
