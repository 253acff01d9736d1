"""Initial conditions of the paper's benchmarks (reference harness.py:183-240)
and the periodic domain they live on.

* isentropic vortex: T = T0 - (gamma-1) eps^2/(8 gamma pi^2)
  exp(1 - r^2), rho = (T/T0)^(1/(gamma-1)), v = v0 + eps/(2 pi) exp((1-r^2)/2)
  (-x2, x1[, 0]), p = rho T, T0 = p0/rho0 = 10, v0 = (1, 1[, 0]), epsilon = 20
  (the paper's strengthened vortex, every log-mean branch is visited), centre
  advected with v0 and wrapped periodically -- exact for all t;
* sinusoidal: rho = 2 + prod_i sin(pi x_i / 5), p = rho^gamma, at rest;
* free stream: rho = 1, v = (0.1, -0.2[, 0.3]), p = 1;
* random: rho, p uniform in [1, 2], v in [-1, 1] from default_rng(seed).
Domain [-5, 5]^d, periodic (harness.py:31-33).
"""

import math

import numpy as np

DOMAIN_LO, DOMAIN_HI = -5.0, 5.0
DOMAIN_LENGTH = DOMAIN_HI - DOMAIN_LO
FREE_STREAM_VELOCITY = (0.1, -0.2, 0.3)
IC_NAMES = ("isentropic_vortex", "sinusoidal", "random", "free_stream")


def wrap_periodic(x):
    return (x - DOMAIN_LO) % DOMAIN_LENGTH + DOMAIN_LO


def vortex_primitives(x, t=0.0, epsilon=20.0, gamma=1.4):
    """The isentropic vortex at time t (primitive variables, last axis)."""
    d = x.shape[-1]
    background = np.array((1.0, 1.0, 0.0)[:d])
    xr = wrap_periodic(x - t * background)
    r2 = xr[..., 0] ** 2 + xr[..., 1] ** 2
    t0 = 10.0
    temp = t0 - (gamma - 1.0) * epsilon**2 / (8.0 * gamma * math.pi**2) * np.exp(1.0 - r2)
    rho = (temp / t0) ** (1.0 / (gamma - 1.0))
    swirl = epsilon / (2.0 * math.pi) * np.exp(0.5 * (1.0 - r2))
    q = np.zeros(x.shape[:-1] + (d + 2,))
    q[..., 0] = rho
    q[..., 1] = background[0] - swirl * xr[..., 1]
    q[..., 2] = background[1] + swirl * xr[..., 0]
    q[..., d + 1] = rho * temp
    return q


def sinusoidal_primitives(x, gamma=1.4):
    d = x.shape[-1]
    rho = 2.0 + np.prod(np.sin(math.pi * x / 5.0), axis=-1)
    q = np.zeros(x.shape[:-1] + (d + 2,))
    q[..., 0] = rho
    q[..., d + 1] = rho**gamma
    return q


def free_stream_primitives(x):
    d = x.shape[-1]
    q = np.empty(x.shape[:-1] + (d + 2,))
    q[..., 0] = 1.0
    for i in range(d):
        q[..., 1 + i] = FREE_STREAM_VELOCITY[i]
    q[..., d + 1] = 1.0
    return q


def random_primitives(x, seed):
    d = x.shape[-1]
    rng = np.random.default_rng(seed)
    q = np.empty(x.shape[:-1] + (d + 2,))
    q[..., 0] = 1.0 + rng.random(x.shape[:-1])
    for i in range(d):
        q[..., 1 + i] = 2.0 * rng.random(x.shape[:-1]) - 1.0
    q[..., d + 1] = 1.0 + rng.random(x.shape[:-1])
    return q


def initial_state(ic, coords, gas, epsilon=20.0, seed=0):
    """Conserved initial state of benchmark ``ic`` on the nodal coordinates."""
    from .euler import prim2cons

    if ic == "isentropic_vortex":
        q = vortex_primitives(coords, 0.0, epsilon, gas.gamma)
    elif ic == "sinusoidal":
        q = sinusoidal_primitives(coords, gas.gamma)
    elif ic == "random":
        q = random_primitives(coords, seed)
    elif ic == "free_stream":
        q = free_stream_primitives(coords)
    else:
        from .errors import ConfigurationError

        raise ConfigurationError("ic: expected one of %s, got %r" % (", ".join(IC_NAMES), ic))
    return np.ascontiguousarray(prim2cons(q, gas))
