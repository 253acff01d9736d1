"""Flux kinds and evaluation counters (reference fluxes.py:30-101).

The device kernels do not count per evaluation; the host bumps the active
counters with the exact analytic totals the reference's loops would have
produced (two-point evaluations: n_elem d (p+1)^(d-1) |pair table| for the
volume term plus n_elem d (p+1)^(d-1) for the surface term; two log means per
Ranocha / Chandrashekar volume pair), so ``rhs(..., counter=c)`` keeps the
reference's contract (tests/test_discretization.py:314-355 of the reference).
"""

import threading
from contextlib import contextmanager

from .errors import ConfigurationError

VOLUME_KINDS = ("shima", "ranocha", "central", "kennedy_gruber", "chandrashekar")
SURFACE_KINDS = VOLUME_KINDS + ("llf", "hll")


class FluxCounter:
    __slots__ = ("two_point_evals", "one_point_evals", "logmean_evals")

    def __init__(self):
        self.reset()

    def reset(self):
        self.two_point_evals = 0
        self.one_point_evals = 0
        self.logmean_evals = 0

    def __repr__(self):
        return "FluxCounter(two_point=%d, one_point=%d, logmean=%d)" % (
            self.two_point_evals,
            self.one_point_evals,
            self.logmean_evals,
        )


_local = threading.local()


def _stack():
    stack = getattr(_local, "stack", None)
    if stack is None:
        stack = []
        _local.stack = stack
    return stack


@contextmanager
def count_guard(counter):
    """Activate ``counter`` on this thread; nested guards all see every count."""
    stack = _stack()
    stack.append(counter)
    try:
        yield counter
    finally:
        stack.remove(counter)


def bump(extra=None, two_point=0, one_point=0, logmean=0):
    """Add analytic totals to every active counter (and ``extra``, once)."""
    targets = list(getattr(_local, "stack", None) or [])
    if extra is not None and extra not in targets:
        targets.append(extra)
    for c in targets:
        c.two_point_evals += two_point
        c.one_point_evals += one_point
        c.logmean_evals += logmean


def require_volume_kind(kind):
    if kind not in VOLUME_KINDS:
        raise ConfigurationError(
            "volume flux must be symmetric (%s), got %r" % (", ".join(VOLUME_KINDS), kind)
        )
