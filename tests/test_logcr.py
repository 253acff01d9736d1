"""log_cr (paper_2112_10517_b200/csrc/fdg_logcr.h) is the correctly rounded
natural log: checked against 200-bit mpmath on random and adversarial inputs.
The same source is compiled into the GPU FAITHFUL kernels and into
oracle/liboracle_cr.so (exercised here)."""

import ctypes
import math

import numpy as np
import pytest

from oracle import oracle

mpmath = pytest.importorskip("mpmath")


def _log_cr():
    L = oracle.lib("cr")
    L.or_log.argtypes = [ctypes.c_double]
    L.or_log.restype = ctypes.c_double
    return L.or_log


def _cr(x):
    with mpmath.workprec(200):
        return float(mpmath.log(mpmath.mpf(x)))


def test_log_cr_is_correctly_rounded():
    f = _log_cr()
    rng = np.random.default_rng(42)
    xs = np.concatenate([
        rng.uniform(0.2, 5.0, 20000),
        1.0 + rng.uniform(-0.02, 0.02, 10000),
        1.0 + rng.uniform(-1e-7, 1e-7, 5000),
        np.exp(rng.uniform(-700.0, 700.0, 5000)),
        np.array([1.0 + 2.0**-52, 1.0 - 2.0**-53, 2.0, 0.5, 5e-324, 1e-310, np.finfo(float).max]),
    ])
    bad = [x for x in xs.tolist() if f(x) != _cr(x)]
    assert not bad, bad[:5]


def test_log_cr_special_values():
    f = _log_cr()
    assert f(1.0) == 0.0
    assert f(0.0) == -math.inf
    assert f(math.inf) == math.inf
    assert math.isnan(f(-1.0))
    assert math.isnan(f(math.nan))


def test_glibc_log_is_not_correctly_rounded_here():
    """Why FAITHFUL uses log_cr: glibc (the reference's math.log) misrounds
    a small fraction of inputs, which no GPU log can reproduce bit for bit."""
    rng = np.random.default_rng(1)
    xs = rng.uniform(0.2, 5.0, 20000).tolist()
    mis = sum(1 for x in xs if math.log(x) != _cr(x))
    assert 0 < mis < 0.01 * len(xs)
