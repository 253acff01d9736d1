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


def test_fast_table_log_accuracy_and_header():
    """log_tab (the per-node table log of the FAST volume-only kernels,
    csrc/fdg_fast.cuh): the device algorithm re-run in exactly rounded
    arithmetic stays within 1.5 ulp of max(|log x|, 2^-7) of 60-digit logs,
    and the committed table is what scripts/gen_logtab_fast.py generates."""
    import importlib.util
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("gen_logtab_fast", os.path.join(root, "scripts", "gen_logtab_fast.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    with open(gen.HEADER) as fh:
        assert fh.read() == gen.header_text()
    worst, n = gen.max_error_ulps(n=1500, seed=7)
    assert n > 4000 and worst < 1.6
