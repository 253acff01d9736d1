"""Helpers to read the committed golden fixtures (tests/golden/*.npz).

The fixtures were produced by tests/golden/make_golden.py from the reference
package; nothing here imports the reference.
"""

import functools
import os
from types import SimpleNamespace

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

CASES = [
    "c2d_cart_p3",
    "c2d_curv_p3",
    "c2d_curv_p5",
    "c2d_cart_p1",
    "c2d_dim1_p3",
    "c3d_cart_p3",
    "c3d_curv_p4",
    "c3d_curv_p2",
    "c3d_cart_p7",
    "c3d_curv_p6",
]


@functools.lru_cache(maxsize=None)
def operators():
    return dict(np.load(os.path.join(GOLDEN, "operators.npz")))


@functools.lru_cache(maxsize=None)
def case(name):
    return dict(np.load(os.path.join(GOLDEN, "case_%s.npz" % name)))


@functools.lru_cache(maxsize=None)
def config(k):
    path = os.path.join(GOLDEN, "cfg%s.npz" % k)
    if not os.path.exists(path):
        return None
    return dict(np.load(path))


@functools.lru_cache(maxsize=None)
def golden_operator(p):
    """The reference's own lgl_operator(p) tables as an Operator1D (its exact
    bits, for tests that rebuild reference states or setups bit for bit)."""
    from paper_2112_10517_b200.operators import Operator1D

    ops = operators()
    return Operator1D(p, "lgl", ops["nodes_%d" % p], ops["weights_%d" % p], ops["D_%d" % p], ops["R_%d" % p])


def golden_setup(name, gamma=1.4):
    """Duck-typed setup built only from the reference's recorded arrays."""
    c = case(name)
    p = int(c["p"])
    ops = operators()
    d = len(c["dims"])
    gas = SimpleNamespace(gamma=gamma, inv_gamma_minus_one=1.0 / (gamma - 1.0))
    return SimpleNamespace(
        d=d,
        op=SimpleNamespace(weights=ops["weights_%d" % p], degree=p, n_nodes=p + 1, family="lgl"),
        dsplit=SimpleNamespace(matrix=ops["dsplit_%d" % p]),
        metrics=SimpleNamespace(
            ja=c["ja"],
            jac=c["jac"],
            cartesian=bool(c["cartesian"]),
            face_ja=tuple(c["face_ja_%d" % n] for n in range(d)),
        ),
        plus_neighbor=tuple(c["plus_%d" % n] for n in range(d)),
        gas=gas,
        n_elements=c["ja"].shape[0],
        n_nodes=c["ja"].shape[1],
    )


def states(name):
    c = case(name)
    return [k[2:] for k in c if k.startswith("u_")]


GAUSS_CASES = ["g2d_cart_p3", "g2d_curv_p3", "g3d_cart_p2", "g3d_curv_p3"]


@functools.lru_cache(maxsize=None)
def gauss_case(name):
    return dict(np.load(os.path.join(GOLDEN, "gauss_%s.npz" % name)))


def gauss_setup(name, gamma=1.4):
    """Duck-typed Gauss-family setup from the reference's recorded arrays."""
    from paper_2112_10517_b200.operators import Operator1D

    c = gauss_case(name)
    p = int(c["p"])
    d = len(c["dims"])
    gas = SimpleNamespace(gamma=gamma, inv_gamma_minus_one=1.0 / (gamma - 1.0))
    op = Operator1D(p, "gauss", c["nodes"], c["weights"], c["D"], c["R"])
    return SimpleNamespace(
        d=d, op=op, gas=gas, dsplit=None,
        metrics=SimpleNamespace(
            ja=c["ja"], jac=c["jac"], cartesian=bool(c["cartesian"]),
            face_ja=tuple(c["face_ja_%d" % n] for n in range(d)),
            elem_face_ja=tuple(c["elem_face_ja_%d" % n] for n in range(d)),
        ),
        plus_neighbor=tuple(c["plus_%d" % n] for n in range(d)),
        n_elements=c["ja"].shape[0], n_nodes=c["ja"].shape[1],
        mesh=SimpleNamespace(dims=tuple(int(x) for x in c["dims"]), d=d),
    )
