"""Golden fixtures for the diagnostics reductions, from the REFERENCE package.

Like make_golden.py this imports the reference (`fluxdg`, read-only at
/root/reference/pkg/src) and runs only in the build container. It rebuilds
each small case's reference setup from the parameters recorded in
case_<name>.npz, takes that case's recorded states and reference RHS outputs,
and writes diagnostics.npz with, per case and state:

* cons_<case>_<state>          conserved_totals(u, setup)            discretization.py:1027-1031
* ent_<case>_<state>_<vf>_<sf> entropy_rate(u, rhs(u), setup)        discretization.py:1011-1024
* err_<case>                   error_norm_l2(u_rand, u_wave|1.01 u_rand, setup)   discretization.py:1033-1037
* dt_<case>_<state>            stable_dt(u, mesh, metrics, gas, p, StepController(0.5))  timeint.py:138-146

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_diagnostics.py
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from fluxdg import GasParams, build_mesh, build_setup, lgl_operator  # noqa: E402
from fluxdg.discretization import conserved_totals, entropy_rate, error_norm_l2  # noqa: E402
from fluxdg.timeint import StepController, stable_dt  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from tests.golden_io import CASES  # noqa: E402

GAS = GasParams(1.4)


def main():
    out = {}
    for name in CASES:
        c = dict(np.load(os.path.join(HERE, "case_%s.npz" % name)))
        dims = tuple(int(x) for x in c["dims"])
        bounds = tuple(float(x) for x in c["bounds"])
        mesh = build_mesh(dims, bounds=bounds, amplitude=float(c["amplitude"]))
        setup = build_setup(mesh, lgl_operator(int(c["p"])), GAS)
        states = [k[2:] for k in c if k.startswith("u_")]
        for s in states:
            u = c["u_" + s]
            out["cons_%s_%s" % (name, s)] = conserved_totals(u, setup)
            out["dt_%s_%s" % (name, s)] = np.array(
                stable_dt(u, mesh, setup.metrics, GAS, int(c["p"]), StepController(0.5))
            )
            for vf, sf in (("ranocha", "ranocha"), ("ranocha", "llf")):
                key = "rhs_%s_%s_%s" % (s, vf, sf)
                if key in c:
                    out["ent_%s_%s_%s_%s" % (name, s, vf, sf)] = np.array(entropy_rate(u, c[key], setup))
        u_exact = c["u_wave"] if "u_wave" in c else 1.01 * c["u_rand"]
        out["err_%s" % name] = error_norm_l2(c["u_rand"], u_exact, setup)
        print(name, "done")
    np.savez_compressed(os.path.join(HERE, "diagnostics.npz"), **out)


if __name__ == "__main__":
    main()
