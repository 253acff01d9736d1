"""Golden fixtures of the reference's benchmark initial conditions and of a
short run of its simulation protocol (harness.py:183-240, 271-345, 445-477).
Build container only (imports /root/reference); writes tests/golden/ics.npz.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_ics.py
"""

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from fluxdg import harness as H  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rec = {}
    for d in (2, 3):
        cfg = H.RunConfig(d=d, p=3, elements=8 if d == 2 else 4, n_steps=3)
        run = H.build_run(cfg)
        x = run.setup.coords
        rec["coords_%dd" % d] = x
        rec["vortex_%dd" % d] = H.vortex_primitives(x, 0.0, 20.0, 1.4)
        rec["vortex_t_%dd" % d] = H.vortex_primitives(x, 0.7, 20.0, 1.4)
        rec["sinus_%dd" % d] = H.sinusoidal_primitives(x, 1.4)
        rec["free_%dd" % d] = H.free_stream_primitives(x)
        rec["random_%dd" % d] = H.random_primitives(x, 3)
        rec["u0_%dd" % d] = run.u0
        res = H.run_simulation(run)
        rec["final_%dd" % d] = res.fields
        rec["t_%dd" % d] = np.array(res.t)
        rec["err_%dd" % d] = res.error_l2
        rec["dt0_%dd" % d] = np.array(H.stable_dt(run.u0, run.mesh, run.setup.metrics, run.gas, 3,
                                                  H.StepController(cfl=0.5)))
    np.savez_compressed(os.path.join(HERE, "ics.npz"), **rec)
    print("ics done")


if __name__ == "__main__":
    main()
