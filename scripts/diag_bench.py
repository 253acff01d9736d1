"""Time the fdg_diagnostic reductions (CUDA events, mean of --reps calls after
warm-up) on a BASELINE configuration and report achieved HBM GB/s against the
algorithmic bytes (every input state read once: 8 (d+2) B per node per state,
plus 8 B per node of J on curved meshes). One JSON line per kind.

    python scripts/diag_bench.py [--k 5] [--dims 128,128,128] [--reps 20]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2112_10517_b200 import workloads  # noqa: E402
from paper_2112_10517_b200.device import (  # noqa: E402
    DIAG_CONSERVED,
    DIAG_DT,
    DIAG_ENTROPY,
    DIAG_ERROR_SQ,
    device_mesh_for,
)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=5)
    ap.add_argument("--dims", default=None)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    dims = tuple(int(x) for x in a.dims.split(",")) if a.dims else None
    setup, u, _ = workloads.build(a.k, dims=dims)
    dm = device_mesh_for(setup)
    ud = torch.as_tensor(u, device="cuda")
    vd = ud * 1.001
    del u
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
    except OSError:
        pass
    peak = float(peaks.get("hbm_gbs", 0.0)) or None
    nodes = ud.shape[0] * ud.shape[1]
    row = 8 * ud.shape[2]
    jac = 0 if dm.cartesian else 8
    for name, kind, b, nstates in (
        ("conserved", DIAG_CONSERVED, None, 1),
        ("entropy", DIAG_ENTROPY, vd, 2),
        ("error_sq", DIAG_ERROR_SQ, vd, 2),
        ("dt", DIAG_DT, None, 1),
    ):
        for _ in range(3):
            dm.diagnostic(kind, ud, b)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(a.reps):
            dm.diagnostic(kind, ud, b)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / a.reps
        nbytes = nodes * (row * nstates + jac)
        gbs = nbytes / (ms * 1e-3) / 1e9
        print(
            json.dumps(
                {
                    "diagnostic": name,
                    "config": "cfg%d %s" % (a.k, "x".join(str(x) for x in (dims or workloads.CONFIGS[a.k]["dims"]))),
                    "ms": ms,
                    "algorithmic_bytes": nbytes,
                    "gbs": gbs,
                    "hbm_frac": None if peak is None else gbs / peak,
                    "l2": "state %.1f GB >> 126 MB L2" % (nodes * row / 1e9),
                }
            )
        )


if __name__ == "__main__":
    main()
