"""Time on-device geometry (fdg_build_geometry) against the host setup for a
BASELINE mesh: CUDA events around the kernel, wall clock around the host
build_setup. One JSON line.

    python scripts/geom_bench.py [--k 4] [--dims 48,48,48] [--host]
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2112_10517_b200 import workloads  # noqa: E402
from paper_2112_10517_b200.geometry import build_mesh, device_geometry  # noqa: E402
from paper_2112_10517_b200.discretization import build_setup  # noqa: E402
from paper_2112_10517_b200.euler import GasParams  # noqa: E402
from paper_2112_10517_b200.operators import lgl_operator  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--dims", default=None)
    ap.add_argument("--host", action="store_true")
    a = ap.parse_args()
    c = workloads.CONFIGS[a.k]
    dims = tuple(int(x) for x in a.dims.split(",")) if a.dims else c["dims"]
    mesh = build_mesh(dims, bounds=(-1.0, 1.0), amplitude=c["amplitude"])
    op = lgl_operator(c["p"])
    device_geometry(mesh, op)  # warm-up (module load)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    coords, ja, jac = device_geometry(mesh, op)
    e.record()
    torch.cuda.synchronize()
    rec = {"config": "cfg%d %s" % (a.k, "x".join(map(str, dims))), "device_ms": s.elapsed_time(e),
           "bytes_written": sum(t.numel() * 8 for t in (coords, ja, jac) if t is not None)}
    if a.host:
        t0 = time.perf_counter()
        build_setup(mesh, op, GasParams(1.4))
        rec["host_build_setup_s"] = time.perf_counter() - t0
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
