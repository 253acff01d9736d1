"""Timing sweep of the device kernels (CUDA events, L2 flushed between launches).

python scripts/sweep.py [--quick]   -> one JSON line per case on stdout
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2112_10517_b200 import workloads  # noqa: E402
from paper_2112_10517_b200.device import DeviceMesh  # noqa: E402


def time_launch(fn, reps, flush):
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(reps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(reps)]
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    for i in range(reps):
        flush.sum()
        starts[i].record()
        fn()
        ends[i].record()
    torch.cuda.synchronize()
    return statistics.median(s.elapsed_time(e) for s, e in zip(starts, ends))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="all")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    cases = [
        # (cfg, dims, flux, kernel, precompute, what)
        (2, None, "ranocha", "batched", "primitives_and_logs", "volume"),
        (2, (32, 32, 32), "ranocha", "batched", "primitives_and_logs", "volume"),
        (2, (64, 64, 64), "ranocha", "batched", "primitives_and_logs", "volume"),
        (5, None, "ranocha", "batched", "primitives_and_logs", "volume"),
        (5, None, "shima", "batched", "none", "volume"),
        (2, None, "ranocha", "batched", "none", "volume"),
        (2, None, "ranocha", "reference", "none", "volume"),
        (2, None, "ranocha", "batched", "primitives_and_logs", "rhs"),
        (3, None, "chandrashekar", "batched", "primitives_and_logs", "volume"),
        (3, None, "ranocha", "batched", "primitives_and_logs", "volume"),
        (4, None, "kennedy_gruber", "batched", "none", "volume"),
        (4, None, "kennedy_gruber", "batched", "none", "rhs"),
        (4, None, "ranocha", "batched", "primitives_and_logs", "volume"),
        (1, None, "ranocha", "batched", "primitives_and_logs", "rhs"),
    ]
    if args.cases != "all":
        keep = set(int(x) for x in args.cases.split(","))
        cases = [c for i, c in enumerate(cases) if i in keep]
    for cfg, dims, flux, kernel, pre, what in cases:
        setup, u_host, config = workloads.build(cfg, dims=dims, kernel=kernel, volume_flux=flux, precompute=pre)
        dm = DeviceMesh(setup)
        u = torch.as_tensor(u_host, device="cuda")
        out = dm.empty()
        s = config.scheme()
        fn = (lambda: dm.volume(u, s, out=out)) if what == "volume" else (lambda: dm.rhs(u, s, out=out))
        ms = time_launch(fn, args.reps, flush)
        nodes = u_host.shape[0] * u_host.shape[1]
        mult = 2 if not setup.metrics.cartesian else 1
        print(json.dumps({
            "cfg": cfg, "dims": list(setup.mesh.dims), "p": setup.op.degree, "flux": flux, "kernel": kernel,
            "precompute": pre, "what": what, "ms": ms, "nodes_per_s": nodes / (ms * 1e-3),
            "hbm_frac_vol": (80.0 * mult * nodes / (ms * 1e-3) / 1e9) / 6547.8,
        }), flush=True)
        del dm, u, out, u_host, setup


if __name__ == "__main__":
    main()
