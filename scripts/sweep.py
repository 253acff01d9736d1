"""Timing sweep of the device kernels. ms: each launch alone (CUDA events, L2
flushed before it); ms_graph: K launches over rotating (u, out) replicas
(> 3x L2) in one CUDA graph, total / K.

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


def time_graph(make_step, n_rep, reps):
    """K = reps steps over n_rep rotating (u, out) replicas in one CUDA graph."""
    for i in range(3):
        make_step(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            make_step(i)
    g.replay()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


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
        (5, None, "ranocha", "batched", "primitives_and_logs", "rhs"),
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
        n_rep = max(2, -(-3 * 126 * 2**20 // (2 * u_host.nbytes)))
        us = [u] + [u.clone() for _ in range(n_rep - 1)]
        outs = [out] + [dm.empty() for _ in range(n_rep - 1)]
        if what == "volume":
            def stepf(i):
                dm.volume(us[i % n_rep], s, out=outs[i % n_rep])
        else:
            def stepf(i):
                dm.rhs(us[i % n_rep], s, out=outs[i % n_rep])
        ms_graph = time_graph(stepf, n_rep, args.reps)
        del us, outs
        nodes = u_host.shape[0] * u_host.shape[1]
        mult = 2 if not setup.metrics.cartesian else 1
        print(json.dumps({
            "cfg": cfg, "dims": list(setup.mesh.dims), "p": setup.op.degree, "flux": flux, "kernel": kernel,
            "precompute": pre, "what": what, "ms": ms, "nodes_per_s": nodes / (ms * 1e-3),
            "hbm_frac_vol": (80.0 * mult * nodes / (ms * 1e-3) / 1e9) / 6547.8,
            "ms_graph": ms_graph, "nodes_per_s_graph": nodes / (ms_graph * 1e-3),
        }), flush=True)
        del dm, u, out, u_host, setup


if __name__ == "__main__":
    main()
