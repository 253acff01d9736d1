"""Volume-integral throughput and roofline fraction per polynomial degree:
3D Cartesian meshes, N = 3..7, Ranocha (log tables) and Shima, the cfg5 state
generator (noisy density wave) on meshes of ~55-134 M nodes (>= 17x L2, so no
L2 flush is needed between launches). One JSON line per case on stdout.

Roofline: bytes/node = 80; flop/node = 1.5 N (pair + 22) + 19
with pair = 69 (Ranocha, log tables, log branch) or 38 (Shima), +0 logs for
Shima (17 per node); bound = the slower of flops at the measured DFMA peak
(fdg_probe) and bytes at MEASURED_PEAKS.json hbm_gbs.

python scripts/degree_sweep.py [--steps 10] [--warmup 3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2112_10517_b200 import _native as N  # noqa: E402
from paper_2112_10517_b200 import workloads  # noqa: E402
from paper_2112_10517_b200.device import device_mesh_for  # noqa: E402
from paper_2112_10517_b200.operators import lgl_operator  # noqa: E402

DIMS = {3: (128, 128, 128), 4: (80, 80, 80), 5: (64, 64, 64), 6: (56, 56, 56), 7: (48, 48, 48)}


def flop_per_node(p, flux):
    pair = {"ranocha": 69, "shima": 38}[flux]
    node = 19 if flux == "ranocha" else 17
    return 1.5 * p * (pair + 22) + node


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--degrees", default="3,4,5,6,7")
    ap.add_argument("--fluxes", default="ranocha,shima")
    ap.add_argument("--what", default="volume", choices=["volume", "rhs"],
                    help="rhs: the full RHS (Rusanov interfaces), fractions against the volume integral's bound")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    hbm, peak_src = bench._peaks()
    fp64_peak = N.fp64_peak_tflops()
    stream = torch.cuda.current_stream()
    for p in [int(x) for x in args.degrees.split(",")]:
        for flux in args.fluxes.split(","):
            setup, u, config = workloads.build_device(5, dims=DIMS[p], kernel="batched", volume_flux=flux,
                                                      op=lgl_operator(p))
            dm = device_mesh_for(setup)
            scheme = config.scheme()
            out = dm.empty()
            launch = dm.rhs if args.what == "rhs" else dm.volume
            for _ in range(args.warmup):
                launch(u, scheme, out=out)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(args.steps):
                launch(u, scheme, out=out)
            b.record(stream)
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / args.steps
            nodes = setup.n_elements * setup.n_nodes
            rate = nodes / (ms * 1e-3)
            flop = flop_per_node(p, flux)
            hbm_frac = 80.0 * rate / 1e9 / hbm
            fp_frac = flop * rate / 1e12 / fp64_peak
            print(json.dumps({
                "what": args.what, "N": p, "dims": DIMS[p], "flux": flux, "precompute": config.precompute, "nodes": nodes,
                "state_mb": u.numel() * 8 / 1e6, "ms": ms, "nodes_per_s": rate,
                "flop_per_node": flop, "hbm_frac": hbm_frac, "fp64_frac": fp_frac,
                "bound": "fp64" if fp_frac > hbm_frac else "hbm", "roofline_frac": max(hbm_frac, fp_frac),
                "hbm_peak_gbs": hbm, "fp64_peak_tflops": fp64_peak, "peak_source": peak_src,
            }), flush=True)
            del u, out, dm, setup
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
