"""Single-GPU evidence for the halo / interior overlap of the sharded RHS.

Rank r's slab of an N-rank partition of cfg5 (128^3) or cfg4 (48^3) is set
up on ONE GPU; the face-trace exchange is emulated on a side stream by the
same packing kernels plus device-to-device copies into the ghost buffer,
followed by a delay of ``--comm-us`` (a stand-in for the NCCL latency).
Timed with CUDA events (median of 20):
  whole      one launch over the slab, ghosts ready
  split      interior launch, then the two boundary-plane launches
  serial     exchange, then the whole launch (the round-1 order)
  overlapped exchange on the side stream || interior, then boundary
The overlapped figure staying at `split` while `serial` grows by the
exchange time is the off-critical-path evidence; results must be bitwise.

  python scripts/overlap_probe.py [--cfg 5] [--world 8] [--comm-us 40]
"""

import argparse
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2112_10517_b200 import workloads
    from paper_2112_10517_b200.device import DeviceMesh
    from paper_2112_10517_b200.parallel import slab_partition

    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=5)
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--comm-us", type=float, default=40.0)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--reserve", type=int, default=8, help="SMs left free in interface launches")
    a = ap.parse_args()
    setup, u_full, config = workloads.build_device(a.cfg, kernel="batched")
    part = slab_partition(setup, a.rank, a.world)
    dm = DeviceMesh(setup, partition=part)
    dm.reserve_sms(a.reserve)
    lo, hi = part["lo"], part["hi"]
    u = u_full[lo:hi].clone()
    F, n = part["plane"], hi - lo
    d, p1 = setup.d, setup.op.degree + 1
    fn, nvar = p1 ** (d - 1), d + 2
    # ghosts from the true neighbours' planes (periodic): packed from u_full
    nxt_first = torch.arange(hi % setup.n_elements, hi % setup.n_elements + F, device="cuda", dtype=torch.int32)
    prv_last = torch.arange((lo - F) % setup.n_elements, (lo - F) % setup.n_elements + F, device="cuda",
                            dtype=torch.int32)
    ghost = torch.empty((2 * F, fn, nvar), dtype=torch.float64, device="cuda")
    stage = torch.empty_like(ghost)
    scheme = config.scheme()
    out = dm.empty()
    ref = dm.empty()
    main_s = torch.cuda.Stream() if os.environ.get("PROBE_MAIN_STREAM", "own") == "own" else torch.cuda.current_stream()
    torch.cuda.set_stream(main_s)
    side = torch.cuda.Stream()
    clock = torch.cuda.get_device_properties(0).clock_rate if hasattr(torch.cuda.get_device_properties(0), "clock_rate") else 1965000
    cycles = int(a.comm_us * 1e-6 * clock * 1e3)

    def exchange(stream):
        with torch.cuda.stream(stream):
            dm.pack_faces(u_full, nxt_first, 0, 0, stage[:F], stream=stream)
            dm.pack_faces(u_full, prv_last, 0, 1, stage[F:], stream=stream)
            torch.cuda._sleep(cycles)  # the wire
            ghost.copy_(stage)

    exchange(main_s)
    dm.rhs(u, scheme, out=ref, ghost_u=ghost)
    torch.cuda.synchronize()

    def timed(fn_):
        ts = []
        for _ in range(a.reps + 3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(main_s)
            fn_()
            e1.record(main_s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts[3:])

    def whole():
        dm.rhs(u, scheme, out=out, ghost_u=ghost)

    def split():
        dm.rhs(u, scheme, out=out, lo=F, hi=n - F)
        dm.rhs(u, scheme, out=out, ghost_u=ghost, ranges=[(0, F), (n - F, n)])

    def serial():
        exchange(main_s)
        whole()

    def overlapped():
        # the real order (parallel.split_launch): pack on the compute stream,
        # the wire (NCCL) on its own stream beside the interior launch
        dm.pack_faces(u_full, nxt_first, 0, 0, stage[:F], stream=main_s)
        dm.pack_faces(u_full, prv_last, 0, 1, stage[F:], stream=main_s)
        ev = torch.cuda.Event()
        ev.record(main_s)
        side.wait_event(ev)
        with torch.cuda.stream(side):
            torch.cuda._sleep(cycles)  # the wire
            ghost.copy_(stage)
        dm.rhs(u, scheme, out=out, lo=F, hi=n - F)
        done = torch.cuda.Event()
        done.record(side)
        main_s.wait_event(done)
        dm.rhs(u, scheme, out=out, ghost_u=ghost, ranges=[(0, F), (n - F, n)])

    def exchange_only():
        exchange(main_s)

    def interior_only():
        dm.rhs(u, scheme, out=out, lo=F, hi=n - F)

    res = {"cfg": a.cfg, "world": a.world, "rank": a.rank, "slab_elements": n, "plane": F, "reserve_sms": a.reserve,
           "comm_emulated_us": a.comm_us}
    for name, f in (("exchange_only", exchange_only), ("interior_only", interior_only), ("whole", whole),
                    ("split", split), ("serial", serial), ("overlapped", overlapped)):
        res[name + "_ms"] = timed(f)
        if name not in ("exchange_only", "interior_only"):
            res[name + "_bitwise"] = bool(torch.equal(out, ref))
    res["hidden_fraction"] = (res["serial_ms"] - res["overlapped_ms"]) / max(res["exchange_only_ms"], 1e-9)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
