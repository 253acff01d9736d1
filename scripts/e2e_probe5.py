"""Host<->device probe of the cfg5 (5.4 GB state) end-to-end volume path:
raw pinned H2D, raw D2H, both directions concurrently (the PCIe floor of the
path), and fdg_volume_host at several chunk counts. CUDA events, best / mean
of 5 after 2 warm-ups. Prints one JSON line."""

import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2112_10517_b200 import _native as N  # noqa: E402
from paper_2112_10517_b200 import workloads  # noqa: E402
from paper_2112_10517_b200.device import device_mesh_for  # noqa: E402


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        out.append(a.elapsed_time(b))
    return {"min": min(out), "mean": statistics.mean(out)}


def main():
    setup, u, cfg = workloads.build_device(5, kernel="batched")
    dm = device_mesh_for(setup)
    s = cfg.scheme()
    u_pin = N.pinned_empty(dm.shape)
    o_pin = N.pinned_empty(dm.shape)
    u_pin.copy_(u)
    torch.cuda.synchronize()
    d_in = dm.empty()
    d_out = dm.empty()
    side = torch.cuda.Stream()
    res = {"bytes_each_way": u_pin.numel() * 8}
    res["h2d"] = timed(lambda: d_in.copy_(u_pin, non_blocking=True))
    res["d2h"] = timed(lambda: o_pin.copy_(d_out, non_blocking=True))

    def both():
        ev = torch.cuda.Event()
        with torch.cuda.stream(side):
            o_pin.copy_(d_out, non_blocking=True)
            ev.record()
        d_in.copy_(u_pin, non_blocking=True)
        torch.cuda.current_stream().wait_event(ev)

    res["h2d_and_d2h_concurrent"] = timed(both)
    res["kernel_only"] = timed(lambda: dm.volume(u, s, out=d_out))
    for n in (4, 8, 16, 24, 32):
        res["volume_host_chunks_%d" % n] = timed(lambda n=n: dm.volume_host(u_pin, s, o_pin, n_chunks=n))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
