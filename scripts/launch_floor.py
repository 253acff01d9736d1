"""Fixed per-launch cost seen by CUDA events: a 1-element torch op, the volume
kernel on 8 elements (one CTA pair), and cfg2, each timed alone between events
after an L2 flush (median of 50)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2112_10517_b200 import workloads  # noqa: E402
from paper_2112_10517_b200.device import DeviceMesh  # noqa: E402

flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")


def t(fn, reps=50):
    for _ in range(5):
        fn()
    ts = []
    for _ in range(reps):
        flush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1000)
    return statistics.median(ts)


x = torch.zeros(1, device="cuda")
print("torch add_ 1 elem: %.2f us" % t(lambda: x.add_(1)))
print("empty event pair: %.2f us" % t(lambda: None))
for dims in [(2, 2, 2), (4, 4, 4), (8, 8, 8), (16, 16, 16), (16, 16, 32)]:
    setup, u_host, cfg = workloads.build(2, dims=dims, kernel="batched")
    dm = DeviceMesh(setup)
    u = torch.as_tensor(u_host, device="cuda")
    out = dm.empty()
    s = cfg.scheme()
    print("volume %s (%d elements): %.2f us" % (dims, setup.n_elements, t(lambda: dm.volume(u, s, out=out))))
