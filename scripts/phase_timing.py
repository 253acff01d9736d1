"""Per-phase SM cycles of the element kernel (needs a -DFDG_PHASE_TIMING build via FDG_LIB)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2112_10517_b200 import _native as N  # noqa: E402
from paper_2112_10517_b200 import workloads  # noqa: E402
from paper_2112_10517_b200.device import DeviceMesh  # noqa: E402

L = N.lib()
L.fdg_debug_phase_cycles.argtypes = [ctypes.c_void_p, ctypes.c_int]
names = ["load", "stage", "dir0", "dir1", "dir2", "epilogue", "-", "gap"]
for dims in [(16, 16, 16), (64, 64, 64)]:
    setup, u_host, cfg = workloads.build(2, dims=dims, kernel="batched")
    dm = DeviceMesh(setup)
    u = torch.as_tensor(u_host, device="cuda")
    out = dm.empty()
    s = cfg.scheme()
    dm.volume(u, s, out=out)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 8)()
    L.fdg_debug_phase_cycles(buf, 1)
    for _ in range(5):
        dm.volume(u, s, out=out)
    torch.cuda.synchronize()
    L.fdg_debug_phase_cycles(buf, 1)
    tot = sum(buf)
    batches = 5 * (setup.n_elements // 8)
    print(dims, "cycles per batch per CTA:", {n: round(buf[i] / batches) for i, n in enumerate(names) if buf[i]},
          "total", round(tot / batches))
