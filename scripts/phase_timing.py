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
    batches = 5 * (setup.n_elements // 4)  # EPB = 4 (64-thread CTAs at N = 3)
    print(dims, "cycles per batch per CTA:", {n: round(buf[i] / batches) for i, n in enumerate(names) if buf[i]},
          "total", round(tot / batches))

# per-CTA start/end (globaltimer) of one cfg2 launch
L.fdg_debug_cta_ns.argtypes = [ctypes.c_void_p, ctypes.c_int]
setup, u_host, cfg = workloads.build(2, kernel="batched")
dm = DeviceMesh(setup)
u = torch.as_tensor(u_host, device="cuda")
out = dm.empty()
s = cfg.scheme()
for _ in range(3):
    dm.volume(u, s, out=out)
torch.cuda.synchronize()
flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
flush.sum()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); dm.volume(u, s, out=out); e1.record(); torch.cuda.synchronize()
n = 1024
buf = (ctypes.c_ulonglong * (3 * n))()
L.fdg_debug_cta_ns(buf, n)
import numpy as np
a = np.array(buf[:], dtype=np.float64).reshape(n, 3)
t0 = a[:, 0].min()
st, en, sm = a[:, 0] - t0, a[:, 1] - t0, a[:, 2].astype(int)
print("event ms %.4f | CTA start: min %.0f med %.0f max %.0f ns | end: min %.0f med %.0f max %.0f ns | dur med %.0f max %.0f"
      % (e0.elapsed_time(e1), st.min(), np.median(st), st.max(), en.min(), np.median(en), en.max(), np.median(en - st), (en - st).max()))
per_sm = np.bincount(sm, minlength=148)
print("CTAs per SM: histogram", {int(k): int(v) for k, v in zip(*np.unique(per_sm, return_counts=True))})
sm_end = np.zeros(148)
for i in range(n):
    sm_end[sm[i]] = max(sm_end[sm[i]], en[i])
for c in sorted(set(per_sm)):
    sel = per_sm == c
    if sel.any():
        print("  SMs with %d CTAs: %d, last CTA end med %.0f max %.0f ns" % (c, sel.sum(), np.median(sm_end[sel]), sm_end[sel].max()))
