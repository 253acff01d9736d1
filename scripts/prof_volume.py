"""Small driver for ncu: a few volume-integral launches on one config."""
import argparse
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=2)
ap.add_argument("--kernel", default="batched")
ap.add_argument("--flux", default=None)
ap.add_argument("--launches", type=int, default=5)
ap.add_argument("--rhs", action="store_true")
ap.add_argument("--dims", default=None)
args = ap.parse_args()

import torch  # noqa: E402

from paper_2112_10517_b200 import workloads  # noqa: E402
from paper_2112_10517_b200.device import device_mesh_for  # noqa: E402

dims = tuple(int(x) for x in args.dims.split(",")) if args.dims else None
if args.cfg in (3, 5) and dims is None:
    # device-built geometry and state: no 22 GB host setup at 128^3
    setup, u, cfg = workloads.build_device(args.cfg, kernel=args.kernel, volume_flux=args.flux)
else:
    setup, u_host, cfg = workloads.build(args.cfg, dims=dims, kernel=args.kernel, volume_flux=args.flux)
    u = torch.as_tensor(u_host, device="cuda")
dm = device_mesh_for(setup)
out = dm.empty()
s = cfg.scheme()
for _ in range(args.launches):
    if args.rhs:
        dm.rhs(u, s, out=out)
    else:
        dm.volume(u, s, out=out)
torch.cuda.synchronize()
print("ok", float(out.abs().max()))
