"""Quick FAST-path accuracy check against the oracle (variant libs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2112_10517_b200 import RhsConfig, mesh_fluxdiff_volume, rhs, workloads  # noqa: E402

CFG = int(os.environ.get("CHECK_CFG", "2"))  # BASELINE config whose degree the variant lib holds
for cfg, dims in ((CFG, (4, 4, 4)), (CFG, (6, 5, 4))):
    setup, u, _ = workloads.build(cfg, dims=dims)
    for pre in ("primitives_and_logs", "none"):
        c = RhsConfig(volume_flux="ranocha", surface_flux="llf", precompute=pre, kernel="batched")
        vol = mesh_fluxdiff_volume(u, setup, c)
        vref = oracle.volume(u, setup, "ranocha", pre)
        du = rhs(u, setup, c)
        dref = oracle.rhs(u, setup, "ranocha", "llf", pre)
        sref = oracle.surface(u, setup, "llf")
        scale = max(np.abs(vref).max(), np.abs(sref).max())
        print(dims, pre, "vol rel %.2e" % (np.abs(vol - vref).max() / np.abs(vref).max()),
              "rhs rel(cancel-aware) %.2e" % (np.abs(du - dref).max() / scale))
