import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
from oracle import oracle
from paper_2112_10517_b200 import RhsConfig, mesh_fluxdiff_volume, rhs, workloads
for dims in ((4, 4, 4), (3, 2, 3)):
    setup, u, _ = workloads.build(3, dims=dims)
    for pre in ("primitives_and_logs", "none"):
        c = RhsConfig(volume_flux="chandrashekar", surface_flux="llf", precompute=pre, kernel="batched")
        vol = mesh_fluxdiff_volume(u, setup, c)
        vref = oracle.volume(u, setup, "chandrashekar", pre, variant="cr")
        du = rhs(u, setup, c)
        dref = oracle.rhs(u, setup, "chandrashekar", "llf", pre, variant="cr")
        print(dims, pre, "vol rel %.2e" % (np.abs(vol - vref).max() / np.abs(vref).max()), "rhs rel %.2e" % (np.abs(du - dref).max() / np.abs(vref).max()))
