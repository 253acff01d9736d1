"""paper_2112_10517_b200 -- B200-native (sm_100a, FP64) flux-differencing DGSEM
volume integral and RHS for the compressible Euler equations: the hot path of
arXiv 2112.10517, behind the reference artifact's (`fluxdg`) own call
signatures. All arithmetic of the path runs in libfdg.so (include/fdg.h);
this package is the host-side mirror of the reference's interface.
"""

from .discretization import (
    KERNELS,
    PRECOMPUTE_MODES,
    RhsConfig,
    SpatialSetup,
    build_setup,
    conserved_totals,
    entropy_rate,
    error_norm_l2,
    mesh_fluxdiff_volume,
    mesh_surface,
    rhs,
    surface_terms,
    volume_fluxdiff,
)
from .errors import (
    AdmissibilityError,
    BenchmarkError,
    ConfigurationError,
    DivergenceError,
    DomainError,
    FluxdgError,
    MeshError,
    NativeLibraryError,
    UnsupportedOperatorError,
)
from .euler import GasParams, cons2prim, prim2cons
from .fluxes import FluxCounter, count_guard
from .geometry import StructuredMesh, build_mesh, compute_metrics
from .operators import build_dsplit, gauss_operator, gauss_scatter_tables, lgl_operator, make_operator, node_lines, pair_table
from .timeint import RK54, SSPRK43, DeviceStepper, RKMethod, ShuOsherMethod, StepController, integrate, rk_step, stable_dt

__version__ = "0.1.0"
