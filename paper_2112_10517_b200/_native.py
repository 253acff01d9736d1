"""ctypes binding of libfdg.so (include/fdg.h).

The product path has no CPU fallback: if the library is missing or fails to
load, every entry point raises NativeLibraryError.
"""

import ctypes
import os

from .errors import ConfigurationError, NativeLibraryError, UnsupportedOperatorError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FDG_LIB") or os.path.join(HERE, "libfdg.so")  # FDG_LIB: tuning variants only

FLUX_IDS = {
    "central": 0,
    "shima": 1,
    "ranocha": 2,
    "kennedy_gruber": 3,
    "chandrashekar": 4,
    "llf": 5,
    "hll": 6,
}
PRECOMPUTE_IDS = {"none": 0, "primitives": 1, "primitives_and_logs": 2}
MODE_IDS = {"reference": 0, "batched": 1}  # RhsConfig.kernel -> FAITHFUL / FAST

FDG_OK, FDG_ERR_CONFIG, FDG_ERR_UNSUPPORTED, FDG_ERR_CUDA, FDG_ERR_ARG = range(5)


class MeshDesc(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int32),
        ("degree", ctypes.c_int32),
        ("n_elem", ctypes.c_int64),
        ("elem_base", ctypes.c_int64),
        ("gamma", ctypes.c_double),
        ("inv_gamma_minus_one", ctypes.c_double),
        ("dsplit", ctypes.c_void_p),
        ("weights", ctypes.c_void_p),
        ("cartesian", ctypes.c_int32),
        ("areas", ctypes.c_double * 3),
        ("jac_const", ctypes.c_double),
        ("ja", ctypes.c_void_p),
        ("jac", ctypes.c_void_p),
        ("plus", ctypes.c_void_p),
        ("minus", ctypes.c_void_p),
        ("ghost_nrm", ctypes.c_void_p),
    ]


class GeometryDesc(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int32),
        ("degree", ctypes.c_int32),
        ("dims", ctypes.c_int32 * 3),
        ("lo", ctypes.c_double * 3),
        ("hi", ctypes.c_double * 3),
        ("amplitude", ctypes.c_double),
        ("nodes", ctypes.c_void_p),
        ("dmat", ctypes.c_void_p),
    ]


class GaussDesc(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int32),
        ("degree", ctypes.c_int32),
        ("n_elem", ctypes.c_int64),
        ("gamma", ctypes.c_double),
        ("inv_gamma_minus_one", ctypes.c_double),
        ("boundary_interp", ctypes.c_void_p),
        ("vv", ctypes.c_void_p),
        ("cvol", ctypes.c_void_p),
        ("cface", ctypes.c_void_p),
        ("lift", ctypes.c_void_p),
        ("ja", ctypes.c_void_p),
        ("jac", ctypes.c_void_p),
        ("plus", ctypes.c_void_p),
        ("minus", ctypes.c_void_p),
    ]


class Scheme(ctypes.Structure):
    _fields_ = [
        ("volume_flux", ctypes.c_int32),
        ("surface_flux", ctypes.c_int32),
        ("precompute", ctypes.c_int32),
        ("mode", ctypes.c_int32),
    ]


class Stage(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("index", ctypes.c_uint32),
        ("a", ctypes.c_double),
        ("b", ctypes.c_double),
        ("cdt", ctypes.c_double),
        ("dt", ctypes.c_double),
    ]


class StatusRec(ctypes.Structure):
    _fields_ = [("first_bad", ctypes.c_int64), ("bad_stage", ctypes.c_int32), ("pad", ctypes.c_int32)]


EXPORTS = (
    "fdg_abi_version",
    "fdg_last_error",
    "fdg_supported",
    "fdg_launch_count",
    "fdg_host_alloc",
    "fdg_host_free",
    "fdg_mesh_create",
    "fdg_mesh_destroy",
    "fdg_volume",
    "fdg_volume_range",
    "fdg_volume_host",
    "fdg_surface",
    "fdg_rhs",
    "fdg_rhs_range",
    "fdg_rk_stage",
    "fdg_rk_stage_range",
    "fdg_gate",
    "fdg_reset_status",
    "fdg_read_status",
    "fdg_mesh_set_reserve_sms",
    "fdg_pack_faces",
    "fdg_fp64_probe",
    "fdg_gauss_create",
    "fdg_gauss_destroy",
    "fdg_gauss_project",
    "fdg_gauss_rhs",
    "fdg_gauss_gate",
    "fdg_gauss_reset_status",
    "fdg_gauss_read_status",
)

_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            "libfdg.so not found at %s; build it with `python -c \"import __graft_entry__ as g; g.build()\"`"
            % LIB_PATH
        )
    try:
        L = ctypes.CDLL(LIB_PATH)
    except OSError as err:
        raise NativeLibraryError("libfdg.so failed to load: %s" % err) from err
    vp, i32, P = ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER
    L.fdg_abi_version.restype = ctypes.c_int
    L.fdg_last_error.restype = ctypes.c_char_p
    L.fdg_supported.argtypes = [i32, i32]
    L.fdg_launch_count.restype = ctypes.c_ulonglong
    L.fdg_host_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]
    L.fdg_host_free.argtypes = [ctypes.c_void_p]
    L.fdg_mesh_create.argtypes = [P(MeshDesc), P(vp)]
    L.fdg_mesh_destroy.argtypes = [vp]
    L.fdg_mesh_destroy.restype = None
    L.fdg_volume.argtypes = [vp, P(Scheme), vp, vp, vp]
    L.fdg_volume_range.argtypes = [vp, P(Scheme), vp, vp, ctypes.c_int64, ctypes.c_int64, vp]
    L.fdg_volume_host.argtypes = [vp, P(Scheme), vp, vp, vp, vp, i32, vp]
    L.fdg_surface.argtypes = [vp, P(Scheme), vp, vp, vp, vp]
    L.fdg_rhs.argtypes = [vp, P(Scheme), vp, vp, vp, vp]
    L.fdg_rk_stage.argtypes = [vp, P(Scheme), P(Stage), vp, vp, vp, vp, vp, vp]
    i64 = ctypes.c_int64
    L.fdg_rhs_range.argtypes = [vp, P(Scheme), vp, vp, vp, i64, i64, i64, i64, vp]
    L.fdg_rk_stage_range.argtypes = [vp, P(Scheme), P(Stage), vp, vp, vp, vp, vp, i64, i64, i64, i64, vp]
    L.fdg_gate.argtypes = [vp, vp, vp]
    L.fdg_reset_status.argtypes = [vp, vp]
    L.fdg_read_status.argtypes = [vp, P(StatusRec), vp]
    L.fdg_mesh_set_traversal.argtypes = [vp, vp, ctypes.c_int64]
    L.fdg_mesh_set_reserve_sms.argtypes = [vp, i32]
    L.fdg_build_geometry.argtypes = [P(GeometryDesc), vp, vp, vp, vp]
    L.fdg_diagnostic.argtypes = [vp, i32, vp, vp, vp, vp]
    L.fdg_pack_faces.argtypes = [vp, vp, i32, i32, i32, i32, i32, vp, vp]
    L.fdg_fp64_probe.argtypes = [P(ctypes.c_double), vp]
    L.fdg_gauss_create.argtypes = [P(GaussDesc), P(vp)]
    L.fdg_gauss_destroy.argtypes = [vp]
    L.fdg_gauss_project.argtypes = [vp, vp, vp, vp, vp]
    L.fdg_gauss_rhs.argtypes = [vp, P(Scheme), vp, vp, vp, vp, vp, vp]
    L.fdg_gauss_gate.argtypes = [vp, vp, vp]
    L.fdg_gauss_reset_status.argtypes = [vp, vp]
    L.fdg_gauss_read_status.argtypes = [vp, P(StatusRec), vp]
    if L.fdg_abi_version() != 1:
        raise NativeLibraryError("libfdg.so ABI version %d, expected 1" % L.fdg_abi_version())
    _lib = L
    return L


def check(rc):
    if rc == FDG_OK:
        return
    msg = lib().fdg_last_error().decode("utf-8", "replace")
    if rc == FDG_ERR_CONFIG:
        raise ConfigurationError(msg)
    if rc == FDG_ERR_UNSUPPORTED:
        raise UnsupportedOperatorError(msg)
    raise NativeLibraryError(msg)


def launch_count():
    return int(lib().fdg_launch_count())


def pinned_empty(shape, dtype="float64"):
    """torch CPU tensor on a cudaHostAlloc buffer (fdg_host_alloc), freed with
    the tensor: the host-buffer path's copies run at the copy engines' full
    rate on it (profiles/r01_e2e.md)."""
    import weakref

    import numpy as np
    import torch

    dt = np.dtype(dtype)
    n = int(np.prod(shape))
    ptr = ctypes.c_void_p()
    check(lib().fdg_host_alloc(n * dt.itemsize, ctypes.byref(ptr)))
    buf = (ctypes.c_char * max(n * dt.itemsize, 1)).from_address(ptr.value)
    arr = np.frombuffer(buf, dtype=dt, count=n).reshape(shape)
    t = torch.from_numpy(arr)
    weakref.finalize(arr, lib().fdg_host_free, ptr)
    return t


def fp64_peak_tflops(stream=None):
    out = ctypes.c_double(0.0)
    check(lib().fdg_fp64_probe(ctypes.byref(out), stream))
    return out.value
