"""The C-ABI library loads without a GPU and exports every symbol include/fdg.h declares."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fdg.h")
LIB = os.path.join(ROOT, "paper_2112_10517_b200", "libfdg.so")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_ ]+\**\s*\**(fdg_[a-z0-9_]+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("fdg_mesh_create", "fdg_volume", "fdg_surface", "fdg_rhs", "fdg_rk_stage", "fdg_gate"):
        assert must in names


@pytest.mark.skipif(not os.path.exists(LIB), reason="libfdg.so not built")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


@pytest.mark.skipif(not os.path.exists(LIB), reason="libfdg.so not built")
def test_abi_version_and_errors_without_gpu():
    from paper_2112_10517_b200 import _native as N

    L = N.lib()
    assert L.fdg_abi_version() == 1
    assert L.fdg_supported(3, 3) == 1
    assert L.fdg_supported(3, 8) == 0
    assert L.fdg_supported(1, 3) == 0
    # argument validation happens before any CUDA call
    handle = ctypes.c_void_p()
    desc = N.MeshDesc()
    desc.d, desc.degree = 3, 9
    rc = L.fdg_mesh_create(ctypes.byref(desc), ctypes.byref(handle))
    assert rc == N.FDG_ERR_UNSUPPORTED
    assert b"degree 9" in L.fdg_last_error()
    from paper_2112_10517_b200.errors import UnsupportedOperatorError

    with pytest.raises(UnsupportedOperatorError, match="degree 9"):
        N.check(rc)
