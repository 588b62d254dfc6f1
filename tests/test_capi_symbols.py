"""The C-ABI library loads without a GPU and exports every symbol declared
in include/npcg.h, with the binding's declared signatures. CPU only: no
compute call is made here."""
import ctypes
import os
import re

import pytest

from paper_2305_16432_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "npcg.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(npcg_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = header_functions()
    for must in ("npcg_pattern_create", "npcg_spmv", "npcg_ldlt_apply_inverse", "npcg_gnn_build_factor",
                 "npcg_pcg_solve", "npcg_solver_create"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _native.load_library()
    missing = [n for n in header_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_every_symbol():
    assert set(header_functions()) == set(_native.SIGNATURES)


def test_abi_version_and_error_string_without_gpu():
    lib = _native.load_library()
    assert lib.npcg_abi_version() == 1
    assert isinstance(lib.npcg_last_error(), bytes)


def test_pattern_validation_errors_before_touching_the_device():
    """Invalid CSR is rejected with DimensionMismatchError (sparse.py:49-65)
    by the C side, without needing a GPU."""
    import numpy as np
    lib = _native.load_library()
    h = ctypes.c_void_p()
    rp = np.array([0, 2, 1], dtype=np.int64)
    ci = np.array([0, 1], dtype=np.int64)
    rc = lib.npcg_pattern_create(2, rp.ctypes.data, ci.ctypes.data, 0, ctypes.byref(h))
    assert rc == _native.ERR_DIMENSION
    rp = np.array([0, 2, 2], dtype=np.int64)
    ci = np.array([1, 0], dtype=np.int64)
    rc = lib.npcg_pattern_create(2, rp.ctypes.data, ci.ctypes.data, 0, ctypes.byref(h))
    assert rc == _native.ERR_DIMENSION
    with pytest.raises(Exception):
        _native.check(rc)


def test_struct_layouts_match_header():
    assert ctypes.sizeof(_native.SolveOpts) == 4 + 4 + 16 * 8 + 8 + 4 * 4
    assert ctypes.sizeof(_native.SolveReportC) == 11 * 8
    assert ctypes.sizeof(_native.GnnDesc) == 10 * 4  # + north_star, dim
    assert ctypes.sizeof(_native.PatternInfo) == 3 * 8 + 9 * 4 + 4
