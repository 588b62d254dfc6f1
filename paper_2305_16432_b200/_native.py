"""ctypes binding of libnpcg.so (include/npcg.h) -- the only compute backend.

There is no CPU fallback: importing works without a GPU (so the host logic
and the ABI can be inspected on a CPU box), but every compute call goes
through ``lib()``, which raises ``NativeUnavailableError`` when the shared
library is missing or no sm_100a device is visible.
"""
from __future__ import annotations

import ctypes
import os

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NPCG_LIB") or os.path.join(_HERE, "libnpcg.so")

# status / error codes (npcg.h)
OK = 0
ERR_DIMENSION = 1
ERR_INVALID_FACTOR = 2
ERR_NOT_SPD = 3
ERR_BREAKDOWN = 4
ERR_CUDA = 5
ERR_DATA_FORMAT = 6
ERR_ARGUMENT = 7

STATUS_ACTIVE = 0
STATUS_CONVERGED = 1
STATUS_MAXITER = 2
STATUS_BREAKDOWN = 3

PATTERN_FACTOR = 1
MAX_THRESHOLDS = 16
MAX_BATCH = 256


class NativeUnavailableError(RuntimeError):
    """libnpcg.so is missing or no B200 (sm_100a) device is usable."""


class PatternInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nnz", ctypes.c_int64), ("nnz_lower", ctypes.c_int64),
                ("full_diagonal", ctypes.c_int32), ("structurally_symmetric", ctypes.c_int32),
                ("has_factor_schedule", ctypes.c_int32), ("levels_lower", ctypes.c_int32),
                ("levels_upper", ctypes.c_int32), ("chunks", ctypes.c_int32),
                ("chunk_rows", ctypes.c_int32), ("window", ctypes.c_int32),
                ("max_level_width", ctypes.c_int32)]


class GnnDesc(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("h", ctypes.c_int32), ("l", ctypes.c_int32),
                ("h_mp", ctypes.c_int32), ("l_mp", ctypes.c_int32), ("n_mp", ctypes.c_int32),
                ("normalize", ctypes.c_int32), ("with_x0_head", ctypes.c_int32),
                ("north_star", ctypes.c_int32), ("dim", ctypes.c_int32)]


class SolveOpts(ctypes.Structure):
    _fields_ = [("n_thresholds", ctypes.c_int32), ("thresholds", ctypes.c_double * MAX_THRESHOLDS),
                ("max_iter", ctypes.c_int64), ("absolute", ctypes.c_int32),
                ("check_every", ctypes.c_int32), ("profile", ctypes.c_int32),
                ("history", ctypes.c_int32)]


PROF_SLOTS = 8
# line path: "trsv_fwd" is the one-launch P^{-1} (ldlt_line_kernel) and "spmv_apdot" carries the
# p / x updates; the level path launches all five classes
PROF_NAMES = ("spmv_apdot", "trsv_fwd", "spmv_drift", "trsv_bwd", "pupd", "other")


class SolveReportC(ctypes.Structure):
    _fields_ = [("status", ctypes.c_void_p), ("iterations", ctypes.c_void_p),
                ("iterations_to", ctypes.c_void_p), ("seconds_to", ctypes.c_void_p),
                ("final_relative_residual", ctypes.c_void_p), ("history", ctypes.c_void_p),
                ("history_cap", ctypes.c_int64), ("breakdown_iteration", ctypes.c_void_p),
                ("kernel_ms", ctypes.c_void_p), ("kernel_launches", ctypes.c_void_p),
                ("passes", ctypes.c_int64)]


P = ctypes.c_void_p
I32 = ctypes.c_int
I64 = ctypes.c_int64

# name -> (restype, argtypes); every symbol declared in include/npcg.h
SIGNATURES = {
    "npcg_last_error": (ctypes.c_char_p, []),
    "npcg_abi_version": (I32, []),
    "npcg_device_ok": (I32, []),
    "npcg_pattern_create": (I32, [I64, P, P, I32, ctypes.POINTER(P)]),
    "npcg_pattern_destroy": (I32, [P]),
    "npcg_pattern_get_info": (I32, [P, ctypes.POINTER(PatternInfo)]),
    "npcg_pattern_device_arrays": (I32, [P, P, P, P, P, P]),
    "npcg_check_symmetric_values": (I32, [P, I32, P, I32, P, P]),
    "npcg_spmv": (I32, [P, I32, P, I32, P, P, P]),
    "npcg_factor_from_lower": (I32, [P, I32, P, I32, P, P]),
    "npcg_factor_to_lower": (I32, [P, I32, P, P, P]),
    "npcg_ldlt_apply_inverse": (I32, [P, I32, P, I32, P, I32, P, P, P]),
    "npcg_gnn_create": (I32, [ctypes.POINTER(GnnDesc), P, I64, ctypes.POINTER(P)]),
    "npcg_gnn_destroy": (I32, [P]),
    "npcg_gnn_build_factor": (I32, [P, P, I32, P, I32, P, P, P, P, P, ctypes.POINTER(I64), P]),
    "npcg_gnn_build_factor_mesh": (I32, [P, P, I32, P, I32, P, P, P, P, P, P, ctypes.POINTER(I64), P]),
    "npcg_solver_create": (I32, [P, P, I32, ctypes.POINTER(P)]),
    "npcg_solver_destroy": (I32, [P]),
    "npcg_pcg_solve": (I32, [P, P, I32, P, I32, P, I32, P, P, P, ctypes.POINTER(SolveOpts),
                             ctypes.POINTER(SolveReportC), P]),
    "npcg_solver_history": (I32, [P, P, I64, I64, P]),
    "npcg_pattern_line_info": (I32, [P, P, P, P, P, I32]),
    "npcg_launch_count": (I64, []),
    "npcg_debug_line_trace": (I32, [P, I32]),
    "npcg_fem_plan_create": (I32, [I64, I64, P, ctypes.POINTER(P)]),
    "npcg_fem_plan_create_p1": (I32, [I64, I64, I32, P, ctypes.POINTER(P)]),
    "npcg_gather_values": (I32, [I64, I32, I32, P, P, P, P]),
    "npcg_trainer_create": (I32, [P, P, I64, ctypes.POINTER(P)]),
    "npcg_trainer_destroy": (I32, [P]),
    "npcg_trainer_get_weights": (I32, [P, P]),
    "npcg_trainer_set_weights": (I32, [P, P, I32]),
    "npcg_trainer_tuple_grad": (I32, [P, P, P, P, P, P, P, ctypes.c_double, P, P, P]),
    "npcg_trainer_adam_step": (I32, [P, P, ctypes.c_double, I64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, P, P]),
    "npcg_fem_plan_destroy": (I32, [P]),
    "npcg_fem_plan_pattern": (I32, [P, ctypes.POINTER(I64), P, P]),
    "npcg_fem_assemble": (I32, [P, I32, P, I32, P, I32, I32, ctypes.c_double, P, P, P]),
}

_lib = None


def load_library(path: str = LIB_PATH):
    """Load the shared library and declare every exported symbol (no GPU needed)."""
    if not os.path.exists(path):
        raise NativeUnavailableError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a); there is no CPU fallback")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def lib():
    """The loaded library, after checking that a B200 device is usable."""
    global _lib
    if _lib is None:
        l = load_library()
        if not l.npcg_device_ok():
            raise NativeUnavailableError("no CUDA device with compute capability 10.0 (B200) is visible")
        _lib = l
    return _lib


def check(rc: int, pivot: int | None = None) -> None:
    """Map a libnpcg return code onto the pcgkit exception taxonomy."""
    if rc == OK:
        return
    msg = (_lib or load_library()).npcg_last_error().decode(errors="replace")
    if rc == ERR_DIMENSION:
        raise errors.DimensionMismatchError(msg)
    if rc == ERR_INVALID_FACTOR:
        raise errors.InvalidFactorError(msg)
    if rc == ERR_NOT_SPD:
        raise errors.NotSpdError(msg, pivot=pivot)
    if rc == ERR_BREAKDOWN:
        raise errors.BreakdownError(msg)
    if rc == ERR_DATA_FORMAT:
        raise errors.DataFormatError(msg)
    if rc == ERR_ARGUMENT:
        raise ValueError(msg)
    raise RuntimeError(f"libnpcg CUDA failure: {msg}")


def stream_handle():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> ctypes.c_void_p:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return ctypes.c_void_p(0 if t is None else t.data_ptr())
