"""ctypes binding of the C ABI in include/holo_b200.h (libholo_b200.so).

The library is built in-tree by ``make`` (or ``__graft_entry__.build()``).
There is no fallback: if the library is missing or no CUDA device is usable,
every entry point raises instead of computing anything on the CPU.
"""

from __future__ import annotations

import ctypes
import os
import re
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libholo_b200.so")
# HOLO_LIB_PATH: another build of the same ABI, e.g. the bounds-checked
# libholo_b200_checked.so (make checked) for tests/test_gpu_checked.py
LIB_PATH = os.environ.get("HOLO_LIB_PATH", LIB_PATH)
CHECKED_LIB_PATH = os.path.join(_HERE, "libholo_b200_checked.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "holo_b200.h")

HOLO_OK = 0
HOLO_ERR_INVALID = 1
HOLO_ERR_UNSUPPORTED = 2
HOLO_ERR_DIVERGED = 3
HOLO_ERR_CUDA = 4
HOLO_ERR_NCCL = 5
POLICY = {"backtracking": 0, "fixed": 1}


class Geometry(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("pitch", ctypes.c_double), ("dz", ctypes.c_double), ("z0", ctypes.c_double),
                ("wavelength", ctypes.c_double)]


class SolverConfig(ctypes.Structure):
    _fields_ = [("lambda_l1", ctypes.c_double), ("lambda_tv", ctypes.c_double),
                ("max_iters", ctypes.c_int32), ("tv_inner_iters", ctypes.c_int32),
                ("step_policy", ctypes.c_int32), ("step_size", ctypes.c_double),
                ("bt_shrink", ctypes.c_double), ("stop_tol", ctypes.c_double),
                ("log_objective", ctypes.c_int32), ("real_nonnegative", ctypes.c_int32)]


class Report(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("restarts", ctypes.c_int32), ("diverged", ctypes.c_int32),
                ("guard_fixups", ctypes.c_int32), ("attempts", ctypes.c_int32),
                ("step_size", ctypes.c_double), ("final_sparsity", ctypes.c_double),
                ("wall_time", ctypes.c_double), ("f0", ctypes.c_double), ("nnz", ctypes.c_int64),
                ("skipped_planes", ctypes.c_int64)]


_P = ctypes.c_void_p
_I = ctypes.c_int32
_D = ctypes.c_double
_H = ctypes.c_void_p  # holo_handle*

# name -> (restype, argtypes); every name here is declared in include/holo_b200.h
SIGNATURES = {
    "holo_last_error": (ctypes.c_char_p, []),
    "holo_version": (ctypes.c_int, []),
    "holo_debug_checks": (ctypes.c_int, [ctypes.POINTER(ctypes.c_uint32)]),
    "holo_shape_supported": (ctypes.c_int, [_I, _I]),
    "holo_create": (ctypes.c_int, [ctypes.POINTER(Geometry), ctypes.c_int, ctypes.POINTER(_H)]),
    "holo_nccl_unique_id": (ctypes.c_int, [_P]),
    "holo_create_sharded": (ctypes.c_int, [ctypes.POINTER(Geometry), ctypes.c_int, _P, ctypes.c_int, ctypes.c_int,
                                           ctypes.POINTER(_H)]),
    "holo_create_local_group": (ctypes.c_int, [ctypes.POINTER(Geometry), ctypes.c_int, ctypes.c_int,
                                               ctypes.POINTER(_H)]),
    "holo_peer_export": (ctypes.c_int, [_H, _P, ctypes.POINTER(ctypes.c_int64)]),
    "holo_peer_import": (ctypes.c_int, [_H, _P, ctypes.c_int64]),
    "holo_peer_slice": (ctypes.c_int64, [ctypes.c_int64, ctypes.c_int32]),
    "holo_destroy": (ctypes.c_int, [_H]),
    "holo_local_planes": (ctypes.c_int, [_H, ctypes.POINTER(_I), ctypes.POINTER(_I)]),
    "holo_operator_norm": (ctypes.c_int, [_H, _I, ctypes.POINTER(_D)]),
    "holo_power_iteration": (ctypes.c_int, [_H, _P, _I, _I, ctypes.POINTER(_D), _P]),
    "holo_solve": (ctypes.c_int, [_H, _P, ctypes.POINTER(SolverConfig), ctypes.POINTER(Report)]),
    "holo_solve_device": (ctypes.c_int, [_H, _P, ctypes.POINTER(SolverConfig), ctypes.POINTER(Report), _P]),
    "holo_history": (ctypes.c_int, [_H, _P, _I, ctypes.POINTER(_I)]),
    "holo_plane_nnz": (ctypes.c_int, [_H, _P]),
    "holo_export_coo_host": (ctypes.c_int, [_H, _P, _P, _P, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]),
    "holo_export_coo_device": (ctypes.c_int, [_H, _P, _P, _P, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64), _P]),
    "holo_solution_device": (ctypes.c_int, [_H, ctypes.POINTER(_P)]),
    "holo_op_transfer": (ctypes.c_int, [_H, _I, _I, _I, _P, _P]),
    "holo_op_fft2": (ctypes.c_int, [_H, _P, _I, _I, _P]),
    "holo_op_forward": (ctypes.c_int, [_H, _P, _P, _P]),
    "holo_op_adjoint": (ctypes.c_int, [_H, _P, _P, _D, _P]),
    "holo_op_prox_fl": (ctypes.c_int, [_H, _P, _P, _I, _I, _I, _D, _D, _I, _P]),
    "holo_label_components": (ctypes.c_int, [_P, ctypes.c_int64, _I, _I, _I, _P, _P]),
    "holo_render_spectrum": (ctypes.c_int, [_P, _P, _P, _P, _I, _I, _I, _D, _D, _P, _P]),
    "holo_background": (ctypes.c_int, [_P, _I, _I, _I, _I, _P, _P]),
    "holo_profile_enable": (ctypes.c_int, [_H, _I]),
    "holo_profile_read": (ctypes.c_int, [_H, ctypes.POINTER(_I), _P, _P, _P]),
    "holo_profile_classes": (ctypes.c_int, [_H, ctypes.c_uint32]),
    "holo_launch_count": (ctypes.c_int64, []),
}

_lib = None
_lock = threading.Lock()


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def header_functions(path: str = HEADER_PATH) -> list[str]:
    """Function names declared in include/holo_b200.h."""
    text = open(path).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(holo_\w+)\s*\(", text, re.M)))


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the library (no GPU needed just to load it)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: build the sm_100a extension first (`make` or __graft_entry__.build()); "
                "there is no CPU fallback")
        lib = ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().holo_last_error()
    return msg.decode() if msg else ""


def check(code: int, what: str = ""):
    if code == HOLO_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if code in (HOLO_ERR_INVALID, HOLO_ERR_UNSUPPORTED):
        raise ValueError(msg)
    raise NativeError(code, msg)


def geometry(g) -> Geometry:
    return Geometry(int(g.nx), int(g.ny), int(g.nz), float(g.pitch), float(g.dz), float(g.z0), float(g.wavelength))
