"""ctypes loader for libpht.so (the C ABI of include/pht.h).  Argument marshalling only.

The library is built in-tree (paper_2111_14317_b200/lib/libpht.so, `make -C csrc`).  There is
no fallback: if it is missing, importing the package raises, so no CPU path can stand in for
the CUDA kernels.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PHT_LIB overrides the library path (kernel-variant experiments only; still the CUDA library)
LIB_PATH = os.environ.get("PHT_LIB") or os.path.join(_HERE, "lib", "libpht.so")

PHT_MAX_N = 24
PT_OK, PT_ZERO_COORD, PT_NONFINITE, PT_SINGULAR = 0, 1, 2, 4
PT_STEP_UNDERFLOW, PT_MAX_STEPS, PT_DIVERGED, PT_FLOOR = 8, 16, 32, 64
SYS_DENSE, SYS_SPECIALIZED, SYS_PROJECTIVE = 1, 2, 4
SPEC_EVAL, SPEC_STEP, SPEC_TRACK, SPEC_ALL = 1, 2, 4, 7
SOLVER_LU, SOLVER_QR = 0, 1
KERNELS = {"auto": 0, "tile": 1, "warp": 2, "dense": 3, "specialized": 4, "lane": 5}   # PHT_KERNELS_*

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64

# name -> (restype, argtypes); mirrors include/pht.h exactly
SIGNATURES = {
    "pht_system_create": (ctypes.c_int, [_i32, _i32, _vp, _vp, _vp, _vp, _i32, ctypes.POINTER(_vp)]),
    "pht_system_create_projective": (ctypes.c_int, [_i32, _i32, _vp, _vp, _vp, _vp, _i32, ctypes.POINTER(_vp)]),
    "pht_homogenize": (ctypes.c_int, [_vp, _i64, _vp, _i32, _vp, _vp]),
    "pht_system_destroy": (None, [_vp]),
    "pht_system_info": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "pht_system_flags": (ctypes.c_int, [_vp]),
    "pht_evaluate": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pht_evaluate_log": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pht_euler_newton": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pht_pc_step": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _i32, _vp, _vp, _vp]),
    "pht_pc_step_host": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _i32, _vp, _vp, _vp]),
    "pht_pc_step_host_async": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _i32, _vp, _vp, _vp]),
    "pht_host_wait": (ctypes.c_int, [_vp, _vp]),
    "pht_track_opts_default": (None, [ctypes.c_void_p]),
    "pht_track": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pht_track_cells": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp]),
    "pht_system_set_solver": (ctypes.c_int, [_vp, _i32]),
    "pht_system_set_kernels": (ctypes.c_int, [_vp, _i32]),
    "pht_system_kernels": (ctypes.c_int, [_vp]),
    "pht_system_specialize": (ctypes.c_int, [_vp, _i32]),
    "pht_specialize_compile": (ctypes.c_int, [_i32, _i32, _vp, _vp, _vp, _vp, _i32, _vp]),
    "pht_specialize_source": (_i64, [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _i64]),
    "pht_launch_count": (_i64, []),
    "pht_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "pht_last_cuda_error": (ctypes.c_char_p, []),
    "pht_version": (ctypes.c_int, []),
}


class TrackOpts(ctypes.Structure):
    """pht_track_opts (include/pht.h)."""
    _fields_ = [("dtau_init", ctypes.c_double), ("dtau_min", ctypes.c_double), ("dtau_max", ctypes.c_double),
                ("newton_tol", ctypes.c_double), ("shrink", ctypes.c_double), ("grow", ctypes.c_double),
                ("final_tol", ctypes.c_double), ("inf_norm", ctypes.c_double), ("newton_iters", ctypes.c_int32),
                ("grow_after", ctypes.c_int32), ("max_steps", ctypes.c_int32), ("final_iters", ctypes.c_int32),
                ("log_state", ctypes.c_int32), ("pred_log", ctypes.c_int32), ("pred_tol", ctypes.c_double),
                ("predictor", ctypes.c_int32), ("reuse_tangent", ctypes.c_int32)]


class PhtError(RuntimeError):
    pass


_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `make -C {os.path.join(_HERE, 'csrc')}` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int, what: str):
    if rc != 0:
        lib = load()
        msg = lib.pht_strerror(rc).decode()
        if rc in (-6, -9):
            msg += ": " + lib.pht_last_cuda_error().decode()
        raise PhtError(f"{what} failed ({rc}): {msg}")
