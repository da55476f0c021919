"""ctypes binding of libhdd_b200.so (the C ABI declared in include/hdd.h).

The library is built in-tree by `paper_1708_02207_b200.build`; there is no
fallback implementation: if the shared library is missing or fails to load,
`lib()` raises and every forward call fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import ConfigError, NumericalError, UsageError

# HDD_LIB_PATH: developer hook for A/B builds of the same sources (tools/ab_build.py)
LIB_PATH = Path(os.environ.get("HDD_LIB_PATH") or Path(__file__).resolve().parent / "libhdd_b200.so")

HDD_OK = 0
HDD_ERR_CONFIG = -1
HDD_ERR_USAGE = -2
HDD_ERR_NUMERICAL = -3
HDD_ERR_CUDA = -4
HDD_ERR_NOMEM = -5
HDD_OBS_POINT = 0
HDD_OBS_MEAN = 1

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)


class HddPlanDesc(C.Structure):
    _fields_ = [
        ("level", C.c_int32), ("n_z", C.c_int32),
        ("sx", _f64p), ("sy", _f64p), ("coef", _f64p), ("f", _f64p),
        ("n_obs", C.c_int32), ("obs_kind", _i32p), ("obs_id", _i64p),
        ("sigma", _f64p), ("y", _f64p),
        ("max_batch", C.c_int32), ("device", C.c_int32), ("keep_nodes", C.c_int32),
        ("mode", C.c_int32), ("lr_eps", C.c_double), ("lr_kmax", C.c_int32), ("lr_nmin", C.c_int32),
        ("g", _f64p), ("full_solve", C.c_int32), ("solve_target", C.c_int64),
    ]


class HddRhs(C.Structure):
    _fields_ = [("f", C.c_void_p), ("f_stride", C.c_int64), ("g", C.c_void_p), ("g_stride", C.c_int64)]


class HddError(C.Structure):
    _fields_ = [("code", C.c_int32), ("sample", C.c_int32), ("node_id", C.c_int64),
                ("message", C.c_char * 256)]


class HddPlanInfo(C.Structure):
    _fields_ = [("level", C.c_int32), ("n_cells", C.c_int32), ("leaf_cells", C.c_int32),
                ("leaf_depth", C.c_int32), ("n_upper", C.c_int32), ("n_leaves", C.c_int32),
                ("n_obs", C.c_int32), ("leaf_cols", C.c_int32), ("max_batch", C.c_int32),
                ("n_kernels_per_batch", C.c_int32), ("workspace_bytes", C.c_int64), ("mode", C.c_int32),
                ("n_topdown", C.c_int32), ("tiny", C.c_int32), ("separable", C.c_int32), ("full_solve", C.c_int32),
                ("n_omega", C.c_int32), ("factor_doubles", C.c_int64)]


class HddNodeInfo(C.Structure):
    _fields_ = [("ref_id", C.c_int64), ("depth", C.c_int32), ("i0", C.c_int32), ("i1", C.c_int32),
                ("j0", C.c_int32), ("j1", C.c_int32), ("son", C.c_int32 * 2),
                ("k", C.c_int32), ("ng", C.c_int32), ("nc", C.c_int32),
                ("bnd", _i64p), ("gamma", _i64p), ("gmap", _i32p), ("csrc", _i32p),
                ("ccoef", _f64p), ("cbirth", _i32p)]


class HddLeafInfo(C.Structure):
    _fields_ = [("ref_id", C.c_int64), ("i0", C.c_int32), ("j0", C.c_int32),
                ("ncols", C.c_int32), ("has_mean", C.c_int32), ("birth", _i32p), ("ccode", _i32p),
                ("gperim", _f64p)]


class HddObsInfo(C.Structure):
    _fields_ = [("kind", C.c_int32), ("col", C.c_int32), ("value", C.c_double), ("node", C.c_int32),
                ("slot", C.c_int32)]


EXPORTS = {
    "hdd_plan_create": (C.c_int, [C.POINTER(HddPlanDesc), C.POINTER(C.c_void_p)]),
    "hdd_plan_destroy": (C.c_int, [C.c_void_p]),
    "hdd_forward_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "hdd_forward_batch_timed": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                          _f64p, C.c_int32]),
    "hdd_forward_batch_host": (C.c_int, [C.c_void_p, _f64p, C.c_int64, _f64p, _f64p]),
    "hdd_sync": (C.c_int, [C.c_void_p, C.c_void_p]),
    "hdd_forward_batch_kappa": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "hdd_forward_batch_kappa_host": (C.c_int, [C.c_void_p, _f64p, C.c_int64, _f64p, _f64p]),
    "hdd_solve_batch_kappa": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "hdd_forward_batch_ex": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(HddRhs), C.c_void_p,
                                       C.c_void_p, C.c_void_p]),
    "hdd_forward_batch_ex_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(HddRhs),
                                            C.c_void_p, C.c_void_p]),
    "hdd_solve_batch_ex": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(HddRhs), C.c_void_p,
                                     C.c_void_p]),
    "hdd_solve_batch_ex_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(HddRhs),
                                          C.c_void_p]),
    "hdd_solve_batch_kappa_host": (C.c_int, [C.c_void_p, _f64p, C.c_int64, _f64p]),
    "hdd_solve_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "hdd_solve_batch_host": (C.c_int, [C.c_void_p, _f64p, C.c_int64, _f64p]),
    "hdd_kappa_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "hdd_posterior_weights": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p]),
    "hdd_last_error": (C.c_int, [C.c_void_p, C.POINTER(HddError)]),
    "hdd_create_error": (C.c_int, [C.POINTER(HddError)]),
    "hdd_plan_info": (C.c_int, [C.c_void_p, C.POINTER(HddPlanInfo)]),
    "hdd_plan_node_info": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(HddNodeInfo)]),
    "hdd_plan_leaf_info": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(HddLeafInfo)]),
    "hdd_plan_obs_info": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(HddObsInfo)]),
    "hdd_leaf_template": (C.c_int, [C.c_int32, _i32p, _i32p, _i32p, C.POINTER(_i32p), C.POINTER(_i32p)]),
    "hdd_debug_node_output": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, _f64p, _f64p, _f64p]),
    "hdd_debug_leaf_clocks": (C.c_int, [C.POINTER(C.c_longlong)]),
    "hdd_debug_merge_clocks": (C.c_int, [C.POINTER(C.c_longlong)]),
    "hdd_debug_lowrank_wide": (C.c_int, [C.c_void_p, _i64p]),
    "hdd_solve_subdomain_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(HddRhs),
                                            C.c_void_p, C.c_void_p]),
    "hdd_solve_subdomain_batch_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(HddRhs),
                                                 C.c_void_p]),
    "hdd_plan_stage_kernel": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_char_p, C.c_int32]),
    "hdd_version": (C.c_char_p, []),
}

_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """Load libhdd_b200.so (raises if it is missing — no fallback path)."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_1708_02207_b200.build` "
                    "(there is no CPU fallback for the HDD likelihood)")
            L = C.CDLL(str(LIB_PATH))
            for name, (res, args) in EXPORTS.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
        return _lib


def raise_for(code: int, err: HddError | None = None):
    """Map a C status to the reference exception types (errors.py:4-21)."""
    if code == HDD_OK:
        return
    msg = err.message.decode(errors="replace") if err is not None else f"status {code}"
    node = int(err.node_id) if err is not None and err.node_id >= 0 else None
    if code == HDD_ERR_CONFIG:
        raise ConfigError(msg)
    if code == HDD_ERR_USAGE:
        raise UsageError(msg)
    if code == HDD_ERR_NUMERICAL:
        raise NumericalError(msg, node)
    raise RuntimeError(f"libhdd_b200: {msg}")
