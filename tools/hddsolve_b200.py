"""hddsolve/b200.py — the binding a reference maintainer would add.

Plugs libhdd_b200.so into the UNMODIFIED reference through its own plug-in points:
`log_likelihood(problem, z, forward=...)` (bayes.py:227-231) and the duck-typed
`problem.param.kappa(z)` (bayes.py:183).  Any reference `param` works — the coefficient
field is evaluated by the reference's own code and handed to the device through
`hdd_forward_batch_kappa_host` — so no separable tables are needed.

    from hddsolve import bayes
    from hddsolve_b200 import device_forward_factory
    fwd = device_forward_factory(problem)
    ll = bayes.log_likelihood(problem, z, forward=fwd)       # reference call site, device forward
    S = fwd.batch(problem, Z)                                 # [B, n_y] in one C call
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

try:   # inside the reference package (hddsolve/b200.py)
    from .errors import ConfigError, NumericalError, UsageError  # type: ignore
except ImportError:   # standalone (tests): the reference's exceptions from the installed package
    from hddsolve.errors import ConfigError, NumericalError, UsageError

_f64 = C.POINTER(C.c_double)
_i32 = C.POINTER(C.c_int32)
_i64 = C.POINTER(C.c_int64)


class _Desc(C.Structure):            # HddPlanDesc, include/hdd.h (field order matters)
    _fields_ = [("level", C.c_int32), ("n_z", C.c_int32), ("sx", _f64), ("sy", _f64),
                ("coef", _f64), ("f", _f64), ("n_obs", C.c_int32),
                ("obs_kind", _i32), ("obs_id", _i64),
                ("sigma", _f64), ("y", _f64), ("max_batch", C.c_int32),
                ("device", C.c_int32), ("keep_nodes", C.c_int32), ("mode", C.c_int32),
                ("lr_eps", C.c_double), ("lr_kmax", C.c_int32), ("lr_nmin", C.c_int32),
                ("g", _f64), ("full_solve", C.c_int32), ("solve_target", C.c_int64)]


class _Err(C.Structure):             # HddError
    _fields_ = [("code", C.c_int32), ("sample", C.c_int32), ("node_id", C.c_int64),
                ("message", C.c_char * 256)]


def _load(path=None):
    L = C.CDLL(path or os.environ.get("HDD_B200_LIB", "libhdd_b200.so"))
    L.hdd_plan_create.argtypes = [C.POINTER(_Desc), C.POINTER(C.c_void_p)]
    L.hdd_plan_destroy.argtypes = [C.c_void_p]
    L.hdd_forward_batch_kappa_host.argtypes = [C.c_void_p, _f64, C.c_int64, _f64, _f64]
    L.hdd_last_error.argtypes = [C.c_void_p, C.POINTER(_Err)]
    L.hdd_create_error.argtypes = [C.POINTER(_Err)]
    return L


_EXC = {-1: ConfigError, -2: UsageError, -3: NumericalError}


def _raise(L, rc, h=None):
    e = _Err()
    (L.hdd_last_error(h, C.byref(e)) if h is not None else L.hdd_create_error(C.byref(e)))
    exc = _EXC.get(rc, RuntimeError)
    raise exc(e.message.decode()) if exc is not NumericalError else exc(e.message.decode(),
                                                                        e.node_id if e.node_id >= 0 else None)


class DeviceForward:
    """forward(problem, z) -> S for the reference's log_likelihood(..., forward=);
    .batch(problem, Z) -> S[B, n_y]."""

    def __init__(self, problem, device=0, lib=None, compression=None):
        L = _load(lib)
        obs = problem.model.observations
        kind = np.array([0 if k == "point" else (1 if k == "mean" else -1) for k, _ in obs], np.int32)
        if (kind < 0).any():
            raise ConfigError("unknown observation kind")
        ids = np.array([int(i) for _, i in obs], np.int64)
        sig = np.ascontiguousarray(problem.model.sigma, dtype=float)
        y = None if problem.model.y is None else np.ascontiguousarray(problem.model.y, dtype=float)
        f = np.ascontiguousarray(problem.f, dtype=float)     # nodal right-hand side
        g = np.ascontiguousarray(problem.g, dtype=float)     # Dirichlet data, root.idx_boundary order
        tol = compression if compression is not None else problem.compression
        d = _Desc(level=problem.tree.mesh.level, n_z=0, sx=None, sy=None, coef=None, f=f.ctypes.data_as(_f64),
                  n_obs=len(obs), obs_kind=kind.ctypes.data_as(_i32), obs_id=ids.ctypes.data_as(_i64),
                  sigma=sig.ctypes.data_as(_f64), y=None if y is None else y.ctypes.data_as(_f64),
                  max_batch=0, device=device, keep_nodes=0, mode=-1,
                  lr_eps=float(tol.eps) if tol else 0.0, lr_kmax=int(tol.k_max) if tol else 0,
                  lr_nmin=int(tol.n_min) if tol else 0, g=g.ctypes.data_as(_f64), full_solve=0,
                  solve_target=-1)
        h = C.c_void_p()
        rc = L.hdd_plan_create(C.byref(d), C.byref(h))
        if rc != 0:
            _raise(L, rc)
        self.L, self.h, self.n_y = L, h, len(obs)
        self.n_tri = problem.tree.mesh.n_triangles

    def batch(self, problem, Z):
        Z = np.atleast_2d(np.asarray(Z, dtype=float))
        K = np.empty((Z.shape[0], self.n_tri))
        for b, z in enumerate(Z):                     # the reference's own coefficient code
            K[b] = np.asarray(problem.param.kappa(z).values, dtype=float)
        S = np.empty((Z.shape[0], self.n_y))
        rc = self.L.hdd_forward_batch_kappa_host(self.h, K.ctypes.data_as(_f64), K.shape[0],
                                                 S.ctypes.data_as(_f64), None)
        if rc != 0:
            _raise(self.L, rc, self.h)
        problem.forward_calls += Z.shape[0]
        return S

    def __call__(self, problem, z):                  # forward_functionals(problem, z) signature
        return self.batch(problem, np.asarray(z, dtype=float)[None])[0]

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            self.L.hdd_plan_destroy(h)
            self.h = None


def device_forward_factory(problem, device=0, lib=None):
    return DeviceForward(problem, device=device, lib=lib)
