"""Bayesian likelihood API — drop-in for the reference's likelihood path.

Same names, argument meaning and error behaviour as
/root/reference/pkg/src/hddsolve/bayes.py, with the forward map running on
the B200 through libhdd_b200.so:

  reference                                   here
  ParamField.build / .kappa (bayes.py:50-77)  ParamField (indicator) / SineKLField
  Prior (bayes.py:80-120)                     Prior (same draw order)
  MeasurementModel (bayes.py:123-147)         MeasurementModel
  mean_observations (bayes.py:150-152)        mean_observations
  BayesProblem (bayes.py:155-177)             BayesProblem (+ device, max_batch)
  forward_functionals (bayes.py:180-198)      forward_functionals  (B = 1 wrapper)
  gaussian_log_likelihood (bayes.py:222-224)  gaussian_log_likelihood
  log_likelihood (bayes.py:227-231)           log_likelihood       (B = 1 wrapper)
  posterior_grid weights (bayes.py:325-330)   posterior_weights
  (per-sample Python loop)                    forward_functionals_batch /
                                              log_likelihood_batch (one C call)

Any nodal right-hand side f and any Dirichlet data g (over the boundary nodes in
increasing id order, like the reference's root.idx_boundary) are supported; both are
fixed per plan.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ConfigError, UsageError
from .geometry import DDTree, Mesh, Rect, cell_centroid_tables

__all__ = [
    "ParamField", "SineKLField", "Prior", "ToleranceSpec", "MeasurementModel", "BayesProblem", "mean_observations",
    "aligned_partition", "kl_pairs", "forward_functionals", "forward_functionals_batch", "log_likelihood",
    "log_likelihood_batch", "gaussian_log_likelihood", "posterior_weights", "synchronize", "prolong_rhs", "solve_subdomain_batch",
]


def aligned_partition(count: int):
    """Tree-aligned power-of-two partition of the unit square (bayes.py:29-47)."""
    if count < 1 or count & (count - 1):
        raise ConfigError(f"partition size must be a power of two, got {count}")
    rects = [Rect(0.0, 1.0, 0.0, 1.0)]
    depth = 0
    while len(rects) < count:
        nxt = []
        for r in rects:
            if depth % 2 == 0:
                mid = 0.5 * (r.x0 + r.x1)
                nxt += [Rect(r.x0, mid, r.y0, r.y1), Rect(mid, r.x1, r.y0, r.y1)]
            else:
                mid = 0.5 * (r.y0 + r.y1)
                nxt += [Rect(r.x0, r.x1, r.y0, mid), Rect(r.x0, r.x1, mid, r.y1)]
        rects = nxt
        depth += 1
    return rects


def kl_pairs(n: int):
    """Positive-integer pairs (a, b) ordered by a + b, then a (BASELINE.json)."""
    out, s = [], 2
    while len(out) < n:
        for a in range(1, s):
            out.append((a, s - a))
            if len(out) == n:
                break
        s += 1
    return out


class _Separable:
    """log kappa_t = sum_k coef_k z_k sx_k(cx_t) sy_k(cy_t) — the form the
    device kernel evaluates (csrc/hdd_kernels.cu, kappa_kernel)."""

    n_z: int
    sx: np.ndarray
    sy: np.ndarray
    coef: np.ndarray
    mesh: Mesh

    def kappa_values(self, z) -> np.ndarray:
        """Host evaluation (API convenience; the batched path computes kappa on the GPU)."""
        z = np.asarray(z, dtype=float)
        if z.shape != (self.n_z,):
            raise ConfigError(f"parameter vector must have length {self.n_z}")
        N = self.mesh.n_cells
        sx = self.sx.reshape(self.n_z, N, 2)
        sy = self.sy.reshape(self.n_z, N, 2)
        q = np.einsum("k,kit,kjt->ijt", self.coef * z, sx, sy)
        return np.exp(q).reshape(-1)

    def kappa(self, z):
        return self.kappa_values(z)


class SineKLField(_Separable):
    """BASELINE field kappa = exp(0.5 sum_k z_k/k sin(pi a_k x1) sin(pi b_k x2))
    at triangle centroids."""

    kind = "sine_kl"

    def __init__(self, tree_or_mesh, n_z: int):
        self.mesh = tree_or_mesh.mesh if isinstance(tree_or_mesh, DDTree) else tree_or_mesh
        if n_z < 1:
            raise ConfigError("n_z must be positive")
        self.n_z = int(n_z)
        self.pairs = kl_pairs(self.n_z)
        cx, cy = cell_centroid_tables(self.mesh)
        a = np.array([p[0] for p in self.pairs], dtype=float)
        b = np.array([p[1] for p in self.pairs], dtype=float)
        self.sx = np.ascontiguousarray(np.sin(math.pi * a[:, None] * cx[None, :]))
        self.sy = np.ascontiguousarray(np.sin(math.pi * b[:, None] * cy[None, :]))
        self.coef = 0.5 / np.arange(1, self.n_z + 1, dtype=float)


@dataclass(frozen=True)
class ParamField(_Separable):
    """Reference indicator parametrization kappa_t = exp(z[region(t)])
    over `aligned_partition(n_z)` (bayes.py:50-77)."""

    n_z: int
    regions: tuple
    mesh: Mesh
    sx: np.ndarray = field(repr=False)
    sy: np.ndarray = field(repr=False)
    coef: np.ndarray = field(repr=False)
    kind = "indicator"

    @classmethod
    def build(cls, tree: DDTree, n_z: int) -> "ParamField":
        regions = aligned_partition(n_z)
        cx, cy = cell_centroid_tables(tree.mesh)
        sx = np.stack([((cx >= r.x0) & (cx <= r.x1)).astype(float) for r in regions])
        sy = np.stack([((cy >= r.y0) & (cy <= r.y1)).astype(float) for r in regions])
        # every centroid must be covered exactly once (bayes.py:69-70)
        cover = np.einsum("kx,ky->xy", sx, sy)
        if not np.all(cover >= 1):
            raise ConfigError("partition does not cover the mesh")
        return cls(n_z, tuple(regions), tree.mesh, np.ascontiguousarray(sx), np.ascontiguousarray(sy),
                   np.ones(n_z))


@dataclass(frozen=True)
class ToleranceSpec:
    """Truncation tolerance (relative Frobenius), rank cap and dense-block size
    of the low-rank map storage (lowrank.py:20-30).  The device sketches each
    admissible block with k_max + 8 random columns (k_max <= 24: one 16/24/32-column
    pass; 25..64: blocks needing a rank above 24 are re-sketched with 72 columns);
    k_max > 64 is a ConfigError naming the device limit."""

    eps: float = 1e-6
    k_max: int = 64
    n_min: int = 32

    def __post_init__(self):
        if self.eps < 0 or self.n_min < 1 or self.k_max < 1:
            raise UsageError("invalid tolerance spec")


@dataclass(frozen=True)
class Prior:
    """Independent per-component prior, standard normal or uniform (bayes.py:80-120)."""

    components: tuple

    @classmethod
    def normal(cls, n_z):
        return cls(tuple(("normal",) for _ in range(n_z)))

    @classmethod
    def uniform(cls, n_z, a, b):
        if not a < b:
            raise ConfigError("uniform prior requires a < b")
        return cls(tuple(("uniform", float(a), float(b)) for _ in range(n_z)))

    @property
    def n_z(self):
        return len(self.components)

    def log_pdf(self, z) -> float:
        z = np.atleast_1d(np.asarray(z, dtype=float))
        total = 0.0
        for zi, comp in zip(z, self.components):
            if comp[0] == "normal":
                total += -0.5 * zi * zi - 0.5 * math.log(2.0 * math.pi)
            else:
                if zi < comp[1] or zi > comp[2]:
                    return -np.inf
                total += -math.log(comp[2] - comp[1])
        return total

    def sample(self, rng, size=None):
        cols = [rng.standard_normal(size) if c[0] == "normal" else rng.uniform(c[1], c[2], size)
                for c in self.components]
        return np.stack(cols, axis=-1)


@dataclass(frozen=True)
class MeasurementModel:
    """Observation functionals ("point", node index) / ("mean", tree node id),
    noise levels and data (bayes.py:123-147)."""

    observations: tuple
    sigma: np.ndarray
    y: np.ndarray | None = None

    def __post_init__(self):
        sigma = np.asarray(self.sigma, dtype=float)
        if sigma.shape != (len(self.observations),) or not np.all(sigma > 0):
            raise ConfigError("one positive noise level per observation required")
        object.__setattr__(self, "sigma", sigma)
        if self.y is not None:
            y = np.asarray(self.y, dtype=float)
            if y.shape != sigma.shape:
                raise ConfigError("data vector length must match the observations")
            object.__setattr__(self, "y", y)

    @property
    def n_y(self):
        return len(self.observations)

    def with_data(self, y):
        return MeasurementModel(self.observations, self.sigma, np.asarray(y, dtype=float))


def mean_observations(tree: DDTree, depth: int):
    """One mean observation per tree node at `depth`, post-order (bayes.py:150-152)."""
    return tuple(("mean", nd.id) for nd in tree.nodes_at_depth(depth))


class _Plan:
    """Owns one HddPlan* (device tables + workspace)."""

    def __init__(self, problem: "BayesProblem", device: int, max_batch: int, keep_nodes: bool = False,
                 mode: int = -1, full_solve: bool = False, solve_target: int = -1):
        L = _lib.lib()
        mesh = problem.tree.mesh
        param = problem.param
        model = problem.model
        obs = model.observations
        kinds = np.array([_lib.HDD_OBS_POINT if k == "point" else
                          (_lib.HDD_OBS_MEAN if k == "mean" else -1) for k, _ in obs], dtype=np.int32)
        if (kinds < 0).any():
            bad = [k for k, _ in obs if k not in ("point", "mean")][0]
            raise ConfigError(f"unknown observation kind {bad!r}")
        # separable fields are evaluated on the device (K1); any other duck-typed
        # param (only .kappa(z) is used, bayes.py:183) hands its fields to the plan
        self.separable = all(hasattr(param, a) for a in ("sx", "sy", "coef"))
        sep = self.separable
        self._keep = dict(
            sx=np.ascontiguousarray(param.sx, dtype=np.float64) if sep else None,
            sy=np.ascontiguousarray(param.sy, dtype=np.float64) if sep else None,
            coef=np.ascontiguousarray(param.coef, dtype=np.float64) if sep else None,
            f=None if problem._f_is_one else np.ascontiguousarray(problem.f, dtype=np.float64),
            g=np.ascontiguousarray(problem.g, dtype=np.float64) if np.any(problem.g != 0.0) else None,
            kind=kinds, ids=np.array([int(i) for _, i in obs], dtype=np.int64),
            sigma=np.ascontiguousarray(model.sigma, dtype=np.float64),
            y=None if model.y is None else np.ascontiguousarray(model.y, dtype=np.float64))
        k = self._keep
        ptr = lambda a, t: None if a is None else a.ctypes.data_as(t)  # noqa: E731
        desc = _lib.HddPlanDesc(
            level=mesh.level, n_z=int(getattr(param, "n_z", 0)),
            sx=ptr(k["sx"], _lib._f64p), sy=ptr(k["sy"], _lib._f64p), coef=ptr(k["coef"], _lib._f64p),
            f=ptr(k["f"], _lib._f64p), n_obs=len(obs), obs_kind=ptr(k["kind"], _lib._i32p),
            obs_id=ptr(k["ids"], _lib._i64p), sigma=ptr(k["sigma"], _lib._f64p), y=ptr(k["y"], _lib._f64p),
            max_batch=int(max_batch), device=int(device), keep_nodes=int(keep_nodes), mode=int(mode),
            lr_eps=float(getattr(problem.compression, "eps", 0.0) or 0.0) if problem.compression is not None else 0.0,
            lr_kmax=int(getattr(problem.compression, "k_max", 64)) if problem.compression is not None else 0,
            lr_nmin=int(getattr(problem.compression, "n_min", 32)) if problem.compression is not None else 0,
            g=ptr(k["g"], _lib._f64p), full_solve=int(full_solve), solve_target=int(solve_target))
        h = C.c_void_p()
        rc = L.hdd_plan_create(C.byref(desc), C.byref(h))
        if rc != _lib.HDD_OK:
            e = _lib.HddError()
            L.hdd_create_error(C.byref(e))
            _lib.raise_for(rc, e)
        self.handle = h
        self.lib = L
        self.n_z = int(getattr(param, "n_z", 0))
        self.n_obs = len(obs)
        self.device = device
        self.n_tri = mesh.n_triangles

    def check(self, rc):
        if rc != _lib.HDD_OK:
            e = _lib.HddError()
            self.lib.hdd_last_error(self.handle, C.byref(e))
            _lib.raise_for(rc, e)

    def info(self) -> _lib.HddPlanInfo:
        out = _lib.HddPlanInfo()
        self.check(self.lib.hdd_plan_info(self.handle, C.byref(out)))
        return out

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self.lib.hdd_plan_destroy(h)
            except Exception:
                pass
            self.handle = None


@dataclass
class BayesProblem:
    """Forward setup shared by every likelihood evaluation (bayes.py:155-177).

    `compression` (a ToleranceSpec) switches on the low-rank storage of the
    boundary maps Psi: every admissible block of every node with more than
    n_min boundary nodes is replaced by its rank-truncated form, as the
    reference does (hdd.py:280-286), by the batched randomized truncated-SVD
    kernel (csrc/hdd_kernels.cu, K5).  `device` selects the
    CUDA device; `max_batch` caps the internal sub-batch (0 = size to memory).
    """

    tree: DDTree
    param: object
    f: np.ndarray
    g: np.ndarray
    model: MeasurementModel
    compression: object = None
    threads: int = 1
    forward_calls: int = 0
    device: int = 0
    max_batch: int = 0
    mode: int = -1          # -1 auto, 0 adjoint functionals, 1 primal top-down for points
    _plan: object = field(default=None, repr=False)
    _solve_plan: object = field(default=None, repr=False)
    _sub_plans: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        mesh = self.tree.mesh
        f = np.asarray(self.f, dtype=float)
        g = np.asarray(self.g, dtype=float)
        if f.shape != (mesh.n_nodes,):
            raise UsageError("data sizes do not match the mesh")
        if g.shape != (4 * mesh.n_cells,):
            raise UsageError("data sizes do not match the mesh")
        if not np.all(np.isfinite(g)):
            raise ConfigError("Dirichlet data g is not finite")
        self.f = f
        self.g = g
        self._f_is_one = bool(np.all(f == 1.0))

    def plan(self) -> _Plan:
        if self._plan is None:
            self._plan = _Plan(self, self.device, self.max_batch, mode=self.mode)
        return self._plan

    def solve_plan(self) -> _Plan:
        """A full-solution plan (primal, every factor kept) for the full-solution
        sweep; a single-leaf or sub-leaf mesh reuses the likelihood plan."""
        info = self.plan().info()
        if info.leaf_depth == 0:
            return self.plan()
        if self._solve_plan is None:
            self._solve_plan = _Plan(self, self.device, self.max_batch, mode=1, full_solve=True)
        return self._solve_plan


def _as_batch(Z, n_z):
    try:
        import torch
    except ImportError:   # pragma: no cover
        torch = None
    if torch is not None and isinstance(Z, torch.Tensor):
        if Z.dim() == 1:
            Z = Z[None]
        if Z.dim() != 2 or Z.shape[-1] != n_z:
            raise ConfigError(f"parameter vector must have length {n_z}")
        if not Z.is_cuda:     # host tensors (pinned or not) take the host entry point
            return np.ascontiguousarray(Z.detach().to(torch.float64).numpy())
        return Z
    Z = np.asarray(Z, dtype=np.float64)
    if Z.ndim == 1:
        Z = Z[None]
    if Z.ndim != 2 or Z.shape[1] != n_z:
        raise ConfigError(f"parameter vector must have length {n_z}")
    return np.ascontiguousarray(Z)


def _kappa_rows(problem: BayesProblem, Z) -> np.ndarray:
    """Coefficient fields of a duck-typed param (only .kappa(z) is used, bayes.py:183),
    evaluated by the caller's own host code, one row per sample: [B, 2 N^2]."""
    if not isinstance(Z, np.ndarray):
        Z = Z.detach().cpu().numpy()
    n_tri = problem.tree.mesh.n_triangles
    K = np.empty((Z.shape[0], n_tri))
    for b, z in enumerate(Z):
        kap = problem.param.kappa(z)
        v = np.asarray(getattr(kap, "values", kap), dtype=np.float64).reshape(-1)
        if v.shape != (n_tri,):
            raise ConfigError(f"coefficient field must have {n_tri} triangle values, got {v.size}")
        K[b] = v
    return K


def _device_check(plan: _Plan, Zb):
    if Zb.device.index != plan.device:
        raise UsageError(f"torch inputs must live on the plan's CUDA device cuda:{plan.device}, got {Zb.device}")


class _Rows:
    """Per-call right-hand sides (f rows [n_nodes], g rows [4N]; one shared row or one
    per sample) as an HddRhs: the general Psi^f / Phi^f maps applied to new data
    (hdd.py:58-105) without rebuilding the plan."""

    def __init__(self, problem: BayesProblem, B: int, f, g, device=None):
        mesh = problem.tree.mesh
        self.keep = []
        self.rhs = _lib.HddRhs()
        for name, arr, width in (("f", f, mesh.n_nodes), ("g", g, 4 * mesh.n_cells)):
            if arr is None:
                continue
            if device is not None:
                import torch
                t = torch.as_tensor(arr, dtype=torch.float64).to(device).contiguous()
                shape, ptr = tuple(t.shape), t.data_ptr()
                self.keep.append(t)
            else:
                t = np.ascontiguousarray(np.asarray(arr, dtype=np.float64))
                shape, ptr = t.shape, t.ctypes.data
                self.keep.append(t)
            if shape == (width,):
                stride = 0
            elif shape == (B, width):
                stride = width
            else:
                raise UsageError(f"{name} must have shape ({width},) or ({B}, {width}), got {shape}")
            setattr(self.rhs, name, ptr)
            setattr(self.rhs, f"{name}_stride", stride)


def _run(problem: BayesProblem, Z, want_S: bool, want_ll: bool, sync: bool = True, f=None, g=None):
    plan = problem.plan()
    n_z = plan.n_z if plan.separable else int(getattr(problem.param, "n_z", np.asarray(Z).shape[-1]))
    Zb = _as_batch(Z, n_z)
    B = Zb.shape[0]
    f64 = _lib._f64p
    general = f is not None or g is not None
    if not plan.separable or (general and isinstance(Zb, np.ndarray)):
        # host entry point: caller-evaluated fields and/or per-call right-hand sides
        K = None if plan.separable else _kappa_rows(problem, Zb)
        Zh = None if K is not None else (Zb if isinstance(Zb, np.ndarray) else Zb.detach().cpu().numpy())
        S = np.empty((B, plan.n_obs)) if want_S else None
        ll = np.empty(B) if want_ll else None
        rows = _Rows(problem, B, f, g) if general else None
        plan.check(plan.lib.hdd_forward_batch_ex_host(
            plan.handle, None if Zh is None else Zh.ctypes.data, None if K is None else K.ctypes.data, B,
            None if rows is None else C.byref(rows.rhs),
            None if S is None else S.ctypes.data, None if ll is None else ll.ctypes.data))
        if not isinstance(Zb, np.ndarray):
            import torch
            S = None if S is None else torch.from_numpy(S).to(Zb.device)
            ll = None if ll is None else torch.from_numpy(ll).to(Zb.device)
        return S, ll
    if isinstance(Zb, np.ndarray):
        S = np.empty((B, plan.n_obs)) if want_S else None
        ll = np.empty(B) if want_ll else None
        rc = plan.lib.hdd_forward_batch_host(
            plan.handle, Zb.ctypes.data_as(f64), B,
            S.ctypes.data_as(f64) if S is not None else None,
            ll.ctypes.data_as(f64) if ll is not None else None)
        plan.check(rc)
        return S, ll
    import torch
    _device_check(plan, Zb)
    Zb = Zb.to(torch.float64).contiguous()
    S = torch.empty((B, plan.n_obs), dtype=torch.float64, device=Zb.device) if want_S else None
    ll = torch.empty(B, dtype=torch.float64, device=Zb.device) if want_ll else None
    stream = C.c_void_p(torch.cuda.current_stream(Zb.device).cuda_stream)
    if general:
        rows = _Rows(problem, B, f, g, device=Zb.device)
        rc = plan.lib.hdd_forward_batch_ex(plan.handle, C.c_void_p(Zb.data_ptr()), None, B, C.byref(rows.rhs),
                                           C.c_void_p(S.data_ptr()) if S is not None else None,
                                           C.c_void_p(ll.data_ptr()) if ll is not None else None, stream)
        plan.check(rc)
        plan.check(plan.lib.hdd_sync(plan.handle, stream))     # rows must outlive the launches
        return S, ll
    rc = plan.lib.hdd_forward_batch(plan.handle, C.c_void_p(Zb.data_ptr()), B,
                                    C.c_void_p(S.data_ptr()) if S is not None else None,
                                    C.c_void_p(ll.data_ptr()) if ll is not None else None, stream)
    plan.check(rc)
    if sync:
        plan.check(plan.lib.hdd_sync(plan.handle, stream))
    return S, ll


def forward_functionals_batch(problem: BayesProblem, Z, sync: bool = True, f=None, g=None):
    """S[B, n_y] for every row of Z (numpy / host torch -> numpy; CUDA torch tensor ->
    CUDA torch tensor).  With CUDA tensors and sync=False the call returns as soon as
    the work is queued on the current stream; failures then surface at the next call
    on the problem or at `synchronize(problem)`.

    `f` ([n_nodes] or [B, n_nodes]) and `g` ([4N] or [B, 4N], boundary nodes in
    increasing id order) replace the problem's right-hand side / Dirichlet data for
    this call only — one shared row or one row per sample (the general maps of
    hdd.py:58-105 applied to new data, "multiple right-hand sides")."""
    S, _ = _run(problem, Z, True, False, sync, f, g)
    problem.forward_calls += int(S.shape[0])
    return S


def log_likelihood_batch(problem: BayesProblem, Z, sync: bool = True, f=None, g=None):
    """ll[B] for every row of Z; raises UsageError without data (bayes.py:228-229).
    `sync`, `f`, `g` as in forward_functionals_batch."""
    if problem.model.y is None:
        raise UsageError("measurement model carries no data")
    _, ll = _run(problem, Z, False, True, sync, f, g)
    problem.forward_calls += int(ll.shape[0])
    return ll


def synchronize(problem: BayesProblem, stream=None):
    """Wait for the problem's queued device work and raise its recorded failure
    (ConfigError / NumericalError naming the lowest failing sample), if any."""
    import torch
    plan = problem.plan()
    st = stream if stream is not None else torch.cuda.current_stream(plan.device)
    plan.check(plan.lib.hdd_sync(plan.handle, C.c_void_p(st.cuda_stream)))


def forward_functionals(problem: BayesProblem, z) -> np.ndarray:
    """Observation vector S(z) (bayes.py:180-198), one sample."""
    z = np.asarray(z, dtype=float)
    n_z = getattr(problem.param, "n_z", z.shape[-1] if z.ndim else 0)
    if z.shape != (n_z,):
        raise ConfigError(f"parameter vector must have length {n_z}")
    return forward_functionals_batch(problem, z[None])[0]


def solve_batch(problem: BayesProblem, Z, f=None, g=None):
    """u at every mesh node for every row of Z: U[B, n_nodes] (node id j * m + i).

    Bottom-up sweep, primal top-down sweep over the interfaces and the in-leaf
    interior solves on the device — leaves_to_root(keep_all) + root_to_leaves
    (hdd.py:289-432) for a batch.  numpy in -> numpy out; a CUDA torch tensor in ->
    CUDA torch tensor out.  `f` / `g`: per-call right-hand sides as in
    forward_functionals_batch (root_to_leaves(store, f, g) for new data)."""
    plan = problem.solve_plan()
    n_z = plan.n_z if plan.separable else int(getattr(problem.param, "n_z", np.asarray(Z).shape[-1]))
    Zb = _as_batch(Z, n_z)
    B = Zb.shape[0]
    n = problem.tree.mesh.n_nodes
    general = f is not None or g is not None
    if not plan.separable or isinstance(Zb, np.ndarray):
        K = None if plan.separable else _kappa_rows(problem, Zb)
        Zh = None if K is not None else (Zb if isinstance(Zb, np.ndarray) else Zb.detach().cpu().numpy())
        rows = _Rows(problem, B, f, g) if general else None
        U = np.empty((B, n))
        plan.check(plan.lib.hdd_solve_batch_ex_host(
            plan.handle, None if Zh is None else Zh.ctypes.data, None if K is None else K.ctypes.data, B,
            None if rows is None else C.byref(rows.rhs), U.ctypes.data))
        if not isinstance(Zb, np.ndarray):
            import torch
            return torch.from_numpy(U).to(Zb.device)
        return U
    import torch
    _device_check(plan, Zb)
    Zb = Zb.to(torch.float64).contiguous()
    U = torch.empty((B, n), dtype=torch.float64, device=Zb.device)
    stream = C.c_void_p(torch.cuda.current_stream(Zb.device).cuda_stream)
    rows = _Rows(problem, B, f, g, device=Zb.device) if general else None
    plan.check(plan.lib.hdd_solve_batch_ex(plan.handle, C.c_void_p(Zb.data_ptr()), None, B,
                                           None if rows is None else C.byref(rows.rhs), C.c_void_p(U.data_ptr()),
                                           stream))
    plan.check(plan.lib.hdd_sync(plan.handle, stream))
    return U


def prolong_rhs(f_coarse, level_coarse: int, level_fine: int) -> np.ndarray:
    """Two-grid right-hand side: nodal values on the level_coarse grid prolonged to the
    level_fine grid by bilinear interpolation (the reference SPEC's "coarse RHS given
    on a coarser grid injected to fine nodes", PAPER.md:286 / :319 property 1, f_h in
    V_H subset V_h).  Node ids j * m + i on both grids."""
    if not (1 <= level_coarse <= level_fine):
        raise ConfigError("two-grid right-hand side needs 1 <= level_coarse <= level_fine")
    mc = (1 << level_coarse) + 1
    fc = np.asarray(f_coarse, dtype=float)
    if fc.shape != (mc * mc,):
        raise ConfigError(f"coarse right-hand side must have {mc * mc} nodal values")
    fc = fc.reshape(mc, mc)                         # [j][i]
    r = 1 << (level_fine - level_coarse)
    mf = (1 << level_fine) + 1
    x = np.arange(mf) / r
    i0 = np.minimum(np.floor(x).astype(int), mc - 2) if mc > 1 else np.zeros(mf, dtype=int)
    t = x - i0
    rows = fc[i0] * (1 - t)[:, None] + fc[i0 + 1] * t[:, None]          # interpolate in j
    return (rows[:, i0] * (1 - t)[None, :] + rows[:, i0 + 1] * t[None, :]).reshape(-1)


def mean_over_cells(mesh, u, cells) -> float:
    """Mean of the P1 function u over a grid-aligned cell rectangle by the exact
    per-triangle rule sum |t|/3 (u1+u2+u3) / |region| (oracle.py:74-83): per cell
    (2 u_a + u_b + u_c + 2 u_d) / 6 for its triangles (a,b,d), (a,d,c)."""
    i0, i1, j0, j1 = cells
    if i1 <= i0 or j1 <= j0:
        raise ConfigError("region contains no triangles")
    m = mesh.m
    u = np.asarray(u, dtype=float).reshape(m, m)     # [j][i]
    a = u[j0:j1, i0:i1]
    b = u[j0:j1, i0 + 1:i1 + 1]
    c = u[j0 + 1:j1 + 1, i0:i1]
    d = u[j0 + 1:j1 + 1, i0 + 1:i1 + 1]
    return float((2.0 * a + b + c + 2.0 * d).sum() / (6.0 * a.size))


def observe_solution(tree: DDTree, u, model: MeasurementModel) -> np.ndarray:
    """Observation operators applied to an assembled solution (bayes.py:211-219)."""
    out = np.empty(model.n_y)
    u = np.asarray(u, dtype=float)
    for k, (kind, ident) in enumerate(model.observations):
        if kind == "mean":
            out[k] = mean_over_cells(tree.mesh, u, tree.node(int(ident)).cells)
        else:
            out[k] = u[int(ident)]
    return out


def forward_full_solve(problem: BayesProblem, z) -> np.ndarray:
    """Observation vector via the full solve plus the per-triangle mean rule — the
    comparison route of the likelihood-equivalence checks (bayes.py:201-208)."""
    z = np.asarray(z, dtype=float)
    if z.ndim != 1:
        raise ConfigError("parameter vector must be one-dimensional")
    u = solve_batch(problem, z[None])[0]
    return observe_solution(problem.tree, u, problem.model)


def solve_subdomain_batch(problem: BayesProblem, Z, target_id: int, f=None, g=None) -> np.ndarray:
    """Solution restricted to one tree node for every row of Z: [B, |idx_omega|], aligned
    with the node's idx_omega (sorted global ids of the closed subdomain).  A partial
    inverse like the reference's solve_subdomain with SolveMode.keep_path(target)
    (hdd.py:435-490, :186-203): the device plan factors, sweeps top-down and solves
    in-leaf only on the root-to-target path and the target's subtree
    (hdd_solve_subdomain_batch).  `f` / `g` as in forward_functionals_batch."""
    tid = int(target_id)
    problem.tree.node(tid)                                   # UsageError for an unknown id
    plan = problem._sub_plans.get(tid)
    if plan is None:
        plan = _Plan(problem, problem.device, problem.max_batch, mode=1, solve_target=tid)
        problem._sub_plans[tid] = plan
    n_z = plan.n_z if plan.separable else int(getattr(problem.param, "n_z", np.asarray(Z).shape[-1]))
    Zb = _as_batch(Z, n_z)
    if not isinstance(Zb, np.ndarray):
        Zb = Zb.detach().cpu().numpy()
    B = Zb.shape[0]
    K = None if plan.separable else _kappa_rows(problem, Zb)
    rows = _Rows(problem, B, f, g) if (f is not None or g is not None) else None
    Us = np.empty((B, plan.info().n_omega))
    plan.check(plan.lib.hdd_solve_subdomain_batch_host(
        plan.handle, None if K is not None else Zb.ctypes.data, None if K is None else K.ctypes.data, B,
        None if rows is None else C.byref(rows.rhs), Us.ctypes.data))
    return Us


def solve_subdomain(problem: BayesProblem, z, target_id: int) -> np.ndarray:
    """Solution restricted to one tree node, aligned with its idx_omega (sorted
    global node ids of the closed subdomain) — solve_subdomain, hdd.py:435-490, as a
    partial inverse (solve_subdomain_batch)."""
    z = np.asarray(z, dtype=float)
    if z.ndim != 1:
        raise ConfigError("parameter vector must be one-dimensional")
    return solve_subdomain_batch(problem, z[None], target_id)[0]


def gaussian_log_likelihood(y, s, sigma) -> float:
    resid = (np.asarray(y) - np.asarray(s)) / sigma
    return float(-0.5 * np.sum(resid ** 2) - np.sum(np.log(sigma * math.sqrt(2.0 * math.pi))))


def log_likelihood(problem: BayesProblem, z, forward=None) -> float:
    """bayes.py:227-231; `forward` keeps the reference's plug-in point."""
    if problem.model.y is None:
        raise UsageError("measurement model carries no data")
    if forward is None:
        z = np.asarray(z, dtype=float)
        n_z = getattr(problem.param, "n_z", z.shape[-1] if z.ndim else 0)
        if z.shape != (n_z,):
            raise ConfigError(f"parameter vector must have length {n_z}")
        return float(log_likelihood_batch(problem, z[None])[0])
    s = forward(problem, z)
    return gaussian_log_likelihood(problem.model.y, s, problem.model.sigma)


def posterior_weights(log_like, log_prior=None):
    """Self-normalised posterior weights and the mode index.

    joint = log_prior + log_like (prior omitted for prior draws), weights =
    exp(joint - logsumexp(joint)), index = argmax(joint) with numpy's
    first-occurrence tie rule — the pieces of posterior_grid reused for
    batches (bayes.py:325-330)."""
    ll = np.asarray(log_like, dtype=float)
    joint = ll if log_prior is None else ll + np.asarray(log_prior, dtype=float)
    mx = np.max(joint)
    lse = mx + math.log(np.sum(np.exp(joint - mx)))
    return np.exp(joint - lse), int(np.argmax(joint)), float(lse)
