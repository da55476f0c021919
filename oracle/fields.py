"""Coefficient parametrizations kappa(z) on the triangles (oracle restatement).

* `IndicatorField` restates the reference `ParamField`: kappa_t =
  exp(z[region(t)]) over the tree-aligned power-of-two partition
  (/root/reference/pkg/src/hddsolve/bayes.py:29-47 aligned_partition,
  :58-71 owner assignment by centroid, first covering region wins,
  :73-77 kappa).
* `SineKLField` is the BASELINE.json field (not in the reference):
  q = 0.5 * sum_k z_k / k * sin(pi a_k x1) sin(pi b_k x2), pairs ordered by
  a+b then a, evaluated at triangle centroids computed as the float mean of
  the three vertex coordinates, exactly like
  `CoefficientField.from_callable` (fem.py:39-43); kappa = exp(q).

Both return plain float arrays of per-triangle values in reference triangle
order; wrapping them in `hddsolve.fem.CoefficientField` is the caller's job.
"""
from __future__ import annotations

import math

import numpy as np

from .geometry import Grid


def kl_pairs(n: int):
    """First n positive-integer pairs ordered by a+b, then a."""
    out = []
    s = 2
    while len(out) < n:
        for a in range(1, s):
            out.append((a, s - a))
            if len(out) == n:
                break
        s += 1
    return out


def aligned_rects(count: int):
    """Tree-aligned partition of the unit square into `count` rectangles
    (x0, x1, y0, y1), same alternating bisection as bayes.py:29-47."""
    if count < 1 or count & (count - 1):
        raise ValueError(f"partition size must be a power of two, got {count}")
    rects = [(0.0, 1.0, 0.0, 1.0)]
    depth = 0
    while len(rects) < count:
        nxt = []
        for x0, x1, y0, y1 in rects:
            if depth % 2 == 0:
                mid = 0.5 * (x0 + x1)
                nxt += [(x0, mid, y0, y1), (mid, x1, y0, y1)]
            else:
                mid = 0.5 * (y0 + y1)
                nxt += [(x0, x1, y0, mid), (x0, x1, mid, y1)]
        rects = nxt
        depth += 1
    return rects


class SineKLField:
    """kappa = exp(0.5 sum_k z_k k^-1 sin(pi a_k x1) sin(pi b_k x2))."""

    kind = "sine_kl"

    def __init__(self, grid: Grid, n_z: int):
        self.grid = grid
        self.n_z = n_z
        self.pairs = kl_pairs(n_z)
        cent = grid.centroids()
        a = np.array([p[0] for p in self.pairs], dtype=float)
        b = np.array([p[1] for p in self.pairs], dtype=float)
        k = np.arange(1, n_z + 1, dtype=float)
        # basis[k, t]; the sin arguments follow the literal formula.
        self.basis = (0.5 / k)[:, None] * np.sin(math.pi * a[:, None] * cent[None, :, 0]) \
            * np.sin(math.pi * b[:, None] * cent[None, :, 1])

    def log_kappa(self, z) -> np.ndarray:
        z = np.asarray(z, dtype=float)
        if z.shape != (self.n_z,):
            raise ValueError(f"parameter vector must have length {self.n_z}")
        return z @ self.basis

    def kappa_values(self, z) -> np.ndarray:
        return np.exp(self.log_kappa(z))

    def kappa(self, z):
        """Duck-typed `ParamField.kappa` (bayes.py:73-77) returning a reference
        `CoefficientField` when hddsolve is importable, else the raw array."""
        vals = self.kappa_values(z)
        try:
            from hddsolve.fem import CoefficientField  # only in the build container
        except ImportError:
            return vals
        return CoefficientField(vals)


class IndicatorField:
    """Reference ParamField semantics: kappa_t = exp(z[region(t)])."""

    kind = "indicator"

    def __init__(self, grid: Grid, n_z: int):
        self.grid = grid
        self.n_z = n_z
        self.rects = aligned_rects(n_z)
        cent = grid.centroids()
        owner = np.full(grid.n_triangles, -1)
        for k, (x0, x1, y0, y1) in enumerate(self.rects):
            inside = (cent[:, 0] >= x0) & (cent[:, 0] <= x1) & (cent[:, 1] >= y0) & (cent[:, 1] <= y1)
            owner[inside & (owner < 0)] = k
        if (owner < 0).any():
            raise ValueError("partition does not cover the mesh")
        self.region = owner

    def kappa_values(self, z) -> np.ndarray:
        z = np.asarray(z, dtype=float)
        if z.shape != (self.n_z,):
            raise ValueError(f"parameter vector must have length {self.n_z}")
        return np.exp(z[self.region])
