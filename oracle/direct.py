"""Sparse direct FEM solve and exact P1 means (oracle restatement).

* `stiffness_and_load` restates `assemble_global`
  (/root/reference/pkg/src/hddsolve/fem.py:93-123): per-triangle P1 stiffness
  kappa/(2 det) G G^T scattered into a CSR matrix, lumped load area/3 per
  vertex.
* `solve` restates `oracle.direct_solve` (oracle.py:26-48): Dirichlet rows
  eliminated, interior block factored (dense below 4000 nodes, SuperLU above).
* `region_mean` restates `oracle.direct_mean` (oracle.py:74-83): sum over
  triangles inside the region of |t|/3 (u1+u2+u3), divided by the area.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .geometry import Grid

_DENSE_LIMIT = 4000


def element_stiffness(coords, kappa: float) -> np.ndarray:
    """3x3 P1 stiffness kappa/(2 det) G G^T of one triangle (fem.py:75-81)."""
    c = np.asarray(coords, dtype=float)
    x, y = c[:, 0], c[:, 1]
    det = (x[1] - x[0]) * (y[2] - y[0]) - (x[2] - x[0]) * (y[1] - y[0])
    if det <= 1e-14:
        raise ValueError("triangle is degenerate or negatively oriented")
    g = np.array([[y[(v + 1) % 3] - y[(v + 2) % 3], x[(v + 2) % 3] - x[(v + 1) % 3]] for v in range(3)])
    return (kappa / (2.0 * det)) * (g @ g.T)


def stiffness_and_load(grid: Grid, kappa: np.ndarray):
    kappa = np.asarray(kappa, dtype=float)
    if kappa.shape != (grid.n_triangles,):
        raise ValueError("coefficient field does not match the mesh")
    xy = grid.coords()
    tri = grid.triangles()
    p = xy[tri]                                   # (nt, 3, 2)
    x, y = p[:, :, 0], p[:, :, 1]
    # hat-function gradient directions (rotated opposite edges)
    g = np.empty((tri.shape[0], 3, 2))
    for v in range(3):
        a, b = (v + 1) % 3, (v + 2) % 3
        g[:, v, 0] = y[:, a] - y[:, b]
        g[:, v, 1] = x[:, b] - x[:, a]
    det = np.full(tri.shape[0], grid.h * grid.h)   # 2 * area
    loc = np.einsum("tik,tjk->tij", g, g) * (kappa / (2.0 * det))[:, None, None]
    rows = np.repeat(tri, 3, axis=1).ravel()
    cols = np.tile(tri, (1, 3)).ravel()
    A = sp.coo_matrix((loc.ravel(), (rows, cols)), shape=(grid.n_nodes, grid.n_nodes)).tocsr()
    area = 0.5 * grid.h * grid.h
    load = np.bincount(tri.ravel(), weights=np.full(tri.size, area / 3.0), minlength=grid.n_nodes)
    return A, load


def solve(grid: Grid, kappa: np.ndarray, f=None, g=None) -> np.ndarray:
    """Galerkin solution over all nodes; f nodal (default 1), g on the sorted
    global perimeter (default 0)."""
    A, load = stiffness_and_load(grid, kappa)
    full = (0, grid.N, 0, grid.N)
    bnd = grid.perimeter_ids(full)
    inner = np.sort(grid.interior_ids(full))
    f = np.ones(grid.n_nodes) if f is None else np.asarray(f, dtype=float)
    g = np.zeros(bnd.size) if g is None else np.asarray(g, dtype=float)
    rhs = (load * f)[inner] - A[inner][:, bnd] @ g
    A_ii = A[inner][:, inner]
    u = np.empty(grid.n_nodes)
    u[bnd] = g
    if grid.n_nodes <= _DENSE_LIMIT:
        u[inner] = np.linalg.solve(A_ii.toarray(), rhs)
    else:
        u[inner] = spla.splu(A_ii.tocsc()).solve(rhs)
    return u


def region_mean(grid: Grid, u: np.ndarray, rect_cells) -> float:
    """Mean of the P1 function u over a cell rectangle (i0, i1, j0, j1)."""
    i0, i1, j0, j1 = rect_cells
    ci, cj = np.meshgrid(np.arange(i0, i1), np.arange(j0, j1), indexing="ij")
    cells = (ci * grid.N + cj).ravel()
    tris = np.sort(np.concatenate([2 * cells, 2 * cells + 1]))
    tri = grid.triangles()[tris]
    area = np.full(tris.size, 0.5 * grid.h * grid.h)
    return float((area / 3.0 * u[tri].sum(axis=1)).sum() / area.sum())
