"""Mesh and decomposition-tree views with the reference's numbering.

Mirrors the reference geometry API (`build_mesh`, `build_tree`, `Rect`,
`boundary_nodes`, `interior_nodes`, `mean_observations`) without building the
Python per-node index sets: the device plan builds its own index sets in C++
(csrc/hdd_plan.cpp).  Numbering (paths under
/root/reference/pkg/src/hddsolve/):

* node (i, j) -> j*m + i, coordinates (i h, j h)            mesh.py:90-98
* cell (i, j) -> triangles 2(iN+j) = (a,b,d), +1 = (a,d,c)  mesh.py:99-111
* alternating bisection (x cut first), post-order ids       ddtree.py:119-174
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError, GeometryError, UsageError

MAX_LEVEL = 11
MIN_LEVEL = 1


@dataclass(frozen=True)
class Rect:
    x0: float
    x1: float
    y0: float
    y1: float

    @property
    def area(self):
        return (self.x1 - self.x0) * (self.y1 - self.y0)


@dataclass(frozen=True)
class Mesh:
    """Uniform right-triangle mesh of the unit square, m = 2^L + 1 nodes per side."""

    level: int

    @property
    def m(self) -> int:
        return (1 << self.level) + 1

    @property
    def n_cells(self) -> int:
        return 1 << self.level

    @property
    def h(self) -> float:
        return 1.0 / (self.m - 1)

    @property
    def n_nodes(self) -> int:
        return self.m * self.m

    @property
    def n_triangles(self) -> int:
        return 2 * self.n_cells ** 2

    def node_index(self, i, j):
        return j * self.m + i

    @property
    def nodes(self) -> np.ndarray:
        jj, ii = np.meshgrid(np.arange(self.m), np.arange(self.m), indexing="ij")
        return np.column_stack([ii.ravel() * self.h, jj.ravel() * self.h])

    def grid_coord(self, value):
        g = value * (self.m - 1)
        gi = int(round(g))
        if abs(g - gi) > 1e-9 or not (0 <= gi <= self.m - 1):
            raise GeometryError(f"coordinate {value} is not on the level-{self.level} grid")
        return gi


def build_mesh(level: int) -> Mesh:
    if not isinstance(level, (int, np.integer)) or not (MIN_LEVEL <= level <= MAX_LEVEL):
        raise ConfigError(f"mesh level must be an integer in [{MIN_LEVEL}, {MAX_LEVEL}], got {level!r}")
    return Mesh(int(level))


def _cells(mesh: Mesh, region: Rect):
    i0, i1 = mesh.grid_coord(region.x0), mesh.grid_coord(region.x1)
    j0, j1 = mesh.grid_coord(region.y0), mesh.grid_coord(region.y1)
    if i0 >= i1 or j0 >= j1:
        raise GeometryError(f"degenerate region {region}")
    return i0, i1, j0, j1


def boundary_nodes(mesh: Mesh, region: Rect) -> np.ndarray:
    i0, i1, j0, j1 = _cells(mesh, region)
    m = mesh.m
    ii = np.arange(i0, i1 + 1)
    jj = np.arange(j0 + 1, j1)
    return np.sort(np.concatenate([j0 * m + ii, j1 * m + ii, jj * m + i0, jj * m + i1]))


def interior_nodes(mesh: Mesh, region: Rect) -> np.ndarray:
    i0, i1, j0, j1 = _cells(mesh, region)
    if i1 - i0 < 2 or j1 - j0 < 2:
        return np.empty(0, dtype=np.int64)
    ii = np.arange(i0 + 1, i1)
    jj = np.arange(j0 + 1, j1)
    return np.sort((jj[:, None] * mesh.m + ii[None, :]).ravel())


def omega_nodes(mesh: Mesh, cells) -> np.ndarray:
    """Sorted global ids of the mesh nodes of a closed cell rectangle (i0, i1, j0, j1):
    the reference DDNode.idx_omega (ddtree.py:40-57)."""
    i0, i1, j0, j1 = cells
    ii = np.arange(i0, i1 + 1)
    jj = np.arange(j0, j1 + 1)
    return (jj[:, None] * mesh.m + ii[None, :]).ravel()


def cell_centroid_tables(mesh: Mesh):
    """(cx[2N], cy[2N]): centroid coordinates of triangle type t in cell column
    i (cx[2i+t]) and cell row j (cy[2j+t]), computed as the float mean of the
    three vertex coordinates like CoefficientField.from_callable (fem.py:39-43)."""
    N, h = mesh.n_cells, mesh.h
    i = np.arange(N)
    x = lambda k: k * h  # noqa: E731  (node coordinate i*h, mesh.py:97)
    # triangle (a, b, d) x-coords: i, i+1, i+1; (a, d, c): i, i+1, i
    v0 = np.stack([np.stack([x(i), x(i + 1), x(i + 1)], 1), np.stack([x(i), x(i + 1), x(i)], 1)], 1)
    cx = v0.mean(axis=2).reshape(-1)
    # y-coords: (a, b, d): j, j, j+1; (a, d, c): j, j+1, j+1
    v1 = np.stack([np.stack([x(i), x(i), x(i + 1)], 1), np.stack([x(i), x(i + 1), x(i + 1)], 1)], 1)
    cy = v1.mean(axis=2).reshape(-1)
    return cx, cy


# -- decomposition tree -------------------------------------------------------
def _split(r, depth):
    i0, i1, j0, j1 = r
    axis = depth % 2
    if axis == 0 and i1 - i0 == 1:
        axis = 1
    elif axis == 1 and j1 - j0 == 1:
        axis = 0
    if axis == 0:
        mid = (i0 + i1) // 2
        return (i0, mid, j0, j1), (mid, i1, j0, j1)
    mid = (j0 + j1) // 2
    return (i0, i1, j0, mid), (i0, i1, mid, j1)


@dataclass(frozen=True)
class NodeRef:
    """A tree node identified like the reference DDNode: post-order id, depth
    and grid-cell bounds (ddtree.py:40-57)."""

    id: int
    depth: int
    cells: tuple
    rect: Rect

    @property
    def area(self):
        return self.rect.area


class DDTree:
    """The reference's alternating-bisection tree, addressed arithmetically."""

    def __init__(self, mesh: Mesh):
        self.mesh = mesh

    @property
    def depth(self) -> int:
        return 2 * self.mesh.level

    def _size(self, depth: int) -> int:
        return (1 << (self.depth - depth + 1)) - 1

    @property
    def n_nodes(self) -> int:
        return self._size(0)

    def _ref(self, r, depth, nid):
        h = self.mesh.h
        return NodeRef(nid, depth, r, Rect(r[0] * h, r[1] * h, r[2] * h, r[3] * h))

    @property
    def root(self) -> NodeRef:
        N = self.mesh.n_cells
        return self._ref((0, N, 0, N), 0, self.n_nodes - 1)

    @property
    def root_id(self) -> int:
        return self.n_nodes - 1

    def node(self, node_id: int) -> NodeRef:
        if not (0 <= node_id < self.n_nodes):
            raise UsageError(f"no tree node with id {node_id}")
        N = self.mesh.n_cells
        r, depth, lo = (0, N, 0, N), 0, 0
        while lo + self._size(depth) - 1 != node_id:
            s1, s2 = _split(r, depth)
            half = self._size(depth + 1)
            if node_id < lo + half:
                r = s1
            else:
                r, lo = s2, lo + half
            depth += 1
        return self._ref(r, depth, node_id)

    def nodes_at_depth(self, depth: int):
        if not (0 <= depth <= self.depth):
            raise UsageError(f"no tree nodes at depth {depth}")
        N = self.mesh.n_cells
        out = []

        def rec(r, d, lo):
            if d == depth:
                out.append(self._ref(r, d, lo + self._size(d) - 1))
                return
            s1, s2 = _split(r, d)
            rec(s1, d + 1, lo)
            rec(s2, d + 1, lo + self._size(d + 1))

        rec((0, N, 0, N), 0, 0)
        return out


def dump_tree(tree: DDTree) -> str:
    """Text lines `depth region |I(omega)| |I(boundary)| |I(gamma)|` for every node in
    post-order — the reference regression format (ddtree.py:193-202)."""
    h = tree.mesh.h
    lines = []

    def rec(r, depth):
        i0, i1, j0, j1 = r
        w, hh = i1 - i0, j1 - j0
        gamma = 0
        if w * hh > 1:
            s1, s2 = _split(r, depth)
            rec(s1, depth + 1)
            rec(s2, depth + 1)
            gamma = (hh - 1) if s1[1] != i1 else (w - 1)    # vertical cut: interior of the x line
        region = f"[{i0 * h:g},{i1 * h:g}]x[{j0 * h:g},{j1 * h:g}]"
        lines.append(f"{depth} {region} {(w + 1) * (hh + 1)} {2 * (w + hh)} {gamma}")

    N = tree.mesh.n_cells
    rec((0, N, 0, N), 0)
    return "\n".join(lines) + "\n"


def build_tree(mesh: Mesh) -> DDTree:
    return DDTree(mesh)
