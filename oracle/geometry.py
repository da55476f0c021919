"""Structured mesh and alternating-bisection tree (oracle restatement).

Restates the reference geometry so the oracle can run without
`/root/reference` on the GPU box:

* node (i, j) -> global id j*m + i, coordinates (i*h, j*h)
  (/root/reference/pkg/src/hddsolve/mesh.py:90-98);
* cell (i, j) -> triangles 2*(i*N + j) = (a, b, d) and 2*(i*N + j) + 1 =
  (a, d, c) with a=(i,j), b=(i+1,j), c=(i,j+1), d=(i+1,j+1)
  (mesh.py:99-111);
* perimeter / interior / region id sets sorted ascending (mesh.py:114-146);
* tree: cut axis alternates with depth, vertical (x) cut first, switched when
  the node is one cell wide along that axis; sons are the lower / left half
  first; ids are post-order (sons precede father); interface = son-1
  perimeter minus father perimeter (ddtree.py:119-174).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Grid:
    level: int

    @property
    def N(self) -> int:          # cells per side
        return 1 << self.level

    @property
    def m(self) -> int:          # nodes per side
        return self.N + 1

    @property
    def h(self) -> float:
        return 1.0 / self.N

    @property
    def n_nodes(self) -> int:
        return self.m * self.m

    @property
    def n_triangles(self) -> int:
        return 2 * self.N * self.N

    def coords(self) -> np.ndarray:
        """(n, 2) node coordinates, row j-major like mesh.py:96-97."""
        jj, ii = np.meshgrid(np.arange(self.m), np.arange(self.m), indexing="ij")
        return np.column_stack([ii.ravel() * self.h, jj.ravel() * self.h])

    def triangles(self) -> np.ndarray:
        """(2N^2, 3) vertex ids, CCW, numbered like mesh.py:101-109."""
        N, m = self.N, self.m
        ci, cj = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
        ci, cj = ci.ravel(), cj.ravel()
        a = cj * m + ci
        tri = np.empty((2 * a.size, 3), dtype=np.int64)
        tri[0::2] = np.column_stack([a, a + 1, a + m + 1])
        tri[1::2] = np.column_stack([a, a + m + 1, a + m])
        return tri

    def centroids(self) -> np.ndarray:
        """Triangle centroids as the float mean of the vertex coordinates
        (the reference evaluates callables there, fem.py:39-43)."""
        return self.coords()[self.triangles()].mean(axis=1)

    # -- index sets over a cell rectangle (i0, i1, j0, j1) -----------------
    def region_ids(self, r) -> np.ndarray:
        i0, i1, j0, j1 = r
        ii = np.arange(i0, i1 + 1)
        jj = np.arange(j0, j1 + 1)
        return (jj[:, None] * self.m + ii[None, :]).ravel()

    def perimeter_ids(self, r) -> np.ndarray:
        i0, i1, j0, j1 = r
        m = self.m
        ii = np.arange(i0, i1 + 1)
        jj = np.arange(j0 + 1, j1)
        ids = np.concatenate([j0 * m + ii, j1 * m + ii, jj * m + i0, jj * m + i1])
        return np.sort(ids)

    def interior_ids(self, r) -> np.ndarray:
        i0, i1, j0, j1 = r
        if i1 - i0 < 2 or j1 - j0 < 2:
            return np.empty(0, dtype=np.int64)
        ii = np.arange(i0 + 1, i1)
        jj = np.arange(j0 + 1, j1)
        return (jj[:, None] * self.m + ii[None, :]).ravel()

    def on_domain_boundary(self, ids) -> np.ndarray:
        ids = np.asarray(ids)
        i, j = ids % self.m, ids // self.m
        return (i == 0) | (j == 0) | (i == self.N) | (j == self.N)


def split_rect(r, depth):
    """Sons of a cell rectangle under the alternating rule (ddtree.py:139-149)."""
    i0, i1, j0, j1 = r
    nx, ny = i1 - i0, j1 - j0
    axis = depth % 2
    if axis == 0 and nx == 1:
        axis = 1
    elif axis == 1 and ny == 1:
        axis = 0
    if axis == 0:
        mid = (i0 + i1) // 2
        return (i0, mid, j0, j1), (mid, i1, j0, j1)
    mid = (j0 + j1) // 2
    return (i0, i1, j0, mid), (i0, i1, mid, j1)


def subtree_size(level: int, depth: int) -> int:
    """Nodes in a subtree rooted at `depth` of the complete tree of height 2L."""
    return (1 << (2 * level - depth + 1)) - 1


def rect_of_node_id(level: int, node_id: int):
    """(rect, depth) of the reference post-order node id, computed arithmetically."""
    N = 1 << level
    r, depth = (0, N, 0, N), 0
    lo = 0
    total = subtree_size(level, 0)
    if not (0 <= node_id < total):
        raise ValueError(f"node id {node_id} out of range")
    while True:
        own = lo + subtree_size(level, depth) - 1
        if node_id == own:
            return r, depth
        s1, s2 = split_rect(r, depth)
        half = subtree_size(level, depth + 1)
        if node_id < lo + half:
            r = s1
        else:
            r, lo = s2, lo + half
        depth += 1


def node_id_of_path(level: int, path) -> int:
    """Post-order id of the node reached by son choices (0/1) from the root."""
    nid = 0
    for d, b in enumerate(path, start=1):
        if b:
            nid += subtree_size(level, d)
    return nid + subtree_size(level, len(path)) - 1


def nodes_at_depth(level: int, depth: int):
    """[(node_id, rect)] of all nodes at `depth`, in post-order id order."""
    N = 1 << level
    out = []

    def rec(r, d, path):
        if d == depth:
            out.append((node_id_of_path(level, path), r))
            return
        s1, s2 = split_rect(r, d)
        rec(s1, d + 1, path + [0])
        rec(s2, d + 1, path + [1])

    rec((0, N, 0, N), 0, [])
    return out


@dataclass
class TreeNode:
    id: int
    depth: int
    rect: tuple
    sons: tuple | None = None
    parent: int | None = None
    omega: np.ndarray = field(default=None, repr=False)
    bnd: np.ndarray = field(default=None, repr=False)
    gamma: np.ndarray = field(default=None, repr=False)
    # merge plan: son boundary -> positions in [bnd | gamma], son omega -> omega
    kpos: tuple = field(default=None, repr=False)
    wpos: tuple = field(default=None, repr=False)

    @property
    def is_leaf(self):
        return self.sons is None


def full_tree(grid: Grid):
    """Every node of the complete tree (down to single cells), post-order.

    Only used at the small levels the CPU port runs (L <= 8)."""
    nodes: list[TreeNode] = []

    def build(r, depth):
        i0, i1, j0, j1 = r
        omega = grid.region_ids(r)
        omega.sort()
        bnd = grid.perimeter_ids(r)
        if i1 - i0 == 1 and j1 - j0 == 1:
            nd = TreeNode(len(nodes), depth, r, omega=omega, bnd=bnd,
                          gamma=np.empty(0, dtype=np.int64))
            nodes.append(nd)
            return nd
        a, b = split_rect(r, depth)
        s1, s2 = build(a, depth + 1), build(b, depth + 1)
        gamma = np.setdiff1d(s1.bnd, bnd, assume_unique=True)
        nd = TreeNode(len(nodes), depth, r, sons=(s1.id, s2.id), omega=omega, bnd=bnd, gamma=gamma)
        K = np.concatenate([bnd, gamma])
        order = np.argsort(K, kind="stable")
        kp, wp = [], []
        for s in (s1, s2):
            kp.append(order[np.searchsorted(K[order], s.bnd)])
            wp.append(np.searchsorted(omega, s.omega))
            s.parent = nd.id
        nd.kpos, nd.wpos = tuple(kp), tuple(wp)
        nodes.append(nd)
        return nd

    N = grid.N
    build((0, N, 0, N), 0)
    return nodes
