"""Restatement of the reference HDD functional path on the CPU ("port").

Follows the reference algorithm step for step, with dense maps and no
condensation, so it is both the parity checker at small sizes and the
`cpu_baseline` (kind "port") that `bench.py` times:

* cell init: psi_g = kappa_t1 P1 + kappa_t2 P2, psi_f = diag(h^2/6 [2,1,1,2])
  (/root/reference/pkg/src/hddsolve/hdd.py:310-316, fem.py:126-145);
* merge: scatter-add the sons' (psi_g, psi_f) over [boundary | interface]
  (hdd.py:216-238), Cholesky of the interface block, X = A22^-1 [A21 | B2],
  psi_g = A11 - A12 Xa (symmetrised), psi_f = B1 - A12 Xb, phi_g = -Xa,
  phi_f = Xb (hdd.py:241-277);
* depth-synchronous bottom-up order, sons dropped after their father
  (hdd.py:343-384);
* functional tracker: every node's mean (c_i = area ratio), points born as
  phi^T e at the interface owner, tracked functionals lifted with (1,0)/(0,1),
  perimeter points as indicator vectors (functionals.py:47-114, :146-224);
* forward = <l_f, f> + <l_g, g> per observation, Gaussian log-likelihood
  (bayes.py:180-198, :222-231).

Observations are ("point", node_index) or ("mean", node_id) exactly like
`MeasurementModel.observations` (bayes.py:127).
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg

from .geometry import Grid, full_tree


def cell_stencils(h: float):
    """Unit-kappa 4x4 stiffness of the two cell triangles and the load diagonal,
    cell nodes ordered (i,j), (i+1,j), (i,j+1), (i+1,j+1) (fem.py:126-145)."""
    P1 = np.zeros((4, 4))
    P2 = np.zeros((4, 4))
    # triangle (a, b, d): right angle at b -> legs a-b, b-d carry -1/2
    P1[np.ix_([0, 1, 3], [0, 1, 3])] = 0.5 * np.array([[1.0, -1.0, 0.0], [-1.0, 2.0, -1.0], [0.0, -1.0, 1.0]])
    # triangle (a, d, c): right angle at c -> legs a-c, c-d carry -1/2
    P2[np.ix_([0, 3, 2], [0, 3, 2])] = 0.5 * np.array([[1.0, 0.0, -1.0], [0.0, 1.0, -1.0], [-1.0, -1.0, 2.0]])
    load = h * h / 6.0 * np.array([2.0, 1.0, 1.0, 2.0])
    return P1, P2, load


class HDDPort:
    """Geometry + tracker plan built once; `forward(kappa)` runs one sample."""

    def __init__(self, level: int, observations, f=None, g=None):
        self.grid = Grid(level)
        self.nodes = full_tree(self.grid)
        self.root = self.nodes[-1]
        self.obs = tuple((str(k), int(i)) for k, i in observations)
        n = self.grid.n_nodes
        self.f = np.ones(n) if f is None else np.asarray(f, dtype=float)
        self.g = np.zeros(self.root.bnd.size) if g is None else np.asarray(g, dtype=float)
        self.by_depth = {}
        for nd in self.nodes:
            self.by_depth.setdefault(nd.depth, []).append(nd)
        owner = {}
        for nd in self.nodes:
            for idx in nd.gamma:
                owner[int(idx)] = nd.id
        root_bnd = set(int(i) for i in self.root.bnd)
        self.born = {}            # node id -> [point indices born there]
        self.perimeter_points = []
        self.mean_nodes = set()
        for kind, ident in self.obs:
            if kind == "point":
                if ident in root_bnd:
                    self.perimeter_points.append(ident)
                elif ident in owner:
                    self.born.setdefault(owner[ident], []).append(ident)
                else:
                    raise ValueError(f"mesh node {ident} not on any interface")
            elif kind == "mean":
                self.mean_nodes.add(ident)
            else:
                raise ValueError(f"unknown observation kind {kind!r}")
        self.P1, self.P2, self.load = cell_stencils(self.grid.h)

    # -- one merge (hdd.py:216-277) ------------------------------------------
    @staticmethod
    def _eliminate(nd, left, right):
        nb, ng = nd.bnd.size, nd.gamma.size
        nk, nw = nb + ng, nd.omega.size
        At = np.zeros((nk, nk))
        Bt = np.zeros((nk, nw))
        for (pg, pf), kp, wp in zip((left, right), nd.kpos, nd.wpos):
            At[np.ix_(kp, kp)] += pg
            Bt[np.ix_(kp, wp)] += pf
        A11, A12, A22 = At[:nb, :nb], At[:nb, nb:], At[nb:, nb:]
        if ng == 0:
            return (A11.copy(), Bt[:nb].copy()), (np.zeros((0, nb)), np.zeros((0, nw)))
        rhs = np.hstack([At[nb:, :nb], Bt[nb:]])
        fac = scipy.linalg.cho_factor(A22, lower=True, check_finite=False)
        X = scipy.linalg.cho_solve(fac, rhs, check_finite=False)
        Xa, Xb = X[:, :nb], X[:, nb:]
        pg = A11 - A12 @ Xa
        pg = 0.5 * (pg + pg.T)
        pf = Bt[:nb] - A12 @ Xb
        return (pg, pf), (-Xa, Xb)

    # -- functional lift (functionals.py:64-114) -----------------------------
    @staticmethod
    def _lift(nd, phi, parts):
        """parts: [(son index 0/1, coef, (l_g, l_f))]; returns father (l_g, l_f)."""
        nb, ng = nd.bnd.size, nd.gamma.size
        lg = np.zeros(nb)
        lf = np.zeros(nd.omega.size)
        z = np.zeros(ng)
        for s, c, (sg, sf) in parts:
            kp, wp = nd.kpos[s], nd.wpos[s]
            outer = kp < nb
            lg[kp[outer]] += c * sg[outer]
            z[kp[~outer] - nb] += c * sg[~outer]
            lf[wp] += c * sf
        if ng:
            lg += phi[0].T @ z
            lf += phi[1].T @ z
        return lg, lf

    def forward(self, kappa: np.ndarray, keep_psi: dict | None = None) -> np.ndarray:
        """S(kappa); if `keep_psi` is a dict it receives {node id: (psi_g, psi_f @ f)}
        (the reference's BuildDiagnostics(keep_psi=True), hdd.py:158, :376-391)."""
        kappa = np.asarray(kappa, dtype=float)
        N = self.grid.N
        live = {}
        means = {}
        tracked = {}
        for depth in sorted(self.by_depth, reverse=True):
            done = []
            for nd in self.by_depth[depth]:
                if nd.is_leaf:
                    i0, _, j0, _ = nd.rect
                    t = 2 * (i0 * N + j0)
                    live[nd.id] = (kappa[t] * self.P1 + kappa[t + 1] * self.P2, np.diag(self.load))
                    # leaf mean: area/3 per triangle vertex over the cell area
                    means[nd.id] = (np.array([1 / 3, 1 / 6, 1 / 6, 1 / 3]), np.zeros(4))
                    if nd.id in self.mean_nodes:
                        tracked[("mean", nd.id)] = (nd.id, means[nd.id])
                    continue
                s1, s2 = nd.sons
                psi, phi = self._eliminate(nd, live[s1], live[s2])
                live[nd.id] = psi
                if keep_psi is not None:
                    keep_psi[nd.id] = (psi[0], psi[1] @ self.f[nd.omega])
                done.append(nd)
                for idx in self.born.get(nd.id, ()):
                    e = np.zeros(nd.gamma.size)
                    e[int(np.searchsorted(nd.gamma, idx))] = 1.0
                    tracked[("point", idx)] = (nd.id, (phi[0].T @ e, phi[1].T @ e))
                for key, (own, fn) in list(tracked.items()):
                    if own == s1:
                        tracked[key] = (nd.id, self._lift(nd, phi, [(0, 1.0, fn)]))
                    elif own == s2:
                        tracked[key] = (nd.id, self._lift(nd, phi, [(1, 1.0, fn)]))
                means[nd.id] = self._lift(nd, phi, [(0, 0.5, means[s1]), (1, 0.5, means[s2])])
                del means[s1], means[s2]
                if nd.id in self.mean_nodes:
                    tracked[("mean", nd.id)] = (nd.id, means[nd.id])
            for nd in done:
                for s in nd.sons:
                    live.pop(s, None)
        out = np.empty(len(self.obs))
        for k, (kind, ident) in enumerate(self.obs):
            if kind == "point" and ident in self.perimeter_points:
                out[k] = self.g[int(np.searchsorted(self.root.bnd, ident))]
                continue
            own, (lg, lf) = tracked[(kind, ident)]
            assert own == self.root.id
            out[k] = float(lf @ self.f + lg @ self.g)
        if not np.all(np.isfinite(out)):
            raise FloatingPointError("non-finite forward observation")
        return out


def gaussian_ll(y, s, sigma) -> float:
    """bayes.py:222-224."""
    r = (np.asarray(y) - np.asarray(s)) / sigma
    return float(-0.5 * np.sum(r * r) - np.sum(np.log(sigma * math.sqrt(2.0 * math.pi))))
