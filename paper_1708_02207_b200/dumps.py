"""Regression text dumps in the reference formats.

* `dump_store_stats` — hdd.py:532-541: one line per merge node, sorted by
  (depth, node id): `depth |boundary| |gamma| dense_bytes stored_bytes max_block_rank`.
  The reference's MapStats (hdd.py:140-151, filled at :363-372) hold the sizes of
  the dense maps Phi^g (gamma x boundary), Phi^f (gamma x omega), Psi^g
  (boundary x boundary) and Psi^f (boundary x omega) of every merge.  For a dense
  store these depend on the geometry only, so `store_stats(tree)` derives them from
  the tree; compressed stores (per-block SVD ranks of those four maps) are not
  reproducible from the device path, which condenses Psi^f/Phi^f into the load
  column and truncates Psi^g over the pruned boundary only.
* `dump_functionals` — functionals.py:248-255: one line per tracked functional,
  keys sorted by repr: `kind:id |l_g| |l_f| checksum`, checksum = sum(l_g) + sum(l_f).
  The device path never materialises l_g / l_f; the checksum is recovered exactly
  from what it computes:
    - sum(l_f) = <l_f, 1> is the observation S for the load f = 1, g = 0, i.e. one
      forward evaluation of the problem with a unit right-hand side;
    - sum(l_g) = <l_g, 1> is the observation for g = 1, f = 0, whose discrete
      solution is u = 1 (stiffness rows sum to zero); every point value and every
      subdomain mean of u = 1 is 1.
  |l_g| = |boundary of the root| = 4N and |l_f| = |omega of the root| = (N+1)^2 for
  every key (functionals live at the root once finished, functionals.py:209-223).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import UsageError
from .geometry import DDTree, _split

__all__ = ["MapStats", "StoreStats", "store_stats", "dump_store_stats",
           "FunctionalSummary", "functional_summaries", "dump_functionals"]


@dataclass(frozen=True)
class MapStats:
    """Per-merge storage record, field for field the reference's MapStats."""

    node_id: int
    depth: int
    n_boundary: int
    n_interface: int
    phi_dense_bytes: int
    phi_bytes: int
    psi_dense_bytes: int
    psi_bytes: int
    max_block_rank: int


@dataclass
class StoreStats:
    """The `stats` part of a reference MapStore (hdd.py:166-183)."""

    stats: list


def store_stats(tree: DDTree, compression=None) -> StoreStats:
    """MapStats of every merge node of a dense `leaves_to_root` sweep over `tree`."""
    if compression is not None:
        raise UsageError("compressed map statistics are not available on the device path "
                         "(Psi^f / Phi^f are condensed, Psi^g is truncated over the pruned boundary)")
    out = []

    def rec(r, depth, lo):
        i0, i1, j0, j1 = r
        w, hh = i1 - i0, j1 - j0
        nid = lo + (1 << (tree.depth - depth + 1)) - 2
        if w * hh == 1:
            return
        s1, s2 = _split(r, depth)
        rec(s1, depth + 1, lo)
        rec(s2, depth + 1, lo + (1 << (tree.depth - depth)) - 1)
        nb = 2 * (w + hh)
        ng = (hh - 1) if s1[1] != i1 else (w - 1)
        nw = (w + 1) * (hh + 1)
        phi = 8 * (ng * nb + ng * nw)
        psi = 8 * (nb * nb + nb * nw)
        out.append(MapStats(nid, depth, nb, ng, phi, phi, psi, psi, 0))

    N = tree.mesh.n_cells
    rec((0, N, 0, N), 0, 0)
    return StoreStats(stats=out)


def dump_store_stats(store) -> str:
    """Text lines `node_depth |boundary| |gamma| dense_bytes compressed_bytes max_block_rank`
    (hdd.py:532-541); `store` is a StoreStats (or anything with `.stats`)."""
    lines = []
    for st in sorted(store.stats, key=lambda s: (s.depth, s.node_id)):
        dense = st.phi_dense_bytes + st.psi_dense_bytes
        stored = st.phi_bytes + st.psi_bytes
        lines.append(f"{st.depth} {st.n_boundary} {st.n_interface} {dense} {stored} {st.max_block_rank}")
    return "\n".join(lines) + "\n"


@dataclass(frozen=True)
class FunctionalSummary:
    """What dump_functionals reads of a finished reference Functional."""

    node_id: int
    l_g_size: int
    l_f_size: int
    checksum: float


def functional_summaries(problem, z, forward=None) -> dict:
    """{("point", idx) | ("mean", node_id): FunctionalSummary} for the observations of
    `problem` at parameter z — the keys FunctionalTracker.finish returns for
    problem._requests() (functionals.py:138-224, bayes.py:168-177)."""
    from .bayes import BayesProblem, forward_functionals_batch

    if forward is None:
        forward = forward_functionals_batch
    mesh = problem.tree.mesh
    unit = problem
    if not problem._f_is_one or np.any(problem.g != 0.0):
        unit = BayesProblem(problem.tree, problem.param, np.ones(mesh.n_nodes), np.zeros(4 * mesh.n_cells), problem.model,
                            compression=problem.compression, device=problem.device, mode=problem.mode)
    S = np.asarray(forward(unit, np.asarray(z, dtype=float)[None]), dtype=float).reshape(-1)
    root = problem.tree.root_id
    n_b, n_w = 4 * mesh.n_cells, (mesh.n_cells + 1) ** 2
    out = {}
    for k, (kind, ident) in enumerate(problem.model.observations):
        key = ("mean", int(ident)) if kind == "mean" else ("point", int(ident))
        out[key] = FunctionalSummary(root, n_b, n_w, 1.0 + float(S[k]))
    return out


def dump_functionals(functionals) -> str:
    """Text lines `kind:id |l_g| |l_f| checksum` (functionals.py:248-255)."""
    lines = []
    for key in sorted(functionals, key=repr):
        fn = functionals[key]
        lines.append(f"{key[0]}:{key[1]} {fn.l_g_size} {fn.l_f_size} {fn.checksum:.12e}")
    return "\n".join(lines) + "\n"
