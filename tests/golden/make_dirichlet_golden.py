"""Non-zero Dirichlet data goldens from the LIVE reference (build container only).

Run:  python tests/golden/make_dirichlet_golden.py  -> dirichlet.npz

The unmodified reference `forward_functionals` (bayes.py:180-198) on a level-5 problem
with the reference's indicator ParamField (n_z = 4), a nodal f and Dirichlet data g over
root.idx_boundary, observing interior lattice points, boundary points and node means
at several depths (including nodes below the 16x16-cell level), at four z.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import hddsolve as hs  # noqa: E402
from hddsolve import bayes  # noqa: E402

L = 5


def main():
    rng = np.random.default_rng(2024)
    mesh = hs.build_mesh(L)
    tree = hs.build_tree(mesh)
    m = mesh.m
    lat = [4, 12, 20, 28]
    obs = [("point", j * m + i) for j in lat for i in lat]
    obs += [("point", 0), ("point", 9), ("point", 17 * m), ("point", 20 * m + 32), ("point", m * m - 3)]
    for d in (0, 2, 3, 6, 10):
        nodes = tree.nodes_at_depth(d)
        obs += [("mean", nodes[0].id), ("mean", nodes[-1].id)]
    f = rng.uniform(0.5, 1.5, mesh.n_nodes)
    g = np.sin(np.linspace(0.0, 6.0, 4 * (m - 1))) + 0.3
    pf = bayes.ParamField.build(tree, 4)
    model = bayes.MeasurementModel(tuple(obs), np.full(len(obs), 0.01), None)
    prob = bayes.BayesProblem(tree, pf, f, g, model)
    Z = rng.standard_normal((4, 4))
    S = np.stack([bayes.forward_functionals(prob, z) for z in Z])
    np.savez_compressed(HERE / "dirichlet.npz", Z=Z, S=S, f=f, g=g,
                        kind=np.array([k for k, _ in obs]), ident=np.array([i for _, i in obs], dtype=np.int64))


if __name__ == "__main__":
    main()
