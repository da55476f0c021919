"""dump_functionals / dump_store_stats goldens from the LIVE reference (build container only).

Run:  python tests/golden/make_text_dump_golden.py

Imports the unmodified reference package from /root/reference/pkg/src and records
* `functionals.dump_functionals` (functionals.py:248-255) of a level-5 problem with the
  reference's indicator ParamField (n_z = 4), point observations (interior lattice,
  two points on the domain boundary) and node means at depths 1..3, at two z;
* `hdd.dump_store_stats` (hdd.py:532-541) of the dense store of the level-4 and
  level-5 trees (functionals_only mode, no compression).
The GPU box never sees /root/reference; the tests read only the text fixtures.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import hddsolve as hs  # noqa: E402
from hddsolve import bayes, functionals, hdd  # noqa: E402

L = 5
ZS = ([0.3, -0.5, 0.8, 0.1], [-1.1, 0.4, 0.0, 0.9])


def observations(tree):
    m = 2 ** L + 1
    lat = [4, 12, 20, 28]
    obs = [("point", j * m + i) for j in lat for i in lat]
    obs += [("point", 5), ("point", 7 * m)]                        # on the domain boundary
    for d in (1, 2, 3):
        obs += [("mean", nd.id) for nd in tree.nodes_at_depth(d)]
    return obs


def main():
    mesh = hs.build_mesh(L)
    tree = hs.build_tree(mesh)
    obs = observations(tree)
    pf = bayes.ParamField.build(tree, 4)
    model = bayes.MeasurementModel(tuple(obs), np.full(len(obs), 0.01), None)
    prob = bayes.BayesProblem(tree, pf, np.ones(mesh.n_nodes), np.zeros(4 * (mesh.m - 1)), model)
    meta = {"level": L, "observations": obs, "z": ZS}
    for k, z in enumerate(ZS):
        tracker = functionals.FunctionalTracker(tree, prob._requests())
        store = hdd.leaves_to_root(tree, pf.kappa(np.array(z)), hdd.SolveMode.functionals_only(),
                                   tracker=tracker)
        (HERE / f"dump_functionals_L{L}_z{k}.txt").write_text(functionals.dump_functionals(store.functionals))
    (HERE / f"dump_functionals_L{L}.json").write_text(json.dumps(meta))
    for lev in (4, 5):
        t = hs.build_tree(hs.build_mesh(lev))
        pf = bayes.ParamField.build(t, 4)
        store = hdd.leaves_to_root(t, pf.kappa(np.zeros(4)), hdd.SolveMode.functionals_only())
        (HERE / f"dump_store_stats_L{lev}.txt").write_text(hdd.dump_store_stats(store))


if __name__ == "__main__":
    main()
