"""Posterior-driver goldens from the LIVE reference (build container only).

Run:  python tests/golden/make_posterior_golden.py

Imports the unmodified reference package `hddsolve` from /root/reference/pkg/src,
builds a level-5 problem with the reference's own indicator ParamField (n_z = 1
and 2, the C1 lattice observations), attaches data from the reference's
`synthesize_data` (direct-solver truth + seeded noise), and records the results
of `posterior_grid` and `posterior_mcmc` (bayes.py:305-377) into posterior.npz.
The GPU box never sees /root/reference; tests read only the fixture.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parents[1]))

import hddsolve as hs  # noqa: E402
from hddsolve import bayes  # noqa: E402

from oracle import configs  # noqa: E402


def problem(n_z):
    cfg = configs.CONFIGS["C1"]
    m = hs.build_mesh(cfg.level)
    tree = hs.build_tree(m)
    obs = configs.observations(cfg)
    pf = bayes.ParamField.build(tree, n_z)
    model = bayes.MeasurementModel(obs, np.full(len(obs), 0.01), None)
    prob = bayes.BayesProblem(tree, pf, np.ones(m.n_nodes), np.zeros(4 * (m.m - 1)), model)
    z_true = np.array([0.4, -0.3][:n_z])
    model = bayes.synthesize_data(prob, z_true, 0.02, seed=17)
    return bayes.BayesProblem(tree, pf, np.ones(m.n_nodes), np.zeros(4 * (m.m - 1)), model)


def main():
    out = {}
    for n_z, spec in ((1, bayes.GridSpec((-1.5,), (1.5,), (9,))), (2, bayes.GridSpec((-1.0, -1.0), (1.2, 0.8), (6, 5)))):
        prob = problem(n_z)
        prior = bayes.Prior.normal(n_z)
        out[f"y{n_z}"] = prob.model.y
        out[f"sigma{n_z}"] = prob.model.sigma
        g = bayes.posterior_grid(prob, prior, spec)
        for k in ("points", "log_prior", "log_like", "log_post", "mode", "weights"):
            out[f"grid{n_z}_{k}"] = getattr(g, k)
        out[f"grid{n_z}_log_evidence"] = np.array(g.log_evidence)
    prob = problem(2)
    chain = bayes.ChainSpec(length=40, burn=10, proposal=0.2, seed=5)
    c = bayes.posterior_mcmc(prob, bayes.Prior.normal(2), chain)
    for k in ("points", "log_prior", "log_like", "log_post", "accepted"):
        out[f"mcmc_{k}"] = getattr(c, k)
    out["mcmc_acceptance"] = np.array(c.acceptance)
    out["mcmc_spec"] = np.array([chain.length, chain.burn, chain.proposal, chain.seed])
    np.savez_compressed(HERE / "posterior.npz", **out)
    print("wrote", HERE / "posterior.npz", {k: np.shape(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
