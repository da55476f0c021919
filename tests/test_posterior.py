"""Posterior drivers against the live reference's
posterior_grid / posterior_mcmc goldens (tests/golden/make_posterior_golden.py):
on CPU with the oracle port as the likelihood (driver logic), on the GPU through
the device likelihood.  Tolerances: log-likelihood / log-posterior / evidence
relative 1e-10; grid points, weights, mode and the chain's accept pattern exact."""
import numpy as np
import pytest

import paper_1708_02207_b200 as hb
from oracle import hdd_port
from paper_1708_02207_b200 import configs, posterior as post

TOL = 1e-10


def _problem(golden, n_z):
    g = golden("posterior")
    cfg = configs.CONFIGS["C1"]
    mesh = hb.build_mesh(cfg.level)
    tree = hb.build_tree(mesh)
    model = hb.MeasurementModel(configs.observations(cfg), g[f"sigma{n_z}"], g[f"y{n_z}"])
    return hb.BayesProblem(tree, hb.ParamField.build(tree, n_z), np.ones(mesh.n_nodes),
                           np.zeros(4 * mesh.n_cells), model)


def _port_ll(prob):
    port = hdd_port.HDDPort(prob.tree.mesh.level, prob.model.observations)

    def ll_batch(problem, Z):
        return np.array([hdd_port.gaussian_ll(problem.model.y, port.forward(problem.param.kappa_values(z)),
                                              problem.model.sigma) for z in Z])
    return ll_batch


def _check_grid(res, g, n_z):
    p = f"grid{n_z}_"
    assert np.array_equal(res.points, g[p + "points"])
    assert np.array_equal(res.weights, g[p + "weights"])
    assert np.allclose(res.log_prior, g[p + "log_prior"], rtol=0, atol=0)
    assert np.max(np.abs(res.log_like - g[p + "log_like"]) / np.abs(g[p + "log_like"])) <= TOL
    assert np.max(np.abs(res.log_post - g[p + "log_post"])) <= TOL * np.max(np.abs(g[p + "log_post"]))
    assert abs(res.log_evidence - float(g[p + "log_evidence"])) <= TOL * abs(float(g[p + "log_evidence"]))
    assert np.array_equal(res.mode, g[p + "mode"])
    assert abs(res.integral - 1.0) <= 1e-12


def _check_chain(res, g):
    assert np.array_equal(res.accepted, g["mcmc_accepted"])
    assert res.acceptance == float(g["mcmc_acceptance"])
    assert np.max(np.abs(res.points - g["mcmc_points"])) <= 1e-12
    assert np.max(np.abs(res.log_post - g["mcmc_log_post"]) / np.abs(g["mcmc_log_post"])) <= TOL


def _spec(g):
    length, burn, prop, seed = g["mcmc_spec"]
    return post.ChainSpec(length=int(length), burn=int(burn), proposal=float(prop), seed=int(seed))


GRIDS = {1: post.GridSpec((-1.5,), (1.5,), (9,)), 2: post.GridSpec((-1.0, -1.0), (1.2, 0.8), (6, 5))}


@pytest.mark.parametrize("n_z", [1, 2])
def test_grid_driver_matches_reference_cpu(golden, n_z):
    prob = _problem(golden, n_z)
    res = post.posterior_grid(prob, hb.Prior.normal(n_z), GRIDS[n_z], log_like_batch=_port_ll(prob))
    _check_grid(res, golden("posterior"), n_z)


def test_mcmc_driver_matches_reference_cpu(golden):
    prob = _problem(golden, 2)
    g = golden("posterior")
    res = post.posterior_mcmc(prob, hb.Prior.normal(2), _spec(g), log_like_batch=_port_ll(prob))
    _check_chain(res, g)


def test_driver_errors_and_helpers():
    with pytest.raises(hb.UsageError):
        post.posterior_grid(None, hb.Prior.normal(3), post.GridSpec((0,) * 3, (1,) * 3, (2,) * 3))
    with pytest.raises(hb.ConfigError):
        post.posterior_grid(None, hb.Prior.normal(2), post.GridSpec((0,), (1,), (2,)))
    with pytest.raises(hb.UsageError):
        post.posterior_mcmc(None, hb.Prior.normal(5), post.ChainSpec())
    a = np.array([-1000.0, -1001.0, -999.5])
    w = np.array([0.5, 1.0, 0.25])
    assert abs(post.logsumexp_weighted(a, w) - (-999.5 + np.log(np.sum(w * np.exp(a + 999.5))))) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("n_z", [1, 2])
def test_grid_posterior_on_device_matches_reference(golden, n_z):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    prob = _problem(golden, n_z)
    _check_grid(post.posterior_grid(prob, hb.Prior.normal(n_z), GRIDS[n_z]), golden("posterior"), n_z)


@pytest.mark.gpu
def test_mcmc_on_device_matches_reference_and_lockstep_chains(golden):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    prob = _problem(golden, 2)
    g = golden("posterior")
    spec = _spec(g)
    _check_chain(post.posterior_mcmc(prob, hb.Prior.normal(2), spec), g)
    chains = post.posterior_mcmc_chains(prob, hb.Prior.normal(2), spec, 3)
    _check_chain(chains[0], g)
    for c in (1, 2):
        single = post.posterior_mcmc(prob, hb.Prior.normal(2), post.ChainSpec(spec.length, spec.burn,
                                                                              spec.proposal, spec.seed + c))
        assert np.array_equal(chains[c].accepted, single.accepted)
        assert np.array_equal(chains[c].points, single.points)
