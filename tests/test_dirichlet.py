"""Non-zero Dirichlet data g (the reference's BayesProblem.g over root.idx_boundary)
against the live reference's forward_functionals (tests/golden/make_dirichlet_golden.py):
the oracle port and the emulated host plan on CPU, the device path on the GPU.
Tolerance: relative 1e-11 (normwise over the observation vector)."""
import numpy as np
import pytest

import paper_1708_02207_b200 as hb
import plan_emulator as pe
from oracle import direct, fields, geometry, hdd_port

TOL = 1e-11


def _problem(golden, device=0, mode=-1):
    d = golden("dirichlet")
    mesh = hb.build_mesh(5)
    tree = hb.build_tree(mesh)
    obs = tuple((str(k), int(i)) for k, i in zip(d["kind"], d["ident"]))
    model = hb.MeasurementModel(obs, np.full(len(obs), 0.01))
    return hb.BayesProblem(tree, hb.ParamField.build(tree, 4), d["f"], d["g"], model,
                           device=device, mode=mode), d


def _err(S, ref):
    return np.max(np.abs(S - ref)) / np.max(np.abs(ref))


def test_oracle_port_matches_reference(golden):
    prob, d = _problem(golden, device=-1)
    port = hdd_port.HDDPort(5, prob.model.observations, f=d["f"], g=d["g"])
    for z, ref in zip(d["Z"], d["S"]):
        assert _err(port.forward(prob.param.kappa_values(z)), ref) <= TOL


@pytest.mark.parametrize("mode", [0, 1])
def test_emulated_plan_matches_reference(golden, mode):
    prob, d = _problem(golden, device=-1, mode=mode)
    grid = geometry.Grid(5)
    ind = fields.IndicatorField(grid, 4)
    for z, ref in zip(d["Z"], d["S"]):
        S, _, _ = pe.run(prob.plan(), 5, ind.kappa_values(z), d["f"])
        assert _err(S, ref) <= TOL
        u = direct.solve(grid, ind.kappa_values(z), f=d["f"], g=d["g"])
        assert abs(u[0] - d["g"][0]) == 0.0


def test_non_finite_g_rejected():
    mesh = hb.build_mesh(4)
    tree = hb.build_tree(mesh)
    g = np.zeros(4 * mesh.n_cells)
    g[3] = np.nan
    with pytest.raises(hb.ConfigError):
        hb.BayesProblem(tree, hb.ParamField.build(tree, 2), np.ones(mesh.n_nodes), g,
                        hb.MeasurementModel((("point", 20),), np.ones(1)), device=-1)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1])
def test_device_matches_reference(golden, mode):
    prob, d = _problem(golden, mode=mode)
    S = hb.forward_functionals_batch(prob, d["Z"])
    assert _err(S, d["S"]) <= TOL


@pytest.mark.gpu
def test_device_full_solution_with_dirichlet_data(golden):
    """solve_batch: u = g on the domain boundary, the direct solve inside."""
    prob, d = _problem(golden)
    U = hb.solve_batch(prob, d["Z"][:2])
    grid = geometry.Grid(5)
    ind = fields.IndicatorField(grid, 4)
    for b in range(2):
        u = direct.solve(grid, ind.kappa_values(d["Z"][b]), f=d["f"], g=d["g"])
        assert np.max(np.abs(U[b] - u)) <= TOL * np.max(np.abs(u))
    assert np.allclose(hb.forward_full_solve(prob, d["Z"][0]), d["S"][0], rtol=0, atol=TOL * np.abs(d["S"]).max())
