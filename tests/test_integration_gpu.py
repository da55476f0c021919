"""INTEGRATION.md's binding (tools/hddsolve_b200.py) executed against the UNMODIFIED
reference package installed under baseline/_ref: the reference's own BayesProblem,
ParamField (indicator, bayes.py:50-77) and log_likelihood(..., forward=) plug-in point
(bayes.py:227-231), with the device forward, against the reference's pure-Python
forward at relative 1e-10 (levels 3 and 5, the reference tests' level and C1's)."""
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
LIB = ROOT / "paper_1708_02207_b200" / "libhdd_b200.so"

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not (REF / "hddsolve").is_dir():
        pytest.skip("reference not installed under baseline/_ref")
    for p in (str(REF), str(ROOT / "tools")):
        if p not in sys.path:
            sys.path.insert(0, p)
    import hddsolve
    return hddsolve


@pytest.mark.parametrize("level, n_z", [(3, 4), (5, 4)])
def test_reference_call_site_with_device_forward(ref, level, n_z):
    import hddsolve_b200
    from hddsolve import bayes
    mesh = ref.build_mesh(level)
    tree = ref.build_tree(mesh)
    param = bayes.ParamField.build(tree, n_z)
    rng = np.random.default_rng(level)
    m = mesh.m
    obs = [("point", int(i)) for i in rng.choice(mesh.n_nodes, 6, replace=False)]
    obs += list(bayes.mean_observations(tree, 2))
    sigma = np.full(len(obs), 0.01)
    y = rng.normal(0.05, 0.01, len(obs))
    f = rng.standard_normal(mesh.n_nodes)
    g = rng.standard_normal(4 * (m - 1))
    problem = bayes.BayesProblem(tree, param, f, g, bayes.MeasurementModel(tuple(obs), sigma, y))
    fwd = hddsolve_b200.device_forward_factory(problem, lib=str(LIB))
    Z = rng.standard_normal((3, n_z))
    for z in Z:
        ll_dev = bayes.log_likelihood(problem, z, forward=fwd)
        ll_ref = bayes.log_likelihood(problem, z)
        assert abs(ll_dev - ll_ref) <= 1e-10 * abs(ll_ref)
        s_dev = fwd(problem, z)
        s_ref = bayes.forward_functionals(problem, z)
        assert np.max(np.abs(s_dev - s_ref)) <= 1e-10 * np.max(np.abs(s_ref))
    S = fwd.batch(problem, Z)
    assert S.shape == (3, len(obs))
    class Neg:                                  # a param whose field is not positive
        def kappa(self, z):
            return _bad(mesh)

    p2 = bayes.BayesProblem(tree, Neg(), f, g, bayes.MeasurementModel(tuple(obs), sigma, y))
    with pytest.raises(ref.errors.ConfigError):
        hddsolve_b200.device_forward_factory(p2, lib=str(LIB)).batch(p2, np.ones((1, n_z)))


def _bad(mesh):
    class F:
        values = np.full(mesh.n_triangles, -1.0)
    return F()
