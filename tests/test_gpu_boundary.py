"""The widened drop-in boundary on the device:

* duck-typed `problem.param` (only `.kappa(z)` is used, reference bayes.py:183, :204,
  :242): the fields come from the caller's host code and enter through
  hdd_forward_batch_kappa — SPEC #1-style random per-triangle kappa ~ U[0.1, 10]
  (reference tests/conftest.py:19-25), random f and g, points and means;
* mesh levels 1-3 (the reference accepts levels >= 1, mesh.py:92-93; its tests use
  level 3): one warp per sample eliminates the interior (tiny_kernel);
* asynchronous calls and failure reporting: the lowest failing sample of a call,
  across sub-batches, ConfigError for invalid fields, NumericalError for a
  non-finite forward value.

Everything is compared with the oracle's sparse direct solve (oracle/direct.py,
a restatement of reference oracle.direct_solve) at the BASELINE tolerance 1e-10.
"""
import numpy as np
import pytest

import paper_1708_02207_b200 as hb
from paper_1708_02207_b200 import bayes
from oracle import configs as ocfg, direct, fields, geometry

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


class Field:
    """Stand-in for the reference CoefficientField (fem.py:23-43): `.values` per triangle."""

    def __init__(self, values):
        self.values = np.asarray(values, dtype=float)


class TriangleParam:
    """Duck-typed param: kappa(z) = base * exp(z . modes), arbitrary per-triangle base
    (no separable tables, so the plan takes coefficient fields)."""

    def __init__(self, base, modes):
        self.base = np.asarray(base, dtype=float)
        self.modes = np.asarray(modes, dtype=float)
        self.n_z = self.modes.shape[0]

    def kappa(self, z):
        return Field(self.base * np.exp(np.asarray(z) @ self.modes))


def random_obs(rng, level, n_pts):
    mesh = hb.build_mesh(level)
    pts = rng.choice(mesh.n_nodes, size=min(n_pts, mesh.n_nodes), replace=False)
    obs = [("point", int(p)) for p in pts]
    for _ in range(int(rng.integers(1, 6))):
        d = int(rng.integers(0, 2 * level + 1))
        nodes = geometry.nodes_at_depth(level, d)
        obs.append(("mean", int(nodes[int(rng.integers(len(nodes)))][0])))
    rng.shuffle(obs)
    return tuple(obs)


def check_against_direct(level, S, kappas, f, g, obs):
    grid = geometry.Grid(level)
    for b in range(S.shape[0]):
        u = direct.solve(grid, kappas[b], f=f, g=g)
        ref = ocfg.observe(grid, u, obs)
        err = np.max(np.abs(S[b] - ref)) / max(np.max(np.abs(ref)), 1e-300)
        assert err <= TOL, (level, b, err)


@pytest.mark.parametrize("level", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("seed", [0, 1])
def test_random_triangle_kappa_matches_direct(cuda, level, seed):
    """SPEC #1 style: kappa ~ U[0.1, 10] per triangle, f ~ N(0,1), g ~ N(0,1)."""
    rng = np.random.default_rng(100 * level + seed)
    mesh = hb.build_mesh(level)
    tree = hb.build_tree(mesh)
    base = rng.uniform(0.1, 10.0, mesh.n_triangles)
    modes = 0.3 * rng.standard_normal((3, mesh.n_triangles))
    param = TriangleParam(base, modes)
    f = rng.standard_normal(mesh.n_nodes)
    g = rng.standard_normal(4 * mesh.n_cells)
    obs = random_obs(rng, level, 12)
    y = rng.standard_normal(len(obs)) * 0.01
    prob = hb.BayesProblem(tree, param, f, g, hb.MeasurementModel(obs, np.full(len(obs), 0.01), y))
    Z = rng.standard_normal((4, 3))
    S = hb.forward_functionals_batch(prob, Z)
    check_against_direct(level, S, [param.kappa(z).values for z in Z], f, g, obs)
    ll = hb.log_likelihood_batch(prob, Z)
    for b in range(Z.shape[0]):
        ref = hb.gaussian_log_likelihood(y, S[b], prob.model.sigma)
        assert abs(ll[b] - ref) <= 1e-12 * abs(ref)
    # the reference's single-sample plug-in points give the same numbers
    assert abs(hb.log_likelihood(prob, Z[1]) - ll[1]) <= 1e-12 * abs(ll[1])
    np.testing.assert_allclose(hb.forward_functionals(prob, Z[2]), S[2], rtol=0, atol=1e-14 * np.abs(S).max())
    info = prob.plan().info()
    assert info.separable == 0 and info.tiny == int(level < 4)


@pytest.mark.parametrize("level", [1, 2, 3])
def test_sine_kl_small_levels(cuda, level):
    """Separable (device K1) fields on meshes below one kernel leaf, f = 1, g = 0."""
    rng = np.random.default_rng(7 + level)
    mesh = hb.build_mesh(level)
    tree = hb.build_tree(mesh)
    n_z = 5
    obs = random_obs(rng, level, 9)
    prob = hb.BayesProblem(tree, hb.SineKLField(tree, n_z), np.ones(mesh.n_nodes), np.zeros(4 * mesh.n_cells),
                           hb.MeasurementModel(obs, np.full(len(obs), 0.01)))
    Z = rng.standard_normal((6, n_z))
    S = hb.forward_functionals_batch(prob, Z)
    fo = fields.SineKLField(geometry.Grid(level), n_z)
    check_against_direct(level, S, [fo.kappa_values(z) for z in Z], None, None, obs)
    torch = cuda
    Sd = hb.forward_functionals_batch(prob, torch.from_numpy(Z).cuda()).cpu().numpy()
    assert np.array_equal(Sd, S)


@pytest.mark.parametrize("level", [2, 3, 5])
def test_small_level_full_solution(cuda, level):
    rng = np.random.default_rng(level)
    mesh = hb.build_mesh(level)
    tree = hb.build_tree(mesh)
    param = TriangleParam(rng.uniform(0.1, 10.0, mesh.n_triangles), 0.2 * rng.standard_normal((2, mesh.n_triangles)))
    f = rng.standard_normal(mesh.n_nodes)
    g = rng.standard_normal(4 * mesh.n_cells)
    obs = (("point", mesh.n_nodes // 2),)
    prob = hb.BayesProblem(tree, param, f, g, hb.MeasurementModel(obs, np.ones(1)))
    Z = rng.standard_normal((3, 2))
    U = bayes.solve_batch(prob, Z)
    grid = geometry.Grid(level)
    for b in range(3):
        u = direct.solve(grid, param.kappa(Z[b]).values, f=f, g=g)
        assert np.max(np.abs(U[b] - u)) <= TOL * np.max(np.abs(u))


def test_invalid_fields_raise_config_error(cuda):
    mesh = hb.build_mesh(5)
    tree = hb.build_tree(mesh)
    rng = np.random.default_rng(3)

    class Bad(TriangleParam):
        def kappa(self, z):
            v = self.base.copy()
            if z[0] > 0.5:
                v[17] = -1.0
            return Field(v)

    param = Bad(rng.uniform(0.1, 10.0, mesh.n_triangles), np.zeros((1, mesh.n_triangles)))
    obs = (("point", 100),)
    prob = hb.BayesProblem(tree, param, np.ones(mesh.n_nodes), np.zeros(4 * mesh.n_cells),
                           hb.MeasurementModel(obs, np.ones(1), np.zeros(1)))
    Z = np.zeros((5, 1))
    Z[3, 0] = 1.0
    with pytest.raises(hb.ConfigError) as ei:
        hb.log_likelihood_batch(prob, Z)
    assert "positive finite" in str(ei.value)
    # the plan recovers after the failure
    ll = hb.log_likelihood_batch(prob, Z[:3])
    assert np.all(np.isfinite(ll))

    class Short(TriangleParam):
        def kappa(self, z):
            return Field(self.base[:-1])

    prob2 = hb.BayesProblem(tree, Short(param.base, param.modes), np.ones(mesh.n_nodes), np.zeros(4 * mesh.n_cells),
                            hb.MeasurementModel(obs, np.ones(1), np.zeros(1)))
    with pytest.raises(hb.ConfigError):
        hb.log_likelihood_batch(prob2, Z)


def _sub_batched_problem(level=5, max_batch=4):
    mesh = hb.build_mesh(level)
    tree = hb.build_tree(mesh)
    obs = (("point", 5 * mesh.m + 7), ("mean", tree.root_id))
    return hb.BayesProblem(tree, hb.SineKLField(tree, 2), np.ones(mesh.n_nodes), np.zeros(4 * mesh.n_cells),
                           hb.MeasurementModel(obs, np.full(2, 0.01), np.zeros(2)), max_batch=max_batch)


def test_failure_names_lowest_sample_across_sub_batches(cuda):
    """Sub-batches of 4: rows 9 and 6 carry a non-finite Z -> the error names row 6
    (global index, whichever CTA finishes first)."""
    prob = _sub_batched_problem()
    Z = np.zeros((12, 2))
    Z[9, 0] = np.inf
    Z[6, 1] = np.nan
    with pytest.raises(hb.ConfigError):
        hb.log_likelihood_batch(prob, Z)
    import ctypes as C
    from paper_1708_02207_b200 import _lib
    e = _lib.HddError()
    prob.plan().lib.hdd_last_error(prob.plan().handle, C.byref(e))
    assert e.sample == 6
    # torch path, asynchronous: the call returns, synchronize raises
    torch = cuda
    Zd = torch.from_numpy(Z).cuda()
    hb.log_likelihood_batch(prob, Zd, sync=False)
    with pytest.raises(hb.ConfigError):
        bayes.synchronize(prob)
    prob.plan().lib.hdd_last_error(prob.plan().handle, C.byref(e))
    assert e.sample == 6
    # clean batch afterwards: no stale failure
    ll = hb.log_likelihood_batch(prob, Zd[:4])
    assert torch.isfinite(ll).all()


def test_non_finite_forward_value_raises_numerical_error(cuda):
    """Coefficients at the bottom of the double range drive the interface pivots and
    the forward values out of range: NumericalError through the C ABI (the
    reference's non-finite check, bayes.py:196-197, and non-SPD pivot, hdd.py:271)."""
    mesh = hb.build_mesh(6)
    tree = hb.build_tree(mesh)
    param = TriangleParam(np.full(mesh.n_triangles, 1.0), np.ones((1, mesh.n_triangles)))
    obs = (("point", 20 * mesh.m + 30),)
    prob = hb.BayesProblem(tree, param, np.ones(mesh.n_nodes), np.zeros(4 * mesh.n_cells),
                           hb.MeasurementModel(obs, np.ones(1), np.zeros(1)))
    Z = np.array([[0.0], [-745.0], [0.0]])          # kappa = exp(-745) ~ 5e-324
    with pytest.raises(hb.NumericalError):
        hb.log_likelihood_batch(prob, Z)
    assert np.isfinite(hb.log_likelihood_batch(prob, Z[:1])).all()


def test_device_mismatch_is_usage_error(cuda):
    torch = cuda
    if torch.cuda.device_count() < 2:
        prob = _sub_batched_problem()
        prob.device = 0
        prob.plan()
        prob._plan.device = 1       # pretend the plan lives elsewhere
        with pytest.raises(hb.UsageError):
            hb.log_likelihood_batch(prob, torch.zeros((2, 2), dtype=torch.float64, device="cuda:0"))
        prob._plan.device = 0


def test_stage_kernel_names_follow_the_launch_rules(cuda):
    """hdd_plan_stage_kernel names the kernel each tree depth launches (bench.py groups
    its CUDA-event stage times by it): the kernel leaves, then tier-M merges for C2; a
    forced HBM-panel tier switches every depth to merge_l_kernel."""
    import ctypes as C
    import os

    from paper_1708_02207_b200 import configs

    def names(prob, B):
        plan = prob.plan()
        info = plan.info()
        out = []
        buf = C.create_string_buffer(160)
        for dep in [-1] + list(range(info.leaf_depth - 1, -1, -1)):
            plan.check(plan.lib.hdd_plan_stage_kernel(plan.handle, dep, B, buf, 160))
            out.append(buf.value.decode())
        assert plan.lib.hdd_plan_stage_kernel(plan.handle, info.leaf_depth + 3, B, buf, 160) != 0
        return out

    got = names(configs.make_problem("C2", device=0), 1024)
    assert got[0].startswith("leaf2_kernel<") and len(got) == 1 + 6
    assert all(n.startswith("merge_m2_kernel<8,") for n in got[1:])
    os.environ["HDD_FORCE_TIER_L"] = "1"
    try:
        got_l = names(configs.make_problem("C2", device=0), 1024)
    finally:
        del os.environ["HDD_FORCE_TIER_L"]
    assert all("merge_l_kernel<" in n for n in got_l[1:])
