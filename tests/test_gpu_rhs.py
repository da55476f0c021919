"""General maps applied to new data: per-call right-hand sides f
and Dirichlet data g without a new plan — one shared row or one row per sample
("multiple right-hand sides and multiple Dirichlet data"; PsiMap.residual
/ PhiMap.apply, hdd.py:58-105) — and the two-grid right-hand side (f given on a coarser
grid, prolonged bilinearly).  Against the oracle's sparse direct solve at
relative 1e-10 (BASELINE tolerance)."""
import numpy as np
import pytest

import paper_1708_02207_b200 as hb
from oracle import configs as ocfg, direct, fields, geometry

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(np.max(np.abs(b)), 1e-300))


def setup(level, n_z, seed, mode=-1):
    rng = np.random.default_rng(seed)
    mesh = hb.build_mesh(level)
    tree = hb.build_tree(mesh)
    pts = rng.choice(mesh.n_nodes, size=min(20, mesh.n_nodes), replace=False)
    obs = [("point", int(p)) for p in pts]
    for d in (0, min(3, 2 * level), 2 * level):
        nodes = geometry.nodes_at_depth(level, d)
        obs.append(("mean", int(nodes[int(rng.integers(len(nodes)))][0])))
    obs = tuple(obs)
    prob = hb.BayesProblem(tree, hb.SineKLField(tree, n_z), np.ones(mesh.n_nodes), np.zeros(4 * mesh.n_cells),
                           hb.MeasurementModel(obs, np.full(len(obs), 0.01)), mode=mode)
    return rng, mesh, prob, obs


@pytest.mark.parametrize("level, mode", [(3, -1), (5, 0), (5, 1), (6, 0), (7, 1)])
def test_per_sample_rhs_matches_direct(cuda, level, mode):
    rng, mesh, prob, obs = setup(level, 4, 10 * level + mode + 1, mode)
    B = 4
    Z = rng.standard_normal((B, 4))
    F = rng.standard_normal((B, mesh.n_nodes))
    G = rng.standard_normal((B, 4 * mesh.n_cells))
    S = hb.forward_functionals_batch(prob, Z, f=F, g=G)
    grid = geometry.Grid(level)
    fo = fields.SineKLField(grid, 4)
    for b in range(B):
        u = direct.solve(grid, fo.kappa_values(Z[b]), f=F[b], g=G[b])
        assert rel(S[b], ocfg.observe(grid, u, obs)) <= TOL, (level, mode, b)
    # device tensors give the same numbers
    torch = cuda
    Sd = hb.forward_functionals_batch(prob, torch.from_numpy(Z).cuda(), f=torch.from_numpy(F).cuda(),
                                      g=torch.from_numpy(G).cuda()).cpu().numpy()
    assert np.array_equal(Sd, S)
    # the plan's own (f = 1, g = 0) data is untouched afterwards
    S0 = hb.forward_functionals_batch(prob, Z)
    u0 = direct.solve(grid, fo.kappa_values(Z[0]))
    assert rel(S0[0], ocfg.observe(grid, u0, obs)) <= TOL


def test_many_rhs_one_coefficient(cuda):
    """One kappa, eight (f, g) pairs in one batch (the HDD multiple-RHS use case), and a
    shared row broadcast over the batch."""
    rng, mesh, prob, obs = setup(6, 3, 77)
    z = rng.standard_normal(3)
    Z = np.repeat(z[None], 8, axis=0)
    F = rng.standard_normal((8, mesh.n_nodes))
    G = rng.uniform(-1, 1, (8, 4 * mesh.n_cells))
    S = hb.forward_functionals_batch(prob, Z, f=F, g=G)
    grid = geometry.Grid(6)
    kap = fields.SineKLField(grid, 3).kappa_values(z)
    for b in range(8):
        assert rel(S[b], ocfg.observe(grid, direct.solve(grid, kap, f=F[b], g=G[b]), obs)) <= TOL
    Sh = hb.forward_functionals_batch(prob, Z[:3], f=F[5], g=G[5])          # one shared row
    for b in range(3):
        assert np.array_equal(Sh[b], S[5])
    # linearity in (f, g): S(f1 + f2, g1 + g2) = S(f1, g1) + S(f2, g2) - S(0, 0)
    S12 = hb.forward_functionals_batch(prob, Z[:1], f=F[0] + F[1], g=G[0] + G[1])
    S00 = hb.forward_functionals_batch(prob, Z[:1], f=np.zeros(mesh.n_nodes), g=np.zeros(4 * mesh.n_cells))
    assert rel(S12[0], S[0] + S[1] - S00[0]) <= 1e-9


@pytest.mark.parametrize("level", [2, 5, 6])
def test_full_solution_with_new_data(cuda, level):
    rng, mesh, prob, obs = setup(level, 2, 5 + level)
    Z = rng.standard_normal((3, 2))
    F = rng.standard_normal((3, mesh.n_nodes))
    G = rng.standard_normal((3, 4 * mesh.n_cells))
    U = hb.solve_batch(prob, Z, f=F, g=G)
    grid = geometry.Grid(level)
    fo = fields.SineKLField(grid, 2)
    for b in range(3):
        assert rel(U[b], direct.solve(grid, fo.kappa_values(Z[b]), f=F[b], g=G[b])) <= TOL


def test_two_grid_rhs(cuda):
    """f given on the level-4 grid, prolonged to level 7: the device result equals the
    fine run with the prolonged data bit-exactly and matches the direct solve."""
    rng, mesh, prob, obs = setup(7, 4, 3)
    fc = rng.standard_normal(17 * 17)
    fh = hb.prolong_rhs(fc, 4, 7)
    assert fh.shape == (mesh.n_nodes,)
    assert np.array_equal(fh.reshape(129, 129)[::8, ::8], fc.reshape(17, 17))   # injection at coarse nodes
    Z = rng.standard_normal((2, 4))
    S = hb.forward_functionals_batch(prob, Z, f=fh)
    grid = geometry.Grid(7)
    fo = fields.SineKLField(grid, 4)
    for b in range(2):
        assert rel(S[b], ocfg.observe(grid, direct.solve(grid, fo.kappa_values(Z[b]), f=fh), obs)) <= TOL


def test_bad_rows_are_usage_errors(cuda):
    rng, mesh, prob, obs = setup(5, 2, 1)
    with pytest.raises(hb.UsageError):
        hb.forward_functionals_batch(prob, np.zeros((3, 2)), f=np.ones(7))
    with pytest.raises(hb.UsageError):
        hb.forward_functionals_batch(prob, np.zeros((3, 2)), g=np.ones((2, 4 * mesh.n_cells)))


@pytest.mark.parametrize("level, depth", [(2, 2), (4, 5), (6, 0), (6, 3), (7, 6), (7, 9), (7, 13)])
def test_solve_subdomain_partial_inverse(cuda, level, depth):
    """solve_subdomain as a partial inverse (hdd.py:435-490 with keep_path): only the
    path and the target's subtree are factored and swept; the values equal the
    full-solution sweep bitwise (same arithmetic on the visited nodes) and the direct
    solve at 1e-10, also with per-call f and g."""
    rng, mesh, prob, obs = setup(level, 3, 40 + level + depth)
    tree = prob.tree
    nodes = tree.nodes_at_depth(depth)
    target = nodes[int(rng.integers(len(nodes)))]
    Z = rng.standard_normal((3, 3))
    Us = hb.solve_subdomain_batch(prob, Z, target.id)
    U = hb.solve_batch(prob, Z)
    idx = hb.omega_nodes(mesh, target.cells)
    assert Us.shape == (3, idx.size)
    assert np.array_equal(Us, U[:, idx])
    F = rng.standard_normal((3, mesh.n_nodes))
    G = rng.standard_normal((3, 4 * mesh.n_cells))
    Us2 = hb.solve_subdomain_batch(prob, Z, target.id, f=F, g=G)
    grid = geometry.Grid(level)
    fo = fields.SineKLField(grid, 3)
    for b in range(3):
        u = direct.solve(grid, fo.kappa_values(Z[b]), f=F[b], g=G[b])
        assert rel(Us2[b], u[idx]) <= TOL
    assert np.array_equal(hb.solve_subdomain(prob, Z[1], target.id), Us[1])
    sub = prob._sub_plans[target.id].info()
    full = prob.solve_plan().info()
    if full.leaf_depth > 0 and depth > 0:
        assert sub.factor_doubles < full.factor_doubles and sub.n_topdown < full.n_topdown
