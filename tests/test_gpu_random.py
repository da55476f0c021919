"""Randomised parity sweep: random levels, parameter dimensions, observation sets
(interior / interface / boundary points, subdomain means at every depth of the tree,
down to single cells inside the kernel leaves), right-hand sides f, Dirichlet data g
and evaluation modes against the oracle's sparse direct solve
(relative 1e-10, the BASELINE tolerance)."""
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


@pytest.mark.parametrize("seed", range(8))
def test_random_problem_matches_direct_solve(cuda, seed):
    rng = np.random.default_rng(1000 + seed)
    level = int(rng.choice([4, 5, 6, 7]))
    n_z = int(rng.integers(1, 12))
    mesh = hb.build_mesh(level)
    tree = hb.build_tree(mesh)
    m = mesh.m
    pts = rng.choice(mesh.n_nodes, size=int(rng.integers(1, 40)), replace=False)
    obs = [("point", int(p)) for p in pts]
    for _ in range(int(rng.integers(0, 8))):
        d = int(rng.integers(0, 2 * level + 1))
        nodes = geometry.nodes_at_depth(level, d)
        obs.append(("mean", int(nodes[int(rng.integers(len(nodes)))][0])))
    rng.shuffle(obs)
    obs = tuple(obs)
    f = rng.uniform(-1.0, 2.0, mesh.n_nodes) if rng.random() < 0.5 else np.ones(mesh.n_nodes)
    g = rng.uniform(-1.0, 1.0, 4 * mesh.n_cells) if rng.random() < 0.5 else np.zeros(4 * mesh.n_cells)
    mode = int(rng.choice([-1, 0, 1]))
    prob = hb.BayesProblem(tree, hb.SineKLField(tree, n_z), f, g,
                           hb.MeasurementModel(obs, np.full(len(obs), 0.01)), mode=mode)
    grid = geometry.Grid(level)
    fo = fields.SineKLField(grid, n_z)
    Z = 1.5 * rng.standard_normal((3, n_z))
    S = hb.forward_functionals_batch(prob, Z)
    for b in range(Z.shape[0]):
        u = direct.solve(grid, fo.kappa_values(Z[b]), f=f, g=g)
        ref = ocfg.observe(grid, u, obs)
        assert np.max(np.abs(S[b] - ref)) <= TOL * max(np.max(np.abs(ref)), 1e-300), (level, n_z, mode, obs)
    assert m == grid.m


@pytest.mark.parametrize("level, n_pts, mode", [(4, 50, 0), (4, 50, 1), (6, 30, 0), (6, 30, 1)])
def test_many_points_inside_one_leaf(cuda, level, n_pts, mode):
    """Leaves with more observation columns than one 8-column pass: the 8-column leaf
    class runs ceil((ncols - 1) / 7) passes (load + 7 columns each)."""
    rng = np.random.default_rng(level * 100 + n_pts + mode)
    mesh = hb.build_mesh(level)
    tree = hb.build_tree(mesh)
    m = mesh.m
    # points strictly inside the first 16x16-cell leaf (not on its in-leaf interfaces only)
    inner = np.array([j * m + i for j in range(1, 16) for i in range(1, 16)])
    obs = tuple(("point", int(p)) for p in rng.choice(inner, n_pts, replace=False))
    prob = hb.BayesProblem(tree, hb.SineKLField(tree, 5), np.ones(mesh.n_nodes), np.zeros(4 * mesh.n_cells),
                           hb.MeasurementModel(obs, np.full(len(obs), 0.01)), mode=mode)
    grid = geometry.Grid(level)
    fo = fields.SineKLField(grid, 5)
    Z = rng.standard_normal((2, 5))
    S = hb.forward_functionals_batch(prob, Z)
    for b in range(2):
        ref = ocfg.observe(grid, direct.solve(grid, fo.kappa_values(Z[b])), obs)
        assert np.max(np.abs(S[b] - ref)) <= TOL * np.max(np.abs(ref))


@pytest.mark.parametrize("mode", [0, 1])
def test_sub_leaf_means(cuda, mode):
    """Means of tree nodes below the 16x16-cell kernel leaves (functionals.py:47-61 at
    any depth): every depth 5..12 of a level-6 tree, a dozen inside one leaf (two
    column passes), next to own-leaf means, in-leaf points and a nodal f."""
    rng = np.random.default_rng(77 + mode)
    level = 6
    mesh = hb.build_mesh(level)
    tree = hb.build_tree(mesh)
    obs = []
    for d in range(5, 13):
        nodes = geometry.nodes_at_depth(level, d)
        obs += [("mean", int(nodes[int(i)][0])) for i in rng.choice(len(nodes), 3, replace=False)]
    first_leaf = [nid for nid, rect in geometry.nodes_at_depth(level, 8) if rect[1] <= 16 and rect[3] <= 16]
    obs += [("mean", int(n)) for n in first_leaf[:12]]
    obs += [("mean", int(geometry.nodes_at_depth(level, 4)[0][0])), ("point", 65 * 5 + 7), ("point", 65 * 40 + 41)]
    obs = tuple(obs)
    f = rng.uniform(0.5, 2.0, mesh.n_nodes)
    prob = hb.BayesProblem(tree, hb.SineKLField(tree, 6), f, np.zeros(4 * mesh.n_cells),
                           hb.MeasurementModel(obs, np.full(len(obs), 0.01)), mode=mode)
    assert prob.plan().info().mode == mode
    grid = geometry.Grid(level)
    fo = fields.SineKLField(grid, 6)
    Z = rng.standard_normal((3, 6))
    S = hb.forward_functionals_batch(prob, Z)
    for b in range(3):
        ref = ocfg.observe(grid, direct.solve(grid, fo.kappa_values(Z[b]), f=f), obs)
        assert np.max(np.abs(S[b] - ref)) <= TOL * np.max(np.abs(ref))
