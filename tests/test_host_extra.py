"""CPU checks of the round-2 host logic: two-grid prolongation, plans below one kernel
leaf (levels 1-3), the restricted primal top-down lists, the per-call right-hand-side
checks, and the new golden files pinned against the oracle."""
import numpy as np
import pytest

import paper_1708_02207_b200 as hb
from oracle import configs as ocfg, direct, fields, geometry


def test_prolong_rhs_is_exact_on_bilinear_functions():
    for lc, lf in ((1, 1), (2, 5), (3, 4)):
        mc, mf = (1 << lc) + 1, (1 << lf) + 1
        xc = np.linspace(0, 1, mc)
        xf = np.linspace(0, 1, mf)
        fcoarse = (1 + 2 * xc[None, :] - 3 * xc[:, None] + 0.5 * xc[None, :] * xc[:, None]).reshape(-1)
        want = (1 + 2 * xf[None, :] - 3 * xf[:, None] + 0.5 * xf[None, :] * xf[:, None]).reshape(-1)
        assert np.max(np.abs(hb.prolong_rhs(fcoarse, lc, lf) - want)) <= 1e-14
    with pytest.raises(hb.ConfigError):
        hb.prolong_rhs(np.zeros(9), 2, 1)
    with pytest.raises(hb.ConfigError):
        hb.prolong_rhs(np.zeros(8), 1, 3)


def _host_problem(level, obs, **kw):
    mesh = hb.build_mesh(level)
    tree = hb.build_tree(mesh)
    return hb.BayesProblem(tree, hb.SineKLField(tree, 3), np.ones(mesh.n_nodes), np.zeros(4 * mesh.n_cells),
                           hb.MeasurementModel(obs, np.ones(len(obs))), device=-1, **kw)


@pytest.mark.parametrize("level", [1, 2, 3])
def test_small_level_plans(level):
    mesh = hb.build_mesh(level)
    tree = hb.build_tree(mesh)
    obs = (("point", 0), ("point", mesh.n_nodes // 2), ("mean", tree.root_id),
           ("mean", tree.nodes_at_depth(2 * level)[0].id))
    info = _host_problem(level, obs).plan().info()
    assert info.tiny == 1 and info.leaf_depth == 0 and info.n_upper == 0 and info.n_leaves == 0
    with pytest.raises(hb.UsageError):
        _host_problem(level, (("mean", tree.n_nodes),)).plan()


def test_restricted_top_down_lists():
    """Primal plans visit only the ancestors of the observation owners: one point deep in
    the tree visits one node per depth; points everywhere visit more."""
    level = 7
    mesh = hb.build_mesh(level)
    one = _host_problem(level, (("point", 40 * mesh.m + 41),), mode=1).plan().info()
    assert one.mode == 1 and one.n_topdown == 2 * (level - 4)      # one node per upper depth
    pts = tuple(("point", int(i)) for i in range(mesh.m + 1, mesh.n_nodes - mesh.m - 1, 97))
    many = _host_problem(level, pts, mode=1).plan().info()
    assert one.n_topdown < many.n_topdown <= many.n_upper


def test_wide_goldens_consistent_with_oracle(golden):
    """wide_C4 rows (reference direct solve) against the oracle restatement at 1e-12."""
    g = golden("wide_C4")
    cfg = ocfg.CONFIGS["C4"]
    grid = geometry.Grid(cfg.level)
    fo = fields.SineKLField(grid, cfg.n_z)
    obs = ocfg.observations(cfg)
    for b in (0, len(g["rows"]) - 1):
        s = ocfg.observe(grid, direct.solve(grid, fo.kappa_values(g["Z"][b])), obs)
        assert np.max(np.abs(s - g["S"][b])) <= 1e-12 * np.max(np.abs(s))


def test_lowrank_goldens_dense_rows_match_oracle(golden):
    """The dense rows of the low-rank goldens (reference HDD, compression=None) equal
    the oracle direct solve; the compressed rows lie inside the reference envelope."""
    g = golden("lowrank_L5")
    level = int(g["level"])
    grid = geometry.Grid(level)
    fo = fields.SineKLField(grid, int(g["n_z"]))
    for b in range(g["Z"].shape[0]):
        u = direct.solve(grid, fo.kappa_values(g["Z"][b]))
        s = u[g["obs_id"]]
        assert np.max(np.abs(s - g["S_dense"][b])) <= 1e-12 * np.max(np.abs(s))
        e = [np.max(np.abs(g[f"S_{k}"][b] - s)) / np.max(np.abs(s)) for k in ("e4", "c5", "e8")]
        assert e[0] > e[1] > e[2] and e[1] <= 1e-6
