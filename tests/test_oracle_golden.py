"""Pin the CPU oracle against the golden vectors recorded from the live reference
(tests/golden/make_golden.py) and the reference tests' known FEM answers."""
import numpy as np
import pytest

from oracle import configs, direct, fields, geometry, hdd_port


def test_known_fem_answers(golden):
    g = golden("fem_known")
    P1, P2, load = hdd_port.cell_stencils(float(g["h"]))
    assert np.array_equal(P1, g["p1"]) and np.array_equal(P2, g["p2"])
    assert np.allclose(load, g["load"], rtol=0, atol=1e-18)
    # frozen right-triangle stiffness of the reference tests (test_fem.py:12-16)
    rt = direct.element_stiffness([(0.0, 0.0), (0.25, 0.0), (0.0, 0.25)], 1.0)
    assert np.allclose(rt, 0.5 * np.array([[2, -1, -1], [-1, 1, 0], [-1, 0, 1.0]]), atol=1e-15)
    assert np.allclose(rt, g["right_triangle"], atol=1e-15)
    # load diag h^2/6 [2,1,1,2] (test_fem.py:161-171)
    assert np.allclose(load, g["h"] ** 2 / 6 * np.array([2, 1, 1, 2]))


def test_affine_exactness_direct():
    """direct solve reproduces u = x1 exactly (test_fem.py:144-149)."""
    grid = geometry.Grid(3)
    xy = grid.coords()
    bnd = grid.perimeter_ids((0, grid.N, 0, grid.N))
    u = direct.solve(grid, np.ones(grid.n_triangles), f=np.zeros(grid.n_nodes), g=xy[bnd, 0])
    assert np.max(np.abs(u - xy[:, 0])) <= 1e-12


def test_protocol_matches_golden(golden):
    for name in ["C1", "C2", "C3", "C4", "C5"]:
        g = golden(f"cfg_{name}")
        cfg = configs.CONFIGS[name]
        obs = configs.observations(cfg)
        assert [0 if k == "point" else 1 for k, _ in obs] == g["obs_kind"].tolist()
        assert [i for _, i in obs] == g["obs_id"].tolist()
        z_true, _, Z = configs.draw(cfg)
        assert np.array_equal(z_true, g["z_true"])
        assert np.array_equal(Z[: g["Z"].shape[0]], g["Z"])


def test_port_matches_reference_c1(golden):
    g = golden("cfg_C1")
    cfg = configs.CONFIGS["C1"]
    obs = configs.observations(cfg)
    port = hdd_port.HDDPort(cfg.level, obs)
    fo = fields.SineKLField(geometry.Grid(cfg.level), cfg.n_z)
    for b in range(0, 64, 7):
        s = port.forward(fo.kappa_values(g["Z"][b]))
        assert np.max(np.abs(s - g["S"][b])) <= 1e-13 * np.max(np.abs(g["S"][b]))
        ll = hdd_port.gaussian_ll(g["y"], s, g["sigma"])
        assert abs(ll - g["ll"][b]) <= 1e-12 * abs(g["ll"][b])


def test_port_per_node_maps_match_reference(golden):
    """Psi^g and Psi^f f of every node at depth <= 2 (BuildDiagnostics keep_psi)."""
    g = golden("c1_nodes")
    cfg = configs.CONFIGS["C1"]
    port = hdd_port.HDDPort(cfg.level, configs.observations(cfg))
    fo = fields.SineKLField(geometry.Grid(cfg.level), cfg.n_z)
    Z = golden("cfg_C1")["Z"]
    for si in range(2):
        keep = {}
        port.forward(fo.kappa_values(Z[si]), keep_psi=keep)
        n = 0
        for key in g:
            if key.startswith(f"s{si}_n") and key.endswith("_g"):
                nid = int(key.split("_n")[1].split("_")[0])
                pg, pf = keep[nid]
                assert np.allclose(pg, g[key], rtol=0, atol=1e-13 * np.abs(g[key]).max())
                assert np.allclose(pf, g[f"s{si}_n{nid}_f"], rtol=0, atol=1e-13 * np.abs(pf).max())
                assert np.array_equal(port.nodes[nid].bnd, g[f"n{nid}_bnd"])
                n += 1
        assert n == 7   # root, 2 depth-1 nodes, 4 leaves (16x16 cells)


def test_indicator_field_matches_reference(golden):
    g = golden("c1_indicator")
    cfg = configs.CONFIGS["C1"]
    grid = geometry.Grid(cfg.level)
    fi = fields.IndicatorField(grid, 4)
    assert np.array_equal(fi.kappa_values(g["Z"][0]), g["kappa0"])
    port = hdd_port.HDDPort(cfg.level, configs.observations(cfg))
    y, sigma = golden("cfg_C1")["y"], golden("cfg_C1")["sigma"]
    for b in range(g["Z"].shape[0]):
        s = port.forward(fi.kappa_values(g["Z"][b]))
        assert np.max(np.abs(s - g["S"][b])) <= 1e-13 * np.max(np.abs(g["S"][b]))
        assert abs(hdd_port.gaussian_ll(y, s, sigma) - g["ll"][b]) <= 1e-12 * abs(g["ll"][b])


@pytest.mark.slow
def test_port_matches_reference_c2(golden):
    g = golden("cfg_C2")
    cfg = configs.CONFIGS["C2"]
    port = hdd_port.HDDPort(cfg.level, configs.observations(cfg))
    fo = fields.SineKLField(geometry.Grid(cfg.level), cfg.n_z)
    s = port.forward(fo.kappa_values(g["Z"][0]))
    assert np.max(np.abs(s - g["S"][0])) <= 1e-12 * np.max(np.abs(g["S"][0]))


def test_direct_matches_reference_c3(golden):
    """Oracle direct solve vs the reference HDD at C3 (257^2 nodes)."""
    g = golden("cfg_C3")
    cfg = configs.CONFIGS["C3"]
    grid = geometry.Grid(cfg.level)
    fo = fields.SineKLField(grid, cfg.n_z)
    obs = configs.observations(cfg)
    u = direct.solve(grid, fo.kappa_values(g["Z"][0]))
    s = configs.observe(grid, u, obs)
    assert np.max(np.abs(s - g["S"][0])) <= 1e-10 * np.max(np.abs(g["S"][0]))
