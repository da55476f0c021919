"""Host logic of the device path, no GPU needed: the C ABI loads and exports
every declared symbol, the C++ plan builder reproduces the reference geometry
and observation routing, and the plan executed by the NumPy emulator
(tests/plan_emulator.py, same algebra as the kernels) matches the oracle."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1708_02207_b200 as hb
import plan_emulator as pe
from oracle import configs, direct, fields, geometry, hdd_port
from paper_1708_02207_b200 import _lib, parallel

ROOT = Path(__file__).resolve().parents[1]


def host_problem(level, n_z, obs, param="kl", sigma=0.01, y=None, f=None, mode=0, g=None):
    mesh = hb.build_mesh(level)
    tree = hb.build_tree(mesh)
    p = hb.SineKLField(tree, n_z) if param == "kl" else hb.ParamField.build(tree, n_z)
    model = hb.MeasurementModel(obs, np.full(len(obs), sigma), y)
    f = np.ones(mesh.n_nodes) if f is None else f
    g = np.zeros(4 * mesh.n_cells) if g is None else g
    return hb.BayesProblem(tree, p, f, g, model, device=-1, mode=mode)


def test_library_exports_header_symbols():
    L = _lib.lib()
    header = (ROOT / "include" / "hdd.h").read_text()
    declared = set(re.findall(r"\b(hdd_[a-z_]+)\s*\(", header))
    assert len(declared) >= 14
    for name in declared:
        assert hasattr(L, name), name
        assert name in _lib.EXPORTS, name
    assert b"sm_100a" in L.hdd_version()


def test_plan_geometry_matches_reference_tree():
    level = 6
    prob = host_problem(level, 4, (("point", 65 * 10 + 7),))
    plan = prob.plan()
    info = plan.info()
    assert info.leaf_depth == 4 and info.n_leaves == 16 and info.n_upper == 15
    nodes = {nd.id: nd for nd in geometry.full_tree(geometry.Grid(level))}
    grid = geometry.Grid(level)
    for u in range(info.n_upper):
        nd = _lib.HddNodeInfo()
        assert plan.lib.hdd_plan_node_info(plan.handle, u, C.byref(nd)) == 0
        ref = nodes[nd.ref_id]
        assert (nd.i0, nd.i1, nd.j0, nd.j1) == ref.rect and nd.depth == ref.depth
        bnd = ref.bnd[~grid.on_domain_boundary(ref.bnd)]
        assert np.array_equal(np.ctypeslib.as_array(nd.bnd, (nd.k,)), bnd) if nd.k else bnd.size == 0
        assert np.array_equal(np.ctypeslib.as_array(nd.gamma, (nd.ng,)), ref.gamma)
    for li in range(info.n_leaves):
        lf = _lib.HddLeafInfo()
        assert plan.lib.hdd_plan_leaf_info(plan.handle, li, C.byref(lf)) == 0
        ref = nodes[lf.ref_id]
        assert ref.rect == (lf.i0, lf.i0 + 16, lf.j0, lf.j0 + 16)


def test_leaf_template_shapes():
    K = [pe.leaf_template()[r][0] for r in range(8)]
    assert K == [79, 55, 39, 27, 19, 13, 9, 6]
    for r, (Kr, k, ng, m1, m2) in enumerate(pe.leaf_template()):
        assert Kr == k + ng
        covered = (m1 >= 0) | (m2 >= 0)
        assert covered.all()                       # every father index comes from a son
        assert ((m1 >= 0) & (m2 >= 0))[k:].all()   # interface shared by both sons


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("case", ["C1", "points6", "means6", "submeans6", "indicator5", "f_nodal5",
                                  "dirichlet4", "dirichlet6"])
def test_emulated_plan_matches_direct_solve(case, mode):
    rng = np.random.default_rng(5)
    f = None
    g = None
    param = "kl"
    if case == "C1":
        level, n_z = 5, 4
        obs = configs.observations(configs.CONFIGS["C1"])
    elif case == "points6":
        level, n_z = 6, 8
        obs = configs.observations(configs.Config("x", 6, 8, 4, 0.01, 1, "random64")) + (("point", 0), ("point", 64))
    elif case == "means6":
        level, n_z = 6, 8
        obs = tuple(("mean", nid) for nid, _ in geometry.nodes_at_depth(6, 2)) + \
            tuple(("mean", nid) for nid, _ in geometry.nodes_at_depth(6, 4))[:6] + \
            (("mean", geometry.nodes_at_depth(6, 0)[0][0]), ("point", 65 * 30 + 33))
    elif case == "submeans6":
        # means of nodes below the 16x16-cell kernel leaves (depths 5..12, down to one
        # cell), next to a leaf's own mean and in-leaf points, with a nodal f
        level, n_z = 6, 8
        obs = tuple(("mean", geometry.nodes_at_depth(6, d)[i][0])
                    for d, i in ((5, 3), (6, 0), (6, 57), (7, 100), (8, 31), (9, 400), (11, 1500), (12, 4095),
                                 (4, 9), (10, 1023))) + (("point", 65 * 30 + 33), ("point", 65 * 3 + 5))
        f = rng.uniform(0.5, 2.0, (65 * 65))
    elif case.startswith("dirichlet"):
        # non-zero Dirichlet data: points on and next to the domain boundary, means
        # touching it (whole domain, a boundary leaf, a sub-leaf corner node)
        level, n_z = int(case[-1]), 5
        m = 2 ** level + 1
        obs = (("point", 0), ("point", 3), ("point", m + 1), ("point", m * (m // 2) + m // 2),
               ("point", m * (m - 2) + m - 2), ("mean", geometry.nodes_at_depth(level, 0)[0][0]),
               ("mean", geometry.nodes_at_depth(level, 2 * level - 8)[0][0]),
               ("mean", geometry.nodes_at_depth(level, 2 * level)[-1][0]))
        f = rng.uniform(0.5, 2.0, m * m)
        g = rng.uniform(-1.0, 1.0, 4 * (m - 1))
    elif case == "indicator5":
        level, n_z = 5, 4
        param = "ind"
        obs = configs.observations(configs.CONFIGS["C1"])
    else:
        level, n_z = 5, 4
        obs = configs.observations(configs.CONFIGS["C1"])
        f = rng.uniform(0.5, 2.0, (33 * 33))
    prob = host_problem(level, n_z, obs, param=param, f=f, mode=mode, g=g)
    assert prob.plan().info().mode == (0 if level == 4 else mode)
    grid = geometry.Grid(level)
    fo = fields.SineKLField(grid, n_z) if param == "kl" else fields.IndicatorField(grid, n_z)
    for z in rng.standard_normal((2, n_z)):
        kap = fo.kappa_values(z)
        S, _, _ = pe.run(prob.plan(), level, kap, f)
        u = direct.solve(grid, kap, f=f, g=g)
        Sd = configs.observe(grid, u, obs)
        assert np.max(np.abs(S - Sd)) <= 1e-12 * np.max(np.abs(Sd))


def test_emulated_leaf_maps_match_reference_nodes(golden):
    """Leaf outputs (unpruned 16x16-cell Schur complements) equal the
    reference's Psi^g / Psi^f f of the same tree nodes."""
    g = golden("c1_nodes")
    Z = golden("cfg_C1")["Z"]
    cfg = configs.CONFIGS["C1"]
    prob = host_problem(cfg.level, cfg.n_z, configs.observations(cfg))
    plan = prob.plan()
    fo = fields.SineKLField(geometry.Grid(cfg.level), cfg.n_z)
    _, leaves, uppers = pe.run(plan, cfg.level, fo.kappa_values(Z[0]))
    for li, (psi, R, _) in enumerate(leaves):
        lf = _lib.HddLeafInfo()
        plan.lib.hdd_plan_leaf_info(plan.handle, li, C.byref(lf))
        ref = g[f"s0_n{lf.ref_id}_g"]
        assert np.max(np.abs(psi - ref)) <= 1e-13 * np.abs(ref).max()
        assert np.max(np.abs(R[:, 0] - g[f"s0_n{lf.ref_id}_f"])) <= 1e-13 * np.abs(R[:, 0]).max()


def test_plan_errors():
    obs = (("point", 100),)
    with pytest.raises(hb.ConfigError):
        hb.build_mesh(0)                                    # the reference accepts levels >= 1 (mesh.py:92-93)
    with pytest.raises(hb.ConfigError):
        hb.build_mesh(12)
    with pytest.raises(hb.ConfigError):
        hb.MeasurementModel(obs, np.array([0.0]))
    mesh = hb.build_mesh(5)
    tree = hb.build_tree(mesh)
    p = hb.SineKLField(tree, 4)
    with pytest.raises(hb.UsageError):
        hb.BayesProblem(tree, p, np.ones(mesh.n_nodes), np.ones(127), hb.MeasurementModel(obs, np.ones(1)))
    deep = geometry.nodes_at_depth(5, 10)[0][0]               # one cell inside a kernel leaf
    host_problem(5, 4, (("mean", deep),)).plan()
    with pytest.raises(hb.UsageError):
        host_problem(5, 4, (("mean", -1),)).plan()
    with pytest.raises(hb.UsageError):
        host_problem(5, 4, (("mean", 10 ** 9),)).plan()
    with pytest.raises(hb.UsageError):
        host_problem(5, 4, (("point", 33 * 33),)).plan()
    with pytest.raises(hb.ConfigError):
        host_problem(5, 4, (("volume", 3),)).plan()
    prob = host_problem(5, 4, obs, y=np.zeros(1))
    with pytest.raises(hb.UsageError):
        hb.log_likelihood_batch(prob, np.zeros((2, 4)))      # host-only plan cannot run
    with pytest.raises(hb.ConfigError):
        hb.forward_functionals(prob, np.zeros(3))
    with pytest.raises(hb.UsageError):
        hb.log_likelihood(host_problem(5, 4, obs), np.zeros(4))   # no data


def test_tree_ids_and_means_api():
    tree = hb.build_tree(hb.build_mesh(6))
    ref = geometry.nodes_at_depth(6, 3)
    mine = tree.nodes_at_depth(3)
    assert [n.id for n in mine] == [i for i, _ in ref]
    assert [n.cells for n in mine] == [r for _, r in ref]
    for nid, r in ref:
        assert tree.node(nid).cells == r
    assert tree.root_id == geometry.subtree_size(6, 0) - 1
    assert hb.mean_observations(tree, 3) == tuple(("mean", i) for i, _ in ref)


def test_posterior_weights_ties_and_normalisation():
    from scipy.special import logsumexp
    ll = np.array([-3.0, 1.5, -0.25, 1.5, -10.0])
    w, idx, lse = hb.posterior_weights(ll)
    assert idx == 1 == int(np.argmax(ll))
    assert abs(lse - logsumexp(ll)) <= 1e-14
    assert abs(w.sum() - 1.0) <= 1e-15
    import torch
    wt, it, lt = parallel.posterior_weights_device(torch.from_numpy(ll))
    assert int(it) == 1 and np.allclose(wt.numpy(), w, rtol=1e-15)


def test_shard_rows():
    for n in [1, 7, 64, 1000]:
        for world in [1, 2, 3, 8]:
            spans = [parallel.shard_rows(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _gloo_worker(rank, world, port, out_path):
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = configs.CONFIGS["C1"]
    obs = configs.observations(cfg)
    port_ = hdd_port.HDDPort(cfg.level, obs)
    fo = fields.SineKLField(geometry.Grid(cfg.level), cfg.n_z)
    y, sigma = hb.configs.observed_data(cfg)

    def forward(problem, Zb):
        return np.array([hdd_port.gaussian_ll(y, port_.forward(fo.kappa_values(z)), sigma) for z in Zb])

    Z = hb.configs.draw_Z(cfg)[:11]
    ll, w, idx, lse = parallel.sharded_log_likelihood(None, Z, forward=forward)
    if rank == 0:
        np.savez(out_path, ll=ll.numpy(), w=w.numpy(), idx=idx, lse=lse)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_likelihood_gloo_world2(tmp_path, golden):
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = tmp_path / "r.npz"
    mp.spawn(_gloo_worker, args=(2, port, str(out)), nprocs=2, join=True)
    r = np.load(out)
    g = golden("cfg_C1")
    assert np.allclose(r["ll"], g["ll"][:11], rtol=1e-12)
    w, idx, lse = hb.posterior_weights(g["ll"][:11])
    assert int(r["idx"]) == idx and np.allclose(r["w"], w, rtol=1e-12)


def test_primal_routing_auto_selection():
    """Auto mode: many point observations -> primal top-down (routes 2/3),
    few -> adjoint (root columns), means stay adjoint."""
    cfg = configs.CONFIGS["C3"]
    p2 = host_problem(cfg.level, cfg.n_z, configs.observations(cfg), mode=-1).plan()
    assert p2.info().mode == 1
    kinds = []
    for o in range(p2.info().n_obs):
        ob = _lib.HddObsInfo()
        p2.lib.hdd_plan_obs_info(p2.handle, o, C.byref(ob))
        kinds.append(ob.kind)
    assert set(kinds) <= {1, 2, 3} and 2 in kinds and 3 in kinds
    for name in ("C1", "C2"):
        c1 = configs.CONFIGS[name]
        p1 = host_problem(c1.level, c1.n_z, configs.observations(c1), mode=-1).plan()
        assert p1.info().mode == 0


@pytest.mark.parametrize("level", [4, 5])
def test_dump_tree_matches_reference_format(level):
    """geometry.dump_tree reproduces the reference's regression dump line for line."""
    from pathlib import Path
    from paper_1708_02207_b200.geometry import dump_tree
    ref = (Path(__file__).resolve().parent / "golden" / f"dump_tree_L{level}.txt").read_text()
    assert dump_tree(hb.build_tree(hb.build_mesh(level))) == ref
