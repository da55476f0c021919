"""Wider golden coverage of the large configs and the restricted primal sweep.

* tests/golden/wide_C3.npz: 16 Z rows spread over the C3 batch through the LIVE
  reference HDD functional path (make_wide_golden.py);
* wide_C4.npz (16 rows) and wide_C5.npz (8 rows): the reference direct solve.
Rows are taken from anywhere in the BASELINE batch (including the last row), so
late sub-batches are covered.  Tolerance: relative 1e-10 (BASELINE north star).
"""
import numpy as np
import pytest

import paper_1708_02207_b200 as hb
from paper_1708_02207_b200 import configs

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("name, n_rows", [("C3", 16), ("C4", 16), ("C5", 8)])
def test_wide_goldens(cuda, golden, name, n_rows):
    g = golden(f"wide_{name}")
    assert g["Z"].shape[0] == n_rows
    # the recorded rows are the protocol's rows
    Zfull = configs.draw_Z(configs.CONFIGS[name])
    assert np.array_equal(Zfull[g["rows"]], g["Z"])
    prob = configs.make_problem(name)
    S = hb.forward_functionals_batch(prob, g["Z"])
    ll = hb.log_likelihood_batch(prob, g["Z"])
    for b in range(n_rows):
        assert rel(S[b], g["S"][b]) <= TOL, (name, int(g["rows"][b]))
    assert np.max(np.abs(ll - g["ll"]) / np.abs(g["ll"])) <= TOL


def test_wide_rows_inside_full_batches(cuda, golden):
    """The golden rows evaluated inside a large batch (sub-batched on the device) give
    the bitwise-same values as evaluated alone (batch-composition invariance)."""
    torch = cuda
    g = golden("wide_C4")
    prob = configs.make_problem("C4")
    Z = configs.draw_Z(configs.CONFIGS["C4"])[:4500]
    ll = hb.log_likelihood_batch(prob, torch.from_numpy(Z).cuda()).cpu().numpy()
    inside = g["rows"] < 4500
    alone = hb.log_likelihood_batch(prob, g["Z"][inside])
    assert np.array_equal(ll[g["rows"][inside]], alone)


def test_primal_top_down_visits_only_needed_nodes(cuda, golden):
    """north_star item 4: the primal sweep (C3: 1089 coarse points) stores factors and
    runs the top-down kernel only on the ancestors of the observation owners; a plan
    with a handful of points visits a handful of nodes and still matches the goldens."""
    g = golden("cfg_C2")
    full = configs.make_problem("C2", mode=1)
    info = full.plan().info()
    assert info.mode == 1 and 0 < info.n_topdown <= info.n_upper
    mesh = full.tree.mesh
    obs = full.model.observations[:3]
    few = hb.BayesProblem(full.tree, full.param, np.ones(mesh.n_nodes), np.zeros(4 * mesh.n_cells),
                          hb.MeasurementModel(obs, np.full(3, 0.01)), mode=1)
    fi = few.plan().info()
    assert fi.n_topdown < info.n_topdown
    S = hb.forward_functionals_batch(few, g["Z"])
    for b in range(g["Z"].shape[0]):
        assert rel(S[b], g["S"][b][:3]) <= TOL
