"""Small forward / solve batches for compute-sanitizer (memcheck, racecheck, synccheck,
initcheck).  usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py CASE

CASE: c1 | c2 | c2_tier_l (HDD_FORCE_TIER_L=1: every merge depth on the HBM panel) |
      c3_lowrank (compress kernel) | c3_primal | tiny (level 3) | kappa (caller fields, level 5) |
      c2_solve (full-solution path) | posterior
"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
case = sys.argv[1]
if case == "c2_tier_l":
    os.environ["HDD_FORCE_TIER_L"] = "1"

import torch  # noqa: E402

import paper_1708_02207_b200 as hb  # noqa: E402
from paper_1708_02207_b200 import configs, parallel  # noqa: E402


def run(name, B, **kw):
    cfg = configs.CONFIGS[name]
    prob = configs.make_problem(name, max_batch=B, **kw)
    Z = configs.draw_Z(cfg, batch=max(B, cfg.batch))[:B]
    ll = hb.log_likelihood_batch(prob, Z)
    S = hb.forward_functionals_batch(prob, torch.from_numpy(Z).cuda())
    torch.cuda.synchronize()
    return ll, S


if case == "c1":
    ll, _ = run("C1", 4)
elif case in ("c2", "c2_tier_l"):
    ll, _ = run("C2", 2)
elif case == "c3_lowrank":
    ll, _ = run("C3", 1, compression=hb.ToleranceSpec(1e-6, 16, 32))
elif case == "c3_primal":
    ll, _ = run("C3", 1, mode=1)
elif case == "c2_solve":
    prob = configs.make_problem("C2", max_batch=2)
    U = hb.solve_batch(prob, configs.draw_Z(configs.CONFIGS["C2"], batch=2))
    ll = U[:, 0]
elif case in ("tiny", "kappa"):
    level = 3 if case == "tiny" else 5
    mesh = hb.build_mesh(level)
    tree = hb.build_tree(mesh)
    rng = np.random.default_rng(0)
    base = rng.uniform(0.1, 10.0, mesh.n_triangles)

    class P:
        n_z = 2

        def kappa(self, z):
            return base * np.exp(0.1 * z[0])

    obs = (("point", mesh.n_nodes // 2), ("mean", tree.root_id))
    param = P() if case == "kappa" else hb.SineKLField(tree, 2)
    prob = hb.BayesProblem(tree, param, rng.standard_normal(mesh.n_nodes), rng.standard_normal(4 * mesh.n_cells),
                           hb.MeasurementModel(obs, np.ones(2), np.zeros(2)))
    ll = hb.log_likelihood_batch(prob, rng.standard_normal((3, 2)))
elif case == "posterior":
    ll = torch.from_numpy(np.random.default_rng(1).normal(size=5000)).cuda()
    w, i, l = parallel.posterior_weights_device(ll)
    torch.cuda.synchronize()
    ll = w.cpu().numpy()
else:
    raise SystemExit(f"unknown case {case}")
print(case, "ok", np.asarray(ll)[:2])
