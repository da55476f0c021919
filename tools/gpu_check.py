"""Quick GPU diagnostics: device path vs the plan emulator and the direct solve,
node by node when they disagree, then a timing of the C2 batch."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import plan_emulator as pe  # noqa: E402
import paper_1708_02207_b200 as hb  # noqa: E402
from paper_1708_02207_b200 import _lib  # noqa: E402
from paper_1708_02207_b200.bayes import _Plan  # noqa: E402
from oracle import configs, direct, fields, geometry  # noqa: E402


def problem(cfg, keep=False, device=0):
    obs = configs.observations(cfg)
    mesh = hb.build_mesh(cfg.level)
    tree = hb.build_tree(mesh)
    param = hb.SineKLField(tree, cfg.n_z)
    model = hb.MeasurementModel(obs, np.full(len(obs), cfg.sigma), np.zeros(len(obs)))
    prob = hb.BayesProblem(tree, param, np.ones(mesh.n_nodes), np.zeros(4 * mesh.n_cells), model,
                           device=device)
    if keep:
        prob._plan = _Plan(prob, device, 8, keep_nodes=True)
    return prob, obs


def check(name, nsamp=3):
    cfg = configs.CONFIGS[name]
    prob, obs = problem(cfg, keep=True)
    host, _ = problem(cfg, device=-1)
    hplan = host.plan()
    g = geometry.Grid(cfg.level)
    fo = fields.SineKLField(g, cfg.n_z)
    _, _, Z = configs.draw(cfg)
    Z = Z[:nsamp]
    S = hb.forward_functionals_batch(prob, Z)
    plan = prob.plan()
    L = plan.lib
    for b in range(nsamp):
        kap = fo.kappa_values(Z[b])
        Se, leaves, uppers = pe.run(hplan, cfg.level, kap)
        u = direct.solve(g, kap)
        Sd = configs.observe(g, u, obs)
        err_e = np.max(np.abs(S[b] - Se)) / np.max(np.abs(Se))
        err_d = np.max(np.abs(S[b] - Sd)) / np.max(np.abs(Sd))
        print(f"{name} sample {b}: rel err vs emulator {err_e:.3e}  vs direct {err_d:.3e}", flush=True)
        if err_e > 1e-10 and b == 0:
            for li in range(min(4, len(leaves))):
                psi = np.empty((64, 64))
                nc = leaves[li][1].shape[1]
                R = np.empty((64, nc))
                sg = np.empty(nc)
                rc = L.hdd_debug_node_output(plan.handle, -1 - li, b, psi.ctypes.data_as(_lib._f64p),
                                             R.ctypes.data_as(_lib._f64p), sg.ctypes.data_as(_lib._f64p))
                assert rc == 0, rc
                print(f"  leaf {li}: psi {np.max(np.abs(psi - leaves[li][0])):.3e} R {np.max(np.abs(R - leaves[li][1])):.3e}"
                      f" sig {np.max(np.abs(sg - leaves[li][2])) if nc else 0:.3e}")
            for u, (psi_e, R_e, s_e) in list(uppers.items())[:8]:
                nd = _lib.HddNodeInfo()
                L.hdd_plan_node_info(plan.handle, u, C.byref(nd))
                psi = np.empty((nd.k, nd.k))
                R = np.empty((nd.k, nd.nc))
                sg = np.empty(nd.nc)
                L.hdd_debug_node_output(plan.handle, u, b, psi.ctypes.data_as(_lib._f64p),
                                        R.ctypes.data_as(_lib._f64p), sg.ctypes.data_as(_lib._f64p))
                print(f"  upper {u} depth {nd.depth} k {nd.k} ng {nd.ng} nc {nd.nc}: psi "
                      f"{np.max(np.abs(psi - psi_e)) if nd.k else 0:.3e} R {np.max(np.abs(R - R_e)) if nd.k else 0:.3e}"
                      f" sig {np.max(np.abs(sg - s_e)):.3e}")


def timing(name, reps=5):
    import torch
    cfg = configs.CONFIGS[name]
    prob, obs = problem(cfg)
    _, _, Z = configs.draw(cfg)
    Zd = torch.from_numpy(Z).cuda()
    hb.forward_functionals_batch(prob, Zd)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record()
        hb.forward_functionals_batch(prob, Zd)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    info = prob.plan().info()
    print(f"{name}: B={Z.shape[0]} best {best:.3f} ms -> {Z.shape[0] / best * 1e3:.1f} samples/s "
          f"(bcap {info.max_batch})", flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["C1", "C2"]
    for n in which:
        check(n)
    for n in which:
        timing(n)
