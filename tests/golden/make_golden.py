"""Generate the golden fixtures from the LIVE reference (build container only).

Run:  PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden.py

It imports the unmodified reference package `hddsolve` from
/root/reference/pkg/src and records, for the BASELINE protocol
(oracle/configs.py):

* cfg_<C>.npz      observations, y (reference direct_solve truth + noise),
                   sigma, z_true, a prefix of the Z batch, and reference
                   S / ll for that prefix (HDD functional path
                   `bayes.log_likelihood` for C1-C3, `oracle.direct_solve` +
                   `observe_solution` for C4/C5 where the reference HDD needs a
                   patched MAX_LEVEL and hours);
* c1_nodes.npz     per-node Psi^g and Psi^f f of the C1 tree (BuildDiagnostics
                   keep_psi) at the 16x16 leaves, depth 1 and the root;
* c1_indicator.npz S / ll with the reference's own indicator ParamField;
* fem_known.npz    the reference tests' known FEM answers (cell patterns).

The GPU box never sees /root/reference: tests read only these fixtures.
"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parents[1]))

import hddsolve as hs  # noqa: E402
from hddsolve import bayes, hdd, mesh as hmesh, oracle as horacle  # noqa: E402

from oracle import configs, fields, geometry  # noqa: E402

hmesh.MAX_LEVEL = 10   # module global read at call time


class KLParam:
    """Duck-typed `problem.param` (bayes.py:183) for the BASELINE sine-KL field."""

    def __init__(self, level, n_z):
        self.f = fields.SineKLField(geometry.Grid(level), n_z)
        self.n_z = n_z

    def kappa(self, z):
        return hs.CoefficientField(self.f.kappa_values(z))


def protocol(cfg):
    obs = configs.observations(cfg)
    m = hs.build_mesh(cfg.level)
    z_true, eps, Z = configs.draw(cfg)
    param = KLParam(cfg.level, cfg.n_z)
    u = horacle.direct_solve(m, param.kappa(z_true), np.ones(m.n_nodes), np.zeros(4 * (m.m - 1)))
    clean = np.empty(len(obs))
    for k, (kind, ident) in enumerate(obs):
        if kind == "point":
            clean[k] = u[ident]
        else:
            rect, _ = geometry.rect_of_node_id(cfg.level, ident)
            h = m.h
            clean[k] = horacle.direct_mean(m, u, hs.Rect(rect[0] * h, rect[1] * h, rect[2] * h, rect[3] * h))
    y = clean + eps
    sigma = np.full(len(obs), cfg.sigma)
    return m, obs, y, sigma, z_true, Z, param


def ref_hdd(cfg, m, obs, y, sigma, param, Zs):
    tree = hs.build_tree(m)
    model = bayes.MeasurementModel(obs, sigma, y)
    prob = bayes.BayesProblem(tree, param, np.ones(m.n_nodes), np.zeros(4 * (m.m - 1)), model)
    S = np.stack([bayes.forward_functionals(prob, z) for z in Zs])
    ll = np.array([bayes.gaussian_log_likelihood(y, s, sigma) for s in S])
    return S, ll, tree, prob


def ref_direct(cfg, m, obs, y, sigma, param, Zs):
    S = []
    for z in Zs:
        u = horacle.direct_solve(m, param.kappa(z), np.ones(m.n_nodes), np.zeros(4 * (m.m - 1)))
        row = []
        for kind, ident in obs:
            if kind == "point":
                row.append(u[ident])
            else:
                rect, _ = geometry.rect_of_node_id(cfg.level, ident)
                h = m.h
                row.append(horacle.direct_mean(m, u, hs.Rect(rect[0] * h, rect[1] * h, rect[2] * h, rect[3] * h)))
        S.append(row)
    S = np.array(S)
    ll = np.array([bayes.gaussian_log_likelihood(y, s, sigma) for s in S])
    return S, ll


def main():
    n_prefix = {"C1": 64, "C2": 8, "C3": 2, "C4": 2, "C5": 1}
    for name in ["C1", "C2", "C3", "C4", "C5"]:
        cfg = configs.CONFIGS[name]
        t0 = time.time()
        m, obs, y, sigma, z_true, Z, param = protocol(cfg)
        Zs = Z[: n_prefix[name]]
        if name in ("C1", "C2", "C3"):
            S, ll, tree, prob = ref_hdd(cfg, m, obs, y, sigma, param, Zs)
            path = "hdd.forward_functionals"
        else:
            S, ll = ref_direct(cfg, m, obs, y, sigma, param, Zs)
            path = "oracle.direct_solve"
        kinds = np.array([0 if k == "point" else 1 for k, _ in obs], dtype=np.int32)
        ids = np.array([i for _, i in obs], dtype=np.int64)
        np.savez_compressed(HERE / f"cfg_{name}.npz", obs_kind=kinds, obs_id=ids, y=y, sigma=sigma,
                            z_true=z_true, Z=Zs, S=S, ll=ll, path=path, level=cfg.level, n_z=cfg.n_z)
        print(name, path, S.shape, f"{time.time() - t0:.1f}s", flush=True)
        if name == "C1":
            # per-node maps for two samples
            diag_rec = {}
            for si in range(2):
                diag = hdd.BuildDiagnostics(keep_psi=True)
                store = hdd.leaves_to_root(tree, param.kappa(Zs[si]), hdd.SolveMode.functionals_only(),
                                           diagnostics=diag)
                for nd in tree.nodes:
                    if nd.depth <= 2:
                        ps = store.psi[nd.id]
                        fo = np.ones(nd.idx_omega.size)
                        diag_rec[f"s{si}_n{nd.id}_g"] = np.asarray(ps.psi_g)
                        diag_rec[f"s{si}_n{nd.id}_f"] = np.asarray(ps.psi_f) @ fo
                        diag_rec[f"n{nd.id}_bnd"] = nd.idx_boundary
            np.savez_compressed(HERE / "c1_nodes.npz", **diag_rec)
            # the reference's own indicator parametrization
            pf = bayes.ParamField.build(tree, 4)
            model = bayes.MeasurementModel(obs, sigma, y)
            prob_i = bayes.BayesProblem(tree, pf, np.ones(m.n_nodes), np.zeros(4 * (m.m - 1)), model)
            Zi = Zs[:8]
            Si = np.stack([bayes.forward_functionals(prob_i, z) for z in Zi])
            lli = np.array([bayes.log_likelihood(prob_i, z) for z in Zi])
            np.savez_compressed(HERE / "c1_indicator.npz", Z=Zi, S=Si, ll=lli,
                                kappa0=pf.kappa(Zi[0]).values)
            # kappa of the sine-KL field (from_callable-equivalent centroids)
            np.savez_compressed(HERE / "c1_kappa.npz", Z=Zs[:4],
                                kappa=np.stack([param.kappa(z).values for z in Zs[:4]]))
    # reference FEM known answers (test_fem.py:12-16, :161-171)
    from hddsolve.fem import cell_patterns, local_stiffness
    h = 0.125
    p1, p2, load = cell_patterns(h)
    rt = local_stiffness([(0.0, 0.0), (0.25, 0.0), (0.0, 0.25)], 1.0)
    np.savez_compressed(HERE / "fem_known.npz", p1=p1, p2=p2, load=load, h=h, right_triangle=rt)
    print("done")


if __name__ == "__main__":
    main()
