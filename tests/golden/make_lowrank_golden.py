"""Low-rank (H-matrix) goldens from the LIVE reference's compressed path (build container only).

Run:  PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_lowrank_golden.py [levels]

For mesh levels 5-8 and the C5-style protocol scaled to the level (n_z = 32, 256 seeded
random interior points, sigma 0.005, f = 1, g = 0, y = reference direct solve at z_true +
noise), it runs the unmodified reference `bayes.forward_functionals` (hdd.py:289-394 with
`compression=ToleranceSpec(...)`, i.e. `_maybe_compress` hdd.py:280-286 on all four maps
Psi^g, Psi^f, Phi^g, Phi^f with the exact-SVD truncation lowrank.py:52-77) for:

* dense (compression=None),
* ToleranceSpec(1e-6, 16, 32)  — the BASELINE C5 spec,
* ToleranceSpec()              — the reference default (1e-6, 64, 32),
* ToleranceSpec(1e-4, 16, 32) and ToleranceSpec(1e-8, 16, 32) — the error envelope,
* ToleranceSpec(1e-13, 24 | 64, 32) — ranks above 24 (the device's wide-sketch path).

and records S and ll per (spec, row) in lowrank_L<level>.npz together with Z, y, sigma and
the observations.  The device tests compare the device low-rank path against these.
"""
from __future__ import annotations

import multiprocessing as mp
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
import make_golden as mg  # noqa: E402  (imports the live reference, patches MAX_LEVEL)

import hddsolve as hs  # noqa: E402
from hddsolve import bayes, lowrank  # noqa: E402

from oracle import configs  # noqa: E402

SPECS = {
    "dense": None,
    "c5": (1e-6, 16, 32),
    "default": (1e-6, 64, 32),
    "e4": (1e-4, 16, 32),
    "e8": (1e-8, 16, 32),
    "e13k24": (1e-13, 24, 32),   # eps near the 1e-14 floor: ranks above 24 appear
    "e13k64": (1e-13, 64, 32),   # ... and the device wide (72-column) sketch is needed
}
N_ROWS = 3


def cfg_for(level):
    return configs.Config(f"LR{level}", level, 32, 2 * (level - 5), 0.005, N_ROWS, "random256")


_CTX = {}


def _ctx(level):
    if level not in _CTX:
        cfg = cfg_for(level)
        m, obs, y, sigma, z_true, Z, param = mg.protocol(cfg)
        tree = hs.build_tree(m)
        _CTX[level] = (cfg, m, obs, y, sigma, Z, param, tree)
    return _CTX[level]


def _run(args):
    level, spec_name, i = args
    cfg, m, obs, y, sigma, Z, param, tree = _ctx(level)
    spec = SPECS[spec_name]
    comp = None if spec is None else lowrank.ToleranceSpec(*spec)
    model = bayes.MeasurementModel(obs, sigma, y)
    prob = bayes.BayesProblem(tree, param, np.ones(m.n_nodes), np.zeros(4 * (m.m - 1)), model, compression=comp)
    t0 = time.time()
    s = bayes.forward_functionals(prob, Z[i])
    return spec_name, i, s, bayes.gaussian_log_likelihood(y, s, sigma), time.time() - t0


def main(levels):
    for level in levels:
        t0 = time.time()
        cfg, m, obs, y, sigma, Z, param, tree = _ctx(level)
        jobs = [(level, sn, i) for sn in SPECS for i in range(N_ROWS)]
        with mp.get_context("fork").Pool(6) as pool:
            res = pool.map(_run, jobs)
        out = dict(Z=Z[:N_ROWS], y=y, sigma=sigma, level=level, n_z=cfg.n_z,
                   obs_id=np.array([i for _, i in obs], dtype=np.int64))
        for sn, spec in SPECS.items():
            rows = sorted((r for r in res if r[0] == sn), key=lambda r: r[1])
            out[f"S_{sn}"] = np.stack([r[2] for r in rows])
            out[f"ll_{sn}"] = np.array([r[3] for r in rows])
            out[f"sec_{sn}"] = np.array([r[4] for r in rows])
            if spec is not None:
                out[f"spec_{sn}"] = np.array(spec, dtype=float)
        np.savez_compressed(HERE / f"lowrank_L{level}.npz", **out)
        d = out["S_dense"]
        msg = " ".join(f"{sn} {np.max(np.abs(out[f'S_{sn}'] - d)) / np.max(np.abs(d)):.2e}" for sn in SPECS
                       if sn != "dense")
        print(f"L{level}: {msg} ({time.time() - t0:.0f}s)", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [5, 6, 7, 8])
