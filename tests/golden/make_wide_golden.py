"""Wider golden prefixes for the large configs, from the LIVE reference (build container only).

Run:  PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_wide_golden.py [C3 C4 C5]

Same protocol as make_golden.py (observations, y, Z order); records more Z rows:

* wide_C3.npz  16 rows through the reference HDD functional path
               (`bayes.forward_functionals`, hdd.py:289-394 + functionals.py:138-224);
* wide_C4.npz  16 rows through the reference `oracle.direct_solve` + `direct_mean`
               (its HDD at level 9 needs a patched MAX_LEVEL and ~136 s per sample);
* wide_C5.npz  8 rows through `oracle.direct_solve` (level 10).

Rows are spread over the batch (indices recorded in `rows`), not only the prefix, so the
device tests also cover samples from late sub-batches.  Rows run in a process pool.
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

from oracle import configs  # noqa: E402

ROWS = {
    "C3": list(range(8)) + [1000, 2047, 4096, 5000, 6143, 7000, 8000, 8191],
    "C4": list(range(8)) + [2229, 2230, 4460, 20000, 33333, 50000, 65000, 65535],
    "C5": [0, 1, 2, 543, 544, 8000, 12345, 16383],
}

_CTX = {}


def _row(args):
    name, i = args
    cfg = configs.CONFIGS[name]
    if name not in _CTX:
        _CTX[name] = mg.protocol(cfg)
    m, obs, y, sigma, z_true, Z, param = _CTX[name]
    Zs = Z[i:i + 1]
    if name == "C3":
        S, ll, _, _ = mg.ref_hdd(cfg, m, obs, y, sigma, param, Zs)
    else:
        S, ll = mg.ref_direct(cfg, m, obs, y, sigma, param, Zs)
    return i, S[0], ll[0]


def main(names):
    for name in names:
        cfg = configs.CONFIGS[name]
        t0 = time.time()
        rows = ROWS[name]
        procs = 4 if name == "C5" else 6
        with mp.get_context("fork").Pool(procs) as pool:
            res = sorted(pool.map(_row, [(name, i) for i in rows]))
        _, obs, y, sigma, z_true, Z, _ = mg.protocol(cfg)
        S = np.stack([r[1] for r in res])
        ll = np.array([r[2] for r in res])
        path = "hdd.forward_functionals" if name == "C3" else "oracle.direct_solve"
        np.savez_compressed(HERE / f"wide_{name}.npz", rows=np.array(rows, dtype=np.int64), Z=Z[rows], S=S, ll=ll,
                            y=y, sigma=sigma, path=path, level=cfg.level, n_z=cfg.n_z)
        print(name, path, S.shape, f"{time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C3", "C4", "C5"])
