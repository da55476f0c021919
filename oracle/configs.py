"""BASELINE configurations C1-C5 and the seeded observation/draw protocol.

The reference fixes neither the observation sets nor the seeds (SURVEY.md
D5, D7); this module is the builder's documented protocol (SURVEY.md
Appendix A), shared by the golden generator, the tests and the CPU baseline:

* C1 lattice: i, j in {4, 12, 20, 28}, node j*m + i, j outer;
* C2 / C5: np.sort(default_rng(seed + 1).choice(interior nodes, n, replace=False));
* C3 coarse grid: i, j in {0, 8, ..., 256}, j outer (128 of them on the
  domain boundary, value 0);
* C4: ("mean", id) for the 16 depth-4 tree nodes in post-order id order
  (bayes.py:150-152 `mean_observations`);
* draws: rng = default_rng(seed); z_true = rng.standard_normal(n_z);
  eps = rng.normal(0, sigma, n_y); Z = stack([rng.standard_normal(B) for k]),
  i.e. `Prior.sample` column order (bayes.py:113-120);
* y = observe(direct solve(kappa(z_true)), f = 1, g = 0) + eps.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import direct
from .fields import SineKLField
from .geometry import Grid, nodes_at_depth, rect_of_node_id

SEED = 170802207


@dataclass(frozen=True)
class Config:
    name: str
    level: int
    n_z: int
    depth: int            # BASELINE truncation depth (32x32-cell leaves; 16x16 for C1)
    sigma: float
    batch: int
    obs_kind: str
    compression: tuple | None = None   # (eps, k_max, n_min)


CONFIGS = {
    "C1": Config("C1", 5, 4, 2, 0.01, 64, "lattice"),
    "C2": Config("C2", 7, 8, 4, 0.01, 1024, "random64"),
    "C3": Config("C3", 8, 20, 6, 0.005, 8192, "coarse8"),
    "C4": Config("C4", 9, 32, 8, 0.005, 65536, "means4"),
    "C5": Config("C5", 10, 32, 10, 0.005, 16384, "random256", (1e-6, 16, 32)),
}


def observations(cfg: Config, seed: int = SEED):
    grid = Grid(cfg.level)
    m = grid.m
    if cfg.obs_kind == "lattice":
        lat = [4, 12, 20, 28]
        return tuple(("point", j * m + i) for j in lat for i in lat)
    if cfg.obs_kind.startswith("random"):
        n = int(cfg.obs_kind[len("random"):])
        inner = np.sort(grid.interior_ids((0, grid.N, 0, grid.N)))
        pick = np.sort(np.random.default_rng(seed + 1).choice(inner, n, replace=False))
        return tuple(("point", int(p)) for p in pick)
    if cfg.obs_kind == "coarse8":
        c = list(range(0, grid.N + 1, 8))
        return tuple(("point", j * m + i) for j in c for i in c)
    if cfg.obs_kind == "means4":
        return tuple(("mean", nid) for nid, _ in nodes_at_depth(cfg.level, 4))
    raise ValueError(cfg.obs_kind)


def observe(grid: Grid, u: np.ndarray, obs) -> np.ndarray:
    """Observation operator on an assembled solution (bayes.py:211-219)."""
    out = np.empty(len(obs))
    for k, (kind, ident) in enumerate(obs):
        if kind == "point":
            out[k] = u[ident]
        else:
            rect, _ = rect_of_node_id(grid.level, ident)
            out[k] = direct.region_mean(grid, u, rect)
    return out


def draw(cfg: Config, seed: int = SEED, batch: int | None = None):
    """(z_true, eps, Z) in the protocol's draw order."""
    rng = np.random.default_rng(seed)
    n_y = len(observations(cfg, seed))
    z_true = rng.standard_normal(cfg.n_z)
    eps = rng.normal(0.0, cfg.sigma, n_y)
    B = cfg.batch if batch is None else batch
    Z = np.stack([rng.standard_normal(B) for _ in range(cfg.n_z)], axis=-1)
    return z_true, eps, Z


def synthesize(cfg: Config, seed: int = SEED):
    """Observed data y from the direct solver at z_true plus noise."""
    grid = Grid(cfg.level)
    obs = observations(cfg, seed)
    z_true, eps, _ = draw(cfg, seed, batch=1)
    field = SineKLField(grid, cfg.n_z)
    u = direct.solve(grid, field.kappa_values(z_true))
    clean = observe(grid, u, obs)
    return obs, clean + eps, np.full(len(obs), cfg.sigma), z_true
