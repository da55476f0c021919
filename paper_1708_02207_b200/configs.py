"""The five BASELINE configurations as ready-to-run BayesProblems.

Observation sets and the Z draw order follow the protocol documented in
DESIGN.md; the observed data y (truth from the
reference's direct solver at z_true plus seeded noise) was produced in the
build container by tests/golden/make_golden.py and ships as
data/protocol.npz — synthetic measurement data, not a computation of the
forward map.
"""
from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .bayes import BayesProblem, MeasurementModel, SineKLField, mean_observations
from .geometry import build_mesh, build_tree, interior_nodes, Rect

SEED = 170802207
DATA = Path(__file__).resolve().parent / "data" / "protocol.npz"


@dataclass(frozen=True)
class Config:
    name: str
    level: int
    n_z: int
    depth: int            # BASELINE truncation depth (32x32-cell leaves; 16x16 for C1)
    sigma: float
    batch: int
    obs_kind: str
    compression: tuple | None = None


CONFIGS = {
    "C1": Config("C1", 5, 4, 2, 0.01, 64, "lattice"),
    "C2": Config("C2", 7, 8, 4, 0.01, 1024, "random64"),
    "C3": Config("C3", 8, 20, 6, 0.005, 8192, "coarse8"),
    "C4": Config("C4", 9, 32, 8, 0.005, 65536, "means4"),
    "C5": Config("C5", 10, 32, 10, 0.005, 16384, "random256", (1e-6, 16, 32)),
}


def observations(cfg: Config, seed: int = SEED):
    mesh = build_mesh(cfg.level)
    m = mesh.m
    if cfg.obs_kind == "lattice":
        lat = [4, 12, 20, 28]
        return tuple(("point", j * m + i) for j in lat for i in lat)
    if cfg.obs_kind.startswith("random"):
        n = int(cfg.obs_kind[len("random"):])
        inner = interior_nodes(mesh, Rect(0.0, 1.0, 0.0, 1.0))
        pick = np.sort(np.random.default_rng(seed + 1).choice(inner, n, replace=False))
        return tuple(("point", int(p)) for p in pick)
    if cfg.obs_kind == "coarse8":
        c = list(range(0, mesh.n_cells + 1, 8))
        return tuple(("point", j * m + i) for j in c for i in c)
    if cfg.obs_kind == "means4":
        return mean_observations(build_tree(mesh), 4)
    raise ValueError(cfg.obs_kind)


def draw_Z(cfg: Config, batch: int | None = None, seed: int = SEED) -> np.ndarray:
    """Z[B, n_z] in the protocol's draw order (z_true, noise, then Prior.sample
    columns, bayes.py:113-120)."""
    rng = np.random.default_rng(seed)
    n_y = len(observations(cfg, seed))
    rng.standard_normal(cfg.n_z)
    rng.normal(0.0, cfg.sigma, n_y)
    B = cfg.batch if batch is None else batch
    return np.stack([rng.standard_normal(B) for _ in range(cfg.n_z)], axis=-1)


def observed_data(cfg: Config):
    """(y, sigma) of the synthetic experiment."""
    with np.load(DATA) as d:
        y = d[f"{cfg.name}_y"]
        sigma = d[f"{cfg.name}_sigma"]
    return y, sigma


def make_problem(name: str, device: int = 0, max_batch: int = 0, with_data: bool = True,
                 mode: int = -1, compression=False) -> BayesProblem:
    """`compression=True` applies the config's ToleranceSpec (C5: eps 1e-6,
    k_max 16, n_min 32); a ToleranceSpec instance is used as given."""
    cfg = CONFIGS[name]
    mesh = build_mesh(cfg.level)
    tree = build_tree(mesh)
    obs = observations(cfg)
    if with_data:
        y, sigma = observed_data(cfg)
    else:
        y, sigma = None, np.full(len(obs), cfg.sigma)
    model = MeasurementModel(obs, sigma, y)
    tol = None
    if compression is True and cfg.compression is not None:
        from .bayes import ToleranceSpec
        tol = ToleranceSpec(*cfg.compression)
    elif compression not in (None, False, True):
        tol = compression
    return BayesProblem(tree, SineKLField(tree, cfg.n_z), np.ones(mesh.n_nodes), np.zeros(4 * mesh.n_cells),
                        model, compression=tol, device=device, max_batch=max_batch, mode=mode)
