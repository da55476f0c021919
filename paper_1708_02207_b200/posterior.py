"""Posterior drivers on the batched device likelihood.

Restates the reference's `posterior_grid` / `posterior_mcmc`
(/root/reference/pkg/src/hddsolve/bayes.py:251-377) with every likelihood
evaluation routed through `log_likelihood_batch`:

* `posterior_grid` evaluates all tensor-grid points in ONE device batch instead
  of the reference's per-point loop (bayes.py:326); quadrature, normalisation,
  evidence and mode follow bayes.py:318-333 exactly;
* `posterior_mcmc` is the reference random-walk Metropolis chain, step for step
  (same RNG stream, same accept rule, same bookkeeping), one device call per step;
* `posterior_mcmc_chains` runs C independent chains (chain c seeded chain.seed + c)
  in lockstep with one device batch of C proposals per step — chain c reproduces
  `posterior_mcmc` with ChainSpec(seed=chain.seed + c).
"""
from __future__ import annotations

import math
import warnings
from dataclasses import dataclass

import numpy as np

from .bayes import BayesProblem, Prior, log_likelihood_batch
from .errors import ConfigError, UsageError


@dataclass(frozen=True)
class GridSpec:
    lo: tuple
    hi: tuple
    n: tuple

    def axes(self):
        return [np.linspace(l, h, k) for l, h, k in zip(self.lo, self.hi, self.n)]


@dataclass(frozen=True)
class ChainSpec:
    length: int = 4000
    burn: int = 1000
    proposal: float = 0.15
    seed: int = 0


@dataclass
class PosteriorResult:
    points: np.ndarray            # (N, n_z) grid points or chain samples
    log_prior: np.ndarray
    log_like: np.ndarray
    log_post: np.ndarray          # normalized on grids, unnormalized for chains
    log_evidence: float | None = None
    mode: np.ndarray | None = None
    weights: np.ndarray | None = None
    acceptance: float | None = None
    accepted: np.ndarray | None = None

    @property
    def integral(self):
        if self.weights is None:
            return None
        return float(np.sum(np.exp(self.log_post) * self.weights))

    def posterior_mean(self):
        return self.points.mean(axis=0)

    def posterior_std(self):
        return self.points.std(axis=0)


def _trapezoid_weights(axis):
    w = np.full(axis.size, axis[1] - axis[0]) if axis.size > 1 else np.ones(1)
    if axis.size > 1:
        w[0] *= 0.5
        w[-1] *= 0.5
    return w


def logsumexp_weighted(a, b=None) -> float:
    """log(sum(b * exp(a))), the scipy.special.logsumexp(a, b=b) value used by
    bayes.py:328 (shifted by max(a); b >= 0)."""
    a = np.asarray(a, dtype=float)
    b = np.ones_like(a) if b is None else np.asarray(b, dtype=float)
    mask = b != 0
    if not mask.any():
        return -math.inf
    amax = float(np.max(a[mask]))
    if not np.isfinite(amax):
        return amax
    return amax + math.log(float(np.sum(b * np.exp(a - amax))))


def posterior_grid(problem: BayesProblem, prior: Prior, grid: GridSpec,
                   log_like_batch=log_likelihood_batch) -> PosteriorResult:
    """Tensor-grid posterior for one or two parameters (bayes.py:305-333); the
    evidence is a trapezoidal quadrature in log space and the returned log
    density is normalized so the same quadrature integrates it to one."""
    n_z = prior.n_z
    if n_z > 2:
        raise UsageError("grid posteriors support at most two parameters")
    if len(grid.lo) != n_z or len(grid.hi) != n_z or len(grid.n) != n_z:
        raise ConfigError("grid spec dimensions do not match the prior")
    axes = grid.axes()
    if n_z == 1:
        points = axes[0][:, None]
        weights = _trapezoid_weights(axes[0])
    else:
        xx, yy = np.meshgrid(axes[0], axes[1], indexing="ij")
        points = np.column_stack([xx.ravel(), yy.ravel()])
        weights = np.outer(_trapezoid_weights(axes[0]), _trapezoid_weights(axes[1])).ravel()
    log_prior = np.array([prior.log_pdf(p) for p in points])
    log_like = np.asarray(log_like_batch(problem, np.ascontiguousarray(points)), dtype=float)
    joint = log_prior + log_like
    log_evidence = logsumexp_weighted(joint, weights)
    log_post = joint - log_evidence
    mode = points[int(np.argmax(joint))].copy()
    return PosteriorResult(points=points, log_prior=log_prior, log_like=log_like,
                           log_post=log_post, log_evidence=log_evidence, mode=mode,
                           weights=weights)


def _run_chains(problem, prior, chain, seeds, log_like_batch):
    if prior.n_z > 4:
        raise UsageError("random-walk chains support at most four parameters")
    C = len(seeds)
    n_z = prior.n_z
    rngs = [np.random.default_rng(s) for s in seeds]
    z = np.stack([prior.sample(r).reshape(n_z) for r in rngs])
    has_data = problem.model.n_y > 0

    def log_target(Zc):
        lp = np.array([prior.log_pdf(zc) for zc in Zc])
        lt = lp.copy()
        ok = np.isfinite(lp)
        if has_data and ok.any():
            lt[ok] = lp[ok] + np.asarray(log_like_batch(problem, np.ascontiguousarray(Zc[ok])), dtype=float)
        return lp, lt

    lp, lt = log_target(z)
    total = chain.burn + chain.length
    samples = np.empty((C, total, n_z))
    log_posts = np.empty((C, total))
    log_priors = np.empty((C, total))
    accepted = np.zeros((C, total), dtype=bool)
    for it in range(total):
        prop = np.stack([z[c] + chain.proposal * rngs[c].standard_normal(n_z) for c in range(C)])
        lp_p, lt_p = log_target(prop)
        for c in range(C):
            if np.log(rngs[c].uniform()) < lt_p[c] - lt[c]:
                z[c], lp[c], lt[c] = prop[c], lp_p[c], lt_p[c]
                accepted[c, it] = True
        samples[:, it] = z
        log_posts[:, it] = lt
        log_priors[:, it] = lp
    out = []
    keep = slice(chain.burn, None)
    for c in range(C):
        rate = float(accepted[c].sum()) / total
        if not 0.05 <= rate <= 0.95:
            warnings.warn(f"Metropolis acceptance rate {rate:.3f} outside [0.05, 0.95]", RuntimeWarning)
        out.append(PosteriorResult(points=samples[c, keep], log_prior=log_priors[c, keep],
                                   log_like=log_posts[c, keep] - log_priors[c, keep],
                                   log_post=log_posts[c, keep], acceptance=rate, accepted=accepted[c, keep]))
    return out


def posterior_mcmc(problem: BayesProblem, prior: Prior, chain: ChainSpec,
                   log_like_batch=log_likelihood_batch) -> PosteriorResult:
    """Random-walk Metropolis chain targeting likelihood times prior (bayes.py:336-377)."""
    return _run_chains(problem, prior, chain, [chain.seed], log_like_batch)[0]


def posterior_mcmc_chains(problem: BayesProblem, prior: Prior, chain: ChainSpec, n_chains: int,
                          log_like_batch=log_likelihood_batch):
    """`n_chains` independent chains in lockstep, one device batch of proposals per
    step; chain c equals posterior_mcmc(..., ChainSpec(seed=chain.seed + c))."""
    if n_chains < 1:
        raise UsageError("n_chains must be positive")
    return _run_chains(problem, prior, chain, [chain.seed + c for c in range(n_chains)], log_like_batch)
