"""B200-native batched HDD likelihood (arXiv 1708.02207 hot path).

Z[B, n_z] -> kappa(Z) -> bottom-up Schur-complement sweep over the
hierarchical domain decomposition -> observation functionals F(u) ->
Gaussian log-likelihood, all in fp64 sm_100a CUDA kernels behind the C ABI of
libhdd_b200.so (include/hdd.h).  The Python surface mirrors the reference
package `hddsolve` (bayes.py / mesh.py / ddtree.py / errors.py).
"""
from .bayes import (  # noqa: F401
    BayesProblem,
    MeasurementModel,
    ParamField,
    Prior,
    SineKLField,
    ToleranceSpec,
    aligned_partition,
    forward_full_solve,
    forward_functionals,
    forward_functionals_batch,
    gaussian_log_likelihood,
    kl_pairs,
    log_likelihood,
    log_likelihood_batch,
    mean_observations,
    mean_over_cells,
    observe_solution,
    posterior_weights,
    prolong_rhs,
    solve_batch,
    solve_subdomain,
    solve_subdomain_batch,
)
from .errors import ConfigError, GeometryError, NumericalError, UsageError  # noqa: F401
from .geometry import (  # noqa: F401
    DDTree, Mesh, Rect, boundary_nodes, build_mesh, build_tree, dump_tree, interior_nodes, omega_nodes,
)

__version__ = "0.1.0"
from . import configs, dumps, parallel, posterior  # noqa: E402,F401
from .dumps import dump_functionals, dump_store_stats, functional_summaries, store_stats  # noqa: E402,F401
from .posterior import ChainSpec, GridSpec, PosteriorResult, posterior_grid, posterior_mcmc, posterior_mcmc_chains  # noqa: E402,F401
