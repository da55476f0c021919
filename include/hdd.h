/*
 * hdd.h — C ABI of libhdd_b200.so, the B200-native batched HDD likelihood.
 *
 * One plan = one BayesProblem of the reference (mesh level, parametrization,
 * right-hand side f, MeasurementModel), compiled into device tables once;
 * every forward call evaluates a whole batch Z[B, n_z] of parameter samples:
 *
 *     Z -> kappa(Z) -> bottom-up Schur sweep -> S(Z) = F(u) -> log L(Z)
 *
 * Entry points and the reference interfaces they replace
 * (paths under /root/reference/pkg/src/hddsolve/):
 *
 *   hdd_plan_create    BayesProblem(...) (bayes.py:155-177) + build_mesh
 *                      (mesh.py:90-111) + build_tree (ddtree.py:119-174) +
 *                      FunctionalTracker.__init__ (functionals.py:146-175):
 *                      geometry, merge plan and observation routing, built once.
 *   hdd_forward_batch  forward_functionals (bayes.py:180-198) and
 *                      log_likelihood / gaussian_log_likelihood
 *                      (bayes.py:222-231), batched over Z rows; internally
 *                      ParamField.kappa (bayes.py:73-77), leaves_to_root in
 *                      functionals_only mode (hdd.py:289-394) and the tracker
 *                      callbacks (functionals.py:182-224).
 *   hdd_plan_destroy   (garbage collection of the problem / MapStore).
 *   hdd_last_error     the reference's exceptions (errors.py:4-21): the
 *                      status code selects ConfigError / UsageError /
 *                      NumericalError(node_id).
 *   hdd_plan_*info     debug views of the plan (DDNode index sets and merge
 *                      plan, ddtree.py:40-57), used by the host-logic tests.
 *
 * Conventions: plain pointers and sizes only.  Device pointers are CUDA
 * device addresses on the plan's device; `stream` is a cudaStream_t passed as
 * void* (NULL = the legacy default stream, like a CUDA launch without one).  All functions return HDD_OK (0) or a negative status; no call
 * falls back to the CPU.
 */
#ifndef HDD_B200_H
#define HDD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  HDD_OK = 0,
  HDD_ERR_CONFIG = -1,     /* ConfigError: invalid level, n_z, sigma, kappa  */
  HDD_ERR_USAGE = -2,      /* UsageError: bad call / observation routing      */
  HDD_ERR_NUMERICAL = -3,  /* NumericalError: non-SPD interface, non-finite S */
  HDD_ERR_CUDA = -4,       /* CUDA runtime failure (message carries detail)   */
  HDD_ERR_NOMEM = -5
};

enum { HDD_OBS_POINT = 0, HDD_OBS_MEAN = 1 };

typedef struct HddPlan HddPlan;

typedef struct {
  int32_t level;           /* mesh level L: 2^L cells per side (1 <= L <= 11);
                              levels 1-3 are solved by one warp per sample   */
  int32_t n_z;             /* parameter dimension                             */
  /* separable log-coefficient: for triangle t = 2(i N + j) + type,
   *   log kappa_t = sum_k coef[k] z[k] sx[k][2 i + type] sy[k][2 j + type]
   * (sine-KL: sin(pi a_k cx), sin(pi b_k cy), coef 0.5/k; reference
   *  indicator ParamField: 0/1 interval masks, coef 1).  Row-major
   *  [n_z][2N] host arrays.  All three NULL: no parametrization, the plan
   *  evaluates caller-supplied fields (hdd_forward_batch_kappa; the
   *  reference's duck-typed param.kappa(z), bayes.py:183).                  */
  const double* sx;
  const double* sy;
  const double* coef;
  const double* f;         /* nodal right-hand side [n nodes], NULL = 1       */
  int32_t n_obs;
  const int32_t* obs_kind; /* HDD_OBS_POINT (mesh node index) or HDD_OBS_MEAN */
  const int64_t* obs_id;   /* (reference post-order tree node id)            */
  const double* sigma;     /* [n_obs] noise std, > 0                          */
  const double* y;         /* [n_obs] data, NULL = no likelihood             */
  int32_t max_batch;       /* samples per internal sub-batch (0 = auto)       */
  int32_t device;          /* CUDA device, -1 = host-only plan (tests)        */
  int32_t keep_nodes;      /* 1 = keep every depth's outputs (debug hooks)    */
  int32_t mode;            /* -1 auto, 0 adjoint (all functionals carried to
                              the root, functionals.py:138-224), 1 primal
                              (points by the top-down interface back-solve,
                              hdd.py:397-432, restricted to what F needs)     */
  /* low-rank storage of the boundary maps (reference ToleranceSpec,
   * lowrank.py:20-30; hdd.py:280-286): eps <= 0 disables it               */
  double lr_eps;
  int32_t lr_kmax;
  int32_t lr_nmin;
  /* Dirichlet data on the domain boundary, [4N] in increasing mesh-node order
   * (the reference's root.idx_boundary order, bayes.py:162); NULL = 0.  Known
   * boundary values are folded into the load and functional columns at the
   * kernel-leaf outputs, so the upper merges never see them.                 */
  const double* g;
  /* 1 = keep the primal factors of EVERY upper node (required by
   * hdd_solve_batch, the root_to_leaves analogue of SolveMode.keep_all(),
   * hdd.py:120-138); 0 = likelihood plans keep them only on the
   * root-to-observation paths the top-down sweep visits.                      */
  int32_t full_solve;
  /* >= 0: reference node id of a solve_subdomain target (hdd.py:435-490): the plan
   * keeps factors only on the root-to-target path and the target's subtree (the
   * reference's SolveMode.keep_path, hdd.py:186-203) for hdd_solve_subdomain_batch;
   * -1 = none.                                                                 */
  int64_t solve_target;
} HddPlanDesc;

typedef struct {
  int32_t code;
  int32_t sample;          /* failing sample (-1 if n/a)                      */
  int64_t node_id;         /* failing reference tree node id (-1 if n/a)     */
  char message[256];
} HddError;

typedef struct {
  int32_t level, n_cells, leaf_cells, leaf_depth;
  int32_t n_upper, n_leaves, n_obs, leaf_cols;
  int32_t max_batch, n_kernels_per_batch;
  int64_t workspace_bytes;
  int32_t mode;
  int32_t n_topdown;       /* primal: upper nodes the top-down sweep visits   */
  int32_t tiny;            /* 1: level <= 3, one warp per sample (no tree)    */
  int32_t separable;       /* 1: Z entry points (K1); 0: kappa entry points   */
  int32_t full_solve;      /* 1: factors of every node kept (hdd_solve_batch) */
  int32_t n_omega;         /* solve_subdomain plans: |idx_omega| of the target */
  int64_t factor_doubles;  /* primal factor storage per sample (doubles)      */
} HddPlanInfo;

typedef struct {
  int64_t ref_id;          /* reference post-order node id                    */
  int32_t depth, i0, i1, j0, j1;
  int32_t son[2];          /* plan indices of the sons; -1-leaf for leaves    */
  int32_t k, ng, nc;       /* |pruned boundary|, |interface|, output columns */
  const int64_t* bnd;      /* [k] pruned boundary ids (sorted)                */
  const int64_t* gamma;    /* [ng] interface ids (sorted)                     */
  const int32_t* gmap;     /* [2][k+ng] son output row of each father index  */
  const int32_t* csrc;     /* [nc][2] son column feeding each column, -1 none */
  const double* ccoef;     /* [nc][2] coefficients                            */
  const int32_t* cbirth;   /* [nc] interface position of a born point, -1    */
} HddNodeInfo;

typedef struct {
  int64_t ref_id;
  int32_t i0, j0, ncols, has_mean;
  const int32_t* birth;    /* [ncols][3]: in-leaf level, node, gamma pos     */
  const int32_t* ccode;    /* [ncols] 0 load, 1 own mean, 2 point, or a mean
                              over a sub-leaf node: (1 << 24) | i0 | i1 << 5 |
                              j0 << 10 | j1 << 15 (leaf-local cell range)    */
  const double* gperim;    /* [64] Dirichlet value of each perimeter node on the
                              domain boundary (NULL when g = 0)                */
} HddLeafInfo;

typedef struct {
  int32_t kind;            /* 0 root column, 1 constant, 2 leaf point (primal),
                              3 interface point (primal)                       */
  int32_t col;
  double value;
  int32_t node;            /* leaf (kind 2) / upper node (kind 3) plan index  */
  int32_t slot;
} HddObsInfo;

int hdd_plan_create(const HddPlanDesc* desc, HddPlan** out);
int hdd_plan_destroy(HddPlan* plan);

/* Z_dev [B][n_z], S_dev [B][n_obs] (nullable), ll_dev [B] (nullable).
 * ASYNCHRONOUS: returns once the launches are queued on `stream`.  Failures
 * (non-SPD interface, non-finite S, invalid kappa) are recorded on the device
 * and reported by hdd_sync, by the synchronous (_host) calls, or by the next
 * call on the plan once the record has reached the host; the HddError then
 * names the lowest failing sample of that call. */
int hdd_forward_batch(HddPlan* plan, const double* Z_dev, int64_t B,
                      double* S_dev, double* ll_dev, void* stream);

/* Waits for `stream` and returns the status of the calls queued since the last
 * check: HDD_OK, or the recorded failure (hdd_last_error has the details). */
int hdd_sync(HddPlan* plan, void* stream);

/* Same as hdd_forward_batch with caller-supplied coefficient fields instead of
 * Z: K_dev [B][2 N^2], triangle order t = 2(i N + j) + type (the reference's
 * CoefficientField.values, fem.py:23-43) — the drop-in for a duck-typed
 * problem.param whose .kappa(z) is arbitrary host code (bayes.py:183, :204,
 * :242).  Values are checked positive and finite on the device (ConfigError). */
int hdd_forward_batch_kappa(HddPlan* plan, const double* K_dev, int64_t B,
                            double* S_dev, double* ll_dev, void* stream);
int hdd_forward_batch_kappa_host(HddPlan* plan, const double* K_host, int64_t B,
                                 double* S_host, double* ll_host);

/* Same as hdd_forward_batch, plus per-stage device time (CUDA events on the
 * launching stream), accumulated over the internal sub-batches into
 * stage_ms[n_stages]: [0] kappa, [1] leaf, [2 + i] merges of depth
 * leaf_depth-1-i (deepest first), [n_stages-1] finalize.  n_stages must be
 * leaf_depth + 3. Synchronizes the stream. */
int hdd_forward_batch_timed(HddPlan* plan, const double* Z_dev, int64_t B,
                            double* S_dev, double* ll_dev, void* stream,
                            double* stage_ms, int32_t n_stages);

/* Same call with HOST buffers (synchronous): sub-batch i+1's H2D copy and
 * sub-batch i-1's D2H copy run on two copy streams beside sub-batch i's
 * compute; returns when the results are in host memory. */
int hdd_forward_batch_host(HddPlan* plan, const double* Z_host, int64_t B,
                           double* S_host, double* ll_host);

/* Full solution u at every mesh node for every row of Z: U_dev[B][n_nodes]
 * (n_nodes = (2^level + 1)^2, node id j * (2^level + 1) + i).  The bottom-up
 * sweep and the primal top-down sweep give u on every interface; each kernel
 * leaf then solves for its interior nodes.  Requires a plan created with
 * mode = 1 and full_solve = 1 (every factor kept), else HDD_ERR_USAGE — the
 * analogue of root_to_leaves requiring a store built with SolveMode.keep_all().
 * Asynchronous like hdd_forward_batch.
 * Replaces root_to_leaves / forward_full_solve (reference hdd.py:397-432,
 * bayes.py:201-208). */
int hdd_solve_batch(HddPlan* plan, const double* Z_dev, int64_t B, double* U_dev, void* stream);

/* Same call with HOST buffers. */
int hdd_solve_batch_host(HddPlan* plan, const double* Z_host, int64_t B, double* U_host);
/* Full solution from caller-supplied coefficient fields K [B][2 N^2]. */
int hdd_solve_batch_kappa(HddPlan* plan, const double* K_dev, int64_t B, double* U_dev, void* stream);
int hdd_solve_batch_kappa_host(HddPlan* plan, const double* K_host, int64_t B, double* U_host);

/* Per-triangle kappa for a batch (parity hook for the assembly kernel). */
int hdd_kappa_batch(HddPlan* plan, const double* Z_dev, int64_t B,
                    double* kappa_dev, void* stream);

/* Posterior weights of a batch of log-likelihoods, on the device (the pieces of the
 * reference posterior_grid, bayes.py:325-330, for prior draws): joint = ll (+ log_prior
 * when non-NULL), lse = logsumexp(joint), w = exp(joint - lse), idx = the first index
 * of max(joint) (numpy argmax tie rule).  Device pointers on the current device; one
 * kernel launch on `stream`, deterministic (fixed reduction order), so every rank of an
 * all-gathered batch gets bitwise-identical weights.  HDD_ERR_USAGE for n <= 0 or NULL
 * ll / w / idx / lse. */
int hdd_posterior_weights(const double* ll_dev, const double* log_prior_dev, int64_t n, double* w_dev,
                          int64_t* idx_dev, double* lse_dev, void* stream);

/* Per-call right-hand sides: the general maps Psi^f / Phi^f (hdd.py:58-105,
 * PsiMap.residual / PhiMap.apply) applied to new data without a new plan — a
 * batch row may carry its own f and g ("multiple right-hand sides and multiple
 * Dirichlet data").  f rows hold n_nodes values (mesh-node order),
 * g rows 4N values (boundary nodes in increasing id order, the reference's
 * root.idx_boundary); stride 0 = one row shared by the whole batch; NULL = the
 * plan's f / g.  Host variants take host rows (stride 0 or the row length). */
typedef struct {
  const double* f;
  int64_t f_stride;
  const double* g;
  int64_t g_stride;
} HddRhs;

/* Forward / likelihood with exactly one of Z_dev [B][n_z] and K_dev [B][2N^2]
 * (caller fields) and optional per-call rows (asynchronous, like
 * hdd_forward_batch). */
int hdd_forward_batch_ex(HddPlan* plan, const double* Z_dev, const double* K_dev, int64_t B, const HddRhs* rhs,
                         double* S_dev, double* ll_dev, void* stream);
int hdd_forward_batch_ex_host(HddPlan* plan, const double* Z_host, const double* K_host, int64_t B,
                              const HddRhs* rhs_host, double* S_host, double* ll_host);
/* Full solution u with per-call rows (full-solution plans). */
int hdd_solve_batch_ex(HddPlan* plan, const double* Z_dev, const double* K_dev, int64_t B, const HddRhs* rhs,
                       double* U_dev, void* stream);
int hdd_solve_batch_ex_host(HddPlan* plan, const double* Z_host, const double* K_host, int64_t B,
                            const HddRhs* rhs_host, double* U_host);

/* solve_subdomain (hdd.py:435-490) as a partial inverse: the solution on the plan's
 * target node only, Usub [B][n_omega] aligned with the target's idx_omega (sorted
 * global ids of the closed subdomain).  Only the root-to-target path and the target's
 * subtree are factored, swept top-down and solved in-leaf.  Exactly one of Z / K;
 * rhs optional (as in hdd_forward_batch_ex).  HDD_ERR_USAGE unless the plan was
 * created with solve_target >= 0. */
int hdd_solve_subdomain_batch(HddPlan* plan, const double* Z_dev, const double* K_dev, int64_t B,
                              const HddRhs* rhs, double* Usub_dev, void* stream);
int hdd_solve_subdomain_batch_host(HddPlan* plan, const double* Z_host, const double* K_host, int64_t B,
                                   const HddRhs* rhs_host, double* Usub_host);

int hdd_last_error(const HddPlan* plan, HddError* out);
/* Error of the last failed hdd_plan_create (no plan exists then). */
int hdd_create_error(HddError* out);

int hdd_plan_info(const HddPlan* plan, HddPlanInfo* out);
int hdd_plan_node_info(const HddPlan* plan, int32_t idx, HddNodeInfo* out);
int hdd_plan_leaf_info(const HddPlan* plan, int32_t idx, HddLeafInfo* out);
int hdd_plan_obs_info(const HddPlan* plan, int32_t idx, HddObsInfo* out);
/* In-leaf template: level r = 0..7 -> K, k, ng and the son gather maps. */
int hdd_leaf_template(int32_t r, int32_t* K, int32_t* k, int32_t* ng,
                      const int32_t** map1, const int32_t** map2);

/* Debug: copy node `idx` (plan index; leaves are -1-leaf) outputs of the last
 * forward call for sample b: psi [k][k], R [k][nc], sigma [nc] to host. */
int hdd_debug_node_output(HddPlan* plan, int32_t idx, int32_t b,
                          double* psi, double* R, double* sigma);

/* Profiling hook: clock64 stamps of leaf CTA (0,0) of the last launch
 * ([0] start, [1] after the register base, [10 + 8 (5-r) + phase] per level). */
int hdd_debug_leaf_clocks(long long* out64);
/* Per-phase clock64 stamps [32 depths][8] of CTA (sample 0, node 0) of each merge
 * launch of the last batch (profiling hook): 0 start, 1 maps staged, 2 panel
 * gathered, 3 eliminated, 4 sigma/factors written, 5 Schur update written. */
int hdd_debug_merge_clocks(long long* out);
/* Low-rank plans with k_max > 24: number of (block, sample) pairs handed to the
 * 72-column wide sketch since the plan was created (0 otherwise). */
int hdd_debug_lowrank_wide(HddPlan* plan, int64_t* total);

/* Which kernel(s) the merge of tree depth `depth` launches for a sub-batch of B
 * samples, as the ncu launch list names them (e.g. "merge_l_kernel<3,64>", or
 * "assemble_l_kernel+merge_l_kernel<2,128>+schur_l_kernel" on the split tier-L
 * depths); depth = -1: the kernel-leaf launch.  Used by bench.py to group the
 * CUDA-event stage times by kernel (reference: one `schur_eliminate` call per
 * node, hdd.py:241-277).  Returns HDD_ERR_USAGE for a depth without nodes. */
int hdd_plan_stage_kernel(const HddPlan* plan, int32_t depth, int32_t B, char* buf, int32_t cap);

const char* hdd_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HDD_B200_H */
