// Host-side plan of the batched HDD likelihood (internal header).
//
// The plan is the compiled form of one reference BayesProblem: the
// alternating-bisection tree truncated at 16x16-cell "kernel leaves", the
// pruned (Dirichlet-free) boundary/interface index sets of every upper node,
// the gather maps that replace the reference's scatter-add merge plan
// (ddtree.py:40-57 bpos/opos, hdd.py:216-238), and the column plan that
// routes the load vector and every observation functional up the tree
// (functionals.py:146-224).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "hdd.h"

namespace hdd {

constexpr int kLeafCells = 16;                 // kernel-leaf subdomain (cells per side)
constexpr int kLeafPerim = 4 * kLeafCells;     // 64 perimeter nodes
constexpr int kLeafLevels = 8;                 // in-leaf merge levels r = 0..7

enum ColKind { COL_LOAD = 0, COL_MEAN = 1, COL_OBS = 2, COL_SUBMEAN = 3 };

// Device column code of a mean over a sub-leaf tree node (functionals.py:47-61 mean
// rule restricted to the node's cells): tag | i0 | i1 << 5 | j0 << 10 | j1 << 15, the
// node's cell range in leaf-local coordinates.
constexpr int kSubMeanTag = 1 << 24;
inline int submean_code(int i0, int i1, int j0, int j1) {
  return kSubMeanTag | i0 | (i1 << 5) | (j0 << 10) | (j1 << 15);
}

struct Col {
  int kind;      // ColKind
  int obs;       // observation index for COL_OBS / COL_SUBMEAN
  int code = 0;  // COL_SUBMEAN: submean_code of the node's cells
};

struct UpperNode {
  int64_t ref_id = -1;
  int depth = 0, i0 = 0, i1 = 0, j0 = 0, j1 = 0;
  int son[2] = {0, 0};          // >= 0 upper index, < 0: -1 - leaf index
  int k = 0, ng = 0, K = 0, nc = 0;
  bool own_mean = false;
  std::vector<int64_t> bnd, gamma;
  std::vector<int32_t> gmap;    // [2][K]
  std::vector<int32_t> csrc;    // [nc][2]
  std::vector<double> ccoef;    // [nc][2]
  std::vector<int32_t> cbirth;  // [nc]
  std::vector<Col> cols;
  // low-rank blocks of Psi (admissible pairs of the boundary cluster tree)
  std::vector<int32_t> lr_rows, lr_cols;   // concatenated position lists
  std::vector<int32_t> lr_desc;            // [n][4]: row offset, p, col offset, q
  // output layout (per sample): rows k, leading dim ld, then nc sigmas
  int out_ld = 0;
  int64_t out_elems = 0;
  int64_t out_off = 0;          // element offset of sample 0 in its depth buffer
  int buf = 0;                  // output buffer id
  int tier = 0;                 // 0 = smem panel, 1 = global panel
  // primal mode: interface solution u_K = [u_B | u_gamma] and stored factors
  int parent = -1;              // upper index of the father (-1 for the root)
  std::vector<int32_t> cmap;    // [k] father K-index of each pruned boundary node
  int64_t fac_off = 0, u_off = 0;   // per-sample element offsets
};

struct Leaf {
  int64_t ref_id = -1;
  int i0 = 0, j0 = 0;
  bool own_mean = false;
  std::vector<Col> cols;
  std::vector<int32_t> birth;   // [ncols][3] (level r, node q, gamma pos) or -1
  int parent = -1;              // upper index of the father
  std::vector<int32_t> cmap;    // [64] father K-index of each perimeter node, -1 on the domain boundary
  std::vector<int32_t> fslot;   // [ncols] functional slot of a primal point column, -1
  std::vector<int32_t> ccode;   // [ncols] device column code: 0 load, 1 own mean, 2 point, submean_code
  std::vector<double> gperim;   // [64] Dirichlet value of each perimeter node on the domain boundary, else 0
  std::vector<int32_t> gpos;    // [64] position in the boundary vector g (increasing ids), -1 inside
};

struct ObsRoute {
  int kind;      // 0 = root column, 1 = constant, 2 = leaf point (primal), 3 = interface point (primal)
  int col;       // root column / leaf column / interface position
  double value;
  int node = -1; // leaf index (kind 2), upper index (kind 3), boundary position (kind 1 point)
  int slot = -1; // leaf functional slot (kind 2)
};

struct LeafLevel {                // in-leaf template level r (father shape)
  int w, h, K, k, ng, kson;
  std::vector<int32_t> map1, map2; // [K]
};

struct Plan {
  int level = 0, N = 0, m = 0, n_z = 0, leaf_depth = 0;
  double h = 0;
  std::vector<double> sx, sy, coef, f;
  bool f_is_one = true;
  std::vector<double> g;        // [4N] Dirichlet data (sorted boundary ids), empty = 0
  bool has_g = false;
  std::vector<int32_t> obs_kind;
  std::vector<int64_t> obs_id;
  std::vector<double> sigma, y;
  bool has_y = false;
  std::vector<UpperNode> upper;               // grouped by depth, deepest first
  std::vector<std::vector<int>> upper_by_depth;  // depth -> indices
  std::vector<Leaf> leaves;                   // post-order (left to right)
  int leaf_cols = 1;                          // NCL (max columns over leaves)
  int leaf_ld = 0;
  int64_t leaf_elems = 0;
  int leaf_buf = 0;
  std::vector<ObsRoute> route;
  int root = -1;                              // upper index of the root, or -1 (root is leaf 0)
  int root_nc = 0;
  int n_buffers = 2;
  int mode = 0;                               // 0 adjoint (functionals to the root), 1 primal top-down
  double lr_eps = 0.0;                        // low-rank truncation (0 = dense maps)
  int lr_kmax = 64, lr_nmin = 32;
  int n_fslots = 0;                           // leaf point functionals kept for the top-down pass
  int64_t fac_elems = 0, u_elems = 0;         // per-sample sizes of the primal buffers
  std::vector<int64_t> buf_elems_per_sample;  // per buffer
  bool full_solve = false;                    // primal factors kept for every node
  int64_t solve_target = -1;                  // solve_subdomain plan: reference node id, -1 none
  struct { int i0, i1, j0, j1; } solve_rect{0, 0, 0, 0};
  std::vector<int32_t> solve_leaves;          // kernel leaves of the target's subtree (or its container)
  std::vector<int32_t> omega_pos;             // [m*m] position in the target's idx_omega, -1 outside
  int n_omega = 0;
  std::vector<std::vector<int>> td_by_depth;  // primal: upper nodes the top-down sweep visits
  bool separable = true;                      // sx/sy/coef given (else kappa per call)
  bool tiny = false;                          // level <= 3: tiny_kernel, no tree sweep
  std::vector<double> gfull;                  // tiny: [m*m] boundary values
  int64_t root_ref = 0;
};

// Build the plan; returns empty string on success, else the ConfigError /
// UsageError message (code in *code).
std::string build_plan(const HddPlanDesc* desc, Plan& plan, int* code);
std::string build_tiny_plan(const HddPlanDesc* desc, Plan& plan, int* code);

const std::vector<LeafLevel>& leaf_template();
int64_t postorder_id(int level, const std::vector<int>& path);

}  // namespace hdd
