// Plan construction for the batched HDD likelihood (host side, C++17).
//
// Geometry follows the reference exactly (paths under
// /root/reference/pkg/src/hddsolve/):
//   * node (i, j) -> id j*m + i                                  mesh.py:90-98
//   * perimeter ids sorted ascending                             mesh.py:123-135
//   * alternating bisection, x cut first, axis switched when the
//     node is one cell wide, son 1 = lower/left half            ddtree.py:139-149
//   * interface = son-1 perimeter minus father perimeter         ddtree.py:155
//   * post-order node ids (sons precede father)                  ddtree.py:152-173
// Departures (exact algebraic identities):
//   * g = 0 on the domain boundary, so every boundary row/column is pruned
//     from the upper nodes' index sets;
//   * f is fixed per plan, so the reference's |omega|-wide psi_f / phi_f maps
//     are condensed to one load column (hdd.py:276-277);
//   * observation functionals travel as extra columns of the same Schur
//     complement ("bordered" elimination), which is the reference's
//     Algorithms 1-2 (functionals.py:77-106) in matrix form.
#include "hdd_plan.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>

namespace hdd {
namespace {

struct Rect {
  int i0, i1, j0, j1;
};

// Sons of a cell rectangle (ddtree.py:139-149).
void split(const Rect& r, int depth, Rect& a, Rect& b, int* axis_out) {
  int nx = r.i1 - r.i0, ny = r.j1 - r.j0;
  int axis = depth % 2;
  if (axis == 0 && nx == 1) axis = 1;
  else if (axis == 1 && ny == 1) axis = 0;
  if (axis == 0) {
    int mid = (r.i0 + r.i1) / 2;
    a = {r.i0, mid, r.j0, r.j1};
    b = {mid, r.i1, r.j0, r.j1};
  } else {
    int mid = (r.j0 + r.j1) / 2;
    a = {r.i0, r.i1, r.j0, mid};
    b = {r.i0, r.i1, mid, r.j1};
  }
  if (axis_out) *axis_out = axis;
}

// Perimeter node ids in ascending order (rows bottom to top).
std::vector<int64_t> perimeter(const Rect& r, int64_t m) {
  std::vector<int64_t> out;
  out.reserve(2 * (r.i1 - r.i0) + 2 * (r.j1 - r.j0));
  for (int i = r.i0; i <= r.i1; ++i) out.push_back(int64_t(r.j0) * m + i);
  for (int j = r.j0 + 1; j < r.j1; ++j) {
    out.push_back(int64_t(j) * m + r.i0);
    out.push_back(int64_t(j) * m + r.i1);
  }
  for (int i = r.i0; i <= r.i1; ++i) out.push_back(int64_t(r.j1) * m + i);
  return out;
}

// Interface of a split node: the cut line without its two perimeter ends.
std::vector<int64_t> interface_ids(const Rect& r, int depth, int64_t m) {
  Rect a, b;
  int axis;
  split(r, depth, a, b, &axis);
  std::vector<int64_t> out;
  if (axis == 0) {
    for (int j = r.j0 + 1; j < r.j1; ++j) out.push_back(int64_t(j) * m + a.i1);
  } else {
    for (int i = r.i0 + 1; i < r.i1; ++i) out.push_back(int64_t(a.j1) * m + i);
  }
  return out;
}

int find_pos(const std::vector<int64_t>& sorted, int64_t id) {
  auto it = std::lower_bound(sorted.begin(), sorted.end(), id);
  if (it == sorted.end() || *it != id) return -1;
  return int(it - sorted.begin());
}

int64_t subtree_size(int level, int depth) { return (int64_t(1) << (2 * level - depth + 1)) - 1; }

// Geometric cluster tree over point positions (lowrank.py:101-115): split at the
// bbox midpoint of the longer axis (x on ties), fall back to sorted halves.
struct Cluster {
  std::vector<int32_t> pos;
  double bb[4];          // xmin, xmax, ymin, ymax
  int child[2] = {-1, -1};
};

int build_cluster(std::vector<Cluster>& cl, std::vector<int32_t> pos, const std::vector<double>& x,
                  const std::vector<double>& y, int n_min) {
  Cluster c;
  c.bb[0] = c.bb[2] = 1e300;
  c.bb[1] = c.bb[3] = -1e300;
  for (int p : pos) {
    c.bb[0] = std::min(c.bb[0], x[p]); c.bb[1] = std::max(c.bb[1], x[p]);
    c.bb[2] = std::min(c.bb[2], y[p]); c.bb[3] = std::max(c.bb[3], y[p]);
  }
  c.pos = pos;
  const int me = int(cl.size());
  cl.push_back(c);
  if (int(pos.size()) <= n_min) return me;
  const bool ax = (c.bb[1] - c.bb[0]) >= (c.bb[3] - c.bb[2]);
  const double mid = ax ? 0.5 * (c.bb[0] + c.bb[1]) : 0.5 * (c.bb[2] + c.bb[3]);
  std::vector<int32_t> l, r;
  for (int p : pos) ((ax ? x[p] : y[p]) < mid ? l : r).push_back(p);
  if (l.empty() || r.empty()) {
    std::vector<int32_t> srt = pos;
    std::stable_sort(srt.begin(), srt.end(), [&](int a, int b) { return (ax ? x[a] : y[a]) < (ax ? x[b] : y[b]); });
    l.assign(srt.begin(), srt.begin() + srt.size() / 2);
    r.assign(srt.begin() + srt.size() / 2, srt.end());
    // keep the original relative order inside each half (reference uses pos[left])
    std::vector<char> inl(x.size(), 0);
    for (int p : l) inl[p] = 1;
    l.clear(); r.clear();
    for (int p : pos) (inl[p] ? l : r).push_back(p);
  }
  const int a = build_cluster(cl, l, x, y, n_min);
  const int b = build_cluster(cl, r, x, y, n_min);
  cl[me].child[0] = a;
  cl[me].child[1] = b;
  return me;
}

bool disjoint(const Cluster& a, const Cluster& b) {
  return a.bb[1] < b.bb[0] || b.bb[1] < a.bb[0] || a.bb[3] < b.bb[2] || b.bb[3] < a.bb[2];
}

// Admissible (disjoint-bbox) block pairs of the partition (lowrank.py:166-179).
void collect_blocks(const std::vector<Cluster>& cl, int rc, int cc, std::vector<std::pair<int, int>>& out) {
  const Cluster& R = cl[rc];
  const Cluster& Cc = cl[cc];
  if (R.pos.empty() || Cc.pos.empty()) return;
  if (disjoint(R, Cc)) { out.push_back({rc, cc}); return; }
  const bool rl = R.child[0] < 0, cl_ = Cc.child[0] < 0;
  if (rl && cl_) return;   // dense leaf block
  std::vector<int> rch = rl ? std::vector<int>{rc} : std::vector<int>{R.child[0], R.child[1]};
  std::vector<int> cch = cl_ ? std::vector<int>{cc} : std::vector<int>{Cc.child[0], Cc.child[1]};
  for (int a : rch)
    for (int b : cch) collect_blocks(cl, a, b, out);
}

}  // namespace

int64_t postorder_id(int level, const std::vector<int>& path) {
  int64_t id = 0;
  for (size_t d = 1; d <= path.size(); ++d)
    if (path[d - 1]) id += subtree_size(level, int(d));
  return id + subtree_size(level, int(path.size())) - 1;
}

const std::vector<LeafLevel>& leaf_template() {
  static std::vector<LeafLevel> tmpl = [] {
    std::vector<LeafLevel> t;
    Rect r{0, kLeafCells, 0, kLeafCells};
    // local ids: y * 64 + x keeps (y, x) order = global-id order
    const int64_t M = 64;
    for (int lev = 0; lev < kLeafLevels; ++lev) {
      LeafLevel L;
      L.w = r.i1 - r.i0;
      L.h = r.j1 - r.j0;
      Rect a, b;
      split(r, lev, a, b, nullptr);
      auto per = perimeter(r, M);
      auto gam = interface_ids(r, lev, M);
      L.k = int(per.size());
      L.ng = int(gam.size());
      L.K = L.k + L.ng;
      std::vector<int64_t> K = per;
      K.insert(K.end(), gam.begin(), gam.end());
      auto p1 = perimeter(a, M), p2 = perimeter(b, M);
      L.kson = int(p1.size());
      for (int64_t id : K) {
        L.map1.push_back(find_pos(p1, id));
        L.map2.push_back(find_pos(p2, id));
      }
      t.push_back(std::move(L));
      r = a;
    }
    return t;
  }();
  return tmpl;
}

namespace {
// Cell rectangle of a reference post-order tree node id (ddtree.py:152-173): descend
// from the root, the first son's subtree holds the smaller ids.
bool rect_of_id(int level, int64_t id, Rect* out) {
  if (id < 0 || id >= subtree_size(level, 0)) return false;
  const int N = 1 << level;
  Rect r{0, N, 0, N};
  int depth = 0;
  int64_t lo = 0;
  while (lo + subtree_size(level, depth) - 1 != id) {
    Rect a, b;
    split(r, depth, a, b, nullptr);
    const int64_t half = subtree_size(level, depth + 1);
    if (id < lo + half) r = a;
    else { r = b; lo += half; }
    ++depth;
  }
  *out = r;
  return true;
}
}  // namespace

// Levels 1-3: the whole mesh is smaller than one kernel leaf; one warp per sample
// eliminates the interior directly (tiny_kernel).  Observation routes: 1 constant
// (boundary point: g there), 4 interior point (col = node id), 5 mean (col = packed cells).
std::string build_tiny_plan(const HddPlanDesc* d, Plan& P, int* code) {
  P.tiny = true;
  P.leaf_depth = 0;
  P.mode = 0;
  P.root = -1;
  P.root_ref = subtree_size(P.level, 0) - 1;
  P.leaf_cols = 1;
  P.n_buffers = 0;
  const int N = P.N;
  const int64_t m = P.m;
  auto is_boundary = [&](int64_t id) {
    const int64_t i = id % m, j = id / m;
    return i == 0 || j == 0 || i == N || j == N;
  };
  P.gfull.assign(size_t(m) * m, 0.0);
  if (P.has_g) {
    size_t pos = 0;   // boundary nodes in increasing id order (root.idx_boundary)
    for (int64_t id = 0; id < m * m; ++id)
      if (is_boundary(id)) P.gfull[size_t(id)] = P.g[pos++];
  }
  P.route.assign(P.obs_kind.size(), ObsRoute{1, -1, 0.0});
  for (size_t o = 0; o < P.obs_kind.size(); ++o) {
    const int64_t id = P.obs_id[o];
    if (P.obs_kind[o] == HDD_OBS_POINT) {
      if (id < 0 || id >= m * m) { *code = HDD_ERR_USAGE; return "mesh node " + std::to_string(id) + " not found on any interface"; }
      if (is_boundary(id)) {
        const int64_t i = id % m, j = id / m;
        const int pos = int(j == 0 ? i : (j == N ? m + 2 * (N - 1) + i : m + 2 * (j - 1) + (i == N ? 1 : 0)));
        P.route[o] = ObsRoute{1, -1, P.gfull[size_t(id)], pos};
      } else {
        P.route[o] = ObsRoute{4, int(id), 0.0};
      }
    } else if (P.obs_kind[o] == HDD_OBS_MEAN) {
      Rect r;
      if (!rect_of_id(P.level, id, &r)) { *code = HDD_ERR_USAGE; return "no tree node with id " + std::to_string(id); }
      P.route[o] = ObsRoute{5, r.i0 | (r.i1 << 5) | (r.j0 << 10) | (r.j1 << 15), 0.0};
    } else {
      return "unknown observation kind " + std::to_string(P.obs_kind[o]);
    }
  }
  P.lr_eps = d->lr_eps > 0 ? d->lr_eps : 0.0;   // no map is larger than n_min: nothing to compress
  *code = HDD_OK;
  return "";
}

std::string build_plan(const HddPlanDesc* d, Plan& P, int* code) {
  *code = HDD_ERR_CONFIG;
  if (!d) { *code = HDD_ERR_USAGE; return "null plan descriptor"; }
  if (d->level < 1 || d->level > 11)
    return "mesh level must be an integer in [1, 11], got " + std::to_string(d->level);
  // separable tables are optional: without them the plan evaluates caller-supplied
  // coefficient fields only (hdd_forward_batch_kappa; the reference's duck-typed
  // param.kappa(z), bayes.py:183)
  P.separable = d->sx && d->sy && d->coef;
  if ((d->sx || d->sy || d->coef) && !P.separable) return "separable parametrization needs all of sx, sy, coef";
  if (P.separable && (d->n_z < 1 || d->n_z > 256)) return "parameter dimension n_z must be in [1, 256]";
  if (!P.separable && (d->n_z < 0 || d->n_z > 256)) return "parameter dimension n_z must be in [0, 256]";
  if (d->n_obs < 1) return "at least one observation is required";
  if (!d->obs_kind || !d->obs_id || !d->sigma) return "observation arrays are required";
  P.level = d->level;
  P.N = 1 << d->level;
  P.m = P.N + 1;
  P.h = 1.0 / P.N;
  P.n_z = d->n_z;
  const int N = P.N;
  const int64_t m = P.m;
  if (P.separable) {
    P.sx.assign(d->sx, d->sx + size_t(d->n_z) * 2 * N);
    P.sy.assign(d->sy, d->sy + size_t(d->n_z) * 2 * N);
    P.coef.assign(d->coef, d->coef + d->n_z);
  }
  for (double v : P.sx) if (!std::isfinite(v)) return "parametrization table sx is not finite";
  for (double v : P.sy) if (!std::isfinite(v)) return "parametrization table sy is not finite";
  P.f_is_one = (d->f == nullptr);
  if (d->f) {
    P.f.assign(d->f, d->f + size_t(m) * m);
    for (double v : P.f) if (!std::isfinite(v)) return "right-hand side f is not finite";
  }
  if (d->g) {
    P.g.assign(d->g, d->g + size_t(4) * N);
    for (double v : P.g) {
      if (!std::isfinite(v)) return "Dirichlet data g is not finite";
      if (v != 0.0) P.has_g = true;
    }
  }
  const int n_obs = d->n_obs;
  P.obs_kind.assign(d->obs_kind, d->obs_kind + n_obs);
  P.obs_id.assign(d->obs_id, d->obs_id + n_obs);
  P.sigma.assign(d->sigma, d->sigma + n_obs);
  for (double s : P.sigma)
    if (!(s > 0) || !std::isfinite(s)) return "one positive noise level per observation required";
  P.has_y = d->y != nullptr;
  if (P.has_y) {
    P.y.assign(d->y, d->y + n_obs);
    for (double v : P.y) if (!std::isfinite(v)) return "data vector y is not finite";
  }
  P.root_ref = subtree_size(P.level, 0) - 1;
  P.solve_target = d->solve_target;
  if (d->solve_target >= 0) {
    Rect r;
    if (!rect_of_id(P.level, d->solve_target, &r)) {
      *code = HDD_ERR_USAGE;
      return "no tree node with id " + std::to_string(d->solve_target);
    }
    P.solve_rect = {r.i0, r.i1, r.j0, r.j1};
    P.omega_pos.assign(size_t(m) * m, -1);
    for (int j = r.j0; j <= r.j1; ++j)          // idx_omega: sorted global ids (ddtree.py:40-57)
      for (int i = r.i0; i <= r.i1; ++i) P.omega_pos[size_t(j) * m + i] = P.n_omega++;
  }
  if (P.level < 4) return build_tiny_plan(d, P, code);
  const int dl = 2 * (P.level - 4);   // depth of the 16x16-cell kernel leaves
  P.leaf_depth = dl;

  // ---- enumerate the truncated tree (post-order within each depth) -------
  struct Tmp { Rect r; int depth; std::vector<int> path; int parent; int son[2]; };
  std::vector<Tmp> all;
  {
    std::vector<int> path;
    // recursive lambda via explicit stack-free recursion
    struct Rec {
      std::vector<Tmp>& all; int dl;
      int go(Rect r, int depth, std::vector<int>& path) {
        int me = int(all.size());
        all.push_back({r, depth, path, -1, {-1, -1}});
        if (depth == dl) return me;
        Rect a, b;
        split(r, depth, a, b, nullptr);
        path.push_back(0);
        int s1 = go(a, depth + 1, path);
        path.back() = 1;
        int s2 = go(b, depth + 1, path);
        path.pop_back();
        all[me].son[0] = s1;
        all[me].son[1] = s2;
        all[s1].parent = me;
        all[s2].parent = me;
        return me;
      }
    } rec{all, dl};
    rec.go({0, N, 0, N}, 0, path);
  }
  // depth lists in left-to-right order (preorder visit order keeps that)
  std::vector<std::vector<int>> by_depth(dl + 1);
  for (int t = 0; t < int(all.size()); ++t) by_depth[all[t].depth].push_back(t);
  std::vector<int> to_plan(all.size(), 0);   // tmp -> upper idx or -1-leaf
  for (int li = 0; li < int(by_depth[dl].size()); ++li) to_plan[by_depth[dl][li]] = -1 - li;
  P.upper_by_depth.assign(dl, {});
  for (int dep = dl - 1; dep >= 0; --dep)
    for (int t : by_depth[dep]) {
      to_plan[t] = int(P.upper.size());
      P.upper_by_depth[dep].push_back(int(P.upper.size()));
      P.upper.emplace_back();
    }
  P.leaves.resize(by_depth[dl].size());
  auto is_boundary = [&](int64_t id) {
    int64_t i = id % m, j = id / m;
    return i == 0 || j == 0 || i == N || j == N;
  };
  // position of a boundary node in increasing-id order: the bottom row (m), then two
  // per interior row (left, right), then the top row
  auto bpos_of = [&](int64_t id) -> int {
    const int64_t i = id % m, j = id / m;
    return int(j == 0 ? i : (j == N ? m + 2 * (N - 1) + i : m + 2 * (j - 1) + (i == N ? 1 : 0)));
  };
  auto g_of = [&](int64_t id) -> double { return P.has_g ? P.g[size_t(bpos_of(id))] : 0.0; };
  for (int t = 0; t < int(all.size()); ++t) {
    const Tmp& T = all[t];
    int64_t rid = postorder_id(P.level, T.path);
    if (T.depth == dl) {
      Leaf& L = P.leaves[-1 - to_plan[t]];
      L.ref_id = rid;
      L.i0 = T.r.i0;
      L.j0 = T.r.j0;
      L.gperim.assign(kLeafPerim, 0.0);
      L.gpos.assign(kLeafPerim, -1);
      {
        const std::vector<int64_t> per = perimeter(T.r, m);
        for (int a = 0; a < kLeafPerim; ++a)
          if (is_boundary(per[a])) {
            L.gperim[a] = g_of(per[a]);
            L.gpos[a] = bpos_of(per[a]);
          }
      }
      continue;
    }
    UpperNode& U = P.upper[to_plan[t]];
    U.ref_id = rid;
    U.depth = T.depth;
    U.i0 = T.r.i0; U.i1 = T.r.i1; U.j0 = T.r.j0; U.j1 = T.r.j1;
    U.son[0] = to_plan[T.son[0]];
    U.son[1] = to_plan[T.son[1]];
    for (int64_t id : perimeter(T.r, m))
      if (!is_boundary(id)) U.bnd.push_back(id);
    U.gamma = interface_ids(T.r, T.depth, m);
    U.k = int(U.bnd.size());
    U.ng = int(U.gamma.size());
    U.K = U.k + U.ng;
  }
  P.root = dl > 0 ? P.upper_by_depth[0][0] : -1;

  // ---- route observations (functionals.py:146-175) -----------------------
  // owner: ("upper", idx, gpos) | ("leaf", leaf, r, q, gpos) | constant
  struct Birth { int where; int node; int r; int q; int gpos; };   // where: 0 upper, 1 leaf
  std::vector<Birth> births(n_obs, Birth{-1, -1, -1, -1, -1});
  std::vector<int> mean_tmp(n_obs, -1);
  std::vector<int> sub_code(n_obs, 0);      // sub-leaf means: device column code
  P.route.assign(n_obs, ObsRoute{1, -1, 0.0});
  std::map<int64_t, int> tmp_of_refid;
  for (int t = 0; t < int(all.size()); ++t) tmp_of_refid[postorder_id(P.level, all[t].path)] = t;
  for (int o = 0; o < n_obs; ++o) {
    int64_t id = P.obs_id[o];
    if (P.obs_kind[o] == HDD_OBS_POINT) {
      if (id < 0 || id >= m * m) { *code = HDD_ERR_USAGE; return "mesh node " + std::to_string(id) + " not found on any interface"; }
      if (is_boundary(id)) { P.route[o] = ObsRoute{1, -1, g_of(id), bpos_of(id)}; continue; }  // u = g there
      int64_t pi = id % m, pj = id / m;
      int t = 0;
      while (true) {
        const Tmp& T = all[t];
        if (T.depth == dl) {
          // strictly inside this kernel leaf: descend the in-leaf template
          int x = int(pi - T.r.i0), y = int(pj - T.r.j0);
          Rect r{0, kLeafCells, 0, kLeafCells};
          int q = 0;
          for (int lev = 0; lev < kLeafLevels; ++lev) {
            Rect a, b;
            int axis;
            split(r, lev, a, b, &axis);
            if (axis == 0 && x == a.i1 && y > r.j0 && y < r.j1) { births[o] = {1, -1 - to_plan[t], lev, q, y - r.j0 - 1}; break; }
            if (axis == 1 && y == a.j1 && x > r.i0 && x < r.i1) { births[o] = {1, -1 - to_plan[t], lev, q, x - r.i0 - 1}; break; }
            bool second = axis == 0 ? (x > a.i1) : (y > a.j1);
            r = second ? b : a;
            q = 2 * q + (second ? 1 : 0);
          }
          if (births[o].where < 0) { *code = HDD_ERR_USAGE; return "mesh node " + std::to_string(id) + " not found on any interface"; }
          break;
        }
        const UpperNode& U = P.upper[to_plan[t]];
        int gp = find_pos(U.gamma, id);
        if (gp >= 0) { births[o] = {0, to_plan[t], -1, -1, gp}; break; }
        Rect a, b;
        int axis;
        split(T.r, T.depth, a, b, &axis);
        bool second = axis == 0 ? (pi > a.i1) : (pj > a.j1);
        t = T.son[second ? 1 : 0];
      }
    } else if (P.obs_kind[o] == HDD_OBS_MEAN) {
      auto it = tmp_of_refid.find(id);
      if (it == tmp_of_refid.end()) {
        if (id < 0 || id >= subtree_size(P.level, 0)) {
          *code = HDD_ERR_USAGE;
          return "no tree node with id " + std::to_string(id);
        }
        // a node below the kernel-leaf level: locate its cells by descending the
        // post-order numbering, then the kernel leaf that contains them
        Rect r{0, int(P.N), 0, int(P.N)};
        int depth = 0;
        int64_t lo = 0;
        while (lo + subtree_size(P.level, depth) - 1 != id) {
          Rect a, b;
          split(r, depth, a, b, nullptr);
          const int64_t half = subtree_size(P.level, depth + 1);
          if (id < lo + half) r = a;
          else { r = b; lo += half; }
          ++depth;
        }
        int t = 0;
        while (all[t].depth < dl) {
          const Rect& s0 = all[all[t].son[0]].r;
          t = (r.i0 >= s0.i0 && r.i1 <= s0.i1 && r.j0 >= s0.j0 && r.j1 <= s0.j1) ? all[t].son[0] : all[t].son[1];
        }
        const Rect& lr = all[t].r;
        births[o] = {1, -1 - to_plan[t], -1, -1, -1};
        sub_code[o] = submean_code(r.i0 - lr.i0, r.i1 - lr.i0, r.j0 - lr.j0, r.j1 - lr.j0);
        continue;
      }
      mean_tmp[o] = it->second;
    } else {
      return "unknown observation kind " + std::to_string(P.obs_kind[o]);
    }
  }
  // ---- adjoint vs primal (top-down back-solve) ---------------------------
  {
    int n_points = 0;
    for (int o = 0; o < n_obs; ++o) n_points += births[o].where >= 0;
    P.mode = d->mode >= 0 ? d->mode : (n_points > 384 ? 1 : 0);   // measured crossover
    if (d->solve_target >= 0) P.mode = 1;   // the subdomain sweep is a primal top-down
    if (dl == 0) P.mode = 0;     // the root is a kernel leaf: nothing to solve top-down
  }
  const bool primal = P.mode == 1;
  // own-mean flags: every node in the subtree of a requested mean node
  std::vector<char> own_mean(all.size(), 0);
  for (int o = 0; o < n_obs; ++o) {
    if (mean_tmp[o] < 0) continue;
    std::vector<int> st{mean_tmp[o]};
    while (!st.empty()) {
      int t = st.back();
      st.pop_back();
      if (own_mean[t]) continue;
      own_mean[t] = 1;
      if (all[t].son[0] >= 0) { st.push_back(all[t].son[0]); st.push_back(all[t].son[1]); }
    }
  }
  // ---- column plans, bottom-up --------------------------------------------
  // obs -> column at each node (map per tmp node)
  std::vector<std::map<int, int>> colmap(all.size());
  P.leaf_cols = 1;
  for (int t : by_depth[dl]) {
    Leaf& L = P.leaves[-1 - to_plan[t]];
    L.own_mean = own_mean[t];
    L.cols.push_back({COL_LOAD, -1});
    L.birth.insert(L.birth.end(), {-1, -1, -1});
    int mean_col = -1;
    if (L.own_mean) {
      mean_col = int(L.cols.size());
      L.cols.push_back({COL_MEAN, -1});
      L.birth.insert(L.birth.end(), {-1, -1, -1});
    }
    L.fslot.assign(L.cols.size(), -1);
    for (int o = 0; o < n_obs; ++o) {
      if (births[o].where == 1 && births[o].node == -1 - to_plan[t]) {
        const int c = int(L.cols.size());
        if (primal) {
          L.fslot.push_back(P.n_fslots);
          P.route[o] = ObsRoute{2, c, 0.0, -1 - to_plan[t], P.n_fslots};
          ++P.n_fslots;
        } else {
          colmap[t][o] = c;
          L.fslot.push_back(-1);
        }
        if (sub_code[o]) L.cols.push_back({COL_SUBMEAN, o, sub_code[o]});
        else L.cols.push_back({COL_OBS, o});
        L.birth.insert(L.birth.end(), {births[o].r, births[o].q, births[o].gpos});
      }
      if (mean_tmp[o] == t) colmap[t][o] = mean_col;
    }
    for (const Col& c : L.cols)
      L.ccode.push_back(c.kind == COL_LOAD ? 0 : (c.kind == COL_MEAN ? 1 : (c.kind == COL_SUBMEAN ? c.code : 2)));
    P.leaf_cols = std::max(P.leaf_cols, int(L.cols.size()));
  }
  for (int dep = dl - 1; dep >= 0; --dep) {
    for (int t : by_depth[dep]) {
      UpperNode& U = P.upper[to_plan[t]];
      U.own_mean = own_mean[t];
      auto add = [&](Col c, int s1, double c1, int s2, double c2, int birth) {
        U.cols.push_back(c);
        U.csrc.push_back(s1); U.csrc.push_back(s2);
        U.ccoef.push_back(c1); U.ccoef.push_back(c2);
        U.cbirth.push_back(birth);
      };
      int st1 = all[t].son[0], st2 = all[t].son[1];
      add({COL_LOAD, -1}, 0, 1.0, 0, 1.0, -1);
      int mean_col = -1;
      auto son_mean_col = [&](int st) {
        // own mean column of a son: leaf -> 1, upper -> 1 (always right after load)
        (void)st;
        return 1;
      };
      if (U.own_mean) {
        mean_col = int(U.cols.size());
        add({COL_MEAN, -1}, son_mean_col(st1), 0.5, son_mean_col(st2), 0.5, -1);
      }
      for (int si = 0; si < 2; ++si) {
        int st = si == 0 ? st1 : st2;
        for (auto& kv : colmap[st]) {
          int o = kv.first;
          if (mean_tmp[o] == t) continue;   // handled below as alias
          colmap[t][o] = int(U.cols.size());
          if (si == 0) add({COL_OBS, o}, kv.second, 1.0, -1, 0.0, -1);
          else add({COL_OBS, o}, -1, 0.0, kv.second, 1.0, -1);
        }
      }
      for (int o = 0; o < n_obs; ++o) {
        if (births[o].where == 0 && births[o].node == to_plan[t]) {
          if (primal) {
            P.route[o] = ObsRoute{3, births[o].gpos, 0.0, to_plan[t], -1};
          } else {
            colmap[t][o] = int(U.cols.size());
            add({COL_OBS, o}, -1, 0.0, -1, 0.0, births[o].gpos);
          }
        }
        if (mean_tmp[o] == t) colmap[t][o] = mean_col;
      }
      U.nc = int(U.cols.size());
      // gather maps: father index -> son output row
      for (int si = 0; si < 2; ++si) {
        int sp = U.son[si];
        std::vector<int64_t> sset;
        if (sp >= 0) sset = P.upper[sp].bnd;
        else {
          const Leaf& L = P.leaves[-1 - sp];
          sset = perimeter({L.i0, L.i0 + kLeafCells, L.j0, L.j0 + kLeafCells}, m);
        }
        for (int a = 0; a < U.K; ++a) {
          int64_t id = a < U.k ? U.bnd[a] : U.gamma[a - U.k];
          U.gmap.push_back(find_pos(sset, id));
        }
      }
    }
  }
  // root routing
  int root_tmp = 0;   // preorder index 0 is the root
  for (int o = 0; o < n_obs; ++o) {
    if (P.route[o].kind == 1 && births[o].where < 0 && mean_tmp[o] < 0) continue;  // constant
    if (P.route[o].kind >= 2) continue;                                             // primal point
    auto it = colmap[root_tmp].find(o);
    if (it == colmap[root_tmp].end()) { *code = HDD_ERR_USAGE; return "functional was not carried to the root"; }
    P.route[o] = ObsRoute{0, it->second, 0.0};
  }
  P.root_nc = dl > 0 ? P.upper[P.root].nc : int(P.leaves[0].cols.size());

  // ---- low-rank block structure of every large Psi (hdd.py:280-286) -------
  P.lr_eps = d->lr_eps > 0 ? d->lr_eps : 0.0;
  P.lr_kmax = d->lr_kmax > 0 ? d->lr_kmax : 64;
  P.lr_nmin = d->lr_nmin > 0 ? d->lr_nmin : 32;
  if (P.lr_eps > 0) {
    // sketch width k_max + 8: 16 / 24 / 32 columns for k_max <= 24 (compress_kernel),
    // 72 for 25..64 (compress_wide_kernel takes the blocks the narrow sketch cannot decide)
    if (P.lr_kmax > 64)
      return "low-rank rank cap k_max = " + std::to_string(P.lr_kmax) +
             " exceeds the device limit of 64 (sketch width k_max + 8 <= 72)";
    for (UpperNode& U : P.upper) {
      if (U.k <= P.lr_nmin) continue;
      std::vector<double> x(U.k), y(U.k);
      for (int i = 0; i < U.k; ++i) { x[i] = double(U.bnd[i] % m) * P.h; y[i] = double(U.bnd[i] / m) * P.h; }
      std::vector<Cluster> cl;
      std::vector<int32_t> all(U.k);
      for (int i = 0; i < U.k; ++i) all[i] = i;
      const int root = build_cluster(cl, all, x, y, P.lr_nmin);
      std::vector<std::pair<int, int>> blocks;
      collect_blocks(cl, root, root, blocks);
      for (auto& b : blocks) {
        const auto& R = cl[b.first].pos;
        const auto& Cc = cl[b.second].pos;
        // Psi is symmetric: keep one block of each transposed pair, rows = the smaller cluster
        if (*std::min_element(R.begin(), R.end()) > *std::min_element(Cc.begin(), Cc.end())) continue;
        const auto& rr = R.size() <= Cc.size() ? R : Cc;
        const auto& cc = R.size() <= Cc.size() ? Cc : R;
        U.lr_desc.push_back(int32_t(U.lr_rows.size()));
        U.lr_desc.push_back(int32_t(rr.size()));
        U.lr_desc.push_back(int32_t(U.lr_cols.size()));
        U.lr_desc.push_back(int32_t(cc.size()));
        U.lr_rows.insert(U.lr_rows.end(), rr.begin(), rr.end());
        U.lr_cols.insert(U.lr_cols.end(), cc.begin(), cc.end());
      }
    }
  }

  // ---- father links and child-boundary maps (primal top-down) -------------
  for (int u = 0; u < int(P.upper.size()); ++u) {
    UpperNode& U = P.upper[u];
    for (int si = 0; si < 2; ++si) {
      const int sp = U.son[si];
      const int32_t* gm = U.gmap.data() + si * U.K;
      if (sp >= 0) {
        UpperNode& S = P.upper[sp];
        S.parent = u;
        S.cmap.assign(S.k, -1);
        for (int a = 0; a < U.K; ++a)
          if (gm[a] >= 0) S.cmap[gm[a]] = a;
      } else {
        Leaf& L = P.leaves[-1 - sp];
        L.parent = u;
        L.cmap.assign(kLeafPerim, -1);
        for (int a = 0; a < U.K; ++a)
          if (gm[a] >= 0) L.cmap[gm[a]] = a;
      }
    }
  }
  if (primal) {
    // nodes the top-down sweep must visit: the ancestors of every observation's
    // owner (north_star item 4: restricted to what F needs); a full-solution plan
    // (hdd_solve_batch) visits every node
    P.full_solve = d->full_solve != 0;
    std::vector<char> need(P.upper.size(), P.full_solve ? 1 : 0);
    auto mark_up = [&](int u) {
      while (u >= 0 && !need[u]) { need[u] = 1; u = P.upper[u].parent; }
    };
    for (const ObsRoute& r : P.route) {
      if (r.kind == 2) mark_up(P.leaves[r.node].parent);
      else if (r.kind == 3) mark_up(r.node);
    }
    if (d->solve_target >= 0) {
      // solve_subdomain (hdd.py:435-490, SolveMode.keep_path, hdd.py:186-203): the
      // root-to-target path and the target's subtree only — the partial inverse
      int t = 0;
      const Rect tr{P.solve_rect.i0, P.solve_rect.i1, P.solve_rect.j0, P.solve_rect.j1};
      while (all[t].depth < dl && !(all[t].r.i0 == tr.i0 && all[t].r.i1 == tr.i1 && all[t].r.j0 == tr.j0 &&
                                    all[t].r.j1 == tr.j1)) {
        const Rect& s0 = all[all[t].son[0]].r;
        t = (tr.i0 >= s0.i0 && tr.i1 <= s0.i1 && tr.j0 >= s0.j0 && tr.j1 <= s0.j1) ? all[t].son[0] : all[t].son[1];
      }
      std::vector<int> st{t};
      while (!st.empty()) {
        const int q = st.back();
        st.pop_back();
        if (all[q].depth == dl) {
          const int li = -1 - to_plan[q];
          P.solve_leaves.push_back(li);
          mark_up(P.leaves[li].parent);
        } else {
          mark_up(to_plan[q]);
          st.push_back(all[q].son[0]);
          st.push_back(all[q].son[1]);
        }
      }
      std::sort(P.solve_leaves.begin(), P.solve_leaves.end());
    }
    int64_t fo = 0, uo = 0;
    P.td_by_depth.assign(P.upper_by_depth.size(), {});
    for (size_t dep = 0; dep < P.upper_by_depth.size(); ++dep)
      for (int u : P.upper_by_depth[dep]) {
        UpperNode& U = P.upper[u];
        if (!need[u]) { U.fac_off = -1; U.u_off = -1; continue; }
        P.td_by_depth[dep].push_back(u);
        U.fac_off = fo;
        fo += int64_t(U.ng) * (U.k + U.ng + 1);
        U.u_off = uo;
        uo += U.K;
      }
    P.fac_elems = fo;
    P.u_elems = uo;
  }

  // ---- output layouts -----------------------------------------------------
  // node outputs: [Psi lower-packed | R (k x nc) | sigma (nc)]; *_ld is the R row stride
  P.leaf_ld = P.leaf_cols;
  // per-sample blocks padded to an even number of doubles: 16-byte aligned bulk (TMA) copies
  P.leaf_elems = (int64_t(kLeafPerim) * (kLeafPerim + 1) / 2 + int64_t(kLeafPerim) * P.leaf_cols + P.leaf_cols + 1) & ~int64_t(1);
  const bool keep = d->keep_nodes != 0;
  P.n_buffers = keep ? dl + 1 : 2;
  P.buf_elems_per_sample.assign(P.n_buffers, 0);
  P.leaf_buf = keep ? dl : (dl & 1);
  P.buf_elems_per_sample[P.leaf_buf] = int64_t(P.leaves.size()) * P.leaf_elems;
  for (int dep = dl - 1; dep >= 0; --dep) {
    int b = keep ? dep : (dep & 1);
    int64_t acc = 0;
    for (int u : P.upper_by_depth[dep]) {
      UpperNode& U = P.upper[u];
      U.out_ld = U.nc;
      U.out_elems = (int64_t(U.k) * (U.k + 1) / 2 + int64_t(U.k) * U.nc + U.nc + 1) & ~int64_t(1);
      U.buf = b;
      U.out_off = acc;          // scaled by the sub-batch size at allocation
      acc += U.out_elems;
    }
    P.buf_elems_per_sample[b] = std::max(P.buf_elems_per_sample[b], acc);
  }
  *code = HDD_OK;
  return "";
}

}  // namespace hdd
