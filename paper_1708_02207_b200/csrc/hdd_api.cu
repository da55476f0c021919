// C ABI of libhdd_b200.so (see include/hdd.h): plan lifetime, device memory,
// sub-batch scheduling of the kernels, error mapping.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "hdd.h"
#include "hdd_device.h"
#include "hdd_plan.h"

using namespace hdd;

struct HddPlan {
  Plan plan;
  DevPlan dev{};
  int device = -1;
  int bcap = 0;
  cudaStream_t stream = nullptr;
  std::vector<void*> allocs;
  DevUpper* d_upper = nullptr;
  std::vector<DevUpper> h_upper;
  std::vector<size_t> depth_smem;      // merge smem per depth
  std::vector<int> depth_tier;         // 0 = shared-memory panel, 1 = global panel
  std::vector<int64_t> depth_ws;       // panel doubles per (node, sample)
  std::vector<int> depth_rows;         // max k + ngp over the depth's nodes
  std::vector<int> depth_nb;           // elimination block rows (8 or 32)
  std::vector<int> depth_kng;          // max k + 2 ng (top-down smem)
  std::vector<int> lr_blk0, lr_nblk, lr_pmax;   // low-rank blocks per depth (lr_pmax: large blocks)
  std::vector<int> lr_nsmall, lr_pmax_s, lr_qmax_s;   // leading small blocks (one warp each)
  double* ws = nullptr;                // tier-L workspace
  size_t leaf_smem = 0;
  HddError err{};
  // host-API staging
  double* h_Z = nullptr;               // device copies for hdd_forward_batch_host
  double* d_Z = nullptr;
  double* d_S = nullptr;
  double* d_ll = nullptr;
  int64_t io_cap = 0;
  int n_launches = 0;
  // CUDA graph of one forward sub-batch (captured on the plan's stream, replayed on the
  // caller's), keyed by the batch size and the caller's buffers; captured once the same
  // key is seen on two consecutive calls (callers that allocate fresh buffers per call
  // keep the direct launches and never pay a capture)
  cudaGraphExec_t graph = nullptr;
  const double* g_Z = nullptr;
  double* g_S = nullptr;
  double* g_ll = nullptr;
  int g_B = 0;
  bool g_seen = false;
  // asynchronous failure reporting: pinned mirror of the device record
  unsigned long long* h_err = nullptr;
  // pipelined host entry points: copy streams, per-sub-batch events
  cudaStream_t cs_in = nullptr, cs_out = nullptr;
  std::vector<cudaEvent_t> pipe_ev;
  bool io_kappa = false;
  // primal top-down: DevUpper copies of the visited nodes, grouped by depth
  DevUpper* d_td = nullptr;
  std::vector<int> td_first, td_count;
  // tier-L Schur update (schur_l_kernel): one TMA tensor map per tier-L node, grouped
  // by depth in launch order, and the largest tile count of the depth
  std::vector<CUtensorMap> h_tmaps;     // host copies, passed as __grid_constant__ parameters
  std::vector<int> tm_ntiles;           // tile count per map
  std::vector<int> tm_first, tm_tiles;
  std::vector<int> depth_split;         // tier-L depths run split (assemble / eliminate / schur_l)
  // solve_subdomain plans: the target's kernel leaves and the idx_omega position map
  const int32_t* d_solve_leaves = nullptr;
  const int32_t* d_omega_pos = nullptr;
  bool schur_split = false;
};

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

static HddError g_create_err{};
constexpr int kWideSketch = 72;   // compress_wide_kernel sketch columns (kLWW)
static std::mutex g_mu;

static int set_err(HddError* e, int code, const std::string& msg, int sample = -1, int64_t node = -1) {
  e->code = code;
  e->sample = sample;
  e->node_id = node;
  std::snprintf(e->message, sizeof(e->message), "%s", msg.c_str());
  return code;
}

#define CU(call)                                                                            \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return set_err(&pl->err, HDD_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <class T>
static int upload(HddPlan* pl, const std::vector<T>& v, const T** out) {
  if (v.empty()) { *out = nullptr; return 0; }
  void* p = nullptr;
  CU(cudaMalloc(&p, v.size() * sizeof(T)));
  pl->allocs.push_back(p);
  CU(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  *out = static_cast<const T*>(p);
  return 0;
}

// panel row stride: the smallest ld >= w with ld = 8 (mod 16) doubles (conflict-free
// DMMA fragments of 4 rows x 8 columns)
// panel row stride: = 4 (mod 8) doubles, so the DMMA operand fragments (4 rows x 8
// consecutive doubles, one 16-lane half-warp = 4 rows x 4 columns) hit 16 distinct 8-byte
// banks; HDD_PANEL_LD8=1 restores the earlier = 8 (mod 16) stride (A/B hook)
static int panel_ld(int w) {
  static const bool ld8 = std::getenv("HDD_PANEL_LD8") && std::getenv("HDD_PANEL_LD8")[0] == '1';
  return ld8 ? w + ((24 - (w & 15)) & 15) : w + ((12 - (w & 7)) & 7);
}

static int setup_device(HddPlan* pl, int max_batch) {
  Plan& P = pl->plan;
  CU(cudaSetDevice(pl->device));
  CU(cudaStreamCreateWithFlags(&pl->stream, cudaStreamNonBlocking));
  CU(cudaStreamCreateWithFlags(&pl->cs_in, cudaStreamNonBlocking));
  CU(cudaStreamCreateWithFlags(&pl->cs_out, cudaStreamNonBlocking));
  CU(cudaHostAlloc(reinterpret_cast<void**>(&pl->h_err), sizeof(DevError), cudaHostAllocDefault));
  *pl->h_err = kNoError;
  int up_rc;
  {   // per-device leaf tables are built once per process; plans may be created concurrently
    std::lock_guard<std::mutex> lk(g_mu);
    up_rc = upload_leaf_template();
  }
  if (up_rc != 0) return set_err(&pl->err, HDD_ERR_CUDA, "leaf template upload failed");
  DevPlan& D = pl->dev;
  D.N = P.N;
  D.m = P.m;
  D.n_z = P.n_z;
  D.n_obs = int(P.obs_kind.size());
  D.n_leaves = int(P.leaves.size());
  D.leaf_cols = P.leaf_cols;
  D.leaf_ld = P.leaf_ld;
  D.h = P.h;
  D.leaf_elems = P.leaf_elems;
  D.leaf_buf = P.leaf_buf;
  if (P.leaf_cols > kMaxLeafCols)
    return set_err(&pl->err, HDD_ERR_CONFIG,
                   "more than 63 observations strictly inside one 16x16-cell leaf are not supported");
  int rc;
  if ((rc = upload(pl, P.sx, &D.sx))) return rc;
  if ((rc = upload(pl, P.sy, &D.sy))) return rc;
  if ((rc = upload(pl, P.coef, &D.coef))) return rc;
  D.f = nullptr;
  if (!P.f_is_one && (rc = upload(pl, P.f, &D.f))) return rc;
  // leaves
  std::vector<DevLeaf> dl(P.leaves.size());
  for (size_t l = 0; l < P.leaves.size(); ++l) {
    const Leaf& L = P.leaves[l];
    DevLeaf& d = dl[l];
    std::memset(&d, 0, sizeof(d));
    d.i0 = L.i0;
    d.j0 = L.j0;
    d.ncols = int(L.cols.size());
    d.ref_id = L.ref_id;
    for (int c = 0; c < kMaxLeafCols; ++c) {
      d.ctype[c] = 2; d.birth_r[c] = -1; d.birth_q[c] = -1; d.birth_g[c] = -1; d.fslot[c] = -1;
    }
    for (int c = 0; c < d.ncols; ++c) {
      d.ctype[c] = L.ccode[c];
      if (L.ccode[c] >= kSubMeanTag) D.has_submean = 1;
      d.birth_r[c] = L.birth[3 * c];
      d.birth_q[c] = L.birth[3 * c + 1];
      d.birth_g[c] = L.birth[3 * c + 2];
      d.fslot[c] = c < int(L.fslot.size()) ? L.fslot[c] : -1;
    }
    d.parent = L.parent;
  }
  if ((rc = upload(pl, dl, &D.leaves))) return rc;
  D.leaf_g = nullptr;
  if (P.has_g) {
    std::vector<double> lg;
    for (const Leaf& L : P.leaves) lg.insert(lg.end(), L.gperim.begin(), L.gperim.end());
    if ((rc = upload(pl, lg, &D.leaf_g))) return rc;
  }
  {
    std::vector<int32_t> gp;
    for (const Leaf& L : P.leaves) gp.insert(gp.end(), L.gpos.begin(), L.gpos.end());
    if ((rc = upload(pl, gp, &D.leaf_gpos))) return rc;
    D.gcall = nullptr;
    D.f_stride = 0;
    D.g_stride = 0;
  }
  {
    std::vector<int32_t> lc;
    for (const Leaf& L : P.leaves) {
      if (L.cmap.empty()) lc.insert(lc.end(), kLeafPerim, -1);
      else lc.insert(lc.end(), L.cmap.begin(), L.cmap.end());
    }
    if ((rc = upload(pl, lc, &D.leaf_cmap))) return rc;
  }
  {
    std::vector<int32_t> order;
    for (int cls = 0; cls < 3; ++cls) {
      D.leaf_class_start[cls] = int(order.size());
      const int lo = cls == 0 ? 0 : (cls == 1 ? 3 : 5), hi = cls == 0 ? 2 : (cls == 1 ? 4 : kMaxLeafCols);
      D.leaf_class_passes[cls] = 1;
      for (size_t l = 0; l < P.leaves.size(); ++l) {
        int nc = int(P.leaves[l].cols.size());
        if (nc >= lo && nc <= hi) {
          order.push_back(int32_t(l));
          if (cls == 2) D.leaf_class_passes[cls] = std::max(D.leaf_class_passes[cls], nc <= 8 ? 1 : (nc - 1 + 6) / 7);
        }
      }
      D.leaf_class_count[cls] = int(order.size()) - D.leaf_class_start[cls];
    }
    if ((rc = upload(pl, order, &D.leaf_order))) return rc;
  }
  // upper nodes
  std::vector<int32_t> gmap, csrc, cbirth, cmapool;
  std::vector<double> ccoef;
  pl->depth_kng.assign(P.upper_by_depth.size(), 0);
  pl->h_upper.resize(P.upper.size());
  pl->depth_smem.assign(P.upper_by_depth.size(), 0);
  pl->depth_tier.assign(P.upper_by_depth.size(), 0);
  pl->depth_ws.assign(P.upper_by_depth.size(), 0);
  pl->depth_rows.assign(P.upper_by_depth.size(), 0);
  pl->depth_nb.assign(P.upper_by_depth.size(), 32);
  const char* force_l = std::getenv("HDD_FORCE_TIER_L");   // test hook: every depth on the HBM panel
  // panels above this many KB of shared memory run on the HBM-panel tier (tuning hook)
  const int tier_l_kb = std::getenv("HDD_TIER_L_KB") ? std::atoi(std::getenv("HDD_TIER_L_KB")) : 220;
  for (size_t u = 0; u < P.upper.size(); ++u) {
    const UpperNode& U = P.upper[u];
    const int ngp32 = (U.ng + 31) / 32 * 32;
    const int ldp32 = panel_ld(U.k + ngp32 + U.nc);
    if (merge_m2_smem_bytes(ngp32, ldp32, U.K, U.nc) > size_t(tier_l_kb) * 1024 || (force_l && force_l[0] == '1'))
      pl->depth_tier[U.depth] = 1;
  }
  for (size_t u = 0; u < P.upper.size(); ++u) {
    const UpperNode& U = P.upper[u];
    const int nbk = pl->depth_tier[U.depth] ? 32 : 8;
    const int ngp = (U.ng + nbk - 1) / nbk * nbk;
    const int ldp = panel_ld(U.k + ngp + U.nc);
    pl->depth_nb[U.depth] = nbk;
    if (pl->depth_tier[U.depth]) pl->depth_ws[U.depth] = std::max<int64_t>(pl->depth_ws[U.depth], int64_t(ngp) * ldp);
    pl->depth_rows[U.depth] = std::max(pl->depth_rows[U.depth], U.k + ngp);
  }
  for (size_t u = 0; u < P.upper.size(); ++u) {
    const UpperNode& U = P.upper[u];
    DevUpper& d = pl->h_upper[u];
    std::memset(&d, 0, sizeof(d));
    d.k = U.k; d.ng = U.ng; d.K = U.K; d.nc = U.nc;
    const int nbk = pl->depth_nb[U.depth];
    const int ngp_u = (U.ng + nbk - 1) / nbk * nbk;
    d.ldp = panel_ld(U.k + ngp_u + U.nc);
    d.nb = nbk;
    d.out_ld = U.out_ld;
    d.out_elems = U.out_elems;
    d.out_off = U.out_off;
    d.buf = U.buf;
    d.ref_id = U.ref_id;
    for (int sn = 0; sn < 2; ++sn) {
      int s = U.son[sn];
      if (s >= 0) {
        const UpperNode& S = P.upper[s];
        d.son_buf[sn] = S.buf;
        d.son_k[sn] = S.k;
        d.son_ld[sn] = S.out_ld;
        d.son_elems[sn] = S.out_elems;
        d.son_off[sn] = S.out_off;
      } else {
        int l = -1 - s;
        d.son_buf[sn] = P.leaf_buf;
        d.son_k[sn] = kLeafPerim;
        d.son_ld[sn] = P.leaf_ld;
        d.son_elems[sn] = P.leaf_elems;
        d.son_off[sn] = int64_t(l) * P.leaf_elems;
      }
    }
    {   // boundary nodes held by both sons: the two ends of the interface (fewer when an
        // end lies on the domain boundary); their pairs get both sons' Psi entries
      d.sh[0] = d.sh[1] = -1;
      int nsh = 0;
      for (int a = 0; a < U.k; ++a)
        if (U.gmap[a] >= 0 && U.gmap[U.K + a] >= 0) {
          if (nsh >= 2) return set_err(&pl->err, HDD_ERR_CONFIG, "more than two boundary nodes shared by both sons");
          d.sh[nsh++] = a;
        }
    }
    d.gmap_off = int(gmap.size());
    gmap.insert(gmap.end(), U.gmap.begin(), U.gmap.end());
    d.parent = U.parent;
    d.cmap_off = int(cmapool.size());
    cmapool.insert(cmapool.end(), U.cmap.begin(), U.cmap.end());
    d.fac_off = U.fac_off;
    d.u_off = U.u_off;
    pl->depth_kng[U.depth] = std::max(pl->depth_kng[U.depth], U.k + 2 * U.ng);
    d.col_off = int(cbirth.size());
    csrc.insert(csrc.end(), U.csrc.begin(), U.csrc.end());
    ccoef.insert(ccoef.end(), U.ccoef.begin(), U.ccoef.end());
    cbirth.insert(cbirth.end(), U.cbirth.begin(), U.cbirth.end());
    size_t sm = pl->depth_tier[U.depth] ? merge_l_smem_bytes(U.K, U.nc) : merge_m2_smem_bytes(ngp_u, d.ldp, U.K, U.nc);
    if (!pl->depth_tier[U.depth]) {
      // stage the sons in smem when panel + sons still allow two CTAs per SM
      const size_t sons = sizeof(double) * size_t(((d.son_elems[0] + 1) & ~1) + ((d.son_elems[1] + 1) & ~1));
      // measured: pays off only on the first merge level (sons = kernel leaves)
      d.stage = (U.son[0] < 0 && U.son[1] < 0 && sm + sons <= 110 * 1024) ? 1 : 0;
#ifdef HDD_NO_STAGE
      d.stage = 0;
#endif
      if (d.stage) sm += sons;
    }
    pl->depth_smem[U.depth] = std::max(pl->depth_smem[U.depth], sm);
  }
  if ((rc = upload(pl, gmap, &D.gmap))) return rc;
  if ((rc = upload(pl, csrc, &D.csrc))) return rc;
  if ((rc = upload(pl, ccoef, &D.ccoef))) return rc;
  if ((rc = upload(pl, cbirth, &D.cbirth))) return rc;
  if ((rc = upload(pl, cmapool, &D.cmap))) return rc;
  // low-rank block lists, grouped by depth (node index local to the depth launch)
  D.lr_eps = P.lr_eps;
  D.lr_kmax = P.lr_kmax;
  D.lr_l = std::min(32, P.lr_kmax + 8);
  pl->lr_blk0.assign(P.upper_by_depth.size(), 0);
  pl->lr_nblk.assign(P.upper_by_depth.size(), 0);
  pl->lr_pmax.assign(P.upper_by_depth.size(), 0);
  pl->lr_nsmall.assign(P.upper_by_depth.size(), 0);
  pl->lr_pmax_s.assign(P.upper_by_depth.size(), 0);
  pl->lr_qmax_s.assign(P.upper_by_depth.size(), 0);
  // HDD_LR_NO_WARP=1: every block on the CTA kernel (A/B hook)
  const bool no_warp = std::getenv("HDD_LR_NO_WARP") && std::getenv("HDD_LR_NO_WARP")[0] == '1';
  int lr_qmax = 0;
  int lr_nodes_max = 0;
  if (P.lr_eps > 0) {
    std::vector<int32_t> rows, cols, blk;
    for (size_t dep = 0; dep < P.upper_by_depth.size(); ++dep) {
      const auto& ids = P.upper_by_depth[dep];
      lr_nodes_max = std::max(lr_nodes_max, int(ids.size()));
      pl->lr_blk0[dep] = int(blk.size() / 5);
      // small blocks (p, q <= 64: one warp each, compress_warp_kernel) first, then the
      // large ones (one CTA each, compress_kernel)
      for (int pass_small = 1; pass_small >= 0; --pass_small) {
        for (size_t li = 0; li < ids.size(); ++li) {
          const UpperNode& U = P.upper[ids[li]];
          for (size_t b = 0; b + 3 < U.lr_desc.size(); b += 4) {
            const int pb = U.lr_desc[b + 1], qb = U.lr_desc[b + 3];
            const bool small = pb <= 64 && qb <= 64 && !no_warp;
            if (small != bool(pass_small)) continue;
            blk.push_back(int32_t(li));
            blk.push_back(int32_t(rows.size()));
            blk.push_back(pb);
            blk.push_back(int32_t(cols.size()));
            blk.push_back(qb);
            rows.insert(rows.end(), U.lr_rows.begin() + U.lr_desc[b], U.lr_rows.begin() + U.lr_desc[b] + pb);
            cols.insert(cols.end(), U.lr_cols.begin() + U.lr_desc[b + 2], U.lr_cols.begin() + U.lr_desc[b + 2] + qb);
            if (small) {
              pl->lr_pmax_s[dep] = std::max(pl->lr_pmax_s[dep], pb);
              pl->lr_qmax_s[dep] = std::max(pl->lr_qmax_s[dep], qb);
            } else {
              pl->lr_pmax[dep] = std::max(pl->lr_pmax[dep], pb);
            }
            lr_qmax = std::max(lr_qmax, qb);
          }
        }
        if (pass_small) pl->lr_nsmall[dep] = int(blk.size() / 5) - pl->lr_blk0[dep];
      }
      pl->lr_nblk[dep] = int(blk.size() / 5) - pl->lr_blk0[dep];
      if (std::getenv("HDD_LR_STATS")) {   // diagnostics: admissible blocks per depth
        long long area = 0, small = 0;
        int qm = 0;
        for (size_t t = size_t(pl->lr_blk0[dep]) * 5; t < blk.size(); t += 5) {
          area += (long long)blk[t + 2] * blk[t + 4];
          small += (blk[t + 2] <= 64 && blk[t + 4] <= 64);
          qm = std::max(qm, int(blk[t + 4]));
        }
        std::fprintf(stderr, "lr depth %zu: nodes %zu blocks %d (<=64x64: %lld) pmax %d qmax %d area %lld\n", dep,
                     ids.size(), pl->lr_nblk[dep], small, pl->lr_pmax[dep], qm, area);
      }
      if (pl->lr_pmax[dep] > 760)
        return set_err(&pl->err, HDD_ERR_CONFIG, "low-rank block with more than 760 rows does not fit the device sketch");
    }
    if ((rc = upload(pl, rows, &D.lr_rows))) return rc;
    if ((rc = upload(pl, cols, &D.lr_cols))) return rc;
    if ((rc = upload(pl, blk, &D.lr_blk))) return rc;
    // fixed Gaussian test matrix (deterministic: splitmix64 + Box-Muller)
    std::vector<double> om(size_t(std::max(lr_qmax, 1)) * 32);
    uint64_t st = 0x9E3779B97F4A7C15ull;
    auto next = [&]() {
      st += 0x9E3779B97F4A7C15ull;
      uint64_t z = st;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      return double((z ^ (z >> 31)) >> 11) * (1.0 / 9007199254740992.0);
    };
    for (size_t i = 0; i < om.size(); i += 2) {
      const double u1 = std::max(next(), 1e-300), u2 = next();
      const double rr = std::sqrt(-2.0 * std::log(u1));
      om[i] = rr * std::cos(2.0 * M_PI * u2);
      if (i + 1 < om.size()) om[i + 1] = rr * std::sin(2.0 * M_PI * u2);
    }
    if ((rc = upload(pl, om, &D.lr_omega))) return rc;
    D.lr_pmax = 0;
    for (size_t dep = 0; dep < pl->lr_pmax.size(); ++dep)    // wide scratch rows: any queued block
      D.lr_pmax = std::max(D.lr_pmax, std::max(pl->lr_pmax[dep], pl->lr_pmax_s[dep]));
    D.lr_qmax = std::max(lr_qmax, 1);
    if (P.lr_kmax > 24) {
      std::vector<double> omw(size_t(D.lr_qmax) * kWideSketch);
      for (size_t i = 0; i < omw.size(); i += 2) {
        const double u1 = std::max(next(), 1e-300), u2 = next();
        const double rr = std::sqrt(-2.0 * std::log(u1));
        omw[i] = rr * std::cos(2.0 * M_PI * u2);
        if (i + 1 < omw.size()) omw[i + 1] = rr * std::sin(2.0 * M_PI * u2);
      }
      if ((rc = upload(pl, omw, &D.lr_omega_w))) return rc;
    }
  }
  {
    const DevUpper* du = nullptr;
    if ((rc = upload(pl, pl->h_upper, &du))) return rc;
    pl->d_upper = const_cast<DevUpper*>(du);
    D.upper = du;
  }
  pl->td_first.assign(P.upper_by_depth.size(), -1);
  pl->td_count.assign(P.upper_by_depth.size(), 0);
  if (P.mode == 1) {
    std::vector<DevUpper> td;
    for (size_t dep = 0; dep < P.td_by_depth.size(); ++dep) {
      if (P.td_by_depth[dep].empty()) continue;
      pl->td_first[dep] = int(td.size());
      pl->td_count[dep] = int(P.td_by_depth[dep].size());
      for (int u : P.td_by_depth[dep]) td.push_back(pl->h_upper[u]);
    }
    const DevUpper* dt = nullptr;
    if ((rc = upload(pl, td, &dt))) return rc;
    pl->d_td = const_cast<DevUpper*>(dt);
  }
  if (P.solve_target >= 0) {
    if ((rc = upload(pl, P.solve_leaves, &pl->d_solve_leaves))) return rc;
    if ((rc = upload(pl, P.omega_pos, &pl->d_omega_pos))) return rc;
  }
  D.tiny = P.tiny ? 1 : 0;
  D.root_ref = P.root_ref;
  D.gfull = nullptr;
  if (P.tiny && P.has_g && (rc = upload(pl, P.gfull, &D.gfull))) return rc;
  // observations
  std::vector<int32_t> rk, rcol, rnode, rslot;
  std::vector<double> rv;
  double llc = 0.0;
  for (size_t o = 0; o < P.route.size(); ++o) {
    rk.push_back(P.route[o].kind);
    rcol.push_back(P.route[o].col);
    rv.push_back(P.route[o].value);
    rnode.push_back(P.route[o].node);
    rslot.push_back(P.route[o].slot);
    llc += std::log(P.sigma[o] * std::sqrt(2.0 * M_PI));
  }
  D.ll_const = llc;
  if ((rc = upload(pl, rk, &D.route_kind))) return rc;
  if ((rc = upload(pl, rcol, &D.route_col))) return rc;
  if ((rc = upload(pl, rv, &D.route_val))) return rc;
  if ((rc = upload(pl, rnode, &D.route_node))) return rc;
  if ((rc = upload(pl, rslot, &D.route_slot))) return rc;
  D.mode = P.mode;
  D.fac_elems = P.fac_elems;
  D.u_elems = P.u_elems;
  D.n_fslots = P.n_fslots;
  if ((rc = upload(pl, P.sigma, &D.sigma))) return rc;
  D.y = nullptr;
  if (P.has_y && (rc = upload(pl, P.y, &D.y))) return rc;
  // buffers: size the sub-batch
  int64_t per_sample = int64_t(2) * P.N * P.N;
  for (int64_t e : P.buf_elems_per_sample) per_sample += e;
  int64_t ws_per_sample = 0;
  for (size_t d = 0; d < P.upper_by_depth.size(); ++d)
    ws_per_sample = std::max<int64_t>(ws_per_sample, pl->depth_ws[d] * int64_t(P.upper_by_depth[d].size()));
  per_sample += ws_per_sample;
  per_sample += P.fac_elems + P.u_elems + int64_t(P.n_fslots) * 65;
  int64_t bytes_per_sample = per_sample * 8;
  int bcap = max_batch;
  if (bcap <= 0) {
    size_t freeb = 0, totb = 0;
    CU(cudaMemGetInfo(&freeb, &totb));
    int64_t budget = int64_t(double(freeb) * 0.6);
    bcap = int(std::min<int64_t>(4096, std::max<int64_t>(1, budget / bytes_per_sample)));
  }
  pl->bcap = bcap;
  D.bcap = bcap;
  for (int b = 0; b < kMaxBuffers; ++b) D.buf[b] = nullptr;
  if (P.n_buffers > kMaxBuffers) return set_err(&pl->err, HDD_ERR_CONFIG, "tree too deep for debug buffers");
  for (int b = 0; b < P.n_buffers; ++b) {
    void* p = nullptr;
    size_t nb = size_t(P.buf_elems_per_sample[b]) * bcap * sizeof(double);
    if (nb == 0) continue;
    if (cudaMalloc(&p, nb) != cudaSuccess) {
      cudaGetLastError();
      return set_err(&pl->err, HDD_ERR_NOMEM, "device allocation of " + std::to_string(nb) + " bytes failed");
    }
    pl->allocs.push_back(p);
    D.buf[b] = static_cast<double*>(p);
  }
  D.lr_scale = nullptr;
  D.lr_wide_list = nullptr;
  D.lr_wide_n = nullptr;
  D.lr_wide_scr = nullptr;
  D.lr_wide_cap = 0;
  D.lr_wide_ctas = 0;
  D.lr_force_wide = (std::getenv("HDD_LR_FORCE_WIDE") && std::getenv("HDD_LR_FORCE_WIDE")[0] == '1') ? 1 : 0;
  if (P.lr_eps > 0) {
    void* q = nullptr;
    CU(cudaMalloc(&q, sizeof(double) * size_t(std::max(lr_nodes_max, 1)) * bcap));
    pl->allocs.push_back(q);
    D.lr_scale = static_cast<double*>(q);
    if (P.lr_kmax > 24) {
      int nb_max = 1;
      for (int v : pl->lr_nblk) nb_max = std::max(nb_max, v);
      D.lr_wide_cap = int(std::min<int64_t>(int64_t(nb_max) * bcap, 1 << 26));
      D.lr_wide_ctas = 2 * 148;
      D.lr_wide_stride = (int64_t(std::max(D.lr_pmax, 1)) * kWideSketch + int64_t(kWideSketch) * D.lr_qmax + 1) & ~int64_t(1);
      CU(cudaMalloc(&q, sizeof(int2) * size_t(D.lr_wide_cap)));
      pl->allocs.push_back(q);
      D.lr_wide_list = static_cast<int2*>(q);
      CU(cudaMalloc(&q, 2 * sizeof(int)));    // [0] per-depth queue length, [1] running total
      pl->allocs.push_back(q);
      D.lr_wide_n = static_cast<int*>(q);
      CU(cudaMemset(q, 0, 2 * sizeof(int)));
      CU(cudaMalloc(&q, sizeof(double) * size_t(D.lr_wide_ctas) * D.lr_wide_stride));
      pl->allocs.push_back(q);
      D.lr_wide_scr = static_cast<double*>(q);
    }
  }
  D.fac = D.ubuf = D.fbuf = nullptr;
  for (auto pr : {std::make_pair(&D.fac, P.fac_elems), std::make_pair(&D.ubuf, P.u_elems),
                  std::make_pair(&D.fbuf, int64_t(P.n_fslots) * 65)}) {
    if (pr.second <= 0) continue;
    void* q = nullptr;
    if (cudaMalloc(&q, size_t(pr.second) * bcap * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      return set_err(&pl->err, HDD_ERR_NOMEM, "device allocation of the top-down buffers failed");
    }
    pl->allocs.push_back(q);
    *pr.first = static_cast<double*>(q);
  }
  if (ws_per_sample > 0) {
    void* p = nullptr;
    if (cudaMalloc(&p, size_t(ws_per_sample) * bcap * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      return set_err(&pl->err, HDD_ERR_NOMEM, "device allocation of the merge workspace failed");
    }
    pl->allocs.push_back(p);
    pl->ws = static_cast<double*>(p);
  }
  // tier-L Schur update kernel: tensor maps over each tier-L node's panel slice
  // [bcap][ngp][ldp] of the workspace
  {
    // split tier L (assemble / eliminate / TMA Schur update) on the depths whose
    // interface is deep enough (ng >= 255 by default, HDD_SCHUR_L_MIN_NG): measured
    // C4 d2 34.6 -> 33.3 ms, C5 d2 120.1 -> 104.8 ms, d1 71.4 -> 60.1 ms per batch;
    // shallower interfaces keep the fused kernel.  HDD_SCHUR_L_SPLIT=0: off
    const char* sv = std::getenv("HDD_SCHUR_L_SPLIT");
    pl->schur_split = !(sv && sv[0] == '0');
    pl->tm_first.assign(P.upper_by_depth.size(), -1);
    pl->tm_tiles.assign(P.upper_by_depth.size(), 0);
    std::vector<CUtensorMap> maps;
    auto enc = tensor_map_encoder();
    if (!enc) pl->schur_split = false;
    for (size_t dep = 0; dep < P.upper_by_depth.size() && pl->schur_split; ++dep) {
      if (!pl->depth_tier[dep]) continue;
      const auto& ids = P.upper_by_depth[dep];
      pl->tm_first[dep] = int(maps.size());
      for (size_t li = 0; li < ids.size(); ++li) {
        const DevUpper& d = pl->h_upper[ids[li]];
        const int ngp = (d.ng + d.nb - 1) / d.nb * d.nb;
        CUtensorMap m;
        std::memset(&m, 0, sizeof(m));
        void* base = pl->ws + int64_t(li) * pl->depth_ws[dep] * bcap;
        const cuuint64_t dims[3] = {cuuint64_t(d.ldp), cuuint64_t(ngp), cuuint64_t(bcap)};
        const cuuint64_t strides[2] = {cuuint64_t(d.ldp) * 8, cuuint64_t(pl->depth_ws[dep]) * 8};
        const cuuint32_t box[3] = {8, cuuint32_t(schur_l_box_rows()), 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS)
          return set_err(&pl->err, HDD_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
        if (std::getenv("HDD_SCHUR_L_DEBUG"))
          std::fprintf(stderr, "tmap dep %zu node %zu: base %p ldp %d ngp %d bcap %d stride2 %lld k %d nc %d tiles %d\n",
                       dep, li, base, d.ldp, ngp, bcap, (long long)pl->depth_ws[dep], d.k, d.nc,
                       schur_l_tiles(d.k, d.nc, ngp));
        maps.push_back(m);
        pl->tm_ntiles.push_back(schur_l_tiles(d.k, d.nc, ngp));
        pl->tm_tiles[dep] = std::max(pl->tm_tiles[dep], schur_l_tiles(d.k, d.nc, ngp));
      }
    }
    if (maps.empty()) pl->schur_split = false;
    pl->h_tmaps = std::move(maps);
    // split only where the interface is deep enough for the GEMM to amortise its
    // pipeline and the extra A~ round trip through HBM (HDD_SCHUR_L_MIN_NG, default 256)
    const int min_ng = std::getenv("HDD_SCHUR_L_MIN_NG") ? std::atoi(std::getenv("HDD_SCHUR_L_MIN_NG")) : 256;
    pl->depth_split.assign(P.upper_by_depth.size(), 0);
    for (size_t dep = 0; dep < P.upper_by_depth.size(); ++dep) {
      int ngmin = 1 << 30;
      for (int u : P.upper_by_depth[dep]) ngmin = std::min(ngmin, P.upper[u].ng);
      pl->depth_split[dep] = pl->schur_split && pl->depth_tier[dep] && ngmin >= min_ng - 1;
    }
    D.schur_split = pl->schur_split ? 1 : 0;
  }
  {
    void* p = nullptr;
    CU(cudaMalloc(&p, size_t(2) * P.N * P.N * bcap * sizeof(double)));
    pl->allocs.push_back(p);
    D.kappa = static_cast<double*>(p);
    CU(cudaMalloc(&p, sizeof(DevError)));
    pl->allocs.push_back(p);
    D.err = static_cast<DevError*>(p);
    CU(cudaMemset(p, 0xff, sizeof(DevError)));     // kNoError
  }
  if (P.root >= 0) {
    const UpperNode& R = P.upper[P.root];
    D.root_buf = R.buf;
    D.root_off = R.out_off * bcap;
    D.root_elems = R.out_elems;
    D.root_sig = int64_t(R.k) * (R.k + 1) / 2 + int64_t(R.k) * R.nc;
  } else {
    D.root_buf = P.leaf_buf;
    D.root_off = 0;
    D.root_elems = P.leaf_elems;
    D.root_sig = int64_t(kLeafPerim) * (kLeafPerim + 1) / 2 + int64_t(kLeafPerim) * P.leaf_cols;
  }
  pl->leaf_smem = leaf_smem_bytes(P.leaf_cols <= 2 ? 2 : (P.leaf_cols <= 4 ? 4 : 8));
  {
    // kernels one forward sub-batch launches (run_sub_batch): kappa, one leaf launch per
    // column class, per depth one merge (+ psi_norm and compress with low-rank blocks),
    // per depth one top-down solve in primal mode, finalize
    int ncls = 0;
    for (int c = 0; c < 3; ++c) ncls += D.leaf_class_count[c] > 0;
    int n = 2 + ncls;
    for (size_t dep = 0; dep < P.upper_by_depth.size(); ++dep) {
      if (P.upper_by_depth[dep].empty()) continue;
      n += 1 + (D.mode == 1 && pl->td_count[dep] > 0 ? 1 : 0);
      if (pl->depth_tier[dep] && D.schur_split && pl->depth_split[dep]) {
        n += 1;                                             // assemble_l
        for (size_t li = 0; li < P.upper_by_depth[dep].size(); ++li) n += pl->tm_ntiles[pl->tm_first[dep] + li] > 0;
      }
      if (D.lr_eps > 0 && dep > 0 && pl->lr_nblk[dep] > 0)
        n += 1 + (pl->lr_nblk[dep] > pl->lr_nsmall[dep]) + (pl->lr_nsmall[dep] > 0) + (D.lr_wide_list ? 1 : 0);
    }
    pl->n_launches = n;
  }
  return HDD_OK;
}

extern "C" {

int hdd_debug_leaf_clocks(long long* out) { return read_leaf_clocks(out); }
int hdd_debug_merge_clocks(long long* out) { return read_merge_clocks(out); }

const char* hdd_version(void) { return "hdd_b200 0.1 (sm_100a)"; }

int hdd_plan_stage_kernel(const HddPlan* pl, int32_t depth, int32_t B, char* buf, int32_t cap) {
  if (!pl || !buf || cap <= 0 || pl->device < 0) return HDD_ERR_USAGE;
  const Plan& P = pl->plan;
  std::string name;
  if (depth < 0) {
    if (P.tiny) name = "tiny_kernel";
    else {
      const bool sub = pl->dev.has_submean || pl->dev.leaf_g;
      for (int c = 0; c < 3; ++c)
        if (pl->dev.leaf_class_count[c] > 0)
          name += std::string(name.empty() ? "" : "+") + "leaf2_kernel<" + (c == 0 ? "2" : (c == 1 ? "4" : "8")) +
                  ",256," + (sub ? "true" : "false") + ">";
    }
  } else {
    if (depth >= int(P.upper_by_depth.size()) || P.upper_by_depth[depth].empty()) return HDD_ERR_USAGE;
    DevPlan Dd = pl->dev;
    Dd.schur_split = (pl->depth_tier[depth] && pl->dev.schur_split && pl->depth_split[depth]) ? 1 : 0;
    const int v = merge_variant(Dd, int(P.upper_by_depth[depth].size()), B, pl->depth_tier[depth],
                                pl->depth_smem[depth], depth);
    name = merge_variant_name(v);
    if (Dd.schur_split) {
      name = "assemble_l_kernel+" + name;
      if (pl->tm_tiles[depth] > 0) name += "+schur_l_kernel";
    }
  }
  std::snprintf(buf, size_t(cap), "%s", name.c_str());
  return HDD_OK;
}

int hdd_create_error(HddError* out) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (out) *out = g_create_err;
  return HDD_OK;
}

int hdd_plan_create(const HddPlanDesc* desc, HddPlan** out) {
  if (!out) return HDD_ERR_USAGE;
  *out = nullptr;
  HddPlan* pl = new HddPlan();
  int code = HDD_OK;
  std::string msg = build_plan(desc, pl->plan, &code);
  if (code != HDD_OK) {
    std::lock_guard<std::mutex> lk(g_mu);
    set_err(&g_create_err, code, msg);
    delete pl;
    return code;
  }
  pl->device = desc->device;
  if (pl->device >= 0) {
    int rc = setup_device(pl, desc->max_batch);
    if (rc != HDD_OK) {
      std::lock_guard<std::mutex> lk(g_mu);
      g_create_err = pl->err;
      hdd_plan_destroy(pl);
      return rc;
    }
  }
  *out = pl;
  return HDD_OK;
}

int hdd_plan_destroy(HddPlan* pl) {
  if (!pl) return HDD_OK;
  if (pl->device >= 0) {
    cudaSetDevice(pl->device);
    cudaDeviceSynchronize();
    for (void* p : pl->allocs) cudaFree(p);
    if (pl->d_Z) cudaFree(pl->d_Z);
    if (pl->d_S) cudaFree(pl->d_S);
    if (pl->d_ll) cudaFree(pl->d_ll);
    if (pl->graph) cudaGraphExecDestroy(pl->graph);
    for (cudaEvent_t e : pl->pipe_ev) cudaEventDestroy(e);
    if (pl->cs_in) cudaStreamDestroy(pl->cs_in);
    if (pl->cs_out) cudaStreamDestroy(pl->cs_out);
    if (pl->h_err) cudaFreeHost(pl->h_err);
    if (pl->stream) cudaStreamDestroy(pl->stream);
  }
  delete pl;
  return HDD_OK;
}

// One sub-batch through the whole launch sequence.  Z (n_z per row) or, when Kin is
// given, caller-supplied coefficient fields Kin [B][2N^2] (K1 replaced by a check
// kernel); U non-NULL: the full-solution path (primal sweep + in-leaf solves).
// sample0 = global index of the sub-batch's first row (failure records).
static int run_sub_batch(HddPlan* pl, const double* Z, const double* Kin, int B, double* S, double* ll, double* U,
                         cudaStream_t st, int64_t sample0, cudaEvent_t* ev = nullptr, const HddRhs* rhs = nullptr,
                         bool sub = false) {
  Plan& P = pl->plan;
  DevPlan D = pl->dev;                 // by-value copy: per-sub-batch fields
  D.sample0 = sample0;
  if (Kin) D.kappa = const_cast<double*>(Kin);
  if (rhs && rhs->f) {                 // per-call rows (base pointers of the call, offset here)
    D.f = rhs->f + sample0 * rhs->f_stride;
    D.f_stride = rhs->f_stride;
  }
  if (rhs && rhs->g) {
    D.gcall = rhs->g + sample0 * rhs->g_stride;
    D.g_stride = rhs->g_stride;
  }
  const int64_t nn = int64_t(P.m) * P.m;
  int e = 0;
  auto mark = [&]() -> int {
    if (ev) CU(cudaEventRecord(ev[e++], st));
    return HDD_OK;
  };
  int rc;
  if ((rc = mark())) return rc;
  if (Kin) CU(launch_kappa_check(D, Kin, B, st));
  else CU(launch_kappa(D, Z, B, D.kappa, st));
  if ((rc = mark())) return rc;
  if (P.tiny) {
    CU(launch_tiny(D, B, S, ll, U, nn, st));
    if ((rc = mark())) return rc;
    return mark();                     // empty finalize stage
  }
  CU(launch_leaf(D, B, st, nullptr));
  if ((rc = mark())) return rc;
  for (int dep = int(P.upper_by_depth.size()) - 1; dep >= 0; --dep) {
    const auto& ids = P.upper_by_depth[dep];
    if (!ids.empty()) {
      // split tier L (opt-in per depth): assemble -> eliminate -> TMA Schur update
      DevPlan Dd = D;
      Dd.schur_split = (pl->depth_tier[dep] && D.schur_split && pl->depth_split[dep]) ? 1 : 0;
      if (Dd.schur_split)
        CU(launch_assemble_l(Dd, pl->d_upper + ids.front(), int(ids.size()), B, pl->ws, pl->depth_ws[dep],
                             pl->depth_rows[dep], st));
      CU(launch_merge(Dd, pl->d_upper + ids.front(), int(ids.size()), B, pl->ws, pl->depth_ws[dep],
                      pl->depth_tier[dep], pl->depth_rows[dep], pl->depth_smem[dep], pl->depth_nb[dep], st, dep));
      if (Dd.schur_split && pl->tm_tiles[dep] > 0)   // the root (k = 0) has no update
        CU(launch_schur_l(Dd, pl->d_upper + ids.front(), pl->h_tmaps.data() + pl->tm_first[dep],
                          pl->tm_ntiles.data() + pl->tm_first[dep], int(ids.size()), B, st));
      if (D.lr_eps > 0 && dep > 0 && pl->lr_nblk[dep] > 0) {
        if (D.lr_wide_list) CU(cudaMemsetAsync(D.lr_wide_n, 0, sizeof(int), st));
        const int ns = pl->lr_nsmall[dep];
        // psi norms, then the large blocks (CTA each), then the small ones (warp each)
        CU(launch_compress(D, pl->d_upper + ids.front(), int(ids.size()), pl->lr_blk0[dep] + ns,
                           pl->lr_nblk[dep] - ns, B, pl->lr_pmax[dep], st));
        CU(launch_compress_warp(D, pl->d_upper + ids.front(), pl->lr_blk0[dep], ns, B, pl->lr_pmax_s[dep],
                                pl->lr_qmax_s[dep], st));
        if (D.lr_wide_list) CU(launch_compress_wide(D, pl->d_upper + ids.front(), st));
      }
    }
    if ((rc = mark())) return rc;
  }
  if (D.mode == 1) {
    // only the nodes on root-to-observation paths (every node in a full-solution plan)
    for (int dep = 0; dep < int(P.upper_by_depth.size()); ++dep)
      if (pl->td_count[dep] > 0)
        CU(launch_topdown(D, pl->d_td + pl->td_first[dep], pl->td_count[dep], B, pl->depth_kng[dep], st));
  }
  if (U && sub)   // the target's leaves, written in idx_omega order
    CU(launch_leaf_solve(D, B, U, P.n_omega, st, pl->d_solve_leaves, int(P.solve_leaves.size()), pl->d_omega_pos));
  else if (U)
    CU(launch_leaf_solve(D, B, U, nn, st));
  else
    CU(launch_finalize(D, B, S, ll, st));
  return mark();
}

// Failures are recorded on the device (sticky atomicMin key, DevError) and copied
// to a pinned host word at the end of every call, on the call's stream: a call
// returns as soon as its work is queued.  take_error() turns a recorded failure
// into the plan's HddError (lowest failing sample of the call that failed) and
// resets the record; it is reached from hdd_sync, from the synchronous entry
// points, and at the start of the next call when the copy has already landed.
static int enqueue_error_copy(HddPlan* pl, cudaStream_t st) {
  CU(cudaMemcpyAsync(pl->h_err, pl->dev.err, sizeof(DevError), cudaMemcpyDeviceToHost, st));
  return HDD_OK;
}

static int take_error(HddPlan* pl) {
  const unsigned long long key = *reinterpret_cast<volatile unsigned long long*>(pl->h_err);
  if (key == kNoError) return HDD_OK;
  CU(cudaDeviceSynchronize());          // error path: drain every queued copy first
  const unsigned long long k2 = *reinterpret_cast<volatile unsigned long long*>(pl->h_err);
  CU(cudaMemset(pl->dev.err, 0xff, sizeof(DevError)));
  *pl->h_err = kNoError;
  int code;
  long long sample, node;
  dev_error_decode(std::min(key, k2), &code, &sample, &node);
  std::string msg;
  if (code == HDD_ERR_NUMERICAL)
    msg = node >= 0 ? "interface block at node " + std::to_string(node) + " is not positive definite"
                    : "non-finite forward observation";
  else
    msg = "coefficient values must be positive finite reals";
  return set_err(&pl->err, code, msg, int(sample), node);
}

static int sync_and_check(HddPlan* pl, cudaStream_t st) {
  CU(cudaStreamSynchronize(st));
  return take_error(pl);
}

static int check_call(HddPlan* pl, int64_t B, const void* in, bool want_separable) {
  if (!pl) return HDD_ERR_USAGE;
  if (pl->device < 0) return set_err(&pl->err, HDD_ERR_USAGE, "host-only plan cannot run a forward batch");
  if (B < 0 || (B > 0 && !in)) return set_err(&pl->err, HDD_ERR_USAGE, "invalid batch");
  if (want_separable && !pl->plan.separable)
    return set_err(&pl->err, HDD_ERR_USAGE,
                   "plan has no separable parametrization: pass coefficient fields (hdd_forward_batch_kappa)");
  return HDD_OK;
}

// Sub-batched launch of a whole batch on `st` (asynchronous).
static int run_batch(HddPlan* pl, const double* Z, const double* Kin, int64_t B, double* S, double* ll, double* U,
                     cudaStream_t st, const HddRhs* rhs = nullptr, bool sub = false) {
  const int nz = pl->plan.n_z, no = int(pl->plan.obs_kind.size());
  const int64_t nt = int64_t(2) * pl->plan.N * pl->plan.N;
  const int64_t nn = sub ? int64_t(pl->plan.n_omega) : int64_t(pl->plan.m) * pl->plan.m;
  for (int64_t done = 0; done < B;) {
    const int b = int(std::min<int64_t>(pl->bcap, B - done));
    const int rc = run_sub_batch(pl, Z ? Z + done * nz : nullptr, Kin ? Kin + done * nt : nullptr, b,
                                 S ? S + done * no : nullptr, ll ? ll + done : nullptr, U ? U + done * nn : nullptr, st,
                                 done, nullptr, rhs, sub);
    if (rc != HDD_OK) return rc;
    done += b;
  }
  return enqueue_error_copy(pl, st);
}

int hdd_sync(HddPlan* pl, void* stream) {
  if (!pl) return HDD_ERR_USAGE;
  if (pl->device < 0) return HDD_OK;
  CU(cudaSetDevice(pl->device));
  return sync_and_check(pl, static_cast<cudaStream_t>(stream));
}

int hdd_forward_batch(HddPlan* pl, const double* Z, int64_t B, double* S, double* ll, void* stream) {
  int rc = check_call(pl, B, Z, true);
  if (rc != HDD_OK) return rc;
  if (B == 0) return HDD_OK;
  CU(cudaSetDevice(pl->device));
  if ((rc = take_error(pl)) != HDD_OK) return rc;     // an earlier call's failure has landed
  cudaStream_t st = static_cast<cudaStream_t>(stream);   // NULL = legacy default stream
  static const bool no_graph = [] { const char* v = std::getenv("HDD_NO_GRAPH"); return v && v[0] == '1'; }();
  if (B <= pl->bcap && !no_graph) {
    const bool same = pl->g_seen && pl->g_Z == Z && pl->g_S == S && pl->g_ll == ll && pl->g_B == int(B);
    if (!same) {
      // new key: direct launches this time, remember the key
      if (pl->graph) {
        cudaGraphExecDestroy(pl->graph);
        pl->graph = nullptr;
      }
      pl->g_Z = Z;
      pl->g_S = S;
      pl->g_ll = ll;
      pl->g_B = int(B);
      pl->g_seen = true;
      return run_batch(pl, Z, nullptr, B, S, ll, nullptr, st);
    }
    if (!pl->graph) {
      // second call with the same buffers: capture the launch sequence (kappa, leaf
      // classes, one merge per depth, ..., finalize) once, replay it from now on
      CU(cudaStreamBeginCapture(pl->stream, cudaStreamCaptureModeThreadLocal));
      rc = run_sub_batch(pl, Z, nullptr, int(B), S, ll, nullptr, pl->stream, 0);
      cudaGraph_t g = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(pl->stream, &g);
      if (rc != HDD_OK) {
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      CU(ce);
      const cudaError_t ie = cudaGraphInstantiate(&pl->graph, g, 0);
      cudaGraphDestroy(g);
      CU(ie);
    }
    CU(cudaGraphLaunch(pl->graph, st));
    return enqueue_error_copy(pl, st);
  }
  return run_batch(pl, Z, nullptr, B, S, ll, nullptr, st);
}

int hdd_forward_batch_kappa(HddPlan* pl, const double* K, int64_t B, double* S, double* ll, void* stream) {
  int rc = check_call(pl, B, K, false);
  if (rc != HDD_OK) return rc;
  if (B == 0) return HDD_OK;
  CU(cudaSetDevice(pl->device));
  if ((rc = take_error(pl)) != HDD_OK) return rc;
  return run_batch(pl, nullptr, K, B, S, ll, nullptr, static_cast<cudaStream_t>(stream));
}

int hdd_forward_batch_timed(HddPlan* pl, const double* Z, int64_t B, double* S, double* ll, void* stream,
                            double* stage_ms, int32_t n_stages) {
  int rc = check_call(pl, B, Z, true);
  if (rc != HDD_OK) return rc;
  const int ns = pl->plan.leaf_depth + 3;
  if (n_stages != ns || !stage_ms) return set_err(&pl->err, HDD_ERR_USAGE, "stage_ms must hold leaf_depth + 3 entries");
  if (B <= 0) return set_err(&pl->err, HDD_ERR_USAGE, "invalid batch");
  CU(cudaSetDevice(pl->device));
  if ((rc = take_error(pl)) != HDD_OK) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);   // NULL = legacy default stream
  std::vector<cudaEvent_t> ev(ns + 1);
  for (auto& e : ev) CU(cudaEventCreate(&e));
  const int nz = pl->plan.n_z, no = int(pl->plan.obs_kind.size());
  int64_t done = 0;
  while (done < B && rc == HDD_OK) {
    int b = int(std::min<int64_t>(pl->bcap, B - done));
    rc = run_sub_batch(pl, Z + done * nz, nullptr, b, S ? S + done * no : nullptr, ll ? ll + done : nullptr, nullptr,
                       st, done, ev.data());
    if (rc == HDD_OK) {
      CU(cudaEventSynchronize(ev[ns]));
      for (int i = 0; i < ns; ++i) {
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
        stage_ms[i] += ms;
      }
    }
    done += b;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  if (rc != HDD_OK) return rc;
  if ((rc = enqueue_error_copy(pl, st)) != HDD_OK) return rc;
  return sync_and_check(pl, st);
}

// Host buffers: the batch is cut into sub-batches; the H2D copy of sub-batch i+1 (copy
// stream in) and the D2H copy of sub-batch i-1's results (copy stream out) overlap
// the compute of sub-batch i on the plan's stream.  Returns when the results are in
// host memory.  `in_w` doubles per input row (n_z for Z, 2N^2 for kappa fields).
static int run_host(HddPlan* pl, const double* Xh, int in_w, bool is_kappa, int64_t B, double* Sh, double* llh,
                    const HddRhs* rhs = nullptr) {
  const int no = int(pl->plan.obs_kind.size());
  const int64_t nb = (B + pl->bcap - 1) / pl->bcap;
  if (B > pl->io_cap || (is_kappa && !pl->io_kappa) || (!is_kappa && pl->io_kappa)) {
    if (pl->d_Z) cudaFree(pl->d_Z);
    if (pl->d_S) cudaFree(pl->d_S);
    if (pl->d_ll) cudaFree(pl->d_ll);
    pl->d_Z = pl->d_S = pl->d_ll = nullptr;
    pl->io_cap = 0;
    CU(cudaMalloc(&pl->d_Z, size_t(B) * std::max(in_w, 1) * 8));
    CU(cudaMalloc(&pl->d_S, size_t(B) * no * 8));
    CU(cudaMalloc(&pl->d_ll, size_t(B) * 8));
    pl->io_cap = B;
    pl->io_kappa = is_kappa;
  }
  cudaStream_t st = pl->stream;
  while (int64_t(pl->pipe_ev.size()) < 2 * nb) {
    cudaEvent_t e;
    CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    pl->pipe_ev.push_back(e);
  }
  auto rows = [&](int64_t i) { return std::min<int64_t>(pl->bcap, B - i * pl->bcap); };
  auto h2d = [&](int64_t i) -> int {
    const int64_t r0 = i * pl->bcap;
    CU(cudaMemcpyAsync(pl->d_Z + r0 * in_w, Xh + r0 * in_w, size_t(rows(i)) * in_w * 8, cudaMemcpyHostToDevice,
                       pl->cs_in));
    CU(cudaEventRecord(pl->pipe_ev[2 * i], pl->cs_in));
    return HDD_OK;
  };
  int rc;
  if ((rc = h2d(0))) return rc;
  for (int64_t i = 0; i < nb; ++i) {
    const int64_t r0 = i * pl->bcap;
    const int b = int(rows(i));
    CU(cudaStreamWaitEvent(st, pl->pipe_ev[2 * i], 0));
    const double* x = pl->d_Z + r0 * in_w;
    rc = run_sub_batch(pl, is_kappa ? nullptr : x, is_kappa ? x : nullptr, b, Sh ? pl->d_S + r0 * no : nullptr,
                       llh ? pl->d_ll + r0 : nullptr, nullptr, st, r0, nullptr, rhs);
    if (rc != HDD_OK) return rc;
    CU(cudaEventRecord(pl->pipe_ev[2 * i + 1], st));
    if (i + 1 < nb && (rc = h2d(i + 1))) return rc;
    CU(cudaStreamWaitEvent(pl->cs_out, pl->pipe_ev[2 * i + 1], 0));
    if (Sh) CU(cudaMemcpyAsync(Sh + r0 * no, pl->d_S + r0 * no, size_t(b) * no * 8, cudaMemcpyDeviceToHost, pl->cs_out));
    if (llh) CU(cudaMemcpyAsync(llh + r0, pl->d_ll + r0, size_t(b) * 8, cudaMemcpyDeviceToHost, pl->cs_out));
  }
  if ((rc = enqueue_error_copy(pl, st)) != HDD_OK) return rc;
  CU(cudaStreamSynchronize(pl->cs_out));
  return sync_and_check(pl, st);
}

int hdd_forward_batch_host(HddPlan* pl, const double* Zh, int64_t B, double* Sh, double* llh) {
  int rc = check_call(pl, B, Zh, true);
  if (rc != HDD_OK) return rc;
  if (B == 0) return HDD_OK;
  CU(cudaSetDevice(pl->device));
  if ((rc = take_error(pl)) != HDD_OK) return rc;
  return run_host(pl, Zh, pl->plan.n_z, false, B, Sh, llh);
}

int hdd_forward_batch_kappa_host(HddPlan* pl, const double* Kh, int64_t B, double* Sh, double* llh) {
  int rc = check_call(pl, B, Kh, false);
  if (rc != HDD_OK) return rc;
  if (B == 0) return HDD_OK;
  CU(cudaSetDevice(pl->device));
  if ((rc = take_error(pl)) != HDD_OK) return rc;
  return run_host(pl, Kh, 2 * pl->plan.N * pl->plan.N, true, B, Sh, llh);
}

static int solve_common(HddPlan* pl, const double* Z, const double* K, int64_t B, double* U, void* stream) {
  if ((pl->dev.mode != 1 || !pl->plan.full_solve) && pl->plan.leaf_depth > 0)   // a single-leaf tree has no interfaces
    return set_err(&pl->err, HDD_ERR_USAGE,
                   "the full-solution sweep requires a full-solution plan (mode = 1, full_solve = 1 keeps every factor)");
  if (B > 0 && !U) return set_err(&pl->err, HDD_ERR_USAGE, "invalid batch");
  if (B == 0) return HDD_OK;
  CU(cudaSetDevice(pl->device));
  int rc = take_error(pl);
  if (rc != HDD_OK) return rc;
  return run_batch(pl, Z, K, B, nullptr, nullptr, U, static_cast<cudaStream_t>(stream));
}

int hdd_solve_batch(HddPlan* pl, const double* Z, int64_t B, double* U, void* stream) {
  int rc = check_call(pl, B, Z, true);
  if (rc != HDD_OK) return rc;
  return solve_common(pl, Z, nullptr, B, U, stream);
}

int hdd_solve_batch_kappa(HddPlan* pl, const double* K, int64_t B, double* U, void* stream) {
  int rc = check_call(pl, B, K, false);
  if (rc != HDD_OK) return rc;
  return solve_common(pl, nullptr, K, B, U, stream);
}

static int solve_host(HddPlan* pl, const double* Xh, bool is_kappa, int64_t B, double* Uh) {
  if (B == 0) return HDD_OK;
  CU(cudaSetDevice(pl->device));
  const int64_t in_w = is_kappa ? int64_t(2) * pl->plan.N * pl->plan.N : pl->plan.n_z;
  const int64_t nn = int64_t(pl->plan.m) * pl->plan.m;
  double* dX = nullptr;
  double* dU = nullptr;
  CU(cudaMalloc(&dX, size_t(B) * std::max<int64_t>(in_w, 1) * 8));
  if (cudaMalloc(&dU, size_t(B) * nn * 8) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(dX);
    return set_err(&pl->err, HDD_ERR_NOMEM, "device allocation of the solution buffer failed");
  }
  cudaStream_t st = pl->stream;
  int rc = HDD_OK;
  if (cudaMemcpyAsync(dX, Xh, size_t(B) * in_w * 8, cudaMemcpyHostToDevice, st) != cudaSuccess) rc = HDD_ERR_CUDA;
  if (rc == HDD_OK) rc = solve_common(pl, is_kappa ? nullptr : dX, is_kappa ? dX : nullptr, B, dU, st);
  if (rc == HDD_OK && cudaMemcpyAsync(Uh, dU, size_t(B) * nn * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    rc = HDD_ERR_CUDA;
  if (rc == HDD_OK) rc = sync_and_check(pl, st);
  cudaFree(dX);
  cudaFree(dU);
  return rc;
}

int hdd_solve_batch_host(HddPlan* pl, const double* Zh, int64_t B, double* Uh) {
  int rc = check_call(pl, B, Zh, true);
  if (rc != HDD_OK) return rc;
  if (B > 0 && !Uh) return set_err(&pl->err, HDD_ERR_USAGE, "invalid batch");
  return solve_host(pl, Zh, false, B, Uh);
}

int hdd_solve_batch_kappa_host(HddPlan* pl, const double* Kh, int64_t B, double* Uh) {
  int rc = check_call(pl, B, Kh, false);
  if (rc != HDD_OK) return rc;
  if (B > 0 && !Uh) return set_err(&pl->err, HDD_ERR_USAGE, "invalid batch");
  return solve_host(pl, Kh, true, B, Uh);
}

// ---- per-call right-hand sides (general Psi^f / Phi^f maps applied to new data) ----
static int check_rhs(HddPlan* pl, const HddRhs* rhs, bool host) {
  if (!rhs) return HDD_OK;
  const int64_t nn = int64_t(pl->plan.m) * pl->plan.m, ng = int64_t(4) * pl->plan.N;
  if (rhs->f && rhs->f_stride != 0 && (host ? rhs->f_stride != nn : rhs->f_stride < nn))
    return set_err(&pl->err, HDD_ERR_USAGE, "f_stride must be 0 (one row) or the row length (n_nodes)");
  if (rhs->g && rhs->g_stride != 0 && (host ? rhs->g_stride != ng : rhs->g_stride < ng))
    return set_err(&pl->err, HDD_ERR_USAGE, "g_stride must be 0 (one row) or the row length (4N)");
  return HDD_OK;
}

int hdd_forward_batch_ex(HddPlan* pl, const double* Z, const double* K, int64_t B, const HddRhs* rhs, double* S,
                         double* ll, void* stream) {
  if (!pl) return HDD_ERR_USAGE;
  if ((Z != nullptr) == (K != nullptr) && B > 0) return set_err(&pl->err, HDD_ERR_USAGE, "pass exactly one of Z and K");
  int rc = check_call(pl, B, Z ? Z : K, Z != nullptr);
  if (rc != HDD_OK) return rc;
  if ((rc = check_rhs(pl, rhs, false)) != HDD_OK) return rc;
  if (B == 0) return HDD_OK;
  CU(cudaSetDevice(pl->device));
  if ((rc = take_error(pl)) != HDD_OK) return rc;
  return run_batch(pl, Z, K, B, S, ll, nullptr, static_cast<cudaStream_t>(stream), rhs);
}

// device copies of a host HddRhs (rows of n_nodes / 4N doubles)
struct DevRhs {
  HddRhs r{};
  double* f = nullptr;
  double* g = nullptr;
  ~DevRhs() {
    if (f) cudaFree(f);
    if (g) cudaFree(g);
  }
};
static int upload_rhs(HddPlan* pl, const HddRhs* h, int64_t B, DevRhs& d) {
  if (!h) return HDD_OK;
  const int64_t nn = int64_t(pl->plan.m) * pl->plan.m, ng = int64_t(4) * pl->plan.N;
  if (h->f) {
    const size_t n = size_t(h->f_stride ? B : 1) * nn;
    CU(cudaMalloc(&d.f, n * 8));
    CU(cudaMemcpy(d.f, h->f, n * 8, cudaMemcpyHostToDevice));
    d.r.f = d.f;
    d.r.f_stride = h->f_stride;
  }
  if (h->g) {
    const size_t n = size_t(h->g_stride ? B : 1) * ng;
    CU(cudaMalloc(&d.g, n * 8));
    CU(cudaMemcpy(d.g, h->g, n * 8, cudaMemcpyHostToDevice));
    d.r.g = d.g;
    d.r.g_stride = h->g_stride;
  }
  return HDD_OK;
}

int hdd_forward_batch_ex_host(HddPlan* pl, const double* Zh, const double* Kh, int64_t B, const HddRhs* rhs,
                              double* Sh, double* llh) {
  if (!pl) return HDD_ERR_USAGE;
  if ((Zh != nullptr) == (Kh != nullptr) && B > 0) return set_err(&pl->err, HDD_ERR_USAGE, "pass exactly one of Z and K");
  int rc = check_call(pl, B, Zh ? Zh : Kh, Zh != nullptr);
  if (rc != HDD_OK) return rc;
  if ((rc = check_rhs(pl, rhs, true)) != HDD_OK) return rc;
  if (B == 0) return HDD_OK;
  CU(cudaSetDevice(pl->device));
  if ((rc = take_error(pl)) != HDD_OK) return rc;
  DevRhs d;
  if ((rc = upload_rhs(pl, rhs, B, d)) != HDD_OK) return rc;
  const int in_w = Zh ? pl->plan.n_z : 2 * pl->plan.N * pl->plan.N;
  return run_host(pl, Zh ? Zh : Kh, in_w, Kh != nullptr, B, Sh, llh, rhs ? &d.r : nullptr);
}

int hdd_solve_batch_ex(HddPlan* pl, const double* Z, const double* K, int64_t B, const HddRhs* rhs, double* U,
                       void* stream) {
  if (!pl) return HDD_ERR_USAGE;
  if ((Z != nullptr) == (K != nullptr) && B > 0) return set_err(&pl->err, HDD_ERR_USAGE, "pass exactly one of Z and K");
  int rc = check_call(pl, B, Z ? Z : K, Z != nullptr);
  if (rc != HDD_OK) return rc;
  if ((rc = check_rhs(pl, rhs, false)) != HDD_OK) return rc;
  if ((pl->dev.mode != 1 || !pl->plan.full_solve) && pl->plan.leaf_depth > 0)
    return set_err(&pl->err, HDD_ERR_USAGE,
                   "the full-solution sweep requires a full-solution plan (mode = 1, full_solve = 1 keeps every factor)");
  if (B > 0 && !U) return set_err(&pl->err, HDD_ERR_USAGE, "invalid batch");
  if (B == 0) return HDD_OK;
  CU(cudaSetDevice(pl->device));
  if ((rc = take_error(pl)) != HDD_OK) return rc;
  return run_batch(pl, Z, K, B, nullptr, nullptr, U, static_cast<cudaStream_t>(stream), rhs);
}

int hdd_solve_batch_ex_host(HddPlan* pl, const double* Zh, const double* Kh, int64_t B, const HddRhs* rhs,
                            double* Uh) {
  if (!pl) return HDD_ERR_USAGE;
  if ((Zh != nullptr) == (Kh != nullptr) && B > 0) return set_err(&pl->err, HDD_ERR_USAGE, "pass exactly one of Z and K");
  int rc = check_call(pl, B, Zh ? Zh : Kh, Zh != nullptr);
  if (rc != HDD_OK) return rc;
  if ((rc = check_rhs(pl, rhs, true)) != HDD_OK) return rc;
  if (B > 0 && !Uh) return set_err(&pl->err, HDD_ERR_USAGE, "invalid batch");
  if (B == 0) return HDD_OK;
  CU(cudaSetDevice(pl->device));
  DevRhs d;
  if ((rc = upload_rhs(pl, rhs, B, d)) != HDD_OK) return rc;
  const bool is_kappa = Kh != nullptr;
  const int64_t in_w = is_kappa ? int64_t(2) * pl->plan.N * pl->plan.N : pl->plan.n_z;
  const int64_t nn = int64_t(pl->plan.m) * pl->plan.m;
  double* dX = nullptr;
  double* dU = nullptr;
  CU(cudaMalloc(&dX, size_t(B) * std::max<int64_t>(in_w, 1) * 8));
  if (cudaMalloc(&dU, size_t(B) * nn * 8) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(dX);
    return set_err(&pl->err, HDD_ERR_NOMEM, "device allocation of the solution buffer failed");
  }
  cudaStream_t st = pl->stream;
  if (cudaMemcpyAsync(dX, is_kappa ? Kh : Zh, size_t(B) * in_w * 8, cudaMemcpyHostToDevice, st) != cudaSuccess)
    rc = HDD_ERR_CUDA;
  if (rc == HDD_OK)
    rc = hdd_solve_batch_ex(pl, is_kappa ? nullptr : dX, is_kappa ? dX : nullptr, B, rhs ? &d.r : nullptr, dU, st);
  if (rc == HDD_OK && cudaMemcpyAsync(Uh, dU, size_t(B) * nn * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    rc = HDD_ERR_CUDA;
  if (rc == HDD_OK) rc = sync_and_check(pl, st);
  cudaFree(dX);
  cudaFree(dU);
  return rc;
}

// ---- solve_subdomain as a partial inverse ----
__global__ void gather_omega_kernel(const double* __restrict__ U, int64_t nn, const int32_t* __restrict__ pos,
                                    double* __restrict__ Us, int n_omega, int B) {
  const int s = blockIdx.y;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < nn; t += int64_t(gridDim.x) * blockDim.x)
    if (pos[t] >= 0) Us[int64_t(s) * n_omega + pos[t]] = U[int64_t(s) * nn + t];
}

int hdd_solve_subdomain_batch(HddPlan* pl, const double* Z, const double* K, int64_t B, const HddRhs* rhs,
                              double* Us, void* stream) {
  if (!pl) return HDD_ERR_USAGE;
  if ((Z != nullptr) == (K != nullptr) && B > 0) return set_err(&pl->err, HDD_ERR_USAGE, "pass exactly one of Z and K");
  int rc = check_call(pl, B, Z ? Z : K, Z != nullptr);
  if (rc != HDD_OK) return rc;
  if ((rc = check_rhs(pl, rhs, false)) != HDD_OK) return rc;
  if (pl->plan.solve_target < 0)
    return set_err(&pl->err, HDD_ERR_USAGE,
                   "plan has no subdomain target: create it with solve_target (the SolveMode.keep_path analogue)");
  if (B > 0 && !Us) return set_err(&pl->err, HDD_ERR_USAGE, "invalid batch");
  if (B == 0) return HDD_OK;
  CU(cudaSetDevice(pl->device));
  if ((rc = take_error(pl)) != HDD_OK) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (pl->plan.leaf_depth > 0) return run_batch(pl, Z, K, B, nullptr, nullptr, Us, st, rhs, true);
  // a single-leaf or sub-leaf mesh: the whole solution, then the target's nodes
  const int64_t nn = int64_t(pl->plan.m) * pl->plan.m;
  double* U = nullptr;
  CU(cudaMallocAsync(reinterpret_cast<void**>(&U), size_t(B) * nn * 8, st));
  rc = run_batch(pl, Z, K, B, nullptr, nullptr, U, st, rhs);
  if (rc == HDD_OK) {
    gather_omega_kernel<<<dim3(unsigned((nn + 255) / 256), unsigned(B)), 256, 0, st>>>(U, nn, pl->d_omega_pos, Us,
                                                                                       pl->plan.n_omega, int(B));
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) rc = set_err(&pl->err, HDD_ERR_CUDA, cudaGetErrorString(e));
  }
  cudaFreeAsync(U, st);
  return rc;
}

int hdd_solve_subdomain_batch_host(HddPlan* pl, const double* Zh, const double* Kh, int64_t B, const HddRhs* rhs,
                                   double* Ush) {
  if (!pl) return HDD_ERR_USAGE;
  if ((Zh != nullptr) == (Kh != nullptr) && B > 0) return set_err(&pl->err, HDD_ERR_USAGE, "pass exactly one of Z and K");
  int rc = check_call(pl, B, Zh ? Zh : Kh, Zh != nullptr);
  if (rc != HDD_OK) return rc;
  if ((rc = check_rhs(pl, rhs, true)) != HDD_OK) return rc;
  if (B > 0 && !Ush) return set_err(&pl->err, HDD_ERR_USAGE, "invalid batch");
  if (B == 0) return HDD_OK;
  CU(cudaSetDevice(pl->device));
  DevRhs d;
  if ((rc = upload_rhs(pl, rhs, B, d)) != HDD_OK) return rc;
  const bool is_kappa = Kh != nullptr;
  const int64_t in_w = is_kappa ? int64_t(2) * pl->plan.N * pl->plan.N : pl->plan.n_z;
  const int64_t no = pl->plan.n_omega;
  double* dX = nullptr;
  double* dU = nullptr;
  CU(cudaMalloc(&dX, size_t(B) * std::max<int64_t>(in_w, 1) * 8));
  if (cudaMalloc(&dU, size_t(B) * std::max<int64_t>(no, 1) * 8) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(dX);
    return set_err(&pl->err, HDD_ERR_NOMEM, "device allocation of the subdomain buffer failed");
  }
  cudaStream_t st = pl->stream;
  if (cudaMemcpyAsync(dX, is_kappa ? Kh : Zh, size_t(B) * in_w * 8, cudaMemcpyHostToDevice, st) != cudaSuccess)
    rc = HDD_ERR_CUDA;
  if (rc == HDD_OK)
    rc = hdd_solve_subdomain_batch(pl, is_kappa ? nullptr : dX, is_kappa ? dX : nullptr, B, rhs ? &d.r : nullptr, dU, st);
  if (rc == HDD_OK && cudaMemcpyAsync(Ush, dU, size_t(B) * no * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    rc = HDD_ERR_CUDA;
  if (rc == HDD_OK) rc = sync_and_check(pl, st);
  cudaFree(dX);
  cudaFree(dU);
  return rc;
}

int hdd_posterior_weights(const double* ll, const double* lp, int64_t n, double* w, int64_t* idx, double* lse,
                          void* stream) {
  if (n <= 0 || !ll || !w || !idx || !lse) return HDD_ERR_USAGE;
  if (launch_posterior(ll, lp, n, w, idx, lse, static_cast<cudaStream_t>(stream)) != cudaSuccess)
    return HDD_ERR_CUDA;
  return HDD_OK;
}

int hdd_kappa_batch(HddPlan* pl, const double* Z, int64_t B, double* kappa, void* stream) {
  int rc = check_call(pl, B, Z, true);
  if (rc != HDD_OK) return rc;
  if (B > 0 && !kappa) return set_err(&pl->err, HDD_ERR_USAGE, "invalid batch");
  CU(cudaSetDevice(pl->device));
  if ((rc = take_error(pl)) != HDD_OK) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);   // NULL = legacy default stream
  const int64_t nt = int64_t(2) * pl->plan.N * pl->plan.N;
  for (int64_t done = 0; done < B;) {
    int b = int(std::min<int64_t>(pl->bcap, B - done));
    DevPlan D = pl->dev;
    D.sample0 = done;
    CU(launch_kappa(D, Z + done * pl->plan.n_z, b, kappa + done * nt, st));
    done += b;
  }
  if ((rc = enqueue_error_copy(pl, st)) != HDD_OK) return rc;
  return sync_and_check(pl, st);
}

int hdd_debug_lowrank_wide(HddPlan* pl, int64_t* total) {
  if (!pl || !total || pl->device < 0) return HDD_ERR_USAGE;
  *total = 0;
  if (!pl->dev.lr_wide_n) return HDD_OK;
  CU(cudaSetDevice(pl->device));
  int v[2] = {0, 0};
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(v, pl->dev.lr_wide_n, sizeof(v), cudaMemcpyDeviceToHost));
  *total = v[1];
  return HDD_OK;
}

int hdd_last_error(const HddPlan* pl, HddError* out) {
  if (!pl || !out) return HDD_ERR_USAGE;
  *out = pl->err;
  return HDD_OK;
}

int hdd_plan_info(const HddPlan* pl, HddPlanInfo* out) {
  if (!pl || !out) return HDD_ERR_USAGE;
  const Plan& P = pl->plan;
  out->level = P.level;
  out->n_cells = P.N;
  out->leaf_cells = kLeafCells;
  out->leaf_depth = P.leaf_depth;
  out->n_upper = int(P.upper.size());
  out->n_leaves = int(P.leaves.size());
  out->n_obs = int(P.obs_kind.size());
  out->leaf_cols = P.leaf_cols;
  out->max_batch = pl->bcap;
  out->n_kernels_per_batch = pl->device >= 0 ? pl->n_launches : 3 + int(P.upper_by_depth.size());
  int64_t ws = int64_t(2) * P.N * P.N;
  for (int64_t e : P.buf_elems_per_sample) ws += e;
  out->workspace_bytes = ws * 8 * std::max(1, pl->bcap);
  out->mode = P.mode;
  int ntd = 0;
  for (const auto& v : P.td_by_depth) ntd += int(v.size());
  out->n_topdown = ntd;
  out->tiny = P.tiny ? 1 : 0;
  out->separable = P.separable ? 1 : 0;
  out->full_solve = P.full_solve ? 1 : 0;
  out->n_omega = P.n_omega;
  out->factor_doubles = P.fac_elems;
  return HDD_OK;
}

int hdd_plan_node_info(const HddPlan* pl, int32_t idx, HddNodeInfo* out) {
  if (!pl || !out || idx < 0 || idx >= int(pl->plan.upper.size())) return HDD_ERR_USAGE;
  const UpperNode& U = pl->plan.upper[idx];
  out->ref_id = U.ref_id;
  out->depth = U.depth;
  out->i0 = U.i0; out->i1 = U.i1; out->j0 = U.j0; out->j1 = U.j1;
  out->son[0] = U.son[0];
  out->son[1] = U.son[1];
  out->k = U.k; out->ng = U.ng; out->nc = U.nc;
  out->bnd = U.bnd.data();
  out->gamma = U.gamma.data();
  out->gmap = U.gmap.data();
  out->csrc = U.csrc.data();
  out->ccoef = U.ccoef.data();
  out->cbirth = U.cbirth.data();
  return HDD_OK;
}

int hdd_plan_leaf_info(const HddPlan* pl, int32_t idx, HddLeafInfo* out) {
  if (!pl || !out || idx < 0 || idx >= int(pl->plan.leaves.size())) return HDD_ERR_USAGE;
  const Leaf& L = pl->plan.leaves[idx];
  out->ref_id = L.ref_id;
  out->i0 = L.i0;
  out->j0 = L.j0;
  out->ncols = int(L.cols.size());
  out->has_mean = L.own_mean ? 1 : 0;
  out->birth = L.birth.data();
  out->ccode = L.ccode.data();
  out->gperim = pl->plan.has_g ? L.gperim.data() : nullptr;
  return HDD_OK;
}

int hdd_plan_obs_info(const HddPlan* pl, int32_t idx, HddObsInfo* out) {
  if (!pl || !out || idx < 0 || idx >= int(pl->plan.route.size())) return HDD_ERR_USAGE;
  out->kind = pl->plan.route[idx].kind;
  out->col = pl->plan.route[idx].col;
  out->value = pl->plan.route[idx].value;
  out->node = pl->plan.route[idx].node;
  out->slot = pl->plan.route[idx].slot;
  return HDD_OK;
}

int hdd_leaf_template(int32_t r, int32_t* K, int32_t* k, int32_t* ng, const int32_t** map1, const int32_t** map2) {
  const auto& T = leaf_template();
  if (r < 0 || r >= int(T.size())) return HDD_ERR_USAGE;
  if (K) *K = T[r].K;
  if (k) *k = T[r].k;
  if (ng) *ng = T[r].ng;
  if (map1) *map1 = T[r].map1.data();
  if (map2) *map2 = T[r].map2.data();
  return HDD_OK;
}

int hdd_debug_node_output(HddPlan* pl, int32_t idx, int32_t b, double* psi, double* R, double* sigma) {
  if (!pl || pl->device < 0) return HDD_ERR_USAGE;
  const Plan& P = pl->plan;
  if (P.n_buffers != P.leaf_depth + 1) return set_err(&pl->err, HDD_ERR_USAGE, "plan was not created with keep_nodes");
  if (b < 0 || b >= pl->bcap) return set_err(&pl->err, HDD_ERR_USAGE, "sample index out of range");
  const double* base;
  int k, ld, nc;
  if (idx >= 0) {
    if (idx >= int(P.upper.size())) return HDD_ERR_USAGE;
    const UpperNode& U = P.upper[idx];
    base = pl->dev.buf[U.buf] + U.out_off * pl->bcap + int64_t(b) * U.out_elems;
    k = U.k; ld = U.out_ld; nc = U.nc;
  } else {
    int l = -1 - idx;
    if (l >= int(P.leaves.size())) return HDD_ERR_USAGE;
    base = pl->dev.buf[P.leaf_buf] + int64_t(l) * P.leaf_elems * pl->bcap + int64_t(b) * P.leaf_elems;
    k = kLeafPerim; ld = P.leaf_ld; nc = int(P.leaves[l].cols.size());
  }
  const size_t tk = size_t(k) * (k + 1) / 2;
  std::vector<double> tmp(tk + size_t(k) * ld + ld);
  CU(cudaSetDevice(pl->device));
  CU(cudaStreamSynchronize(pl->stream));
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(tmp.data(), base, (tk + size_t(k) * ld + nc) * 8, cudaMemcpyDeviceToHost));
  for (int a = 0; a < k; ++a) {
    if (psi)
      for (int c = 0; c < k; ++c) psi[size_t(a) * k + c] = a >= c ? tmp[size_t(a) * (a + 1) / 2 + c] : tmp[size_t(c) * (c + 1) / 2 + a];
    if (R) for (int c = 0; c < nc; ++c) R[size_t(a) * nc + c] = tmp[tk + size_t(a) * ld + c];
  }
  if (sigma) for (int c = 0; c < nc; ++c) sigma[c] = tmp[tk + size_t(k) * ld + c];
  return HDD_OK;
}

}  // extern "C"
