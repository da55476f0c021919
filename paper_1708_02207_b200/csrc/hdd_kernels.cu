// sm_100a kernels of the batched HDD likelihood (fp64 throughout).
//
//   K1 kappa_kernel     kappa_t = exp(sum_k coef_k z_k sx_k(x_t) sy_k(y_t)) for every
//                       triangle of every sample; HBM-streaming, double2 stores.
//                       Replaces ParamField.kappa (bayes.py:73-77) / the sine-KL
//                       CoefficientField.from_callable (fem.py:39-43).
//   K2 leaf_kernel      one CTA per (16x16-cell leaf, sample): the reference's
//                       sub-tree recursion below the leaf (hdd.py:313-341 on the
//                       leaf's 8 in-leaf depths) done level-synchronously in shared
//                       memory — gather sons (assemble_father, hdd.py:216-238),
//                       warp Cholesky of the interface block, column-parallel
//                       forward substitution, Schur update (schur_eliminate,
//                       hdd.py:241-277) — with the load and observation
//                       functionals carried as extra columns (functionals.py:77-106).
//   K3 merge_m_kernel   one CTA per (upper node, sample): the interface panel
//                       [A21 | A22 | R_gamma] gathered into shared memory, eliminated
//                       row by row, and the Schur update Psi = A11 - W^T W streamed
//                       out with FP64 DMMA (mma.sync m8n8k4 -> DMMA.8x8x4).
//   K4 finalize_kernel  S = root functionals, ll = -1/2 sum r^2 - sum log(sigma sqrt(2pi))
//                       (bayes.py:192-198, :222-224), non-finite check.
#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cstdio>

#include <cuda.h>

#include "hdd.h"
#include "hdd_device.h"
#include "hdd_plan.h"

namespace hdd {

// ---------------------------------------------------------------------------
// shared helpers
// ---------------------------------------------------------------------------
// Failure record: one 64-bit key, atomicMin over (global sample, kind, node) so the
// reported failure is the lowest failing sample of the batch — the one the reference's
// per-sample loop would raise on — independent of CTA scheduling and sub-batching.
__device__ __forceinline__ void record_error(const DevPlan& p, int code, int sample, long long node) {
  atomicMin(&p.err->key, dev_error_key(p.sample0 + sample, code, node));
}

// Right-hand side of sample s: per-call rows (f_stride, hdd_forward_batch_ex) or the
// plan's fixed f; NULL = f = 1.
__device__ __forceinline__ const double* sample_f(const DevPlan& p, int s) {
  return p.f ? p.f + int64_t(s) * p.f_stride : nullptr;
}
// Dirichlet value of perimeter node t of leaf `leaf` for sample s: per-call data
// (leaf_gpos: position in the boundary vector, -1 off the domain boundary) or the plan's.
__device__ __forceinline__ double leaf_gval(const DevPlan& p, int leaf, int s, int t) {
  if (p.gcall) {
    const int pos = p.leaf_gpos[int64_t(leaf) * 64 + t];
    return pos >= 0 ? p.gcall[int64_t(s) * p.g_stride + pos] : 0.0;
  }
  return p.leaf_g ? p.leaf_g[int64_t(leaf) * 64 + t] : 0.0;
}
// Value of a constant observation route (boundary point: g there).
__device__ __forceinline__ double route_const(const DevPlan& p, int o, int s) {
  const int pos = p.route_node[o];
  return (p.gcall && pos >= 0) ? p.gcall[int64_t(s) * p.g_stride + pos] : p.route_val[o];
}

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// K1: coefficient field
// ---------------------------------------------------------------------------
// grid: (ceil(N/128), ceil(N/32), B); block 128.  Thread = column j of 32 consecutive
// cell rows, in groups of 8: each sy_k(j) pair is loaded once per group and feeds 8
// cells; double2 stores (each warp writes 512 contiguous bytes per cell row).  32 rows
// per CTA amortise the czx setup (dependent loads + barrier) over 32 KB of output.
constexpr int kKappaRows = 8, kKappaGroups = 4;
__global__ void __launch_bounds__(128) kappa_kernel(DevPlan p, const double* __restrict__ Z, int B,
                                                    double* __restrict__ kappa) {
  extern __shared__ double czx[];   // [n_z][kKappaGroups * kKappaRows][2]: coef_k z_k sx_k(2i + type)
  constexpr int RB = kKappaRows * kKappaGroups;
  const int N = p.N, nz = p.n_z;
  const int i0 = blockIdx.y * RB, s = blockIdx.z;
  const int nrow = min(RB, N - i0);
  const double* z = Z + int64_t(s) * nz;
  for (int t = threadIdx.x; t < nz * RB * 2; t += blockDim.x) {
    const int k = t / (RB * 2), r = t - k * (RB * 2);
    czx[t] = r < 2 * nrow ? p.coef[k] * z[k] * p.sx[int64_t(k) * 2 * N + 2 * i0 + r] : 0.0;
  }
  __syncthreads();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  const double2* sy2 = reinterpret_cast<const double2*>(p.sy);
  double2* out = reinterpret_cast<double2*>(kappa + int64_t(s) * 2 * N * N);
  bool bad = false;
  for (int g = 0; g < nrow; g += kKappaRows) {
    double q[kKappaRows][2] = {};
    for (int k = 0; k < nz; ++k) {
      const double2 t = __ldg(sy2 + int64_t(k) * N + j);
      const double* c = czx + k * RB * 2 + 2 * g;
#pragma unroll
      for (int r = 0; r < kKappaRows; ++r) {
        q[r][0] = fma(c[2 * r], t.x, q[r][0]);
        q[r][1] = fma(c[2 * r + 1], t.y, q[r][1]);
      }
    }
#pragma unroll
    for (int r = 0; r < kKappaRows; ++r) {
      const double2 v = make_double2(exp(q[r][0]), exp(q[r][1]));
      bad |= !(v.x > 0.0) || !(v.y > 0.0) || !isfinite(v.x) || !isfinite(v.y);
      if (g + r < nrow) out[int64_t(i0 + g + r) * N + j] = v;
    }
  }
  if (bad) record_error(p, HDD_ERR_CONFIG, s, -1);
}

cudaError_t launch_kappa(const DevPlan& p, const double* Z, int B, double* kappa, cudaStream_t s) {
  constexpr int RB = kKappaRows * kKappaGroups;
  dim3 grid((p.N + 127) / 128, (p.N + RB - 1) / RB, B);
  kappa_kernel<<<grid, 128, size_t(2) * RB * p.n_z * sizeof(double), s>>>(p, Z, B, kappa);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K2: leaf condensation
// ---------------------------------------------------------------------------
// compile-time in-leaf level shapes (checked against leaf_template() at upload)
struct LeafLevelShape {
  int K, k, ng, ks;
};
__host__ __device__ constexpr LeafLevelShape leaf_shape(int r) {
  return r == 0 ? LeafLevelShape{79, 64, 15, 48}
       : r == 1 ? LeafLevelShape{55, 48, 7, 32}
       : r == 2 ? LeafLevelShape{39, 32, 7, 24}
       : r == 3 ? LeafLevelShape{27, 24, 3, 16}
       : r == 4 ? LeafLevelShape{19, 16, 3, 12}
       : r == 5 ? LeafLevelShape{13, 12, 1, 8}
       : r == 6 ? LeafLevelShape{9, 8, 1, 6}
                : LeafLevelShape{6, 6, 0, 4};
}
__host__ __device__ constexpr int ctri(int a) { return (a * (a + 1)) / 2; }

struct LeafTmplDev {
  int K[8], k[8], ng[8], kson[8], moff[8];
};
__constant__ LeafTmplDev c_tmpl;
__constant__ int16_t c_map[2][256];
__constant__ uint16_t c_orig[512];   // in-leaf node origin (x | y << 8), index 2^r - 1 + q
// lower-triangle tile coordinates of tile index tt (row-major over the triangle)
__constant__ uint8_t c_tile_i[64];
__constant__ uint8_t c_tile_j[64];

// Precomputed per-level gather programs of the leaf kernel (one set per column
// class NC = 2, 4, 8): every panel / update item of level r knows its source
// offsets in the two sons' packed blocks, so the kernel does no index decoding.
struct LeafItemP { int16_t o1, o2, c, pad; };     // panel item t = g * W + j
struct LeafItemU { int16_t a, bx, o1, o2; };      // update item: row a, X column bx
struct LeafTabDev {
  const LeafItemP* P[3];
  const LeafItemU* U[3];
  int poff[3][6];
  int uoff[3][6];
};
__constant__ LeafTabDev c_ltab;

// per-phase clock64 stamps of CTA (0,0) of the last leaf launch (profiling hook)
__device__ long long g_leaf_clk[64];
#ifndef HDD_PROFILE_TICKS
#define LEAF_TICK(i) do { } while (0)
#else
#ifndef HDD_TICK_X          // which CTA stamps (default the first; a mid-launch CTA shows the steady state)
#define HDD_TICK_X 0
#define HDD_TICK_Y 0
#endif
#define LEAF_TICK(i) \
  do { if (blockIdx.x == HDD_TICK_X && blockIdx.y == HDD_TICK_Y && threadIdx.x == 0) g_leaf_clk[i] = clock64(); } while (0)
#endif
int read_leaf_clocks(long long* out) {
  return cudaMemcpyFromSymbol(out, g_leaf_clk, sizeof(long long) * 64) == cudaSuccess ? 0 : -1;
}
// per-phase clock64 stamps of CTA (sample 0, node 0) of every merge launch, by depth
__device__ long long g_merge_clk[32][8];
#ifndef HDD_PROFILE_TICKS
#define MERGE_TICK(i) do { (void)slot; } while (0)
#else
#define MERGE_TICK(i) \
  do { if (blockIdx.x == HDD_TICK_X && blockIdx.y == HDD_TICK_Y && threadIdx.x == 0 && slot >= 0 && slot < 32) g_merge_clk[slot][i] = clock64(); } while (0)
#endif
int read_merge_clocks(long long* out) {
  return cudaMemcpyFromSymbol(out, g_merge_clk, sizeof(long long) * 32 * 8) == cudaSuccess ? 0 : -1;
}


int upload_leaf_template() {
  const auto& T = leaf_template();
  LeafTmplDev t{};
  int16_t maps[2][256] = {};
  int off = 0;
  for (int r = 0; r < kLeafLevels; ++r) {
    const LeafLevelShape sh = leaf_shape(r);
    if (sh.K != T[r].K || sh.k != T[r].k || sh.ng != T[r].ng || sh.ks != T[r].kson) return -2;
    t.K[r] = T[r].K;
    t.k[r] = T[r].k;
    t.ng[r] = T[r].ng;
    t.kson[r] = T[r].kson;
    t.moff[r] = off;
    for (int a = 0; a < T[r].K; ++a) {
      maps[0][off + a] = int16_t(T[r].map1[a]);
      maps[1][off + a] = int16_t(T[r].map2[a]);
    }
    off += T[r].K;
  }
  uint16_t orig[512] = {};
  for (int r = 0; r <= kLeafLevels; ++r) {
    for (int q = 0; q < (1 << r); ++q) {
      int x = 0, y = 0, w = kLeafCells, h = kLeafCells;
      for (int l = 0; l < r; ++l) {
        int b = (q >> (r - 1 - l)) & 1;
        if (l % 2 == 0) { w /= 2; if (b) x += w; }
        else { h /= 2; if (b) y += h; }
      }
      orig[(1 << r) - 1 + q] = uint16_t(x | (y << 8));
    }
  }
  {
    // one set of tables per device (the __constant__ pointers are per device too)
    static bool built_dev[64] = {};
    static LeafTabDev tab_dev[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return -1;
    bool& built = built_dev[dev];
    LeafTabDev& tab = tab_dev[dev];
    if (!built) {
      for (int ci = 0; ci < 3; ++ci) {
        const int NC = ci == 0 ? 2 : (ci == 1 ? 4 : 8);
        std::vector<LeafItemP> vp;
        std::vector<LeafItemU> vu;
        for (int r = 0; r < 6; ++r) {
          const LeafLevel& L = T[r];
          const int K = L.K, k = L.k, ng = L.ng, ks = L.kson;
          const int W = K + NC;
          auto tri_h = [](int a) { return a * (a + 1) / 2; };
          auto symoff = [&](int i, int j) { return i >= j ? tri_h(i) + j : tri_h(j) + i; };
          const int zs = tri_h(ks) + ks * NC;        // son zero slot: sigma_0 (always 0, see leaf_level)
          tab.poff[ci][r] = int(vp.size());
          for (int g = 0; g < ng; ++g)
            for (int j = 0; j < W; ++j) {
              const int a = k + g;
              LeafItemP it{int16_t(zs), int16_t(zs), -1, 0};
              if (j < K) {
                if (L.map1[a] >= 0 && L.map1[j] >= 0) it.o1 = int16_t(symoff(L.map1[a], L.map1[j]));
                if (L.map2[a] >= 0 && L.map2[j] >= 0) it.o2 = int16_t(symoff(L.map2[a], L.map2[j]));
              } else {
                const int c = j - K;
                it.c = int16_t(c);
                if (L.map1[a] >= 0) it.o1 = int16_t(tri_h(ks) + L.map1[a] * NC + c);
                if (L.map2[a] >= 0) it.o2 = int16_t(tri_h(ks) + L.map2[a] * NC + c);
              }
              vp.push_back(it);
            }
          tab.uoff[ci][r] = int(vu.size());
          for (int a = 0; a < k; ++a)
            for (int b = 0; b <= a; ++b) {
              LeafItemU it{int16_t(a), int16_t(b), int16_t(zs), int16_t(zs)};
              if (L.map1[a] >= 0 && L.map1[b] >= 0) it.o1 = int16_t(symoff(L.map1[a], L.map1[b]));
              if (L.map2[a] >= 0 && L.map2[b] >= 0) it.o2 = int16_t(symoff(L.map2[a], L.map2[b]));
              vu.push_back(it);
            }
          for (int a = 0; a < k; ++a)
            for (int c = 0; c < NC; ++c) {
              LeafItemU it{int16_t(a), int16_t(k + c), int16_t(zs), int16_t(zs)};
              if (L.map1[a] >= 0) it.o1 = int16_t(tri_h(ks) + L.map1[a] * NC + c);
              if (L.map2[a] >= 0) it.o2 = int16_t(tri_h(ks) + L.map2[a] * NC + c);
              vu.push_back(it);
            }
        }
        void* dp = nullptr;
        void* du = nullptr;
        if (cudaMalloc(&dp, vp.size() * sizeof(LeafItemP)) != cudaSuccess) return -1;
        if (cudaMalloc(&du, vu.size() * sizeof(LeafItemU)) != cudaSuccess) return -1;
        cudaMemcpy(dp, vp.data(), vp.size() * sizeof(LeafItemP), cudaMemcpyHostToDevice);
        cudaMemcpy(du, vu.data(), vu.size() * sizeof(LeafItemU), cudaMemcpyHostToDevice);
        tab.P[ci] = static_cast<const LeafItemP*>(dp);
        tab.U[ci] = static_cast<const LeafItemU*>(du);
      }
      built = true;
    }
    if (cudaMemcpyToSymbol(c_ltab, &tab, sizeof(tab)) != cudaSuccess) return -1;
  }
  if (cudaMemcpyToSymbol(c_tmpl, &t, sizeof(t)) != cudaSuccess) return -1;
  if (cudaMemcpyToSymbol(c_map, maps, sizeof(maps)) != cudaSuccess) return -1;
  if (cudaMemcpyToSymbol(c_orig, orig, sizeof(orig)) != cudaSuccess) return -1;
  {
    uint8_t ti[64] = {}, tj[64] = {};
    for (int i = 0, t = 0; t < 64; ++i)
      for (int j = 0; j <= i && t < 64; ++j, ++t) { ti[t] = uint8_t(i); tj[t] = uint8_t(j); }
    if (cudaMemcpyToSymbol(c_tile_i, ti, sizeof(ti)) != cudaSuccess) return -1;
    if (cudaMemcpyToSymbol(c_tile_j, tj, sizeof(tj)) != cudaSuccess) return -1;
  }
  return 0;
}

// subtree-relative post-order id of in-leaf node (r, q) (for error reports)
__device__ long long inleaf_ref_id(long long leaf_id, int r, int q) {
  const int H = 8;   // in-leaf height
  long long size_leaf = (1LL << (H + 1)) - 1;
  long long id = 0;
  for (int d = 1; d <= r; ++d)
    if ((q >> (r - d)) & 1) id += (1LL << (H - d + 1)) - 1;
  id += (1LL << (H - r + 1)) - 2;
  return leaf_id - size_leaf + 1 + id;
}

__device__ __forceinline__ int tri(int a) { return (a * (a + 1)) >> 1; }

// lower-packed symmetric read
__device__ __forceinline__ double sym(const double* P, int i, int j) {
  return i >= j ? P[tri(i) + j] : P[tri(j) + i];
}

// Panel row stride of level r: >= K + NC and = 4 (mod 8), so that the DMMA operand
// fragments (4 rows x 8 consecutive doubles) hit distinct banks.
__host__ __device__ constexpr int leaf_wpad(int w) { return w + ((12 - (w & 7)) & 7); }

// Mean over a sub-leaf tree node (column code kSubMeanTag | i0 | i1 << 5 | j0 << 10 |
// j1 << 15, leaf-local cells): the lumped mean weight of leaf-local node (X, Y) —
// 2, 1, 1, 2 sixths of h^2 from the cells it is the (i,j), (i+1,j), (i,j+1), (i+1,j+1)
// corner of (functionals.py:47-61: a third of each triangle's area per vertex) —
// counting only the cells of the mean's node that lie in the block [bx0,bx1) x [by0,by1).
constexpr int kSubMeanCode = 1 << 24;
__device__ __forceinline__ double submean_weight(int code, int X, int Y, int bx0, int bx1, int by0, int by1) {
  const int x0 = max(bx0, code & 31), x1 = min(bx1, (code >> 5) & 31);
  const int y0 = max(by0, (code >> 10) & 31), y1 = min(by1, (code >> 15) & 31);
  auto cin = [&](int cx, int cy) { return (cx >= x0 && cx < x1 && cy >= y0 && cy < y1) ? 1.0 : 0.0; };
  return 2.0 * cin(X, Y) + cin(X - 1, Y) + cin(X, Y - 1) + 2.0 * cin(X - 1, Y - 1);
}
__device__ __forceinline__ double submean_inv_area(int code, double h) {
  return 1.0 / (double((((code >> 5) & 31) - (code & 31)) * (((code >> 15) & 31) - ((code >> 10) & 31))) * h * h);
}

// Gather programs: read through L1 (__ldg; the tables of a class are shared by every
// CTA) — no staging buffers, so the 2-column class fits 3 CTAs per SM and the
// 8-column class 2 (measured: C2 leaf 7.01 -> 6.11 ms, C4 26.8 -> 22.8 ms against
// cp.async staging in smem, which HDD_LEAF_STAGE_ITEMS restores).
#ifdef HDD_LEAF_STAGE_ITEMS
constexpr bool kLeafStage = true;
#else
constexpr bool kLeafStage = false;
#endif

// Leaf smem layout (doubles): col info [hdr] | arena [T] | gather programs (only with
// HDD_LEAF_STAGE_ITEMS: panel program of even levels [tp0] | of odd levels [tp1] | update
// program [tu]).  In the arena the level outputs ping-pong between its two ends: even
// levels write at the bottom, odd levels (and the fused 6+5 output) at the top, and a
// level's interface panel sits right above the bottom region.  kappa[512] and f[289]
// occupy the bottom until level 4 writes it.  T is the largest (input + output + panel)
// of any level, so the 2-column class fits four CTAs per SM.
// A node block is [Psi packed tri(k) | R k x NC | sigma NC]; sigma_0 (the load column)
// is 0 at every in-leaf level and doubles as the gather programs' zero slot.
__host__ __device__ constexpr int leaf_node_elems(int k, int nc) { return ctri(k) + k * nc + nc; }
// node blocks of a level sit at an odd stride (doubles): lane-per-node accesses (the fused
// 6+5 build) hit 16 distinct 8-byte banks
__host__ __device__ constexpr int leaf_node_stride(int k, int nc) { return leaf_node_elems(k, nc) | 1; }
__host__ __device__ constexpr int leaf_out_elems(int r, int nc) { return (1 << r) * leaf_node_stride(leaf_shape(r).k, nc); }
// panel row stride: DMMA-conflict-free padding where phase D runs on DMMA (ng > 3)
__host__ __device__ constexpr int leaf_panel_w(int r, int nc) {
  return leaf_shape(r).ng == 3 ? leaf_shape(r).K + nc : leaf_wpad(leaf_shape(r).K + nc);
}
__host__ __device__ constexpr int leaf_panel_elems(int r, int nc) { return (1 << r) * leaf_shape(r).ng * leaf_panel_w(r, nc); }
__host__ __device__ constexpr int leaf_hdr(int nc) { return (3 * nc + 1) & ~1; }   // 6 NC ints
struct LeafSmem {
  int T, hdr, tp0, tp1, tu;
  int group_doubles;       // smem doubles per (leaf, sample) group of a CTA (HDD_LEAF_G)
};
static LeafSmem leaf_sizes(int ncl) {
  const auto& Tm = leaf_template();
  LeafSmem s{808 + leaf_out_elems(5, ncl), leaf_hdr(ncl), 0, 0, 0};   // kappa + f below the fused 6+5 output
  for (int r = 0; r <= 4; ++r)
    s.T = std::max(s.T, leaf_out_elems(r, ncl) + leaf_out_elems(r + 1, ncl) + leaf_panel_elems(r, ncl));
  for (int r = 0; r < kLeafLevels && r <= 5; ++r) {
    const int k = Tm[r].k, K = Tm[r].K, ng = Tm[r].ng;
    int& tp = (r & 1) ? s.tp1 : s.tp0;
    if (kLeafStage) {
      tp = std::max(tp, ng * (K + ncl));
      s.tu = std::max(s.tu, k * (k + 1) / 2 + k * ncl);
    }
  }
  for (int* v : {&s.T, &s.tp0, &s.tp1, &s.tu}) *v = (*v + 1) & ~1;
  return s;
}

size_t leaf_smem_bytes(int ncl) {
  const LeafSmem s = leaf_sizes(ncl);
  return sizeof(double) * (size_t(s.hdr) + s.T + s.tp0 + s.tp1 + s.tu);
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Gather programs: staged in smem (cp.async) or, with HDD_LEAF_GLOBAL_ITEMS, read
// through L1 (__ldg) — no staging buffers, so the 2-column class fits 3 CTAs per SM.
template <typename T>
__device__ __forceinline__ T load_item(const T* p, int t) {
  static_assert(sizeof(T) == 8, "8-byte gather items");
  const unsigned long long v = __ldg(reinterpret_cast<const unsigned long long*>(p) + t);
  T it;
  memcpy(&it, &v, 8);
  return it;
}

template <int R, int NC, int NTH>
__device__ __forceinline__ void stage_panel_program(uint64_t* dst) {
  constexpr LeafLevelShape S = leaf_shape(R);
  constexpr int CI = NC == 2 ? 0 : (NC == 4 ? 1 : 2);
  constexpr int NPI = S.ng * (S.K + NC);
  const LeafItemP* g = c_ltab.P[CI] + c_ltab.poff[CI][R];
  if constexpr (kLeafStage)
    for (int t = threadIdx.x % NTH; t < NPI; t += NTH) cp_async8(dst + t, g + t);
  cp_async_commit();
}

// TMA bulk copies (cp.async.bulk, global -> shared) completing on an mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// TMA bulk store shared -> global (bulk group; wait with bulk_wait_read0 before the smem
// is reused or the CTA exits); generic-proxy smem writes need fence_proxy_async_smem first
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
               ::"l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// TMA bulk prefetch of a global range into L2 (no shared memory, no completion)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n"
               ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

// 1/d: MUFU seed + two Newton steps (full double precision)
__device__ __forceinline__ double rcp_nr(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  y = fma(y, fma(-d, y, 1.0), y);
  y = fma(y, fma(-d, y, 1.0), y);
  return y;
}

// 1/sqrt(d): MUFU seed + two Newton steps (full double precision for the
// well-scaled pivots of the in-leaf factorizations)
__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double hd = 0.5 * d;
  y = y * fma(-hd * y, y, 1.5);
  y = y * fma(-hd * y, y, 1.5);
  return y;
}

// One in-leaf level: sons (level R+1, packed) in `in`, outputs (level R) to `out`
// (level 0: `out` is shared-memory staging, copied to the leaf's global block at the end).
//   A  gather the interface panel [A21 | A22 | R_gamma] (all warps)
//   B  Cholesky of A22 in registers (1-2 warps) || the other warps gather the
//      sons' contributions A~ = Psi_s1 + Psi_s2 (and R_B) into `out`
//   C  [W | V] = L^-1 [A21 | R_gamma] in place (thread per column)
//   D  out -= W^T [W | V] on 8x8 DMMA tiles; sigma += V_0^T V
#ifndef HDD_LEAF_G
#define HDD_LEAF_G 1     // (leaf, sample) groups per leaf CTA, see leaf2_kernel
#endif
// barrier of one (leaf, sample) group: the CTA barrier, or with HDD_LEAF_G > 1 and
// HDD_LEAF_NAMED a named barrier per group (groups start together and may drift)
#if defined(HDD_LEAF_NAMED) && HDD_LEAF_G > 1
#define LEAF_SYNC() asm volatile("bar.sync %0, %1;" ::"r"(int(threadIdx.x / NTH) + 1), "n"(NTH) : "memory")
#else
#define LEAF_SYNC() __syncthreads()
#endif
template <int R, int NC, int NTH, bool EXT = false>
__device__ __forceinline__ void leaf_level(const DevPlan& p, const double* __restrict__ in, double* __restrict__ out,
                                           double* __restrict__ pan, const int* __restrict__ cinfo, int leaf,
                                           int s, long long leaf_ref, const uint64_t* __restrict__ tabP,
                                           uint64_t* __restrict__ tabPnext, uint64_t* __restrict__ tabU) {
  constexpr LeafLevelShape S = leaf_shape(R);
  constexpr int K = S.K, k = S.k, ng = S.ng, ks = S.ks;
  constexpr int nf = 1 << R;
  constexpr int Sin = leaf_node_stride(ks, NC);
  constexpr int Sout = leaf_node_stride(k, NC);
  constexpr int Zin = ctri(ks) + ks * NC;              // zero slot: the sons' sigma_0
  constexpr int WL = K + NC;                // logical panel row (program layout)
  constexpr int W = leaf_panel_w(R, NC);    // panel row stride
  constexpr int WX = k + NC;
  constexpr int NT = NTH, NW = NTH / 32;
  constexpr int gsz = nf >= NW ? 1 : NW / nf;
  constexpr int qstep = NW / gsz;
  constexpr int CI = NC == 2 ? 0 : (NC == 4 ? 1 : 2);
  constexpr int NPI = ng * WL, NUI = ctri(k) + k * NC;
  // ng = 3 levels (4 and 3): the sons' contributions and the rank-3 Schur update run as
  // one pass per output element (phase E) instead of B' plus DMMA blocks
  constexpr bool kE = ng == 3;
  constexpr int LPN = ng <= 1 ? 1 : (ng <= 4 ? 4 : (ng <= 8 ? 8 : 16));   // Cholesky lanes per node
  constexpr int NPW = 32 / LPN;                                           // nodes per Cholesky warp
  constexpr int NWB = (nf + NPW - 1) / NPW;                               // Cholesky warps
  static_assert(NWB < NW, "the sons' gather needs free warps");
  const int tid = threadIdx.x % NTH, lane = tid & 31;   // NTH threads per (leaf, sample) group
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);   // provably warp-uniform
  const int sub = warp % gsz;
  const int* ctype = cinfo;
  const int* br = cinfo + NC;
  const int* bq = cinfo + 2 * NC;
  const int* bg = cinfo + 3 * NC;
  double* Pp = pan;

  {   // this level's update program (the single U buffer is free: the previous level is done)
    const LeafItemU* gu = c_ltab.U[CI] + c_ltab.uoff[CI][R];
    if constexpr (kLeafStage)
      for (int t = tid; t < NUI; t += NT) cp_async8(tabU + t, gu + t);
    cp_async_commit();
  }
  cp_async_wait<1>();   // this level's panel program (issued one level earlier) has landed
  LEAF_SYNC();
  // ---- A: gather the interface panel (precomputed program) ----
  // The program of a level is the same for its nf nodes: a thread decodes item t once
  // and applies it to every node q (compile-time strides 2 Sin / ng W), UT items in
  // flight when nf is small.
  {
    const LeafItemP* prog = kLeafStage ? reinterpret_cast<const LeafItemP*>(tabP) : c_ltab.P[CI] + c_ltab.poff[CI][R];
    constexpr int UT = nf >= 4 ? 1 : 4 / nf;
    for (int t0 = tid; t0 < NPI; t0 += UT * NT) {
      int o1[UT], o2[UT];
#pragma unroll
      for (int u = 0; u < UT; ++u) {
        const int t = t0 + u * NT;
        LeafItemP it = LeafItemP{int16_t(Zin), int16_t(Zin), -1, 0};
        if (t < NPI) {
          if constexpr (kLeafStage) it = prog[t];
          else it = load_item(prog, t);
        }
        o1[u] = it.o1;
        o2[u] = Sin + it.o2;
      }
      double v[UT][nf];
#pragma unroll
      for (int u = 0; u < UT; ++u)
#pragma unroll
        for (int q = 0; q < nf; ++q) v[u][q] = in[2 * q * Sin + o1[u]] + in[2 * q * Sin + o2[u]];
#pragma unroll
      for (int u = 0; u < UT; ++u) {
        const int t = t0 + u * NT;
        if (t < NPI) {
          double* P = Pp + (t / WL) * W + (t - (t / WL) * WL);
#pragma unroll
          for (int q = 0; q < nf; ++q) P[q * ng * W] = v[u][q];
        }
      }
    }
  }
  cp_async_wait<0>();   // update program landed
  LEAF_SYNC();
  if constexpr (R > 0) stage_panel_program<R - 1, NC, NTH>(tabPnext);
  LEAF_TICK(10 + 8 * (5 - R) + 0);
  if (warp < NWB) {
    // ---- B: Cholesky A22 = L L^T, a lane per row, LPN lanes per node, column
    // broadcasts by shuffles; L back below the diagonal, 1/L_jj on it.  A
    // non-positive pivot is a NumericalError, exactly like the reference's failed
    // Cholesky (hdd.py:263-270 without the indefinite fallback).
    const int i = lane % LPN;
    const int q = warp * NPW + lane / LPN;
    const bool act = q < nf && i < ng;
    double* P = Pp + (act ? q : 0) * ng * W + k;     // A22[i][l] = P[i * W + l]
    double a[ng];
#pragma unroll
    for (int l = 0; l < ng; ++l) a[l] = (act && l <= i) ? P[i * W + l] : (l == i ? 1.0 : 0.0);
    bool bad = false;
    // unscaled (LDL^T-ordered) elimination: a_il -= a_ij a_lj / d_j.  The column
    // broadcast a_lj does not wait for the pivot's reciprocal, so the serial chain per
    // step is shuffle -> rcp -> mul -> fma; the sqrt scaling of column j runs beside it
#pragma unroll
    for (int j = 0; j < ng; ++j) {
      const double dj = __shfl_sync(0xffffffffu, a[j], j, LPN);
      bad |= !(dj > 0.0);
      const double rj = rcp_nr(dj);
      const double sj = a[j] * rj;
#pragma unroll
      for (int l = j + 1; l < ng; ++l) a[l] = fma(-sj, __shfl_sync(0xffffffffu, a[j], l, LPN), a[l]);
      const double il = rsqrt_nr(dj);
      a[j] = i == j ? il : a[j] * il;
    }
    if (act) {
#pragma unroll
      for (int l = 0; l < ng; ++l)
        if (l <= i) P[i * W + l] = a[l];
      if (i == 0 && bad) record_error(p, HDD_ERR_NUMERICAL, s, inleaf_ref_id(leaf_ref, R, q));
    }
    LEAF_TICK(10 + 8 * (5 - R) + 4);
#ifdef HDD_AB_SERIAL_B
    if (R == 0) asm volatile("bar.arrive 1, %0;" ::"n"(NT));
#endif
  } else {
#ifdef HDD_AB_SERIAL_B
    if (R == 0) asm volatile("bar.sync 1, %0;" ::"n"(NT));
#endif
    // ---- B': sons' contributions to the outputs, A~ = Psi_s1 + Psi_s2 | R_s1 + R_s2 ----
    // (item t decoded once for the level's nf nodes, as in A)
    const LeafItemU* uprog = kLeafStage ? reinterpret_cast<const LeafItemU*>(tabU) : c_ltab.U[CI] + c_ltab.uoff[CI][R];
    constexpr int UB = nf >= 4 ? 1 : 4 / nf;
    const int wt = (warp - NWB) * 32 + lane, nth = (NW - NWB) * 32;
    for (int t0 = wt; !kE && t0 < NUI; t0 += UB * nth) {
      int o1[UB], o2[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int t = t0 + u * nth;
        LeafItemU it = LeafItemU{0, 0, int16_t(Zin), int16_t(Zin)};
        if (t < NUI) {
          if constexpr (kLeafStage) it = uprog[t];
          else it = load_item(uprog, t);
        }
        o1[u] = it.o1;
        o2[u] = Sin + it.o2;
      }
      double v[UB][nf];
#pragma unroll
      for (int u = 0; u < UB; ++u)
#pragma unroll
        for (int q = 0; q < nf; ++q) v[u][q] = in[2 * q * Sin + o1[u]] + in[2 * q * Sin + o2[u]];
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int t = t0 + u * nth;
        if (t < NUI)
#pragma unroll
          for (int q = 0; q < nf; ++q) out[q * Sout + t] = v[u][q];
      }
    }
    // functional births at this level: +1 in the panel's R_gamma column
    if (warp == NW - 1 && lane < NC && br[lane] == R)
      Pp[bq[lane] * ng * W + bg[lane] * W + K + lane] += 1.0;
  }
  LEAF_SYNC();
  LEAF_TICK(10 + 8 * (5 - R) + 1);
  // ---- C: [W | V] = L^-1 [A21 | R_gamma] in place, a thread per column ----
  for (int t = tid; t < nf * WX; t += NT) {
    const int q = t / WX, jj = t - (t / WX) * WX;
    const int col = jj < k ? jj : K + (jj - k);
    double* P = Pp + q * ng * W;
    double w[ng];
#pragma unroll
    for (int g = 0; g < ng; ++g) w[g] = P[g * W + col];     // all loads ahead of the stores
#pragma unroll
    for (int g = 0; g < ng; ++g) {
      double v = w[g];
#pragma unroll
      for (int h = 0; h < g; ++h) v = fma(-P[g * W + k + h], w[h], v);
      w[g] = v * P[g * W + k + g];
    }
#pragma unroll
    for (int g = 0; g < ng; ++g) P[g * W + col] = w[g];
  }
  LEAF_SYNC();
  LEAF_TICK(10 + 8 * (5 - R) + 2);
  // ---- D: out -= W^T [W | V]; sigma += V_0^T V ----
  if constexpr (kE) {
    // ---- E: out = Psi_s1 + Psi_s2 - W^T [W | V] per output element (item t decoded once
    // for the nf nodes; rank-3 update in DFMA) ----
    const LeafItemU* uprog = kLeafStage ? reinterpret_cast<const LeafItemU*>(tabU) : c_ltab.U[CI] + c_ltab.uoff[CI][R];
    for (int t = tid; t < NUI; t += NT) {
      const LeafItemU it = kLeafStage ? uprog[t] : load_item(uprog, t);
      const int a = it.a, bc = it.bx < k ? it.bx : K + (it.bx - k);
      const int o1 = it.o1, o2 = Sin + it.o2;
      double v[nf];
#pragma unroll
      for (int q = 0; q < nf; ++q) v[q] = in[2 * q * Sin + o1] + in[2 * q * Sin + o2];
#pragma unroll
      for (int q = 0; q < nf; ++q) {
        const double* P = Pp + q * ng * W;
#pragma unroll
        for (int g = 0; g < ng; ++g) v[q] = fma(-P[g * W + a], P[g * W + bc], v[q]);
        out[q * Sout + t] = v[q];
      }
    }
  } else if constexpr (ng >= 3) {
    // 16x16 output blocks (2x2 DMMA m8n8k4 tiles; interface dimension padded to 4):
    // lower-triangle Psi blocks, then 16x8 blocks for the R columns
    constexpr int nB = (k + 15) / 16, TPN = ctri(nB) + nB, KS = (ng + 3) / 4;
    constexpr int NBLK = nf * TPN;
    const int lr = lane >> 2, lc = lane & 3;
    for (int w = warp; w < NBLK; w += NW) {
      const int q = w / TPN;
      const int tt = w - q * TPN;
      const bool rt = tt >= ctri(nB);
      const int bi = rt ? tt - ctri(nB) : c_tile_i[tt];
      const int bj = rt ? 0 : c_tile_j[tt];
      const double* P = Pp + q * ng * W;
      double* o = out + q * Sout;
      if (!rt && bj < bi && 16 * bi + 16 <= k) {
        // strictly-lower 16x16 block with every row inside: no per-element predicates
        const int a0 = 16 * bi + lr, b0 = 16 * bj + 2 * lc;
        double* o0 = o + ctri(a0) + b0;
        double* o1 = o + ctri(a0 + 8) + b0;
        double old[2][2][2], acc[2][2][2];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            old[0][j][e] = o0[8 * j + e];
            old[1][j][e] = o1[8 * j + e];
            acc[0][j][e] = 0.0;
            acc[1][j][e] = 0.0;
          }
        const int ca0 = 16 * bi + lr, cb0 = 16 * bj + lr;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
          const int g = 4 * kk + lc;
          const bool gv = g < ng;
          const double* pr = P + g * W;
          const double x0 = gv ? pr[ca0] : 0.0, x1 = gv ? pr[ca0 + 8] : 0.0;
          const double y0 = gv ? pr[cb0] : 0.0, y1 = gv ? pr[cb0 + 8] : 0.0;
          dmma884(acc[0][0], x0, y0);
          dmma884(acc[0][1], x0, y1);
          dmma884(acc[1][0], x1, y0);
          dmma884(acc[1][1], x1, y1);
        }
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            o0[8 * j + e] = old[0][j][e] - acc[0][j][e];
            o1[8 * j + e] = old[1][j][e] - acc[1][j][e];
          }
        continue;
      }
      if (!rt && bj == bi && 16 * bi + 16 <= k) {
        // diagonal 16x16 block: the upper-right 8x8 is never stored (no DMMA), the
        // lower-left one always is, the two diagonal 8x8 keep b <= a
        const int a0 = 16 * bi + lr, b0 = 16 * bi + 2 * lc;
        double* o0 = o + ctri(a0) + b0;
        double* o1 = o + ctri(a0 + 8) + b0;
        double old00[2], old10[2], old11[2], acc00[2] = {0.0, 0.0}, acc10[2] = {0.0, 0.0}, acc11[2] = {0.0, 0.0};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const bool dg = 2 * lc + e <= lr;
          old00[e] = dg ? o0[e] : 0.0;
          old10[e] = o1[e];
          old11[e] = dg ? o1[8 + e] : 0.0;
        }
        const int ca0 = 16 * bi + lr;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
          const int g = 4 * kk + lc;
          const bool gv = g < ng;
          const double* pr = P + g * W;
          const double x0 = gv ? pr[ca0] : 0.0, x1 = gv ? pr[ca0 + 8] : 0.0;
          dmma884(acc00, x0, x0);
          dmma884(acc10, x1, x0);
          dmma884(acc11, x1, x1);
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const bool dg = 2 * lc + e <= lr;
          if (dg) o0[e] = old00[e] - acc00[e];
          o1[e] = old10[e] - acc10[e];
          if (dg) o1[8 + e] = old11[e] - acc11[e];
        }
        continue;
      }
      if (rt && 16 * bi + 16 <= k) {
        // R block with every row inside: columns c = 2 lc + e < NC
        const int a0 = 16 * bi + lr, c0 = 2 * lc;
        double* o0 = o + ctri(k) + a0 * NC + c0;
        double* o1 = o0 + 8 * NC;
        const bool cv0 = c0 < NC, cv1 = c0 + 1 < NC;
        double old0[2], old1[2], acc0[2] = {0.0, 0.0}, acc1[2] = {0.0, 0.0};
        old0[0] = cv0 ? o0[0] : 0.0; old0[1] = cv1 ? o0[1] : 0.0;
        old1[0] = cv0 ? o1[0] : 0.0; old1[1] = cv1 ? o1[1] : 0.0;
        const int ca0 = 16 * bi + lr;
        const bool vy = lr < NC;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
          const int g = 4 * kk + lc;
          const bool gv = g < ng;
          const double* pr = P + g * W;
          const double x0 = gv ? pr[ca0] : 0.0, x1 = gv ? pr[ca0 + 8] : 0.0;
          const double y0 = (gv && vy) ? pr[K + lr] : 0.0;
          dmma884(acc0, x0, y0);
          dmma884(acc1, x1, y0);
        }
        if (cv0) { o0[0] = old0[0] - acc0[0]; o1[0] = old1[0] - acc1[0]; }
        if (cv1) { o0[1] = old0[1] - acc0[1]; o1[1] = old1[1] - acc1[1]; }
        continue;
      }
      // output offsets of this lane's accumulator elements (-1: not stored), old
      // values (the sons' contributions, written by B') fetched ahead of the DMMAs
      int ov[2][2][2];
      double old[2][2][2], acc[2][2][2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int a = 16 * bi + 8 * i + lr;
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            int t = -1;
            if (a < k) {
              if (!rt) {
                const int b = 16 * bj + 8 * j + 2 * lc + e;
                if (b <= a) t = ctri(a) + b;
              } else if (j == 0 && 2 * lc + e < NC) {
                t = ctri(k) + a * NC + 2 * lc + e;
              }
            }
            ov[i][j][e] = t;
            old[i][j][e] = t < 0 ? 0.0 : o[t];
            acc[i][j][e] = 0.0;
          }
      }
      int ca[2], cb[2];
      bool vca[2], vcb[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        ca[i] = 16 * bi + 8 * i + lr;
        vca[i] = ca[i] < k;
        cb[i] = rt ? K + lr : 16 * bj + 8 * i + lr;
        vcb[i] = rt ? (i == 0 && lr < NC) : cb[i] < k;
      }
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        const int g = 4 * kk + lc;
        const double* pr = P + g * W;
        double x[2], y[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          x[i] = (vca[i] && g < ng) ? pr[ca[i]] : 0.0;
          y[i] = (vcb[i] && g < ng) ? pr[cb[i]] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          dmma884(acc[i][0], x[i], y[0]);
          if (!rt) dmma884(acc[i][1], x[i], y[1]);
        }
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            if (ov[i][j][e] >= 0) o[ov[i][j][e]] = old[i][j][e] - acc[i][j][e];
    }
  } else {
    // ng = 1: rank-1 update, a thread per output element
    const double* P0 = Pp;
    for (int idx = tid; idx < nf * NUI; idx += NT) {
      const int q = idx / NUI, t = idx - q * NUI;
      const LeafItemU it = kLeafStage ? reinterpret_cast<const LeafItemU*>(tabU)[t]
                                      : load_item(c_ltab.U[CI] + c_ltab.uoff[CI][R], t);
      const int bx = it.bx;
      const double* P = P0 + q * ng * W;
      out[q * Sout + t] -= P[it.a] * P[bx < k ? bx : K + (bx - k)];
    }
  }
  // sigma row: sigma_c = sigma_s1 + sigma_s2 + V_0^T V_c (column 0 is the load)
  for (int q = warp; q < nf; q += NW) {
    if (lane < NC) {
      const double* P = Pp + q * ng * W;
      const int c = lane;
      double sg = in[(2 * q) * Sin + ctri(ks) + ks * NC + c] + in[(2 * q + 1) * Sin + ctri(ks) + ks * NC + c];
      if (c >= 1)
#pragma unroll
        for (int g = 0; g < ng; ++g) sg = fma(P[g * W + K], P[g * W + K + c], sg);
      double* o = out + q * Sout;
      o[ctri(k) + k * NC + c] = sg;        // sigma_0 = 0 + 0: the next level's zero slot
    }
  }
  if constexpr (R == 0) fence_proxy_async_smem();   // the Psi block is read by the bulk copy below
  LEAF_SYNC();
  if constexpr (R == 0) {
    // leaf output: Psi packed lower, R [64][leaf_cols] (mean columns rescaled by
    // 1/|leaf|, an exact power of two), sigma; primal-mode leaf functionals
    const double inv_area = 1.0 / (double(kLeafCells * kLeafCells) * p.h * p.h);
    double* gdst = p.buf[p.leaf_buf] + int64_t(leaf) * p.leaf_elems * p.bcap + int64_t(s) * p.leaf_elems;
    // Psi (tri(64) doubles, 16-byte aligned at both ends): one TMA bulk store, waited
    // for (smem reads done) before the CTA exits
    static_assert((ctri(k) * 8) % 16 == 0, "bulk copies move 16-byte multiples");
    if (blockIdx.z == 0 && tid == 0) bulk_s2g(gdst, out, uint32_t(ctri(k) * 8));
    // Dirichlet data g on the domain boundary (known perimeter values u_D = g_D):
    // load rows r_a -= Psi_aD g_D, functional columns sigma_c += R_c(D)^T g_D
    const bool hasg = EXT && (p.leaf_g || p.gcall);
    for (int t = tid; t < (k + 1) * NC; t += NT) {
      const int a = t / NC, c = t - (t / NC) * NC;
      const int col = cinfo[5 * NC + c];
      if (col < 0) continue;
      const int ct = ctype[c];
      double raw = out[ctri(k) + a * NC + c];
      if (hasg) {
        if (ct == 0 && a < k) {
          for (int d = 0; d < k; ++d) {
            const double gd = leaf_gval(p, leaf, s, d);
            if (gd != 0.0) raw -= out[a >= d ? tri(a) + d : tri(d) + a] * gd;
          }
        } else if (ct != 0 && a == k) {
          for (int d = 0; d < k; ++d) {
            const double gd = leaf_gval(p, leaf, s, d);
            if (gd != 0.0) raw += out[ctri(k) + d * NC + c] * gd;
          }
        }
      }
      const double val = raw * (ct == 1 ? inv_area : ((EXT && ct >= kSubMeanCode) ? submean_inv_area(ct, p.h) : 1.0));
      gdst[ctri(k) + a * p.leaf_cols + col] = val;
      const int fs = cinfo[4 * NC + c];
      if (fs >= 0) p.fbuf[(int64_t(s) * p.n_fslots + fs) * 65 + a] = val;
    }
  }
  LEAF_TICK(10 + 8 * (5 - R) + 3);
}

// ---- levels 6 + 5 fused: per-node algebra (leaf2_kernel) ----
// A level-5 node (2 x 4 cells, 3 x 5 nodes) has 12 boundary nodes and 3 interior ones
// (the 2x2-block centres c1 = (1,1), c2 = (1,3) and the level-5 interface node
// m = (1,2)); A_II is tridiagonal and every boundary node couples to at most one
// interior node, so  Psi = A_BB - v_a M(g_a, g_b) v_b,  R = r_B - v_a (M r_I)(g_a),
// sigma_c = r_0I^T M r_cI  with M = A_II^-1 in closed form: the block elimination of
// the level-6 and level-5 steps (fem.py:126-145 cell patterns).
// Boundary index <-> local node (sorted (y, x) like the leaf template); interior
// neighbour 0 = c1, 1 = m, 2 = c2, -1 none.
__host__ __device__ constexpr int l56_bx(int i) { return i < 3 ? i : (i < 9 ? (((i - 3) & 1) ? 2 : 0) : i - 9); }
__host__ __device__ constexpr int l56_by(int i) { return i < 3 ? 0 : (i < 9 ? (i - 3) / 2 + 1 : 4); }
__host__ __device__ constexpr int l56_bg(int i) {
  return i == 1 || i == 3 || i == 4 ? 0 : (i == 5 || i == 6 ? 1 : (i == 7 || i == 8 || i == 10 ? 2 : -1));
}
// boundary neighbours of row a with a smaller index: left (x - 1) and down (y - 1), -1 none
__host__ __device__ constexpr int l56_left(int a) {
  return (l56_bx(a) >= 1 && (l56_by(a) == 0 || l56_by(a) == 4 || l56_bx(a) == 2))
             ? (l56_bx(a) == 2 && l56_by(a) >= 1 && l56_by(a) <= 3 ? -1 : a - 1) : -1;
}
__host__ __device__ constexpr int l56_down(int a) {
  return (l56_by(a) >= 1 && l56_bx(a) != 1)
             ? (l56_by(a) == 1 ? (l56_bx(a) == 0 ? 0 : 2) : (l56_by(a) == 4 ? (l56_bx(a) == 0 ? 7 : 8) : a - 2)) : -1;
}

struct L56Node {
  const double* kap;    // the leaf's kappa, [x][2 y + type]
  const double* fl;     // nodal f of the leaf (17 x 17) or null
  int ox, oy;
  double h2_6, h2;
  // kappa rows are rotated by (x >> 1) & 7 doubles (leaf2_kernel's load): the 32 nodes'
  // lane-parallel reads spread over the banks
  __device__ __forceinline__ double k0(int cx, int cy) const {
    return kap[(ox + cx) * 32 + ((2 * (oy + cy) + (ox >> 1)) & 31)];
  }
  __device__ __forceinline__ double k1(int cx, int cy) const {
    return kap[(ox + cx) * 32 + ((2 * (oy + cy) + 1 + (ox >> 1)) & 31)];
  }
  static __device__ __forceinline__ bool in_(int cx, int cy) { return cx >= 0 && cx < 2 && cy >= 0 && cy < 4; }
  __device__ __forceinline__ double Dl(int x, int y) const {
    double d = 0.0;
    if (in_(x, y)) d += 0.5 * (k0(x, y) + k1(x, y));
    if (in_(x - 1, y)) d += k0(x - 1, y);
    if (in_(x, y - 1)) d += k1(x, y - 1);
    if (in_(x - 1, y - 1)) d += 0.5 * (k0(x - 1, y - 1) + k1(x - 1, y - 1));
    return d;
  }
  __device__ __forceinline__ double El(int x, int y) const {   // (x,y)-(x+1,y)
    double e = 0.0;
    if (in_(x, y)) e -= 0.5 * k0(x, y);
    if (in_(x, y - 1)) e -= 0.5 * k1(x, y - 1);
    return e;
  }
  __device__ __forceinline__ double Nl(int x, int y) const {   // (x,y)-(x,y+1)
    double e = 0.0;
    if (in_(x, y)) e -= 0.5 * k1(x, y);
    if (in_(x - 1, y)) e -= 0.5 * k0(x - 1, y);
    return e;
  }
  __device__ __forceinline__ double wl(int x, int y) const {   // lumped load weight
    double w = 0.0;
    if (in_(x, y)) w += 2.0;
    if (in_(x - 1, y)) w += 1.0;
    if (in_(x, y - 1)) w += 1.0;
    if (in_(x - 1, y - 1)) w += 2.0;
    return w * h2_6;
  }
  __device__ __forceinline__ double fv(int x, int y) const { return fl ? fl[(oy + y) * 17 + ox + x] : 1.0; }
  // boundary-interior coupling of boundary node b (compile-time b)
  __device__ __forceinline__ double vb(int b) const {
    return b == 1 ? Nl(1, 0) : b == 3 ? El(0, 1) : b == 4 ? El(1, 1) : b == 5 ? El(0, 2) : b == 6 ? El(1, 2)
         : b == 7 ? El(0, 3) : b == 8 ? El(1, 3) : b == 10 ? Nl(1, 3) : 0.0;
  }
};

// Row A of one node's outputs (Psi row, R row; sigma and the zero slot with row 0): the
// lane owns the node, the warp owns the row, so every index below is a compile-time
// constant and only the kappa-dependent values are computed.
template <int A, int NC, bool SUB>
__device__ __forceinline__ void l56_row(const L56Node& n, const double (&M)[6], double* __restrict__ out,
                                        const int* ctype, const int* br, const int* bq, int q) {
  constexpr int k5 = 12;
  constexpr int xa = l56_bx(A), ya = l56_by(A), ga = l56_bg(A);
  constexpr int il = l56_left(A), idn = l56_down(A);
  // M = [[M0 M1 M2] [M1 M3 M4] [M2 M4 M5]]
  auto Mg = [&](int g, int h) -> double {
    const int lo = g < h ? g : h, hi = g < h ? h : g;
    return lo == 0 ? M[hi] : (lo == 1 ? M[2 + hi] : M[5]);
  };
  double ma0 = 0.0, ma1 = 0.0, ma2 = 0.0;      // row g_a of M, times v_a
  if constexpr (ga >= 0) {
    const double va = n.vb(A);
    ma0 = Mg(ga, 0) * va;
    ma1 = Mg(ga, 1) * va;
    ma2 = Mg(ga, 2) * va;
  }
#pragma unroll
  for (int b = 0; b <= A; ++b) {
    double val = b == A ? n.Dl(xa, ya) : (b == il ? n.El(xa - 1, ya) : (b == idn ? n.Nl(xa, ya - 1) : 0.0));
    const int gb = l56_bg(b);
    if (ga >= 0 && gb >= 0) val -= (gb == 0 ? ma0 : (gb == 1 ? ma1 : ma2)) * n.vb(b);
    out[ctri(A) + b] = val;
  }
  const double wa = n.wl(xa, ya), fa = n.fv(xa, ya);
  const double fI0 = n.fv(1, 1), fI1 = n.fv(1, 2), fI2 = n.fv(1, 3);
  double r00 = 0.0, r01 = 0.0, r02 = 0.0;        // load column interior rhs
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int ct = ctype[c];
    double r0 = 0.0, r1 = 0.0, r2 = 0.0;
    if (ct == 0) { r0 = n.h2 * fI0; r1 = n.h2 * fI1; r2 = n.h2 * fI2; }
    else if (ct == 1) { r0 = n.h2; r1 = n.h2; r2 = n.h2; }
    else if (SUB && ct >= kSubMeanCode) {
      r0 = n.h2_6 * submean_weight(ct, n.ox + 1, n.oy + 1, n.ox, n.ox + 2, n.oy, n.oy + 4);
      r1 = n.h2_6 * submean_weight(ct, n.ox + 1, n.oy + 2, n.ox, n.ox + 2, n.oy, n.oy + 4);
      r2 = n.h2_6 * submean_weight(ct, n.ox + 1, n.oy + 3, n.ox, n.ox + 2, n.oy, n.oy + 4);
    }
    if (br[c] == 6 && bq[c] == 2 * q) r0 += 1.0;
    if (br[c] == 6 && bq[c] == 2 * q + 1) r2 += 1.0;
    if (br[c] == 5 && bq[c] == q) r1 += 1.0;
    if (c == 0) { r00 = r0; r01 = r1; r02 = r2; }
    double val = ct == 0 ? wa * fa : (ct == 1 ? wa : 0.0);
    if (SUB && ct >= kSubMeanCode) val = n.h2_6 * submean_weight(ct, n.ox + xa, n.oy + ya, n.ox, n.ox + 2, n.oy, n.oy + 4);
    if constexpr (ga >= 0) val -= ma0 * r0 + ma1 * r1 + ma2 * r2;
    out[ctri(k5) + A * NC + c] = val;
    if constexpr (A == 0) {
      double sg = 0.0;
      if (c >= 1) {
        const double t0 = M[0] * r0 + M[1] * r1 + M[2] * r2;
        const double t1 = M[1] * r0 + M[3] * r1 + M[4] * r2;
        const double t2 = M[2] * r0 + M[4] * r1 + M[5] * r2;
        sg = r00 * t0 + r01 * t1 + r02 * t2;
      }
      out[ctri(k5) + k5 * NC + c] = sg;
    }
  }
}

// One CTA per (16x16-cell leaf, sample).  Level 6 (2x2-cell blocks) is built per
// thread in registers straight from the cells' kappa; levels 5..0 run
// level-synchronously in shared memory with lower-packed Schur complements:
// gather the interface panel, Gauss-Jordan interface inverse (warp per node),
// Y = A22^-1 [A21 | R], then the Schur update A11 - A21^T Y on DMMA tiles.
// HDD_LEAF_G > 1: G (leaf, sample) groups of NTH threads per CTA, the same leaf for G
// consecutive samples.  The groups run in lockstep (every barrier is CTA-wide), so they
// fetch each instruction line together: the kernel is ~120 KB of straight-line code run
// once per item, far beyond the 32 KB L1.5 instruction cache (ncu: icc hit rate 75 %).
__host__ __device__ constexpr int leaf_minb(int nc) { return kLeafStage ? 2 : (nc == 2 ? 4 : (nc == 4 ? 3 : 2)); }
__host__ __device__ constexpr int leaf_groups(int nc) { return leaf_minb(nc) % HDD_LEAF_G == 0 ? HDD_LEAF_G : 1; }
template <int NC, int NTH, bool SUB>   // SUB: sub-leaf mean columns or Dirichlet data present
__global__ void __launch_bounds__(NTH * leaf_groups(NC), leaf_minb(NC) / leaf_groups(NC)) leaf2_kernel(DevPlan p, const int* __restrict__ order, LeafSmem ls,
                                                       int B) {
  extern __shared__ __align__(16) double sm_all[];
  constexpr int G = leaf_groups(NC);
  const int grp = G > 1 ? threadIdx.x / NTH : 0;
  double* sm = sm_all + size_t(grp) * ls.group_doubles;
  const int leaf = order[blockIdx.x];
  // a ragged last CTA recomputes the last sample in its spare groups (identical stores)
  const int s = G > 1 ? min(int(blockIdx.y) * G + grp, B - 1) : int(blockIdx.y);
  const int pass = blockIdx.z;
  LEAF_TICK(0);
  const int tid = threadIdx.x % NTH;
  constexpr int NT = NTH;
  const DevLeaf& L = p.leaves[leaf];
  if (pass > 0 && 1 + (NC - 1) * pass >= L.ncols) return;   // no columns left for this pass
  int* cinfo = reinterpret_cast<int*>(sm);                       // ctype, br, bq, bg, fslot
  double* arena = sm + leaf_hdr(NC);
  const int T = ls.T;
  // level r output: even r at the bottom of the arena, odd r at the top; level r's panel
  // right above the bottom region (its output for even r, its input for odd r)
  auto lout = [&](int r) -> double* { return (r & 1) ? arena + T - leaf_out_elems(r, NC) : arena; };
  auto lpan = [&](int r) -> double* { return arena + leaf_out_elems((r & 1) ? r + 1 : r, NC); };
  uint64_t* tab0 = reinterpret_cast<uint64_t*>(arena + T);      // panel programs, even levels
  uint64_t* tab1 = tab0 + ls.tp0;                                // odd levels
  uint64_t* tabU = tab1 + ls.tp1;
  double* kap = arena;                                            // [512], the bottom until level 4
  double* fl = kap + 512;                                         // [289]
  const int N = p.N;
  {
    const double* kb = p.kappa + int64_t(s) * 2 * N * N;
    for (int t = tid; t < 512; t += NT) {
      const int x = t >> 5, r = t & 31;
      cp_async8(kap + x * 32 + ((r + ((x >> 1) & 7)) & 31), kb + 2 * (int64_t(L.i0 + x) * N + L.j0) + r);
    }
    cp_async_commit();
    stage_panel_program<5, NC, NTH>(tab1);
    if (p.f) {
      const double* fs = sample_f(p, s);
      for (int t = tid; t < 289; t += NT) {
        int y = t / 17, x = t - y * 17;
        fl[t] = fs[int64_t(L.j0 + y) * p.m + L.i0 + x];
      }
    }
    if (tid < NC) {
      // local column tid of this pass -> leaf column lc (column 0 = the load, in every pass)
      const int lc = tid == 0 ? 0 : 1 + (NC - 1) * pass + (tid - 1);
      const bool ok = lc < L.ncols;
      cinfo[tid] = ok ? L.ctype[lc] : 3;     // 3 = unused column
      cinfo[NC + tid] = ok ? L.birth_r[lc] : -1;
      cinfo[2 * NC + tid] = ok ? L.birth_q[lc] : -1;
      cinfo[3 * NC + tid] = ok ? L.birth_g[lc] : -1;
      cinfo[4 * NC + tid] = ok ? L.fslot[lc] : -1;
      cinfo[5 * NC + tid] = ok && !(tid == 0 && pass > 0) ? lc : -1;   // output column
    }
    cp_async_wait<1>();
  }
  LEAF_SYNC();
  const int* ctype = cinfo;
  const int* br = cinfo + NC;
  const int* bq = cinfo + 2 * NC;
  const double h2_6 = p.h * p.h / 6.0;

  // ---------------- levels 6 + 5 fused: 2x4-cell nodes condensed directly ----------------
  // (l56_row): lane = node (32 nodes), warp w = boundary rows w and w + 8
  {
    constexpr int k5 = 12;
    constexpr int S5 = leaf_node_stride(k5, NC);
    static_assert(NTH == 256, "8 warps x 32 nodes");
    const int q = tid & 31, wid = tid >> 5;
    const int o = c_orig[31 + q];
    L56Node n;
    n.kap = kap;
    n.fl = p.f ? fl : nullptr;
    n.ox = o & 255;
    n.oy = o >> 8;
    n.h2_6 = h2_6;
    n.h2 = p.h * p.h;
    // interior block (tridiagonal) and its inverse M
    const double ia = n.Dl(1, 1), ib = n.Nl(1, 1), ic = n.Dl(1, 2), idd = n.Nl(1, 2), ie = n.Dl(1, 3);
    const double p1 = ia * ic - ib * ib;
    const double det = p1 * ie - ia * idd * idd;
    if (wid == 0 && (!(ia > 0.0) || !(p1 > 0.0) || !(det > 0.0)))
      record_error(p, HDD_ERR_NUMERICAL, s, inleaf_ref_id(L.ref_id, 5, q));
    const double rdet = 1.0 / det;
    const double M[6] = {(ic * ie - idd * idd) * rdet, -ib * ie * rdet, ib * idd * rdet,
                         ia * ie * rdet, -ia * idd * rdet, p1 * rdet};
    double* out = lout(5) + q * S5;
    switch (wid) {   // warp-uniform
      case 0: l56_row<0, NC, SUB>(n, M, out, ctype, br, bq, q); l56_row<8, NC, SUB>(n, M, out, ctype, br, bq, q); break;
      case 1: l56_row<1, NC, SUB>(n, M, out, ctype, br, bq, q); l56_row<9, NC, SUB>(n, M, out, ctype, br, bq, q); break;
      case 2: l56_row<2, NC, SUB>(n, M, out, ctype, br, bq, q); l56_row<10, NC, SUB>(n, M, out, ctype, br, bq, q); break;
      case 3: l56_row<3, NC, SUB>(n, M, out, ctype, br, bq, q); l56_row<11, NC, SUB>(n, M, out, ctype, br, bq, q); break;
      case 4: l56_row<4, NC, SUB>(n, M, out, ctype, br, bq, q); break;
      case 5: l56_row<5, NC, SUB>(n, M, out, ctype, br, bq, q); break;
      case 6: l56_row<6, NC, SUB>(n, M, out, ctype, br, bq, q); break;
      default: l56_row<7, NC, SUB>(n, M, out, ctype, br, bq, q); break;
    }
  }
  LEAF_SYNC();

  LEAF_TICK(1);
  // ---------------- levels 5..0 in shared memory ----------------
  leaf_level<4, NC, NTH>(p, lout(5), lout(4), lpan(4), cinfo, leaf, s, L.ref_id, tab0, tab1, tabU);
  leaf_level<3, NC, NTH>(p, lout(4), lout(3), lpan(3), cinfo, leaf, s, L.ref_id, tab1, tab0, tabU);
  leaf_level<2, NC, NTH>(p, lout(3), lout(2), lpan(2), cinfo, leaf, s, L.ref_id, tab0, tab1, tabU);
  leaf_level<1, NC, NTH>(p, lout(2), lout(1), lpan(1), cinfo, leaf, s, L.ref_id, tab1, tab0, tabU);
  leaf_level<0, NC, NTH, SUB>(p, lout(1), lout(0), lpan(0), cinfo, leaf, s, L.ref_id, tab0, tab1, tabU);
  if (tid == 0) bulk_wait_read0();   // the Psi bulk store has read its shared memory
  LEAF_TICK(63);
}

cudaError_t launch_leaf(const DevPlan& p, int B, cudaStream_t s, size_t* smem_out) {
  for (int cls = 0; cls < 3; ++cls) {
    const int cnt = p.leaf_class_count[cls];
    if (cnt == 0) continue;
    const int ncl = cls == 0 ? 2 : (cls == 1 ? 4 : 8);
    LeafSmem ls = leaf_sizes(ncl);
    const int G = leaf_groups(ncl);
    ls.group_doubles = int((leaf_smem_bytes(ncl) / sizeof(double) + 1) & ~size_t(1));   // 16-byte aligned groups
    const size_t smem = G > 1 ? size_t(G) * ls.group_doubles * sizeof(double) : leaf_smem_bytes(ncl);
    if (smem_out) *smem_out = smem;
    dim3 grid(cnt, (B + G - 1) / G, p.leaf_class_passes[cls]);
    const int* ord = p.leaf_order + p.leaf_class_start[cls];
    cudaError_t e;
#define HDD_LAUNCH_LEAF(NCV, SUBV)                                                                             \
  e = cudaFuncSetAttribute(leaf2_kernel<NCV, 256, SUBV>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); \
  if (e != cudaSuccess) return e;                                                                              \
  leaf2_kernel<NCV, 256, SUBV><<<grid, 256 * G, smem, s>>>(p, ord, ls, B);
    // sub-leaf mean columns and Dirichlet data only exist in plans that need them
    // (separate instantiation: the likelihood configs never pay for them)
    if (p.has_submean || p.leaf_g || p.gcall) {
      if (ncl == 2) { HDD_LAUNCH_LEAF(2, true) }
      else if (ncl == 4) { HDD_LAUNCH_LEAF(4, true) }
      else { HDD_LAUNCH_LEAF(8, true) }
    } else {
      if (ncl == 2) { HDD_LAUNCH_LEAF(2, false) }
      else if (ncl == 4) { HDD_LAUNCH_LEAF(4, false) }
      else { HDD_LAUNCH_LEAF(8, false) }
    }
#undef HDD_LAUNCH_LEAF
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// ---------------------------------------------------------------------------
// K3: upper merges.  Three steps per depth:
//   assemble_kernel   gathers the sons into the father's output block (lower
//                     part of A11 and R_B: assemble_father, hdd.py:216-238) and
//                     into the interface panel [A21 | A22 (padded to 32) | R_gamma]
//                     in HBM — memory-bound, every (row, node, sample) in parallel;
//   merge_m2_kernel   panel <= ~200 KB: one CTA per (node, sample) loads it to
//                     shared memory, 32-row blocked right-looking elimination with
//                     FP64 DMMA trailing updates, then the Schur update
//                     out -= X_B^T [X_B | X_R] on lower-triangle tiles (mirrored);
//   merge_l2_kernel   same with the panel kept in HBM (tier L).
// ---------------------------------------------------------------------------
template <int FM, int FN>
__device__ __forceinline__ void warp_gemm_tn(double (&acc)[FM][FN][2], const double* __restrict__ A, int lda, int m0,
                                             const double* __restrict__ B, int ldb, int n0, int kd) {
  const int lane = threadIdx.x & 31;
  const int gq = lane & 3, gr = lane >> 2;
  for (int k0 = 0; k0 < kd; k0 += 4) {
    double av[FM], bv[FN];
#pragma unroll
    for (int i = 0; i < FM; ++i) av[i] = A[(k0 + gq) * lda + m0 + 8 * i + gr];
#pragma unroll
    for (int j = 0; j < FN; ++j) bv[j] = B[(k0 + gq) * ldb + n0 + 8 * j + gr];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) dmma884(acc[i][j], av[i], bv[j]);
  }
}

constexpr int kLB = 32;     // elimination block (rows)
#ifdef HDD_LDS8
constexpr int kLds = 72;    // smem leading dim for 64-wide tiles (= 8 mod 16)
constexpr int kLdd = 40;    // smem leading dim for 32-wide tiles (= 8 mod 16)
#else
// = 4 or 12 (mod 16): a half-warp's DMMA fragment (4 rows x 4 columns) hits 16 distinct
// 8-byte banks (= 8 (mod 16) put rows 0 and 2 on the same banks)
constexpr int kLds = 76;    // smem leading dim for 64-wide tiles (+ 8 folded R columns)
constexpr int kLdd = 36;    // smem leading dim for 32-wide tiles
#endif
#ifdef HDD_LDS8
constexpr int kLwPad = 8;
#else
constexpr int kLwPad = 12;  // elimination chunk rows: LW + 12 = 12 (mod 16)
#endif

__device__ __forceinline__ int upper_ngp(const DevUpper& U) { return (U.ng + U.nb - 1) / U.nb * U.nb; }

// -- shared building blocks ------------------------------------------------
// Cholesky of the NB x NB diagonal block (rows read from `src`, ld `ld`) by one
// warp, lane = row, the row of L in registers and L[j][c] broadcast with
// shuffles; then L^-1 by forward row elimination with the rows of L^-1 kept in
// LiT (LiT[c][r] = (L^-1)[r][c]).  Sets *bad on a non-positive pivot.
template <int NB>
__device__ __forceinline__ double reg_get(const double (&a)[NB], int c) {
  double v = 0.0;
#pragma unroll
  for (int t = 0; t < NB; ++t) v = (t == c) ? a[t] : v;
  return v;
}
template <int NB>
__device__ __forceinline__ void reg_set(double (&a)[NB], int c, double v) {
#pragma unroll
  for (int t = 0; t < NB; ++t) a[t] = (t == c) ? v : a[t];
}

template <int NB>
__device__ __forceinline__ void factor_diag_block(const double* src, int ld, double* LiT, int* bad) {
  const int lane = threadIdx.x & 31;
  double a[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) a[j] = lane < NB ? src[lane * ld + j] : (lane == j ? 1.0 : 0.0);
  for (int c = 0; c < NB; ++c) {
    const double ac = reg_get<NB>(a, c);
    const double d = __shfl_sync(0xffffffffu, ac, c);
    if (!(d > 0.0) && lane == 0) *bad = 1;
    const double l = sqrt(d), inv = 1.0 / l;
    const double lc = lane == c ? l : (lane > c ? ac * inv : 0.0);
    reg_set<NB>(a, c, lane >= c ? lc : reg_get<NB>(a, c));
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const double ljc = __shfl_sync(0xffffffffu, lc, j);
      if (j > c && lane >= j) a[j] = fma(-lc, ljc, a[j]);
    }
  }
  // rows of L^-1: lane r accumulates row r in LiT[.][r]
  if (lane < NB)
#pragma unroll
    for (int c = 0; c < NB; ++c) LiT[c * kLdd + lane] = lane == c ? 1.0 : 0.0;
  __syncwarp();
  for (int h = 0; h < NB; ++h) {
    const double lrh = reg_get<NB>(a, h);     // L[lane][h]
    if (lane == h) {
      const double inv = 1.0 / lrh;
      for (int c = 0; c <= h; ++c) LiT[c * kLdd + h] *= inv;
    }
    __syncwarp();
    if (lane > h && lane < NB)
      for (int c = 0; c <= h; ++c) LiT[c * kLdd + lane] = fma(-lrh, LiT[c * kLdd + h], LiT[c * kLdd + lane]);
    __syncwarp();
  }
}

// Cholesky of a 32x32 SPD block (rows from `src`, stride ld) by one warp: lane =
// row in registers, column broadcasts by shuffles (fully unrolled); L goes to Ls
// column-major (Ls[c * kLdd + r] = L[r][c], 1/L_cc on the diagonal), then L^-1 by
// right-looking forward substitution, lane = column, into LiT[c * kLdd + r] =
// (L^-1)[r][c].  Sets *bad on a non-positive pivot.
__device__ __forceinline__ void factor_block32(const double* src, int ld, double* Ls, double* LiT, int* bad) {
  const int lane = threadIdx.x & 31;
  {
    double a[32];
#pragma unroll
    for (int l = 0; l < 32; ++l) a[l] = l <= lane ? src[lane * ld + l] : (l == lane ? 1.0 : 0.0);
    bool nb = false;
    double ild = 1.0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const double dj = __shfl_sync(0xffffffffu, a[j], j);
      nb |= !(dj > 0.0);
      const double il = rsqrt_nr(dj);
      const double lij = a[j] * il;
#pragma unroll
      for (int l = j + 1; l < 32; ++l) a[l] = fma(-lij, __shfl_sync(0xffffffffu, lij, l), a[l]);
      if (lane == j) ild = il;
      a[j] = lij;
    }
#pragma unroll
    for (int l = 0; l < 32; ++l)
      if (l <= lane) Ls[l * kLdd + lane] = l == lane ? ild : a[l];
    if (lane == 0 && nb) *bad = 1;
  }
  __syncwarp();
  // L^-1 = [L11^-1, 0; -L22^-1 L21 L11^-1, L22^-1] on 16x16 blocks (keeps 32 doubles live)
  const int c = lane & 15, base = lane & 16;
  double x[16];
  {
    double v[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = m == c ? 1.0 : 0.0;
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      x[m] = v[m] * Ls[(base + m) * kLdd + base + m];
      LiT[lane * kLdd + base + m] = x[m];
#pragma unroll
      for (int q = m + 1; q < 16; ++q) v[q] = fma(-Ls[(base + m) * kLdd + base + q], x[m], v[q]);
    }
    if (base)
#pragma unroll
      for (int m = 0; m < 16; ++m) LiT[lane * kLdd + m] = 0.0;    // upper-right block of L^-1
  }
  __syncwarp();
  if (!base) {
    double y[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      double t = 0.0;
#pragma unroll
      for (int m = 0; m < 16; ++m) t = fma(Ls[m * kLdd + 16 + r], x[m], t);     // (L21 x)[r]
      y[r] = t;
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      double t = 0.0;
#pragma unroll
      for (int q = 0; q <= r; ++q) t = fma(LiT[(16 + q) * kLdd + 16 + r], y[q], t);   // (L22^-1 y)[r]
      LiT[lane * kLdd + 16 + r] = -t;
    }
  }
  __syncwarp();
}

// Cholesky + L^-1 of an N x N SPD block (N <= 24) by one warp: lane = row, shuffles;
// L^-1 right-looking, lane = column.  Same conventions as factor_block32.
template <int N>
__device__ __forceinline__ void factor_blockN(const double* src, int ld, double* Ls, double* LiT, int* bad) {
  static_assert(N <= 24, "use factor_block32");
  const int lane = threadIdx.x & 31;
  const int row = lane < N ? lane : N - 1;
  {
    double a[N];
#pragma unroll
    for (int l = 0; l < N; ++l) a[l] = l <= row ? src[row * ld + l] : (l == row ? 1.0 : 0.0);
    bool nb = false;
    double ild = 1.0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const double dj = __shfl_sync(0xffffffffu, a[j], j);
      nb |= !(dj > 0.0);
      const double il = rsqrt_nr(dj);
      const double lij = a[j] * il;
#pragma unroll
      for (int l = j + 1; l < N; ++l) a[l] = fma(-lij, __shfl_sync(0xffffffffu, lij, l), a[l]);
      if (row == j) ild = il;
      a[j] = lij;
    }
    __syncwarp();
    if (lane < N)
#pragma unroll
      for (int l = 0; l < N; ++l)
        if (l <= lane) Ls[l * kLdd + lane] = l == lane ? ild : a[l];
    if (lane == 0 && nb) *bad = 1;
  }
  __syncwarp();
  if (lane < N) {
    double v[N];
#pragma unroll
    for (int m = 0; m < N; ++m) v[m] = m == lane ? 1.0 : 0.0;
#pragma unroll
    for (int m = 0; m < N; ++m) {
      const double x = v[m] * Ls[m * kLdd + m];
      LiT[lane * kLdd + m] = x;
#pragma unroll
      for (int q = m + 1; q < N; ++q) v[q] = fma(-Ls[m * kLdd + q], x, v[q]);
    }
  }
  __syncwarp();
}

// -- son views (packed-lower node outputs) ----------------------------------
// A node output per sample is [Psi lower-packed tri(k) | R k x nc | sigma nc].
struct SonView {
  const double* b;
  int k, nc;
};
__device__ __forceinline__ double son_psi(const SonView& s, int i, int j) {
  return i >= j ? s.b[tri(i) + j] : s.b[tri(j) + i];
}
__device__ __forceinline__ double son_R(const SonView& s, int i, int c) { return s.b[tri(s.k) + i * s.nc + c]; }
__device__ __forceinline__ double son_sig(const SonView& s, int c) { return s.b[tri(s.k) + s.k * s.nc + c]; }

struct MergeCtx {
  SonView sv[2];
  const int32_t* gm;     // [2][K]
  const int32_t* csrc;   // [nc][2]
  const double* ccoef;   // [nc][2]
  const int32_t* cbirth; // [nc]
  int K;
  int sh[2];             // son-shared boundary nodes (DevUpper::sh)
};

__device__ __forceinline__ MergeCtx merge_ctx(const DevPlan& p, const DevUpper& U, int s) {
  MergeCtx c;
#pragma unroll
  for (int sn = 0; sn < 2; ++sn) {
    c.sv[sn].b = p.buf[U.son_buf[sn]] + U.son_off[sn] * p.bcap + int64_t(s) * U.son_elems[sn];
    c.sv[sn].k = U.son_k[sn];
    c.sv[sn].nc = U.son_ld[sn];
  }
  c.gm = p.gmap + U.gmap_off;
  c.csrc = p.csrc + 2 * U.col_off;
  c.ccoef = p.ccoef + 2 * U.col_off;
  c.cbirth = p.cbirth + U.col_off;
  c.K = U.K;
  c.sh[0] = U.sh[0];
  c.sh[1] = U.sh[1];
  return c;
}

// assembled A~(a, j) for father indices a, j (gather form of assemble_father)
__device__ __forceinline__ double gather_A(const MergeCtx& c, int a, int j) {
  double v = 0.0;
  const int pa0 = c.gm[a], pa1 = c.gm[c.K + a];
  const int pb0 = c.gm[j], pb1 = c.gm[c.K + j];
  if (pa0 >= 0 && pb0 >= 0) v += son_psi(c.sv[0], pa0, pb0);
  if (pa1 >= 0 && pb1 >= 0) v += son_psi(c.sv[1], pa1, pb1);
  return v;
}
// gather_A with ONE load and no add: the entry of the first son that holds the pair
// (a, j).  Only the pairs of two nodes shared by both sons (the ends of the interface,
// MergeCtx::sh: at most three lower pairs per node) have a second term; the Schur
// epilogues add it afterwards (shared_pair_fixup), so the gathered value is first used
// after the DMMA loop.
__device__ __forceinline__ double gather_A1(const MergeCtx& c, int a, int j) {
  const int pa0 = c.gm[a], pa1 = c.gm[c.K + a];
  const int pb0 = c.gm[j], pb1 = c.gm[c.K + j];
  const bool h0 = (pa0 | pb0) >= 0, h1 = (pa1 | pb1) >= 0;
  const double* b = h0 ? c.sv[0].b : c.sv[1].b;
  const int pi = h0 ? pa0 : pa1, pj = h0 ? pb0 : pb1;
  const int hi = max(pi, pj), lo = min(pi, pj);
  return (h0 || h1) ? b[tri(hi) + lo] : 0.0;
}
// second son's term of the son-shared pairs, added to the written output (call after
// a CTA barrier that follows the epilogue's stores)
__device__ __forceinline__ void shared_pair_fixup(const MergeCtx& c, double* __restrict__ out) {
  const int t = threadIdx.x;
  if (t < 3) {
    int a = c.sh[t == 0 ? 0 : 1], b = c.sh[t == 2 ? 1 : 0];
    if (a >= 0 && b >= 0) {
      if (a < b) { const int u = a; a = b; b = u; }
      out[tri(a) + b] += son_psi(c.sv[1], c.gm[c.K + a], c.gm[c.K + b]);
    }
  }
}
// father index a (< k) on the boundary of BOTH sons
__device__ __forceinline__ bool gather_shared(const MergeCtx& c, int a, int k) {
  return a < k && (c.gm[a] | c.gm[c.K + a]) >= 0;
}
// assembled R~(a, col)
__device__ __forceinline__ double gather_R(const MergeCtx& c, int a, int col) {
  double v = 0.0;
  const int pa0 = c.gm[a], pa1 = c.gm[c.K + a];
  const int s0 = c.csrc[2 * col], s1 = c.csrc[2 * col + 1];
  if (pa0 >= 0 && s0 >= 0) v += c.ccoef[2 * col] * son_R(c.sv[0], pa0, s0);
  if (pa1 >= 0 && s1 >= 0) v += c.ccoef[2 * col + 1] * son_R(c.sv[1], pa1, s1);
  return v;
}
// the two sons' contributions kept apart (the add is deferred past the DMMA chain so
// the loads' latency overlaps it)
__device__ __forceinline__ void gather_A2(const MergeCtx& c, int a, int j, double& v0, double& v1) {
  const int pa0 = c.gm[a], pa1 = c.gm[c.K + a];
  const int pb0 = c.gm[j], pb1 = c.gm[c.K + j];
  v0 = (pa0 >= 0 && pb0 >= 0) ? son_psi(c.sv[0], pa0, pb0) : 0.0;
  v1 = (pa1 >= 0 && pb1 >= 0) ? son_psi(c.sv[1], pa1, pb1) : 0.0;
}
__device__ __forceinline__ void gather_R2(const MergeCtx& c, int a, int col, double& v0, double& v1) {
  const int pa0 = c.gm[a], pa1 = c.gm[c.K + a];
  const int s0 = c.csrc[2 * col], s1 = c.csrc[2 * col + 1];
  v0 = (pa0 >= 0 && s0 >= 0) ? c.ccoef[2 * col] * son_R(c.sv[0], pa0, s0) : 0.0;
  v1 = (pa1 >= 0 && s1 >= 0) ? c.ccoef[2 * col + 1] * son_R(c.sv[1], pa1, s1) : 0.0;
}
__device__ __forceinline__ double gather_sig(const MergeCtx& c, int col) {
  double v = 0.0;
  const int s0 = c.csrc[2 * col], s1 = c.csrc[2 * col + 1];
  if (s0 >= 0) v += c.ccoef[2 * col] * son_sig(c.sv[0], s0);
  if (s1 >= 0) v += c.ccoef[2 * col + 1] * son_sig(c.sv[1], s1);
  return v;
}

// panel row g of [A21 | A22 (padded) | R_gamma] -> dst (smem or HBM); four entries
// per thread in flight (the son reads are independent, predicated loads)
template <int U = 4>
__device__ __forceinline__ void gather_panel_row(const MergeCtx& c, int k, int ng, int Kp, int W, int g,
                                                 double* dst, int lane0, int step, int jfirst = 0) {
  if (g >= ng) {
    for (int j = jfirst + lane0; j < W; j += step) dst[j] = (j == k + g) ? 1.0 : 0.0;
    return;
  }
  const int a = k + g;
  const int pa0 = c.gm[a], pa1 = c.gm[c.K + a];
  for (int j0 = jfirst + lane0; j0 < W; j0 += U * step) {
    double v0[U], v1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * step;
      v0[u] = 0.0;
      v1[u] = 0.0;
      if (j < k + ng) {
        const int pb0 = c.gm[j], pb1 = c.gm[c.K + j];
        if (pa0 >= 0 && pb0 >= 0) v0[u] = son_psi(c.sv[0], pa0, pb0);
        if (pa1 >= 0 && pb1 >= 0) v1[u] = son_psi(c.sv[1], pa1, pb1);
      } else if (j >= Kp && j < W) {
        const int col = j - Kp;
        const int s0 = c.csrc[2 * col], s1 = c.csrc[2 * col + 1];
        if (pa0 >= 0 && s0 >= 0) v0[u] = c.ccoef[2 * col] * son_R(c.sv[0], pa0, s0);
        if (pa1 >= 0 && s1 >= 0) v1[u] = c.ccoef[2 * col + 1] * son_R(c.sv[1], pa1, s1);
        if (c.cbirth[col] == g) v0[u] += 1.0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * step;
      if (j < W) dst[j] = v0[u] + v1[u];
    }
  }
}

// Tier M (panel in shared memory, sons in global memory): the A21 columns j < k of panel
// row g have ONE term except at the (at most two) son-shared columns, so they go straight
// from the son's packed Psi into the panel with cp.async: no registers, every element of
// the row in flight at once (the register gather keeps U elements per thread in flight and
// pays one L2 round trip per U x 32 columns).  The A22 / R columns and the shared columns
// keep the register path (two terms, coefficients).  The caller commits and waits.
__device__ __forceinline__ void gather_panel_row_async(const MergeCtx& c, int k, int ng, int g, double* dst,
                                                       int lane) {
  if (g >= ng) {
    for (int j = lane; j < k; j += 32) dst[j] = 0.0;
    return;
  }
  const int pa0 = c.gm[k + g], pa1 = c.gm[c.K + k + g];
  const int ta0 = tri(pa0), ta1 = tri(pa1);
  for (int j = lane; j < k; j += 32) {
    const int pb0 = c.gm[j], pb1 = c.gm[c.K + j];
    if (pb0 >= 0 && pb1 >= 0) {              // son-shared column: both terms
      dst[j] = son_psi(c.sv[0], pa0, pb0) + son_psi(c.sv[1], pa1, pb1);
    } else if (pb0 >= 0) {
      cp_async8(dst + j, c.sv[0].b + (pa0 >= pb0 ? ta0 + pb0 : tri(pb0) + pa0));
    } else if (pb1 >= 0) {
      cp_async8(dst + j, c.sv[1].b + (pa1 >= pb1 ? ta1 + pb1 : tri(pb1) + pa1));
    } else {
      dst[j] = 0.0;
    }
  }
}

// Panel gather on 16-row x 32-column tiles through a per-warp smem tile, so that every
// read of a son's packed-lower Psi is contiguous along the lanes: a son entry (pa, pb)
// sits at tri(max) + min, i.e. it is contiguous along the COLUMNS j where pa >= pb and
// along the ROWS g where pa < pb.  Pass 1 (lane = column) takes the terms with pa >= pb,
// pass 2 (half-warp lane = row, the two half-warps on even / odd columns) the terms with
// pa < pb; the tile then leaves as 32-column row segments.  The row-wise gather
// (gather_panel_row) read the pa < pb half with one 32-byte sector per lane (VERDICT r01:
// 2.5-2.8x the ideal L2 sectors).  Columns [0, Kp) only; the R columns stay row-wise.
// OFF by default (HDD_GATHER_TILE): measured slower, C4 d5 / d4 / d3 25.5 / 31.8 / 23.3 ->
// 27.6 / 33.2 / 23.9 ms: the gather is bound by the load round trips per thread (twice as
// many here), not by the sectors.
// Each element has at most two terms (one per son), so the sum does not depend on which
// pass brings which term.
constexpr int kGT = 16;                      // tile rows
constexpr int kGTs = 33;                     // tile row stride (doubles)
__device__ __forceinline__ void gather_panel_tile(const MergeCtx& c, int k, int ng, int Kp, int g0, int j0,
                                                  double* __restrict__ tile, double* __restrict__ P, int64_t ldp,
                                                  int lane) {
  const int KA = k + ng;                     // A columns end
  // ---- pass 1: lane = column j, rows in turn; terms with pa >= pb ----
  {
    const int j = j0 + lane;
    const bool jl = j < KA;
    const int pb0 = jl ? c.gm[j] : -1, pb1 = jl ? c.gm[c.K + j] : -1;
#pragma unroll
    for (int r0 = 0; r0 < kGT; r0 += 8) {
      double v0[8], v1[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int g = g0 + r0 + u;
        v0[u] = 0.0;
        v1[u] = 0.0;
        if (g < ng) {
          const int pa0 = c.gm[k + g], pa1 = c.gm[c.K + k + g];
          if (pb0 >= 0 && pa0 >= pb0) v0[u] = c.sv[0].b[tri(pa0) + pb0];
          if (pb1 >= 0 && pa1 >= pb1) v1[u] = c.sv[1].b[tri(pa1) + pb1];
        } else if (j == k + g) {
          v0[u] = 1.0;                       // padding rows: identity
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) tile[(r0 + u) * kGTs + lane] = v0[u] + v1[u];
    }
  }
  __syncwarp();
  // ---- pass 2: lane & 15 = row, lane >> 4 = column parity; terms with pa < pb ----
  {
    const int g = g0 + (lane & 15);
    const bool gl = g < ng;
    const int pa0 = gl ? c.gm[k + g] : -1, pa1 = gl ? c.gm[c.K + k + g] : -1;
    double* trow = tile + (lane & 15) * kGTs;
#pragma unroll
    for (int c0 = 0; c0 < 32; c0 += 16) {
      double v0[8], v1[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + c0 + 2 * u + (lane >> 4);
        v0[u] = 0.0;
        v1[u] = 0.0;
        if (j < KA) {
          const int pb0 = c.gm[j], pb1 = c.gm[c.K + j];
          if (pa0 >= 0 && pa0 < pb0) v0[u] = c.sv[0].b[tri(pb0) + pa0];
          if (pa1 >= 0 && pa1 < pb1) v1[u] = c.sv[1].b[tri(pb1) + pa1];
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) trow[c0 + 2 * u + (lane >> 4)] += v0[u] + v1[u];
    }
  }
  __syncwarp();
  // ---- the tile's rows to the panel (32 consecutive columns per row) ----
  if (j0 + lane < Kp) {
#pragma unroll 4
    for (int r = 0; r < kGT; ++r) P[int64_t(g0 + r) * ldp + j0 + lane] = tile[r * kGTs + lane];
  }
  __syncwarp();
}

// Schur-update epilogue on 32 x 64 output tiles (lower-triangle Psi tiles and
// the R columns), the assembled A~ values gathered from the sons and issued
// before the DMMA loop; output packed-lower.
template <bool SMEM, bool FAST = false, bool SPLIT = false, bool G1 = false>
__device__ __forceinline__ void schur_epilogue(const MergeCtx& mc, const double* __restrict__ P, int ldp, int k,
                                               int ngp, int Kp, int nc, double* __restrict__ out, double* Ea,
                                               double* Eb) {
  const int tid = threadIdx.x & 255, lane = tid & 31, warp = tid >> 5;
  const int grp = threadIdx.x >> 8, ngrp = SMEM ? (blockDim.x >> 8) : 1;   // 8-warp groups
  const int gq = lane & 3, gr = lane >> 2;
  const int ow = k + nc;
  const int m0 = (warp >> 2) * 16, n0 = (warp & 3) * 16;
  const int na = (k + 31) / 32, nbt = (ow + 63) / 64;
  const int tk = tri(k);
  // tiles t = ta * nbt + tb, walked without integer division
  int ta = 0, tb = grp;
  while (tb >= nbt && nbt > 0) { tb -= nbt; ++ta; }
  for (int t = grp; t < na * nbt; t += ngrp) {
    const int a0 = ta * 32, b0 = tb * 64;
    tb += ngrp;
    while (tb >= nbt) { tb -= nbt; ++ta; }
    if (b0 + 64 <= k && b0 > a0 + 31) continue;   // strictly upper Psi tile
    // 8x8 DMMA blocks of this warp's 16x16 sub-tile that hold outputs (warp-uniform):
    // rows < k, columns < k + nc, not strictly above the diagonal of Psi
    bool live[2][2];
    bool any = false;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int ar = a0 + m0 + 8 * i, bc = b0 + n0 + 8 * j;
        live[i][j] = ar < k && bc < ow && !(bc + 8 <= k && bc > ar + 7);
        any |= live[i][j];
      }
    if constexpr (SMEM) {
      if (!any) continue;                          // no barriers in the smem-panel loop
      const int ar0 = a0 + m0, bc0 = b0 + n0;
      if (FAST && ar0 + 16 <= k && bc0 + 16 <= k && bc0 + 15 < ar0) {
        // this warp's 16x16 sub-tile is strictly lower and inside Psi: no per-element
        // predicates (the common case on big nodes)
        double pre[2][2][2], pre1[2][2][2], acc[2][2][2] = {};
        int trow[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int aa = ar0 + 8 * i + gr;
          trow[i] = tri(aa);
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              if constexpr (G1) { pre[i][j][e] = gather_A1(mc, aa, bc0 + 8 * j + 2 * gq + e); pre1[i][j][e] = 0.0; }
              else if constexpr (SPLIT) gather_A2(mc, aa, bc0 + 8 * j + 2 * gq + e, pre[i][j][e], pre1[i][j][e]);
              else { pre[i][j][e] = gather_A(mc, aa, bc0 + 8 * j + 2 * gq + e); pre1[i][j][e] = 0.0; }
            }
        }
        for (int g0 = 0; g0 < ngp; g0 += 4) {
          const double* pr = P + size_t(g0 + gq) * ldp;
          double av[2], bv[2];
#pragma unroll
          for (int i = 0; i < 2; ++i) { av[i] = pr[ar0 + 8 * i + gr]; bv[i] = pr[bc0 + 8 * i + gr]; }
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) dmma884(acc[i][j], av[i], bv[j]);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              out[trow[i] + bc0 + 8 * j + 2 * gq + e] = (SPLIT ? pre[i][j][e] + pre1[i][j][e] : pre[i][j][e]) - acc[i][j][e];
        continue;
      }
    }
    double acc[2][2][2] = {};
    int acol[2], bcol[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int aa = a0 + m0 + 8 * i + gr;
      acol[i] = aa < k ? aa : 0;
      const int bb = b0 + n0 + 8 * i + gr;
      bcol[i] = bb < k ? bb : (bb < ow ? Kp + (bb - k) : 0);
    }
    double pre[2][2][2], pre1[2][2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int aa = a0 + m0 + 8 * i + gr;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int bb = b0 + n0 + 8 * j + 2 * gq + e;
          double v = 0.0, v1 = 0.0;
          if (aa < k && bb < ow) {
            if constexpr (SPLIT) {
              if (bb < k) {
                if (bb <= aa) {
                  if constexpr (G1) v = gather_A1(mc, aa, bb);
                  else gather_A2(mc, aa, bb, v, v1);
                }
              } else gather_R2(mc, aa, bb - k, v, v1);
            } else {
              if (bb < k) {
                if (bb <= aa) {
                  if constexpr (G1) v = gather_A1(mc, aa, bb);
                  else v = gather_A(mc, aa, bb);
                }
              } else v = gather_R(mc, aa, bb - k);
            }
          }
          pre[i][j][e] = v;
          pre1[i][j][e] = v1;
        }
    }
    if constexpr (SMEM) {
      for (int g0 = 0; g0 < ngp; g0 += 4) {
        const double* pr = P + size_t(g0 + gq) * ldp;
        double av[2], bv[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) { av[i] = pr[acol[i]]; bv[i] = pr[bcol[i]]; }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j)
            if (live[i][j]) dmma884(acc[i][j], av[i], bv[j]);
      }
    } else {
      for (int g0 = 0; g0 < ngp; g0 += 32) {
        __syncthreads();
        for (int tt = tid; tt < 32 * 32; tt += 256) {
          const int g = tt >> 5, i = tt & 31;
          const int aa = a0 + i;
          Ea[g * kLds + i] = aa < k ? P[int64_t(g0 + g) * ldp + aa] : 0.0;
        }
        for (int tt = tid; tt < 32 * 64; tt += 256) {
          const int g = tt >> 6, j = tt & 63;
          const int bb = b0 + j;
          const int col = bb < k ? bb : (bb < ow ? Kp + (bb - k) : -1);
          Eb[g * kLds + j] = col >= 0 ? P[int64_t(g0 + g) * ldp + col] : 0.0;
        }
        __syncthreads();
        warp_gemm_tn<2, 2>(acc, Ea, kLds, m0, Eb, kLds, n0, 32);
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int aa = a0 + m0 + 8 * i + gr;
      if (aa >= k) continue;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int bb = b0 + n0 + 8 * j + 2 * gq + e;
          if (bb >= ow) continue;
          if (bb < k) {
            if (bb <= aa) out[tri(aa) + bb] = (pre[i][j][e] + pre1[i][j][e]) - acc[i][j][e];
          } else {
            out[tk + aa * nc + (bb - k)] = (pre[i][j][e] + pre1[i][j][e]) - acc[i][j][e];
          }
        }
    }
  }
  if constexpr (G1) {          // single-load gathers: the son-shared pairs' second term
    __syncthreads();
    shared_pair_fixup(mc, out);
  }
}


constexpr int kEC = 16;     // tier-L epilogue: interface rows per staged chunk
#ifndef HDD_EPI_STAGES
#define HDD_EPI_STAGES 2    // smem buffers of the tier-L epilogue's X chunks
#endif
// Tier-L Schur update on 64 x 64 output tiles: the lower Psi tiles (b0 <= a0, columns
// < k) and, when nc > 8, 64-column R tiles.  With nc <= 8 (most depths: the load column
// and a few functionals) the R block rides on the diagonal tiles: their two strictly
// upper 32 x 16 warp tiles compute rows a0..a0+63 x the R columns instead (B chunk
// columns 64..71), so no tile pass stages A for a mostly empty R tile and no DMMA runs
// on padding columns.  X chunks of kEC interface rows are double-buffered HBM -> smem
// with cp.async; 8 warps as 2 x 4 of 32 x 16 DMMA tiles.
// E: [2][2][kEC][kLds] smem (A chunk, B chunk) x double buffer.
__device__ __forceinline__ void schur_epilogue_l(const MergeCtx& mc, const double* __restrict__ P, int ldp, int k,
                                                 int ngp, int Kp, int nc, double* __restrict__ out, double* E) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane & 3, gr = lane >> 2;
  const int m0 = (warp >> 2) * 32, n0 = (warp & 3) * 16;
  const int na = (k + 63) / 64;
  const bool fold = nc <= 8;
  const int nbr = fold ? 0 : (nc + 63) / 64;
  const int nch = ngp / kEC;
  const int tk = tri(k);
  for (int ia = 0; ia < na; ++ia) {
    const int a0 = ia * 64;
    for (int jb = 0; jb <= ia + nbr; ++jb) {
      const bool is_r = jb > ia;
      const int b0 = is_r ? (jb - ia - 1) * 64 : jb * 64;   // Psi column / R column origin
      const bool rfold = fold && jb == ia;
      // warp role: 0 idle, 1 its 32 x 16 part of the tile, 2 folded R rows (a0 + rm0 ..)
      int role = 1, rm0 = 0;
      if (is_r) {
        if (b0 + n0 >= nc || a0 + m0 >= k) role = 0;
      } else if (b0 + n0 > a0 + m0 + 31 || b0 + n0 >= k || a0 + m0 >= k) {
        role = 0;
        if (rfold && m0 == 0 && n0 >= 32) {
          rm0 = n0 == 32 ? 0 : 32;
          role = a0 + rm0 < k ? 2 : 0;
        }
      }
      const int lim = is_r ? nc : k;          // B columns: R columns or Psi columns
      const int base = is_r ? Kp : 0;
      auto stage = [&](int c, int buf) {
        double* Ea = E + buf * 2 * kEC * kLds;
        double* Eb = Ea + kEC * kLds;
        const int g0 = c * kEC;
        // column pairs as 16-byte copies (even ldp, even starts); odd starts element-wise
        for (int tt = tid; tt < kEC * 32; tt += 256) {
          const int g = tt >> 5, i = 2 * (tt & 31);
          const double* src = P + int64_t(g0 + g) * ldp;
          double* ea = Ea + g * kLds + i;
          double* eb = Eb + g * kLds + i;
          const int aa = a0 + i;
          if (aa + 1 < k) cp_async16(ea, src + aa);
          else {
            if (aa < k) cp_async8(ea, src + aa);
            else ea[0] = 0.0;
            ea[1] = 0.0;
          }
          const int bb = b0 + i;
          if (bb + 1 < lim && ((base + bb) & 1) == 0) cp_async16(eb, src + base + bb);
          else {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              if (bb + e < lim) cp_async8(eb + e, src + base + bb + e);
              else eb[e] = 0.0;
            }
          }
        }
        if (rfold)
          for (int tt = tid; tt < kEC * 8; tt += 256) {
            const int g = tt >> 3, cc = tt & 7;
            double* eb = Eb + g * kLds + 64 + cc;
            if (cc < nc) cp_async8(eb, P + int64_t(g0 + g) * ldp + Kp + cc);
            else *eb = 0.0;
          }
        cp_async_commit();
      };
      __syncthreads();
      stage(0, 0);
#if HDD_EPI_STAGES == 3
      if (nch > 1) stage(1, 1);
#endif
      // the assembled A~ / R~ values of this warp's outputs, loaded ahead of the DMMAs
      double pre[4][2][2];
      // warp-uniform: can this warp's 32 rows x 16 columns hold a pair of two nodes shared
      // by both sons?  (two such nodes per merge: almost every warp tile takes the
      // single-load gather)
      const bool both = role == 1 && !is_r &&
                        __any_sync(0xffffffffu, gather_shared(mc, a0 + m0 + lane, k)) &&
                        __any_sync(0xffffffffu, gather_shared(mc, b0 + n0 + (lane & 15), k));
      if (role == 1 && !is_r && !both) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int aa = a0 + m0 + 8 * i + gr;
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int bb = b0 + n0 + 8 * j + 2 * gq + e;
              pre[i][j][e] = (aa < k && bb <= aa) ? gather_A1(mc, aa, bb) : 0.0;
            }
        }
      } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int aa = a0 + (role == 2 ? rm0 : m0) + 8 * i + gr;
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            double v = 0.0;
            if (role == 1 && aa < k) {
              const int bb = b0 + n0 + 8 * j + 2 * gq + e;
              if (is_r) { if (bb < nc) v = gather_R(mc, aa, bb); }
              else if (bb <= aa) v = gather_A(mc, aa, bb);
            } else if (role == 2 && j == 0 && aa < k) {
              const int rc = 2 * gq + e;
              if (rc < nc) v = gather_R(mc, aa, rc);
            }
            pre[i][j][e] = v;
          }
      }
      }
      double acc[4][2][2] = {};
      for (int c = 0; c < nch; ++c) {
#if HDD_EPI_STAGES == 3
        // three buffers, one barrier per chunk: it publishes chunk c and frees the
        // buffer of chunk c - 1 for chunk c + 2
        if (c + 1 < nch) cp_async_wait<1>();
        else cp_async_wait<0>();
        __syncthreads();
        if (c + 2 < nch) stage(c + 2, (c + 2) % 3);
        const double* Ea = E + (c % 3) * 2 * kEC * kLds;
#elif defined(HDD_ONE_BARRIER)
        // two buffers, one barrier per chunk: the barrier publishes chunk c and tells that
        // every warp has left chunk c - 1, whose buffer then takes chunk c + 1 (same
        // prefetch distance as staging before the wait: one chunk of DMMAs)
        cp_async_wait<0>();
        __syncthreads();
        if (c + 1 < nch) stage(c + 1, (c + 1) & 1);
        const double* Ea = E + (c & 1) * 2 * kEC * kLds;
#else
        if (c + 1 < nch) {
          stage(c + 1, (c + 1) & 1);
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncthreads();
        const double* Ea = E + (c & 1) * 2 * kEC * kLds;
#endif
        const double* Eb = Ea + kEC * kLds;
        if (role == 1) {
          warp_gemm_tn<4, 2>(acc, Ea, kLds, m0, Eb, kLds, n0, kEC);
        } else if (role == 2) {
#pragma unroll
          for (int kk = 0; kk < kEC; kk += 4) {
            double av[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = Ea[(kk + gq) * kLds + rm0 + 8 * i + gr];
            const double bv = Eb[(kk + gq) * kLds + 64 + gr];
#pragma unroll
            for (int i = 0; i < 4; ++i) dmma884(acc[i][0], av[i], bv);
          }
        }
#if HDD_EPI_STAGES != 3 && !defined(HDD_ONE_BARRIER)
        __syncthreads();
#endif
      }
      if (role == 0) continue;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int aa = a0 + (role == 2 ? rm0 : m0) + 8 * i + gr;
        if (aa >= k) continue;
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if (role == 2) {
              const int rc = 2 * gq + e;
              if (j == 0 && rc < nc) out[tk + aa * nc + rc] = pre[i][0][e] - acc[i][0][e];
            } else {
              const int bb = b0 + n0 + 8 * j + 2 * gq + e;
              if (is_r) {
                if (bb < nc) out[tk + aa * nc + bb] = pre[i][j][e] - acc[i][j][e];
              } else if (bb <= aa) {
                out[tri(aa) + bb] = pre[i][j][e] - acc[i][j][e];
              }
            }
          }
      }
    }
  }
}

__device__ __forceinline__ void store_factors(const DevPlan& p, const DevUpper& U, int s, const double* P, int ldp,
                                              int Kp, bool diag_unscaled, int tid, int nthr) {
  const int k = U.k, ng = U.ng;
  const int fw = k + ng + 1;
  double* F = p.fac + int64_t(s) * p.fac_elems + U.fac_off;
  for (int t = tid; t < ng * fw; t += nthr) {
    const int g = t / fw, j = t - g * fw;
    double v;
    if (j < k) v = P[int64_t(g) * ldp + j];
    else if (j < k + ng) {
      const int jj = j - k;
      v = jj < g ? 0.0 : P[int64_t(g) * ldp + k + jj];
      if (jj == g && diag_unscaled) v = sqrt(v);
    } else v = P[int64_t(g) * ldp + Kp];
    F[t] = v;
  }
}

// Cholesky of an 8x8 SPD block D (row stride ld) by one warp: lane = row in
// registers, column broadcasts by shuffles; L -> Ls (lower, zero upper), 1/L_ii ->
// Ld, then L^-1 -> Li column by column (lane = column).  *bad = 1 on a
// non-positive pivot.
#ifdef HDD_FACTOR8_NOINLINE     // A/B: one copy of the ~500-instruction factor (instruction-cache footprint)
__device__ __noinline__ void factor_block8(const double* D, int ld, double* Ls, double* Li, double* Ld,
                                           int* bad) {
#else
__device__ __forceinline__ void factor_block8(const double* D, int ld, double* Ls, double* Li, double* Ld,
                                              int* bad) {
#endif
  const int lane = threadIdx.x & 31, i = lane & 7;
  double a[8];
#pragma unroll
  for (int l = 0; l < 8; ++l) a[l] = l <= i ? D[i * ld + l] : (l == i ? 1.0 : 0.0);
  bool nb = false;
  double ild = 1.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double dj = __shfl_sync(0xffffffffu, a[j], j, 8);
    nb |= !(dj > 0.0);
    const double il = rsqrt_nr(dj);
    const double lij = a[j] * il;
#pragma unroll
    for (int l = j + 1; l < 8; ++l) a[l] = fma(-lij, __shfl_sync(0xffffffffu, lij, l, 8), a[l]);
    if (i == j) ild = il;
    a[j] = i == j ? dj * il : lij;
  }
  if (lane < 8) {
#pragma unroll
    for (int l = 0; l < 8; ++l) Ls[i * 8 + l] = l <= i ? a[l] : 0.0;
    Ld[i] = ild;
  }
  if (lane == 0 && nb) *bad = 1;
  __syncwarp();
  if (lane < 8) {
    double x[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      double v = m == lane ? 1.0 : 0.0;
#pragma unroll
      for (int q = 0; q < m; ++q) v = fma(-Ls[m * 8 + q], x[q], v);
      x[m] = v * Ld[m];
    }
#pragma unroll
    for (int m = 0; m < 8; ++m) Li[m * 8 + lane] = x[m];
  }
  __syncwarp();
}

// -- tier M: panel in shared memory ------------------------------------------
// smem: panel [ngp][ldp] | scratch [8] + L, L^-1 of the diagonal block [2][64] | son maps [2][K] int | column plan (csrc
// [nc][2], cbirth [nc]) int | ccoef [nc][2] | staged sons (optional)
size_t merge_m2_smem_bytes(int ngp, int ldp, int K, int nc) {
  const size_t ints = (size_t(2 * K + 3 * nc) + 1) & ~size_t(1);
  return sizeof(double) * (size_t(ngp) * ldp + 8 + 128 + ints / 2 + 2 * size_t(nc) + 2) + 64;   // +2: 16-byte alignment of the staged sons
}

#ifndef HDD_M2_GATHER8_MINB
#define HDD_M2_GATHER8_MINB 2   // tier-M instantiations (by CTAs/SM) whose panel gather keeps 8 loads per thread in flight
#endif
template <int NB, int NTH, int MINB>
__global__ void __launch_bounds__(NTH, MINB) merge_m2_kernel(DevPlan p, const DevUpper* __restrict__ nodes, int slot) {
  extern __shared__ __align__(16) double sm[];
  MERGE_TICK(0);
  const DevUpper& U = nodes[blockIdx.y];
  const int s = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NT = NTH, NWp = NTH >> 5;
  const int k = U.k, ng = U.ng, nc = U.nc, ldp = U.ldp;
  const int ngp = upper_ngp(U);
  const int Kp = k + ngp;
  const int W = Kp + nc;
  double* P = sm;                          // [ngp][ldp]
  double* piv = P + size_t(ngp) * ldp;     // [NB] pivots of the current block
  int32_t* gms = reinterpret_cast<int32_t*>(piv + 8 + 128);
  int32_t* cis = gms + 2 * U.K;
  double* ccs = reinterpret_cast<double*>(gms + ((2 * U.K + 3 * nc + 1) & ~1));
  double* st = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(ccs + 2 * nc) + 15) & ~uintptr_t(15));
  __shared__ int s_bad;
  __shared__ __align__(8) uint64_t s_bar;
  MergeCtx mc = merge_ctx(p, U, s);
  if (U.stage) {
    // stage both sons' packed outputs in shared memory: two TMA bulk copies (the
    // per-sample blocks are even-sized, hence 16-byte aligned) on one mbarrier
    if (tid == 0) {
      mbar_init(&s_bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      const uint32_t b0 = uint32_t(U.son_elems[0]) * 8u, b1 = uint32_t(U.son_elems[1]) * 8u;
      mbar_arrive_expect_tx(&s_bar, b0 + b1);
      bulk_g2s(st, mc.sv[0].b, b0, &s_bar);
      bulk_g2s(st + U.son_elems[0], mc.sv[1].b, b1, &s_bar);
    }
    mc.sv[0].b = st;
    mc.sv[1].b = st + U.son_elems[0];
  }
#ifndef HDD_NO_L2_PREFETCH
  else if (tid == 0) {
    // the sons' packed outputs are read twice (panel gather now, A11 / R_B in the Schur
    // epilogue after the elimination): pull them into L2 while the maps are staged
    bulk_prefetch_l2(mc.sv[0].b, uint32_t(U.son_elems[0] * 8) & ~15u);
    bulk_prefetch_l2(mc.sv[1].b, uint32_t(U.son_elems[1] * 8) & ~15u);
  }
#endif
  for (int t = tid; t < 2 * U.K; t += NT) gms[t] = __ldg(mc.gm + t);
  for (int t = tid; t < 2 * nc; t += NT) {
    cis[t] = __ldg(mc.csrc + t);
    ccs[t] = __ldg(mc.ccoef + t);
  }
  for (int t = tid; t < nc; t += NT) cis[2 * nc + t] = __ldg(mc.cbirth + t);
  mc.gm = gms;
  mc.csrc = cis;
  mc.cbirth = cis + 2 * nc;
  mc.ccoef = ccs;
  __syncthreads();                         // maps staged; the mbarrier is initialised
  if (U.stage) mbar_wait(&s_bar, 0);
  MERGE_TICK(1);
#ifdef HDD_M2_GATHER_ASYNC
  if (!U.stage) {
    for (int g = warp; g < ngp; g += NWp) gather_panel_row_async(mc, k, ng, g, P + g * ldp, lane);
    cp_async_commit();
    for (int g = warp; g < ngp; g += NWp)
      gather_panel_row<(MINB <= HDD_M2_GATHER8_MINB) ? 8 : 4>(mc, k, ng, Kp, W, g, P + g * ldp, lane, 32, k);
    cp_async_wait<0>();
  } else
#endif
  for (int g = warp; g < ngp; g += NWp) gather_panel_row<(MINB <= HDD_M2_GATHER8_MINB) ? 8 : 4>(mc, k, ng, Kp, W, g, P + g * ldp, lane, 32);
  if (tid == 0) s_bad = 0;
  const int gq = lane & 3, gr = lane >> 2;
  double* Ls = piv + 8;                    // [8][8] diagonal-block factor L (piv: 1/L_ii)
  double* Li = Ls + 64;                    // [8][8] L^-1
  static_assert(NB == 8, "8-row elimination blocks");
  // Right-looking blocked Cholesky of A22 on 8-row blocks with look-ahead: warp 0
  // updates and factors the next diagonal block while warps 1.. apply the trailing
  // update of the current block row (two barriers per block).
  __syncthreads();                         // panel gathered
  MERGE_TICK(2);
  if (warp == 0) factor_block8(P + k, ldp, Ls, Li, piv, &s_bad);
#ifdef HDD_PROFILE_TICKS
  if (blockIdx.x == HDD_TICK_X && blockIdx.y == HDD_TICK_Y && threadIdx.x == 0 && slot >= 0 && slot < 16) g_merge_clk[slot + 16][0] = clock64();
#endif
  __syncthreads();
  MERGE_TICK(6);                           // first diagonal block factored
  for (int r0 = 0; r0 < ngp; r0 += NB) {
    // block rows X = L^-1 P[r0:r0+8, :] in place, 8-column DMMA tiles across warps
    for (int t = warp; t < (W + 7) / 8; t += NWp) {
      const int c0 = 8 * t;
      double acc[2] = {0.0, 0.0};
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const double av = Li[gr * 8 + 4 * kk + gq];
        const double bv = c0 + gr < W ? P[(r0 + 4 * kk + gq) * ldp + c0 + gr] : 0.0;
        dmma884(acc, av, bv);
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = c0 + 2 * gq + e;
        if (col < W) P[(r0 + gr) * ldp + col] = acc[e];
      }
    }
    __syncthreads();
    if (r0 == 0) MERGE_TICK(7);            // first block row applied
    const int rn = r0 + NB;                // next block
    if (rn >= ngp) break;
    if (warp == 0) {
      // look-ahead: D_next -= X[:, next]^T X[:, next], then factor it
      const double* X = P + r0 * ldp + k + rn;
      double acc[2] = {0.0, 0.0};
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const double x = X[(4 * kk + gq) * ldp + gr];
        dmma884(acc, x, x);
      }
      double* D = P + rn * ldp + k + rn;
      D[gr * ldp + 2 * gq] -= acc[0];
      D[gr * ldp + 2 * gq + 1] -= acc[1];
      __syncwarp();
      factor_block8(D, ldp, Ls, Li, piv, &s_bad);
    } else {
      const int nrt = (ngp - rn) / 8;
      const int nct = (W + 31) / 32;
      for (int t = warp - 1; t < nrt * nct; t += NWp - 1) {
        const int rt = rn + (t / nct) * 8;
        const int c0 = (t % nct) * 32;
        if (c0 >= k && c0 + 32 <= k + rt) continue;     // A22 columns left of the tile rows: never read again
        double acc[1][4][2] = {};
        warp_gemm_tn<1, 4>(acc, P + r0 * ldp + k, ldp, rt, P + r0 * ldp, ldp, c0, NB);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = c0 + 8 * j + 2 * gq + e;
            const bool diag_next = rt == rn && col >= k + rn && col < k + rn + 8;   // warp 0's block
            if (col < W && !diag_next) P[(rt + gr) * ldp + col] -= acc[0][j][e];
          }
      }
    }
    __syncthreads();
  }
  __syncthreads();
  MERGE_TICK(3);
  if (s_bad && tid == 0) record_error(p, HDD_ERR_NUMERICAL, s, U.ref_id);
  if (p.mode == 1 && U.fac_off >= 0) store_factors(p, U, s, P, ldp, Kp, false, tid, NT);
  double* out = p.buf[U.buf] + U.out_off * p.bcap + int64_t(s) * U.out_elems;
  const int tk = tri(k);
  for (int c = tid; c < nc; c += NT) {
    double v = gather_sig(mc, c);
    if (c >= 1)
      for (int g = 0; g < ng; ++g) v = fma(P[g * ldp + Kp], P[g * ldp + Kp + c], v);
    out[tk + k * nc + c] = v;
  }
  MERGE_TICK(4);
#ifndef HDD_G1_MINB_LO
#define HDD_G1_MINB_LO 3   // tier-M instantiations (by CTAs/SM) whose epilogue uses the single-load gather
#endif
  schur_epilogue<true, MINB <= 3, MINB <= 2, (MINB <= 3 && MINB >= HDD_G1_MINB_LO)>(mc, P, ldp, k, ngp, Kp, nc, out, nullptr, nullptr);
  MERGE_TICK(5);
}

// -- tier L: panel in HBM ----------------------------------------------------
// smem: F phases (L scratch / LiT / Xc / Lt) and the epilogue's 2 x (A, B) chunks of
// 32 x kLds share the front region; the son maps and column plan follow it.
// left-looking elimination: column chunks of LW (64, or 128 for the 2-CTA/SM variant),
// staged rows per step kLH
constexpr int kLH = 16;
__host__ __device__ constexpr size_t l_region(int lw) {
  const size_t lws = size_t(lw) + kLwPad;
  const size_t stream = 2 * size_t(kLH) * (kLdd + lws);                 // 2 x (A chunk | B chunk)
  const size_t ll = 2 * 32 * kLdd + (stream > 32 * lws ? stream : 32 * lws);
  const size_t epi = 2 * HDD_EPI_STAGES * kEC * kLds;                    // Schur epilogue chunks
  return epi > ll ? epi : ll;
}
constexpr size_t kLRegion = l_region(64);
size_t merge_l_smem_bytes(int K, int nc) {
  const size_t ints = (size_t(2 * K + 3 * nc) + 1) & ~size_t(1);
  return sizeof(double) * (kLRegion + ints / 2 + 2 * size_t(nc)) + 1024;
}

template <int MINB, int LW>
__global__ void __launch_bounds__(256, MINB) merge_l_kernel(DevPlan p, const DevUpper* __restrict__ nodes,
                                                          double* __restrict__ ws, int64_t ws_stride, int slot) {
  extern __shared__ __align__(16) double sm[];
  MERGE_TICK(0);
  const DevUpper& U = nodes[blockIdx.y];
  const int s = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = U.k, ng = U.ng, nc = U.nc, ldp = U.ldp;
  const int ngp = upper_ngp(U);
  const int Kp = k + ngp;
  const int W = Kp + nc;
  double* P = ws + int64_t(blockIdx.y) * ws_stride * p.bcap + int64_t(s) * ws_stride;
  __shared__ int s_bad;
  MergeCtx mc = merge_ctx(p, U, s);
  {   // son maps and column plan in smem (the gathers' first hop)
    int32_t* gms = reinterpret_cast<int32_t*>(sm + l_region(LW));
    int32_t* cis = gms + 2 * U.K;
    double* ccs = reinterpret_cast<double*>(gms + ((2 * U.K + 3 * nc + 1) & ~1));
    for (int t = tid; t < 2 * U.K; t += 256) gms[t] = __ldg(mc.gm + t);
    for (int t = tid; t < 2 * nc; t += 256) {
      cis[t] = __ldg(mc.csrc + t);
      ccs[t] = __ldg(mc.ccoef + t);
    }
    for (int t = tid; t < nc; t += 256) cis[2 * nc + t] = __ldg(mc.cbirth + t);
    mc.gm = gms;
    mc.csrc = cis;
    mc.cbirth = cis + 2 * nc;
    mc.ccoef = ccs;
    __syncthreads();
  }
  MERGE_TICK(1);
  if (!p.schur_split)     // split mode: assemble_l_kernel has written the panel
#ifndef HDD_GATHER_TILE    // A/B: the tile gather below measured slower (latency-bound, not sector-bound)
    for (int g = warp; g < ngp; g += 8) gather_panel_row<8>(mc, k, ng, Kp, W, g, P + int64_t(g) * ldp, lane, 32);
#else
  {
    // columns [0, Kp) on 16 x 32 tiles (coalesced son reads), the R columns row-wise
    double* tile = sm + warp * (kGT * kGTs);             // the front region is idle until the elimination
    const int nct = (Kp + 31) / 32, nt = (ngp / kGT) * nct;
    for (int t = warp; t < nt; t += 8) {
      const int gb = t / nct;
      gather_panel_tile(mc, k, ng, Kp, gb * kGT, (t - gb * nct) * 32, tile, P, ldp, lane);
    }
    for (int g = warp; g < ngp; g += 8) gather_panel_row<8>(mc, k, ng, Kp, W, g, P + int64_t(g) * ldp, lane, 32, Kp);
  }
#endif
  if (tid == 0) s_bad = 0;
  __syncthreads();
  MERGE_TICK(2);
  // Left-looking blocked elimination.  For each 32-row block r0 and each chunk of
  // kLW columns c of C(r0) = [k + r0, W) u [0, k) (the diagonal block's own A22
  // columns first, then the rest of A22, R_gamma, then A21):
  //   T = P[r0 rows][c] - sum_{h < r0} U[h][r0 rows]^T P[h][c]     (depth-r0 DMMA GEMM,
  //       rows h streamed through smem in kLH-row chunks, double-buffered cp.async)
  //   chunk 0 only: Cholesky of T's leading 32x32 block -> L_bb, L_bb^-1 (warp 0)
  //   P[r0 rows][c] = L_bb^-1 T                                   (the row block of U / W / V)
  // Every panel element is written once (no trailing read-modify-write sweeps); the
  // accumulators stay in registers for the whole depth.
  {
    double* LsB = sm;                        // [32][kLdd] factor scratch
    double* LiB = sm + 32 * kLdd;            // [32][kLdd] L_bb^-1 (transposed)
    double* St = sm + 2 * 32 * kLdd;         // stream buffers / T tile [32][kLWs]
    constexpr int kLW = LW, kLWs = LW + kLwPad;
    constexpr int SB = kLH * (kLdd + kLWs);
    constexpr int FN = kLW / 32;
    const int gq = lane & 3, gr = lane >> 2;
    const int m0 = (warp >> 2) * 16, n0 = (warp & 3) * (kLW / 4);
    for (int r0 = 0; r0 < ngp; r0 += kLB) {
      const int nseg = W - k - r0;           // [k + r0, W) first, then [0, k)
      const int nv = nseg + k;
      const double* Arow = P + k + r0;       // A operand columns of row h: Arow[h * ldp + i]
      for (int v0 = 0; v0 < nv; v0 += kLW) {
        auto phys = [&](int v) { return v < nseg ? k + r0 + v : v - nseg; };
        auto stage = [&](int h0, int buf) {
          double* Sa = St + buf * SB;
          double* Sb = Sa + kLH * kLdd;
#ifdef HDD_ELIM_CP8
          for (int t = tid; t < kLH * 32; t += 256) {
            const int g = t >> 5, i = t & 31;
            cp_async8(Sa + g * kLdd + i, Arow + int64_t(h0 + g) * ldp + i);
          }
          for (int t = tid; t < kLH * kLW; t += 256) {
            const int g = t / kLW, j = t - (t / kLW) * kLW;
            const int v = v0 + j;
            if (v < nv) cp_async8(Sb + g * kLWs + j, P + int64_t(h0 + g) * ldp + phys(v));
            else Sb[g * kLWs + j] = 0.0;
          }
#else
          // column pairs as 16-byte copies where the panel columns are even-aligned and
          // contiguous (even ldp; a pair never straddles the segment wrap), else per element
          const bool a16 = ((k + r0) & 1) == 0;
          for (int t = tid; t < kLH * 16; t += 256) {
            const int g = t >> 4, i = 2 * (t & 15);
            const double* src = Arow + int64_t(h0 + g) * ldp + i;
            double* dst = Sa + g * kLdd + i;
            if (a16) cp_async16(dst, src);
            else { cp_async8(dst, src); cp_async8(dst + 1, src + 1); }
          }
          for (int t = tid; t < kLH * (kLW / 2); t += 256) {
            const int g = t / (kLW / 2), j = 2 * (t - (t / (kLW / 2)) * (kLW / 2));
            const int v = v0 + j;
            double* dst = Sb + g * kLWs + j;
            const double* row = P + int64_t(h0 + g) * ldp;
            const int pc = phys(v);
            if (v + 1 < nv && (pc & 1) == 0 && (v + 1 < nseg || v >= nseg)) cp_async16(dst, row + pc);
            else {
              if (v < nv) cp_async8(dst, row + pc); else dst[0] = 0.0;
              if (v + 1 < nv) cp_async8(dst + 1, row + phys(v + 1)); else dst[1] = 0.0;
            }
          }
#endif
          cp_async_commit();
        };
        // the block's own panel values, loaded ahead of the depth-r0 GEMM
        double pv[2][FN][2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int row = m0 + 8 * i + gr, v = v0 + n0 + 8 * j + 2 * gq + e;
              pv[i][j][e] = v < nv ? P[int64_t(r0 + row) * ldp + phys(v)] : 0.0;
            }
        double acc[2][FN][2] = {};
        const int nch = r0 / kLH;
        if (nch > 0) {
          __syncthreads();                   // previous users of the stream buffers are done
          stage(0, 0);
#ifdef HDD_ONE_BARRIER
          for (int c = 0; c < nch; ++c) {     // one barrier per chunk, see schur_epilogue_l
            cp_async_wait<0>();
            __syncthreads();
            if (c + 1 < nch) stage((c + 1) * kLH, (c + 1) & 1);
            const double* Sa = St + (c & 1) * SB;
            warp_gemm_tn<2, FN>(acc, Sa, kLdd, m0, Sa + kLH * kLdd, kLWs, n0, kLH);
          }
          __syncthreads();                    // the T tile below overwrites the stream buffers
#else
          for (int c = 0; c < nch; ++c) {
            if (c + 1 < nch) {
              stage((c + 1) * kLH, (c + 1) & 1);
              cp_async_wait<1>();
            } else {
              cp_async_wait<0>();
            }
            __syncthreads();
            const double* Sa = St + (c & 1) * SB;
            warp_gemm_tn<2, FN>(acc, Sa, kLdd, m0, Sa + kLH * kLdd, kLWs, n0, kLH);
            __syncthreads();
          }
#endif
        } else {
          __syncthreads();
        }
        // T = P[r0 rows][chunk] - acc -> smem
        double* T = St;
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int row = m0 + 8 * i + gr, cc = n0 + 8 * j + 2 * gq + e;
              T[row * kLWs + cc] = pv[i][j][e] - acc[i][j][e];
            }
        __syncthreads();
        if (v0 == 0) {
          if (warp == 0) factor_block32(T, kLWs, LsB, LiB, &s_bad);
          __syncthreads();
        }
        double x[2][FN][2] = {};
        warp_gemm_tn<2, FN>(x, LiB, kLdd, m0, T, kLWs, n0, 32);
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int row = m0 + 8 * i + gr, cc = n0 + 8 * j + 2 * gq + e;
              const int v = v0 + cc;
              if (v < nv) P[int64_t(r0 + row) * ldp + phys(v)] = x[i][j][e];
            }
      }
    }
    __syncthreads();
  }
  MERGE_TICK(3);
  if (s_bad && tid == 0) record_error(p, HDD_ERR_NUMERICAL, s, U.ref_id);
  if (p.mode == 1 && U.fac_off >= 0) store_factors(p, U, s, P, ldp, Kp, false, tid, 256);
  double* out = p.buf[U.buf] + U.out_off * p.bcap + int64_t(s) * U.out_elems;
  const int tk = tri(k);
  for (int c = tid; c < nc; c += 256) {
    double v = gather_sig(mc, c);
    if (c >= 1)
      for (int g = 0; g < ng; ++g) v = fma(P[int64_t(g) * ldp + Kp], P[int64_t(g) * ldp + Kp + c], v);
    out[tk + k * nc + c] = v;
  }
  MERGE_TICK(4);
  if (!p.schur_split) schur_epilogue_l(mc, P, ldp, k, ngp, Kp, nc, out, sm);   // else schur_l_kernel
  MERGE_TICK(5);
}

// ---------------------------------------------------------------------------
// Tier-L Schur update as its own batched GEMM (after merge_l_kernel has left the
// eliminated panel [W | L^T | V] in the HBM workspace):
//   out(a, b) = A~(a, b) - sum_g W[g][a] W[g][b]      (lower Psi, packed)
//   out(a, c) = R~(a, c) - sum_g W[g][a] V[g][c]      (R block)
// One CTA per (128 x 64 output tile, sample, node); the tiles of one node-sample are
// adjacent in the grid so their panel re-reads hit L2.  The panel rows stream through
// a kSS-stage ring of TMA tensor tiles (cp.async.bulk.tensor, one tensor map per
// node: [bcap][ngp][ldp] doubles, box 8 columns x kSR rows -> [col block][row][8]
// in smem, so every DMMA fragment load is bank-conflict free), completing on
// mbarriers; 8 warps as 4 x 2 of 32 x 32 DMMA tiles (16 m8n8k4 per k-step).  The
// assembled A~ / R~ values are gathered from the sons after the K loop.
// ---------------------------------------------------------------------------
constexpr int kSA = 128, kSB = 64, kSR = 32, kSS = 4;
constexpr int kSBX = kSB / 8 + 1;                        // B boxes: one extra for an odd R-block start
constexpr int kSRB = kSA / 8 + kSBX;                     // box index of the folded R columns
constexpr int kSRN = 2;                                  // R boxes (up to 16 folded R columns)
constexpr int kStageD = (kSA + 8 * kSBX + 8 * kSRN) * kSR;   // doubles per stage (A | B | R boxes)
size_t schur_l_smem_bytes() { return sizeof(double) * size_t(kSS) * kStageD + 128; }

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
      ::"r"(smem_u32(dst)), "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)) : "memory");
}

// The R block (nc columns at panel column Kp) rides on tile (a0, a0 + 64) of a 128-row
// block when it fits two 8-column boxes (nc <= 16 - (Kp & 1)) and that tile exists: the
// tile's strictly upper warp tiles compute rows a0..a0+127 x the R columns.  Other row
// blocks get 64-column R tiles.
__host__ __device__ inline bool schur_fold_row(int ia, int k, int nc, int kp_odd) {
  return nc <= 8 * kSRN - kp_odd && ia * kSA + kSB < k;
}
__host__ __device__ inline int schur_l_tiles_dev(int k, int nc, int kp_odd) {
  const int na = (k + kSA - 1) / kSA, nbk = (k + kSB - 1) / kSB, nr = (nc + kSB - 1) / kSB;
  int t = 0;
  for (int ia = 0; ia < na; ++ia) {
    t += (nbk < (ia * kSA + kSA) / kSB ? nbk : (ia * kSA + kSA) / kSB);
    if (!schur_fold_row(ia, k, nc, kp_odd)) t += nr;
  }
  return t;
}

// tile t of a node -> (a0, b0, is_r, fold: carries the R columns); false past the end
__device__ __forceinline__ bool schur_tile(int t, int k, int nc, int kp_odd, int& a0, int& b0, bool& is_r,
                                           bool& fold) {
  const int na = (k + kSA - 1) / kSA, nbk = (k + kSB - 1) / kSB, nr = (nc + kSB - 1) / kSB;
  for (int ia = 0; ia < na; ++ia) {
    const int nb = min(nbk, (ia * kSA + kSA) / kSB);     // b tiles with b0 <= a0 + 127 (lower part)
    const bool fr = schur_fold_row(ia, k, nc, kp_odd);
    a0 = ia * kSA;
    if (t < nb) { b0 = t * kSB; is_r = false; fold = fr && b0 == a0 + kSB; return true; }
    t -= nb;
    if (!fr) {
      if (t < nr) { b0 = t * kSB; is_r = true; fold = false; return true; }
      t -= nr;
    }
  }
  return false;
}

constexpr int kSTPC = 4;                                 // tiles per CTA (the ring runs across them)

// Warp-specialised: warps 0-7 compute (4 x 2 of 32 x 32 DMMA tiles), warp 8 produces
// (waits for a free slot, lane 0 posts the expected bytes, lanes 0..26 issue one TMA box
// each).  full[slot] completes on the TMA bytes, empty[slot] on the 8 consumer warps.
// In a tile that carries the R columns, the warps whose 32 x 32 part is strictly upper
// compute the R rows instead.
__global__ void __launch_bounds__(288, 1) schur_l_kernel(DevPlan p, const DevUpper* __restrict__ nodes,
                                                       const __grid_constant__ CUtensorMap tmap, int node) {
  extern __shared__ __align__(128) double sst_raw[];
  // TMA tensor destinations must be 128-byte aligned
  double* sst = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(sst_raw) + 127) & ~uintptr_t(127));
  __shared__ __align__(8) uint64_t s_full[kSS], s_empty[kSS];
  const int s = blockIdx.y;
  const DevUpper& U = nodes[node];
  const int k = U.k, nc = U.nc;
  const int ngp = upper_ngp(U), Kp = k + ngp;
  const int kp_odd = Kp & 1;
  const int n_tiles = schur_l_tiles_dev(k, nc, kp_odd);
  const int t0 = blockIdx.x * kSTPC;
  if (t0 >= n_tiles) return;
  const int ntl = min(kSTPC, n_tiles - t0);
  const int nch = ngp / kSR;
  const int nq = ntl * nch;                                // (tile, chunk) stream of this CTA
  const int ldp = U.ldp;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < kSS; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == 8) {
    // ---- producer ----
    for (int q = 0; q < nq; ++q) {
      const int slot = q % kSS;
      if (q >= kSS) mbar_wait(&s_empty[slot], uint32_t(((q / kSS) - 1) & 1));
      int a0, b0;
      bool is_r, fold;
      schur_tile(t0 + q / nch, k, nc, kp_odd, a0, b0, is_r, fold);
      const int c = q - (q / nch) * nch;
      // B columns start at bcol; TMA box starts must be 16-byte aligned, so the boxes
      // start at the even column below it (the consumers skip boff columns); boxes
      // that start past the panel row are not issued (their columns are never stored)
      const int bstart = (is_r ? Kp + b0 : b0) & ~1;
      const int col = lane < kSA / 8 ? a0 + 8 * lane
                    : (lane < kSRB ? bstart + 8 * (lane - kSA / 8) : (Kp & ~1) + 8 * (lane - kSRB));
      const bool live = (lane < kSRB || (lane < kSRB + kSRN && fold && 8 * (lane - kSRB) < nc + kp_odd)) &&
                        col < ldp;
      const unsigned nbox = __popc(__ballot_sync(0xffffffffu, live));
      if (lane == 0) mbar_arrive_expect_tx(&s_full[slot], uint32_t(nbox * kSR * 8 * 8));
      __syncwarp();
      if (live) tma_load_3d(sst + slot * kStageD + lane * kSR * 8, &tmap, col, c * kSR, s, &s_full[slot]);
    }
    return;
  }
  // ---- consumers ----
  const int gq = lane & 3, gr = lane >> 2;
  const int wa = (warp >> 1) * 32, wb = (warp & 1) * 32;  // warp tile origin inside the CTA tile
  double* out = p.buf[U.buf] + U.out_off * p.bcap + int64_t(s) * U.out_elems;
  const int tk = tri(k);
  double acc[4][4][2];
  int role = 1, ra = 0;
  for (int q = 0; q < nq; ++q) {
    int a0, b0;
    bool is_r, fold;
    schur_tile(t0 + q / nch, k, nc, kp_odd, a0, b0, is_r, fold);
    const int c = q - (q / nch) * nch;
    const int boff = (is_r ? Kp + b0 : b0) & 1;
    if (c == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      // role: 1 its 32 x 32 part of the tile, 2 the folded R columns of rows a0 + ra ..
      // + 31 (a strictly upper warp tile of an R-carrying tile)
      role = 1;
      ra = wa;
      if (fold && wa < 64) {
        ra = wa + (wb ? 64 : 0);
        role = 2;
      }
    }
    const int slot = q % kSS;
    mbar_wait(&s_full[slot], uint32_t((q / kSS) & 1));
    const double* st = sst + slot * kStageD;
    if (role == 1) {
      const double* As = st + (wa / 8) * kSR * 8;         // 4 A boxes of [kSR][8]
      const double* Bs = st + (kSA / 8) * kSR * 8;        // B boxes
#pragma unroll
      for (int kk = 0; kk < kSR; kk += 4) {
        double av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = As[i * kSR * 8 + (kk + gq) * 8 + gr];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int cb = wb + 8 * j + gr + boff;
          bv[j] = Bs[(cb >> 3) * kSR * 8 + (kk + gq) * 8 + (cb & 7)];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma884(acc[i][j], av[i], bv[j]);
      }
    } else {
      const double* As = st + (ra / 8) * kSR * 8;
      const double* Rs = st + kSRB * kSR * 8;
      // R column 8 j + gr sits at box column 8 j + gr + (Kp & 1)
      const int cr0 = gr + kp_odd, cr1 = 8 + gr + kp_odd;
      const bool two = nc + kp_odd > 8;
#pragma unroll
      for (int kk = 0; kk < kSR; kk += 4) {
        double av[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = As[i * kSR * 8 + (kk + gq) * 8 + gr];
        const double bv0 = Rs[(cr0 >> 3) * kSR * 8 + (kk + gq) * 8 + (cr0 & 7)];
#pragma unroll
        for (int i = 0; i < 4; ++i) dmma884(acc[i][0], av[i], bv0);
        if (two) {
          const double bv1 = cr1 < 16 ? Rs[kSR * 8 + (kk + gq) * 8 + (cr1 & 7)] : 0.0;
#pragma unroll
          for (int i = 0; i < 4; ++i) dmma884(acc[i][1], av[i], bv1);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&s_empty[slot]);           // this warp is done with the slot
    if (c == nch - 1) {
      // epilogue: out already holds A~ / R~ (assemble_l_kernel); out -= W^T [W | V],
      // two rows of fragments at a time (loads first, then the stores)
#pragma unroll
      for (int ih = 0; ih < 4; ih += 2) {
        int idx[2][4][2];
        double old[2][4][2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int a = a0 + ra + 8 * (ih + i) + gr;
              int t = -1;
              if (a < k) {
                if (role == 2) {
                  const int rc = 8 * j + 2 * gq + e;
                  t = (j < kSRN && rc < nc) ? tk + a * nc + rc : -1;
                } else {
                  const int b = b0 + wb + 8 * j + 2 * gq + e;
                  t = !is_r ? (b <= a ? tri(a) + b : -1) : (b < nc ? tk + a * nc + b : -1);
                }
              }
              idx[i][j][e] = t;
              old[i][j][e] = t >= 0 ? out[t] : 0.0;
            }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              if (idx[i][j][e] >= 0) out[idx[i][j][e]] = old[i][j][e] - acc[ih + i][j][e];
      }
    }
  }
}

// Tier-L assembly (split mode): the father's interface panel [A21 | A22 | R_gamma] into
// the HBM workspace and the assembled A11 / R_B (lower packed) into the node output,
// one warp per row, every (row, sample, node) in parallel — the son gathers of
// assemble_father (hdd.py:216-238) as a memory-bound pass, off the elimination's and
// the Schur update's critical paths.
__global__ void __launch_bounds__(256) assemble_l_kernel(DevPlan p, const DevUpper* __restrict__ nodes,
                                                         double* __restrict__ ws, int64_t ws_stride) {
  const DevUpper& U = nodes[blockIdx.z];
  const int s = blockIdx.y;
  const int k = U.k, ng = U.ng, nc = U.nc, ldp = U.ldp;
  const int ngp = upper_ngp(U), Kp = k + ngp, W = Kp + nc;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= ngp + k) return;
  const MergeCtx mc = merge_ctx(p, U, s);
  if (row < ngp) {
    double* P = ws + int64_t(blockIdx.z) * ws_stride * p.bcap + int64_t(s) * ws_stride;
    gather_panel_row<8>(mc, k, ng, Kp, W, row, P + int64_t(row) * ldp, lane, 32);
    return;
  }
  const int a = row - ngp;
  double* out = p.buf[U.buf] + U.out_off * p.bcap + int64_t(s) * U.out_elems;
  for (int b = lane; b <= a; b += 32) out[tri(a) + b] = gather_A(mc, a, b);
  for (int c = lane; c < nc; c += 32) out[tri(k) + a * nc + c] = gather_R(mc, a, c);
}

cudaError_t launch_assemble_l(const DevPlan& p, const DevUpper* nodes_dev, int n_nodes, int B, double* ws,
                              int64_t ws_stride, int max_rows, cudaStream_t s) {
  assemble_l_kernel<<<dim3((max_rows + 7) / 8, B, n_nodes), 256, 0, s>>>(p, nodes_dev, ws, ws_stride);
  return cudaGetLastError();
}

// one launch per node: the node's tensor map travels as a __grid_constant__ parameter
cudaError_t launch_schur_l(const DevPlan& p, const DevUpper* nodes_dev, const CUtensorMap* tmaps, const int* tiles,
                           int n_nodes, int B, cudaStream_t s) {
  const size_t smem = schur_l_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(schur_l_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  for (int n = 0; n < n_nodes; ++n) {
    if (tiles[n] == 0) continue;                          // k = 0 (root): nothing to update
    schur_l_kernel<<<dim3((tiles[n] + kSTPC - 1) / kSTPC, B, 1), 288, smem, s>>>(p, nodes_dev, tmaps[n], n);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

int schur_l_tiles(int k, int nc, int ngp) { return schur_l_tiles_dev(k, nc, (k + ngp) & 1); }
int schur_l_box_rows() { return kSR; }

// Which merge kernel instantiation a depth launches (shared by launch_merge and the
// bench's per-kernel grouping, hdd_plan_stage_kernel): 0..3 merge_m2_kernel<8,256,2> /
// <8,512,1> / <8,256,4> / <8,256,3>, 4 merge_l_kernel<3,64>, 5 merge_l_kernel<2,128>.
int merge_variant(const DevPlan& p, int n_nodes, int B, int tier, size_t smem, int slot) {
  if (tier == 0) {
    // occupancy by panel size: 1 x 512 threads for big panels; 4 x 256 threads (64
    // registers) when 4 panels fit an SM, else 3 x 256 (80 registers; measured)
    static const int force_minb = std::getenv("HDD_M2_MINB") ? std::atoi(std::getenv("HDD_M2_MINB")) : 0;   // A/B hook
    if ((smem > 100 * 1024 && smem <= 113 * 1024) || (force_minb == 2 && smem <= 113 * 1024)) return 0;
    if (smem > 100 * 1024) return 1;
    if (smem <= 55 * 1024 && force_minb != 3) return 2;
    return 3;
  }
  // 3 CTAs/SM (80 registers, some spills) pays when the launch has enough CTAs to
  // fill them and the panel region fits three per SM (measured: C4 depths 3-5 -12 %)
  // (the 2-CTA/SM variant has the smem for 128-column elimination chunks: twice the
  // DMMA work per staged A operand, measured -18 % on the C5 root)
  // (split depths below the root run only the elimination here: the 128-column chunks of
  // the 2-CTA/SM variant win there, measured C5 d2 104.8 -> 99.1 ms, d1 60.3 -> 54.0 ms
  // per 512; the root (slot = depth 0) keeps 3 CTAs/SM: C3 3.15 vs 3.53 ms)
  if ((!p.schur_split || slot == 0) && int64_t(n_nodes) * B >= 148 * 3 * 2 && smem <= 74 * 1024) return 4;
  return 5;
}

const char* merge_variant_name(int v) {
  static const char* names[] = {"merge_m2_kernel<8,256,2>", "merge_m2_kernel<8,512,1>", "merge_m2_kernel<8,256,4>",
                                "merge_m2_kernel<8,256,3>", "merge_l_kernel<3,64>",     "merge_l_kernel<2,128>"};
  return names[v];
}

cudaError_t launch_merge(const DevPlan& p, const DevUpper* nodes_dev, int n_nodes, int B, double* ws,
                         int64_t ws_stride, int tier, int max_rows, size_t smem, int nb, cudaStream_t s, int slot) {
  (void)max_rows;
  (void)nb;
  cudaError_t e;
  dim3 grid(B, n_nodes);
  switch (merge_variant(p, n_nodes, B, tier, smem, slot)) {
    case 0:
      e = cudaFuncSetAttribute(merge_m2_kernel<8, 256, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e != cudaSuccess) return e;
      merge_m2_kernel<8, 256, 2><<<grid, 256, smem, s>>>(p, nodes_dev, slot);
      break;
    case 1:
      e = cudaFuncSetAttribute(merge_m2_kernel<8, 512, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e != cudaSuccess) return e;
      merge_m2_kernel<8, 512, 1><<<grid, 512, smem, s>>>(p, nodes_dev, slot);
      break;
    case 2:
      e = cudaFuncSetAttribute(merge_m2_kernel<8, 256, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e != cudaSuccess) return e;
      merge_m2_kernel<8, 256, 4><<<grid, 256, smem, s>>>(p, nodes_dev, slot);
      break;
    case 3:
      e = cudaFuncSetAttribute(merge_m2_kernel<8, 256, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e != cudaSuccess) return e;
      merge_m2_kernel<8, 256, 3><<<grid, 256, smem, s>>>(p, nodes_dev, slot);
      break;
    case 4:
      e = cudaFuncSetAttribute(merge_l_kernel<3, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e != cudaSuccess) return e;
      merge_l_kernel<3, 64><<<grid, 256, smem, s>>>(p, nodes_dev, ws, ws_stride, slot);
      break;
    default: {
      const size_t sm2 = smem + sizeof(double) * (l_region(128) - kLRegion);
      e = cudaFuncSetAttribute(merge_l_kernel<2, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm2));
      if (e != cudaSuccess) return e;
      merge_l_kernel<2, 128><<<grid, 256, sm2, s>>>(p, nodes_dev, ws, ws_stride, slot);
    }
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K4 (primal): top-down interface back-solve (root_to_leaves, hdd.py:397-432):
// u_gamma = L^-T (v - W u_B), one CTA per (node, sample), depth by depth from the
// root.  The likelihood sweep launches it only on the nodes of the plan's td lists
// (ancestors of the observation owners, hdd_plan.cpp); the merges store factors
// only for those nodes.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) topdown_kernel(DevPlan p, const DevUpper* __restrict__ nodes) {
  extern __shared__ __align__(16) double sm[];
  const DevUpper& U = nodes[blockIdx.y];
  const int s = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = U.k, ng = U.ng;
  const int fw = k + ng + 1;
  double* uB = sm;              // [k]
  double* y = uB + k;           // [ng]
  double* u = y + ng;           // [ng]
  double* dblk = u + ng;        // [32][33]
  double* ub = p.ubuf + int64_t(s) * p.u_elems;
  const double* F = p.fac + int64_t(s) * p.fac_elems + U.fac_off;
  // u_B from the father's u_K (cmap entries are father K-indices)
  if (U.parent >= 0) {
    for (int i = tid; i < k; i += 256) uB[i] = ub[p.upper[U.parent].u_off + p.cmap[U.cmap_off + i]];
  }
  __syncthreads();
  // y = v - W u_B
  for (int g = warp; g < ng; g += 8) {
    const double* row = F + int64_t(g) * fw;
    double acc = 0.0;
    for (int i = lane; i < k; i += 32) acc = fma(row[i], uB[i], acc);
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) y[g] = row[k + ng] - acc;
  }
  __syncthreads();
  // L^T u = y, 32-row blocks from the bottom
  for (int i1 = ng; i1 > 0; i1 -= 32) {
    const int i0 = i1 > 32 ? i1 - 32 : 0;
    for (int r = i0 + warp; r < i1; r += 8) {
      const double* row = F + int64_t(r) * fw + k;
      double acc = 0.0;
      for (int j = i1 + lane; j < ng; j += 32) acc = fma(row[j], u[j], acc);
      for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (lane == 0) y[r] -= acc;
    }
    // stage the diagonal block (coalesced rows) for the serial part
    {
      const int nb = i1 - i0;
      for (int t = tid; t < 32 * 32; t += 256) {
        const int r = t >> 5, j = t & 31;
        dblk[r * 33 + j] = (r < nb && j < nb) ? F[int64_t(i0 + r) * fw + k + i0 + j] : 0.0;
      }
    }
    __syncthreads();
    if (warp == 0) {
      // diagonal block from smem (lane = row), column-oriented back substitution
      const int nb = i1 - i0;
      const int row_i = i0 + lane;
      const double* arow = dblk + lane * 33;
      double yv = lane < nb ? y[row_i] : 0.0;
      double uv = 0.0;
      const double inv_own = lane < nb ? 1.0 / arow[lane] : 0.0;   // off the serial chain
      for (int r = nb - 1; r >= 0; --r) {
        if (lane == r) uv = yv * inv_own;
        const double v = __shfl_sync(0xffffffffu, uv, r);
        if (lane < r) yv = fma(-arow[r], v, yv);
      }
      if (lane < nb) u[row_i] = uv;
    }
    __syncthreads();
  }
  double* mine = ub + U.u_off;
  for (int i = tid; i < k; i += 256) mine[i] = uB[i];
  for (int g = tid; g < ng; g += 256) mine[k + g] = u[g];
}

// ---------------------------------------------------------------------------
// K5: low-rank storage of Psi (lowrank.py:52-77 compress, :155-179 partition,
// hdd.py:280-286).  For every admissible (disjoint-bbox) block A (p x q) of a
// large node's Psi and every sample: randomized range finder Y = A Omega
// (Omega q x l Gaussian, l = k_max + 8), Q = orth(Y) by shifted CholeskyQR2,
// B = Q^T A, pivoted Cholesky of M = B B^T gives a rank-k A_k = (Q C)(L_SS^-1 B_S)
// with EXACT error ||A - A_k||_F^2 = ||A||^2 - ||B||^2 + trace(Schur_k).  k is the
// smallest rank meeting the reference's relative Frobenius criterion eps; the
// block stays dense when k > k_max or k (p + q) >= p q (the reference's rule);
// ||A|| <= 1e-14 ||Psi|| collapses the block to rank 0.  The node's maps are then
// the re-densified compressed maps, as in the reference (hdd.py:227-228).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) psi_norm_kernel(DevPlan p, const DevUpper* __restrict__ nodes, int n_nodes) {
  const DevUpper& U = nodes[blockIdx.y];
  const int s = blockIdx.x;
  const double* psi = p.buf[U.buf] + U.out_off * p.bcap + int64_t(s) * U.out_elems;
  const int k = U.k;
  const int n = tri(k);
  double acc = 0.0;
  for (int t = threadIdx.x; t < n; t += 256) {
    int a = int((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
    if (tri(a + 1) <= t) ++a;
    if (tri(a) > t) --a;
    const double v = psi[t];
    acc += (t - tri(a) == a) ? v * v : 2.0 * v * v;
  }
  __shared__ double red[8];
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t2 = 0.0;
    for (int w = 0; w < 8; ++w) t2 += red[w];
    p.lr_scale[int64_t(blockIdx.y) * p.bcap + s] = t2;
  }
}

// LW: sketch width rounded up (16 / 24 / 32).  Every pass reads each entry of the
// block once: a thread owns a row (pass 1) or a column (passes 2, 3) and keeps the LW
// sketch / projection values of it in registers; partial sums over row or column
// groups meet in shared memory.
template <int LW, int MINB, int NT = 256>   // NT = 512: one CTA per SM (sketches above 113 KB), twice the warps
__global__ void __launch_bounds__(NT, MINB) compress_kernel(DevPlan p, const DevUpper* __restrict__ nodes, int blk0) {
  extern __shared__ __align__(16) double sm[];
  const int32_t* bd = p.lr_blk + 5 * (blk0 + blockIdx.y);
  const int ln = bd[0], roff = bd[1], P_ = bd[2], coff = bd[3], Q_ = bd[4];
  const DevUpper& U = nodes[ln];
  const int s = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int L = p.lr_l;
  double* psi = p.buf[U.buf] + U.out_off * p.bcap + int64_t(s) * U.out_elems;
  const int32_t* R = p.lr_rows + roff;
  const int32_t* Cc = p.lr_cols + coff;
  constexpr int YS = LW + 1;              // sketch row stride (odd: conflict-free column reads)
  double* Y = sm;                         // [P_][YS]
  double* G = Y + size_t(P_) * YS;        // [32][kLdd] gram / pivoted factor C
  double* LiT = G + 32 * kLdd;            // [32][kLdd]
  double* Bc = LiT + 32 * kLdd;           // [LW][65] chunk of B (or D)
  double* red = Bc + LW * 65;             // [64]
  __shared__ int s_bad, s_k, s_conv, s_piv[32];
  __shared__ double s_an2, s_bn2;
  auto A = [&](int i, int j) { const int r = R[i], c = Cc[j]; return r >= c ? psi[tri(r) + c] : psi[tri(c) + r]; };
  // ---- pass 1: Y = A Omega (thread per row, all sketch columns), ||A||^2 ----
  // JG thread groups split the columns when the block has few rows
  const int JG = P_ >= NT ? 1 : (P_ >= NT / 2 ? 2 : (P_ >= NT / 4 ? 4 : 8));
  const int RS = NT / JG;
  double an = 0.0;
  {
    // the JG column groups of a row meet in smem in a fixed order (group 0 stores,
    // groups 1.. add one after another): bitwise reproducible, no atomics
    const int jg = tid / RS, ir = tid - (tid / RS) * RS;
    for (int i0 = 0; i0 < P_; i0 += RS) {     // uniform trip count (barriers below)
      const int i = i0 + ir;
      const bool live = i < P_;
      double acc[LW];
#pragma unroll
      for (int t = 0; t < LW; ++t) acc[t] = 0.0;
      if (live) {
        const int r = R[i];
        const int tr = tri(r);
        #pragma unroll 4   // the block reads of 4 iterations in flight before their FMAs
        for (int j = jg; j < Q_; j += JG) {
          const int c = Cc[j];
          const double a = r >= c ? psi[tr + c] : psi[tri(c) + r];
          an = fma(a, a, an);
          const double2* om = reinterpret_cast<const double2*>(p.lr_omega + j * 32);
#pragma unroll
          for (int t = 0; t < LW; t += 2) {
            const double2 o = __ldg(om + t / 2);
            acc[t] = fma(a, o.x, acc[t]);
            acc[t + 1] = fma(a, o.y, acc[t + 1]);
          }
        }
      }
      double* yr = Y + i * YS;
      for (int g = 0; g < JG; ++g) {
        if (live && jg == g) {
#pragma unroll
          for (int t = 0; t < LW; ++t) {
            const double v = t < L ? acc[t] : 0.0;
            yr[t] = g == 0 ? v : yr[t] + v;
          }
        }
        if (JG > 1) __syncthreads();
      }
    }
  }
  for (int off = 16; off > 0; off >>= 1) an += __shfl_xor_sync(0xffffffffu, an, off);
  if (lane == 0) red[warp] = an;
  __syncthreads();
  if (tid == 0) {
    double t2 = 0.0;
    for (int w = 0; w < NT / 32; ++w) t2 += red[w];
    s_an2 = t2;
  }
  __syncthreads();
  const double an2 = s_an2;
  const double scale2 = p.lr_scale[int64_t(ln) * p.bcap + s];
  if (p.lr_force_wide && p.lr_wide_list && !(an2 <= 1e-28 * scale2)) {   // test hook: every block to the wide sketch
    if (tid == 0) {
      const int slot = atomicAdd(p.lr_wide_n, 1);
      if (slot < p.lr_wide_cap) p.lr_wide_list[slot] = make_int2(blk0 + blockIdx.y, s);
      atomicAdd(p.lr_wide_n + 1, 1);
    }
    return;
  }
  if (an2 <= 1e-28 * scale2) {          // ||A|| <= 1e-14 ||Psi||: rank 0
    for (int t = tid; t < P_ * Q_; t += NT) {
      const int i = t / Q_, j = t - i * Q_;
      const int r = R[i], c = Cc[j];
      psi[r >= c ? tri(r) + c : tri(c) + r] = 0.0;
    }
    return;
  }
  // ---- shifted CholeskyQR2: Q = Y R^-1 (in place) ----
  for (int pass = 0; pass < 2; ++pass) {
    for (int t = tid; t < 32 * 32; t += NT) {
      const int a = t >> 5, b = t & 31;
      double v = 0.0;
      if (a < L && b < L)
        for (int i = 0; i < P_; ++i) v = fma(Y[i * YS + a], Y[i * YS + b], v);
      G[a * kLdd + b] = v;
    }
    __syncthreads();
    if (tid == 0) {
      double tr = 0.0;
      for (int a = 0; a < L; ++a) tr += G[a * kLdd + a];
      const double shift = 1e-13 * tr + 1e-300;
      for (int a = 0; a < 32; ++a) G[a * kLdd + a] = a < L ? G[a * kLdd + a] + shift : 1.0;
      s_bad = 0;
    }
    __syncthreads();
    if (warp == 0) {                                           // G doubles as the L scratch
      if (L <= 16) factor_blockN<16>(G, kLdd, G, LiT, &s_bad);
      else if (L <= 24) factor_blockN<24>(G, kLdd, G, LiT, &s_bad);
      else factor_block32(G, kLdd, G, LiT, &s_bad);
    }
    __syncthreads();
    // Y <- Y R^-1 in place, 32 rows x 8 column groups of 4 per chunk (compute, barrier, write)
    for (int i0 = 0; i0 < P_; i0 += NT / 8) {
      const int i = i0 + (tid >> 3), c0 = (tid & 7) * 4;
      double v[4] = {0.0, 0.0, 0.0, 0.0};
      if (i < P_ && c0 < LW) {
        const double* yr = Y + i * YS;
        for (int t = 0; t < c0 + 4; ++t) {
          const double yt = yr[t];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (t <= c0 + u) v[u] = fma(yt, LiT[t * kLdd + c0 + u], v[u]);
        }
      }
      __syncthreads();
      if (i < P_ && c0 < LW)
#pragma unroll
        for (int u = 0; u < 4; ++u) Y[i * YS + c0 + u] = c0 + u < L ? v[u] : 0.0;
    }
    __syncthreads();
  }
  // ---- pass 2: M = B B^T with B = Q^T A, in 64-column chunks ----
  for (int t = tid; t < 32 * 32; t += NT) G[(t >> 5) * kLdd + (t & 31)] = 0.0;
  constexpr int MU = 1024 / NT;
  double macc[MU] = {};                      // thread owns M entries tid + NT u
  for (int j0 = 0; j0 < Q_; j0 += 64) {
    __syncthreads();
    {   // B chunk: thread per (column, quarter of the rows), all LW rows of B in
        // registers; each A entry read once, the quarters summed in smem in a fixed
        // order (quarter 0 stores, 1..3 add in turn: bitwise reproducible)
      for (int t = tid; t < LW * 65; t += NT) Bc[t] = 0.0;
      __syncthreads();
      const int jj = tid & 63, ig = tid >> 6, j = j0 + jj;
      double v[LW];
#pragma unroll
      for (int u = 0; u < LW; ++u) v[u] = 0.0;
      if (j < Q_) {
        const int c = Cc[j];
        const int tc = tri(c);
        #pragma unroll 4   // the block reads of 4 iterations in flight before their FMAs
        for (int i = ig; i < P_; i += NT / 64) {
          const int r = R[i];
          const double x = r >= c ? psi[tri(r) + c] : psi[tc + r];
          const double* yr = Y + i * YS;
#pragma unroll
          for (int u = 0; u < LW; ++u) v[u] = fma(yr[u], x, v[u]);
        }
      }
      for (int g = 0; g < NT / 64; ++g) {
        if (ig == g && j < Q_)
#pragma unroll
          for (int u = 0; u < LW; ++u)
            if (u < L) Bc[u * 65 + jj] += v[u];
        __syncthreads();
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < MU; ++u) {
      const int e = tid + NT * u, a = e >> 5, b = e & 31;
      if (a < L && b < L)
        for (int jj = 0; jj < 64; ++jj) macc[u] = fma(Bc[a * 65 + jj], Bc[b * 65 + jj], macc[u]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < MU; ++u) {
    const int e = tid + NT * u;
    G[(e >> 5) * kLdd + (e & 31)] = macc[u];
  }
  __syncthreads();
  // ---- pivoted Cholesky of M (one warp): rank decision ----
  if (warp == 0) {
    double bn2 = 0.0;
    for (int a = 0; a < L; ++a) bn2 += G[a * kLdd + a];
    double dg = lane < L ? G[lane * kLdd + lane] : -1.0;   // residual diagonal
    bool used = lane >= L;
    const double budget = p.lr_eps * p.lr_eps * an2;
    double resid = fmax(an2 - bn2, 0.0);
    double trace = 0.0;
    for (int a = 0; a < L; ++a) trace += G[a * kLdd + a];
    int kk = 0;
    // C column t stored in LiT[.][t] (LiT reused as the pivoted factor C, rows = original index)
    while (kk < L && !(resid + trace <= budget)) {
      double best = used ? -1.0 : dg;
      int bi = lane;
      for (int off = 16; off > 0; off >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (best <= 0.0) break;
      const int piv = bi;
      const double sq = sqrt(best);
      double v = 0.0;
      if (!used || lane == piv) {
        v = G[lane * kLdd + piv];
        for (int u = 0; u < kk; ++u) v = fma(-LiT[lane * kLdd + u], LiT[piv * kLdd + u], v);
        v /= sq;
      }
      __syncwarp();
      if (lane < 32) LiT[lane * kLdd + kk] = (lane == piv) ? sq : ((used && lane != piv) ? 0.0 : v);
      if (lane == piv) used = true;
      if (!used) dg -= v * v;
      if (lane == 0) s_piv[kk] = piv;
      trace = 0.0;
      {
        double mine = used ? 0.0 : fmax(dg, 0.0);
        for (int off = 16; off > 0; off >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, off);
        trace = mine;
      }
      ++kk;
      __syncwarp();
    }
    if (lane == 0) { s_k = kk; s_bn2 = bn2; s_conv = (resid + trace <= budget) ? 1 : 0; }
  }
  __syncthreads();
  const int kk = s_k;
  // ranks this sketch decides: up to L - 8 (the requested k_max when k_max <= 24)
  const int kcap = min(p.lr_kmax, L - 8);
  const bool decided = s_conv && kk <= kcap;
  if (!decided && p.lr_kmax > kcap && p.lr_wide_list) {
    // k_max > 24 requested and the block needs a rank above the 32-column sketch:
    // if a rank in (kcap, k_max] can still satisfy the storage rule, hand the block
    // to the wide-sketch kernel (l = k_max + 8 columns, compress_wide_kernel)
    const int64_t kstore = (int64_t(P_) * Q_ - 1) / (P_ + Q_);    // largest k with k (p + q) < p q
    if (kstore > kcap) {
      if (tid == 0) {
        const int slot = atomicAdd(p.lr_wide_n, 1);
        if (slot < p.lr_wide_cap) p.lr_wide_list[slot] = make_int2(blk0 + blockIdx.y, s);
        atomicAdd(p.lr_wide_n + 1, 1);         // running total (hdd_debug_lowrank_wide)
      }
      return;
    }
  }
  if (!decided || int64_t(kk) * (P_ + Q_) >= int64_t(P_) * Q_) return;   // stays dense
  // ---- pass 3: A_k = Q (C D) with D = L_SS^-1 B_S, per 64-column chunk ----
  double* Ec = red + 64;                  // [LW][65]
  for (int j0 = 0; j0 < Q_; j0 += 64) {
    for (int t = tid; t < LW * 65; t += NT) Bc[t] = 0.0;     // B_S rows (pivot order)
    __syncthreads();
    {
      const int jj = tid & 63, ig = tid >> 6, j = j0 + jj;
      double v[LW];
#pragma unroll
      for (int u = 0; u < LW; ++u) v[u] = 0.0;
      if (j < Q_) {
        const int c = Cc[j];
        const int tc = tri(c);
        int pvt[LW];
#pragma unroll
        for (int u = 0; u < LW; ++u) pvt[u] = u < kk ? s_piv[u] : 0;
        #pragma unroll 4   // the block reads of 4 iterations in flight before their FMAs
        for (int i = ig; i < P_; i += NT / 64) {
          const int r = R[i];
          const double x = r >= c ? psi[tri(r) + c] : psi[tc + r];
          const double* yr = Y + i * YS;
#pragma unroll
          for (int u = 0; u < LW; ++u)
            if (u < kk) v[u] = fma(yr[pvt[u]], x, v[u]);
        }
      }
      for (int g = 0; g < NT / 64; ++g) {     // fixed-order sum of the row groups
        if (ig == g && j < Q_)
#pragma unroll
          for (int u = 0; u < LW; ++u)
            if (u < kk) Bc[u * 65 + jj] += v[u];
        __syncthreads();
      }
    }
    __syncthreads();
    for (int jj = tid; jj < 64; jj += NT) {      // forward substitution with L_SS
      for (int u = 0; u < kk; ++u) {
        double v = Bc[u * 65 + jj];
        for (int w = 0; w < u; ++w) v = fma(-LiT[s_piv[u] * kLdd + w], Bc[w * 65 + jj], v);
        Bc[u * 65 + jj] = v / LiT[s_piv[u] * kLdd + u];
      }
    }
    __syncthreads();
    for (int t = tid; t < LW * 64; t += NT) {    // E = C D  (L x 64)
      const int a = t >> 6, jj = t & 63;
      double v = 0.0;
      if (a < L)
        for (int u = 0; u < kk; ++u) v = fma(LiT[a * kLdd + u], Bc[u * 65 + jj], v);
      Ec[a * 65 + jj] = v;
    }
    __syncthreads();
    for (int t = tid; t < P_ * 64; t += NT) {
      const int i = t >> 6, jj = t & 63, j = j0 + jj;
      if (j >= Q_) continue;
      double v = 0.0;
      for (int a = 0; a < L; ++a) v = fma(Y[i * YS + a], Ec[a * 65 + jj], v);
      const int r = R[i], c = Cc[j];
      psi[r >= c ? tri(r) + c : tri(c) + r] = v;
    }
    __syncthreads();
  }
}

// Wide sketch (k_max in 25..64): the blocks the 32-column kernel could not decide
// (queued in lr_wide_list), l = k_max + 8 <= 72 sketch columns, the same algorithm
// (randomized range finder, shifted CholeskyQR2, B = Q^T A, pivoted Cholesky of
// B B^T with the exact error, storage rule) with Y / B in a global scratch slab per
// CTA.  Rare path (ranks above 24 at the requested eps): plain loops, fixed-order
// reductions (bitwise reproducible).
constexpr int kLWW = 72;
__global__ void __launch_bounds__(256) compress_wide_kernel(DevPlan p, const DevUpper* __restrict__ nodes) {
  extern __shared__ __align__(16) double smw[];
  double* G = smw;                          // [kLWW][kLWW + 1] Gram / M
  double* Cm = G + kLWW * (kLWW + 1);       // [kLWW][kLWW + 1] pivoted factor C
  double* red = Cm + kLWW * (kLWW + 1);     // [256]
  __shared__ int s_piv[kLWW], s_k, s_conv;
  __shared__ double s_an2;
  const int tid = threadIdx.x, lane = tid & 31;
  const int L = min(p.lr_kmax + 8, kLWW);
  double* Y = p.lr_wide_scr + int64_t(blockIdx.x) * p.lr_wide_stride;     // [P][kLWW]
  double* Bm = Y + int64_t(p.lr_pmax) * kLWW;                               // [kLWW][qmax]
  const int n_items = min(*p.lr_wide_n, p.lr_wide_cap);
  for (int e = blockIdx.x; e < n_items; e += gridDim.x) {
    const int2 it = p.lr_wide_list[e];
    const int32_t* bd = p.lr_blk + 5 * it.x;               // absolute block index
    const int ln = bd[0], roff = bd[1], P_ = bd[2], coff = bd[3], Q_ = bd[4];
    const int QM = p.lr_qmax;
    const DevUpper& U = nodes[ln];
    const int s = it.y;
    double* psi = p.buf[U.buf] + U.out_off * p.bcap + int64_t(s) * U.out_elems;
    const int32_t* R = p.lr_rows + roff;
    const int32_t* Cc = p.lr_cols + coff;
    auto A = [&](int i, int j) { const int r = R[i], c = Cc[j]; return r >= c ? psi[tri(r) + c] : psi[tri(c) + r]; };
    // 1. Y = A Omega, ||A||^2
    double an = 0.0;
    for (int idx = tid; idx < P_ * L; idx += 256) {
      const int i = idx / L, t = idx - (idx / L) * L;
      double acc = 0.0;
      for (int j = 0; j < Q_; ++j) acc = fma(A(i, j), p.lr_omega_w[j * kLWW + t], acc);
      Y[int64_t(i) * kLWW + t] = acc;
    }
    for (int idx = tid; idx < P_ * Q_; idx += 256) {
      const double a = A(idx / Q_, idx - (idx / Q_) * Q_);
      an = fma(a, a, an);
    }
    red[tid] = an;
    __syncthreads();
    if (tid == 0) {
      double t2 = 0.0;
      for (int w = 0; w < 256; ++w) t2 += red[w];
      s_an2 = t2;
    }
    __syncthreads();
    const double an2 = s_an2;
    // 2. shifted CholeskyQR2: Q = Y L^-T with Y^T Y + shift = L L^T, twice
    for (int pass = 0; pass < 2; ++pass) {
      for (int idx = tid; idx < L * L; idx += 256) {
        const int a = idx / L, b = idx - (idx / L) * L;
        double v = 0.0;
        for (int i = 0; i < P_; ++i) v = fma(Y[int64_t(i) * kLWW + a], Y[int64_t(i) * kLWW + b], v);
        G[a * (kLWW + 1) + b] = v;
      }
      __syncthreads();
      if (tid == 0) {
        double tr = 0.0;
        for (int a = 0; a < L; ++a) tr += G[a * (kLWW + 1) + a];
        const double shift = 1e-13 * tr + 1e-300;
        for (int a = 0; a < L; ++a) G[a * (kLWW + 1) + a] += shift;
      }
      __syncthreads();
      for (int j = 0; j < L; ++j) {             // right-looking Cholesky, lower triangle
        const double d = sqrt(G[j * (kLWW + 1) + j]);
        __syncthreads();
        for (int i = j + 1 + tid; i < L; i += 256) G[i * (kLWW + 1) + j] /= d;
        if (tid == 0) G[j * (kLWW + 1) + j] = d;
        __syncthreads();
        const int w = L - j - 1;
        for (int t = tid; t < w * w; t += 256) {
          const int i = j + 1 + t / w, c = j + 1 + t % w;
          if (c <= i) G[i * (kLWW + 1) + c] = fma(-G[i * (kLWW + 1) + j], G[c * (kLWW + 1) + j], G[i * (kLWW + 1) + c]);
        }
        __syncthreads();
      }
      for (int i = tid; i < P_; i += 256) {     // row i: q L^T = y
        double* y = Y + int64_t(i) * kLWW;
        for (int c = 0; c < L; ++c) {
          double v = y[c];
          for (int t = 0; t < c; ++t) v = fma(-y[t], G[c * (kLWW + 1) + t], v);
          y[c] = v / G[c * (kLWW + 1) + c];
        }
      }
      __syncthreads();
    }
    // 3. B = Q^T A, M = B B^T
    for (int idx = tid; idx < L * Q_; idx += 256) {
      const int a = idx / Q_, j = idx - (idx / Q_) * Q_;
      double v = 0.0;
      for (int i = 0; i < P_; ++i) v = fma(Y[int64_t(i) * kLWW + a], A(i, j), v);
      Bm[int64_t(a) * QM + j] = v;
    }
    __syncthreads();
    for (int idx = tid; idx < L * L; idx += 256) {
      const int a = idx / L, b = idx - (idx / L) * L;
      double v = 0.0;
      for (int j = 0; j < Q_; ++j) v = fma(Bm[int64_t(a) * QM + j], Bm[int64_t(b) * QM + j], v);
      G[a * (kLWW + 1) + b] = v;
    }
    __syncthreads();
    // 4. pivoted Cholesky of M (warp 0, lane owns rows lane, lane + 32, lane + 64)
    if (tid < 32) {
      constexpr int RPL = (kLWW + 31) / 32;
      double dg[RPL];
      bool used[RPL];
      double bn2 = 0.0;
      for (int a = 0; a < L; ++a) bn2 += G[a * (kLWW + 1) + a];
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        const int r = lane + 32 * u;
        used[u] = r >= L;
        dg[u] = r < L ? G[r * (kLWW + 1) + r] : -1.0;
      }
      const double budget = p.lr_eps * p.lr_eps * an2;
      const double resid = fmax(an2 - bn2, 0.0);
      double trace = bn2;
      int kk = 0;
      while (kk < L && !(resid + trace <= budget)) {
        double best = -1.0;
        int bi = 1 << 30;
#pragma unroll
        for (int u = 0; u < RPL; ++u)
          if (!used[u] && (dg[u] > best)) { best = dg[u]; bi = lane + 32 * u; }
        for (int off = 16; off > 0; off >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, off);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
          if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if (best <= 0.0) break;
        const int piv = bi;
        const double sq = sqrt(best);
        double v[RPL];
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
          const int r = lane + 32 * u;
          v[u] = 0.0;
          if (r < L && (!used[u] || r == piv)) {
            double t = G[r * (kLWW + 1) + piv];
            for (int q = 0; q < kk; ++q) t = fma(-Cm[r * (kLWW + 1) + q], Cm[piv * (kLWW + 1) + q], t);
            v[u] = t / sq;
          }
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
          const int r = lane + 32 * u;
          if (r < L) Cm[r * (kLWW + 1) + kk] = r == piv ? sq : (used[u] ? 0.0 : v[u]);
          if (r == piv) used[u] = true;
          if (!used[u]) dg[u] -= v[u] * v[u];
        }
        if (lane == 0) s_piv[kk] = piv;
        double mine = 0.0;
#pragma unroll
        for (int u = 0; u < RPL; ++u) mine += used[u] ? 0.0 : fmax(dg[u], 0.0);
        for (int off = 16; off > 0; off >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, off);
        trace = mine;
        ++kk;
        __syncwarp();
      }
      if (lane == 0) { s_k = kk; s_conv = (resid + trace <= budget) ? 1 : 0; }
    }
    __syncthreads();
    const int kk = s_k;
    if (s_conv && kk <= p.lr_kmax && int64_t(kk) * (P_ + Q_) < int64_t(P_) * Q_) {
      // 5. A_k = Q (C D), D = L_SS^-1 B_S; column j of E = C D replaces column j of B
      for (int j = tid; j < Q_; j += 256) {
        double d[kLWW];
        for (int u = 0; u < kk; ++u) {
          double v = Bm[int64_t(s_piv[u]) * QM + j];
          for (int w = 0; w < u; ++w) v = fma(-Cm[s_piv[u] * (kLWW + 1) + w], d[w], v);
          d[u] = v / Cm[s_piv[u] * (kLWW + 1) + u];
        }
        for (int a = 0; a < L; ++a) {
          double v = 0.0;
          for (int u = 0; u < kk; ++u) v = fma(Cm[a * (kLWW + 1) + u], d[u], v);
          Bm[int64_t(a) * QM + j] = v;
        }
      }
      __syncthreads();
      for (int idx = tid; idx < P_ * Q_; idx += 256) {
        const int i = idx / Q_, j = idx - (idx / Q_) * Q_;
        double v = 0.0;
        for (int a = 0; a < L; ++a) v = fma(Y[int64_t(i) * kLWW + a], Bm[int64_t(a) * QM + j], v);
        const int r = R[i], c = Cc[j];
        psi[r >= c ? tri(r) + c : tri(c) + r] = v;
      }
    }
    __syncthreads();
  }
}

#ifdef HDD_LR_MINB3_BY_SMEM   // A/B: the 80-register 3-CTA/SM instantiation wherever three sketches fit an SM
#define HDD_LR_MINB3(pmax, smem) ((smem) <= 74 * 1024)
#else
#define HDD_LR_MINB3(pmax, smem) ((pmax) <= 64)
#endif
cudaError_t launch_compress(const DevPlan& p, const DevUpper* nodes_dev, int n_nodes, int blk0, int nblk, int B,
                            int pmax, cudaStream_t s) {
  psi_norm_kernel<<<dim3(B, n_nodes), 256, 0, s>>>(p, nodes_dev, n_nodes);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (nblk == 0) return cudaSuccess;
  const int lw = p.lr_l <= 16 ? 16 : (p.lr_l <= 24 ? 24 : 32);
  const size_t smem = sizeof(double) * (size_t(pmax) * (lw + 1) + 2 * 32 * kLdd + 2 * size_t(lw) * 65 + 64) + 64;
  auto go = [&](auto kern, int nt = 256) -> cudaError_t {
    cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e2 != cudaSuccess) return e2;
    kern<<<dim3(B, nblk), nt, smem, s>>>(p, nodes_dev, blk0);
    return cudaGetLastError();
  };
#ifndef HDD_LR_NO_512
  // sketches too large for two CTAs per SM (blocks above 362 rows at the 24-column
  // sketch): one 512-thread CTA per SM instead of one 256-thread CTA (16 warps, not 8)
  static const bool force512 = std::getenv("HDD_LR_FORCE_512") && std::getenv("HDD_LR_FORCE_512")[0] == '1';   // test hook
  if (smem > 113 * 1024 || force512) {
    if (p.lr_l <= 16) return go(compress_kernel<16, 1, 512>, 512);
    if (p.lr_l <= 24) return go(compress_kernel<24, 1, 512>, 512);
    return go(compress_kernel<32, 1, 512>, 512);
  }
#endif
  // levels of small blocks (<= 64 rows) are latency-bound: three CTAs per SM (80
  // registers) beat the spill-free two (measured on C5 depths 10-11)
  if (HDD_LR_MINB3(pmax, smem)) {
    if (p.lr_l <= 16) return go(compress_kernel<16, 3>);
    if (p.lr_l <= 24) return go(compress_kernel<24, 3>);
    return go(compress_kernel<32, 3>);
  }
  if (p.lr_l <= 16) return go(compress_kernel<16, 2>);
  if (p.lr_l <= 24) return go(compress_kernel<24, 2>);
  return go(compress_kernel<32, 2>);
}

cudaError_t launch_compress_wide(const DevPlan& p, const DevUpper* nodes_dev, cudaStream_t s) {
  const size_t smem = sizeof(double) * (2 * size_t(kLWW) * (kLWW + 1) + 256);
  cudaError_t e = cudaFuncSetAttribute(compress_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  compress_wide_kernel<<<p.lr_wide_ctas, 256, smem, s>>>(p, nodes_dev);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Small admissible blocks (p, q <= 64; 75 % of the C5 blocks, all of the deepest
// levels): one WARP per (block, sample), eight per CTA, no block-wide barriers.  Same
// algorithm and decisions as compress_kernel (randomized range finder with the
// same Omega, shifted CholeskyQR2, B = Q^T A kept as H = A^T Q, pivoted Cholesky
// of M = H^T H with the exact error, storage rule, wide-sketch handoff), with lanes
// owning block rows (sketch, CholeskyQR) or block columns (H, re-densification) and
// the L x L factorizations in registers (lane = row, shuffles).  Per warp smem:
// Q [pmax][LW] | H [qmax][LW] | C [LW][LW + 1] | pivots.
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int cw_stride(int pmax, int qmax, int lw) {
  return ((pmax + qmax) * lw + lw * (lw + 1) + lw / 2 + 2 + 1) & ~1;
}

template <int LW>
__global__ void __launch_bounds__(256) compress_warp_kernel(DevPlan p, const DevUpper* __restrict__ nodes, int blk0,
                                                            int nblk, int B, int pmax, int qmax) {
  extern __shared__ __align__(16) double smc[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * (blockDim.x >> 5) + warp;
  if (item >= nblk * B) return;                            // warp-uniform
  const int bl = item / B, s = item - (item / B) * B;     // samples fastest: a CTA shares the block's tables
  const int32_t* bd = p.lr_blk + 5 * (blk0 + bl);
  const int ln = bd[0], roff = bd[1], P_ = bd[2], coff = bd[3], Q_ = bd[4];
  const DevUpper& U = nodes[ln];
  double* psi = p.buf[U.buf] + U.out_off * p.bcap + int64_t(s) * U.out_elems;
  const int32_t* R = p.lr_rows + roff;
  const int32_t* Cc = p.lr_cols + coff;
  const int L = p.lr_l;
  double* Yw = smc + int64_t(warp) * cw_stride(pmax, qmax, LW);   // [P][LW]  (Y, then Q)
  double* Hw = Yw + pmax * LW;                                    // [Q][LW]  (H = A^T Q = B^T)
  double* Cw = Hw + qmax * LW;                                    // [LW][LW + 1] (CholeskyQR L, then C)
  int* pv = reinterpret_cast<int*>(Cw + LW * (LW + 1));           // [LW] pivots
  auto A = [&](int i, int j) { const int r = R[i], c = Cc[j]; return r >= c ? psi[tri(r) + c] : psi[tri(c) + r]; };
  auto wsum = [&](double v) {
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
  };
  // ---- Y = A Omega (lane owns rows lane, lane + 32), ||A||^2 ----
  double y0[LW], y1[LW];
#pragma unroll
  for (int t = 0; t < LW; ++t) y0[t] = y1[t] = 0.0;
  double an = 0.0;
  const bool v0 = lane < P_, v1 = lane + 32 < P_;
  const int r0 = v0 ? R[lane] : 0, r1 = v1 ? R[lane + 32] : 0;
  for (int j = 0; j < Q_; ++j) {
    const int c = Cc[j];
    const double a0 = v0 ? (r0 >= c ? psi[tri(r0) + c] : psi[tri(c) + r0]) : 0.0;
    const double a1 = v1 ? (r1 >= c ? psi[tri(r1) + c] : psi[tri(c) + r1]) : 0.0;
    an = fma(a0, a0, fma(a1, a1, an));
    const double2* om = reinterpret_cast<const double2*>(p.lr_omega + j * 32);
#pragma unroll
    for (int t = 0; t < LW; t += 2) {
      const double2 o = __ldg(om + t / 2);
      y0[t] = fma(a0, o.x, y0[t]);
      y0[t + 1] = fma(a0, o.y, y0[t + 1]);
      y1[t] = fma(a1, o.x, y1[t]);
      y1[t + 1] = fma(a1, o.y, y1[t + 1]);
    }
  }
  const double an2 = wsum(an);
  const double scale2 = p.lr_scale[int64_t(ln) * p.bcap + s];
  if (p.lr_force_wide && p.lr_wide_list && !(an2 <= 1e-28 * scale2)) {
    if (lane == 0) {
      const int slot = atomicAdd(p.lr_wide_n, 1);
      if (slot < p.lr_wide_cap) p.lr_wide_list[slot] = make_int2(blk0 + bl, s);
      atomicAdd(p.lr_wide_n + 1, 1);
    }
    return;
  }
  if (an2 <= 1e-28 * scale2) {                            // ||A|| <= 1e-14 ||Psi||: rank 0
    for (int t = lane; t < P_ * Q_; t += 32) {
      const int i = t / Q_, j = t - (t / Q_) * Q_;
      const int r = R[i], c = Cc[j];
      psi[r >= c ? tri(r) + c : tri(c) + r] = 0.0;
    }
    return;
  }
#pragma unroll
  for (int t = 0; t < LW; ++t) {                          // columns past L stay zero
    if (t >= L) { y0[t] = 0.0; y1[t] = 0.0; }
  }
  // ---- shifted CholeskyQR2: Q = Y L^-T with Y^T Y + shift = L L^T (twice) ----
  for (int pass = 0; pass < 2; ++pass) {
    if (v0)
#pragma unroll
      for (int t = 0; t < LW; ++t) Yw[lane * LW + t] = y0[t];
    if (v1)
#pragma unroll
      for (int t = 0; t < LW; ++t) Yw[(lane + 32) * LW + t] = y1[t];
    __syncwarp();
    double g[LW];                                           // lane a: row a of Y^T Y
#pragma unroll
    for (int b = 0; b < LW; ++b) g[b] = 0.0;
    const int ar = lane < LW ? lane : 0;
    for (int i = 0; i < P_; ++i) {
      const double ya = Yw[i * LW + ar];
#pragma unroll
      for (int b = 0; b < LW; ++b) g[b] = fma(ya, Yw[i * LW + b], g[b]);
    }
    double gd = 0.0;
#pragma unroll
    for (int b = 0; b < LW; ++b) gd = (b == lane) ? g[b] : gd;
    const double tr = wsum(lane < L ? gd : 0.0);
    const double shift = 1e-13 * tr + 1e-300;
#pragma unroll
    for (int b = 0; b < LW; ++b) {
      if (lane >= L || b >= L) g[b] = (b == lane) ? 1.0 : 0.0;   // identity past the sketch width
      else if (b == lane) g[b] += shift;
    }
    // register Cholesky, lane = row (rows >= LW are idle copies of row LW - 1)
    double ild = 1.0;
#pragma unroll
    for (int j = 0; j < LW; ++j) {
      const double dj = __shfl_sync(0xffffffffu, g[j], j);
      const double il = rsqrt_nr(dj);
      const double lij = g[j] * il;
#pragma unroll
      for (int l = j + 1; l < LW; ++l) g[l] = fma(-lij, __shfl_sync(0xffffffffu, lij, l), g[l]);
      if (lane == j) ild = il;
      g[j] = lij;
    }
    __syncwarp();
    if (lane < LW)                                          // L (lower, row-major) with 1/L_jj on the diagonal
#pragma unroll
      for (int l = 0; l < LW; ++l)
        if (l <= lane) Cw[lane * (LW + 1) + l] = l == lane ? ild : g[l];
    __syncwarp();
    // rows: q L^T = y  ->  q_c = (y_c - sum_{t < c} q_t L_ct) / L_cc
#pragma unroll
    for (int c = 0; c < LW; ++c) {
      double a = y0[c], b = y1[c];
#pragma unroll
      for (int t = 0; t < c; ++t) {
        const double lct = Cw[c * (LW + 1) + t];
        a = fma(-y0[t], lct, a);
        b = fma(-y1[t], lct, b);
      }
      const double il = Cw[c * (LW + 1) + c];
      y0[c] = a * il;
      y1[c] = b * il;
    }
    __syncwarp();
  }
  if (v0)
#pragma unroll
    for (int t = 0; t < LW; ++t) Yw[lane * LW + t] = y0[t];
  if (v1)
#pragma unroll
    for (int t = 0; t < LW; ++t) Yw[(lane + 32) * LW + t] = y1[t];
  __syncwarp();
  // ---- H = A^T Q (lane owns columns lane, lane + 32) ----
  {
    double h0[LW], h1[LW];
#pragma unroll
    for (int t = 0; t < LW; ++t) h0[t] = h1[t] = 0.0;
    const bool w0 = lane < Q_, w1 = lane + 32 < Q_;
    const int c0 = w0 ? Cc[lane] : 0, c1 = w1 ? Cc[lane + 32] : 0;
    for (int i = 0; i < P_; ++i) {
      const int r = R[i];
      const double x0 = w0 ? (r >= c0 ? psi[tri(r) + c0] : psi[tri(c0) + r]) : 0.0;
      const double x1 = w1 ? (r >= c1 ? psi[tri(r) + c1] : psi[tri(c1) + r]) : 0.0;
#pragma unroll
      for (int t = 0; t < LW; ++t) {
        const double q = Yw[i * LW + t];
        h0[t] = fma(q, x0, h0[t]);
        h1[t] = fma(q, x1, h1[t]);
      }
    }
    if (w0)
#pragma unroll
      for (int t = 0; t < LW; ++t) Hw[lane * LW + t] = h0[t];
    if (w1)
#pragma unroll
      for (int t = 0; t < LW; ++t) Hw[(lane + 32) * LW + t] = h1[t];
  }
  __syncwarp();
  // ---- M = H^T H (lane a: row a), pivoted Cholesky in registers ----
  double m[LW];
#pragma unroll
  for (int c = 0; c < LW; ++c) m[c] = 0.0;
  {
    const int ar = lane < LW ? lane : 0;
    for (int j = 0; j < Q_; ++j) {
      const double ha = Hw[j * LW + ar];
#pragma unroll
      for (int c = 0; c < LW; ++c) m[c] = fma(ha, Hw[j * LW + c], m[c]);
    }
  }
  double dg = -1.0;
#pragma unroll
  for (int c = 0; c < LW; ++c) dg = (c == lane) ? m[c] : dg;
  bool used = lane >= L;
  if (used) dg = -1.0;
  const double bn2 = wsum(used ? 0.0 : dg);
  const double budget = p.lr_eps * p.lr_eps * an2;
  const double resid = fmax(an2 - bn2, 0.0);
  double trace = bn2;
  double crow[LW];                                         // row `lane` of C
#pragma unroll
  for (int u = 0; u < LW; ++u) crow[u] = 0.0;
  int kk = 0;
  while (kk < L && !(resid + trace <= budget)) {
    double best = used ? -1.0 : dg;
    int bi = lane;
    for (int off = 16; off > 0; off >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (best <= 0.0) break;
    const int piv = bi;
    const double sq = sqrt(best);
    double mp = 0.0;                                       // M[lane][piv]
#pragma unroll
    for (int c = 0; c < LW; ++c) mp = (c == piv) ? m[c] : mp;
    double v = mp;
#pragma unroll
    for (int u = 0; u < LW; ++u)
      if (u < kk) v = fma(-crow[u], __shfl_sync(0xffffffffu, crow[u], piv), v);
    v /= sq;
    const double cval = lane == piv ? sq : (used ? 0.0 : v);
#pragma unroll
    for (int u = 0; u < LW; ++u)
      if (u == kk) crow[u] = cval;
    if (lane == piv) used = true;
    if (!used) dg -= v * v;
    if (lane == 0) pv[kk] = piv;
    trace = wsum(used ? 0.0 : fmax(dg, 0.0));
    ++kk;
  }
  const bool conv = resid + trace <= budget;
  const int kcap = min(p.lr_kmax, L - 8);
  const bool decided = conv && kk <= kcap;
  if (!decided && p.lr_kmax > kcap && p.lr_wide_list) {
    const int64_t kstore = (int64_t(P_) * Q_ - 1) / (P_ + Q_);
    if (kstore > kcap) {
      if (lane == 0) {
        const int slot = atomicAdd(p.lr_wide_n, 1);
        if (slot < p.lr_wide_cap) p.lr_wide_list[slot] = make_int2(blk0 + bl, s);
        atomicAdd(p.lr_wide_n + 1, 1);
      }
      return;
    }
  }
  if (!decided || int64_t(kk) * (P_ + Q_) >= int64_t(P_) * Q_) return;   // stays dense
  // ---- A_k = Q (C D), D = L_SS^-1 B_S with B_S[u][j] = H[j][piv_u] ----
  __syncwarp();
  if (lane < LW)
#pragma unroll
    for (int u = 0; u < LW; ++u) Cw[lane * (LW + 1) + u] = crow[u];
  __syncwarp();
  for (int j = lane; j < Q_; j += 32) {
    double d[LW], e[LW];
#pragma unroll
    for (int u = 0; u < LW; ++u) {
      d[u] = 0.0;
      if (u < kk) {
        const int pu = pv[u];
        double t = Hw[j * LW + pu];
#pragma unroll
        for (int w = 0; w < u; ++w) t = fma(-Cw[pu * (LW + 1) + w], d[w], t);
        d[u] = t / Cw[pu * (LW + 1) + u];
      }
    }
#pragma unroll
    for (int a = 0; a < LW; ++a) {
      double t = 0.0;
#pragma unroll
      for (int u = 0; u < LW; ++u)
        if (u < kk) t = fma(Cw[a * (LW + 1) + u], d[u], t);
      e[a] = a < L ? t : 0.0;
    }
    const int c = Cc[j];
    for (int i = 0; i < P_; ++i) {
      double t = 0.0;
#pragma unroll
      for (int a = 0; a < LW; ++a) t = fma(Yw[i * LW + a], e[a], t);
      const int r = R[i];
      psi[r >= c ? tri(r) + c : tri(c) + r] = t;
    }
  }
}

cudaError_t launch_compress_warp(const DevPlan& p, const DevUpper* nodes_dev, int blk0, int nblk, int B, int pmax,
                                 int qmax, cudaStream_t s) {
  if (nblk == 0) return cudaSuccess;
  const int lw = p.lr_l <= 16 ? 16 : (p.lr_l <= 24 ? 24 : 32);
  const size_t per_warp = sizeof(double) * size_t(cw_stride(pmax, qmax, lw));
  static const int max_nw = std::getenv("HDD_LR_WARPS") ? std::atoi(std::getenv("HDD_LR_WARPS")) : 8;   // A/B hook
  const int nw = int(std::max<size_t>(1, std::min<size_t>(size_t(max_nw), (220 * 1024) / per_warp)));   // warps per CTA
  const size_t smem = per_warp * nw;
  const int64_t items = int64_t(nblk) * B;
  const dim3 grid(unsigned((items + nw - 1) / nw));
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    kern<<<grid, 32 * nw, smem, s>>>(p, nodes_dev, blk0, nblk, B, pmax, qmax);
    return cudaGetLastError();
  };
  if (lw == 16) return go(compress_warp_kernel<16>);
  if (lw == 24) return go(compress_warp_kernel<24>);
  return go(compress_warp_kernel<32>);
}

cudaError_t launch_topdown(const DevPlan& p, const DevUpper* nodes_dev, int n_nodes, int B, int max_kng,
                           cudaStream_t s) {
  const size_t smem = sizeof(double) * (size_t(max_kng) + 32 * 33) + 64;
  cudaError_t e = cudaFuncSetAttribute(topdown_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  dim3 grid(B, n_nodes);
  topdown_kernel<<<grid, 256, smem, s>>>(p, nodes_dev);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K4: observations + Gaussian log-likelihood
// ---------------------------------------------------------------------------
__global__ void finalize_kernel(DevPlan p, int B, double* __restrict__ S, double* __restrict__ ll) {
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (s >= B) return;
  const double* sig = p.buf[p.root_buf] + p.root_off + int64_t(s) * p.root_elems + p.root_sig;
  const double* ub = p.ubuf ? p.ubuf + int64_t(s) * p.u_elems : nullptr;
  double acc = 0.0;
  for (int o = lane; o < p.n_obs; o += 32) {
    const int kind = p.route_kind[o];
    double v;
    if (kind == 0) {
      v = sig[p.route_col[o]];
    } else if (kind == 1) {
      v = route_const(p, o, s);
    } else if (kind == 2) {
      // leaf point: l^T u_B(leaf) + sigma, u_B from the father's u_K
      const int l = p.route_node[o];
      const double* fn = p.fbuf + (int64_t(s) * p.n_fslots + p.route_slot[o]) * 65;
      const int par = p.leaves[l].parent;
      const double* up = ub + p.upper[par].u_off;
      const int32_t* cm = p.leaf_cmap + int64_t(l) * kLeafPerim;
      double t = fn[64];
      for (int b = 0; b < kLeafPerim; ++b) {
        const int c = cm[b];
        if (c >= 0) t = fma(fn[b], up[c], t);
      }
      v = t;
    } else {
      const DevUpper& U = p.upper[p.route_node[o]];
      v = ub[U.u_off + U.k + p.route_col[o]];
    }
    if (!isfinite(v)) record_error(p, HDD_ERR_NUMERICAL, s, -1);
    if (S) S[int64_t(s) * p.n_obs + o] = v;
    if (p.y) {
      const double r = (p.y[o] - v) / p.sigma[o];
      acc = fma(r, r, acc);
    }
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0 && ll) ll[s] = p.y ? (-0.5 * acc - p.ll_const) : 0.0;
}

// ---------------------------------------------------------------------------
// Posterior weights of a gathered batch (a13): one CTA, two passes over the batch
// (max / first argmax, then sum exp(joint - max)), fixed reduction order.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) posterior_kernel(const double* __restrict__ ll,
                                                         const double* __restrict__ lp, int64_t n,
                                                         double* __restrict__ w, int64_t* __restrict__ idx,
                                                         double* __restrict__ lse) {
  __shared__ double s_v[32];
  __shared__ int64_t s_i[32];
  __shared__ double s_mx, s_lse;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  auto joint = [&](int64_t t) { return lp ? ll[t] + lp[t] : ll[t]; };
  // numpy argmax order: NaN ranks above every number (the first NaN wins), then the
  // largest value, ties to the first index
  auto better = [](double v, int64_t i, double m, int64_t mi_) {
    const bool vn = isnan(v), mn = isnan(m);
    if (vn != mn) return vn;
    return (vn || v == m) ? i < mi_ : v > m;
  };
  double mx = -INFINITY;
  int64_t mi = INT64_MAX;
  for (int64_t t = tid; t < n; t += blockDim.x) {
    const double v = joint(t);
    if (better(v, t, mx, mi)) { mx = v; mi = t; }
  }
  for (int off = 16; off > 0; off >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, mx, off);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, mi, off);
    if (better(ov, oi, mx, mi)) { mx = ov; mi = oi; }
  }
  if (lane == 0) { s_v[warp] = mx; s_i[warp] = mi; }
  __syncthreads();
  if (tid == 0) {
    double m = s_v[0];
    int64_t i = s_i[0];
    for (int q = 1; q < nw; ++q)
      if (better(s_v[q], s_i[q], m, i)) { m = s_v[q]; i = s_i[q]; }
    s_mx = m;
    *idx = i;
  }
  __syncthreads();
  const double m = s_mx;
  double sum = 0.0;
  for (int64_t t = tid; t < n; t += blockDim.x) sum += exp(joint(t) - m);
  for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
  __syncthreads();
  if (lane == 0) s_v[warp] = sum;
  __syncthreads();
  if (tid == 0) {
    double tot = 0.0;
    for (int q = 0; q < nw; ++q) tot += s_v[q];
    s_lse = m + log(tot);
    *lse = s_lse;
  }
  __syncthreads();
  const double l = s_lse;
  for (int64_t t = tid; t < n; t += blockDim.x) w[t] = exp(joint(t) - l);
}

cudaError_t launch_posterior(const double* ll, const double* lp, int64_t n, double* w, int64_t* idx, double* lse,
                             cudaStream_t s) {
  posterior_kernel<<<1, 1024, 0, s>>>(ll, lp, n, w, idx, lse);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const DevPlan& p, int B, double* S, double* ll, cudaStream_t s) {
  finalize_kernel<<<(B + 7) / 8, 256, 0, s>>>(p, B, S, ll);
  return cudaGetLastError();
}

}  // namespace hdd

namespace hdd {

// ---------------------------------------------------------------------------
// K6: full-solution path, the in-leaf part of root_to_leaves (hdd.py:397-432).
// The upper interfaces come from the primal top-down sweep (u_K of every upper
// node); each kernel leaf then solves for its 15 x 15 interior nodes from its 64
// perimeter values: the exact P1 stiffness of the structured triangulation is the
// variable-coefficient 5-point stencil, so the interior system is banded (half
// bandwidth 15) and one warp factors it by a right-looking band Cholesky in
// shared memory, then runs the two triangular solves.
// ---------------------------------------------------------------------------
constexpr int kIn = kLeafCells - 1;        // interior nodes per side
constexpr int kNI = kIn * kIn;             // interior unknowns
constexpr int kBW = kIn + 1;               // band width incl. the diagonal

// perimeter index of local node (x, y) in the sorted-id perimeter order
__device__ __forceinline__ int perim_index(int x, int y) {
  return y == 0 ? x : (y == kLeafCells ? 3 * kLeafCells - 1 + x : kLeafCells + 1 + 2 * (y - 1) + (x == kLeafCells));
}

// leaf_list: the kernel leaves to solve (NULL = all); omega_pos: global node id -> output
// column (solve_subdomain: the target's idx_omega order, -1 = not in the target), NULL =
// full U rows of n_nodes
__global__ void __launch_bounds__(32) leaf_solve_kernel(DevPlan p, double* __restrict__ U, int64_t n_nodes,
                                                        const int32_t* __restrict__ leaf_list,
                                                        const int32_t* __restrict__ omega_pos) {
  __shared__ double band[kNI * kBW];       // column j: rows j .. j+15 of L
  __shared__ double rhs[kNI], invd[kNI];
  __shared__ double kap[512];
  __shared__ double ub[kLeafPerim];
  const int leaf = leaf_list ? leaf_list[blockIdx.x] : int(blockIdx.x), s = blockIdx.y, lane = threadIdx.x;
  const DevLeaf& L = p.leaves[leaf];
  const int N = p.N, m = p.m;
  const double* kb = p.kappa + int64_t(s) * 2 * N * N;
  for (int t = lane; t < 512; t += 32) kap[t] = kb[2 * (int64_t(L.i0 + (t >> 5)) * N + L.j0) + (t & 31)];
  for (int t = lane; t < kLeafPerim; t += 32) {
    const int c = L.parent >= 0 ? p.leaf_cmap[int64_t(leaf) * kLeafPerim + t] : -1;
    ub[t] = c >= 0 ? p.ubuf[int64_t(s) * p.u_elems + p.upper[L.parent].u_off + c]
                   : leaf_gval(p, leaf, s, t);    // u = g on the domain boundary
  }
  __syncwarp();
  auto k0 = [&](int cx, int cy) { return kap[cx * 32 + 2 * cy]; };
  auto k1 = [&](int cx, int cy) { return kap[cx * 32 + 2 * cy + 1]; };
  const double h2 = p.h * p.h;
  for (int j = lane; j < kNI; j += 32) {
    const int x = j % kIn + 1, y = j / kIn + 1;
    // cell contributions of fem.py:126-145 (node = a of (x,y), b of (x-1,y), c of (x,y-1), d of (x-1,y-1))
    const double D = 0.5 * (k0(x, y) + k1(x, y)) + k0(x - 1, y) + k1(x, y - 1) + 0.5 * (k0(x - 1, y - 1) + k1(x - 1, y - 1));
    const double E = -0.5 * k0(x, y) - 0.5 * k1(x, y - 1);           // to (x+1, y)
    const double Nn = -0.5 * k1(x, y) - 0.5 * k0(x - 1, y);          // to (x, y+1)
    const double Wc = -0.5 * k0(x - 1, y) - 0.5 * k1(x - 1, y - 1);  // to (x-1, y)
    const double Sc = -0.5 * k1(x, y - 1) - 0.5 * k0(x - 1, y - 1);  // to (x, y-1)
    double* col = band + j * kBW;
    col[0] = D;
    col[1] = x < kIn ? E : 0.0;
#pragma unroll
    for (int i = 2; i < kBW - 1; ++i) col[i] = 0.0;
    col[kBW - 1] = y < kIn ? Nn : 0.0;
    // lumped load (psi_f = h^2/6 diag(2,1,1,2) per cell -> h^2 f at an interior node)
    double r = h2 * (p.f ? sample_f(p, s)[int64_t(L.j0 + y) * m + L.i0 + x] : 1.0);
    if (x == 1) r -= Wc * ub[perim_index(0, y)];
    if (x == kIn) r -= E * ub[perim_index(kLeafCells, y)];
    if (y == 1) r -= Sc * ub[perim_index(x, 0)];
    if (y == kIn) r -= Nn * ub[perim_index(x, kLeafCells)];
    rhs[j] = r;
  }
  // this lane's (i, m) pairs of the rank-1 band update, 1 <= m <= i <= 15 (120 pairs)
  int pi[4], pm[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    int t = lane + 32 * u, i = 1;
    while (t >= i) { t -= i; ++i; }
    pi[u] = i;
    pm[u] = t + 1;
    if (lane + 32 * u >= 120) pi[u] = 0;
  }
  __syncwarp();
  bool bad = false;
  for (int j = 0; j < kNI; ++j) {
    double* col = band + j * kBW;
    const double d = col[0];
    const double il = rsqrt_nr(d);
    bad |= !(d > 0.0);
    const double li = (lane >= 1 && lane < kBW) ? col[lane] * il : 0.0;
    __syncwarp();
    if (lane >= 1 && lane < kBW) col[lane] = li;
    if (lane == 0) { col[0] = d * il; invd[j] = il; }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = pi[u], mm = pm[u];
      if (i > 0 && j + i < kNI) band[(j + mm) * kBW + (i - mm)] -= col[i] * col[mm];
    }
    __syncwarp();
  }
  if (lane == 0 && bad) record_error(p, HDD_ERR_NUMERICAL, s, L.ref_id);
  // L y = rhs
  for (int j = 0; j < kNI; ++j) {
    if (lane == 0) rhs[j] *= invd[j];
    __syncwarp();
    const double yj = rhs[j];
    if (lane >= 1 && lane < kBW && j + lane < kNI) rhs[j + lane] -= band[j * kBW + lane] * yj;
    __syncwarp();
  }
  // L^T x = y
  for (int j = kNI - 1; j >= 0; --j) {
    if (lane == 0) rhs[j] *= invd[j];
    __syncwarp();
    const double xj = rhs[j];
    if (lane >= 1 && lane < kBW && j - lane >= 0) rhs[j - lane] -= band[(j - lane) * kBW + lane] * xj;
    __syncwarp();
  }
  double* Us = U + int64_t(s) * n_nodes;
  for (int j = lane; j < kNI; j += 32) {
    const int x = j % kIn + 1, y = j / kIn + 1;
    const int64_t id = int64_t(L.j0 + y) * m + L.i0 + x;
    if (!omega_pos) Us[id] = rhs[j];
    else if (omega_pos[id] >= 0) Us[omega_pos[id]] = rhs[j];
  }
  for (int t = lane; t < kLeafPerim; t += 32) {
    int x, y;
    if (t <= kLeafCells) { x = t; y = 0; }
    else if (t >= 3 * kLeafCells - 1) { x = t - (3 * kLeafCells - 1); y = kLeafCells; }
    else { y = (t - kLeafCells - 1) / 2 + 1; x = ((t - kLeafCells - 1) & 1) ? kLeafCells : 0; }
    const int64_t id = int64_t(L.j0 + y) * m + L.i0 + x;
    if (!omega_pos) Us[id] = ub[t];
    else if (omega_pos[id] >= 0) Us[omega_pos[id]] = ub[t];
  }
}

cudaError_t launch_leaf_solve(const DevPlan& p, int B, double* U, int64_t n_nodes, cudaStream_t s,
                              const int32_t* leaf_list, int n_list, const int32_t* omega_pos) {
  dim3 grid(leaf_list ? n_list : p.n_leaves, B);
  leaf_solve_kernel<<<grid, 32, 0, s>>>(p, U, n_nodes, leaf_list, omega_pos);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Caller-supplied coefficient fields (hdd_forward_batch_kappa): the check of
// CoefficientField (fem.py:31-32) — every value positive and finite — on the device.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) kappa_check_kernel(DevPlan p, const double* __restrict__ kappa, int64_t nt) {
  const int s = blockIdx.y;
  const double* kb = kappa + int64_t(s) * nt;
  bool bad = false;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < nt; t += int64_t(gridDim.x) * blockDim.x) {
    const double v = kb[t];
    bad |= !(v > 0.0) || !isfinite(v);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) record_error(p, HDD_ERR_CONFIG, s, -1);
}

cudaError_t launch_kappa_check(const DevPlan& p, const double* kappa, int B, cudaStream_t s) {
  const int64_t nt = int64_t(2) * p.N * p.N;
  const int gx = int(std::min<int64_t>(64, (nt + 255) / 256));
  kappa_check_kernel<<<dim3(gx, B), 256, 0, s>>>(p, kappa, nt);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Meshes below one kernel leaf (levels 1-3, N <= 8 cells per side): the whole
// tree's Schur recursion collapses to the elimination of the (N-1)^2 interior
// unknowns at the root (the reference's leaves_to_root on such a mesh ends in the
// same SPD system).  One warp per sample: 5-point P1 stiffness from the cell
// patterns (fem.py:126-145), lumped load h^2 f (psi_f = h^2/6 diag(2,1,1,2) per
// cell), Dirichlet data moved to the right-hand side, dense Cholesky in shared
// memory, then the observations (points, per-triangle means, oracle.py:74-83 /
// functionals.py:47-61) and the Gaussian log-likelihood (bayes.py:222-224).
// ---------------------------------------------------------------------------
constexpr int kTinyN = 8, kTinyI = kTinyN - 1, kTinyNI = kTinyI * kTinyI;

__global__ void __launch_bounds__(32) tiny_kernel(DevPlan p, int B, double* __restrict__ S, double* __restrict__ ll,
                                                  double* __restrict__ U, int64_t n_nodes) {
  __shared__ double kap[2 * kTinyN * kTinyN];
  __shared__ double A[kTinyNI * kTinyNI];
  __shared__ double rhs[kTinyNI];
  __shared__ double u[(kTinyN + 1) * (kTinyN + 1)];
  const int s = blockIdx.x, lane = threadIdx.x;
  const int N = p.N, m = p.m, ni = N - 1, n = ni * ni;
  const double* kb = p.kappa + int64_t(s) * 2 * N * N;
  for (int t = lane; t < 2 * N * N; t += 32) kap[t] = kb[t];
  for (int t = lane; t < m * m; t += 32) {
    double gv = p.gfull ? p.gfull[t] : 0.0;
    if (p.gcall) {                          // boundary position in increasing-id order
      const int i = t % m, j = t / m;
      const bool bnd = i == 0 || j == 0 || i == N || j == N;
      const int pos = j == 0 ? i : (j == N ? m + 2 * (N - 1) + i : m + 2 * (j - 1) + (i == N ? 1 : 0));
      gv = bnd ? p.gcall[int64_t(s) * p.g_stride + pos] : 0.0;
    }
    u[t] = gv;
  }
  for (int t = lane; t < n * n; t += 32) A[t] = 0.0;
  __syncwarp();
  auto k0 = [&](int cx, int cy) { return kap[2 * (cx * N + cy)]; };
  auto k1 = [&](int cx, int cy) { return kap[2 * (cx * N + cy) + 1]; };
  const double h2 = p.h * p.h;
  // row j = interior node (x, y), x, y in 1..N-1; cells (x-1..x, y-1..y) all exist
  for (int j = lane; j < n; j += 32) {
    const int x = j % ni + 1, y = j / ni + 1;
    const double Dg = 0.5 * (k0(x, y) + k1(x, y)) + k0(x - 1, y) + k1(x, y - 1) + 0.5 * (k0(x - 1, y - 1) + k1(x - 1, y - 1));
    const double E = -0.5 * k0(x, y) - 0.5 * k1(x, y - 1);           // to (x+1, y)
    const double Nn = -0.5 * k1(x, y) - 0.5 * k0(x - 1, y);          // to (x, y+1)
    const double Wc = -0.5 * k0(x - 1, y) - 0.5 * k1(x - 1, y - 1);  // to (x-1, y)
    const double Sc = -0.5 * k1(x, y - 1) - 0.5 * k0(x - 1, y - 1);  // to (x, y-1)
    A[j * n + j] = Dg;
    if (x < ni) A[(j + 1) * n + j] = E;
    if (y < ni) A[(j + ni) * n + j] = Nn;
    double r = h2 * (p.f ? sample_f(p, s)[y * m + x] : 1.0);
    if (x == 1) r -= Wc * u[y * m];
    if (x == ni) r -= E * u[y * m + N];
    if (y == 1) r -= Sc * u[x];
    if (y == ni) r -= Nn * u[N * m + x];
    rhs[j] = r;
  }
  __syncwarp();
  bool bad = false;
  for (int j = 0; j < n; ++j) {            // right-looking Cholesky, lower triangle
    const double d = A[j * n + j];
    bad |= !(d > 0.0);
    const double sq = sqrt(d), il = 1.0 / sq;
    __syncwarp();
    for (int i = j + 1 + lane; i < n; i += 32) A[i * n + j] *= il;
    if (lane == 0) A[j * n + j] = sq;
    __syncwarp();
    const int w = n - j - 1;
    for (int t = lane; t < w * w; t += 32) {
      const int i = j + 1 + t / w, c = j + 1 + t % w;
      if (c <= i) A[i * n + c] = fma(-A[i * n + j], A[c * n + j], A[i * n + c]);
    }
    __syncwarp();
  }
  if (lane == 0 && bad) record_error(p, HDD_ERR_NUMERICAL, s, p.root_ref);
  for (int j = 0; j < n; ++j) {            // L y = rhs
    if (lane == 0) rhs[j] /= A[j * n + j];
    __syncwarp();
    const double yj = rhs[j];
    for (int i = j + 1 + lane; i < n; i += 32) rhs[i] = fma(-A[i * n + j], yj, rhs[i]);
    __syncwarp();
  }
  for (int j = n - 1; j >= 0; --j) {       // L^T x = y
    if (lane == 0) rhs[j] /= A[j * n + j];
    __syncwarp();
    const double xj = rhs[j];
    for (int i = lane; i < j; i += 32) rhs[i] = fma(-A[j * n + i], xj, rhs[i]);
    __syncwarp();
  }
  for (int j = lane; j < n; j += 32) u[(j / ni + 1) * m + j % ni + 1] = rhs[j];
  __syncwarp();
  if (U)
    for (int t = lane; t < m * m; t += 32) U[int64_t(s) * n_nodes + t] = u[t];
  double acc = 0.0;
  for (int o = lane; o < p.n_obs; o += 32) {
    const int kind = p.route_kind[o];
    double v;
    if (kind == 1) {
      v = route_const(p, o, s);
    } else if (kind == 4) {
      v = u[p.route_col[o]];
    } else {                                // kind 5: mean over the node's cells
      const int c = p.route_col[o];
      const int i0 = c & 31, i1 = (c >> 5) & 31, j0 = (c >> 10) & 31, j1 = (c >> 15) & 31;
      double t = 0.0;
      for (int cy = j0; cy < j1; ++cy)
        for (int cx = i0; cx < i1; ++cx)
          t += 2.0 * u[cy * m + cx] + u[cy * m + cx + 1] + u[(cy + 1) * m + cx] + 2.0 * u[(cy + 1) * m + cx + 1];
      v = t / (6.0 * (i1 - i0) * (j1 - j0));
    }
    if (!isfinite(v)) record_error(p, HDD_ERR_NUMERICAL, s, -1);
    if (S) S[int64_t(s) * p.n_obs + o] = v;
    if (p.y) {
      const double r = (p.y[o] - v) / p.sigma[o];
      acc = fma(r, r, acc);
    }
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0 && ll) ll[s] = p.y ? (-0.5 * acc - p.ll_const) : 0.0;
}

cudaError_t launch_tiny(const DevPlan& p, int B, double* S, double* ll, double* U, int64_t n_nodes, cudaStream_t s) {
  tiny_kernel<<<B, 32, 0, s>>>(p, B, S, ll, U, n_nodes);
  return cudaGetLastError();
}

}  // namespace hdd
