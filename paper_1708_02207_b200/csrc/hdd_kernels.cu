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
#include <cstdio>

#include "hdd.h"
#include "hdd_device.h"
#include "hdd_plan.h"

namespace hdd {

// ---------------------------------------------------------------------------
// shared helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ void record_error(DevError* e, int code, int sample, long long node) {
  if (atomicCAS(&e->code, 0, code) == 0) {
    e->sample = sample;
    e->node = node;
  }
}

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// K1: coefficient field
// ---------------------------------------------------------------------------
// grid: (ceil(N/128), N, B); block 128. Thread = cell (i = blockIdx.y, j).
__global__ void __launch_bounds__(128) kappa_kernel(DevPlan p, const double* __restrict__ Z, int B,
                                                    double* __restrict__ kappa) {
  extern __shared__ double czx[];   // [n_z][2]: coef_k z_k sx_k(2i), coef_k z_k sx_k(2i+1)
  const int N = p.N, nz = p.n_z;
  const int i = blockIdx.y, s = blockIdx.z;
  const double* z = Z + int64_t(s) * nz;
  for (int k = threadIdx.x; k < nz; k += blockDim.x) {
    double cz = p.coef[k] * z[k];
    czx[2 * k] = cz * p.sx[int64_t(k) * 2 * N + 2 * i];
    czx[2 * k + 1] = cz * p.sx[int64_t(k) * 2 * N + 2 * i + 1];
  }
  __syncthreads();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  double q0 = 0.0, q1 = 0.0;
  const double2* sy2 = reinterpret_cast<const double2*>(p.sy);
  for (int k = 0; k < nz; ++k) {
    double2 t = __ldg(sy2 + int64_t(k) * N + j);
    q0 = fma(czx[2 * k], t.x, q0);
    q1 = fma(czx[2 * k + 1], t.y, q1);
  }
  double2 out = make_double2(exp(q0), exp(q1));
  if (!(out.x > 0.0) || !(out.y > 0.0) || !isfinite(out.x) || !isfinite(out.y))
    record_error(p.err, HDD_ERR_CONFIG, s, -1);
  reinterpret_cast<double2*>(kappa + int64_t(s) * 2 * N * N)[int64_t(i) * N + j] = out;
}

cudaError_t launch_kappa(const DevPlan& p, const double* Z, int B, double* kappa, cudaStream_t s) {
  dim3 grid((p.N + 127) / 128, p.N, B);
  kappa_kernel<<<grid, 128, size_t(2) * p.n_z * sizeof(double), s>>>(p, Z, B, kappa);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K2: leaf condensation
// ---------------------------------------------------------------------------
struct LeafTmplDev {
  int K[8], k[8], ng[8], kson[8], moff[8];
};
__constant__ LeafTmplDev c_tmpl;
__constant__ int16_t c_map[2][256];
__constant__ uint16_t c_orig[512];   // in-leaf node origin (x | y << 8), index 2^r - 1 + q

int upload_leaf_template() {
  const auto& T = leaf_template();
  LeafTmplDev t{};
  int16_t maps[2][256] = {};
  int off = 0;
  for (int r = 0; r < kLeafLevels; ++r) {
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
  if (cudaMemcpyToSymbol(c_tmpl, &t, sizeof(t)) != cudaSuccess) return -1;
  if (cudaMemcpyToSymbol(c_map, maps, sizeof(maps)) != cudaSuccess) return -1;
  if (cudaMemcpyToSymbol(c_orig, orig, sizeof(orig)) != cudaSuccess) return -1;
  return 0;
}

// level-r buffer size (doubles) for nf nodes
__host__ __device__ constexpr int leaf_level_doubles(int nf, int K, int ncl) {
  return nf * (K * (K + ncl) + ncl);
}

static int leaf_buf_doubles(int ncl) {
  const auto& T = leaf_template();
  int mx = 0;
  for (int r = 0; r < kLeafLevels; ++r) {
    int v = leaf_level_doubles(1 << r, T[r].K, ncl);
    mx = v > mx ? v : mx;
  }
  return (mx + 15) / 16 * 16;
}

size_t leaf_smem_bytes(int ncl) {
  // kappa 512 + f 17x17 (pad 296) + maps (2x256 int16 = 128 doubles) + 2 buffers
  return sizeof(double) * (512 + 296 + 128 + 2 * size_t(leaf_buf_doubles(ncl)));
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

template <int NCL>
__global__ void __launch_bounds__(256) leaf_kernel(DevPlan p, int bufd) {
  extern __shared__ __align__(16) double sm[];
  const int leaf = blockIdx.x, s = blockIdx.y;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nthr >> 5;
  const DevLeaf& L = p.leaves[leaf];
  double* kap = sm;                  // [16 x][32 (y, type)]
  double* fl = kap + 512;            // [17 y][17 x]
  int16_t* mp = reinterpret_cast<int16_t*>(fl + 296);   // [2][256]
  double* bufA = fl + 296 + 128;
  double* bufB = bufA + bufd;
  const int N = p.N;
  {
    const double* kb = p.kappa + int64_t(s) * 2 * N * N;
    for (int t = tid; t < 512; t += nthr) {
      int x = t >> 5, r = t & 31;
      kap[t] = kb[2 * (int64_t(L.i0 + x) * N + L.j0) + r];
    }
    for (int t = tid; t < 289; t += nthr) {
      int y = t / 17, x = t % 17;
      fl[t] = p.f ? p.f[int64_t(L.j0 + y) * p.m + L.i0 + x] : 1.0;
    }
    for (int t = tid; t < 512; t += nthr) mp[t] = c_map[t >> 8][t & 255];
  }
  // column coefficients and cell initial values
  const int ncols = L.ncols;
  const double h2_6 = p.h * p.h / 6.0;
  __syncthreads();

  double* in = nullptr;
  double* out = bufA;
  int in_ld = 0, in_K = 0, in_stride = 0;
  for (int r = kLeafLevels - 1; r >= 0; --r) {
    const int K = c_tmpl.K[r], k = c_tmpl.k[r], ng = c_tmpl.ng[r];
    const int nf = 1 << r;
    const int ldo = K + NCL;
    const int stride = K * ldo + NCL;
    const int16_t* m1 = mp + c_tmpl.moff[r];
    const int16_t* m2 = mp + 256 + c_tmpl.moff[r];
    // ---- gather (assemble_father) ----
    const int per = K * ldo;
    for (int idx = tid; idx < nf * per; idx += nthr) {
      const int q = idx / per;
      const int rem = idx - q * per;
      const int a = rem / ldo;
      const int b = rem - a * ldo;
      double v = 0.0;
#pragma unroll
      for (int sn = 0; sn < 2; ++sn) {
        const int pa = sn ? m2[a] : m1[a];
        if (pa < 0) continue;
        const int qs = 2 * q + sn;
        if (r == kLeafLevels - 1) {
          // son = single cell: psi = k0 P1 + k1 P2, loads, mean pattern
          const int o = c_orig[(1 << (r + 1)) - 1 + qs];
          const int cx = o & 255, cy = o >> 8;
          if (b < K) {
            const int pb = sn ? m2[b] : m1[b];
            if (pb < 0) continue;
            const double k0 = kap[cx * 32 + 2 * cy], k1 = kap[cx * 32 + 2 * cy + 1];
            // P1 on (0,1,3), P2 on (0,3,2) with entries +-1/2, 1 (fem.py:126-145)
            const int lo = pa < pb ? pa : pb, hi = pa < pb ? pb : pa;
            double p1 = 0.0, p2 = 0.0;
            if (lo == hi) {
              p1 = (lo == 1) ? 1.0 : ((lo == 0 || lo == 3) ? 0.5 : 0.0);
              p2 = (lo == 2) ? 1.0 : ((lo == 0 || lo == 3) ? 0.5 : 0.0);
            } else {
              p1 = ((lo == 0 && hi == 1) || (lo == 1 && hi == 3)) ? -0.5 : 0.0;
              p2 = ((lo == 0 && hi == 2) || (lo == 2 && hi == 3)) ? -0.5 : 0.0;
            }
            v += fma(k0, p1, k1 * p2);
          } else {
            const int c = b - K;
            if (c >= ncols) continue;
            const int ct = L.ctype[c];
            if (ct == 0) {
              const double w = (pa == 0 || pa == 3) ? (h2_6 + h2_6) : h2_6;
              const int nx = cx + (pa & 1), ny = cy + (pa >> 1);
              v += w * fl[ny * 17 + nx];
            } else if (ct == 1) {
              const double w = (pa == 0 || pa == 3) ? (1.0 / 3.0) : (1.0 / 6.0);
              v += 0.5 * w;
            }
          }
        } else {
          const double* sd = in + qs * in_stride;
          if (b < K) {
            const int pb = sn ? m2[b] : m1[b];
            if (pb < 0) continue;
            v += sd[pa * in_ld + pb];
          } else {
            const int c = b - K;
            if (c >= ncols) continue;
            const double cf = L.ctype[c] == 1 ? 0.5 : 1.0;
            v += cf * sd[pa * in_ld + in_K + c];
          }
        }
      }
      if (b >= K) {
        const int c = b - K;
        if (c < ncols && L.birth_r[c] == r && L.birth_q[c] == q && a == k + L.birth_g[c]) v += 1.0;
      }
      out[q * stride + rem] = v;
    }
    for (int idx = tid; idx < nf * NCL; idx += nthr) {
      const int q = idx / NCL, c = idx - q * NCL;
      double v = 0.0;
      if (r < kLeafLevels - 1 && c < ncols) {
        const double cf = L.ctype[c] == 1 ? 0.5 : 1.0;
        v = cf * in[(2 * q) * in_stride + in_K * in_ld + c] + cf * in[(2 * q + 1) * in_stride + in_K * in_ld + c];
      }
      out[q * stride + K * ldo + c] = v;
    }
    __syncthreads();
    if (ng > 0) {
      // ---- Cholesky of the interface block, one warp per node ----
      for (int q = warp; q < nf; q += nwarp) {
        double* A = out + q * stride;
        for (int c = 0; c < ng; ++c) {
          const double d = A[(k + c) * ldo + k + c];
          if (!(d > 0.0) && lane == 0)
            record_error(p.err, HDD_ERR_NUMERICAL, s, inleaf_ref_id(L.ref_id, r, q));
          const double l = sqrt(d), inv = 1.0 / l;
          __syncwarp();
          for (int rr = c + 1 + lane; rr < ng; rr += 32) A[(k + rr) * ldo + k + c] *= inv;
          if (lane == 0) A[(k + c) * ldo + k + c] = l;
          __syncwarp();
          const int rem = ng - c - 1;
          for (int t = lane; t < rem * rem; t += 32) {
            const int i1 = c + 1 + t / rem, i2 = c + 1 + t % rem;
            if (i2 <= i1) A[(k + i1) * ldo + k + i2] -= A[(k + i1) * ldo + k + c] * A[(k + i2) * ldo + k + c];
          }
          __syncwarp();
        }
      }
      __syncthreads();
      // ---- forward substitution X = L^-1 [A21 | R_gamma], in place ----
      const int wcols = k + NCL;
      for (int idx = tid; idx < nf * wcols; idx += nthr) {
        const int q = idx / wcols, bb = idx - q * wcols;
        const int b = bb < k ? bb : K + (bb - k);
        double* A = out + q * stride;
        for (int g = 0; g < ng; ++g) {
          double x = A[(k + g) * ldo + b];
          for (int hh = 0; hh < g; ++hh) x -= A[(k + g) * ldo + k + hh] * A[(k + hh) * ldo + b];
          A[(k + g) * ldo + b] = x / A[(k + g) * ldo + k + g];
        }
      }
      __syncthreads();
      // ---- Schur update [A11 | R_B] -= X^T X ; sigma += v^T X ----
      const int per2 = k * wcols;
      for (int idx = tid; idx < nf * (per2 + NCL); idx += nthr) {
        const int q = idx / (per2 + NCL);
        const int rem = idx - q * (per2 + NCL);
        double* A = out + q * stride;
        if (rem < per2) {
          const int a = rem / wcols, bb = rem - a * wcols;
          const int b = bb < k ? bb : K + (bb - k);
          double acc = A[a * ldo + b];
          for (int g = 0; g < ng; ++g) acc = fma(-A[(k + g) * ldo + a], A[(k + g) * ldo + b], acc);
          A[a * ldo + b] = acc;
        } else {
          const int c = rem - per2;
          if (c >= 1) {
            double acc = A[K * ldo + c];
            for (int g = 0; g < ng; ++g) acc = fma(A[(k + g) * ldo + K], A[(k + g) * ldo + K + c], acc);
            A[K * ldo + c] = acc;
          }
        }
      }
      __syncthreads();
    }
    in = out;
    in_ld = ldo;
    in_K = K;
    in_stride = stride;
    out = (out == bufA) ? bufB : bufA;
  }
  // ---- write the leaf output: Psi [64][64], R [64][ncl], sigma ----
  const int ld = p.leaf_ld;
  double* dst = p.buf[p.leaf_buf] + int64_t(leaf) * p.leaf_elems * p.bcap + int64_t(s) * p.leaf_elems;
  const int lc = p.leaf_cols;
  for (int idx = tid; idx < kLeafPerim * ld; idx += nthr) {
    const int a = idx / ld, b = idx - a * ld;
    dst[idx] = b < kLeafPerim ? in[a * in_ld + b] : in[a * in_ld + in_K + (b - kLeafPerim)];
  }
  for (int c = tid; c < lc; c += nthr) dst[kLeafPerim * ld + c] = in[in_K * in_ld + c];
}

cudaError_t launch_leaf(const DevPlan& p, int B, cudaStream_t s, size_t* smem_out) {
  const int ncl = p.leaf_cols <= 2 ? 2 : (p.leaf_cols <= 4 ? 4 : 8);
  size_t smem = leaf_smem_bytes(ncl);
  if (smem_out) *smem_out = smem;
  dim3 grid(p.n_leaves, B);
  int bufd = leaf_buf_doubles(ncl);
  cudaError_t e;
  switch (ncl) {
    case 2:
      e = cudaFuncSetAttribute(leaf_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e != cudaSuccess) return e;
      leaf_kernel<2><<<grid, 256, smem, s>>>(p, bufd);
      break;
    case 4:
      e = cudaFuncSetAttribute(leaf_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e != cudaSuccess) return e;
      leaf_kernel<4><<<grid, 256, smem, s>>>(p, bufd);
      break;
    default:
      e = cudaFuncSetAttribute(leaf_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e != cudaSuccess) return e;
      leaf_kernel<8><<<grid, 256, smem, s>>>(p, bufd);
      break;
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K3: upper merge, interface panel in shared memory (tier M)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) merge_m_kernel(DevPlan p, const DevUpper* __restrict__ nodes) {
  extern __shared__ __align__(16) double sm[];
  const DevUpper& U = nodes[blockIdx.y];
  const int s = blockIdx.x;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nthr >> 5;
  const int k = U.k, ng = U.ng, K = U.K, nc = U.nc, ldp = U.ldp;
  const int ngp = (ng + 3) & ~3;
  double* P = sm;                                  // [ngp][ldp]
  double* sig = P + size_t(ngp) * ldp;             // [nc]
  double* ccoef = sig + ((nc + 1) & ~1);           // [nc][2]
  int* gm = reinterpret_cast<int*>(ccoef + 2 * nc); // [2][K]
  int* csrc = gm + 2 * K;                          // [nc][2]
  int* cbirth = csrc + 2 * nc;                     // [nc]
  for (int t = tid; t < 2 * K; t += nthr) gm[t] = p.gmap[U.gmap_off + t];
  for (int t = tid; t < 2 * nc; t += nthr) {
    csrc[t] = p.csrc[2 * U.col_off + t];
    ccoef[t] = p.ccoef[2 * U.col_off + t];
  }
  for (int t = tid; t < nc; t += nthr) cbirth[t] = p.cbirth[U.col_off + t];
  const double* son[2];
#pragma unroll
  for (int sn = 0; sn < 2; ++sn)
    son[sn] = p.buf[U.son_buf[sn]] + U.son_off[sn] * p.bcap + int64_t(s) * U.son_elems[sn];
  const int sk0 = U.son_k[0], sk1 = U.son_k[1], sl0 = U.son_ld[0], sl1 = U.son_ld[1];
  __syncthreads();
  // ---- gather the interface panel [A21 | A22 | R_gamma] ----
  const int W = K + nc;
  for (int g = warp; g < ngp; g += nwarp) {
    double* row = P + size_t(g) * ldp;
    if (g >= ng) {
      for (int b = lane; b < ldp; b += 32) row[b] = 0.0;
      continue;
    }
    const int a = k + g;
    const int pa0 = gm[a], pa1 = gm[K + a];
    const double* r0 = pa0 >= 0 ? son[0] + size_t(pa0) * sl0 : nullptr;
    const double* r1 = pa1 >= 0 ? son[1] + size_t(pa1) * sl1 : nullptr;
    for (int b = lane; b < W; b += 32) {
      double v = 0.0;
      if (b < K) {
        if (r0) { int pb = gm[b]; if (pb >= 0) v += r0[pb]; }
        if (r1) { int pb = gm[K + b]; if (pb >= 0) v += r1[pb]; }
      } else {
        const int c = b - K;
        if (r0 && csrc[2 * c] >= 0) v += ccoef[2 * c] * r0[sk0 + csrc[2 * c]];
        if (r1 && csrc[2 * c + 1] >= 0) v += ccoef[2 * c + 1] * r1[sk1 + csrc[2 * c + 1]];
        if (cbirth[c] == g) v += 1.0;
      }
      row[b] = v;
    }
  }
  for (int c = tid; c < nc; c += nthr) {
    double v = 0.0;
    if (csrc[2 * c] >= 0) v += ccoef[2 * c] * son[0][size_t(sk0) * sl0 + csrc[2 * c]];
    if (csrc[2 * c + 1] >= 0) v += ccoef[2 * c + 1] * son[1][size_t(sk1) * sl1 + csrc[2 * c + 1]];
    sig[c] = v;
  }
  __syncthreads();
  // ---- row-oriented elimination: L = chol(A22), X = L^-1 [A21 | A22 | R] ----
  for (int c = 0; c < ng; ++c) {
    double* rc = P + size_t(c) * ldp;
    const double d = rc[k + c];
    if (!(d > 0.0) && tid == 0) record_error(p.err, HDD_ERR_NUMERICAL, s, U.ref_id);
    const double inv = 1.0 / sqrt(d);
    __syncthreads();
    for (int b = tid; b < W; b += nthr) rc[b] *= inv;
    __syncthreads();
    for (int rr = c + 1 + warp; rr < ng; rr += nwarp) {
      double* rw = P + size_t(rr) * ldp;
      const double lr = rw[k + c] * inv;
      for (int b = lane; b < W; b += 32)
        if (b != k + c) rw[b] = fma(-lr, rc[b], rw[b]);
    }
    __syncthreads();
  }
  // ---- sigma += v^T X (v = load column) ----
  for (int c = 1 + tid; c < nc; c += nthr) {
    double acc = sig[c];
    for (int g = 0; g < ng; ++g) acc = fma(P[size_t(g) * ldp + K], P[size_t(g) * ldp + K + c], acc);
    sig[c] = acc;
  }
  // ---- Schur update out = A~[B, B|cols] - X_B^T X, FP64 DMMA 16x16 warp tiles ----
  double* dst = p.buf[U.buf] + U.out_off * p.bcap + int64_t(s) * U.out_elems;
  const int ow = k + nc;                 // output columns
  const int mt = (k + 15) >> 4, nt = (ow + 15) >> 4;
  const int gq = lane & 3, gr = lane >> 2;
  for (int tile = warp; tile < mt * nt; tile += nwarp) {
    const int a0 = (tile / nt) << 4, b0 = (tile % nt) << 4;
    double acc[2][2][2] = {};
    int acol[2], bcol[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      int a = a0 + 8 * i + gr;
      acol[i] = a < k ? a : 0;
      int b = b0 + 8 * i + gr;
      bcol[i] = b < k ? b : (b < ow ? K + (b - k) : 0);
    }
    for (int g = 0; g < ngp; g += 4) {
      const double* pr = P + size_t(g + gq) * ldp;
      double av[2], bv[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) { av[i] = pr[acol[i]]; bv[i] = pr[bcol[i]]; }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma884(acc[i][j], av[i], bv[j]);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int a = a0 + 8 * i + gr;
      if (a >= k) continue;
      const int pa0 = gm[a], pa1 = gm[K + a];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int b = b0 + 8 * j + 2 * gq + e;
          if (b >= ow) continue;
          double v = 0.0;
          if (b < k) {
            if (pa0 >= 0) { int pb = gm[b]; if (pb >= 0) v += son[0][size_t(pa0) * sl0 + pb]; }
            if (pa1 >= 0) { int pb = gm[K + b]; if (pb >= 0) v += son[1][size_t(pa1) * sl1 + pb]; }
          } else {
            const int c = b - k;
            if (pa0 >= 0 && csrc[2 * c] >= 0) v += ccoef[2 * c] * son[0][size_t(pa0) * sl0 + sk0 + csrc[2 * c]];
            if (pa1 >= 0 && csrc[2 * c + 1] >= 0) v += ccoef[2 * c + 1] * son[1][size_t(pa1) * sl1 + sk1 + csrc[2 * c + 1]];
          }
          dst[size_t(a) * U.out_ld + b] = v - acc[i][j][e];
        }
      }
    }
  }
  __syncthreads();
  for (int c = tid; c < nc; c += nthr) dst[size_t(k) * U.out_ld + c] = sig[c];
}

cudaError_t launch_merge_m(const DevPlan& p, const DevUpper* nodes_dev, int n_nodes, int B, size_t smem,
                           cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(merge_m_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  dim3 grid(B, n_nodes);
  merge_m_kernel<<<grid, 256, smem, s>>>(p, nodes_dev);
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
  double acc = 0.0;
  for (int o = lane; o < p.n_obs; o += 32) {
    const double v = p.route_kind[o] == 0 ? sig[p.route_col[o]] : p.route_val[o];
    if (!isfinite(v)) record_error(p.err, HDD_ERR_NUMERICAL, s, -1);
    if (S) S[int64_t(s) * p.n_obs + o] = v;
    if (p.y) {
      const double r = (p.y[o] - v) / p.sigma[o];
      acc = fma(r, r, acc);
    }
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0 && ll) ll[s] = p.y ? (-0.5 * acc - p.ll_const) : 0.0;
}

cudaError_t launch_finalize(const DevPlan& p, int B, double* S, double* ll, cudaStream_t s) {
  finalize_kernel<<<(B + 7) / 8, 256, 0, s>>>(p, B, S, ll);
  return cudaGetLastError();
}

}  // namespace hdd
