// Device-side plan tables and kernel launchers (internal header).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace hdd {

constexpr int kMaxBuffers = 24;

// One upper (merge) node as the merge kernels see it.
struct DevUpper {
  int k, ng, K, nc;
  int ldp;                 // panel leading dimension
  int nb;                  // elimination block rows (8 or 32); panel rows = ng rounded up to nb
  int stage;               // tier M: stage both sons' outputs in shared memory
  int out_ld;
  int64_t out_elems, out_off;
  int buf;
  int son_buf[2];
  int son_k[2];            // son output rows (= Psi width)
  int son_ld[2];
  int64_t son_elems[2], son_off[2];
  int gmap_off;            // offset into the gmap pool: [2][K]
  int parent;              // upper index of the father, -1 root (primal)
  int cmap_off;            // offset into the cmap pool: [k] father K-index of each boundary node
  int64_t fac_off, u_off;  // per-sample offsets in the factor / interface-solution buffers
  int col_off;             // offset into column pools: csrc/ccoef [nc][2], cbirth [nc]
  int sh[2];               // father indices (< k) of the boundary nodes on BOTH sons (interface ends), -1
  int64_t ref_id;
};

// One kernel leaf.
// leaf columns (load + means + points strictly inside the leaf); the 8-column kernel
// class runs ceil((ncols - 1) / 7) passes of (load + 7 columns) for wider leaves
constexpr int kMaxLeafCols = 64;

struct DevLeaf {
  int i0, j0;
  int ncols;
  int pad;
  int64_t ref_id;
  // per column: coefficient type (0 = load, 1 = mean, 2 = point) and birth
  int ctype[kMaxLeafCols];
  int birth_r[kMaxLeafCols], birth_q[kMaxLeafCols], birth_g[kMaxLeafCols];
  int fslot[kMaxLeafCols]; // primal: functional slot of a point column, -1
  int parent;              // upper index of the father (-1 when the leaf is the root)
};

// Device failure record: key = sample << 33 | (code == NUMERICAL) << 32 | (node + 1),
// ~0 = no failure (reset value).  Reference node ids < 2^31 (level <= 11).
struct DevError {
  unsigned long long key;
};
constexpr unsigned long long kNoError = ~0ull;
__host__ __device__ inline unsigned long long dev_error_key(long long sample, int code, long long node) {
  return (static_cast<unsigned long long>(sample) << 33) | (static_cast<unsigned long long>(code != -1) << 32) |
         static_cast<unsigned long long>((node + 1) & 0xffffffffll);
}
inline void dev_error_decode(unsigned long long key, int* code, long long* sample, long long* node) {
  *sample = static_cast<long long>(key >> 33);
  *code = ((key >> 32) & 1) ? -3 : -1;     // HDD_ERR_NUMERICAL : HDD_ERR_CONFIG
  *node = static_cast<long long>(key & 0xffffffffull) - 1;
}

struct DevPlan {
  int N, m, n_z, n_obs, n_leaves, leaf_cols, leaf_ld;
  int has_submean;         // some leaf column is a mean over a sub-leaf node
  const double* leaf_g;    // [n_leaves][64] Dirichlet values on the domain boundary, NULL = g = 0
  double h;
  int64_t leaf_elems;
  int leaf_buf;
  int bcap;                // allocated sub-batch capacity
  const double* sx;        // [n_z][2N]
  const double* sy;
  const double* coef;
  const double* f;         // nullptr = 1
  const DevLeaf* leaves;
  const int32_t* leaf_order;   // leaf indices grouped by column class (<=2, <=4, <=8)
  int leaf_class_start[3], leaf_class_count[3], leaf_class_passes[3];
  const DevUpper* upper;
  const int32_t* gmap;
  const int32_t* csrc;
  const double* ccoef;
  const int32_t* cbirth;
  const int32_t* route_kind;
  const int32_t* route_col;
  const double* route_val;
  const int32_t* route_node;
  const int32_t* route_slot;
  int mode;                // 0 adjoint, 1 primal
  // low-rank (H-matrix) storage of the boundary maps
  double lr_eps;
  int lr_kmax, lr_l;       // rank cap, sketch width (k_max + 8 <= 32)
  const int32_t* lr_rows;  // position pools
  const int32_t* lr_cols;
  const int32_t* lr_blk;   // [n][5]: node (depth-local), row offset, p, col offset, q
  const double* lr_omega;  // [q_max][32] fixed Gaussian test matrix
  double* lr_scale;        // [max nodes per depth][bcap]  ||Psi||_F^2
  // wide sketch (k_max 25..64): blocks queued by compress_kernel, l = k_max + 8 <= 72
  const double* lr_omega_w;   // [q_max][72]
  int2* lr_wide_list;         // [lr_wide_cap] (depth-local block, sample); NULL when k_max <= 24
  int* lr_wide_n;
  int lr_wide_cap, lr_wide_ctas;
  double* lr_wide_scr;        // [lr_wide_ctas][lr_wide_stride]  Y [p_max][72] | B [72][q_max]
  int64_t lr_wide_stride;
  int lr_pmax, lr_qmax;
  int lr_force_wide;          // test hook (HDD_LR_FORCE_WIDE=1): every block through the wide sketch
  int schur_split;            // tier L: Schur update in schur_l_kernel (TMA-fed GEMM), not in merge_l_kernel
  int64_t fac_elems, u_elems;
  int n_fslots;
  double* fac;             // [bcap][fac_elems]  W | L^T | v rows of every upper node
  double* ubuf;            // [bcap][u_elems]    u_K = [u_B | u_gamma] of every upper node
  double* fbuf;            // [bcap][n_fslots][65] leaf point functionals
  const int32_t* cmap;     // upper cmap pool
  const int32_t* leaf_cmap;   // [n_leaves][64]
  const double* sigma;
  const double* y;         // nullptr = no likelihood
  double ll_const;         // sum log(sigma sqrt(2 pi))
  int root_buf;            // root output: buffer, sample-0 offset, per-sample stride,
  int64_t root_off;        // and the offset of its sigma row inside a sample block
  int64_t root_elems;
  int64_t root_sig;
  double* buf[kMaxBuffers];
  double* kappa;           // [bcap][2 N^2]
  DevError* err;
  int64_t sample0;         // global index of the sub-batch's first sample (error records)
  // meshes below one kernel leaf (levels 1-3): tiny_kernel
  int tiny;
  const double* gfull;     // [m*m] Dirichlet value at every boundary node (interior 0), NULL = g = 0
  long long root_ref;      // reference id of the root (error records)
  // per-call right-hand sides (hdd_forward_batch_ex): f rows with stride f_stride
  // (0 = one row for the batch; f above then points at the call's data), Dirichlet
  // rows gcall [.][4N] with stride g_stride, boundary position of every leaf
  // perimeter node leaf_gpos [n_leaves][64] (-1 off the domain boundary)
  int64_t f_stride;
  const double* gcall;
  int64_t g_stride;
  const int32_t* leaf_gpos;
};

// launchers (hdd_kernels.cu); all return cudaError_t of the launch
cudaError_t launch_kappa(const DevPlan& p, const double* Z, int B, double* kappa, cudaStream_t s);
cudaError_t launch_leaf(const DevPlan& p, int B, cudaStream_t s, size_t* smem_out);
int merge_variant(const DevPlan& p, int n_nodes, int B, int tier, size_t smem, int slot);
const char* merge_variant_name(int v);
cudaError_t launch_merge(const DevPlan& p, const DevUpper* nodes_dev, int n_nodes, int B, double* ws,
                         int64_t ws_stride, int tier, int max_rows, size_t smem, int nb, cudaStream_t s, int slot = -1);
size_t merge_m2_smem_bytes(int ngp, int ldp, int K, int nc);
size_t merge_l_smem_bytes(int K, int nc);
cudaError_t launch_compress(const DevPlan& p, const DevUpper* nodes_dev, int n_nodes, int blk0, int nblk, int B,
                            int pmax, cudaStream_t s);
cudaError_t launch_schur_l(const DevPlan& p, const DevUpper* nodes_dev, const CUtensorMap* tmaps, const int* tiles,
                           int n_nodes, int B, cudaStream_t s);
int schur_l_tiles(int k, int nc, int ngp);   // ngp: padded interface rows
cudaError_t launch_assemble_l(const DevPlan& p, const DevUpper* nodes_dev, int n_nodes, int B, double* ws,
                              int64_t ws_stride, int max_rows, cudaStream_t s);
int schur_l_box_rows();
cudaError_t launch_compress_wide(const DevPlan& p, const DevUpper* nodes_dev, cudaStream_t s);
cudaError_t launch_compress_warp(const DevPlan& p, const DevUpper* nodes_dev, int blk0, int nblk, int B, int pmax,
                                 int qmax, cudaStream_t s);
cudaError_t launch_topdown(const DevPlan& p, const DevUpper* nodes_dev, int n_nodes, int B, int max_ng, cudaStream_t s);
cudaError_t launch_finalize(const DevPlan& p, int B, double* S, double* ll, cudaStream_t s);
cudaError_t launch_posterior(const double* ll, const double* lp, int64_t n, double* w, int64_t* idx, double* lse,
                             cudaStream_t s);
cudaError_t launch_leaf_solve(const DevPlan& p, int B, double* U, int64_t n_nodes, cudaStream_t s,
                              const int32_t* leaf_list = nullptr, int n_list = 0, const int32_t* omega_pos = nullptr);
cudaError_t launch_kappa_check(const DevPlan& p, const double* kappa, int B, cudaStream_t s);
cudaError_t launch_tiny(const DevPlan& p, int B, double* S, double* ll, double* U, int64_t n_nodes, cudaStream_t s);
size_t leaf_smem_bytes(int leaf_cols);
int upload_leaf_template();
int read_leaf_clocks(long long* out);
int read_merge_clocks(long long* out);

}  // namespace hdd
