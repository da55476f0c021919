// Probe: TMA 3-D tile loads of FP64 boxes [rows][8] with the tensor map passed as a
// __grid_constant__ parameter vs read from global memory.  nvcc -arch=sm_100a
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <bool GLOBAL>
__global__ void probe(const __grid_constant__ CUtensorMap tmp, const CUtensorMap* tmg, double* out, int c0, int c1, int c2) {
  __shared__ __align__(128) double box[16 * 8];
  __shared__ __align__(8) uint64_t bar;
  const CUtensorMap* tm = GLOBAL ? tmg : &tmp;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    if (GLOBAL) asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;\n" ::"l"(tm) : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&bar)), "r"(16 * 8 * 8) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
        ::"r"(su32(box)), "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(su32(&bar)) : "memory");
  }
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n"
               ::"r"(su32(&bar)) : "memory");
  for (int t = threadIdx.x; t < 128; t += blockDim.x) out[t] = box[t];
}

int main() {
  const int ld = 40, rows = 32, ns = 3;
  std::vector<double> h(size_t(ld) * rows * ns);
  for (size_t i = 0; i < h.size(); ++i) h[i] = double(i);
  double *d, *o;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&o, 128 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q{};
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  CUtensorMap m;
  const cuuint64_t dims[3] = {cuuint64_t(ld), cuuint64_t(rows), cuuint64_t(ns)};
  const cuuint64_t str[2] = {cuuint64_t(ld) * 8, cuuint64_t(ld) * rows * 8};
  const cuuint32_t box[3] = {8, 16, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", int(r));
  CUtensorMap* gm;
  cudaMalloc(&gm, sizeof(m));
  cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
  for (int g = 0; g < 2; ++g) {
    if (g) probe<true><<<1, 128>>>(m, gm, o, 8, 16, 2);
    else probe<false><<<1, 128>>>(m, gm, o, 8, 16, 2);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> b(128);
    cudaMemcpy(b.data(), o, 128 * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int rr = 0; rr < 16; ++rr)
      for (int c = 0; c < 8; ++c) bad += b[rr * 8 + c] != h[size_t(2) * ld * rows + size_t(16 + rr) * ld + 8 + c];
    printf("%s: %s, mismatches %d\n", g ? "global map" : "param map", cudaGetErrorString(e), bad);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
