// Leaf-kernel-shaped warp Cholesky (A22 rows from smem with the padded panel stride,
// act/bad predicates, FSEL, stores back), one warp working while the CTA's other warps
// wait at a barrier — to compare with chol_bench's register-only loop.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double hd = 0.5 * d;
  y = y * fma(-hd * y, y, 1.5);
  y = y * fma(-hd * y, y, 1.5);
  return y;
}

template <int ng, int LPN, int W, int k>
__global__ void chol_smem(long long* clk, double* out, int nwarps_work) {
  __shared__ double pan[ng * W];
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  for (int t = tid; t < ng * W; t += blockDim.x) {
    const int r = t / W, c = t % W - k;
    pan[t] = (c == r) ? 40.0 + r : ((c >= 0 && c < ng) ? 1.0 / (1 + abs(c - r)) : 0.3);
  }
  __syncthreads();
  long long t0 = clock64();
  if (warp < nwarps_work) {
    const int i = lane % LPN;
    const bool act = lane / LPN == 0 && i < ng;
    double* P = pan + k;
    double a[ng];
#pragma unroll
    for (int l = 0; l < ng; ++l) a[l] = (act && l <= i) ? P[i * W + l] : (l == i ? 1.0 : 0.0);
    bool bad = false;
#pragma unroll
    for (int j = 0; j < ng; ++j) {
      const double dj = __shfl_sync(0xffffffffu, a[j], j, LPN);
      bad |= !(dj > 0.0);
      const double il = rsqrt_nr(dj);
      const double lij = a[j] * il;
#pragma unroll
      for (int l = j + 1; l < ng; ++l) a[l] = fma(-lij, __shfl_sync(0xffffffffu, lij, l, LPN), a[l]);
      a[j] = i == j ? il : lij;
    }
    if (act) {
#pragma unroll
      for (int l = 0; l < ng; ++l)
        if (l <= i) P[i * W + l] = a[l];
      if (i == 0 && bad) out[0] = 1.0;
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (tid == 0) clk[blockIdx.x] = t1 - t0;
  if (tid == 0) out[1 + blockIdx.x] = pan[k + 5 * W + 3];
}

int main() {
  long long* clk;
  double* out;
  cudaMalloc(&clk, 4096 * 8);
  cudaMalloc(&out, 8192 * 8);
  long long c[4];
  for (int threads : {32, 256}) {
    chol_smem<15, 16, 84, 64><<<1, threads>>>(clk, out, 1);
    cudaDeviceSynchronize();
    chol_smem<15, 16, 84, 64><<<1, threads>>>(clk, out, 1);
    cudaDeviceSynchronize();
    cudaMemcpy(c, clk, 8, cudaMemcpyDeviceToHost);
    printf("leaf-shaped chol15, %d threads per CTA: %lld cycles\n", threads, c[0]);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
