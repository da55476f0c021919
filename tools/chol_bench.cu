// Microbenchmark: warp-register Cholesky latency (lane = row, shuffles) for n = 8, 15, 32,
// plus FP64 / SHFL dependent-chain latencies.  One warp per CTA, clock64 around the loop.
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

template <int NG, int LPN>
__global__ void chol(const double* in, double* out, long long* clk, int reps) {
  const int lane = threadIdx.x & 31, i = lane % LPN;
  double a[NG];
#pragma unroll
  for (int l = 0; l < NG; ++l) a[l] = in[(i * NG + l) % 256];
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      const double dj = __shfl_sync(0xffffffffu, a[j], j, LPN);
      const double il = rsqrt_nr(dj);
      const double lij = a[j] * il;
#pragma unroll
      for (int l = j + 1; l < NG; ++l) a[l] = fma(-lij, __shfl_sync(0xffffffffu, lij, l, LPN), a[l]);
      a[j] = i == j ? il : lij;
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int l = 0; l < NG; ++l) s += a[l];
  out[blockIdx.x * 32 + lane] = s;
  if (lane == 0) clk[blockIdx.x] = (t1 - t0) / reps;
}

__global__ void lat_dfma(double* out, long long* clk, int reps) {
  double x = threadIdx.x * 1e-3, y = 1.0000001;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int u = 0; u < 64; ++u) x = fma(x, y, 1e-9);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) clk[0] = (t1 - t0) / (reps * 64);
}
__global__ void lat_shfl(double* out, long long* clk, int reps) {
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int u = 0; u < 64; ++u) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) clk[0] = (t1 - t0) / (reps * 64);
}
__global__ void lat_rsqrt(double* out, long long* clk, int reps) {
  double x = 1.0 + threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = rsqrt_nr(x) + 1.0;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) clk[0] = (t1 - t0) / (reps * 16);
}

int main() {
  double *in, *out;
  long long* clk;
  cudaMalloc(&in, 256 * 8);
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&clk, 1024 * 8);
  double h[256];
  for (int i = 0; i < 256; ++i) h[i] = (i % 17 == 0) ? 100.0 : 0.01 * (i % 7);
  cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
  long long c[4];
  auto run = [&](const char* name, void (*k)(const double*, double*, long long*, int), int blocks) {
    k<<<blocks, 32>>>(in, out, clk, 20);
    cudaDeviceSynchronize();
    cudaMemcpy(c, clk, 8, cudaMemcpyDeviceToHost);
    printf("%s blocks=%d: %lld cycles per factorization\n", name, blocks, c[0]);
  };
  run("chol8 (LPN 8)", chol<8, 8>, 1);
  run("chol15 (LPN 16)", chol<15, 16>, 1);
  run("chol15 (LPN 16)", chol<15, 16>, 148 * 8);
  run("chol32 (LPN 32)", chol<32, 32>, 1);
  lat_dfma<<<1, 32>>>(out, clk, 100); cudaDeviceSynchronize(); cudaMemcpy(c, clk, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %lld cycles\n", c[0]);
  lat_shfl<<<1, 32>>>(out, clk, 100); cudaDeviceSynchronize(); cudaMemcpy(c, clk, 8, cudaMemcpyDeviceToHost);
  printf("SHFL(double) dependent latency: %lld cycles\n", c[0]);
  lat_rsqrt<<<1, 32>>>(out, clk, 100); cudaDeviceSynchronize(); cudaMemcpy(c, clk, 8, cudaMemcpyDeviceToHost);
  printf("rsqrt_nr + add dependent latency: %lld cycles\n", c[0]);
  return 0;
}
