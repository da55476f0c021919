// Do FP64 DMMA and DFMA share one pipe on B200?  Mixed kernel: warps with an even
// id run DMMA chains, odd warps DFMA chains; also a single-warp dependent-chain
// latency probe for DMMA and DFMA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// mode 0: all DMMA, 1: all DFMA, 2: even warps DMMA / odd warps DFMA
__global__ void mix_kernel(double* out, int iters, int mode) {
  const int warp = threadIdx.x >> 5;
  const bool do_mma = mode == 0 || (mode == 2 && (warp & 1) == 0);
  double s = 0;
  if (do_mma) {
    double a = 1e-3 * threadIdx.x, b = 0.5;
    double c[8][2];
#pragma unroll
    for (int k = 0; k < 8; ++k) { c[k][0] = 0; c[k][1] = 0; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < 8; ++k) dmma(c[k][0], c[k][1], a, b);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  } else {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-9 + k;
    const double b = 0.999999, c = 1e-7;
    // same flops per warp as the DMMA branch: 32 DMMA = 8192 FMA per warp-iter = 256 per thread
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < 32; ++u)
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void lat_kernel(long long* out, int n) {
  double d0 = threadIdx.x, d1 = 0, a = 0.5, b = 0.25;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) dmma(d0, d1, a, b);
  long long t1 = clock64();
  double x = d0 + d1;
  for (int i = 0; i < n; ++i) x = fma(x, 0.999, 1e-9);
  long long t2 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; }
  if (x == 12345.0) out[2] = 1;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * 148 * 8 * 1024);
  long long* lo; cudaMalloc(&lo, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[3] = {"dmma", "dfma", "mixed"};
  for (int mode = 0; mode < 3; ++mode)
    for (int threads : {256, 512}) {
      int blocks = sms * (1024 / threads);
      int iters = 2000;
      mix_kernel<<<blocks, threads>>>(out, 100, mode);
      cudaEventRecord(e0);
      mix_kernel<<<blocks, threads>>>(out, iters, mode);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8192 * (double)iters * blocks * (threads / 32);
      printf("{\"bench\":\"%s\",\"threads\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", names[mode], threads, ms, flops / ms / 1e9);
    }
  long long h[2];
  lat_kernel<<<1, 32>>>(lo, 1000);
  cudaMemcpy(h, lo, 16, cudaMemcpyDeviceToHost);
  printf("{\"dmma_dep_latency_clk\":%.1f,\"dfma_dep_latency_clk\":%.1f}\n", h[0] / 1000.0, h[1] / 1000.0);
  printf("{\"err\":\"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
