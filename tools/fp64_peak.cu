// FP64 peak microbenchmarks for the roofline denominators (B200, sm_100a).
//   dfma : independent DFMA chains in registers (CUDA-core FP64 peak)
//   dmma : mma.sync.m8n8k4.f64 chains (FP64 tensor path, DMMA.8x8x4 in SASS)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = 1e-3 * threadIdx.x, b = 0.5;
  double c[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) dmma(c[k][0], c[k][1], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out; cudaMalloc(&out, sizeof(double) * 148 * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) {
    int blocks = sms * (2048 / threads);
    int iters = 4000;
    dfma_kernel<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("{\"bench\":\"dfma\",\"threads\":%d,\"blocks\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", threads, blocks, ms, flops / ms / 1e9);
  }
  for (int threads : {128, 256, 512}) {
    int blocks = sms * (1024 / threads);
    int iters = 2000;
    dmma_kernel<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8 * 4 * (double)iters * blocks * (threads / 32);
    printf("{\"bench\":\"dmma\",\"threads\":%d,\"blocks\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", threads, blocks, ms, flops / ms / 1e9);
  }
  printf("{\"sms\":%d,\"clock_khz\":%d,\"err\":\"%s\"}\n", sms, clk, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
