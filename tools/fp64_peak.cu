// FP64 throughput probe for the roofline denominator of the fp64-bound kernels
// (MEASURED_PEAKS.json only carries HBM and bf16).  Two paths:
//   DFMA : 8 independent FMA chains per thread, all SMs, many warps
//   DMMA : mma.sync m8n8k4 f64 (the fp64 tensor path used by gk_collision)
// Prints one JSON line: {"dfma_tflops": .., "dmma_tflops": .., "sm_count": .., "clock_mhz": ..}
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = p.multiProcessorCount * 8, threads = 256;
  float ms;
  // DFMA: flops = blocks*threads*iters*8*2
  const int it1 = 4096;
  dfma_kernel<<<blocks, threads>>>(d, 64, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) dfma_kernel<<<blocks, threads>>>(d, it1, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double dfma = 5.0 * blocks * threads * (double)it1 * 16.0 / (ms * 1e-3) / 1e12;
  // DMMA: each mma = 8*8*4 FMA = 512 flop per warp
  const int it2 = 2048;
  dmma_kernel<<<blocks, threads>>>(d, 64);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) dmma_kernel<<<blocks, threads>>>(d, it2);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double dmma = 5.0 * blocks * (threads / 32) * (double)it2 * 8 * 512.0 / (ms * 1e-3) / 1e12;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"sm_count\": %d, \"clock_max_mhz\": %d, \"err\": \"%s\"}\n",
         dfma, dmma, p.multiProcessorCount, clk / 1000, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
