// FP64 latency / throughput microbenchmark: W warps per SM, C independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void k(double* out, int iters, double a, double b, long long* cyc) {
  double x[C];
#pragma unroll
  for (int i = 0; i < C; ++i) x[i] = threadIdx.x * 1e-3 + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < C; ++i) x[i] = fma(x[i], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < C; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int C>
void run(int warps_per_sm, int sms, double* d, long long* c) {
  const int iters = 4096;
  k<C><<<sms, warps_per_sm * 32>>>(d, iters, 1.0000001, 1e-9, c);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / iters;                    // cycles per loop iteration
  const double ops_per_clk_sm = warps_per_sm * 32.0 * C / per;  // DFMA lanes per clk per SM
  printf("C=%2d warps/SM=%2d: %.2f clk/iter, %.1f DFMA/clk/SM (peak 64)\n", C, warps_per_sm, per, ops_per_clk_sm);
}
int main() {
  double* d; long long* c;
  cudaMalloc(&d, 8); cudaMalloc(&c, 8);
  run<1>(1, 1, d, c);
  run<2>(1, 1, d, c);
  run<4>(1, 1, d, c);
  run<8>(1, 1, d, c);
  for (int w : {4, 8, 12, 16, 24, 32}) { run<1>(w, 148, d, c); run<2>(w, 148, d, c); run<4>(w, 148, d, c); }
  return 0;
}
