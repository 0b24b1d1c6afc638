// Output write-pattern probe for the int8 collision epilogue: each CTA writes
// tiles of R rows x W bytes (rows `ld` bytes apart) in the GEMM's tile order,
// vs. plain contiguous streaming writes of the same total.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/write_probe tools/write_probe.cu
#include <cstdio>
#include <cstdint>

__global__ void tiles(double* out, int64_t ld, int ncb, int nib, int T, int64_t N, int64_t tiles_total,
                      int rows, int cols) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t tile = blockIdx.x; tile < tiles_total; tile += gridDim.x) {
    const int ib = (int)(tile % nib);
    const int64_t rest = tile / nib;
    const int cb = (int)(rest % ncb), tt = (int)(rest / ncb);
    double* base = out + (int64_t)tt * N + (int64_t)cb * cols;
    for (int r = warp; r < rows; r += nw) {
      double* row = base + (int64_t)(ib * rows + r) * ld;
      for (int c = lane; c < cols; c += 32) __stcs(row + c, 1.0);
    }
  }
}

__global__ void stream(double* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    __stcs(out + i, 1.0);
}

int main() {
  const int M = 576, T = 32;
  const int64_t N = 46080;
  const int64_t n = (int64_t)M * T * N;
  double* out;
  cudaMalloc(&out, n * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    stream<<<148 * 8, 256>>>(out, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("contiguous: %.2f ms  %.0f GB/s\n", ms, n * 8 / ms / 1e6);
  }
  const int shapes[][2] = {{64, 128}, {64, 256}, {32, 512}, {128, 128}};
  for (auto& sh : shapes) {
    const int rows = sh[0], cols = sh[1];
    const int ncb = (int)(N / cols), nib = M / rows;
    const int64_t tt = (int64_t)T * ncb * nib;
    for (int threads : {256, 1024}) {
      cudaEventRecord(e0);
      tiles<<<148, threads>>>(out, T * N, ncb, nib, T, N, tt, rows, cols);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("tiles %3d rows x %4d B, 148 CTAs x %4d thr: %.2f ms  %.0f GB/s\n", rows, cols * 8, threads, ms,
             n * 8 / ms / 1e6);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
