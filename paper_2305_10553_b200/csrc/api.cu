// Library-wide C-ABI entry points: version, error reporting, device queries.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>

#include "gk_common.cuh"
#include "../../include/gk.h"

namespace gk {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static std::atomic<int64_t> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int& sm_reserve() {
  static thread_local int n = 0;
  return n;
}

int check_launch(const char* what) {
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s launch failed: %s", what, cudaGetErrorString(e));
    return GK_ERR_CUDA;
  }
  return GK_OK;
}

// ---- fp64 throughput probe (roofline denominator; MEASURED_PEAKS.json has none)
__global__ void probe_dfma(double* out, int iters, double a, double b) {
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

__global__ void probe_dmma(double* out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  const double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
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

}  // namespace gk

extern "C" {

int64_t gk_launch_counter(void) { return gk::g_launches.load(); }

int gk_probe_fp64_peak(double* dfma_tflops, double* dmma_tflops) {
  int dev = 0, sms = 0;
  GK_CUDA(cudaGetDevice(&dev));
  GK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* d = nullptr;
  GK_CUDA(cudaMalloc(&d, 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256, reps = 5;
  float ms = 0;
  gk::probe_dfma<<<blocks, threads>>>(d, 64, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) gk::probe_dfma<<<blocks, threads>>>(d, 4096, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  if (dfma_tflops) *dfma_tflops = (double)reps * blocks * threads * 4096.0 * 16.0 / (ms * 1e-3) / 1e12;
  gk::probe_dmma<<<blocks, threads>>>(d, 64);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) gk::probe_dmma<<<blocks, threads>>>(d, 2048);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  if (dmma_tflops) *dmma_tflops = (double)reps * blocks * (threads / 32) * 2048.0 * 8 * 512.0 / (ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  return gk::check_launch("gk_probe_fp64_peak");
}

int gk_version(void) { return GK_ABI_VERSION; }

const char* gk_last_error(void) { return gk::g_err; }

int gk_device_info(int device, int* sm_count, int* cc_major, int* cc_minor, int64_t* l2_bytes) {
  cudaDeviceProp p;
  GK_CUDA(cudaGetDeviceProperties(&p, device));
  if (sm_count) *sm_count = p.multiProcessorCount;
  if (cc_major) *cc_major = p.major;
  if (cc_minor) *cc_minor = p.minor;
  if (l2_bytes) *l2_bytes = p.l2CacheSize;
  return GK_OK;
}

}  // extern "C"
