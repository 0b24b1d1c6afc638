// Shared helpers for the gk (gyrokinetic-proxy) sm_100a kernels.
//
// Complex values are double2 (re, im): torch.complex128 / numpy complex128 storage
// is interleaved, so a state pointer is reinterpreted, never relaid.
//
// All arithmetic that must be bit-reproducible across kernels (the FFT butterflies
// feed the exact-zero self-bracket contract, reference test_spectral.py:234-237 and
// test_kernels.py:218-223) goes through the explicit-rounding intrinsics below, so
// nvcc's FMA contraction can never make two instantiations of the same transform
// round differently.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#define GK_OK 0
#define GK_ERR_ARG 1
#define GK_ERR_CUDA 2
#define GK_ERR_NOMEM 3
#define GK_ERR_COMM 4

namespace gk {

void set_error(const char* fmt, ...);
int check_launch(const char* what);
void count_launch();
// SMs the persistent kernels (FFT x/y passes, the int8 GEMM) leave free on this
// thread's launches: the multi-GPU step reserves some while NCCL transfers run
// next to them (a persistent kernel fills every SM's registers / shared memory, so
// an NCCL kernel launched meanwhile would wait for it to finish).
int& sm_reserve();
struct SmReserve {
  int prev;
  explicit SmReserve(int n) : prev(sm_reserve()) { sm_reserve() = n; }
  ~SmReserve() { sm_reserve() = prev; }
};

__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}
// a * b
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)),
                      __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)));
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(__fma_rn(a.x, b.x, __dmul_rn(a.y, b.y)),
                      __fma_rn(a.y, b.x, -__dmul_rn(a.x, b.y)));
}
__device__ __forceinline__ double2 cscale(double2 a, double s) {
  return make_double2(__dmul_rn(a.x, s), __dmul_rn(a.y, s));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
// -i * a
__device__ __forceinline__ double2 cmul_mi(double2 a) { return make_double2(a.y, -a.x); }
// +i * a
__device__ __forceinline__ double2 cmul_pi(double2 a) { return make_double2(-a.y, a.x); }

__host__ __device__ __forceinline__ int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// True the first time it is called for the current device with this mask (kernel
// attributes such as the dynamic shared-memory limit are per device).
inline bool first_on_device(std::atomic<unsigned long long>& mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  return !(mask.fetch_or(bit) & bit);
}

}  // namespace gk

#define GK_CHECK_ARG(cond, ...)        \
  do {                                 \
    if (!(cond)) {                     \
      gk::set_error(__VA_ARGS__);      \
      return GK_ERR_ARG;               \
    }                                  \
  } while (0)

#define GK_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      gk::set_error("%s failed: %s", #call, cudaGetErrorString(e_));               \
      return GK_ERR_CUDA;                                                          \
    }                                                                              \
  } while (0)
