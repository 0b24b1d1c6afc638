// Library-wide C-ABI entry points: version, error reporting, device queries.
#include <cstdarg>
#include <cstdio>
#include <cstring>

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

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s launch failed: %s", what, cudaGetErrorString(e));
    return GK_ERR_CUDA;
  }
  return GK_OK;
}

}  // namespace gk

extern "C" {

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
