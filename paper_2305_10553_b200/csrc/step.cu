// Builder-defined time step: the reference has no step/RHS
// function (its compute API is the five kernels, kernels.py:45-150), so the step
// is the composition of exactly those kernels, in the order the CPU oracle
// (oracle/port.py: step) composes the reference functions:
//   phi = field(h, w); rhs = (stream(h) + nonlinear(h, phi)) + collision(h)
//   h'  = shear(h + dt * rhs, shifts)
// Stream-ordered launches only; all buffers come from the caller's workspace.
#include "gk_common.cuh"
#include "../../include/gk.h"

#include <cstdlib>

namespace {
int64_t align256(int64_t b) { return (b + 255) & ~int64_t(255); }

// Side stream for the collision GEMM: it only needs h, so it can run while the
// field reduction and the nonlinear FFTs run on the caller's stream (DMMA work
// next to DFMA/shared-memory work).  GK_STEP_SERIAL=1 disables the overlap.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  bool ok = false;
  SideStream() {
    const char* e = getenv("GK_STEP_SERIAL");
    if (e && e[0] == '1') return;
    ok = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess &&
         cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&join, cudaEventDisableTiming) == cudaSuccess;
  }
};
SideStream& side() {
  static thread_local SideStream ss;
  return ss;
}
}  // namespace

extern "C" {

int64_t gk_step_workspace_bytes(const gk_spectral_plan* plan, int64_t n_vel, int64_t n_theta,
                                int64_t n_ky, int64_t n_kx) {
  const int64_t cells = n_ky * n_kx;
  const int64_t state = n_vel * n_theta * cells * 16;
  int64_t b = align256(n_theta * cells * 16);  // phi
  b += 3 * align256(state);                    // stream, collision (reused as h + dt rhs), nonlinear
  if (plan) b += align256(gk_bracket_workspace_bytes(plan, n_vel * n_theta, n_theta));
  return b;
}

int gk_step(const gk_spectral_plan* plan, const double* h, const double* weights,
            const double* stencil_host, int width, const double* matrices, const int32_t* shifts,
            double dt, double* h_out, double* phi_out, int64_t n_vel, int64_t n_theta, int64_t n_ky,
            int64_t n_kx, void* workspace, int64_t workspace_bytes, void* stream) {
  GK_CHECK_ARG(h && weights && stencil_host && matrices && shifts && h_out && workspace,
               "gk_step: null pointer");
  GK_CHECK_ARG(h != h_out, "gk_step: h_out must not alias h");
  GK_CHECK_ARG(workspace_bytes >= gk_step_workspace_bytes(plan, n_vel, n_theta, n_ky, n_kx),
               "gk_step: workspace too small");
  const int64_t cells = n_ky * n_kx;
  const int64_t state = n_vel * n_theta * cells * 16;
  char* w = (char*)workspace;
  double* phi = (double*)w;
  w += align256(n_theta * cells * 16);
  double* str = (double*)w;
  w += align256(state);
  double* coll = (double*)w;
  w += align256(state);
  double* nl = (double*)w;
  w += align256(state);
  int rc;
  SideStream& ss = side();
  const bool overlap = ss.ok && plan;
  if (overlap) {  // collision on the side stream, concurrently with field + nonlinear
    GK_CUDA(cudaEventRecord(ss.fork, (cudaStream_t)stream));
    GK_CUDA(cudaStreamWaitEvent(ss.s, ss.fork, 0));
    if ((rc = gk_collision(matrices, h, coll, n_vel, n_theta, cells, ss.s))) return rc;
    GK_CUDA(cudaEventRecord(ss.join, ss.s));
  }
  if ((rc = gk_field(h, weights, phi, n_vel, n_theta, cells, stream))) return rc;
  if (phi_out) GK_CUDA(cudaMemcpyAsync(phi_out, phi, n_theta * cells * 16, cudaMemcpyDeviceToDevice,
                                       (cudaStream_t)stream));
  if (plan) {
    const int64_t wsb = gk_bracket_workspace_bytes(plan, n_vel * n_theta, n_theta);
    if ((rc = gk_nonlinear(plan, h, phi, nl, n_vel, n_theta, w, wsb, stream))) return rc;
  }
  if (overlap) {
    GK_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, ss.join, 0));
  } else if ((rc = gk_collision(matrices, h, coll, n_vel, n_theta, cells, stream))) {
    return rc;
  }
  if (width <= 9)  // fused stream + axpy + shear: one HBM pass
    return gk_step_finish(h, plan ? nl : nullptr, coll, stencil_host, width, shifts, dt, h_out, n_vel, n_theta,
                          n_ky, n_kx, stream);
  if ((rc = gk_stream(h, stencil_host, width, GK_STREAM_OPTIMIZED, str, n_vel, n_theta, cells, stream)))
    return rc;
  // coll <- h + dt * ((str + nl) + coll)  (in place on the collision buffer is safe: elementwise)
  if ((rc = gk_axpy3(h, str, plan ? nl : nullptr, coll, dt, coll, n_vel * n_theta * cells, stream)))
    return rc;
  return gk_shear(coll, shifts, h_out, n_vel * n_theta, n_ky, n_kx, stream);
}

}  // extern "C"
