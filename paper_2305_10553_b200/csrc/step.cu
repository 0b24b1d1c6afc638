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

namespace {

struct StepBufs {
  double *phi, *coll, *nl, *str, *ws;
  int64_t ws_bytes;
};

// workspace: phi | coll | nl | [str, only for stencils wider than 9] | bracket workspace
StepBufs carve(const gk_spectral_plan* plan, int width, int64_t n_vel, int64_t n_theta, int64_t n_ky, int64_t n_kx,
               void* workspace) {
  const int64_t cells = n_ky * n_kx;
  const int64_t state = n_vel * n_theta * cells * 16;
  char* w = (char*)workspace;
  StepBufs b{};
  b.phi = (double*)w;
  w += align256(n_theta * cells * 16);
  b.coll = (double*)w;
  w += align256(state);
  b.nl = (double*)w;
  w += align256(state);
  b.str = nullptr;
  if (width > 9) {
    b.str = (double*)w;
    w += align256(state);
  }
  b.ws = (double*)w;
  b.ws_bytes = plan ? gk_bracket_workspace_bytes(plan, n_vel * n_theta, n_theta) : 0;
  return b;
}

int64_t step_bytes(const gk_spectral_plan* plan, int width, int64_t n_vel, int64_t n_theta, int64_t n_ky,
                   int64_t n_kx) {
  const int64_t cells = n_ky * n_kx;
  const int64_t state = n_vel * n_theta * cells * 16;
  int64_t b = align256(n_theta * cells * 16) + 2 * align256(state);
  if (width > 9) b += align256(state);
  if (plan) b += align256(gk_bracket_workspace_bytes(plan, n_vel * n_theta, n_theta));
  return b;
}

// stage: -1 = whole step; 0 field, 1 nonlinear, 2 collision, 3 finish (stream + axpy + shear)
int step_impl(int stage, const gk_spectral_plan* plan, const double* h, const double* weights,
              const double* stencil_host, int width, const double* matrices, const int32_t* shifts, double dt,
              double* h_out, double* phi_out, int64_t n_vel, int64_t n_theta, int64_t n_ky, int64_t n_kx,
              void* workspace, int64_t workspace_bytes, void* stream) {
  GK_CHECK_ARG(h && weights && stencil_host && matrices && shifts && h_out && workspace, "gk_step: null pointer");
  GK_CHECK_ARG(h != h_out, "gk_step: h_out must not alias h");
  GK_CHECK_ARG(workspace_bytes >= step_bytes(plan, width, n_vel, n_theta, n_ky, n_kx),
               "gk_step: workspace too small");
  const int64_t cells = n_ky * n_kx;
  const StepBufs b = carve(plan, width, n_vel, n_theta, n_ky, n_kx, workspace);
  const cudaStream_t st = (cudaStream_t)stream;
  int rc;
  SideStream& ss = side();
  const bool overlap = stage < 0 && ss.ok && plan;
  if (overlap) {  // collision on the side stream, concurrently with field + nonlinear
    GK_CUDA(cudaEventRecord(ss.fork, st));
    GK_CUDA(cudaStreamWaitEvent(ss.s, ss.fork, 0));
    if ((rc = gk_collision(matrices, h, b.coll, n_vel, n_theta, cells, ss.s))) return rc;
    GK_CUDA(cudaEventRecord(ss.join, ss.s));
  }
  if (stage < 0 || stage == 0) {
    if ((rc = gk_field(h, weights, b.phi, n_vel, n_theta, cells, stream))) return rc;
    if (phi_out) GK_CUDA(cudaMemcpyAsync(phi_out, b.phi, n_theta * cells * 16, cudaMemcpyDeviceToDevice, st));
  }
  if ((stage < 0 || stage == 1) && plan) {
    if ((rc = gk_nonlinear(plan, h, b.phi, b.nl, n_vel, n_theta, b.ws, b.ws_bytes, stream))) return rc;
  }
  if (overlap) {
    GK_CUDA(cudaStreamWaitEvent(st, ss.join, 0));
  } else if (stage < 0 || stage == 2) {
    if ((rc = gk_collision(matrices, h, b.coll, n_vel, n_theta, cells, stream))) return rc;
  }
  if (stage >= 0 && stage != 3) return GK_OK;
  if (width <= 9)  // fused stream + axpy + shear: one HBM pass
    return gk_step_finish(h, plan ? b.nl : nullptr, b.coll, stencil_host, width, shifts, dt, h_out, n_vel, n_theta,
                          n_ky, n_kx, stream);
  if ((rc = gk_stream(h, stencil_host, width, GK_STREAM_OPTIMIZED, b.str, n_vel, n_theta, cells, stream))) return rc;
  // coll <- h + dt * ((str + nl) + coll)  (in place on the collision buffer is safe: elementwise)
  if ((rc = gk_axpy3(h, b.str, plan ? b.nl : nullptr, b.coll, dt, b.coll, n_vel * n_theta * cells, stream)))
    return rc;
  return gk_shear(b.coll, shifts, h_out, n_vel * n_theta, n_ky, n_kx, stream);
}

}  // namespace

extern "C" {

int64_t gk_step_workspace_bytes(const gk_spectral_plan* plan, int64_t n_vel, int64_t n_theta, int64_t n_ky,
                                int64_t n_kx) {
  return step_bytes(plan, 31, n_vel, n_theta, n_ky, n_kx);  // any stencil width
}

int64_t gk_step_workspace_bytes_w(const gk_spectral_plan* plan, int width, int64_t n_vel, int64_t n_theta,
                                  int64_t n_ky, int64_t n_kx) {
  return step_bytes(plan, width, n_vel, n_theta, n_ky, n_kx);
}

int gk_step(const gk_spectral_plan* plan, const double* h, const double* weights, const double* stencil_host,
            int width, const double* matrices, const int32_t* shifts, double dt, double* h_out, double* phi_out,
            int64_t n_vel, int64_t n_theta, int64_t n_ky, int64_t n_kx, void* workspace, int64_t workspace_bytes,
            void* stream) {
  return step_impl(-1, plan, h, weights, stencil_host, width, matrices, shifts, dt, h_out, phi_out, n_vel, n_theta,
                   n_ky, n_kx, workspace, workspace_bytes, stream);
}

int gk_step_stage(int stage, const gk_spectral_plan* plan, const double* h, const double* weights,
                  const double* stencil_host, int width, const double* matrices, const int32_t* shifts, double dt,
                  double* h_out, int64_t n_vel, int64_t n_theta, int64_t n_ky, int64_t n_kx, void* workspace,
                  int64_t workspace_bytes, void* stream) {
  GK_CHECK_ARG(stage >= 0 && stage <= 3, "gk_step_stage: stage must be 0..3");
  return step_impl(stage, plan, h, weights, stencil_host, width, matrices, shifts, dt, h_out, nullptr, n_vel,
                   n_theta, n_ky, n_kx, workspace, workspace_bytes, stream);
}

}  // extern "C"
