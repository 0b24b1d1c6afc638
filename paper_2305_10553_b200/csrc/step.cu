// Builder-defined time step: the reference has no step/RHS
// function (its compute API is the five kernels, kernels.py:45-150), so the step
// is the composition of exactly those kernels, in the order the CPU oracle
// (oracle/port.py: step) composes the reference functions:
//   phi = field(h, w); rhs = (stream(h) + nonlinear(h, phi)) + collision(h)
//   h'  = shear(h + dt * rhs, shifts)
// Stream-ordered launches only; all buffers come from the caller's workspace.
#include <algorithm>
#include "gk_common.cuh"
#include "../../include/gk.h"

#include <cstdlib>
#include <map>
#include <memory>

namespace {
int64_t align256(int64_t b) { return (b + 255) & ~int64_t(255); }

// Optional side stream for the collision (GK_STEP_OVERLAP=1): it only needs h, so
// it can run next to the nonlinear FFTs.  That paid with the fp64 DMMA collision
// (DMMA next to DFMA work); the int8 GEMM and the FFT kernels each fill the SMs,
// and serial measured the same or better (34.1 vs 34.3 ms), so serial is the default.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  bool ok = false;
  SideStream() {
    const char* e = getenv("GK_STEP_OVERLAP");
    if (!(e && e[0] == '1')) return;
    ok = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess &&
         cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&join, cudaEventDisableTiming) == cudaSuccess;
  }
};
// Streams and events belong to the device that was current when they were made:
// keep one set per (thread, device).
template <class T>
T& per_device() {
  static thread_local std::map<int, std::unique_ptr<T>> sets;
  int dev = 0;
  cudaGetDevice(&dev);
  auto& p = sets[dev];
  if (!p) p.reset(new T());
  return *p;
}
SideStream& side() { return per_device<SideStream>(); }

// Field stage in theta chunks on a side stream, next to the nonlinear term: the
// bracket of theta planes [t0, t1) needs only their field moment, so the HBM-bound
// field + B-slicing pass of chunk c+1 streams while the FP64-bound FFTs work on
// chunk c.  GK_FIELD_CHUNKS (0 or 1 = off: the field stage runs whole, first).
struct FieldSide {
  static constexpr int kMax = 64;
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, ev[kMax] = {};
  bool ok = false;
  FieldSide() {
    ok = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess &&
         cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; ok && i < kMax; ++i) ok = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming) == cudaSuccess;
  }
};
FieldSide& field_side() { return per_device<FieldSide>(); }
int field_chunks() {
  static const int k = [] {
    const char* e = getenv("GK_FIELD_CHUNKS");
    return e ? std::max(0, std::min(atoi(e), FieldSide::kMax)) : 0;
  }();
  return k;
}
}  // namespace

namespace gk {
bool collision_use_i8(int64_t M, int64_t N, int64_t T);
int64_t collision_i8_bslice_bytes(int64_t M, int64_t T, int64_t N);
int collision_i8_slices(const double* H, int64_t M, int64_t T, int64_t N, int64_t t0, int64_t t1, void* buf,
                        cudaStream_t st, const double* w, double* phi);
int collision_i8_presliced(const double* A, const void* buf, const double* H, double* C, int64_t M, int64_t T,
                           int64_t N, int64_t t0, int64_t t1, cudaStream_t st, void* abuf, bool reuse_a);
int64_t collision_i8_aslice_bytes(int64_t M, int64_t T);
int collision_i8_range(const double* A, const double* H, double* C, int M, int T, int64_t N, int t0, int t1,
                       cudaStream_t st, const double* w, double* phi, void* scratch, bool reuse_a);
int64_t collision_i8_group_scratch_bytes(int64_t M, int64_t T, int64_t N);
void aslices_forget(const void* base, int64_t bytes, const void* keep, int64_t keep_bytes);
}  // namespace gk

namespace {

// With the int8-slice collision, the field stage is one pass that computes the
// field moment and the collision's B slices of every theta (the step workspace
// holds them), so only the GEMMs run on the side stream next to the nonlinear term.
// The step-level slice buffer is capped (GK_STEP_SLICES_MAX_GB, default 8 GB:
// 5.1 GB at sh03b, 28 GB would not fit next to C5a's 4 x 36 GB state buffers);
// above it the collision slices theta group by theta group on its own.
bool step_i8(int64_t n_vel, int64_t n_theta, int64_t cells) {
  if (!gk::collision_use_i8(n_vel, 2 * cells, n_theta)) return false;
  static const double cap = [] {
    const char* e = getenv("GK_STEP_SLICES_MAX_GB");
    return (e ? atof(e) : 8.0) * 1e9;
  }();
  return (double)gk::collision_i8_bslice_bytes(n_vel, n_theta, 2 * cells) <= cap;
}

struct StepBufs {
  double *phi, *coll, *nl, *str, *ws;
  void* bsl;  // int8 B slices of all thetas (int8 collision only)
  void* asl;  // int8 A slices of all thetas (int8 collision only; kept between steps, see gk_step_ex)
  void* grp;  // grouped int8 collision (B slices too big to keep): one group's B slices + all A slices
  bool reuse_a;
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
  b.bsl = nullptr;
  b.grp = nullptr;
  if (step_i8(n_vel, n_theta, cells)) {
    b.bsl = w;
    w += align256(gk::collision_i8_bslice_bytes(n_vel, n_theta, 2 * cells));
    b.asl = w;
    w += align256(gk::collision_i8_aslice_bytes(n_vel, n_theta));
  } else if (gk::collision_use_i8(n_vel, 2 * cells, n_theta)) {
    b.grp = w;
    w += align256(gk::collision_i8_group_scratch_bytes(n_vel, n_theta, 2 * cells));
  }
  b.ws = (double*)w;
  b.ws_bytes = plan ? gk_bracket_workspace_bytes(plan, n_vel * n_theta, n_theta) : 0;
  // this layout owns the workspace: matrix-slice tags another layout left in it
  // are dropped (only this layout's own A-slice area may be reused)
  const int64_t total = (char*)w - (char*)workspace + b.ws_bytes;
  if (b.asl)
    gk::aslices_forget(workspace, total, b.asl, gk::collision_i8_aslice_bytes(n_vel, n_theta));
  else
    gk::aslices_forget(workspace, total, b.grp, b.grp ? gk::collision_i8_group_scratch_bytes(n_vel, n_theta, 2 * cells) : 0);
  return b;
}

int64_t step_bytes(const gk_spectral_plan* plan, int width, int64_t n_vel, int64_t n_theta, int64_t n_ky,
                   int64_t n_kx) {
  const int64_t cells = n_ky * n_kx;
  const int64_t state = n_vel * n_theta * cells * 16;
  int64_t b = align256(n_theta * cells * 16) + 2 * align256(state);
  if (width > 9) b += align256(state);
  if (step_i8(n_vel, n_theta, cells))
    b += align256(gk::collision_i8_bslice_bytes(n_vel, n_theta, 2 * cells)) +
         align256(gk::collision_i8_aslice_bytes(n_vel, n_theta));
  else if (gk::collision_use_i8(n_vel, 2 * cells, n_theta))
    b += align256(gk::collision_i8_group_scratch_bytes(n_vel, n_theta, 2 * cells));
  if (plan) b += align256(gk_bracket_workspace_bytes(plan, n_vel * n_theta, n_theta));
  return b;
}

// field (+ int8 B slices) and collision over thetas [t0, t1)
int field_stage(const StepBufs& b, const double* h, const double* weights, int64_t n_vel, int64_t n_theta,
                int64_t cells, int64_t t0, int64_t t1, void* stream) {
  if (b.bsl)  // one pass: field moment (gk_field's order, same bits) + the collision's B slices
    return gk::collision_i8_slices(h, n_vel, n_theta, 2 * cells, t0, t1, b.bsl, (cudaStream_t)stream, weights,
                                   b.phi);
  return gk_field_range(h, weights, b.phi, n_vel, n_theta, cells, t0, t1, stream);
}
int collision_stage(const StepBufs& b, const double* matrices, const double* h, int64_t n_vel, int64_t n_theta,
                    int64_t cells, int64_t t0, int64_t t1, void* stream) {
  if (b.bsl)
    return gk::collision_i8_presliced(matrices, b.bsl, h, b.coll, n_vel, n_theta, 2 * cells, t0, t1,
                                      (cudaStream_t)stream, b.asl, b.reuse_a);
  if (b.grp)
    return gk::collision_i8_range(matrices, h, b.coll, (int)n_vel, (int)n_theta, 2 * cells, (int)t0, (int)t1,
                                  (cudaStream_t)stream, nullptr, nullptr, b.grp, b.reuse_a);
  return gk_collision_range(matrices, h, b.coll, n_vel, n_theta, cells, t0, t1, stream);
}

// stage: -1 = whole step; 0 field, 1 nonlinear, 2 collision, 3 finish (stream + axpy + shear)
int step_impl(int stage, const gk_spectral_plan* plan, const double* h, const double* weights,
              const double* stencil_host, int width, const double* matrices, const int32_t* shifts, double dt,
              double* h_out, double* phi_out, int64_t n_vel, int64_t n_theta, int64_t n_ky, int64_t n_kx,
              void* workspace, int64_t workspace_bytes, void* stream, int flags = 0) {
  GK_CHECK_ARG(h && weights && stencil_host && matrices && shifts && h_out && workspace, "gk_step: null pointer");
  GK_CHECK_ARG(h != h_out, "gk_step: h_out must not alias h");
  GK_CHECK_ARG(workspace_bytes >= step_bytes(plan, width, n_vel, n_theta, n_ky, n_kx),
               "gk_step: workspace too small");
  const int64_t cells = n_ky * n_kx;
  StepBufs b = carve(plan, width, n_vel, n_theta, n_ky, n_kx, workspace);
  b.reuse_a = (flags & GK_STEP_REUSE_MATRICES) != 0;
  const cudaStream_t st = (cudaStream_t)stream;
  int rc;
  SideStream& ss = side();
  const bool overlap = stage < 0 && ss.ok && plan;
  // the collision runs on the side stream, concurrently with the nonlinear term
  // (and with the field pass too when that pass does not make its B slices)
  auto fork_collision = [&]() -> int {
    GK_CUDA(cudaEventRecord(ss.fork, st));
    GK_CUDA(cudaStreamWaitEvent(ss.s, ss.fork, 0));
    int r = collision_stage(b, matrices, h, n_vel, n_theta, cells, 0, n_theta, ss.s);
    if (r) return r;
    GK_CUDA(cudaEventRecord(ss.join, ss.s));
    return GK_OK;
  };
  if (overlap && !b.bsl && (rc = fork_collision())) return rc;
  const int fk = (int)std::min<int64_t>(field_chunks(), n_theta);
  bool fused_field = false;
  if (stage < 0 && plan && fk > 1 && field_side().ok) {
    // field chunk c on the side stream; the nonlinear range of chunk c waits for it
    FieldSide& fs = field_side();
    GK_CUDA(cudaEventRecord(fs.fork, st));
    GK_CUDA(cudaStreamWaitEvent(fs.s, fs.fork, 0));
    for (int c = 0; c < fk; ++c) {
      const int64_t t0 = c * n_theta / fk, t1 = (c + 1) * n_theta / fk;
      if ((rc = field_stage(b, h, weights, n_vel, n_theta, cells, t0, t1, fs.s))) return rc;
      GK_CUDA(cudaEventRecord(fs.ev[c], fs.s));
    }
    for (int c = 0; c < fk; ++c) {
      const int64_t t0 = c * n_theta / fk, t1 = (c + 1) * n_theta / fk;
      GK_CUDA(cudaStreamWaitEvent(st, fs.ev[c], 0));
      if ((rc = gk_nonlinear_range(plan, h, b.phi, b.nl, n_vel, n_theta, t0, t1, b.ws, b.ws_bytes, stream)))
        return rc;
    }
    if (phi_out) GK_CUDA(cudaMemcpyAsync(phi_out, b.phi, n_theta * cells * 16, cudaMemcpyDeviceToDevice, st));
    if (overlap && b.bsl && (rc = fork_collision())) return rc;
  } else {
  // int8 collision whose B slices do not fit the step workspace (C5a): its
  // group-by-group slicing also writes the field moment (gk_field's bits), so it
  // runs first and the state is read once for both
  fused_field = stage < 0 && !b.bsl && !overlap && gk::collision_use_i8(n_vel, 2 * cells, n_theta);
  if (fused_field) {
    if ((rc = gk::collision_i8_range(matrices, h, b.coll, (int)n_vel, (int)n_theta, 2 * cells, 0, (int)n_theta, st,
                                     weights, b.phi, b.grp, b.reuse_a)))
      return rc;
    if (phi_out) GK_CUDA(cudaMemcpyAsync(phi_out, b.phi, n_theta * cells * 16, cudaMemcpyDeviceToDevice, st));
    if (plan && (rc = gk_nonlinear(plan, h, b.phi, b.nl, n_vel, n_theta, b.ws, b.ws_bytes, stream))) return rc;
  }
  if (!fused_field && (stage < 0 || stage == 0)) {
    if ((rc = field_stage(b, h, weights, n_vel, n_theta, cells, 0, n_theta, stream))) return rc;
    if (phi_out) GK_CUDA(cudaMemcpyAsync(phi_out, b.phi, n_theta * cells * 16, cudaMemcpyDeviceToDevice, st));
  }
  if (overlap && b.bsl && (rc = fork_collision())) return rc;
  if (!fused_field && (stage < 0 || stage == 1) && plan) {
    if ((rc = gk_nonlinear(plan, h, b.phi, b.nl, n_vel, n_theta, b.ws, b.ws_bytes, stream))) return rc;
  }
  }
  if (overlap) {
    GK_CUDA(cudaStreamWaitEvent(st, ss.join, 0));
  } else if (!fused_field && (stage < 0 || stage == 2)) {
    if ((rc = collision_stage(b, matrices, h, n_vel, n_theta, cells, 0, n_theta, stream))) return rc;
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

struct CopyStreams {
  static constexpr int kMax = 64;  // theta chunks
  static constexpr int kVB = 8;    // velocity blocks per chunk
  static constexpr int kBuf = 8;   // device buffers tracked for overlapped calls
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t in[kMax][kVB], out[kMax][kVB], start = nullptr, done = nullptr;
  // overlapped calls (GK_STEP_HOST_OVERLAP): when each device buffer was last
  // released -- h_dev by the compute stream's last read, out_dev by the last D2H
  struct Release {
    const void* p = nullptr;
    cudaEvent_t ev = nullptr;
    bool recorded = false;
  } rel_h[kBuf], rel_out[kBuf];
  int next_h = 0, next_out = 0;
  bool ok = false;
  CopyStreams() {
    ok = cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking) == cudaSuccess &&
         cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking) == cudaSuccess &&
         cudaEventCreateWithFlags(&start, cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&done, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; ok && i < kMax; ++i)
      for (int j = 0; ok && j < kVB; ++j)
        ok = cudaEventCreateWithFlags(&in[i][j], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&out[i][j], cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; ok && i < kBuf; ++i)
      ok = cudaEventCreateWithFlags(&rel_h[i].ev, cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&rel_out[i].ev, cudaEventDisableTiming) == cudaSuccess;
  }
  static Release& slot(Release* r, int& next, const void* p) {
    for (int i = 0; i < kBuf; ++i)
      if (r[i].p == p) return r[i];
    Release& s = r[next];
    next = (next + 1) % kBuf;
    s.p = p;
    s.recorded = false;
    return s;
  }
};
CopyStreams& copies() { return per_device<CopyStreams>(); }

}  // namespace

extern "C" {

// One step from pinned host memory to pinned host memory, pipelined over theta
// chunks: the H2D copy of chunk c+1 (copy engine 1) overlaps field / nonlinear /
// collision on chunk c, and the D2H copy of finished chunks (copy engine 2)
// overlaps both.  Every theta plane's results are computed by the same kernels as
// gk_step (bit-identical).  finish(c) needs the stencil's neighbour planes, so it
// runs once chunk c+1 has arrived; chunk 0 (which wraps to the last planes) last.
int gk_step_host_ex(const gk_spectral_plan* plan, const double* h_host, double* h_dev, double* out_dev,
                    double* out_host, const double* weights, const double* stencil_host, int width,
                    const double* matrices, const int32_t* shifts, double dt, int64_t n_vel, int64_t n_theta,
                    int64_t n_ky, int64_t n_kx, int n_chunks, void* workspace, int64_t workspace_bytes, int flags,
                    void* stream) {
  GK_CHECK_ARG(h_host && h_dev && out_dev && out_host && weights && stencil_host && matrices && shifts &&
                   workspace, "gk_step_host: null pointer");
  GK_CHECK_ARG(h_dev != out_dev, "gk_step_host: out_dev must not alias h_dev");
  GK_CHECK_ARG(width % 2 == 1 && width <= 9 && width <= n_theta, "gk_step_host: stencil width must be odd <= 9");
  GK_CHECK_ARG(workspace_bytes >= step_bytes(plan, width, n_vel, n_theta, n_ky, n_kx),
               "gk_step_host: workspace too small");
  CopyStreams& cp = copies();
  GK_CHECK_ARG(cp.ok, "gk_step_host: could not create copy streams");
  const int half = width / 2;
  int K = n_chunks < 1 ? 1 : n_chunks;
  if (K > CopyStreams::kMax) K = CopyStreams::kMax;
  if (K > n_theta) K = (int)n_theta;
  // velocity blocks: every chunk moves as VB pieces (planes of the chunk x a block
  // of velocity rows).  field / nonlinear / collision need every velocity row of a
  // plane, but the finish (stream + axpy + shear) is elementwise in v, so the finish
  // of chunk c, block b -- and its D2H -- can start as soon as block b of the
  // neighbour planes is in: the pipeline's head and tail shrink from whole chunks
  // to blocks.  GK_E2E_VBLOCKS (default 4, 1..8).
  static const int vb_env = [] {
    const char* e = getenv("GK_E2E_VBLOCKS");
    const int v = e ? atoi(e) : 4;
    return std::max(1, std::min(v, CopyStreams::kVB));
  }();
  const int VB = (int)std::min<int64_t>(vb_env, n_vel);
  int64_t vb[CopyStreams::kVB + 1];
  for (int j = 0; j <= VB; ++j) vb[j] = (int64_t)j * n_vel / VB;
  const int64_t cells = n_ky * n_kx;
  const int64_t pitch = n_theta * cells * 16;
  GK_CHECK_ARG((flags & ~(GK_STEP_REUSE_MATRICES | GK_STEP_HOST_OVERLAP)) == 0, "gk_step_host_ex: unknown flags 0x%x",
               flags);
  StepBufs b = carve(plan, width, n_vel, n_theta, n_ky, n_kx, workspace);
  b.reuse_a = (flags & GK_STEP_REUSE_MATRICES) != 0;
  const bool overlap = (flags & GK_STEP_HOST_OVERLAP) != 0;
  const cudaStream_t st = (cudaStream_t)stream;
  int64_t tb[CopyStreams::kMax + 1];
  for (int c = 0; c <= K; ++c) tb[c] = (int64_t)c * n_theta / K;
  // (plane t, velocity row v) of a [v][t][cells] array
  auto at = [&](const double* base, int64_t t, int64_t v) { return base + (v * n_theta + t) * cells * 2; };
  CopyStreams::Release& rel_h = CopyStreams::slot(cp.rel_h, cp.next_h, h_dev);
  CopyStreams::Release& rel_out = CopyStreams::slot(cp.rel_out, cp.next_out, out_dev);
  if (overlap) {
    // consecutive overlapped calls on alternating device buffers: this call's
    // copy-in starts as soon as h_dev's last reader (an earlier call's finish) is
    // done -- during the previous call's compute and D2H tail -- and its finishes
    // write out_dev once that buffer's last D2H has drained
    if (rel_h.recorded) GK_CUDA(cudaStreamWaitEvent(cp.h2d, rel_h.ev, 0));
    if (rel_out.recorded) GK_CUDA(cudaStreamWaitEvent(st, rel_out.ev, 0));
  } else {
    GK_CUDA(cudaEventRecord(cp.start, st));
    GK_CUDA(cudaStreamWaitEvent(cp.h2d, cp.start, 0));
    GK_CUDA(cudaStreamWaitEvent(cp.d2h, cp.start, 0));
  }
  // H2D order: the last `half` planes first (chunk 0's periodic stencil reaches
  // them), then chunk by chunk, each as VB velocity blocks (event in[c][j] after
  // block j; the stream is in order, so it also covers everything before).
  // Finishing chunk c needs planes [tb[c] - half, tb[c+1] + half) mod T: block j of
  // it is issued as soon as block j of the chunk holding its highest needed plane
  // is in -- chunks may be thinner than the stencil reach.
  int rc0;
  const bool wrap_first = half > 0 && K >= 2 && tb[1] <= n_theta - half;
  const int64_t tail_end = wrap_first ? n_theta - half : n_theta;
  auto h2d = [&](int64_t a, int64_t e, int64_t v0, int64_t v1) -> int {
    if (e > a && v1 > v0)
      GK_CUDA(cudaMemcpy2DAsync((void*)at(h_dev, a, v0), pitch, at(h_host, a, v0), pitch, (e - a) * cells * 16,
                                v1 - v0, cudaMemcpyHostToDevice, cp.h2d));
    return GK_OK;
  };
  // the last chunk lies inside the wrap planes: its data arrives first, so it is
  // computed first and its finish streams with the last chunk to arrive
  const bool wrap_chunk = wrap_first && tb[K - 1] >= tail_end;
  for (int j = 0; wrap_first && j < VB; ++j) {
    if ((rc0 = h2d(tail_end, n_theta, vb[j], vb[j + 1]))) return rc0;
    if (wrap_chunk) GK_CUDA(cudaEventRecord(cp.in[K - 1][j], cp.h2d));
  }
  for (int c = 0; c < K - (wrap_chunk ? 1 : 0); ++c) {
    const int64_t a0 = tb[c], a1 = std::max(a0, std::min(tb[c + 1], tail_end));  // wrap planes are in already
    for (int j = 0; j < VB; ++j) {
      if ((rc0 = h2d(a0, a1, vb[j], vb[j + 1]))) return rc0;
      GK_CUDA(cudaEventRecord(cp.in[c][j], cp.h2d));
    }
  }
  // arrival rank of a chunk's data (the wrap chunk comes first)
  auto arrival = [&](int c) { return (wrap_chunk && c == K - 1) ? -1 : c; };
  // chunk whose block-j event covers everything finish(c, j) reads: of the chunks
  // holding planes [tb[c] - half, tb[c+1] + half) mod T, the last to arrive (the
  // wrap planes arrive first, then chunks in order)
  auto need = [&](int c) -> int {
    if (!wrap_first && half > 0) return K - 1;  // no early wrap copy: everything must be in
    int d = c, rank = arrival(c);
    for (int64_t q = tb[c] - half; q < tb[c + 1] + half; ++q) {
      const int64_t t = ((q % n_theta) + n_theta) % n_theta;
      if (t >= tail_end) continue;  // a wrap plane: in before any chunk
      int e = 0;
      while (tb[e + 1] <= t) ++e;
      if (arrival(e) > rank) rank = arrival(e), d = e;
    }
    return d;
  };
  int rc;
  auto finish = [&](int c, int j) -> int {
    const int d = need(c);
    GK_CUDA(cudaStreamWaitEvent(st, cp.in[d][d == c ? VB - 1 : j], 0));
    const int64_t off = vb[j] * n_theta * cells * 2;
    int r = gk_step_finish_range(h_dev + off, plan ? b.nl + off : nullptr, b.coll + off, stencil_host, width, shifts,
                                 dt, out_dev + off, vb[j + 1] - vb[j], n_theta, n_ky, n_kx, tb[c], tb[c + 1], stream);
    if (r) return r;
    GK_CUDA(cudaEventRecord(cp.out[c][j], st));
    GK_CUDA(cudaStreamWaitEvent(cp.d2h, cp.out[c][j], 0));
    GK_CUDA(cudaMemcpy2DAsync((void*)at(out_host, tb[c], vb[j]), pitch, at(out_dev, tb[c], vb[j]), pitch,
                              (tb[c + 1] - tb[c]) * cells * 16, vb[j + 1] - vb[j], cudaMemcpyDeviceToHost, cp.d2h));
    return GK_OK;
  };
  bool computed[CopyStreams::kMax] = {}, finished[CopyStreams::kMax] = {};
  // finish every computed chunk whose halo arrives no later than chunk `upto`
  // (all of them for upto = K), block-interleaved: block j of each as chunk
  // `upto`'s block j arrives
  auto finish_ready = [&](int upto) -> int {
    int ready[CopyStreams::kMax], n = 0;
    for (int x = 0; x < K; ++x)
      if (computed[x] && !finished[x] && (upto >= K || arrival(need(x)) <= arrival(upto))) ready[n++] = x;
    for (int j = 0; j < VB; ++j)
      for (int i = 0; i < n; ++i)
        if (int r = finish(ready[i], j)) return r;
    for (int i = 0; i < n; ++i) finished[ready[i]] = true;
    return GK_OK;
  };
  for (int i = 0; i < K; ++i) {
    const int c = wrap_chunk ? (i == 0 ? K - 1 : i - 1) : i;  // compute in arrival order
    if ((rc = finish_ready(c))) return rc;  // before computing chunk c: they only wait on copies
    GK_CUDA(cudaStreamWaitEvent(st, cp.in[c][VB - 1], 0));
    if ((rc = field_stage(b, h_dev, weights, n_vel, n_theta, cells, tb[c], tb[c + 1], stream))) return rc;
    if (plan && (rc = gk_nonlinear_range(plan, h_dev, b.phi, b.nl, n_vel, n_theta, tb[c], tb[c + 1], b.ws,
                                         b.ws_bytes, stream)))
      return rc;
    if ((rc = collision_stage(b, matrices, h_dev, n_vel, n_theta, cells, tb[c], tb[c + 1], stream))) return rc;
    computed[c] = true;
  }
  if ((rc = finish_ready(K))) return rc;
  GK_CUDA(cudaEventRecord(cp.done, cp.d2h));
  if (overlap) {  // the caller joins with gk_step_host_join before reading out_host
    GK_CUDA(cudaEventRecord(rel_h.ev, st));
    rel_h.recorded = true;
    GK_CUDA(cudaEventRecord(rel_out.ev, cp.d2h));
    rel_out.recorded = true;
    return GK_OK;
  }
  GK_CUDA(cudaStreamWaitEvent(st, cp.done, 0));  // syncing `stream` covers the last D2H
  return GK_OK;
}

int gk_step_host(const gk_spectral_plan* plan, const double* h_host, double* h_dev, double* out_dev,
                 double* out_host, const double* weights, const double* stencil_host, int width,
                 const double* matrices, const int32_t* shifts, double dt, int64_t n_vel, int64_t n_theta,
                 int64_t n_ky, int64_t n_kx, int n_chunks, void* workspace, int64_t workspace_bytes,
                 void* stream) {
  return gk_step_host_ex(plan, h_host, h_dev, out_dev, out_host, weights, stencil_host, width, matrices, shifts, dt,
                         n_vel, n_theta, n_ky, n_kx, n_chunks, workspace, workspace_bytes, 0, stream);
}

// `stream` waits for the last D2H of the overlapped gk_step_host_ex calls made on
// this device (synchronising it then covers every out_host written so far)
int gk_step_host_join(void* stream) {
  CopyStreams& cp = copies();
  GK_CHECK_ARG(cp.ok, "gk_step_host_join: no copy streams");
  GK_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, cp.done, 0));
  return GK_OK;
}

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

int gk_step_ex(const gk_spectral_plan* plan, const double* h, const double* weights, const double* stencil_host,
               int width, const double* matrices, const int32_t* shifts, double dt, double* h_out, double* phi_out,
               int64_t n_vel, int64_t n_theta, int64_t n_ky, int64_t n_kx, void* workspace, int64_t workspace_bytes,
               int flags, void* stream) {
  GK_CHECK_ARG((flags & ~GK_STEP_REUSE_MATRICES) == 0, "gk_step_ex: unknown flags 0x%x", flags);
  return step_impl(-1, plan, h, weights, stencil_host, width, matrices, shifts, dt, h_out, phi_out, n_vel, n_theta,
                   n_ky, n_kx, workspace, workspace_bytes, stream, flags);
}

// ---- in-place step: the state is updated in place and the workspace holds one
// state-sized buffer (rhs) instead of two (coll, nl) plus the output, so a state
// of up to ~45% of device memory steps on one GPU (em04b: 64 GB state, ~140 GB in
// all, where gk_step needs ~4 states).  Same kernels, one association changed:
//   phi = field(h); rhs = collision(h); rhs += nonlinear(h, phi);
//   rhs = h + dt * (stream(h) + rhs);  h = shear(rhs)
// i.e. h' = shear(h + dt * (stream + (coll + nl))) -- gk_step rounds
// (stream + nl) + coll; the two agree to a few ulps of the rhs.
// workspace: phi | rhs | bracket workspace.  stage: -1 whole, 0 field, 1 coll,
// 2 nonlinear (accumulate), 3 finish (stream + axpy in place, then shear).
static int64_t inplace_bytes(const gk_spectral_plan* plan, int64_t n_vel, int64_t n_theta, int64_t cells) {
  const int64_t state = n_vel * n_theta * cells * 16;
  int64_t b = align256(n_theta * cells * 16) + align256(state);
  if (plan) b += align256(gk_nonlinear_acc_workspace_bytes(plan, n_vel, n_theta));
  if (gk::collision_use_i8(n_vel, 2 * cells, n_theta))
    b += align256(gk::collision_i8_group_scratch_bytes(n_vel, n_theta, 2 * cells));
  return b;
}

int64_t gk_step_inplace_workspace_bytes(const gk_spectral_plan* plan, int64_t n_vel, int64_t n_theta, int64_t n_ky,
                                        int64_t n_kx) {
  return inplace_bytes(plan, n_vel, n_theta, n_ky * n_kx);
}

int gk_step_inplace(int stage, const gk_spectral_plan* plan, double* h, const double* weights,
                    const double* stencil_host, int width, const double* matrices, const int32_t* shifts, double dt,
                    double* phi_out, int64_t n_vel, int64_t n_theta, int64_t n_ky, int64_t n_kx, void* workspace,
                    int64_t workspace_bytes, void* stream) {
  GK_CHECK_ARG(h && weights && stencil_host && matrices && shifts && workspace, "gk_step_inplace: null pointer");
  GK_CHECK_ARG(stage >= -1 && stage <= 3, "gk_step_inplace: stage must be -1..3");
  GK_CHECK_ARG(width % 2 == 1 && width <= 9 && width <= n_theta, "gk_step_inplace: stencil width %d (1..9, odd)",
               width);
  const int64_t cells = n_ky * n_kx;
  GK_CHECK_ARG(workspace_bytes >= inplace_bytes(plan, n_vel, n_theta, cells), "gk_step_inplace: workspace too small");
  char* w = (char*)workspace;
  double* phi = (double*)w;
  w += align256(n_theta * cells * 16);
  double* rhs = (double*)w;
  w += align256(n_vel * n_theta * cells * 16);
  void* bws = w;
  const int64_t bws_bytes = plan ? gk_nonlinear_acc_workspace_bytes(plan, n_vel, n_theta) : 0;
  w += plan ? align256(bws_bytes) : 0;
  void* grp = gk::collision_use_i8(n_vel, 2 * cells, n_theta) ? (void*)w : nullptr;  // grouped int8 scratch
  gk::aslices_forget(workspace, workspace_bytes, nullptr, 0);  // no reuse across in-place steps
  const cudaStream_t st = (cudaStream_t)stream;
  int rc;
  // int8 collision: its group-by-group B slicing also writes the field moment
  // (gk_field's bits), so the whole step reads the state once for both
  const bool fused_field = stage < 0 && gk::collision_use_i8(n_vel, 2 * cells, n_theta);
  if (fused_field) {
    if ((rc = gk::collision_i8_range(matrices, h, rhs, (int)n_vel, (int)n_theta, 2 * cells, 0, (int)n_theta, st,
                                     weights, phi, grp, false)))
      return rc;
    if (phi_out) GK_CUDA(cudaMemcpyAsync(phi_out, phi, n_theta * cells * 16, cudaMemcpyDeviceToDevice, st));
  }
  if (!fused_field && (stage < 0 || stage == 0)) {
    if ((rc = gk_field(h, weights, phi, n_vel, n_theta, cells, stream))) return rc;
    if (phi_out) GK_CUDA(cudaMemcpyAsync(phi_out, phi, n_theta * cells * 16, cudaMemcpyDeviceToDevice, st));
  }
  if (!fused_field && (stage < 0 || stage == 1) &&
      (rc = gk_collision(matrices, h, rhs, n_vel, n_theta, cells, stream)))
    return rc;
  if ((stage < 0 || stage == 2) && plan &&
      (rc = gk_nonlinear_acc(plan, h, phi, rhs, n_vel, n_theta, bws, bws_bytes, stream)))
    return rc;
  if (stage >= 0 && stage != 3) return GK_OK;
  if ((rc = gk_stream_axpy_inplace(h, rhs, stencil_host, width, dt, n_vel, n_theta, cells, stream))) return rc;
  return gk_shear(rhs, shifts, h, n_vel * n_theta, n_ky, n_kx, stream);
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
