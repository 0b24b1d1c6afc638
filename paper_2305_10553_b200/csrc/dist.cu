// One rank's share of the multi-GPU step (SURVEY.md §8 e; no reference code --
// the reference models this decomposition only analytically, commsim.py:213-219,
// PAPER.md:184-190).  The step is gk_step's composition (step.cu):
//   phi = field(h); h' = shear(h + dt * ((stream(h) + nonlinear(h, phi)) + coll(h)))
// on a toroidal-home shard h[M][T][Y/G][R] of rank r (modes [r Y/G, (r+1) Y/G)).
//
// Local on the home shard: field (a full velocity sum: bitwise G-invariant),
// collision (per cell), stream + axpy + shear (the finish pass).  The bracket
// needs all (ky, kx) of a slice, so velocity rows travel: the home rows are cut
// into K chunks of G * Mk rows, rank q brackets sub-block q of every chunk.
//   fwd(k):    chunk k's home-row blocks to their bracketing ranks -> recv
//              [G src][Mk][T][Y/G][R]   (S/(G K) bytes per chunk)
//   bracket:   the FFT kernels address each toroidal block of their input and
//              output rows through per-block base pointers (no pack / unpack)
//   back(k):   the results home -> nl rows of chunk k, home layout
//   finish(k): stream + axpy + shear of chunk k's rows (elementwise in v)
// and phi's blocks are gathered once.  The rank's own block never travels.
// Two transports:
//  * NCCL (gk_dist_step): fwd/back are all-to-alls issued on the communicator's
//    stream in one fixed order (fwd 0, gather, fwd 1, back 0, fwd 2, back 1, ...),
//    events tie them to the compute stream; 2-deep recv / send / nl rings.
//  * P2P (gk_dist_step_p2p, below): CUDA IPC windows; fwd = copy-engine pushes
//    into the peers' receive rings, back = the x forward transform's own stores
//    into the peers' nl rings; stream-memory-op flags order it on the device.
//
// Every per-element operation is the single-GPU step's (same kernels, same
// orders; the collision picks int8 vs DMMA from the GLOBAL column count), so the
// result is bit-identical to gk_step for any rank count -- checked on one GPU by
// gk_dist_step_sim (G ranks' phases in lock-step, exchanges as device copies) and
// by 2, 4 and 8 processes sharing the GPU over the P2P transport.
#include <cuda.h>
#include <dlfcn.h>

#include <chrono>
#include <thread>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "gk_common.cuh"
#include "comm.cuh"
#include "../../include/gk.h"

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
int nonlinear_fields_blocked(const gk_spectral_plan* p, const double* phi, int64_t n_theta, int64_t n_blocks,
                             void* ws, int64_t ws_bytes, int64_t n_slices, cudaStream_t st);
int nonlinear_slices_blocked(const gk_spectral_plan* p, const double* const* in_base, double* const* out_base,
                             int64_t n_vel, int64_t n_theta, int64_t n_blocks, void* ws, int64_t ws_bytes,
                             cudaStream_t st);
int64_t nonlinear_ws_bytes_sizes(int64_t n_kx, int64_t n_ky, int64_t n_x, int64_t n_y, int64_t n_slices,
                                 int64_t n_theta);
void plan_grid(const gk_spectral_plan* p, int64_t* n_x, int64_t* n_y);
void aslices_forget(const void* base, int64_t bytes, const void* keep, int64_t keep_bytes);
}  // namespace gk

namespace {

int64_t align256(int64_t b) { return (b + 255) & ~int64_t(255); }
constexpr int kMaxRanks = 16;  // toroidal blocks a bracket launch addresses (spectral.cu kMaxLayoutBlocks)

double slices_cap() {
  static const double cap = [] {
    const char* e = getenv("GK_STEP_SLICES_MAX_GB");
    return (e ? atof(e) : 8.0) * 1e9;
  }();
  return cap;
}

struct Geom {
  int G = 1;
  int64_t M, T, Y, Yl, R, cells, row;  // row = complex values per home velocity row (T * Yl * R)
  int64_t K, Mk, chunk_rows, chunk_elems, blk;  // blk = Mk * row (one rank's block of a chunk)
  bool nonlinear, i8, presliced;
  bool p2p = false;  // the P2P transport: the chunk rings and phi blocks live in the IPC window
  Geom(int G_, int64_t M_, int64_t T_, int64_t Y_, int64_t R_, int64_t K_, bool nl)
      : G(G_), M(M_), T(T_), Y(Y_), Yl(Y_ / G_), R(R_), K(K_), nonlinear(nl) {
    cells = Yl * R;
    row = T * cells;
    Mk = nl ? M / (G * K) : M;
    chunk_rows = nl ? (int64_t)G * Mk : M;
    chunk_elems = chunk_rows * row;
    blk = Mk * row;
    // int8 vs DMMA from the global column count (the single-GPU step's choice), so
    // every rank count computes the same bits; the B slices of all thetas are kept
    // (sliced in the field pass) when they fit the cap, else made group by group
    i8 = gk::collision_use_i8(M, 2 * Y * R, T);
    presliced = i8 && (double)gk::collision_i8_bslice_bytes(M, T, 2 * cells) <= slices_cap();
  }
};

struct Bufs {
  double *phi_l, *phi_g, *coll, *recv[2], *send[2], *nl[2];
  void *bsl, *asl, *grp, *bws;
  int64_t bws_bytes, total;
};

// workspace: phi_l | phi_g | coll | recv x2 | send x2 | nl x2 | B slices | A slices | bracket ws
Bufs carve(const Geom& g, int64_t n_x, int64_t n_y, void* base) {
  char* w = (char*)base;
  Bufs b{};
  auto take = [&](int64_t bytes) -> void* {
    void* p = w;
    w += align256(bytes);
    return p;
  };
  b.phi_l = (double*)take(g.T * g.cells * 16);
  b.phi_g = g.nonlinear && !g.p2p ? (double*)take(g.G * g.T * g.cells * 16) : nullptr;
  b.coll = (double*)take(g.M * g.row * 16);
  const bool travel = g.nonlinear && g.G > 1 && !g.p2p;  // recv / send rings (the own block's slot stays unused)
  for (int i = 0; i < 2; ++i) {
    b.recv[i] = travel ? (double*)take(g.chunk_elems * 16) : nullptr;
    b.send[i] = travel ? (double*)take(g.chunk_elems * 16) : nullptr;
    b.nl[i] = g.nonlinear && !g.p2p ? (double*)take(g.chunk_elems * 16) : nullptr;
  }
  b.bsl = g.presliced ? take(gk::collision_i8_bslice_bytes(g.M, g.T, 2 * g.cells)) : nullptr;
  b.asl = g.presliced ? take(gk::collision_i8_aslice_bytes(g.M, g.T)) : nullptr;
  b.grp = (g.i8 && !g.presliced) ? take(gk::collision_i8_group_scratch_bytes(g.M, g.T, 2 * g.cells)) : nullptr;
  b.bws_bytes = g.nonlinear ? gk::nonlinear_ws_bytes_sizes(g.R, g.Y, n_x, n_y, g.Mk * g.T, g.T) : 0;
  b.bws = g.nonlinear ? take(b.bws_bytes) : nullptr;
  b.total = w - (char*)base;
  return b;
}

// One rank's inputs and phases.
struct Rank {
  Geom g;
  Bufs b;
  const gk_spectral_plan* plan;
  const double *h, *weights, *stencil, *matrices;
  const int32_t* shifts;
  int width;
  double dt;
  double *out, *phi_out;
  bool reuse_a;

  // field moment (+ the collision's int8 B slices, or with the grouped int8
  // collision the whole collision: its slicing writes the field moment too)
  int field(cudaStream_t st) const {
    int rc;
    if (b.bsl)
      rc = gk::collision_i8_slices(h, g.M, g.T, 2 * g.cells, 0, g.T, b.bsl, st, weights, b.phi_l);
    else if (g.i8)
      rc = gk::collision_i8_range(matrices, h, b.coll, (int)g.M, (int)g.T, 2 * g.cells, 0, (int)g.T, st, weights,
                                  b.phi_l, b.grp, reuse_a);
    else
      rc = gk_field(h, weights, b.phi_l, g.M, g.T, g.cells, st);
    if (rc == GK_OK && phi_out)
      GK_CUDA(cudaMemcpyAsync(phi_out, b.phi_l, g.T * g.cells * 16, cudaMemcpyDeviceToDevice, st));
    return rc;
  }
  int collision(cudaStream_t st) const {
    if (b.bsl)
      return gk::collision_i8_presliced(matrices, b.bsl, h, b.coll, g.M, g.T, 2 * g.cells, 0, g.T, st, b.asl,
                                        reuse_a);
    if (g.i8) return GK_OK;  // done by field()
    return gk_collision_range(matrices, h, b.coll, g.M, g.T, g.cells, 0, g.T, st);
  }
  int fields(cudaStream_t st) const {
    return gk::nonlinear_fields_blocked(plan, b.phi_g, g.T, g.G, b.bws, b.bws_bytes, g.Mk * g.T, st);
  }
  // chunk k's home rows: the fwd send buffer, and where finish(k) reads and writes
  int64_t chunk_off(int64_t k) const { return k * g.chunk_elems * 2; }  // doubles
  // the rank's own block: read from h, written into the nl ring (no travel)
  int bracket(int64_t k, int self, cudaStream_t st) const {
    const double* in[kMaxRanks];
    double* out_b[kMaxRanks];
    for (int q = 0; q < g.G; ++q) {
      in[q] = q == self ? h + chunk_off(k) + (int64_t)self * g.blk * 2 : b.recv[k & 1] + (int64_t)q * g.blk * 2;
      out_b[q] = q == self ? b.nl[k & 1] + (int64_t)self * g.blk * 2 : b.send[k & 1] + (int64_t)q * g.blk * 2;
    }
    return gk::nonlinear_slices_blocked(plan, in, out_b, g.Mk, g.T, g.G, b.bws, b.bws_bytes, st);
  }
  int finish(int64_t k, cudaStream_t st) const {
    const int64_t o = chunk_off(k);
    return gk_step_finish_range(h + o, g.nonlinear ? b.nl[k & 1] : nullptr, b.coll + o, stencil, width, shifts, dt,
                                out + o, g.chunk_rows, g.T, g.Yl, g.R, 0, g.T, st);
  }
};

int check_args(const Geom& g, int64_t ws_bytes, const Bufs& b, int width) {
  GK_CHECK_ARG(g.G >= 1 && g.G <= kMaxRanks && g.Y % g.G == 0, "gk_dist_step: n_ky %lld not divisible by %d ranks "
               "(at most %d)", (long long)g.Y, g.G, kMaxRanks);
  GK_CHECK_ARG(!g.nonlinear || (g.K >= 1 && g.K <= gk_comm::kMaxChunks && g.M % (g.G * g.K) == 0),
               "gk_dist_step: n_vel %lld not divisible into %d ranks x %lld chunks (<= %d)", (long long)g.M, g.G,
               (long long)g.K, gk_comm::kMaxChunks);
  GK_CHECK_ARG(width % 2 == 1 && width <= 9 && width <= g.T, "gk_dist_step: stencil width %d (odd, <= 9)", width);
  GK_CHECK_ARG(ws_bytes >= b.total, "gk_dist_step: workspace too small (%lld < %lld)", (long long)ws_bytes,
               (long long)b.total);
  return GK_OK;
}

Rank make_rank(const Geom& g, const gk_spectral_plan* plan, const double* h, const double* weights,
               const double* stencil, int width, const double* matrices, const int32_t* shifts, double dt,
               double* out, double* phi_out, void* ws, int flags) {
  int64_t nx, ny;
  gk::plan_grid(plan, &nx, &ny);
  Rank r{g, carve(g, nx, ny, ws), plan, h, weights, stencil, matrices, shifts,
         width, dt, out, phi_out, (flags & GK_STEP_REUSE_MATRICES) != 0};
  // this call's layout owns the workspace: matrix slices another layout left in it
  // are forgotten (only this layout's own A-slice buffer may be reused)
  if (r.b.asl)
    gk::aslices_forget(ws, r.b.total, r.b.asl, gk::collision_i8_aslice_bytes(g.M, g.T));
  else
    gk::aslices_forget(ws, r.b.total, r.b.grp, r.b.grp ? gk::collision_i8_group_scratch_bytes(g.M, g.T, 2 * g.cells) : 0);
  return r;
}

}  // namespace

extern "C" {

int64_t gk_dist_workspace_bytes(int64_t n_x, int64_t n_y, int64_t n_vel, int64_t n_theta, int64_t n_ky,
                                int64_t n_kx, int nranks, int64_t chunks) {
  if (nranks < 1 || n_ky % nranks) return -1;
  const Geom g(nranks, n_vel, n_theta, n_ky, n_kx, chunks, n_x > 0);
  return carve(g, n_x, n_y, nullptr).total;
}

int gk_dist_step(gk_comm* comm, const gk_spectral_plan* plan, const double* h, const double* weights,
                 const double* stencil_host, int width, const double* matrices, const int32_t* shifts, double dt,
                 double* h_out, double* phi_out, int64_t n_vel, int64_t n_theta, int64_t n_ky, int64_t n_kx,
                 int64_t chunks, void* workspace, int64_t workspace_bytes, int flags, void* stream) {
  GK_CHECK_ARG(comm && h && weights && stencil_host && matrices && shifts && h_out && workspace,
               "gk_dist_step: null pointer");
  GK_CHECK_ARG(h != h_out, "gk_dist_step: h_out must not alias h");
  GK_CHECK_ARG((flags & ~GK_STEP_REUSE_MATRICES) == 0, "gk_dist_step: unknown flags 0x%x", flags);
  const Geom g(comm->nranks, n_vel, n_theta, n_ky, n_kx, chunks, plan != nullptr);
  Rank r = make_rank(g, plan, h, weights, stencil_host, width, matrices, shifts, dt, h_out, phi_out, workspace, flags);
  if (int rc = check_args(g, workspace_bytes, r.b, width)) return rc;
  const cudaStream_t st = (cudaStream_t)stream, cs = comm->cs;
  int rc;
  // leave SMs to NCCL while the transposes run next to the persistent kernels
  // (GK_COMM_SMS, default 8 of 148; nothing travels at one rank)
  static const int comm_sms = [] {
    const char* e = getenv("GK_COMM_SMS");
    return e ? std::max(0, atoi(e)) : 8;
  }();
  gk::SmReserve reserve(g.nonlinear && g.G > 1 ? comm_sms : 0);
  if (!g.nonlinear) {  // linear-only: nothing travels
    if ((rc = r.field(st)) || (rc = r.collision(st))) return rc;
    return r.finish(0, st);
  }
  const int64_t K = g.K;
  auto fwd = [&](int64_t k) -> int {  // chunk k of every rank's home rows -> recv[k % 2]
    if ((rc = gk::comm_alltoall(comm, h + r.chunk_off(k), r.b.recv[k & 1], g.blk, cs, true))) return rc;
    GK_CUDA(cudaEventRecord(comm->rf[k], cs));
    return GK_OK;
  };
  GK_CUDA(cudaEventRecord(comm->start, st));
  GK_CUDA(cudaStreamWaitEvent(cs, comm->start, 0));
  if ((rc = fwd(0))) return rc;  // needs only h: overlaps the field pass
  if ((rc = r.field(st))) return rc;
  GK_CUDA(cudaEventRecord(comm->phi, st));
  GK_CUDA(cudaStreamWaitEvent(cs, comm->phi, 0));
  if ((rc = gk::comm_allgather(comm, r.b.phi_l, r.b.phi_g, g.T * g.cells, cs))) return rc;
  GK_CUDA(cudaEventRecord(comm->gathered, cs));
  if (K > 1 && (rc = fwd(1))) return rc;
  if ((rc = r.collision(st))) return rc;  // local, while the exchange runs
  GK_CUDA(cudaStreamWaitEvent(st, comm->gathered, 0));
  if ((rc = r.fields(st))) return rc;
  for (int64_t k = 0; k < K; ++k) {
    GK_CUDA(cudaStreamWaitEvent(st, comm->rf[k], 0));
    if ((rc = r.bracket(k, comm->rank, st))) return rc;  // recv[k % 2] -> send[k % 2]
    GK_CUDA(cudaEventRecord(comm->br[k], st));
    GK_CUDA(cudaStreamWaitEvent(cs, comm->br[k], 0));
    if (k >= 2) GK_CUDA(cudaStreamWaitEvent(cs, comm->fin[k - 2], 0));  // nl[k % 2] read by finish(k - 2)
    if ((rc = gk::comm_alltoall(comm, r.b.send[k & 1], r.b.nl[k & 1], g.blk, cs, true))) return rc;
    GK_CUDA(cudaEventRecord(comm->bk[k], cs));
    if (k + 2 < K && (rc = fwd(k + 2))) return rc;  // recv[k % 2] is free once bracket(k) ran
    if (k >= 1) {
      GK_CUDA(cudaStreamWaitEvent(st, comm->bk[k - 1], 0));
      if ((rc = r.finish(k - 1, st))) return rc;
      GK_CUDA(cudaEventRecord(comm->fin[k - 1], st));
    }
  }
  GK_CUDA(cudaStreamWaitEvent(st, comm->bk[K - 1], 0));
  if ((rc = r.finish(K - 1, st))) return rc;
  GK_CUDA(cudaEventRecord(comm->fin[K - 1], st));
  GK_CUDA(cudaStreamWaitEvent(cs, comm->fin[K - 1], 0));  // the next step's fwd(0) waits for this step
  return GK_OK;
}

// One stage of gk_dist_step on its workspace, for per-stage timing (bench split):
// 0 field, 1 nonlinear (phi all-gather, the pipelined transposes and the
// bracket of every chunk, no finish), 2 collision, 3 finish of every chunk (reads
// whatever the nl ring holds: timing only), 4 the transposes alone (fwd + back of
// every chunk, no compute).  Stream-ordered on `stream`.
int gk_dist_step_stage(int stage, gk_comm* comm, const gk_spectral_plan* plan, const double* h,
                       const double* weights, const double* stencil_host, int width, const double* matrices,
                       const int32_t* shifts, double dt, double* h_out, int64_t n_vel, int64_t n_theta,
                       int64_t n_ky, int64_t n_kx, int64_t chunks, void* workspace, int64_t workspace_bytes,
                       void* stream) {
  GK_CHECK_ARG(comm && h && weights && stencil_host && matrices && shifts && h_out && workspace,
               "gk_dist_step_stage: null pointer");
  GK_CHECK_ARG(stage >= 0 && stage <= 4, "gk_dist_step_stage: stage must be 0..4");
  const Geom g(comm->nranks, n_vel, n_theta, n_ky, n_kx, chunks, plan != nullptr);
  Rank r = make_rank(g, plan, h, weights, stencil_host, width, matrices, shifts, dt, h_out, nullptr, workspace,
                     GK_STEP_REUSE_MATRICES);
  if (int rc = check_args(g, workspace_bytes, r.b, width)) return rc;
  const cudaStream_t st = (cudaStream_t)stream;
  int rc = GK_OK;
  if (stage == 0) return r.field(st);
  if (stage == 2) return r.collision(st);
  if (stage == 3) {
    for (int64_t k = 0; k < (g.nonlinear ? g.K : 1) && rc == GK_OK; ++k) rc = r.finish(k, st);
    return rc;
  }
  if (!g.nonlinear) return GK_OK;
  for (int64_t k = 0; k < g.K && rc == GK_OK; ++k) {  // NCCL on the caller's stream: serial, measurable
    if (stage == 1 && k == 0) {
      if ((rc = gk::comm_allgather(comm, r.b.phi_l, r.b.phi_g, g.T * g.cells, st)) || (rc = r.fields(st))) break;
    }
    if ((rc = gk::comm_alltoall(comm, h + r.chunk_off(k), r.b.recv[k & 1], g.blk, st, true))) break;
    if (stage == 1 && (rc = r.bracket(k, comm->rank, st))) break;
    rc = gk::comm_alltoall(comm, r.b.send[k & 1], r.b.nl[k & 1], g.blk, st, true);
  }
  return rc;
}

// G ranks of gk_dist_step in ONE process on one device (test harness for the
// rank step's layouts and chunk schedule): every rank's phases run in lock-step
// on `stream`, and each exchange is the device copy the all-to-all / all-gather
// would make.  Arrays hold one pointer per rank (host arrays of device pointers).
int gk_dist_step_sim(int nranks, const gk_spectral_plan* plan, const double* const* h, const double* weights,
                     const double* stencil_host, int width, const double* matrices, const int32_t* const* shifts,
                     double dt, double* const* h_out, double* const* phi_out, int64_t n_vel, int64_t n_theta,
                     int64_t n_ky, int64_t n_kx, int64_t chunks, void* const* workspace, int64_t workspace_bytes,
                     void* stream) {
  GK_CHECK_ARG(nranks >= 1 && h && shifts && h_out && workspace && weights && stencil_host && matrices,
               "gk_dist_step_sim: null pointer");
  const Geom g(nranks, n_vel, n_theta, n_ky, n_kx, chunks, plan != nullptr);
  std::vector<Rank> rk;
  for (int q = 0; q < nranks; ++q) {
    GK_CHECK_ARG(h[q] && h_out[q] && shifts[q] && workspace[q], "gk_dist_step_sim: null pointer for rank %d", q);
    rk.push_back(make_rank(g, plan, h[q], weights, stencil_host, width, matrices, shifts[q], dt, h_out[q],
                           phi_out ? phi_out[q] : nullptr, workspace[q], 0));
    if (int rc = check_args(g, workspace_bytes, rk.back().b, width)) return rc;
  }
  const cudaStream_t st = (cudaStream_t)stream;
  int rc;
  auto copy = [&](double* dst, const double* src, int64_t elems) -> int {
    GK_CUDA(cudaMemcpyAsync(dst, src, elems * 16, cudaMemcpyDeviceToDevice, st));
    return GK_OK;
  };
  for (auto& r : rk)
    if ((rc = r.field(st))) return rc;
  if (g.nonlinear)
    for (int r = 0; r < nranks; ++r)
      for (int q = 0; q < nranks; ++q)
        if ((rc = copy(rk[r].b.phi_g + (int64_t)q * g.T * g.cells * 2, rk[q].b.phi_l, g.T * g.cells))) return rc;
  for (auto& r : rk)
    if ((rc = r.collision(st))) return rc;
  if (!g.nonlinear) {
    for (auto& r : rk)
      if ((rc = r.finish(0, st))) return rc;
    return GK_OK;
  }
  for (auto& r : rk)
    if ((rc = r.fields(st))) return rc;
  for (int64_t k = 0; k < g.K; ++k) {
    // fwd: rank r receives block r of chunk k of every rank q's home rows
    // (the own block q == r does not travel: bracket reads / writes it in place)
    for (int r = 0; r < nranks; ++r)
      for (int q = 0; q < nranks; ++q)
        if (q != r && (rc = copy(rk[r].b.recv[k & 1] + (int64_t)q * g.blk * 2,
                                 rk[q].h + rk[q].chunk_off(k) + (int64_t)r * g.blk * 2, g.blk)))
          return rc;
    for (int r = 0; r < nranks; ++r)
      if ((rc = rk[r].bracket(k, r, st))) return rc;
    // back: rank r receives, from every q, q's block r of its bracket output
    for (int r = 0; r < nranks; ++r)
      for (int q = 0; q < nranks; ++q)
        if (q != r && (rc = copy(rk[r].b.nl[k & 1] + (int64_t)q * g.blk * 2,
                                 rk[q].b.send[k & 1] + (int64_t)r * g.blk * 2, g.blk)))
          return rc;
    for (auto& r : rk)
      if ((rc = r.finish(k, st))) return rc;
  }
  return GK_OK;
}

}  // extern "C"

// =====================================================================  P2P transport
// The transposes without a collective library: every rank's exchange window (the
// velocity-chunk receive ring, the nl ring, phi's blocks, flags) is device memory
// exported by CUDA IPC and mapped by every peer.  Per chunk:
//   fwd:  the copy engines push the rank's home-row blocks into the peers' receive
//         rings (cudaMemcpyAsync over NVLink on a copy stream: no SMs), then a
//         stream memory operation writes the arrival flag into the peer's window;
//   back: the bracket's x forward transform stores each toroidal block's rows
//         straight into the owning peer's nl ring (P2P stores from the FFT kernel:
//         the return transpose is fused into the compute, tile by tile);
//   sync: cuStreamWaitValue32 on flags in the own window (arrivals, and "slot
//         free" from the consumers) -- the stream front end waits, no kernel spins,
//         no host round trip.
// Flags hold monotone 32-bit counters (global chunk index c: arrived = c + 1,
// slot freed after consuming c = c + 3, initial "free" = 2), compared wrap-safe.
namespace {

struct Drv {
  CUresult (*wait)(CUstream, CUdeviceptr, cuuint32_t, unsigned) = nullptr;
  CUresult (*write)(CUstream, CUdeviceptr, cuuint32_t, unsigned) = nullptr;
  bool ok = false;
  char why[160] = "";
};
Drv& drv() {
  static Drv d;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libcuda.so.1", RTLD_NOW);
    if (!h) {
      snprintf(d.why, sizeof(d.why), "cannot load libcuda.so.1");
      return;
    }
    d.wait = reinterpret_cast<decltype(d.wait)>(dlsym(h, "cuStreamWaitValue32_v2"));
    d.write = reinterpret_cast<decltype(d.write)>(dlsym(h, "cuStreamWriteValue32_v2"));
    d.ok = d.wait && d.write;
    if (!d.ok) snprintf(d.why, sizeof(d.why), "libcuda.so.1 lacks cuStreamWaitValue32_v2 / cuStreamWriteValue32_v2");
  });
  return d;
}

enum Flag {
  F_RECV_ARRIVED = 0,
  F_NL_ARRIVED = 1,
  F_PHI_ARRIVED = 2,
  F_RECV_FREE = 3,
  F_NL_FREE = 4,
  F_TEST = 5,  // gk_p2p_selftest_*
  F_COUNT = 6
};
constexpr uint32_t kTestMagic = 0x6b500000u;  // | sender rank

// one P2P store per thread into a peer's window (the transport's kernel path)
__global__ void p2p_test_store(uint64_t* dst, uint64_t v) { dst[threadIdx.x] = v + threadIdx.x; }

}  // namespace

struct gk_p2p {
  int G = 1, r = 0, device = 0;
  int64_t M = 0, T = 0, Y = 0, R = 0, K = 1;
  int64_t chunk_elems = 0, blk = 0, phi_elems = 0;  // complex values
  int64_t off_recv = 0, off_nl = 0, off_phi = 0, off_flags = 0, win_bytes = 0;
  char* win = nullptr;
  char* peer[kMaxRanks] = {};
  bool opened[kMaxRanks] = {};
  // one copy stream per peer: the pushes to different peers run on different
  // copy engines at once (a single stream would serialise them)
  cudaStream_t cp[kMaxRanks] = {};
  cudaEvent_t start = nullptr, done[kMaxRanks] = {};
  uint64_t step = 0, chunk_base = 0;
  unsigned wait_flags = CU_STREAM_WAIT_VALUE_GEQ;

  double* recv(int q, uint64_t c) const { return (double*)(peer[q] + off_recv + (c & 1) * chunk_elems * 16); }
  double* nl(int q, uint64_t c) const { return (double*)(peer[q] + off_nl + (c & 1) * chunk_elems * 16); }
  double* phi(int q, uint64_t e) const { return (double*)(peer[q] + off_phi + (e & 1) * G * phi_elems * 16); }
  CUdeviceptr flag(int q, int f, int idx) const {
    return (CUdeviceptr)(peer[q] + off_flags + ((int64_t)f * kMaxRanks + idx) * 4);
  }
};

namespace {
int waitv(const gk_p2p* c, cudaStream_t s, int f, int idx, uint32_t v) {
  const CUresult e = drv().wait((CUstream)s, c->flag(c->r, f, idx), v, c->wait_flags);
  if (e != CUDA_SUCCESS) {
    gk::set_error("cuStreamWaitValue32 failed (%d)", (int)e);
    return GK_ERR_CUDA;
  }
  return GK_OK;
}
int writev(const gk_p2p* c, cudaStream_t s, int q, int f, uint32_t v) {  // flag f, index = this rank, in q's window
  const CUresult e = drv().write((CUstream)s, c->flag(q, f, c->r), v, CU_STREAM_WRITE_VALUE_DEFAULT);
  if (e != CUDA_SUCCESS) {
    gk::set_error("cuStreamWriteValue32 failed (%d)", (int)e);
    return GK_ERR_CUDA;
  }
  return GK_OK;
}
}  // namespace

extern "C" {

int gk_p2p_create(int nranks, int rank, int64_t n_vel, int64_t n_theta, int64_t n_ky, int64_t n_kx, int64_t chunks,
                  gk_p2p** out) {
  GK_CHECK_ARG(out, "gk_p2p_create: null pointer");
  *out = nullptr;
  GK_CHECK_ARG(nranks >= 1 && nranks <= kMaxRanks && rank >= 0 && rank < nranks && n_ky % nranks == 0 &&
                   chunks >= 1 && n_vel % (nranks * chunks) == 0,
               "gk_p2p_create: bad geometry (%d ranks, n_vel %lld, n_ky %lld, %lld chunks)", nranks,
               (long long)n_vel, (long long)n_ky, (long long)chunks);
  GK_CHECK_ARG(drv().ok, "gk_p2p_create: %s", drv().why);
  auto* c = new gk_p2p{};
  c->G = nranks;
  c->r = rank;
  cudaGetDevice(&c->device);
  c->M = n_vel, c->T = n_theta, c->Y = n_ky, c->R = n_kx, c->K = chunks;
  const int64_t cells = n_ky / nranks * n_kx, row = n_theta * cells, Mk = n_vel / (nranks * chunks);
  c->blk = Mk * row;
  c->chunk_elems = nranks * c->blk;
  c->phi_elems = n_theta * cells;
  c->off_recv = 0;
  c->off_nl = align256(2 * c->chunk_elems * 16);
  c->off_phi = c->off_nl + align256(2 * c->chunk_elems * 16);
  c->off_flags = c->off_phi + align256(2 * nranks * c->phi_elems * 16);
  c->win_bytes = c->off_flags + align256((int64_t)F_COUNT * kMaxRanks * 4);
  int flush = 0;
  cudaDeviceGetAttribute(&flush, cudaDevAttrCanFlushRemoteWrites, c->device);
  if (flush) c->wait_flags |= CU_STREAM_WAIT_VALUE_FLUSH;
  bool ok = cudaMalloc(&c->win, c->win_bytes) == cudaSuccess;
  std::vector<uint32_t> init((size_t)F_COUNT * kMaxRanks, 0u);
  for (int i = 0; i < kMaxRanks; ++i) init[F_RECV_FREE * kMaxRanks + i] = init[F_NL_FREE * kMaxRanks + i] = 2u;
  ok = ok && cudaMemcpy(c->win + c->off_flags, init.data(), init.size() * 4, cudaMemcpyHostToDevice) == cudaSuccess;
  ok = ok && cudaEventCreateWithFlags(&c->start, cudaEventDisableTiming) == cudaSuccess;
  for (int q = 0; ok && q < nranks; ++q)
    ok = cudaStreamCreateWithFlags(&c->cp[q], cudaStreamNonBlocking) == cudaSuccess &&
         cudaEventCreateWithFlags(&c->done[q], cudaEventDisableTiming) == cudaSuccess;
  if (!ok) {
    gk::set_error("gk_p2p_create: could not allocate the %lld-byte exchange window", (long long)c->win_bytes);
    gk_p2p_destroy(c);
    return GK_ERR_NOMEM;
  }
  c->peer[rank] = c->win;
  *out = c;
  return GK_OK;
}

int64_t gk_p2p_window_bytes(const gk_p2p* c) { return c ? c->win_bytes : -1; }

// the window's CUDA IPC handle (GK_P2P_HANDLE_BYTES), to be sent to every peer
int gk_p2p_ipc_handle(const gk_p2p* c, void* handle) {
  GK_CHECK_ARG(c && handle, "gk_p2p_ipc_handle: null pointer");
  cudaIpcMemHandle_t h;
  GK_CUDA(cudaIpcGetMemHandle(&h, c->win));
  memcpy(handle, &h, sizeof(h));
  return GK_OK;
}

// handles: nranks consecutive IPC handles (rank order); maps every peer's window
int gk_p2p_connect(gk_p2p* c, const void* handles) {
  GK_CHECK_ARG(c && handles, "gk_p2p_connect: null pointer");
  for (int q = 0; q < c->G; ++q) {
    if (q == c->r) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, (const char*)handles + (size_t)q * sizeof(h), sizeof(h));
    void* p = nullptr;
    GK_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->peer[q] = (char*)p;
    c->opened[q] = true;
  }
  return GK_OK;
}

int gk_p2p_destroy(gk_p2p* c) {
  if (!c) return GK_OK;
  for (int q = 0; q < kMaxRanks; ++q)
    if (c->opened[q]) cudaIpcCloseMemHandle(c->peer[q]);
  if (c->win) cudaFree(c->win);
  if (c->start) cudaEventDestroy(c->start);
  for (int q = 0; q < kMaxRanks; ++q) {
    if (c->done[q]) cudaEventDestroy(c->done[q]);
    if (c->cp[q]) cudaStreamDestroy(c->cp[q]);
  }
  delete c;
  return GK_OK;
}

// Connectivity self-test of a connected window, before any step relies on it: every
// rank sends each peer a token through all three paths the transport uses -- a
// copy-engine push (token 0 of its slot in the peer's receive ring), P2P stores
// from a kernel (tokens 1..31) and a stream memory operation (the F_TEST flag,
// written last on the same stream) -- then (after a host barrier between the two
// calls) polls its own window from the host with a timeout: a transport that
// would leave a step waiting forever on a flag fails here with an error instead.
int gk_p2p_selftest_send(gk_p2p* c) {
  GK_CHECK_ARG(c, "gk_p2p_selftest_send: null pointer");
  for (int q = 0; q < c->G; ++q) {
    if (q == c->r) continue;
    uint64_t* slot = (uint64_t*)(c->peer[q] + c->off_recv) + 32 * c->r;
    uint64_t* src = (uint64_t*)(c->win + c->off_nl) + 32 * q;  // staged in the own window
    const uint64_t tok = ((uint64_t)kTestMagic << 32) | ((uint64_t)c->r << 8);
    p2p_test_store<<<1, 1, 0, c->cp[q]>>>(src, tok);
    GK_CUDA(cudaMemcpyAsync(slot, src, sizeof(tok), cudaMemcpyDeviceToDevice, c->cp[q]));  // copy engine
    p2p_test_store<<<1, 31, 0, c->cp[q]>>>(slot + 1, tok + 1);                             // P2P stores
    int rc = gk::check_launch("gk_p2p_selftest_send");
    if (rc) return rc;
    if ((rc = writev(c, c->cp[q], q, F_TEST, kTestMagic | (uint32_t)c->r))) return rc;
  }
  for (int q = 0; q < c->G; ++q)
    if (q != c->r) GK_CUDA(cudaStreamSynchronize(c->cp[q]));
  return GK_OK;
}

int gk_p2p_selftest_check(gk_p2p* c, int timeout_ms) {
  GK_CHECK_ARG(c, "gk_p2p_selftest_check: null pointer");
  std::vector<uint32_t> f(kMaxRanks);
  std::vector<uint64_t> tok(32);
  const auto t0 = std::chrono::steady_clock::now();
  for (int q = 0; q < c->G; ++q) {
    if (q == c->r) continue;
    for (;;) {
      GK_CUDA(cudaMemcpy(f.data(), c->win + c->off_flags + (int64_t)F_TEST * kMaxRanks * 4, kMaxRanks * 4,
                         cudaMemcpyDeviceToHost));
      if (f[q] == (kTestMagic | (uint32_t)q)) break;
      const auto ms =
          std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
      if (ms > timeout_ms) {
        gk::set_error("gk_p2p_selftest: no flag from rank %d after %d ms (stream memory operations over P2P)", q,
                      timeout_ms);
        return GK_ERR_COMM;
      }
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
    GK_CUDA(cudaMemcpy(tok.data(), (uint64_t*)(c->win + c->off_recv) + 32 * q, 32 * 8, cudaMemcpyDeviceToHost));
    const uint64_t want = ((uint64_t)kTestMagic << 32) | ((uint64_t)q << 8);
    for (int i = 0; i < 32; ++i)
      if (tok[i] != want + (uint64_t)i) {
        gk::set_error("gk_p2p_selftest: token %d from rank %d is %#llx, expected %#llx (%s)", i, q,
                      (unsigned long long)tok[i], (unsigned long long)(want + i),
                      i == 0 ? "copy-engine push" : "P2P store from a kernel");
        return GK_ERR_COMM;
      }
  }
  return GK_OK;
}

int64_t gk_dist_p2p_workspace_bytes(int64_t n_x, int64_t n_y, int64_t n_vel, int64_t n_theta, int64_t n_ky,
                                    int64_t n_kx, int nranks, int64_t chunks) {
  if (nranks < 1 || n_ky % nranks) return -1;
  Geom g(nranks, n_vel, n_theta, n_ky, n_kx, chunks, n_x > 0);
  g.p2p = true;
  return carve(g, n_x, n_y, nullptr).total;
}

// One rank's step over the P2P transport; same composition and bits as gk_step.
int gk_dist_step_p2p(gk_p2p* c, const gk_spectral_plan* plan, const double* h, const double* weights,
                     const double* stencil_host, int width, const double* matrices, const int32_t* shifts,
                     double dt, double* h_out, double* phi_out, int64_t n_vel, int64_t n_theta, int64_t n_ky,
                     int64_t n_kx, void* workspace, int64_t workspace_bytes, int flags, void* stream) {
  GK_CHECK_ARG(c && h && weights && stencil_host && matrices && shifts && h_out && workspace,
               "gk_dist_step_p2p: null pointer");
  GK_CHECK_ARG(h != h_out, "gk_dist_step_p2p: h_out must not alias h");
  GK_CHECK_ARG(n_vel == c->M && n_theta == c->T && n_ky == c->Y && n_kx == c->R,
               "gk_dist_step_p2p: geometry differs from the window's (gk_p2p_create)");
  GK_CHECK_ARG(plan != nullptr, "gk_dist_step_p2p: the P2P transport is for the nonlinear step");
  Geom g(c->G, n_vel, n_theta, n_ky, n_kx, c->K, true);
  g.p2p = true;
  int64_t nx, ny;
  gk::plan_grid(plan, &nx, &ny);
  Rank rk{g, carve(g, nx, ny, workspace), plan, h, weights, stencil_host, matrices, shifts, width, dt, h_out,
          phi_out, (flags & GK_STEP_REUSE_MATRICES) != 0};
  if (rk.b.asl)
    gk::aslices_forget(workspace, rk.b.total, rk.b.asl, gk::collision_i8_aslice_bytes(g.M, g.T));
  else
    gk::aslices_forget(workspace, rk.b.total, rk.b.grp,
                       rk.b.grp ? gk::collision_i8_group_scratch_bytes(g.M, g.T, 2 * g.cells) : 0);
  GK_CHECK_ARG(width % 2 == 1 && width <= 9 && width <= g.T, "gk_dist_step_p2p: stencil width %d (odd, <= 9)", width);
  GK_CHECK_ARG(workspace_bytes >= rk.b.total, "gk_dist_step_p2p: workspace too small (%lld < %lld)",
               (long long)workspace_bytes, (long long)rk.b.total);
  const cudaStream_t st = (cudaStream_t)stream;
  const int G = c->G, me = c->r;
  const uint64_t e = c->step, c0 = c->chunk_base;
  int rc;
  GK_CUDA(cudaEventRecord(c->start, st));
  for (int q = 0; q < G; ++q)
    if (q != me) GK_CUDA(cudaStreamWaitEvent(c->cp[q], c->start, 0));
  // Host issue order matters: an async copy into another process's memory may
  // block the host until its stream reaches it (seen with ranks sharing a device),
  // so a push is issued only after every bracket it waits for (through the peers'
  // "slot free" flags) has been issued here -- the peers issue in the same order.
  auto push = [&](int64_t k) -> int {  // chunk k's home-row blocks into the peers' receive rings
    const uint64_t cc = c0 + k;
    for (int q = 0; q < G; ++q) {
      if (q == me) continue;
      if ((rc = waitv(c, c->cp[q], F_RECV_FREE, q, (uint32_t)(cc + 1)))) return rc;  // q consumed chunk cc - 2
      GK_CUDA(cudaMemcpyAsync(c->recv(q, cc) + (int64_t)me * g.blk * 2, h + rk.chunk_off(k) + (int64_t)q * g.blk * 2,
                              g.blk * 16, cudaMemcpyDeviceToDevice, c->cp[q]));
      if ((rc = writev(c, c->cp[q], q, F_RECV_ARRIVED, (uint32_t)(cc + 1)))) return rc;
    }
    return GK_OK;
  };
  for (int64_t k = 0; k < std::min<int64_t>(2, g.K); ++k)  // the first two need only h
    if ((rc = push(k))) return rc;
  // field moment (+ the collision's B slices), phi's blocks to every rank's window
  if ((rc = rk.field(st))) return rc;
  for (int q = 0; q < G; ++q) {
    GK_CUDA(cudaMemcpyAsync(c->phi(q, e) + (int64_t)me * c->phi_elems * 2, rk.b.phi_l, c->phi_elems * 16,
                            cudaMemcpyDeviceToDevice, st));
    if (q != me && (rc = writev(c, st, q, F_PHI_ARRIVED, (uint32_t)(e + 1)))) return rc;
  }
  if ((rc = rk.collision(st))) return rc;  // local, while the pushes travel
  for (int q = 0; q < G; ++q)
    if (q != me && (rc = waitv(c, st, F_PHI_ARRIVED, q, (uint32_t)(e + 1)))) return rc;
  if ((rc = gk::nonlinear_fields_blocked(plan, c->phi(me, e), g.T, G, rk.b.bws, rk.b.bws_bytes, g.Mk * g.T, st)))
    return rc;
  auto finish = [&](int64_t k) -> int {
    const uint64_t cc = c0 + k;
    for (int q = 0; q < G; ++q)
      if (q != me && (rc = waitv(c, st, F_NL_ARRIVED, q, (uint32_t)(cc + 1)))) return rc;
    const int64_t o = rk.chunk_off(k);
    if ((rc = gk_step_finish_range(h + o, c->nl(me, cc), rk.b.coll + o, stencil_host, width, shifts, dt, h_out + o,
                                   g.chunk_rows, g.T, g.Yl, g.R, 0, g.T, st)))
      return rc;
    for (int q = 0; q < G; ++q)
      if (q != me && (rc = writev(c, st, q, F_NL_FREE, (uint32_t)(cc + 3)))) return rc;
    return GK_OK;
  };
  for (int64_t k = 0; k < g.K; ++k) {
    const uint64_t cc = c0 + k;
    for (int q = 0; q < G; ++q) {
      if (q == me) continue;
      if ((rc = waitv(c, st, F_RECV_ARRIVED, q, (uint32_t)(cc + 1)))) return rc;  // q's block of chunk cc is here
      if ((rc = waitv(c, st, F_NL_FREE, q, (uint32_t)(cc + 1)))) return rc;      // q's nl slot is free
    }
    const double* in[kMaxRanks];
    double* outb[kMaxRanks];
    for (int q = 0; q < G; ++q) {
      in[q] = q == me ? h + rk.chunk_off(k) + (int64_t)me * g.blk * 2 : c->recv(me, cc) + (int64_t)q * g.blk * 2;
      outb[q] = c->nl(q, cc) + (int64_t)me * g.blk * 2;  // block q's rows go home to rank q (P2P stores)
    }
    if ((rc = gk::nonlinear_slices_blocked(plan, in, outb, g.Mk, g.T, G, rk.b.bws, rk.b.bws_bytes, st))) return rc;
    for (int q = 0; q < G; ++q) {
      if (q == me) continue;
      if ((rc = writev(c, st, q, F_NL_ARRIVED, (uint32_t)(cc + 1)))) return rc;
      if ((rc = writev(c, st, q, F_RECV_FREE, (uint32_t)(cc + 3)))) return rc;
    }
    if (k + 2 < g.K && (rc = push(k + 2))) return rc;  // its slot frees when bracket(k) has run everywhere
    if (k >= 1 && (rc = finish(k - 1))) return rc;
  }
  if ((rc = finish(g.K - 1))) return rc;
  for (int q = 0; q < G; ++q) {  // the pushes read h: done before the caller reuses it
    if (q == me) continue;
    GK_CUDA(cudaEventRecord(c->done[q], c->cp[q]));
    GK_CUDA(cudaStreamWaitEvent(st, c->done[q], 0));
  }
  c->step += 1;
  c->chunk_base += (uint64_t)g.K;
  return GK_OK;
}

// One local stage of the P2P rank step for per-stage timing (bench split):
// 0 field, 2 collision, 3 finish of every chunk (reads whatever the window's nl
// ring holds: timing only).  The nonlinear stage with its transposes is the step
// minus these (its transfers are fused into it).
int gk_dist_step_p2p_stage(int stage, gk_p2p* c, const gk_spectral_plan* plan, const double* h,
                           const double* weights, const double* stencil_host, int width, const double* matrices,
                           const int32_t* shifts, double dt, double* h_out, void* workspace, int64_t workspace_bytes,
                           void* stream) {
  GK_CHECK_ARG(c && plan && h && h_out && workspace, "gk_dist_step_p2p_stage: null pointer");
  GK_CHECK_ARG(stage == 0 || stage == 2 || stage == 3, "gk_dist_step_p2p_stage: stage must be 0, 2 or 3");
  Geom g(c->G, c->M, c->T, c->Y, c->R, c->K, true);
  g.p2p = true;
  int64_t nx, ny;
  gk::plan_grid(plan, &nx, &ny);
  Rank rk{g, carve(g, nx, ny, workspace), plan, h, weights, stencil_host, matrices, shifts, width, dt, h_out,
          nullptr, true};
  GK_CHECK_ARG(workspace_bytes >= rk.b.total, "gk_dist_step_p2p_stage: workspace too small");
  const cudaStream_t st = (cudaStream_t)stream;
  if (stage == 0) return rk.field(st);
  if (stage == 2) return rk.collision(st);
  int rc = GK_OK;
  for (int64_t k = 0; k < g.K && rc == GK_OK; ++k) {
    const int64_t o = rk.chunk_off(k);
    rc = gk_step_finish_range(h + o, c->nl(c->r, k), rk.b.coll + o, stencil_host, width, shifts, dt, h_out + o,
                              g.chunk_rows, g.T, g.Yl, g.R, 0, g.T, st);
  }
  return rc;
}

}  // extern "C"
