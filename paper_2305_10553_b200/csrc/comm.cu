// NCCL behind the C-ABI (SURVEY.md §8 b/e): the communicator, the two transposes
// around the nonlinear term and the field all-gather of the multi-GPU step.
// No reference code: the reference only models this exchange analytically
// (commsim.py:213-219 alltoall_volume, PAPER.md:184-190 the 2-D decomposition).
//
// NCCL is loaded at run time (dlopen) so libgk.so has no link-time dependency on
// it: the copy torch already loaded (its bundled libnccl.so.2) is reused when
// present, else GK_NCCL_LIB, else the system libnccl.so.2.  nccl.h provides the
// types only.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "gk_common.cuh"
#include "comm.cuh"
#include "../../include/gk.h"

namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
  ncclResult_t (*GetVersion)(int*);
  bool ok = false;
  char why[256] = "";
};

template <class F>
bool sym(void* h, const char* name, F& f) {
  f = reinterpret_cast<F>(dlsym(h, name));
  return f != nullptr;
}

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's copy, if loaded
    const char* env = getenv("GK_NCCL_LIB");
    if (!h && env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      snprintf(api.why, sizeof(api.why), "cannot load libnccl.so.2: %s", dlerror());
      return;
    }
    api.ok = sym(h, "ncclGetUniqueId", api.GetUniqueId) && sym(h, "ncclCommInitRank", api.CommInitRank) &&
             sym(h, "ncclCommDestroy", api.CommDestroy) && sym(h, "ncclSend", api.Send) &&
             sym(h, "ncclRecv", api.Recv) && sym(h, "ncclGroupStart", api.GroupStart) &&
             sym(h, "ncclGroupEnd", api.GroupEnd) && sym(h, "ncclAllGather", api.AllGather) &&
             sym(h, "ncclGetErrorString", api.GetErrorString) && sym(h, "ncclGetVersion", api.GetVersion);
    if (!api.ok) snprintf(api.why, sizeof(api.why), "libnccl.so.2 lacks a required symbol");
  });
  return api;
}

}  // namespace

#define GK_NCCL(call)                                                                        \
  do {                                                                                       \
    ncclResult_t r_ = (call);                                                                \
    if (r_ != ncclSuccess) {                                                                 \
      gk::set_error("%s failed: %s", #call, nccl().GetErrorString(r_));                      \
      return GK_ERR_COMM;                                                                    \
    }                                                                                        \
  } while (0)

namespace gk {
// block all-to-all: block q of `send` (block_elems complex values at q *
// block_elems) goes to rank q, rank q's block lands at q * block_elems of `recv`
// skip_self: the rank's own block stays put (the caller reads / writes it in place)
int comm_alltoall(gk_comm* c, const double* send, double* recv, int64_t block_elems, cudaStream_t st,
                  bool skip_self) {
  NcclApi& api = nccl();
  const size_t n = (size_t)block_elems * 2;  // doubles
  if (skip_self && c->nranks == 1) return GK_OK;
  GK_NCCL(api.GroupStart());
  for (int q = 0; q < c->nranks; ++q) {
    if (skip_self && q == c->rank) continue;
    GK_NCCL(api.Send(send + (size_t)q * n, n, ncclFloat64, q, c->nc, st));
    GK_NCCL(api.Recv(recv + (size_t)q * n, n, ncclFloat64, q, c->nc, st));
  }
  GK_NCCL(api.GroupEnd());
  return GK_OK;
}
int comm_allgather(gk_comm* c, const double* send, double* recv, int64_t elems, cudaStream_t st) {
  GK_NCCL(nccl().AllGather(send, recv, (size_t)elems * 2, ncclFloat64, c->nc, st));
  return GK_OK;
}
}  // namespace gk

extern "C" {

int gk_comm_unique_id(void* id) {
  GK_CHECK_ARG(id, "gk_comm_unique_id: null pointer");
  NcclApi& api = nccl();
  GK_CHECK_ARG(api.ok, "gk_comm_unique_id: %s", api.why);
  ncclUniqueId u;
  GK_NCCL(api.GetUniqueId(&u));
  memcpy(id, &u, sizeof(u));
  return GK_OK;
}

int gk_comm_init(int nranks, int rank, const void* id, gk_comm** comm) {
  GK_CHECK_ARG(comm && id, "gk_comm_init: null pointer");
  *comm = nullptr;
  GK_CHECK_ARG(nranks >= 1 && rank >= 0 && rank < nranks, "gk_comm_init: rank %d of %d", rank, nranks);
  NcclApi& api = nccl();
  GK_CHECK_ARG(api.ok, "gk_comm_init: %s", api.why);
  auto* c = new gk_comm{};
  c->nranks = nranks;
  c->rank = rank;
  cudaGetDevice(&c->device);
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  ncclResult_t r = api.CommInitRank(&c->nc, nranks, u, rank);
  if (r != ncclSuccess) {
    gk::set_error("ncclCommInitRank failed: %s", api.GetErrorString(r));
    delete c;
    return GK_ERR_COMM;
  }
  bool ok = cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking) == cudaSuccess;
  for (cudaEvent_t* e : {&c->start, &c->phi, &c->gathered, &c->done})
    ok = ok && cudaEventCreateWithFlags(e, cudaEventDisableTiming) == cudaSuccess;
  for (int i = 0; ok && i < gk_comm::kMaxChunks; ++i)
    for (cudaEvent_t* e : {&c->rf[i], &c->br[i], &c->bk[i], &c->fin[i]})
      ok = ok && cudaEventCreateWithFlags(e, cudaEventDisableTiming) == cudaSuccess;
  if (!ok) {
    gk::set_error("gk_comm_init: could not create the communication stream / events");
    gk_comm_destroy(c);
    return GK_ERR_CUDA;
  }
  *comm = c;
  return GK_OK;
}

int gk_comm_destroy(gk_comm* c) {
  if (!c) return GK_OK;
  if (c->nc) nccl().CommDestroy(c->nc);
  for (cudaEvent_t e : {c->start, c->phi, c->gathered, c->done})
    if (e) cudaEventDestroy(e);
  for (int i = 0; i < gk_comm::kMaxChunks; ++i)
    for (cudaEvent_t e : {c->rf[i], c->br[i], c->bk[i], c->fin[i]})
      if (e) cudaEventDestroy(e);
  if (c->cs) cudaStreamDestroy(c->cs);
  delete c;
  return GK_OK;
}

int gk_comm_info(const gk_comm* c, int* nranks, int* rank, int* nccl_version) {
  GK_CHECK_ARG(c, "gk_comm_info: null communicator");
  if (nranks) *nranks = c->nranks;
  if (rank) *rank = c->rank;
  if (nccl_version) {
    int v = 0;
    nccl().GetVersion(&v);
    *nccl_version = v;
  }
  return GK_OK;
}

// Velocity-chunk transposes.  home_rows: a chunk of G * rows_per_rank home-layout
// velocity rows ([M][T][Y/G][R] rows of row_elems complex values); rank q
// brackets rows [q rpr, (q + 1) rpr) of it.  recv: [G src][rpr][T][Y/G][R], the
// blocked layout gk_nonlinear_blocked reads.
int gk_transpose_to_nl(gk_comm* c, const double* home_rows, double* recv, int64_t rows_per_rank, int64_t row_elems,
                       void* stream) {
  GK_CHECK_ARG(c && home_rows && recv, "gk_transpose_to_nl: null pointer");
  return gk::comm_alltoall(c, home_rows, recv, rows_per_rank * row_elems, (cudaStream_t)stream, false);
}
// send: [G dst][rpr][T][Y/G][R] (gk_nonlinear_blocked's output); rank q's block
// lands in rows [q rpr, (q + 1) rpr) of home_rows.
int gk_transpose_to_lin(gk_comm* c, const double* send, double* home_rows, int64_t rows_per_rank, int64_t row_elems,
                        void* stream) {
  GK_CHECK_ARG(c && send && home_rows, "gk_transpose_to_lin: null pointer");
  return gk::comm_alltoall(c, send, home_rows, rows_per_rank * row_elems, (cudaStream_t)stream, false);
}

int gk_comm_allgather(gk_comm* c, const double* send, double* recv, int64_t elems, void* stream) {
  GK_CHECK_ARG(c && send && recv, "gk_comm_allgather: null pointer");
  return gk::comm_allgather(c, send, recv, elems, (cudaStream_t)stream);
}

}  // extern "C"
