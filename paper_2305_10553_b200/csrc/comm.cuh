// The multi-GPU communicator shared by comm.cu (NCCL plumbing) and dist.cu (the
// rank step).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

struct ncclComm;

// The communicator: one NCCL communicator + the communication stream the step
// issues every NCCL operation on (one stream, so every rank enqueues the
// operations in the same order), and the events that pipeline it with the compute.
struct gk_comm {
  ncclComm* nc = nullptr;
  int nranks = 0, rank = 0, device = 0;
  cudaStream_t cs = nullptr;
  static constexpr int kMaxChunks = 64;
  cudaEvent_t start = nullptr, phi = nullptr, gathered = nullptr, done = nullptr;
  cudaEvent_t rf[kMaxChunks] = {}, br[kMaxChunks] = {}, bk[kMaxChunks] = {}, fin[kMaxChunks] = {};
};


namespace gk {
int comm_alltoall(gk_comm* c, const double* send, double* recv, int64_t block_elems, cudaStream_t st,
                  bool skip_self);
int comm_allgather(gk_comm* c, const double* send, double* recv, int64_t elems, cudaStream_t st);
}  // namespace gk
