// comm.cuh — the multi-GPU exchange used by subtree sharding (DESIGN.md
// "Multi-GPU").  The hot path needs exactly one collective: an allgather of fixed-size,
// rank-major slots (subtree-root skeleton data once per build, reduced Schur blocks once per
// factorization, the reduced right-hand side + the w^T q partial once per ADMM iteration).
//
// Two backends:
//  - NCCL (libnccl.so.2 loaded at run time, so the single-GPU library has no NCCL
//    dependency): ncclAllGather on device buffers, stream-ordered, capturable in the ADMM
//    iteration's CUDA graph.  Production path over NVLink 5 / NVSwitch.
//  - host callback: the caller supplies allgather(ctx, send, recv, bytes) on HOST buffers
//    (e.g. torch.distributed/gloo from Python).  The library stages through pinned memory and
//    synchronizes the stream, so it is not capturable; used to run P ranks as P processes on
//    fewer GPUs (P-invariance tests) without any kernel waiting on another rank.
#pragma once
#include <memory>
#include "common.cuh"

namespace svmhss {

struct Comm {
  int size = 1, rank = 0;
  virtual ~Comm() {}
  virtual bool capturable() const = 0;
  // recv[p * bytes .. (p+1) * bytes) = rank p's send (device pointers, ordered on s).
  virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
};

std::shared_ptr<Comm> make_nccl_comm(int nranks, int rank, const void* unique_id);
std::shared_ptr<Comm> make_host_comm(int nranks, int rank, hss_allgather_fn fn, void* ctx);
void nccl_unique_id(void* out128);

}  // namespace svmhss
