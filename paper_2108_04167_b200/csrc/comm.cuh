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

// The level-lg exchange of one ADMM iteration (or mat-vec), as one fused kernel: rank g's slot =
// its own node's rows of `buf` (own_k x ncols at own_koff) + `extra` (nextra), every rank's slot is
// unpacked into buf (node p at koff[p], kk[p] rows) and extra_out (P x nextra).
struct ExchangeArgs {
  double* buf;
  int64_t own_koff;
  int own_k, ncols, nextra, kmax;
  const double* extra;
  double* extra_out;
  const int64_t *koff, *kk;  // device, P entries
  int64_t slot;              // doubles per rank slot (kmax * ncols + nextra)
};
// A symmetric window (NCCL device API): local pointer + opaque handle.
struct DevWindow {
  void* win = nullptr;   // ncclWindow_t
  void* mem = nullptr;   // ncclMemAlloc'd base
  unsigned* parity = nullptr;  // device counter selecting the window half
  size_t bytes = 0;
};

struct Comm {
  int size = 1, rank = 0;
  virtual ~Comm() {}
  virtual bool capturable() const = 0;
  // recv[p * bytes .. (p+1) * bytes) = rank p's send (device pointers, ordered on s).
  virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
  // in-kernel exchange over NVLink through the NCCL device API (LSA symmetric
  // windows + LSA barrier).  device_api(): available on this communicator (every rank an LSA
  // peer).  window_alloc / window_free are COLLECTIVE (every rank, same order).
  virtual bool device_api() const { return false; }
  virtual DevWindow window_alloc(size_t bytes) { (void)bytes; return DevWindow{}; }
  virtual void window_free(DevWindow&) {}
  virtual void device_exchange(const DevWindow&, const ExchangeArgs&, cudaStream_t) {}
};

// device_api: 1 = use the NCCL device API for the per-iteration exchange when every rank is an
// LSA (NVLink load/store) peer, 0 = always ncclAllGather (env SVMHSS_NCCL_DEVICE=0 also disables).
std::shared_ptr<Comm> make_nccl_comm(int nranks, int rank, const void* unique_id, int device_api = 1);
std::shared_ptr<Comm> make_host_comm(int nranks, int rank, hss_allgather_fn fn, void* ctx);
void nccl_unique_id(void* out128);

}  // namespace svmhss
