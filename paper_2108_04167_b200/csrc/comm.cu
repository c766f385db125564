// comm.cu — backends of the subtree-sharding allgather (see comm.cuh).
#include <dlfcn.h>
#include <cstring>
#include "comm.cuh"

namespace svmhss {

// ------------------------------------------------------------------ NCCL (dlopen)
// Minimal NCCL ABI (nccl.h, stable since 2.x): opaque communicator, 128-byte unique id,
// ncclInt8 = 0.
namespace nccl {
typedef struct ncclComm* comm_t;
typedef struct { char internal[128]; } uid_t;
typedef int res_t;
struct Api {
  void* h = nullptr;
  res_t (*GetUniqueId)(uid_t*) = nullptr;
  res_t (*CommInitRank)(comm_t*, int, uid_t, int) = nullptr;
  res_t (*CommDestroy)(comm_t) = nullptr;
  res_t (*AllGather)(const void*, void*, size_t, int, comm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(res_t) = nullptr;
};
static Api& api() {
  static Api a;
  static bool tried = false;
  if (!tried) {
    tried = true;
    // the process's NCCL (torch loads its bundled libnccl.so.2 first), else the system one
    a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!a.h) a.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (a.h) {
      a.GetUniqueId = (res_t(*)(uid_t*))dlsym(a.h, "ncclGetUniqueId");
      a.CommInitRank = (res_t(*)(comm_t*, int, uid_t, int))dlsym(a.h, "ncclCommInitRank");
      a.CommDestroy = (res_t(*)(comm_t))dlsym(a.h, "ncclCommDestroy");
      a.AllGather = (res_t(*)(const void*, void*, size_t, int, comm_t, cudaStream_t))dlsym(a.h, "ncclAllGather");
      a.GetErrorString = (const char* (*)(res_t))dlsym(a.h, "ncclGetErrorString");
    }
  }
  if (!a.h || !a.GetUniqueId || !a.CommInitRank || !a.CommDestroy || !a.AllGather)
    throw Error(HSS_ENCCL, "NCCL not available (dlopen libnccl.so.2 failed)");
  return a;
}
static void check(res_t r, const char* what) {
  if (r != 0)
    throw Error(HSS_ENCCL, std::string(what) + ": " +
                               (api().GetErrorString ? api().GetErrorString(r) : "nccl error"));
}
}  // namespace nccl

struct NcclComm : Comm {
  nccl::comm_t c = nullptr;
  NcclComm(int n, int r, const void* id) {
    size = n;
    rank = r;
    nccl::uid_t u;
    std::memcpy(&u, id, sizeof(u));
    nccl::check(nccl::api().CommInitRank(&c, n, u, r), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (c) nccl::api().CommDestroy(c);
  }
  bool capturable() const override { return true; }
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    if (size == 1) {
      if (send != recv) CUDA_CHECK(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, s));
      return;
    }
    nccl::check(nccl::api().AllGather(send, recv, bytes, /*ncclInt8*/ 0, c, s), "ncclAllGather");
  }
};

void nccl_unique_id(void* out128) {
  nccl::uid_t u;
  nccl::check(nccl::api().GetUniqueId(&u), "ncclGetUniqueId");
  std::memcpy(out128, &u, sizeof(u));
}

std::shared_ptr<Comm> make_nccl_comm(int nranks, int rank, const void* unique_id) {
  return std::make_shared<NcclComm>(nranks, rank, unique_id);
}

// ------------------------------------------------------------------ host callback
struct HostComm : Comm {
  hss_allgather_fn fn;
  void* ctx;
  std::vector<char> hs, hr;  // host staging (the callback may be slow; pinning is not needed)
  HostComm(int n, int r, hss_allgather_fn f, void* c) : fn(f), ctx(c) { size = n; rank = r; }
  bool capturable() const override { return false; }
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    hs.resize(bytes);
    hr.resize(bytes * size);
    if (bytes) CUDA_CHECK(cudaMemcpyAsync(hs.data(), send, bytes, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    const int rc = fn(ctx, hs.data(), hr.data(), bytes);
    if (rc != 0) throw Error(HSS_ENCCL, "host allgather callback failed (rc " + std::to_string(rc) + ")");
    if (bytes) CUDA_CHECK(cudaMemcpyAsync(recv, hr.data(), bytes * size, cudaMemcpyHostToDevice, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
};

std::shared_ptr<Comm> make_host_comm(int nranks, int rank, hss_allgather_fn fn, void* ctx) {
  return std::make_shared<HostComm>(nranks, rank, fn, ctx);
}

}  // namespace svmhss
