// comm.cu — backends of the subtree-sharding allgather (see comm.cuh).
#include <dlfcn.h>
#include <cstdlib>
#include <cstring>
#include "comm.cuh"
#ifdef SVMHSS_HAVE_NCCL_DEVICE
#include <nccl.h>
#include <nccl_device.h>
#endif

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
  // device API (NCCL >= 2.28; nullptr when the loaded NCCL lacks it)
  void* DevCommCreate = nullptr;
  void* DevCommDestroy = nullptr;
  void* WindowRegister = nullptr;
  void* WindowDeregister = nullptr;
  void* MemAlloc = nullptr;
  void* MemFree = nullptr;
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
      a.DevCommCreate = dlsym(a.h, "ncclDevCommCreate");
      a.DevCommDestroy = dlsym(a.h, "ncclDevCommDestroy");
      a.WindowRegister = dlsym(a.h, "ncclCommWindowRegister");
      a.WindowDeregister = dlsym(a.h, "ncclCommWindowDeregister");
      a.MemAlloc = dlsym(a.h, "ncclMemAlloc");
      a.MemFree = dlsym(a.h, "ncclMemFree");
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

#ifdef SVMHSS_HAVE_NCCL_DEVICE
// The fused exchange (N3): pack this rank's slot straight into every peer's window (NVLink
// stores through the LSA pointers), one LSA barrier (release / acquire: every peer's stores are
// visible), unpack all P slots from the local window.  The window has two halves used on
// alternate calls (device parity counter), so a rank that runs ahead into the next iteration
// never overwrites a slot a slower peer has not unpacked yet: to write half h again it must pass
// the next barrier, which every peer reaches only after finishing its unpack of half h.
__global__ void __launch_bounds__(512) lsa_exchange_kernel(ncclDevComm dc, ncclWindow_t win, unsigned* parity,
                                                           int P, int rank, ExchangeArgs A) {
  const unsigned half = *parity & 1u;
  const size_t base = (size_t)half * P * A.slot * sizeof(double);
  const int64_t nrow = (int64_t)A.own_k * A.ncols;
  const double* src = A.buf + A.own_koff * A.ncols;
  for (int peer = 0; peer < P; ++peer) {
    double* dst = (double*)ncclGetLsaPointer(win, base + (size_t)rank * A.slot * sizeof(double), peer);
    for (int64_t e = threadIdx.x; e < nrow; e += blockDim.x) dst[e] = src[e];
    for (int e = threadIdx.x; e < A.nextra; e += blockDim.x) dst[(int64_t)A.kmax * A.ncols + e] = A.extra[e];
  }
  {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), 0);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  }
  const double* loc = (const double*)((const char*)ncclGetLocalPointer(win, 0) + base);
  for (int p = 0; p < P; ++p) {
    const int64_t cnt = A.kk[p] * A.ncols;
    double* dst = A.buf + A.koff[p] * A.ncols;
    for (int64_t e = threadIdx.x; e < cnt; e += blockDim.x) dst[e] = loc[p * A.slot + e];
    if (A.extra_out)
      for (int e = threadIdx.x; e < A.nextra; e += blockDim.x)
        A.extra_out[p * A.nextra + e] = loc[p * A.slot + (int64_t)A.kmax * A.ncols + e];
  }
  __syncthreads();
  if (threadIdx.x == 0) *parity += 1u;
}
#endif

struct NcclComm : Comm {
  nccl::comm_t c = nullptr;
  bool dev = false;
#ifdef SVMHSS_HAVE_NCCL_DEVICE
  ncclDevComm dcomm{};
#endif
  NcclComm(int n, int r, const void* id, int device_api) {
    size = n;
    rank = r;
    nccl::uid_t u;
    std::memcpy(&u, id, sizeof(u));
    nccl::check(nccl::api().CommInitRank(&c, n, u, r), "ncclCommInitRank");
#ifdef SVMHSS_HAVE_NCCL_DEVICE
    const char* e = getenv("SVMHSS_NCCL_DEVICE");
    auto& A = nccl::api();
    if (device_api && !(e && e[0] == '0') && A.DevCommCreate && A.WindowRegister && A.MemAlloc) {
      ncclDevCommRequirements req{};
      req.lsaBarrierCount = 1;
      auto create = (ncclResult_t(*)(ncclComm_t, ncclDevCommRequirements_t const*, ncclDevComm_t*))A.DevCommCreate;
      // collective: every rank creates (or fails) alike; an LSA team smaller than the
      // communicator (ranks not all NVLink load/store peers) keeps ncclAllGather
      if (create((ncclComm_t)c, &req, &dcomm) == ncclSuccess)
        dev = dcomm.lsaSize == n && dcomm.lsaRank == r;
    }
#else
    (void)device_api;
#endif
  }
  ~NcclComm() override {
#ifdef SVMHSS_HAVE_NCCL_DEVICE
    if (dev && nccl::api().DevCommDestroy)
      ((ncclResult_t(*)(ncclComm_t, ncclDevComm_t const*))nccl::api().DevCommDestroy)((ncclComm_t)c, &dcomm);
#endif
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
  bool device_api() const override { return dev; }
#ifdef SVMHSS_HAVE_NCCL_DEVICE
  DevWindow window_alloc(size_t bytes) override {
    DevWindow w;
    auto& A = nccl::api();
    const size_t al = NCCL_WIN_REQUIRED_ALIGNMENT;
    w.bytes = (2 * bytes + al - 1) / al * al;  // two halves (alternate calls)
    nccl::check(((ncclResult_t(*)(void**, size_t))A.MemAlloc)(&w.mem, w.bytes), "ncclMemAlloc");
    ncclWindow_t win = nullptr;
    nccl::check(((ncclResult_t(*)(ncclComm_t, void*, size_t, ncclWindow_t*, int))A.WindowRegister)(
                    (ncclComm_t)c, w.mem, w.bytes, &win, NCCL_WIN_COLL_SYMMETRIC),
                "ncclCommWindowRegister");
    w.win = win;
    CUDA_CHECK(cudaMalloc((void**)&w.parity, sizeof(unsigned)));
    CUDA_CHECK(cudaMemset(w.parity, 0, sizeof(unsigned)));
    return w;
  }
  void window_free(DevWindow& w) override {
    auto& A = nccl::api();
    if (w.win && A.WindowDeregister)
      ((ncclResult_t(*)(ncclComm_t, ncclWindow_t))A.WindowDeregister)((ncclComm_t)c, (ncclWindow_t)w.win);
    if (w.mem && A.MemFree) ((ncclResult_t(*)(void*))A.MemFree)(w.mem);
    if (w.parity) cudaFree(w.parity);
    w = DevWindow{};
  }
  void device_exchange(const DevWindow& w, const ExchangeArgs& a, cudaStream_t s) override {
    lsa_exchange_kernel<<<1, 512, 0, s>>>(dcomm, (ncclWindow_t)w.win, w.parity, size, rank, a);
    LAUNCH_CHECK();
  }
#endif
};

void nccl_unique_id(void* out128) {
  nccl::uid_t u;
  nccl::check(nccl::api().GetUniqueId(&u), "ncclGetUniqueId");
  std::memcpy(out128, &u, sizeof(u));
}

std::shared_ptr<Comm> make_nccl_comm(int nranks, int rank, const void* unique_id, int device_api) {
  return std::make_shared<NcclComm>(nranks, rank, unique_id, device_api);
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
