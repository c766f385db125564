// common.cuh — shared device/host helpers of libsvmhss (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>
#include <vector>
#include <stdexcept>
#include <atomic>

#include "../../include/svmhss.h"

namespace svmhss {

// ------------------------------------------------------------------ errors
struct Error : public std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& s);

#define CUDA_CHECK(x)                                                                 \
  do {                                                                                \
    cudaError_t e__ = (x);                                                            \
    if (e__ != cudaSuccess)                                                           \
      throw ::svmhss::Error(e__ == cudaErrorMemoryAllocation ? HSS_ENOMEM : HSS_ECUDA, \
                            std::string(#x) + ": " + cudaGetErrorString(e__));        \
  } while (0)

extern std::atomic<long long> g_launches;  // kernels launched by this library (api.cu)
#define LAUNCH_CHECK()                         \
  do {                                         \
    ::svmhss::g_launches.fetch_add(1);         \
    CUDA_CHECK(cudaGetLastError());            \
  } while (0)

inline void require(bool ok, const std::string& msg) {
  if (!ok) throw Error(HSS_EINVAL, msg);
}

// ------------------------------------------------------------------ device buffers
// Stream-ordered allocations from the library's own memory pool on the current device
// (cudaMemPoolCreate, release threshold "never" while handles are alive, so steady-state steps
// do not call the driver allocator and cudaFree never forces a device synchronization; trimmed
// when the device's last hss_t / ulv_t is freed).  The device's default pool (torch's
// cudaMallocAsync backend) is never touched.  The allocation stream is the library call's stream.
extern thread_local cudaStream_t g_alloc_stream;
cudaMemPool_t lib_pool();                  // the current device's pool (created on first use)
void lib_malloc(void** p, size_t bytes, cudaStream_t s);   // throws Error on failure
struct StreamScope {  // sets the allocation stream for the duration of an API call
  cudaStream_t prev;
  explicit StreamScope(cudaStream_t s) : prev(g_alloc_stream) { g_alloc_stream = s; }
  ~StreamScope() { g_alloc_stream = prev; }
};

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t st = nullptr;
  DevBuf() {}
  explicit DevBuf(size_t count) { alloc(count); }
  void alloc(size_t count) {
    release();
    n = count;
    st = g_alloc_stream;
    if (count) lib_malloc((void**)&p, count * sizeof(T), st);
  }
  void release() {
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), st(o.st) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    release(); p = o.p; n = o.n; st = o.st; o.p = nullptr; o.n = 0; return *this;
  }
  size_t bytes() const { return n * sizeof(T); }
};

template <typename T>
inline void h2d(T* d, const T* h, size_t n, cudaStream_t s) {
  if (n) CUDA_CHECK(cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
}
template <typename T>
inline void d2h(T* h, const T* d, size_t n, cudaStream_t s) {
  if (n) CUDA_CHECK(cudaMemcpyAsync(h, d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
}

// A device copy of a host vector (uploaded on `s`; host vector must outlive the copy —
// callers synchronize or keep the vector alive).
template <typename T>
inline DevBuf<T> upload(const std::vector<T>& v, cudaStream_t s) {
  DevBuf<T> d(v.size());
  h2d(d.p, v.data(), v.size(), s);
  return d;
}

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// ------------------------------------------------------------------ timing
struct EventTimer {
  cudaEvent_t a, b;
  cudaStream_t s;
  explicit EventTimer(cudaStream_t st) : s(st) {
    CUDA_CHECK(cudaEventCreate(&a));
    CUDA_CHECK(cudaEventCreate(&b));
    CUDA_CHECK(cudaEventRecord(a, s));
  }
  double stop_ms() {
    CUDA_CHECK(cudaEventRecord(b, s));
    CUDA_CHECK(cudaEventSynchronize(b));
    float ms = 0;
    CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
    return ms;
  }
  ~EventTimer() { cudaEventDestroy(a); cudaEventDestroy(b); }
};

// Optional phase trace (env SVMHSS_TRACE=1): host wall time and stream time between marks,
// printed to stderr when the tracer goes out of scope.  Off: no events, no cost.
struct PhaseTrace {
  bool on = false;
  cudaStream_t s = nullptr;
  std::string name;
  std::vector<std::pair<std::string, cudaEvent_t>> ev;
  std::vector<double> host_ms;
  double t0 = 0;
  static double now_ms();
  PhaseTrace(const char* nm, cudaStream_t st);
  void mark(const std::string& tag);
  ~PhaseTrace();
};

// ------------------------------------------------------------------ device helpers
// Programmatic dependent launch (PDL): a kernel launched with launch_pdl lets the next kernel of
// the stream / graph be scheduled once all its CTAs have started (pdl_trigger), and waits for the
// previous kernel's completion and memory (pdl_wait) before touching anything it produced.
// Both are no-ops for kernels launched without the attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum with a fixed reduction order (deterministic). `red` >= 32 doubles.
__device__ __forceinline__ double block_sum(double v, double* red) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < nw ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

// splitmix64 finalizer (reading R1-R3; same constants as oracle/rng.py, independently written)
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// R1-R3: Gaussian keyed by (seed key, i, j).  `key` = splitmix64(seed).
__device__ __forceinline__ double counter_gaussian(uint64_t key, uint64_t i, uint64_t j) {
  uint64_t ctr = (i << 20) | j;
  uint64_t base = key + 2ull * ctr;
  uint64_t a = splitmix64(base), b = splitmix64(base + 1ull);
  double u1 = ((double)(a >> 11) + 0.5) * 0x1.0p-53;
  double u2 = (double)(b >> 11) * 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

}  // namespace svmhss
