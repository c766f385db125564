// api.cu — the C-ABI of libsvmhss.so (include/svmhss.h).  Argument validation, handle
// ownership (reference counted hss_t <- ulv_t), error translation; no arithmetic here.
#include <chrono>
#include <cmath>
#include <cstring>
#include <mutex>
#include "internal.cuh"

namespace svmhss {
static thread_local std::string g_last_error;
std::atomic<long long> g_launches{0};
thread_local cudaStream_t g_alloc_stream = nullptr;
// One pool per device, created on first use (never reconfigure the device's default
// pool, which torch's cudaMallocAsync backend shares).  live[dev] counts this device's alive
// hss_t / ulv_t handles; when it drops to zero the pool is trimmed back to nothing.
static std::mutex g_pool_mu;
static std::vector<cudaMemPool_t> g_pools;
static std::vector<int> g_live;
static std::vector<size_t> g_reserved;   // pool_reserve's current reservation, per device

static int cur_device() {
  int dev = 0;
  CUDA_CHECK(cudaGetDevice(&dev));
  return dev;
}

cudaMemPool_t lib_pool() {
  const int dev = cur_device();
  std::lock_guard<std::mutex> g(g_pool_mu);
  if ((int)g_pools.size() <= dev) {
    g_pools.resize(dev + 1, nullptr);
    g_live.resize(dev + 1, 0);
    g_reserved.resize(dev + 1, 0);
  }
  if (!g_pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool;
    CUDA_CHECK(cudaMemPoolCreate(&pool, &props));
    uint64_t thr = UINT64_MAX;
    CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    g_pools[dev] = pool;
  }
  return g_pools[dev];
}

void lib_malloc(void** p, size_t bytes, cudaStream_t s) {
  CUDA_CHECK(cudaMallocFromPoolAsync(p, bytes, lib_pool(), s));
}

// handle bookkeeping (hss_t / ulv_t of the current device)
static void handle_acquired() {
  const int dev = cur_device();
  lib_pool();
  std::lock_guard<std::mutex> g(g_pool_mu);
  ++g_live[dev];
}
static void handle_released(int dev) {
  cudaMemPool_t pool = nullptr;
  // SVMHSS_POOL_KEEP=1: keep the reservation when the last handle goes (a process that rebuilds
  // repeatedly, e.g. bench.py's steps, avoids re-mapping GBs per build; hss_pool_trim releases)
  static const bool keep = [] { const char* e = getenv("SVMHSS_POOL_KEEP"); return e && e[0] == '1'; }();
  {
    std::lock_guard<std::mutex> g(g_pool_mu);
    if (dev < 0 || dev >= (int)g_live.size()) return;
    if (--g_live[dev] > 0 || keep) return;
    pool = g_pools[dev];
    g_reserved[dev] = 0;
  }
  if (!pool) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(dev);
  cudaDeviceSynchronize();   // every stream-ordered free of the pool has completed
  cudaMemPoolTrimTo(pool, 0);
  cudaSetDevice(prev);
  cudaGetLastError();
}

// Memory-pool reservation ahead of a build: one physical chunk of about the problem's peak
// footprint (sketch operands, generators, factor and its per-level temporaries ~ 24 n (s + r) 8
// bytes), capped at half the free memory, so the stream-ordered allocations of build / factor /
// ADMM sub-allocate from it instead of growing the pool (mapping GBs) in the middle of a
// factorization.  SVMHSS_POOL_RESERVE_GB overrides the estimate (0 disables).
static void pool_reserve(int64_t n, int r, int s_cols, cudaStream_t st) {
  const int dev = cur_device();
  cudaMemPool_t pool = lib_pool();
  const char* e = getenv("SVMHSS_POOL_RESERVE_GB");
  double want = e ? atof(e) * 1e9 : 24.0 * (double)n * (double)(s_cols + r) * 8.0;
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) { cudaGetLastError(); return; }
  size_t reserved;
  {
    std::lock_guard<std::mutex> g(g_pool_mu);
    reserved = g_reserved[dev];
  }
  want = std::min(want, 0.5 * (double)fr + (double)reserved);
  if (want <= (double)reserved + 64e6) return;
  void* p = nullptr;
  if (cudaMallocFromPoolAsync(&p, (size_t)want, pool, st) == cudaSuccess) {
    cudaFreeAsync(p, st);
    std::lock_guard<std::mutex> g(g_pool_mu);
    g_reserved[dev] = (size_t)want;
  } else {
    cudaGetLastError();
  }
}

bool pdl_enabled() {
  static const bool on = [] { const char* e = getenv("SVMHSS_PDL"); return !(e && e[0] == '0'); }();
  return on;
}

void set_last_error(const std::string& s) { g_last_error = s; }

double PhaseTrace::now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
PhaseTrace::PhaseTrace(const char* nm, cudaStream_t st) : s(st), name(nm) {
  const char* e = getenv("SVMHSS_TRACE");
  on = e && e[0] == '1';
  if (on) { t0 = now_ms(); mark("start"); }
}
void PhaseTrace::mark(const std::string& tag) {
  if (!on) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, s);
  ev.push_back({tag, e});
  host_ms.push_back(now_ms() - t0);
}
PhaseTrace::~PhaseTrace() {
  if (!on) return;
  mark("end");
  cudaEventSynchronize(ev.back().second);
  fprintf(stderr, "[svmhss trace] %s\n", name.c_str());
  for (size_t i = 1; i < ev.size(); ++i) {
    float ms = 0;
    cudaEventElapsedTime(&ms, ev[i - 1].second, ev[i].second);
    fprintf(stderr, "  %-28s gpu %9.3f ms   host@ %9.3f ms\n", ev[i].first.c_str(), ms, host_ms[i]);
  }
  for (auto& x : ev) cudaEventDestroy(x.second);
}

static void ensure_device() {
  int cnt = 0;
  cudaError_t e = cudaGetDeviceCount(&cnt);
  if (e != cudaSuccess || cnt == 0) throw Error(HSS_ECUDA, "no CUDA device available (no CPU fallback exists)");
}

template <typename Fn>
static int guarded(Fn&& fn, bool need_device = true) {
  try {
    if (need_device) ensure_device();
    fn();
    return HSS_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    cudaGetLastError();
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return HSS_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return HSS_ECUDA;
  }
}

// node (l, i) has its generators on this rank (always true on one GPU)
static bool held(const HSSImpl& H, int l, int i) {
  if (l < H.sh.lg) return true;
  if (H.sh.on() && l == H.sh.lg) return true;  // exchanged: k and skeletons known everywhere
  return i >= H.sh.first(l) && i < H.sh.last(l);
}

// hss_build with the adaptive sampling loop (N2a-c) when opt.adaptive_s0 > 0
static HSSImpl* build_adaptive(const double* F, int64_t n, int r, double h, const hss_opts& o,
                               std::shared_ptr<Comm> comm, cudaStream_t s) {
  const int s_max = o.max_rank + o.oversample;
  int s_cur = (o.adaptive_s0 > 0) ? std::min(o.adaptive_s0, s_max) : s_max;
  if (s_cur % 2) ++s_cur;  // the sketch kernel needs an even column count
  s_cur = std::min(s_cur, s_max);
  double ms[4] = {0, 0, 0, 0};
  for (int round = 1;; ++round) {
    auto* H = new HSSImpl();
    try {
      hss_build_impl(*H, F, n, r, h, o, comm, s, s_cur);
    } catch (...) {
      delete H;
      throw;
    }
    ms[0] += H->st.ms_tree; ms[1] += H->st.ms_omega; ms[2] += H->st.ms_sketch; ms[3] += H->st.ms_compress;
    const bool done = o.adaptive_s0 <= 0 || s_cur >= s_max || !hss_unconverged(*H, o.oversample, o.max_rank);
    if (done) {
      H->st.s_used = s_cur;
      H->st.sample_rounds = round;
      H->st.ms_tree = ms[0]; H->st.ms_omega = ms[1]; H->st.ms_sketch = ms[2]; H->st.ms_compress = ms[3];
      return H;
    }
    delete H;
    s_cur = std::min(s_max, s_cur + o.adaptive_ds + (o.adaptive_ds % 2));
  }
}

static void release_hss(HSSImpl* H) {
  if (H && H->refs.fetch_sub(1) == 1) delete H;
}

static void validate_opts(const hss_opts* o, int64_t n, int32_t r, double h) {
  require(o != nullptr, "hss_build: opts is NULL");
  require(n >= 1, "hss_build: n must be >= 1");
  require(r >= 1, "hss_build: r must be >= 1");
  require(std::isfinite(h) && h > 0, "hss_build: h must be > 0");
  require(o->leaf_size >= 1, "hss_build: leaf_size must be >= 1");
  require(o->max_rank >= 1, "hss_build: max_rank must be >= 1");
  require(o->oversample >= 0, "hss_build: oversample must be >= 0");
  const int s = o->max_rank + o->oversample;
  require(s <= (1 << 20), "hss_build: s = max_rank + oversample must be <= 2^20 (R1 column field)");
  require(s % 2 == 0, "hss_build: s = max_rank + oversample must be even");
  require(o->rel_tol >= 0 && o->abs_tol >= 0, "hss_build: tolerances must be >= 0");
  require(o->sampling == HSS_SAMPLING_SKETCH || o->sampling == HSS_SAMPLING_ANN, "hss_build: unknown sampling");
  require(o->interp == HSS_INTERP_ID || o->interp == HSS_INTERP_SPD, "hss_build: unknown interp");
  require(o->interp == HSS_INTERP_ID || (std::isfinite(o->spd_eps) && o->spd_eps >= 0),
          "hss_build: spd_eps must be finite and >= 0");
  if (o->adaptive_s0 > 0) {
    require(o->sampling == HSS_SAMPLING_SKETCH, "hss_build: adaptive sampling needs the sketch sampling");
    require(o->adaptive_ds > 0, "hss_build: adaptive_ds must be > 0");
  }
  if (o->sampling == HSS_SAMPLING_ANN) {
    require(o->ann_neighbors >= 1 && o->ann_trees >= 1 && o->ann_leaf >= 2 && o->ann_leaf <= 256,
            "hss_build: ANN needs ann_neighbors >= 1, ann_trees >= 1, 2 <= ann_leaf <= 256");
    require((int64_t)o->ann_trees * o->ann_neighbors <= 256, "hss_build: ann_trees * ann_neighbors must be <= 256");
    require((int64_t)o->ann_leaf * r * 8 <= 227 * 1024, "hss_build: ann_leaf * r too large (lower ann_leaf)");
    require(s <= 1152, "hss_build: s must be <= 1152");
  }
}

}  // namespace svmhss

using namespace svmhss;

struct hss_s { HSSImpl* impl; int dev; };
struct ulv_s { ULVImpl* impl; int dev; };
struct hss_comm_s { std::shared_ptr<Comm> c; };

static std::shared_ptr<Comm> comm_of(const hss_opts* o) {
  return (o && o->comm) ? o->comm->c : std::shared_ptr<Comm>();
}

extern "C" {

const char* hss_last_error(void) { return g_last_error.c_str(); }
const char* hss_version(void) { return "svmhss 0.2 (sm_100a)"; }
int64_t hss_launch_count(void) { return (int64_t)g_launches.load(); }

int hss_build(const double* F, int64_t n, int32_t r, double h, const hss_opts* opt, void* stream,
              hss_t* out) {
  return guarded([&] {
    StreamScope ss__((cudaStream_t)stream);
    require(out != nullptr && F != nullptr, "hss_build: NULL pointer");
    validate_opts(opt, n, r, h);
    pool_reserve(n, r, opt->max_rank + opt->oversample, (cudaStream_t)stream);
    HSSImpl* H = build_adaptive(F, n, r, h, *opt, comm_of(opt), (cudaStream_t)stream);
    handle_acquired();
    *out = new hss_s{H, cur_device()};
  });
}

int hss_info(hss_t Hh, hss_stats* st, int64_t* perm_out, int32_t* ranks_out, int64_t* skel_out) {
  return guarded([&] {
    require(Hh != nullptr, "hss_info: NULL handle");
    const HSSImpl& H = *Hh->impl;
    if (st) *st = H.st;
    if (perm_out) {
      CUDA_CHECK(cudaMemcpy(perm_out, H.perm.p, H.n * sizeof(int64_t), cudaMemcpyDeviceToHost));
    }
    if (ranks_out) {
      const int nn = (1 << (H.L + 1)) - 1;
      for (int t = 0; t < nn; ++t) ranks_out[t] = -1;
      for (int l = 1; l <= H.L; ++l)
        for (size_t i = 0; i < H.lv[l].size(); ++i)
          ranks_out[H.node_id(l, (int)i)] = held(H, l, (int)i) ? H.lv[l][i].k : -2;
    }
    if (skel_out) {
      int64_t off = 0;
      for (int l = 1; l <= H.L; ++l)
        for (size_t i = 0; i < H.lv[l].size(); ++i) {
          if (!held(H, l, (int)i)) continue;
          const auto& nd = H.lv[l][i];
          if (nd.k > 0)
            CUDA_CHECK(cudaMemcpy(skel_out + off, H.J[l].p + nd.koff, nd.k * sizeof(int64_t), cudaMemcpyDeviceToHost));
          off += nd.k;
        }
    }
  });
}

int hss_node(hss_t Hh, int32_t node, int32_t* rows, int32_t* k, double* U, double* B, double* D) {
  return guarded([&] {
    require(Hh != nullptr, "hss_node: NULL handle");
    const HSSImpl& H = *Hh->impl;
    const int nn = (1 << (H.L + 1)) - 1;
    require(node >= 0 && node < nn, "hss_node: node id out of range");
    int l = 0;
    while (((1 << (l + 1)) - 1) <= node) ++l;
    const int i = node - ((1 << l) - 1);
    require(held(H, l, i) && (l != H.sh.lg || !H.sh.on() || i == H.sh.g),
            "hss_node: node is held by another rank");
    const NodeInfo& nd = H.lv[l][i];
    if (rows) *rows = nd.rows;
    if (k) *k = (l == 0) ? -1 : nd.k;
    if (U && l >= 1) {
      if (nd.pt) {
        for (int a = 0; a < nd.rows; ++a)
          for (int b = 0; b < nd.k; ++b) U[(int64_t)a * nd.k + b] = (a == b) ? 1.0 : 0.0;
      } else if (nd.k > 0) {
        CUDA_CHECK(cudaMemcpy(U, H.U[l].p + nd.uoff, (size_t)nd.rows * nd.k * 8, cudaMemcpyDeviceToHost));
      }
    }
    if (B && l < H.L) {
      const int ka = H.lv[l + 1][2 * i].k, kb = H.lv[l + 1][2 * i + 1].k;
      if (ka * kb > 0)
        CUDA_CHECK(cudaMemcpy(B, H.B[l].p + nd.boff, (size_t)ka * kb * 8, cudaMemcpyDeviceToHost));
    }
    if (D && l == H.L) {
      const int64_t m = nd.hi - nd.lo;
      CUDA_CHECK(cudaMemcpy(D, H.D.p + nd.doff, (size_t)m * m * 8, cudaMemcpyDeviceToHost));
    }
  });
}

int hss_matvec(hss_t Hh, const double* v, double* out, int32_t nrhs, void* stream) {
  return guarded([&] {
    StreamScope ss__((cudaStream_t)stream);
    require(Hh && v && out, "hss_matvec: NULL pointer");
    require(nrhs >= 1, "hss_matvec: nrhs must be >= 1");
    const HSSImpl& H = *Hh->impl;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nl = H.nloc();
    DevBuf<double> a((size_t)std::max<int64_t>(1, nl) * nrhs), b((size_t)std::max<int64_t>(1, nl) * nrhs),
        full((size_t)H.n * nrhs);
    gather_rows(v, H.perm.p + H.lo_g, nl, nrhs, a.p, s);
    hss_matvec_tree(H, a.p, b.p, nrhs, s);
    gather_points(H, b.p, nrhs, full.p, s);
    scatter_rows(full.p, H.perm.p, H.n, nrhs, out, s);
    CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

int hss_ulv_factor(hss_t Hh, double beta, void* stream, ulv_t* out) {
  return guarded([&] {
    StreamScope ss__((cudaStream_t)stream);
    require(Hh && out, "hss_ulv_factor: NULL pointer");
    require(std::isfinite(beta) && beta > 0, "hss_ulv_factor: beta must be > 0");
    auto* F = new ULVImpl();
    F->H = Hh->impl;
    F->H->refs.fetch_add(1);
    F->beta = beta;
    try {
      ulv_factor_impl(*F, (cudaStream_t)stream);
    } catch (...) {
      release_hss(F->H);
      delete F;
      throw;
    }
    handle_acquired();
    *out = new ulv_s{F, cur_device()};
  });
}

int ulv_info(ulv_t U, ulv_stats* st) {
  return guarded([&] {
    require(U && st, "ulv_info: NULL pointer");
    *st = U->impl->st;
  });
}

int ulv_solve(ulv_t Uh, const double* b, double* x, int32_t nrhs, void* stream) {
  return guarded([&] {
    StreamScope ss__((cudaStream_t)stream);
    require(Uh && b && x, "ulv_solve: NULL pointer");
    require(nrhs >= 1, "ulv_solve: nrhs must be >= 1");
    const ULVImpl& F = *Uh->impl;
    const HSSImpl& H = *F.H;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nl = H.nloc();
    DevBuf<double> bt((size_t)std::max<int64_t>(1, nl) * nrhs), xt((size_t)std::max<int64_t>(1, nl) * nrhs),
        full((size_t)H.n * nrhs);
    gather_rows(b, H.perm.p + H.lo_g, nl, nrhs, bt.p, s);
    CUDA_CHECK(cudaStreamSynchronize(s));  // b and x may alias
    // the sweep kernels take up to 8 right-hand sides: groups of 8 columns
    for (int c0 = 0; c0 < nrhs; c0 += 8) {
      const int w = std::min(8, nrhs - c0);
      SolveWS ws;
      solve_ws_alloc(F, w, ws);
      if (nl > 0)
        CUDA_CHECK(cudaMemcpy2DAsync(ws.fin[H.L], w * 8, bt.p + c0, nrhs * 8, w * 8, nl, cudaMemcpyDeviceToDevice, s));
      ulv_solve_tree(F, ws, s);
      if (nl > 0)
        CUDA_CHECK(cudaMemcpy2DAsync(xt.p + c0, nrhs * 8, ws.xout[H.L], w * 8, w * 8, nl, cudaMemcpyDeviceToDevice, s));
      CUDA_CHECK(cudaStreamSynchronize(s));
    }
    gather_points(H, xt.p, nrhs, full.p, s);
    scatter_rows(full.p, H.perm.p, H.n, nrhs, x, s);
    CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

int admm_svm_train(ulv_t Uh, const double* y, const double* C, int32_t nC, int32_t max_it,
                   const admm_opts* opt, double* z_out, double* mu_out, double* bias_out,
                   double* obj_out, admm_stats* st, void* stream) {
  return guarded([&] {
    StreamScope ss__((cudaStream_t)stream);
    require(Uh && y && C && z_out, "admm_svm_train: NULL pointer");
    require(nC >= 1, "admm_svm_train: nC must be >= 1");
    require(max_it >= 1, "admm_svm_train: max_it must be >= 1");
    std::vector<double> Cs(C, C + nC);
    for (double c : Cs) require(std::isfinite(c) && c > 0, "admm_svm_train: every C must be > 0");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = Uh->impl->H->n;
    if (nC <= 8) {
      AdmmResult r = admm_train_impl(*Uh->impl, y, Cs, max_it, opt, z_out, mu_out, bias_out, obj_out, s);
      if (st) {
        st->w1 = r.w1; st->ms_precompute = r.ms_pre; st->ms_loop = r.ms_loop; st->ms_bias = r.ms_bias;
        st->iterations = max_it; st->graph = r.graph; st->kernel_launches_per_iter = r.launches;
      }
      return;
    }
    // groups of at most 8 problems (the sweep kernels' widest right-hand side); each group is an
    // independent ADMM run, its outputs copied into its columns of the nC-wide outputs
    const int te = (opt && opt->trace_every > 0) ? opt->trace_every : 0;
    const int64_t ntr = te ? (max_it + te - 1) / te : 0;
    if (st) *st = admm_stats{};
    for (int c0 = 0; c0 < nC; c0 += 8) {
      const int w = std::min(8, nC - c0);
      std::vector<double> Cg(Cs.begin() + c0, Cs.begin() + c0 + w), bg(w), og(w);
      DevBuf<double> zg((size_t)n * w), mg(mu_out ? (size_t)n * w : 0);
      DevBuf<double> tz((te && opt->trace_z) ? (size_t)ntr * n * w : 0), tm((te && opt->trace_mu) ? (size_t)ntr * n * w : 0);
      admm_opts og_opt{};
      if (opt) og_opt = *opt;
      og_opt.trace_z = tz.p;
      og_opt.trace_mu = tm.p;
      AdmmResult r = admm_train_impl(*Uh->impl, y, Cg, max_it, &og_opt, zg.p, mu_out ? mg.p : nullptr,
                                     bg.data(), og.data(), s);
      auto put = [&](double* dst, const double* src, int64_t rows) {
        CUDA_CHECK(cudaMemcpy2DAsync(dst + c0, (size_t)nC * 8, src, (size_t)w * 8, (size_t)w * 8, rows,
                                     cudaMemcpyDeviceToDevice, s));
      };
      put(z_out, zg.p, n);
      if (mu_out) put(mu_out, mg.p, n);
      if (tz.p) put(opt->trace_z, tz.p, ntr * n);
      if (tm.p) put(opt->trace_mu, tm.p, ntr * n);
      CUDA_CHECK(cudaStreamSynchronize(s));
      for (int c = 0; c < w; ++c) {
        if (bias_out) bias_out[c0 + c] = bg[c];
        if (obj_out) obj_out[c0 + c] = og[c];
      }
      if (st) {
        st->w1 = r.w1; st->ms_precompute += r.ms_pre; st->ms_loop += r.ms_loop; st->ms_bias += r.ms_bias;
        st->iterations = max_it; st->graph = r.graph; st->kernel_launches_per_iter += r.launches;
      }
    }
  });
}

int svm_predict(const double* Ftrain, const double* y, const double* z, int64_t n, int32_t r, double h,
                const double* bias, int32_t nC, const double* Ftest, int64_t m, double* dv_out,
                int8_t* label_out, hss_comm_t comm, void* stream) {
  return guarded([&] {
    StreamScope ss__((cudaStream_t)stream);
    require(Ftrain && y && z && bias && (Ftest || m == 0), "svm_predict: NULL pointer");
    require(n >= 1 && r >= 1 && m >= 0, "svm_predict: bad sizes");
    require(nC >= 1 && nC <= 16, "svm_predict: nC must be in 1..16");
    require(std::isfinite(h) && h > 0, "svm_predict: h must be > 0");
    if (m == 0) return;
    predict_impl(Ftrain, y, z, n, r, h, bias, nC, Ftest, m, dv_out, label_out, comm ? comm->c.get() : nullptr,
                 (cudaStream_t)stream);
  });
}

int svm_train_predict_host(const double* F, const double* y, int64_t n, int32_t r, double h,
                           const hss_opts* opt, double beta, const double* C, int32_t nC,
                           int32_t max_it, const double* Ftest, int64_t m, double* z_out,
                           double* bias_out, double* obj_out, int8_t* labels_out,
                           double* timings_ms) {
  return guarded([&] {
    require(F && y && C && z_out, "svm_train_predict_host: NULL pointer");
    require(nC >= 1 && nC <= 8, "svm_train_predict_host: nC must be in 1..8");
    require(!(labels_out && m > 0) || Ftest, "svm_train_predict_host: NULL Ftest");
    validate_opts(opt, n, r, h);
    cudaStream_t s;
    CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct SG { cudaStream_t s; ~SG() { cudaStreamSynchronize(s); cudaStreamDestroy(s); } } sg{s};
    StreamScope ss__(s);
    cudaEvent_t ev[8];
    for (auto& e : ev) CUDA_CHECK(cudaEventCreate(&e));
    struct EG { cudaEvent_t* e; ~EG() { for (int i = 0; i < 8; ++i) cudaEventDestroy(e[i]); } } eg{ev};
    CUDA_CHECK(cudaEventRecord(ev[0], s));
    DevBuf<double> dF((size_t)n * r), dy(n), dFt((size_t)std::max<int64_t>(1, m) * r);
    DevBuf<double> dz((size_t)n * nC);
    DevBuf<int8_t> dl((size_t)std::max<int64_t>(1, m) * nC);
    h2d(dF.p, F, (size_t)n * r, s);
    h2d(dy.p, y, n, s);
    if (labels_out && m > 0) h2d(dFt.p, Ftest, (size_t)m * r, s);
    CUDA_CHECK(cudaEventRecord(ev[1], s));
    HSSImpl* H = build_adaptive(dF.p, n, r, h, *opt, comm_of(opt), s);
    struct HG { HSSImpl* h; ~HG() { release_hss(h); } } hg{H};
    CUDA_CHECK(cudaEventRecord(ev[2], s));
    ULVImpl Fz;
    Fz.H = H;
    Fz.beta = beta;
    require(std::isfinite(beta) && beta > 0, "beta must be > 0");
    ulv_factor_impl(Fz, s);
    CUDA_CHECK(cudaEventRecord(ev[3], s));
    std::vector<double> Cs(C, C + nC), bias(nC), obj(nC);
    for (double c : Cs) require(std::isfinite(c) && c > 0, "every C must be > 0");
    AdmmResult ar = admm_train_impl(Fz, dy.p, Cs, max_it, nullptr, dz.p, nullptr, bias.data(), obj.data(), s);
    CUDA_CHECK(cudaEventRecord(ev[4], s));
    CUDA_CHECK(cudaEventRecord(ev[5], s));
    if (labels_out && m > 0)
      predict_impl(dF.p, dy.p, dz.p, n, r, h, bias.data(), nC, dFt.p, m, nullptr, dl.p, comm_of(opt).get(), s);
    CUDA_CHECK(cudaEventRecord(ev[6], s));
    d2h(z_out, dz.p, (size_t)n * nC, s);
    if (labels_out && m > 0) d2h(labels_out, dl.p, (size_t)m * nC, s);
    CUDA_CHECK(cudaEventRecord(ev[7], s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    for (int c = 0; c < nC; ++c) {
      if (bias_out) bias_out[c] = bias[c];
      if (obj_out) obj_out[c] = obj[c];
    }
    if (timings_ms) {
      float t;
      CUDA_CHECK(cudaEventElapsedTime(&t, ev[0], ev[1])); timings_ms[0] = t;
      CUDA_CHECK(cudaEventElapsedTime(&t, ev[1], ev[2])); timings_ms[1] = t;
      CUDA_CHECK(cudaEventElapsedTime(&t, ev[2], ev[3])); timings_ms[2] = t;
      timings_ms[3] = ar.ms_pre + ar.ms_loop;
      timings_ms[4] = ar.ms_bias;
      CUDA_CHECK(cudaEventElapsedTime(&t, ev[5], ev[6])); timings_ms[5] = t;
      CUDA_CHECK(cudaEventElapsedTime(&t, ev[6], ev[7])); timings_ms[6] = t;
      CUDA_CHECK(cudaEventElapsedTime(&t, ev[0], ev[7])); timings_ms[7] = t;
    }
  });
}

int hss_ann_lists(const double* F, int64_t n, int32_t r, int32_t kappa, int32_t trees, int32_t leaf,
                  uint64_t seed, int64_t* idx_out, double* d_out, void* stream) {
  return guarded([&] {
    StreamScope ss__((cudaStream_t)stream);
    require(F && idx_out && d_out, "hss_ann_lists: NULL pointer");
    require(n >= 1 && r >= 1, "hss_ann_lists: bad sizes");
    cudaStream_t s = (cudaStream_t)stream;
    const int rp = (r + 3) / 4 * 4;
    DevBuf<double> Fpad((size_t)n * rp);
    pad_rows(F, n, r, rp, Fpad.p, s);
    ann_build(Fpad.p, n, r, rp, kappa, trees, leaf, seed, idx_out, d_out, s);
  });
}

int hss_omega(uint64_t seed, const int64_t* idx, int64_t rows, int32_t s, double* out, void* stream) {
  return guarded([&] {
    StreamScope ss__((cudaStream_t)stream);
    require(idx && out, "hss_omega: NULL pointer");
    require(rows >= 0 && s >= 1 && s <= (1 << 20), "hss_omega: bad sizes");
    omega_rows(seed, idx, rows, s, out, (cudaStream_t)stream);
    CUDA_CHECK(cudaStreamSynchronize((cudaStream_t)stream));
  });
}

int hss_tree(const double* F, int64_t n, int32_t r, int32_t leaf_size, uint64_t tree_seed,
             int64_t* perm_out, void* stream) {
  return guarded([&] {
    StreamScope ss__((cudaStream_t)stream);
    require(F && perm_out, "hss_tree: NULL pointer");
    require(n >= 1 && r >= 1 && leaf_size >= 1, "hss_tree: bad sizes");
    cudaStream_t s = (cudaStream_t)stream;
    const int rp = (r + 3) / 4 * 4;
    DevBuf<double> Fpad((size_t)n * rp);
    pad_rows(F, n, r, rp, Fpad.p, s);
    build_tree(Fpad.p, n, r, rp, leaf_size, tree_seed, perm_out, nullptr, s);
  });
}

int hss_kernel_matmul(const double* Fa, int64_t na, const double* Fb, int64_t nb, int32_t r,
                      double h, const double* W, int32_t ncols, int32_t same_set, double* S,
                      void* stream) {
  return guarded([&] {
    StreamScope ss__((cudaStream_t)stream);
    require(Fa && Fb && W && S, "hss_kernel_matmul: NULL pointer");
    require(na >= 0 && nb >= 0 && r >= 1 && ncols >= 1, "hss_kernel_matmul: bad sizes");
    require(std::isfinite(h) && h > 0, "hss_kernel_matmul: h must be > 0");
    cudaStream_t s = (cudaStream_t)stream;
    const int rp = (r + 3) / 4 * 4;
    const int ncp = (ncols + 1) / 2 * 2;
    DevBuf<double> A((size_t)std::max<int64_t>(1, na) * rp), Bm((size_t)std::max<int64_t>(1, nb) * rp),
        nua(std::max<int64_t>(1, na) + kNormPad), nub(std::max<int64_t>(1, nb) + kNormPad);
    pad_rows(Fa, na, r, rp, A.p, s);
    pad_rows(Fb, nb, r, rp, Bm.p, s);
    row_norms(A.p, na, rp, nua.p, s);
    row_norms(Bm.p, nb, rp, nub.p, s);
    DevBuf<double> Wp, Sp;
    const double* Wuse = W;
    double* Suse = S;
    if (ncp != ncols) {  // pad to an even column count
      Wp.alloc((size_t)std::max<int64_t>(1, nb) * ncp);
      Sp.alloc((size_t)std::max<int64_t>(1, na) * ncp);
      CUDA_CHECK(cudaMemsetAsync(Wp.p, 0, Wp.bytes(), s));
      CUDA_CHECK(cudaMemcpy2DAsync(Wp.p, ncp * 8, W, ncols * 8, ncols * 8, nb, cudaMemcpyDeviceToDevice, s));
      Wuse = Wp.p;
      Suse = Sp.p;
    }
    KmmArgs a{};
    a.Fa = A.p; a.nua = nua.p; a.na = na;
    a.Fb = Bm.p; a.nub = nub.p; a.nb = nb;
    a.rp = rp; a.W = Wuse; a.ldw = ncp; a.ncols = ncp; a.S = Suse; a.lds = ncp;
    a.neg_inv_2h2 = -1.0 / (2.0 * h * h);
    a.same_set = same_set ? 1 : 0;
    kernel_matmul(a, s);
    if (ncp != ncols)
      CUDA_CHECK(cudaMemcpy2DAsync(S, ncols * 8, Sp.p, ncp * 8, ncols * 8, na, cudaMemcpyDeviceToDevice, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

int hss_kernel_block(const double* Fa, int64_t na, const double* Fb, int64_t nb, int32_t r, double h,
                     double* K, void* stream) {
  return guarded([&] {
    StreamScope ss__((cudaStream_t)stream);
    require(Fa && Fb && K, "hss_kernel_block: NULL pointer");
    require(na >= 0 && nb >= 0 && r >= 1 && na < (1 << 30) && nb < (1 << 30), "hss_kernel_block: bad sizes");
    cudaStream_t s = (cudaStream_t)stream;
    // stack both point sets in one array; columns index the second half
    DevBuf<double> A((size_t)std::max<int64_t>(1, na + nb) * r);
    CUDA_CHECK(cudaMemcpyAsync(A.p, Fa, (size_t)na * r * 8, cudaMemcpyDeviceToDevice, s));
    CUDA_CHECK(cudaMemcpyAsync(A.p + (size_t)na * r, Fb, (size_t)nb * r * 8, cudaMemcpyDeviceToDevice, s));
    std::vector<KblkProb> p = {{(int)na, (int)nb, nullptr, 0, nullptr, na, K, nb, 0.0}};
    kernel_blocks(A.p, r, r, h, p, s);
    CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

int hss_comm_nccl_id(void* unique_id_out) {
  return guarded([&] {
    require(unique_id_out != nullptr, "hss_comm_nccl_id: NULL pointer");
    nccl_unique_id(unique_id_out);
  });
}

int hss_comm_init_nccl(int32_t nranks, int32_t rank, const void* unique_id, hss_comm_t* out) {
  return guarded([&] {
    require(out && unique_id, "hss_comm_init_nccl: NULL pointer");
    require(nranks >= 1 && rank >= 0 && rank < nranks, "hss_comm_init_nccl: bad rank / nranks");
    *out = new hss_comm_s{make_nccl_comm(nranks, rank, unique_id)};
  });
}

int hss_comm_init_host(int32_t nranks, int32_t rank, hss_allgather_fn fn, void* ctx, hss_comm_t* out) {
  return guarded([&] {
    require(out && fn, "hss_comm_init_host: NULL pointer");
    require(nranks >= 1 && rank >= 0 && rank < nranks, "hss_comm_init_host: bad rank / nranks");
    *out = new hss_comm_s{make_host_comm(nranks, rank, fn, ctx)};
  }, /*need_device=*/false);
}

void hss_comm_free(hss_comm_t c) { delete c; }

int hss_comm_info(hss_comm_t c, int32_t* nranks, int32_t* rank, int32_t* device_api) {
  return guarded([&] {
    require(c != nullptr, "hss_comm_info: NULL comm");
    if (nranks) *nranks = c->c->size;
    if (rank) *rank = c->c->rank;
    if (device_api) *device_api = c->c->device_api() ? 1 : 0;
  }, /*need_device=*/false);
}

int hss_comm_exchange_test(hss_comm_t c, const double* send, int64_t count, double* recv, void* stream) {
  return guarded([&] {
    StreamScope ss__((cudaStream_t)stream);
    require(c && send && recv, "hss_comm_exchange_test: NULL pointer");
    require(count >= 1, "hss_comm_exchange_test: count must be >= 1");
    Comm& C = *c->c;
    cudaStream_t s = (cudaStream_t)stream;
    const int P = C.size;
    if (!C.device_api()) {
      C.allgather(send, recv, (size_t)count * sizeof(double), s);
      CUDA_CHECK(cudaStreamSynchronize(s));
      return;
    }
    // the level-lg exchange kernel with a trivial layout: rank p's `count` values at p * count
    std::vector<int64_t> ko(P), kk(P, count);
    for (int p = 0; p < P; ++p) ko[p] = (int64_t)p * count;
    auto dko = upload(ko, s), dkk = upload(kk, s);
    CUDA_CHECK(cudaMemcpyAsync(recv + (int64_t)C.rank * count, send, (size_t)count * sizeof(double),
                               cudaMemcpyDeviceToDevice, s));
    DevWindow w = C.window_alloc((size_t)P * count * sizeof(double));
    struct WG { Comm& c; DevWindow& w; ~WG() { c.window_free(w); } } wg{C, w};
    ExchangeArgs a{recv, (int64_t)C.rank * count, (int)count, 1, 0, (int)count, nullptr, nullptr, dko.p, dkk.p, count};
    C.device_exchange(w, a, s);
    C.device_exchange(w, a, s);   // twice: both window halves
    CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

void hss_free(hss_t H) {
  if (!H) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(H->dev);  // device buffers are released on their own device
  release_hss(H->impl);
  cudaSetDevice(prev);
  handle_released(H->dev);
  delete H;
}

void ulv_free(ulv_t U) {
  if (!U) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(U->dev);
  HSSImpl* H = U->impl->H;
  delete U->impl;
  release_hss(H);
  cudaSetDevice(prev);
  handle_released(U->dev);
  delete U;
}

int hss_pool_trim(void) {
  return guarded([&] {
    const int dev = cur_device();
    cudaMemPool_t pool = lib_pool();
    CUDA_CHECK(cudaDeviceSynchronize());
    CUDA_CHECK(cudaMemPoolTrimTo(pool, 0));
    std::lock_guard<std::mutex> g(g_pool_mu);
    g_reserved[dev] = 0;
  });
}

}  // extern "C"
