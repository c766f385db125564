// shard.cu — subtree-sharding exchanges and cluster-tree-ordered reductions.
//
// Every reduction of a per-point quantity (w^T q, e^T v, the bias sums) is done leaf by leaf
// and then pairwise up the cluster tree: leaf partials -> subtree root (owner rank) ->
// exchange of the P subtree-root values -> pairwise over the top levels.  The association
// order is the tree's, whatever P is, so results are bitwise identical for P = 1, 2, 4, 8.
#include "internal.cuh"

namespace svmhss {

// in-place pairwise reduction of nl rows of ncols values: row 0 <- total (a[i] += a[i + st]
// for i = 0 mod 2 st, i + st < nl: the cluster tree's association for any nl)
__device__ void pairwise_rows(double* a, int nl, int ncols) {
  for (int st = 1; st < nl; st <<= 1) {
    const int npair = (nl + 2 * st - 1) / (2 * st);
    for (int e = threadIdx.x; e < npair * ncols; e += blockDim.x) {
      const int i = (e / ncols) * 2 * st, c = e % ncols;
      if (i + st < nl) a[(int64_t)i * ncols + c] += a[(int64_t)(i + st) * ncols + c];
    }
    __syncthreads();
  }
}

__global__ void tree_reduce_kernel(double* part, int nl, int ncols, double* out) {
  pairwise_rows(part, nl, ncols);
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) out[c] = part[c];
}

constexpr int kTopMax = 4096;  // P * ncols values reduced in shared memory
__global__ void tree_reduce_top_kernel(const double* in, int nl, int ncols, double* out) {
  __shared__ double tmp[kTopMax];
  for (int e = threadIdx.x; e < nl * ncols; e += blockDim.x) tmp[e] = in[e];
  __syncthreads();
  pairwise_rows(tmp, nl, ncols);
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) out[c] = tmp[c];
}

void tree_reduce_local(const HSSImpl& H, double* part, int ncols, double* out, cudaStream_t s) {
  const int nl = H.sh.last(H.L) - H.sh.first(H.L);
  tree_reduce_kernel<<<1, 256, 0, s>>>(part, nl, ncols, out);
  LAUNCH_CHECK();
}

void tree_reduce_top(int P, const double* in, int ncols, double* out, cudaStream_t s) {
  require(P * ncols <= kTopMax, "tree_reduce_top: too many values");
  tree_reduce_top_kernel<<<1, 256, 0, s>>>(in, P, ncols, out);
  LAUNCH_CHECK();
}

void tree_reduce_all(const HSSImpl& H, double* part, int ncols, double* host_out, cudaStream_t s) {
  DevBuf<double> sub(ncols), all((size_t)H.sh.P * ncols), tot(ncols);
  tree_reduce_local(H, part, ncols, sub.p, s);
  if (H.sh.on()) {
    H.sh.comm->allgather(sub.p, all.p, (size_t)ncols * sizeof(double), s);
    tree_reduce_top(H.sh.P, all.p, ncols, tot.p, s);
    d2h(host_out, tot.p, ncols, s);
  } else {
    d2h(host_out, sub.p, ncols, s);
  }
  CUDA_CHECK(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------------ level-lg exchange
void exch_ws_alloc(const HSSImpl& H, int ncols, int nextra, ExchWS& ws) {
  ws.ncols = ncols;
  ws.nextra = nextra;
  ws.slot = (int64_t)H.kmax_lg * ncols + nextra;
  if (H.sh.on() && H.sh.comm->device_api()) {  // N3: symmetric window (collective allocation)
    ws.comm = H.sh.comm;
    ws.win = ws.comm->window_alloc((size_t)std::max<int64_t>(1, ws.slot * H.sh.P) * sizeof(double));
    return;
  }
  ws.send.alloc(std::max<int64_t>(1, ws.slot));
  ws.recv.alloc(std::max<int64_t>(1, ws.slot * H.sh.P));
}

// buf[(koff_p + i) * ncols + c] = recv[p * slot + i * ncols + c]; extra_out[p * nextra + e]
__global__ void exch_unpack_kernel(const double* __restrict__ recv, int64_t slot, int P, int ncols,
                                   int nextra, int kmax, const int64_t* __restrict__ koff,
                                   const int64_t* __restrict__ kk, double* __restrict__ buf,
                                   double* __restrict__ extra_out) {
  const int p = blockIdx.y;
  const double* src = recv + p * slot;
  const int64_t cnt = kk[p] * ncols;
  double* dst = buf + koff[p] * ncols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < cnt; e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = src[e];
  if (blockIdx.x == 0 && extra_out)
    for (int e = threadIdx.x; e < nextra; e += blockDim.x) extra_out[p * nextra + e] = src[(int64_t)kmax * ncols + e];
}

void exchange_lg(const HSSImpl& H, ExchWS& ws, double* buf, const double* extra, double* extra_out,
                 cudaStream_t s) {
  if (!H.sh.on()) {
    if (extra && extra_out && ws.nextra)
      CUDA_CHECK(cudaMemcpyAsync(extra_out, extra, ws.nextra * sizeof(double), cudaMemcpyDeviceToDevice, s));
    return;
  }
  const auto& own = H.lv[H.sh.lg][H.sh.g];
  if (ws.win.win) {  // N3: pack -> NVLink stores into every peer's window -> LSA barrier -> unpack
    ExchangeArgs a{buf, own.koff, own.k, ws.ncols, ws.nextra, H.kmax_lg, extra, extra_out, H.lg_koff.p, H.lg_k.p,
                   ws.slot};
    H.sh.comm->device_exchange(ws.win, a, s);
    return;
  }
  if (own.k > 0)
    CUDA_CHECK(cudaMemcpyAsync(ws.send.p, buf + own.koff * ws.ncols, (size_t)own.k * ws.ncols * sizeof(double),
                               cudaMemcpyDeviceToDevice, s));
  if (ws.nextra && extra)
    CUDA_CHECK(cudaMemcpyAsync(ws.send.p + (int64_t)H.kmax_lg * ws.ncols, extra, ws.nextra * sizeof(double),
                               cudaMemcpyDeviceToDevice, s));
  H.sh.comm->allgather(ws.send.p, ws.recv.p, ws.slot * sizeof(double), s);
  const int64_t mx = (int64_t)H.kmax_lg * ws.ncols;
  dim3 grid((unsigned)std::max(1, std::min(64, ceil_div(std::max<int64_t>(1, mx), 256))), H.sh.P);
  exch_unpack_kernel<<<grid, 256, 0, s>>>(ws.recv.p, ws.slot, H.sh.P, ws.ncols, ws.nextra, H.kmax_lg,
                                          H.lg_koff.p, H.lg_k.p, buf, extra_out);
  LAUNCH_CHECK();
}

// ------------------------------------------------------------------ point vectors
__global__ void unpack_points_kernel(const double* __restrict__ recv, int64_t slot, int ncols,
                                     const int64_t* __restrict__ lo, const int64_t* __restrict__ cnt,
                                     double* __restrict__ full) {
  const int p = blockIdx.y;
  const int64_t tot = cnt[p] * ncols;
  const double* src = recv + p * slot;
  double* dst = full + lo[p] * ncols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = src[e];
}

void gather_points(const HSSImpl& H, const double* loc, int ncols, double* full, cudaStream_t s) {
  if (!H.sh.on()) {
    if (loc != full)
      CUDA_CHECK(cudaMemcpyAsync(full, loc, (size_t)H.n * ncols * sizeof(double), cudaMemcpyDeviceToDevice, s));
    return;
  }
  const int64_t slot = H.nmax_g * ncols;
  DevBuf<double> send(slot), recv(slot * H.sh.P);
  CUDA_CHECK(cudaMemcpyAsync(send.p, loc, (size_t)H.nloc() * ncols * sizeof(double), cudaMemcpyDeviceToDevice, s));
  H.sh.comm->allgather(send.p, recv.p, slot * sizeof(double), s);
  dim3 grid((unsigned)std::min<int64_t>(1024, ceil_div(slot, 256)), H.sh.P);
  unpack_points_kernel<<<grid, 256, 0, s>>>(recv.p, slot, ncols, H.rank_lo.p, H.rank_cnt.p, full);
  LAUNCH_CHECK();
  CUDA_CHECK(cudaStreamSynchronize(s));
}

}  // namespace svmhss
