// tree.cu — cluster tree by recursive PCA-median bisection on the GPU (readings T1-T4;
// P:72 "clustering ... preprocessing", P:180 hierarchical 2x2 partitioning).
//
// Per level (all nodes of the level at once, features kept in the current tree order):
//   chunk partial sums -> node means (fixed chunk order) -> chunk partial covariances ->
//   per-node reduction + 20 normalized power steps from the counter-RNG start vector ->
//   projections p_i = (f_i - c).v -> three stable global radix sorts (sort.cu: by original
//   index, by an order-preserving key of p, by node) = within every node the stable order by
//   (p, original index) -> permute rows.
#include "internal.cuh"

namespace svmhss {

int num_levels(int64_t n, int m) {
  int L = 0;
  while ((int64_t)m * ((int64_t)1 << L) < n) ++L;
  return L;
}

void node_ranges(int64_t n, int L, std::vector<std::vector<std::pair<int64_t, int64_t>>>& out) {
  out.assign(L + 1, {});
  out[0].push_back({0, n});
  for (int l = 0; l < L; ++l)
    for (auto& pr : out[l]) {
      const int64_t half = (pr.second - pr.first) / 2;
      out[l + 1].push_back({pr.first, pr.first + half});
      out[l + 1].push_back({pr.first + half, pr.second});
    }
}

struct Chunk { int node; int64_t lo, hi; };
constexpr int TREE_CHUNK = 2048;

// partial sums of features over a chunk
__global__ void chunk_sum_kernel(const double* __restrict__ F, int rp, int r,
                                 const Chunk* __restrict__ ch, double* __restrict__ part) {
  const Chunk c = ch[blockIdx.x];
  for (int f = threadIdx.x; f < r; f += blockDim.x) {
    double a = 0.0;
    for (int64_t i = c.lo; i < c.hi; ++i) a += F[i * rp + f];
    part[(int64_t)blockIdx.x * r + f] = a;
  }
}

// node mean = (sum of its chunk partials in chunk order) / count
__global__ void node_mean_kernel(const double* __restrict__ part, const int* __restrict__ cbeg,
                                 const int* __restrict__ cend, const int64_t* __restrict__ cnt,
                                 int r, double* __restrict__ mean) {
  const int nd = blockIdx.x;
  for (int f = threadIdx.x; f < r; f += blockDim.x) {
    double a = 0.0;
    for (int c = cbeg[nd]; c < cend[nd]; ++c) a += part[(int64_t)c * r + f];
    mean[(int64_t)nd * r + f] = a / (double)cnt[nd];
  }
}

// partial covariance over a chunk: sum (f-c)(f-c)^T, full r x r.  Thread = a 4 x 4 block of
// (a, b) pairs (register blocking: 8 shared loads per 16 FMAs); blockIdx.y selects a group of 256
// blocks.  Every pair accumulates its rows in order (32-row shared blocks in order), as before.
__global__ void __launch_bounds__(256) chunk_cov_kernel(const double* __restrict__ F, int rp, int r,
                                                        const Chunk* __restrict__ ch,
                                                        const double* __restrict__ mean,
                                                        double* __restrict__ part) {
  const Chunk c = ch[blockIdx.x];
  extern __shared__ double xs[];  // 32 x r4 centred rows (r4 = r rounded up to 4, zero padded)
  const int r4 = (r + 3) & ~3, nb4 = r4 / 4;
  const double* mu = mean + (int64_t)c.node * r;
  const int blk = blockIdx.y * 256 + threadIdx.x;
  const bool on = blk < nb4 * nb4;
  const int a0 = on ? (blk / nb4) * 4 : 0, b0 = on ? (blk % nb4) * 4 : 0;
  double acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
  for (int64_t i0 = c.lo; i0 < c.hi; i0 += 32) {
    const int nb = (int)min((int64_t)32, c.hi - i0);
    __syncthreads();
    for (int e = threadIdx.x; e < nb * r4; e += blockDim.x) {
      const int ii = e / r4, f = e % r4;
      xs[e] = (f < r) ? F[(i0 + ii) * rp + f] - mu[f] : 0.0;
    }
    __syncthreads();
    if (on) {
      for (int ii = 0; ii < nb; ++ii) {
        const double* x = xs + ii * r4;
        double xa[4], xb[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { xa[u] = x[a0 + u]; xb[u] = x[b0 + u]; }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = fma(xa[u], xb[v], acc[u][v]);
      }
    }
  }
  if (on) {
    const int npair = r * r;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (a0 + u < r && b0 + v < r) part[(int64_t)blockIdx.x * npair + (a0 + u) * r + b0 + v] = acc[u][v];
  }
}

// node covariance (chunk order) + power iteration; one CTA per node
__global__ void __launch_bounds__(256) node_dir_kernel(const double* __restrict__ part,
                                                       const int* __restrict__ cbeg,
                                                       const int* __restrict__ cend, int r,
                                                       uint64_t key, int id0,
                                                       double* __restrict__ dir) {
  const int nd = blockIdx.x;
  extern __shared__ double sh[];
  double* C = sh;            // r*r
  double* v = C + r * r;     // r
  double* w = v + r;         // r
  __shared__ double red[32];
  const int npair = r * r;
  for (int pr = threadIdx.x; pr < npair; pr += blockDim.x) {
    double a = 0.0;
    for (int c = cbeg[nd]; c < cend[nd]; ++c) a += part[(int64_t)c * npair + pr];
    C[pr] = a;
  }
  // v0 = normalized counter-RNG vector (R1-R3 with i = BFS node id, j = feature)
  double p = 0.0;
  for (int f = threadIdx.x; f < r; f += blockDim.x) {
    const double x = counter_gaussian(key, (uint64_t)(id0 + nd), (uint64_t)f);
    v[f] = x;
    p += x * x;
  }
  const double nv = sqrt(block_sum(p, red));
  for (int f = threadIdx.x; f < r; f += blockDim.x) v[f] /= nv;
  __syncthreads();
  for (int it = 0; it < 20; ++it) {
    double q = 0.0;
    for (int a = threadIdx.x; a < r; a += blockDim.x) {
      double s = 0.0;
      for (int b = 0; b < r; ++b) s = fma(C[a * r + b], v[b], s);
      w[a] = s;
      q += s * s;
    }
    const double nw = sqrt(block_sum(q, red));
    if (nw == 0.0) break;  // T2: keep v when Cv = 0
    for (int a = threadIdx.x; a < r; a += blockDim.x) v[a] = w[a] / nw;
    __syncthreads();
  }
  for (int f = threadIdx.x; f < r; f += blockDim.x) dir[(int64_t)nd * r + f] = v[f];
}

__device__ __forceinline__ uint64_t order_key(double p) {
  if (p == 0.0) p = 0.0;  // -0 -> +0
  uint64_t b = (uint64_t)__double_as_longlong(p);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void project_kernel(const double* __restrict__ F, int rp, int r, int64_t n,
                               const int* __restrict__ node_of, const double* __restrict__ mean,
                               const double* __restrict__ dir, uint64_t* __restrict__ key,
                               int* __restrict__ pos) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int nd = node_of[i];
  const double* mu = mean + (int64_t)nd * r;
  const double* v = dir + (int64_t)nd * r;
  double p = 0.0;
  for (int f = 0; f < r; ++f) p = fma(F[i * rp + f] - mu[f], v[f], p);
  key[i] = order_key(p);
  pos[i] = (int)i;
}

// N1: random-projection key p = sum_f s_f F[i, f] (features in order; s_f = +-1 from bit 63 of
// splitmix64(key_t + 2^20 * node_id + f)); s_f * x is exact, so the sum is the same with or
// without contraction.
__global__ void rp_project_kernel(const double* __restrict__ F, int rp, int r, int64_t n,
                                  const int* __restrict__ node_of, uint64_t key_t, int id0,
                                  uint64_t* __restrict__ key, int* __restrict__ pos) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t base = key_t + (uint64_t)(id0 + node_of[i]) * (1ull << 20);
  double p = 0.0;
  for (int f = 0; f < r; ++f) {
    const double x = F[i * rp + f];
    p = __dadd_rn(p, (splitmix64(base + (uint64_t)f) >> 63) ? -x : x);
  }
  key[i] = order_key(p);
  pos[i] = (int)i;
}

__global__ void gather_key_kernel(const uint64_t* __restrict__ key, const int* __restrict__ order,
                                  int64_t n, uint64_t* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = key[order[i]];
}

__global__ void node_key_kernel(const int* __restrict__ node_of_pos, const int* __restrict__ order, int64_t n,
                                unsigned* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = (unsigned)node_of_pos[order[i]];
}

static int bits_for(uint64_t v) { int b = 0; while (b < 63 && (1ull << b) <= v) ++b; return b; }

__global__ void permute_kernel(const double* __restrict__ F, const int64_t* __restrict__ idx,
                               const int* __restrict__ order, int64_t n, int rp,
                               double* __restrict__ F2, int64_t* __restrict__ idx2) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * rp) return;
  const int64_t i = e / rp;
  const int f = (int)(e % rp);
  const int64_t src = order[i];
  F2[e] = F[src * rp + f];
  if (f == 0) idx2[i] = idx[src];
}

__global__ void iota64_kernel(int64_t* a, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}

void build_tree(const double* Fpad, int64_t n, int r, int rp, int m, uint64_t tree_seed,
                int64_t* perm, double* Fp_out, cudaStream_t s, int rp_tree_index) {
  const int L = num_levels(n, m);
  require(n < ((int64_t)1 << 31), "tree: n must be < 2^31");
  std::vector<std::vector<std::pair<int64_t, int64_t>>> rg;
  node_ranges(n, L, rg);
  DevBuf<double> Fa(n * rp), Fb(n * rp);
  DevBuf<int64_t> ia(n), ib(n);
  CUDA_CHECK(cudaMemcpyAsync(Fa.p, Fpad, n * rp * sizeof(double), cudaMemcpyDeviceToDevice, s));
  iota64_kernel<<<ceil_div(n, 256), 256, 0, s>>>(ia.p, n);
  LAUNCH_CHECK();
  const uint64_t key = splitmix64(tree_seed);
  DevBuf<uint64_t> k1(n), k2(n);
  DevBuf<int> p1(n), p2(n), node_of(n);
  DevBuf<unsigned> nk1(n), nk2(n);
  DevBuf<int64_t> ik(n);
  for (int l = 0; l < L; ++l) {
    const auto& nodes = rg[l];
    const int nn = (int)nodes.size();
    std::vector<Chunk> ch;
    std::vector<int> cb(nn), ce(nn), nof(n);
    std::vector<int64_t> cnt(nn);
    for (int i = 0; i < nn; ++i) {
      cb[i] = (int)ch.size();
      for (int64_t lo = nodes[i].first; lo < nodes[i].second; lo += TREE_CHUNK)
        ch.push_back({i, lo, std::min(nodes[i].second, lo + TREE_CHUNK)});
      ce[i] = (int)ch.size();
      cnt[i] = nodes[i].second - nodes[i].first;
      for (int64_t p = nodes[i].first; p < nodes[i].second; ++p) nof[p] = i;
    }
    auto d_ch = upload(ch, s);
    auto d_cb = upload(cb, s), d_ce = upload(ce, s);
    auto d_cnt = upload(cnt, s);
    auto d_nof = upload(nof, s);
    if (rp_tree_index >= 0) {  // N1: random-projection tree
      rp_project_kernel<<<ceil_div(n, 256), 256, 0, s>>>(Fa.p, rp, r, n, d_nof.p,
                                                         splitmix64(tree_seed + (uint64_t)rp_tree_index),
                                                         (1 << l) - 1, k1.p, p1.p);
      LAUNCH_CHECK();
    } else {
    const int nch = (int)ch.size();
    DevBuf<double> part((size_t)nch * r * r), mean((size_t)nn * r), dir((size_t)nn * r);
    chunk_sum_kernel<<<nch, 128, 0, s>>>(Fa.p, rp, r, d_ch.p, part.p);
    LAUNCH_CHECK();
    node_mean_kernel<<<nn, 128, 0, s>>>(part.p, d_cb.p, d_ce.p, d_cnt.p, r, mean.p);
    LAUNCH_CHECK();
    {
      const int r4 = (r + 3) & ~3;
      size_t sm = 32 * (size_t)r4 * sizeof(double);
      dim3 gcov(nch, ceil_div((r4 / 4) * (r4 / 4), 256));
      if (sm > 48 * 1024)
        CUDA_CHECK(cudaFuncSetAttribute(chunk_cov_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      chunk_cov_kernel<<<gcov, 256, sm, s>>>(Fa.p, rp, r, d_ch.p, mean.p, part.p);
      LAUNCH_CHECK();
      size_t sm2 = ((size_t)r * r + 2 * r) * sizeof(double);
      if (sm2 > 48 * 1024)
        CUDA_CHECK(cudaFuncSetAttribute(node_dir_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
      node_dir_kernel<<<nn, 256, sm2, s>>>(part.p, d_cb.p, d_ce.p, r, key, (1 << l) - 1, dir.p);
      LAUNCH_CHECK();
    }
    project_kernel<<<ceil_div(n, 256), 256, 0, s>>>(Fa.p, rp, r, n, d_nof.p, mean.p, dir.p, k1.p, p1.p);
    LAUNCH_CHECK();
    }
    // order of positions within each node by (projection key, original index), as three global
    // stable radix sorts instead of per-node segmented sorts: by original index, by projection
    // key, then by node (node ranges are contiguous and in node order, so each node's positions
    // land in its own range)
    const int qb = std::max(1, bits_for((uint64_t)std::max<int64_t>(1, n - 1)));
    const int nbits = std::max(1, bits_for((uint64_t)std::max(1, nn - 1)));
    const uint64_t* iak = reinterpret_cast<const uint64_t*>(ia.p);
    uint64_t* ikk = reinterpret_cast<uint64_t*>(ik.p);
    // keys1 (the projection keys) must survive pass 1: keep a copy in k2 for the gather
    CUDA_CHECK(cudaMemcpyAsync(k2.p, k1.p, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
    radix_sort_pairs(iak, ikk, p1.p, p2.p, n, 0, qb, s);
    // p2 = positions ordered by original index; gather their projection keys
    gather_key_kernel<<<ceil_div(n, 256), 256, 0, s>>>(k2.p, p2.p, n, k1.p);
    LAUNCH_CHECK();
    radix_sort_pairs(k1.p, k2.p, p2.p, p1.p, n, 0, 64, s);
    node_key_kernel<<<ceil_div(n, 256), 256, 0, s>>>(d_nof.p, p1.p, n, nk1.p);
    LAUNCH_CHECK();
    radix_sort_pairs(nk1.p, nk2.p, p1.p, p2.p, n, 0, nbits, s);
    std::swap(p1, p2);   // final order of positions in p1
    permute_kernel<<<ceil_div(n * rp, 256), 256, 0, s>>>(Fa.p, ia.p, p1.p, n, rp, Fb.p, ib.p);
    LAUNCH_CHECK();
    std::swap(Fa, Fb);
    std::swap(ia, ib);
    CUDA_CHECK(cudaStreamSynchronize(s));  // host vectors above go out of scope
  }
  CUDA_CHECK(cudaMemcpyAsync(perm, ia.p, n * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  if (Fp_out)
    CUDA_CHECK(cudaMemcpyAsync(Fp_out, Fa.p, n * rp * sizeof(double), cudaMemcpyDeviceToDevice, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
}

}  // namespace svmhss
