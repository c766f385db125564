// ann.cu — HSS-ANN column sampling on the GPU (readings N1-N3 in
// DESIGN.md).  Every integer decision (trees, neighbour lists, sampled columns) is made in exact
// arithmetic so it matches the oracle bit for bit:
//   N1  `trees` random-projection trees (tree.cu, rp mode); candidates of a point = the other
//       points of its leaf in every tree; d(i, j) = sum_f (F[i,f] - F[j,f])^2 with each square
//       rounded before the add (__dmul_rn / __dadd_rn: no contraction); ANN(i) = the kappa
//       distinct candidates with the smallest (d, original index).
//   N2  per node: pairs (d(i, j), pos(j)) over its active rows' ANN lists, outside the node;
//       the first s distinct positions in (d, pos) order (= (min d, pos) order), random fill
//       from splitmix64 when fewer exist, sorted by position.
// Selection is a warp-wide repeated lexicographic argmin over register-resident candidates.
#include <algorithm>
#include "internal.cuh"

namespace svmhss {

constexpr int kAnnMaxC = 8;     // candidates per lane: leaves <= 256 points, T * kappa <= 256

// lexicographic (d, j) < (d2, j2)
__device__ __forceinline__ bool lex_less(double d, int64_t j, double d2, int64_t j2) {
  return d < d2 || (d == d2 && j < j2);
}

// warp: pick the kappa smallest distinct (d, j) among lane-held candidates (cd/cj, n_l each);
// out_d/out_j[0..kappa) sorted, padded with +inf / -1.  Same j => same d (distinctness).
__device__ void warp_topk(double (&cd)[kAnnMaxC], int64_t (&cj)[kAnnMaxC], int kappa,
                          double* __restrict__ out_d, int64_t* __restrict__ out_j) {
  const int lane = threadIdx.x & 31;
  for (int q = 0; q < kappa; ++q) {
    double bd = INFINITY;
    int64_t bj = INT64_MAX;
#pragma unroll
    for (int c = 0; c < kAnnMaxC; ++c)
      if (cj[c] >= 0 && lex_less(cd[c], cj[c], bd, bj)) { bd = cd[c]; bj = cj[c]; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, bd, o);
      const int64_t oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (lex_less(od, oj, bd, bj)) { bd = od; bj = oj; }
    }
    if (lane == 0) {
      out_d[q] = (bj == INT64_MAX) ? INFINITY : bd;
      out_j[q] = (bj == INT64_MAX) ? -1 : bj;
    }
    if (bj == INT64_MAX) {
      for (int q2 = q + 1 + lane; q2 < kappa; q2 += 32) { out_d[q2] = INFINITY; out_j[q2] = -1; }
      return;
    }
#pragma unroll
    for (int c = 0; c < kAnnMaxC; ++c)
      if (cj[c] == bj) cj[c] = -1;  // taken (all copies of j)
  }
}

// warp: the kappa smallest (d, j) among DISTINCT lane-held candidates (no repeated j), sorted,
// padded with +inf / -1 -- the same output as warp_topk.  The kappa-th smallest distance T is
// found by a radix select over the bits of d (non-negative doubles order as their bit patterns),
// candidates with d < T are taken, ties at T by increasing j, and the selected <= 64 pairs are
// ordered by a bitonic sort in shared memory (scratch: 64 (d, j) pairs per warp).
__device__ void warp_topk_select(double (&cd)[kAnnMaxC], int64_t (&cj)[kAnnMaxC], int kappa,
                                 double* __restrict__ out_d, int64_t* __restrict__ out_j,
                                 double* __restrict__ sd, int64_t* __restrict__ sj) {
  const int lane = threadIdx.x & 31;
  unsigned long long key[kAnnMaxC];
  int nv = 0;
#pragma unroll
  for (int c = 0; c < kAnnMaxC; ++c) {
    key[c] = (cj[c] >= 0) ? (unsigned long long)__double_as_longlong(cd[c]) : ~0ull;
    nv += (cj[c] >= 0) ? 1 : 0;
  }
  const int nvalid = __reduce_add_sync(0xffffffffu, (unsigned)nv);
  const int K = min(kappa, nvalid);
  int taken = 0;
  if (K > 0) {
    unsigned long long prefix = 0ull;
    int rem = K;
    for (int b = 62; b >= 0; --b) {   // bit 63 (sign) is 0 for every valid key
      const unsigned long long hi = ~((2ull << b) - 1ull);   // bits above b
      int cnt = 0;
#pragma unroll
      for (int c = 0; c < kAnnMaxC; ++c)
        cnt += (cj[c] >= 0 && (key[c] & hi) == prefix && !((key[c] >> b) & 1ull)) ? 1 : 0;
      cnt = (int)__reduce_add_sync(0xffffffffu, (unsigned)cnt);
      if (rem > cnt) { prefix |= (1ull << b); rem -= cnt; }
    }
    // prefix = T (the K-th smallest key); rem = how many candidates equal to T to take
    int pos = 0;   // compaction: this lane's selected entries go after the lower lanes' ones
    int mine = 0;
#pragma unroll
    for (int c = 0; c < kAnnMaxC; ++c) mine += (cj[c] >= 0 && key[c] < prefix) ? 1 : 0;
    pos = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, pos, o);
      if (lane >= o) pos += v;
    }
    pos -= mine;
    const int nless = __shfl_sync(0xffffffffu, pos + mine, 31);
#pragma unroll
    for (int c = 0; c < kAnnMaxC; ++c)
      if (cj[c] >= 0 && key[c] < prefix) { sd[pos] = cd[c]; sj[pos] = cj[c]; ++pos; }
    // ties at T: the rem smallest j (rare: usually rem = 1)
    int64_t last = -1;
    for (int q = 0; q < rem; ++q) {
      int64_t bj = INT64_MAX;
#pragma unroll
      for (int c = 0; c < kAnnMaxC; ++c)
        if (cj[c] >= 0 && key[c] == prefix && cj[c] > last && cj[c] < bj) bj = cj[c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const int64_t oj = __shfl_xor_sync(0xffffffffu, bj, o);
        bj = oj < bj ? oj : bj;
      }
      if (lane == 0) { sd[nless + q] = __longlong_as_double((long long)prefix); sj[nless + q] = bj; }
      last = bj;
    }
    taken = K;
  }
  __syncwarp();
  // bitonic sort of the first `taken` entries (padded to 64 with +inf) by (d, j)
  for (int e = lane; e < 64; e += 32)
    if (e >= taken) { sd[e] = INFINITY; sj[e] = INT64_MAX; }
  __syncwarp();
  for (int size = 2; size <= 64; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int e = lane; e < 64; e += 32) {
        const int partner = e ^ stride;
        if (partner > e) {
          const bool up = (e & size) == 0;
          const double d0 = sd[e], d1 = sd[partner];
          const int64_t j0 = sj[e], j1 = sj[partner];
          const bool gt = lex_less(d1, j1, d0, j0);   // (d0, j0) > (d1, j1)
          if (gt == up) { sd[e] = d1; sd[partner] = d0; sj[e] = j1; sj[partner] = j0; }
        }
      }
      __syncwarp();
    }
  }
  for (int q = lane; q < kappa; q += 32) {
    out_d[q] = (q < taken) ? sd[q] : INFINITY;
    out_j[q] = (q < taken) ? sj[q] : -1;
  }
  __syncwarp();
}

// Phase A (one tree): one CTA per leaf.  Ft: features in this tree's order (stride rp),
// perm: tree position -> original index.  cand rows are ORIGINAL indices.
__global__ void __launch_bounds__(512) ann_leaf_kernel(const double* __restrict__ Ft, int rp, int r,
                                                       const int64_t* __restrict__ perm,
                                                       const int64_t* __restrict__ leaf_lo,
                                                       int kappa, double* __restrict__ cand_d,
                                                       int64_t* __restrict__ cand_j, int xs_rows) {
  extern __shared__ double xs[];  // m x r, then 16 warps x 64 (d, j) selection scratch
  const int64_t lo = leaf_lo[blockIdx.x], hi = leaf_lo[blockIdx.x + 1];
  const int m = (int)(hi - lo), lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* scr_d = xs + (size_t)xs_rows * r;
  int64_t* scr_j = reinterpret_cast<int64_t*>(scr_d + 16 * 64);
  for (int e = threadIdx.x; e < m * r; e += blockDim.x) xs[e] = Ft[(lo + e / r) * rp + e % r];
  __syncthreads();
  const int nw = blockDim.x >> 5;
  for (int i = wid; i < m; i += nw) {
    double cd[kAnnMaxC];
    int64_t cj[kAnnMaxC];
#pragma unroll
    for (int c = 0; c < kAnnMaxC; ++c) {
      const int jj = lane + 32 * c;
      cj[c] = -1;
      cd[c] = INFINITY;
      if (jj < m && jj != i) {
        double d = 0.0;
        for (int f = 0; f < r; ++f) {
          const double t = xs[i * r + f] - xs[jj * r + f];
          d = __dadd_rn(d, __dmul_rn(t, t));
        }
        cd[c] = d;
        cj[c] = perm[lo + jj];
      }
    }
    const int64_t oi = perm[lo + i];
    if (kappa <= 64)
      warp_topk_select(cd, cj, kappa, cand_d + oi * kappa, cand_j + oi * kappa, scr_d + wid * 64, scr_j + wid * 64);
    else
      warp_topk(cd, cj, kappa, cand_d + oi * kappa, cand_j + oi * kappa);
  }
}

// Phase B: merge the T per-tree lists of a point (warp per point).
__global__ void __launch_bounds__(256) ann_merge_kernel(int64_t n, int T, int kappa,
                                                        const double* __restrict__ cand_d,
                                                        const int64_t* __restrict__ cand_j,
                                                        double* __restrict__ out_d, int64_t* __restrict__ out_j) {
  const int64_t i = blockIdx.x * 8LL + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  double cd[kAnnMaxC];
  int64_t cj[kAnnMaxC];
#pragma unroll
  for (int c = 0; c < kAnnMaxC; ++c) {
    const int e = lane + 32 * c;  // entry e of T * kappa: tree e / kappa, rank e % kappa
    cj[c] = -1;
    cd[c] = INFINITY;
    if (e < T * kappa) {
      const int64_t off = ((int64_t)(e / kappa) * n + i) * kappa + e % kappa;
      cj[c] = cand_j[off];
      cd[c] = cand_d[off];
    }
  }
  warp_topk(cd, cj, kappa, out_d + i * kappa, out_j + i * kappa);
}

void ann_build(const double* Fpad, int64_t n, int r, int rp, int kappa, int trees, int leaf, uint64_t seed,
               int64_t* idx_out, double* d_out, cudaStream_t s) {
  require(kappa >= 1 && trees >= 1 && leaf >= 2, "ann: kappa, trees >= 1 and leaf >= 2");
  require(leaf <= 32 * kAnnMaxC, "ann: ann_leaf must be <= 256");
  require((int64_t)trees * kappa <= 32 * kAnnMaxC, "ann: ann_trees * ann_neighbors must be <= 256");
  const size_t smem = ((size_t)leaf * r + 16 * 64 * 2) * sizeof(double);
  require(smem <= 227 * 1024, "ann: ann_leaf * features too large for shared memory (lower ann_leaf)");
  const int L = num_levels(n, leaf);
  std::vector<std::vector<std::pair<int64_t, int64_t>>> rg;
  node_ranges(n, L, rg);
  std::vector<int64_t> llo;
  for (auto& pr : rg[L]) llo.push_back(pr.first);
  llo.push_back(n);
  auto d_llo = upload(llo, s);
  const int nleaf = (int)rg[L].size();
  DevBuf<int64_t> perm(n), cj((size_t)trees * n * kappa);
  DevBuf<double> Ft((size_t)n * rp), cd((size_t)trees * n * kappa);
  if (smem > 48 * 1024)
    CUDA_CHECK(cudaFuncSetAttribute(ann_leaf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int t = 0; t < trees; ++t) {
    build_tree(Fpad, n, r, rp, leaf, seed, perm.p, Ft.p, s, t);
    ann_leaf_kernel<<<nleaf, 512, smem, s>>>(Ft.p, rp, r, perm.p, d_llo.p, kappa, cd.p + (size_t)t * n * kappa,
                                             cj.p + (size_t)t * n * kappa, leaf);
    LAUNCH_CHECK();
  }
  ann_merge_kernel<<<ceil_div(n, 8), 256, 0, s>>>(n, trees, kappa, cd.p, cj.p, d_out, idx_out);
  LAUNCH_CHECK();
  CUDA_CHECK(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------------ N2: sampled columns
// pairs of node segment g (node q of the level, rows x kappa slots from offset roff * kappa):
// key1 = d (or +inf when invalid), val = position (or INT64_MAX)
struct SampNode { int64_t lo, hi, roff; int rows, pad; };

__global__ void samp_pairs_kernel(const SampNode* __restrict__ nodes, int kappa, const int64_t* __restrict__ act,
                                  const int64_t* __restrict__ ann_pos, const double* __restrict__ ann_d,
                                  double* __restrict__ pd, int64_t* __restrict__ pq) {
  const SampNode N = nodes[blockIdx.x];
  const int64_t tot = (int64_t)N.rows * kappa;
  for (int64_t e = threadIdx.x; e < tot; e += blockDim.x) {
    const int64_t a = act[N.roff + e / kappa];  // tree position of the active row
    const int c = (int)(e % kappa);
    const int64_t q = ann_pos[a * kappa + c];
    const bool ok = q >= 0 && (q < N.lo || q >= N.hi);
    pd[N.roff * kappa + e] = ok ? ann_d[a * kappa + c] : INFINITY;
    pq[N.roff * kappa + e] = ok ? q : INT64_MAX;
  }
}

// after sorting each segment by (q, d): keep the first of every q run -> flag 1 (key = d),
// others -> key +inf and q = INT64_MAX (sorted to the end by the next pass)
__global__ void samp_unique_kernel(const SampNode* __restrict__ nodes, int kappa, double* __restrict__ pd,
                                   int64_t* __restrict__ pq, const double* __restrict__ sd,
                                   const int64_t* __restrict__ sq) {
  const SampNode N = nodes[blockIdx.x];
  const int64_t b = N.roff * kappa, tot = (int64_t)N.rows * kappa;
  for (int64_t e = threadIdx.x; e < tot; e += blockDim.x) {
    const int64_t q = sq[b + e];
    const bool first = q != INT64_MAX && (e == 0 || sq[b + e - 1] != q);
    pd[b + e] = first ? sd[b + e] : INFINITY;
    pq[b + e] = first ? q : INT64_MAX;
  }
}

// after sorting each segment by (dmin, q): the first min(s, count) valid positions, sorted by
// position (odd-even sort in shared memory), into C (node q at q * s); count -> cnt[q]
__global__ void __launch_bounds__(256) samp_take_kernel(const SampNode* __restrict__ nodes, int kappa, int s,
                                                        const int64_t* __restrict__ sq, int64_t* __restrict__ C,
                                                        int* __restrict__ cnt) {
  extern __shared__ int64_t cs[];  // s
  const SampNode N = nodes[blockIdx.x];
  const int64_t b = N.roff * kappa, tot = (int64_t)N.rows * kappa;
  __shared__ int nvalid;
  if (threadIdx.x == 0) nvalid = 0;
  __syncthreads();
  for (int e = threadIdx.x; e < s; e += blockDim.x) {
    const int64_t q = (e < tot) ? sq[b + e] : INT64_MAX;
    cs[e] = q;
    if (q != INT64_MAX) atomicAdd(&nvalid, 1);
  }
  __syncthreads();
  for (int ph = 0; ph < s; ++ph) {  // odd-even transposition sort (s <= 1152)
    for (int e = 2 * threadIdx.x + (ph & 1); e + 1 < s; e += 2 * blockDim.x)
      if (cs[e] > cs[e + 1]) { const int64_t t = cs[e]; cs[e] = cs[e + 1]; cs[e + 1] = t; }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < s; e += blockDim.x) C[(int64_t)blockIdx.x * s + e] = (cs[e] == INT64_MAX) ? -1 : cs[e];
  if (threadIdx.x == 0) cnt[blockIdx.x] = nvalid;
}

// Sampled columns for the nodes [f, e) of level l: C (nn x s tree positions, sorted; entries past
// the node's count are filled randomly (N2) or -1 if the complement is exhausted).
// act: row-packed active tree positions of the level (roff per node).
// Global radix formulation of the per-node column choice (same result as sorting each node's
// segment): key1 = node << QB | q (q = n for excluded pairs) -> radix sort (node, q); per
// (node, q) run the minimum d; key2 = bits of dmin (+inf for non-first / excluded) -> stable radix
// sort by dmin, then stable by node -> every node's segment ordered by (dmin, q).
__global__ void samp_keys_kernel(const SampNode* __restrict__ nodes, int kappa, const int64_t* __restrict__ act,
                                 const int64_t* __restrict__ ann_pos, const double* __restrict__ ann_d, int qb,
                                 int64_t n, uint64_t* __restrict__ key, double* __restrict__ pd) {
  const SampNode N = nodes[blockIdx.x];
  const int64_t tot = (int64_t)N.rows * kappa;
  for (int64_t e = threadIdx.x; e < tot; e += blockDim.x) {
    const int64_t a = act[N.roff + e / kappa];
    const int c = (int)(e % kappa);
    const int64_t q = ann_pos[a * kappa + c];
    const bool ok = q >= 0 && (q < N.lo || q >= N.hi);
    pd[N.roff * kappa + e] = ok ? ann_d[a * kappa + c] : INFINITY;
    key[N.roff * kappa + e] = ((uint64_t)blockIdx.x << qb) | (uint64_t)(ok ? q : n);
  }
}

// sorted by (node, q): run starts carry min d of the run; others +inf with q = n (node kept)
__global__ void samp_runmin_kernel(int64_t np, int qb, int64_t n, const uint64_t* __restrict__ key,
                                   const double* __restrict__ d, uint64_t* __restrict__ dkey,
                                   uint64_t* __restrict__ val) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= np) return;
  const uint64_t k = key[e];
  const uint64_t mask = (1ull << qb) - 1ull;
  const bool valid = (int64_t)(k & mask) != n;
  const bool first = valid && (e == 0 || key[e - 1] != k);
  double m = INFINITY;
  if (first) {
    m = d[e];
    for (int64_t f = e + 1; f < np && key[f] == k; ++f) m = fmin(m, d[f]);
  }
  dkey[e] = __double_as_longlong(m);            // non-negative doubles: bit order = value order
  val[e] = first ? k : ((k & ~mask) | (uint64_t)n);
}

__global__ void samp_nodekey_kernel(int64_t np, int qb, const uint64_t* __restrict__ val, unsigned* __restrict__ nk) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < np) nk[e] = (unsigned)(val[e] >> qb);
}

__global__ void samp_q_kernel(int64_t np, int qb, int64_t n, const uint64_t* __restrict__ val, int64_t* __restrict__ q) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= np) return;
  const int64_t v = (int64_t)(val[e] & ((1ull << qb) - 1ull));
  q[e] = (v == n) ? INT64_MAX : v;
}

static int bits_for(uint64_t v) { int b = 0; while (b < 63 && (1ull << b) <= v) ++b; return b; }

void ann_sample_level(const HSSImpl& H, int l, const int64_t* act, const int64_t* ann_pos, const double* ann_d,
                      int kappa, uint64_t seed, int64_t* C, cudaStream_t s) {
  const int f = H.sh.first(l), e = H.sh.last(l), nn = e - f, S = H.s;
  std::vector<SampNode> sn(nn);
  int64_t sumR = 0;
  for (int q = 0; q < nn; ++q) {
    const auto& nd = H.lv[l][f + q];
    sn[q] = {nd.lo, nd.hi, nd.roff, nd.rows, 0};
    sumR = std::max<int64_t>(sumR, nd.roff + nd.rows);
  }
  const int64_t np = std::max<int64_t>(1, sumR * kappa);
  auto dsn = upload(sn, s);
  const int64_t nall = H.n;
  const int qb = bits_for((uint64_t)nall);          // q in [0, n], n = excluded
  const int nb = bits_for((uint64_t)std::max(1, nn - 1));
  require(qb + nb <= 63, "ann_sample_level: key overflow");
  DevBuf<uint64_t> k1(np), k2(np), v1(np), v2(np);
  DevBuf<double> d1(np), d2(np);
  DevBuf<unsigned> nk1(np), nk2(np);
  DevBuf<int64_t> q1(np);
  if (sumR * kappa < np) {  // no rows (empty level): keep the tail defined
    CUDA_CHECK(cudaMemsetAsync(k1.p, 0, np * sizeof(uint64_t), s));
    CUDA_CHECK(cudaMemsetAsync(d1.p, 0, np * sizeof(double), s));
  }
  samp_keys_kernel<<<nn, 256, 0, s>>>(dsn.p, kappa, act, ann_pos, ann_d, qb, nall, k1.p, d1.p);
  LAUNCH_CHECK();
  // (node, q) order
  radix_sort_pairs(k1.p, k2.p, d1.p, d2.p, np, 0, qb + nb, s);
  const unsigned g = (unsigned)((np + 255) / 256);
  samp_runmin_kernel<<<g, 256, 0, s>>>(np, qb, nall, k2.p, d2.p, k1.p, v1.p);
  LAUNCH_CHECK();
  // stable by dmin, then stable by node: (node, dmin, q)
  radix_sort_pairs(k1.p, k2.p, v1.p, v2.p, np, 0, 64, s);
  samp_nodekey_kernel<<<g, 256, 0, s>>>(np, qb, v2.p, nk1.p);
  LAUNCH_CHECK();
  radix_sort_pairs(nk1.p, nk2.p, v2.p, v1.p, np, 0, std::max(1, nb), s);
  samp_q_kernel<<<g, 256, 0, s>>>(np, qb, nall, v1.p, q1.p);
  LAUNCH_CHECK();
  DevBuf<int> cnt(nn);
  samp_take_kernel<<<nn, 256, (size_t)S * sizeof(int64_t), s>>>(dsn.p, kappa, S, q1.p, C, cnt.p);
  LAUNCH_CHECK();
  std::vector<int> hc(nn);
  d2h(hc.data(), cnt.p, nn, s);
  CUDA_CHECK(cudaStreamSynchronize(s));
  // random fill (N2) on the host for the nodes short of min(s, n - w) columns
  const int64_t n = H.n;
  const uint64_t key = splitmix64(seed);
  std::vector<int64_t> row(S);
  for (int q = 0; q < nn; ++q) {
    const int64_t lo = sn[q].lo, hi = sn[q].hi, w = hi - lo;
    const int64_t target = std::min<int64_t>(S, n - w);
    if (hc[q] >= target) continue;
    d2h(row.data(), C + (int64_t)q * S, S, s);
    CUDA_CHECK(cudaStreamSynchronize(s));
    std::vector<int64_t> chosen(row.begin(), row.begin() + hc[q]);
    std::vector<int64_t> sorted = chosen;
    auto has = [&](int64_t p) { return std::binary_search(sorted.begin(), sorted.end(), p); };
    auto add = [&](int64_t p) {
      chosen.push_back(p);
      sorted.insert(std::upper_bound(sorted.begin(), sorted.end(), p), p);
    };
    const int64_t node_id = H.node_id(l, f + q);
    for (uint64_t d = 0; (int64_t)chosen.size() < target && d < 64ull * (uint64_t)S; ++d) {
      const uint64_t u = splitmix64(key + (uint64_t)node_id * (1ull << 20) + d);
      int64_t p = (int64_t)(u % (uint64_t)(n - w));
      if (p >= lo) p += w;
      if (!has(p)) add(p);
    }
    for (int64_t p = 0; (int64_t)chosen.size() < target; ++p)
      if ((p < lo || p >= hi) && !has(p)) add(p);
    for (int c = 0; c < S; ++c) row[c] = (c < (int)sorted.size()) ? sorted[c] : -1;
    h2d(C + (int64_t)q * S, row.data(), S, s);
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
}

// N3: Y_t = K(A_t, C_t) for every node of the level: W[(roff + i) * S + c] = K(act[roff + i], C[q*S + c])
// (direct differences summed in feature order, as kblock_kernel; columns with C = -1 are zero).
// One CTA per (node, 32 rows): the rows' features and 64 sampled columns' features at a time are
// staged in shared memory (odd row stride: conflict-free per-column reads); thread (c, i0) owns
// column c and rows i0, i0 + 4, ... (8 independent distance chains).
constexpr int AYR = 32, AYC = 64;

__global__ void __launch_bounds__(256) ann_y_kernel(const SampNode* __restrict__ nodes, const double* __restrict__ F,
                                                    int rp, int r, double neg_inv_2h2, int S,
                                                    const int64_t* __restrict__ act, const int64_t* __restrict__ C,
                                                    double* __restrict__ W) {
  const SampNode N = nodes[blockIdx.y];
  const int i0 = blockIdx.x * AYR;
  if (i0 >= N.rows) return;
  const int rs = r | 1;                      // odd stride
  extern __shared__ double ysm[];
  double* xa = ysm;                          // AYR x rs
  double* xc = ysm + AYR * rs;               // AYC x rs
  const int nr = min(AYR, N.rows - i0);
  for (int e = threadIdx.x; e < AYR * r; e += blockDim.x) {
    const int i = e / r, f = e % r;
    xa[i * rs + f] = (i < nr) ? F[act[N.roff + i0 + i] * rp + f] : 0.0;
  }
  const int64_t* Cq = C + (int64_t)blockIdx.y * S;
  const int c = threadIdx.x % AYC, ib = threadIdx.x / AYC;   // rows ib + 4 u
  for (int c0 = 0; c0 < S; c0 += AYC) {
    __syncthreads();
    for (int e = threadIdx.x; e < AYC * r; e += blockDim.x) {
      const int cc = e / r, f = e % r;
      const int64_t q = (c0 + cc < S) ? Cq[c0 + cc] : -1;
      xc[cc * rs + f] = (q >= 0) ? F[q * rp + f] : 0.0;
    }
    __syncthreads();
    if (c0 + c >= S) continue;
    const bool valid = Cq[c0 + c] >= 0;
    double d[AYR / 4];
#pragma unroll
    for (int u = 0; u < AYR / 4; ++u) d[u] = 0.0;
    for (int f = 0; f < r; ++f) {
      const double xv = xc[c * rs + f];
#pragma unroll
      for (int u = 0; u < AYR / 4; ++u) {
        const double t = xa[(ib + 4 * u) * rs + f] - xv;
        d[u] = fma(t, t, d[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < AYR / 4; ++u) {
      const int i = ib + 4 * u;
      if (i < nr) W[(N.roff + i0 + i) * (int64_t)S + c0 + c] = valid ? exp(d[u] * neg_inv_2h2) : 0.0;
    }
  }
}

void ann_y_level(const HSSImpl& H, int l, const int64_t* act, const int64_t* C, double* W, cudaStream_t s) {
  const int f = H.sh.first(l), e = H.sh.last(l), nn = e - f;
  std::vector<SampNode> sn(nn);
  int maxr = 1;
  for (int q = 0; q < nn; ++q) {
    const auto& nd = H.lv[l][f + q];
    sn[q] = {nd.lo, nd.hi, nd.roff, nd.rows, 0};
    maxr = std::max(maxr, nd.rows);
  }
  auto dsn = upload(sn, s);
  dim3 grid(ceil_div(maxr, AYR), nn);
  const size_t smem = (size_t)(AYR + AYC) * (H.r | 1) * sizeof(double);
  if (smem > 48 * 1024)
    CUDA_CHECK(cudaFuncSetAttribute(ann_y_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ann_y_kernel<<<grid, 256, smem, s>>>(dsn.p, H.Fp.p, H.rp, H.r, -1.0 / (2.0 * H.h * H.h), H.s, act, C, W);
  LAUNCH_CHECK();
  CUDA_CHECK(cudaStreamSynchronize(s));
}

// ann_pos[p * kappa + c] = iperm[idx[perm[p] * kappa + c]] (-1 kept), ann_dp likewise by position
__global__ void ann_to_tree_kernel(int64_t n, int kappa, const int64_t* __restrict__ perm,
                                   const int64_t* __restrict__ iperm, const int64_t* __restrict__ idx,
                                   const double* __restrict__ d, int64_t* __restrict__ pos,
                                   double* __restrict__ dp) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * kappa) return;
  const int64_t p = e / kappa;
  const int c = (int)(e % kappa);
  const int64_t o = perm[p] * kappa + c;
  const int64_t j = idx[o];
  pos[e] = (j >= 0) ? iperm[j] : -1;
  dp[e] = d[o];
}

void ann_to_tree(const HSSImpl& H, int kappa, const int64_t* idx, const double* d, int64_t* pos, double* dp,
                 cudaStream_t s) {
  ann_to_tree_kernel<<<ceil_div(H.n * kappa, 256), 256, 0, s>>>(H.n, kappa, H.perm.p, H.iperm.p, idx, d, pos, dp);
  LAUNCH_CHECK();
}

}  // namespace svmhss
