// sort.cu — stable LSD radix sort of (key, value) pairs (8-bit digits), used by the cluster tree
// (T3's stable order by (projection, original index) within every node, as three global sorts)
// and by HSS-ANN's per-node column choice (N2).  Per pass: a per-tile digit histogram
// (shared-memory counters), an exclusive scan of the digit-major (digit, tile) counts, and a
// stable scatter: inside a tile items are ranked in (round, warp, lane) order — the rank among
// equal digits within a warp from __match_any_sync, the warps' counts combined in warp order —
// so equal keys keep their input order and the result is deterministic.
#include "internal.cuh"

namespace svmhss {

constexpr int RS_THREADS = 256, RS_ROUNDS = 8, RS_TILE = RS_THREADS * RS_ROUNDS;

template <typename K>
__global__ void __launch_bounds__(RS_THREADS) rs_hist_kernel(const K* __restrict__ keys, int64_t n, int shift,
                                                             unsigned mask, unsigned* __restrict__ counts,
                                                             int64_t ntiles) {
  __shared__ unsigned h[256];
  h[threadIdx.x] = 0u;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * RS_TILE;
#pragma unroll
  for (int q = 0; q < RS_ROUNDS; ++q) {
    const int64_t i = base + q * RS_THREADS + threadIdx.x;
    if (i < n) atomicAdd(&h[(unsigned)(keys[i] >> shift) & mask], 1u);
  }
  __syncthreads();
  counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// exclusive scan, step 1: per block of 4096 counts, its total
__global__ void __launch_bounds__(256) rs_scan_part_kernel(const unsigned* __restrict__ c, int64_t total,
                                                           unsigned* __restrict__ part) {
  __shared__ unsigned red[256];
  const int64_t b0 = (int64_t)blockIdx.x * 4096;
  unsigned a = 0u;
  for (int64_t i = b0 + threadIdx.x; i < min(total, b0 + 4096); i += 256) a += c[i];
  red[threadIdx.x] = a;
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// step 2 (one CTA): exclusive scan of the block totals, in place
__global__ void __launch_bounds__(1024) rs_scan_top_kernel(unsigned* __restrict__ part, int nb) {
  __shared__ unsigned s[1024];
  unsigned carry = 0u;
  for (int b0 = 0; b0 < nb; b0 += 1024) {
    const int i = b0 + threadIdx.x;
    const unsigned v = i < nb ? part[i] : 0u;
    s[threadIdx.x] = v;
    __syncthreads();
    for (int st = 1; st < 1024; st <<= 1) {  // inclusive Hillis-Steele
      const unsigned t = threadIdx.x >= st ? s[threadIdx.x - st] : 0u;
      __syncthreads();
      s[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < nb) part[i] = carry + s[threadIdx.x] - v;
    const unsigned tot = s[1023];
    __syncthreads();
    carry += tot;
  }
}

// step 3: exclusive scan inside each block of 4096 counts, plus the block's offset
__global__ void __launch_bounds__(256) rs_scan_fin_kernel(unsigned* __restrict__ c, int64_t total,
                                                          const unsigned* __restrict__ part) {
  __shared__ unsigned s[256];
  const int64_t b0 = (int64_t)blockIdx.x * 4096;
  // each thread owns 16 consecutive counts
  const int64_t i0 = b0 + (int64_t)threadIdx.x * 16;
  unsigned loc[16], sum = 0u;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    loc[q] = (i0 + q < total) ? c[i0 + q] : 0u;
    sum += loc[q];
  }
  s[threadIdx.x] = sum;
  __syncthreads();
  for (int st = 1; st < 256; st <<= 1) {
    const unsigned t = threadIdx.x >= st ? s[threadIdx.x - st] : 0u;
    __syncthreads();
    s[threadIdx.x] += t;
    __syncthreads();
  }
  unsigned run = part[blockIdx.x] + s[threadIdx.x] - sum;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    if (i0 + q < total) c[i0 + q] = run;
    run += loc[q];
  }
}

template <typename K, typename V>
__global__ void __launch_bounds__(RS_THREADS) rs_scatter_kernel(const K* __restrict__ kin, const V* __restrict__ vin,
                                                                K* __restrict__ kout, V* __restrict__ vout, int64_t n,
                                                                int shift, unsigned mask,
                                                                const unsigned* __restrict__ offs, int64_t ntiles) {
  constexpr int NW = RS_THREADS / 32;
  __shared__ unsigned boff[256], run[256];
  __shared__ unsigned wc[NW][256];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  boff[tid] = offs[(int64_t)tid * ntiles + blockIdx.x];
  run[tid] = 0u;
  const int64_t base = (int64_t)blockIdx.x * RS_TILE;
  const unsigned lt = (1u << lane) - 1u;
  for (int q = 0; q < RS_ROUNDS; ++q) {
#pragma unroll
    for (int e = 0; e < NW; ++e) wc[e][tid] = 0u;
    __syncthreads();
    const int64_t i = base + q * RS_THREADS + tid;
    const bool valid = i < n;
    K k = 0;
    V v{};
    unsigned d = 0xFFFFu;
    if (valid) { k = kin[i]; v = vin[i]; d = (unsigned)(k >> shift) & mask; }
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const unsigned rank = __popc(peers & lt);
    if (valid && (peers & lt) == 0u) wc[w][d] = __popc(peers);  // the lowest lane of the group
    __syncthreads();
    if (valid) {
      unsigned o = boff[d] + run[d] + rank;
      for (int e = 0; e < w; ++e) o += wc[e][d];
      kout[o] = k;
      vout[o] = v;
    }
    __syncthreads();
    unsigned add = 0u;
#pragma unroll
    for (int e = 0; e < NW; ++e) add += wc[e][tid];
    run[tid] += add;
    __syncthreads();
  }
}

template <typename K, typename V>
static void radix_sort_impl(const K* kin, K* kout, const V* vin, V* vout, int64_t n, int begin_bit, int end_bit,
                            cudaStream_t s) {
  if (n <= 0) return;
  require(n < (int64_t)1 << 31, "radix_sort: n must be < 2^31");
  const int64_t ntiles = (n + RS_TILE - 1) / RS_TILE;
  const int64_t total = 256 * ntiles;
  const int64_t nblk = (total + 4095) / 4096;
  DevBuf<unsigned> cnt(total), part(nblk);
  DevBuf<K> kt(n);
  DevBuf<V> vt(n);
  const int npass = std::max(1, (end_bit - begin_bit + 7) / 8);
  // ping-pong so that the last pass writes kout / vout
  const K* ksrc = kin;
  const V* vsrc = vin;
  for (int pss = 0; pss < npass; ++pss) {
    const int shift = begin_bit + 8 * pss;
    const int bits = std::min(8, end_bit - shift);
    const unsigned mask = bits >= 8 ? 255u : ((1u << std::max(bits, 1)) - 1u);
    const bool to_out = ((npass - 1 - pss) % 2) == 0;
    K* kdst = to_out ? kout : kt.p;
    V* vdst = to_out ? vout : vt.p;
    rs_hist_kernel<K><<<(unsigned)ntiles, RS_THREADS, 0, s>>>(ksrc, n, shift, mask, cnt.p, ntiles);
    LAUNCH_CHECK();
    rs_scan_part_kernel<<<(unsigned)nblk, 256, 0, s>>>(cnt.p, total, part.p);
    LAUNCH_CHECK();
    rs_scan_top_kernel<<<1, 1024, 0, s>>>(part.p, (int)nblk);
    LAUNCH_CHECK();
    rs_scan_fin_kernel<<<(unsigned)nblk, 256, 0, s>>>(cnt.p, total, part.p);
    LAUNCH_CHECK();
    rs_scatter_kernel<K, V><<<(unsigned)ntiles, RS_THREADS, 0, s>>>(ksrc, vsrc, kdst, vdst, n, shift, mask, cnt.p,
                                                                      ntiles);
    LAUNCH_CHECK();
    ksrc = kdst;
    vsrc = vdst;
  }
}

void radix_sort_pairs(const uint64_t* kin, uint64_t* kout, const int* vin, int* vout, int64_t n, int begin_bit,
                      int end_bit, cudaStream_t s) {
  radix_sort_impl(kin, kout, vin, vout, n, begin_bit, end_bit, s);
}
void radix_sort_pairs(const unsigned* kin, unsigned* kout, const int* vin, int* vout, int64_t n, int begin_bit,
                      int end_bit, cudaStream_t s) {
  radix_sort_impl(kin, kout, vin, vout, n, begin_bit, end_bit, s);
}
void radix_sort_pairs(const uint64_t* kin, uint64_t* kout, const uint64_t* vin, uint64_t* vout, int64_t n,
                      int begin_bit, int end_bit, cudaStream_t s) {
  radix_sort_impl(kin, kout, vin, vout, n, begin_bit, end_bit, s);
}
void radix_sort_pairs(const unsigned* kin, unsigned* kout, const uint64_t* vin, uint64_t* vout, int64_t n,
                      int begin_bit, int end_bit, cudaStream_t s) {
  radix_sort_impl(kin, kout, vin, vout, n, begin_bit, end_bit, s);
}
void radix_sort_pairs(const uint64_t* kin, uint64_t* kout, const double* vin, double* vout, int64_t n,
                      int begin_bit, int end_bit, cudaStream_t s) {
  radix_sort_impl(kin, kout, vin, vout, n, begin_bit, end_bit, s);
}

}  // namespace svmhss
