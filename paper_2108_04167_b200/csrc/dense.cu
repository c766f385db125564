// dense.cu — batched small dense fp64 kernels (one problem = one HSS tree node).
//
//  bgemm   : FP64 tensor-core (DMMA) batched GEMM with arbitrary strides (sibling updates H4, Omega' = U^T Omega^,
//            R_a B R_b^T, Q^T D Q, the explicit solve operators of the ULV).
//  bpotrf  : left-looking Cholesky, one CTA per node (U: Dc_rr = L_r L_r^T; root).
//  btrsm   : blocked triangular solve with many right-hand sides (T = R11^-1 R12 in H3;
//            L_sr, G_r = L_r^-1 Q_r^T in U).
//  bgeqr2  : Householder QR (LAPACK dlarfg convention) of Ucur (U).
//  blarft  : compact-WY T factor (Q = I - V T V^T).
//  bcpqr   : column-pivoted Householder QR of Y^T with the AMB-10 rank rule (H3): exact
//            trailing column norms recomputed in the update pass; argmax ties -> lowest index.
#include <cstdlib>
#include <cooperative_groups.h>
#include "dense.cuh"

namespace svmhss {
namespace cg = cooperative_groups;

template <typename P>
static P* upload_probs(const std::vector<P>& v, cudaStream_t s) {
  P* d = nullptr;
  lib_malloc((void**)&d, v.size() * sizeof(P), s);
  CUDA_CHECK(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(P), cudaMemcpyHostToDevice, s));
  return d;
}
static void free_probs(void* d, cudaStream_t s) { CUDA_CHECK(cudaFreeAsync(d, s)); }

__device__ __forceinline__ void dmma884_(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// ------------------------------------------------------------------ GEMM
// FP64 tensor-core (DMMA m8n8k4) batched GEMM.  8 warps as 2 (m) x 4 (n); warp tile
// (8 MT) x (8 NT), CTA tile (16 MT) x (32 NT), k in 16-wide shared-memory tiles, register
// prefetch of the next tile (double buffered).  Operands are stored [row][k] (A) and [col][k]
// (B) with row stride 20 = 4 (mod 16) doubles, so every fragment load (row g, k t) is bank-
// conflict free.  Every tile shape runs the same per-element sequence of DMMAs (k = 0, 4, 8,
// ... in order, zero padded), so a node's result does not depend on which shape its batch
// used (bitwise P-invariance of the sharded build).
constexpr int DBK = 16, DSK = 20, DNS = 3;


__device__ __forceinline__ void cp_async8_(double* smem, const double* gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(pred ? 8 : 0));
}

template <int MT, int NT, int MINB>
__global__ void __launch_bounds__(256, MINB) bgemm_dmma_kernel(const GemmProb* __restrict__ probs) {
  constexpr int BM = 16 * MT, BN = 32 * NT;
  constexpr int LA = BM * DBK / 256, LB = BN * DBK / 256;  // elements per thread per tile
  const GemmProb P = probs[blockIdx.z];
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= P.m || n0 >= P.n) return;
  if (P.lower && n0 > m0 + BM - 1) return;  // strictly above the diagonal: not needed
  extern __shared__ __align__(16) double dsm[];
  double* As = dsm;                       // DNS x BM x DSK
  double* Bs = dsm + DNS * BM * DSK;      // DNS x BN x DSK
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  const int wm = (w >> 2) * (8 * MT), wn = (w & 3) * (8 * NT);
  const bool a_k = (P.acs == 1), b_n = (P.bcs == 1);
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // per-thread element (i0 + q di, k0 + kq0 + q dk) of the A tile, (j0 + q dj, k0 + kb0 + q dkb) of B:
  // consecutive threads walk the operand's unit-stride dimension (coalesced loads); the tiles
  // go global -> shared by 8-byte cp.async (zero fill outside the matrix)
  int ai0, ak0, adi, adk, bj0, bk0, bdj, bdk;
  if (a_k) { ai0 = tid / DBK; ak0 = tid % DBK; adi = 256 / DBK; adk = 0; }
  else { ai0 = tid % BM; ak0 = tid / BM; adi = 0; adk = 256 / BM; }
  if (b_n) { bj0 = tid % BN; bk0 = tid / BN; bdj = 0; bdk = 256 / BN; }
  else { bj0 = tid / DBK; bk0 = tid % DBK; bdj = 256 / DBK; bdk = 0; }
  const long long astep = (long long)adi * P.ars + (long long)adk * P.acs;
  const long long bstep = (long long)bdk * P.brs + (long long)bdj * P.bcs;
  const double* Ab = P.A + (long long)(m0 + ai0) * P.ars + (long long)ak0 * P.acs;
  const double* Bb = P.B + (long long)bk0 * P.brs + (long long)(n0 + bj0) * P.bcs;
  auto issue = [&](int kt, int buf) {
    const int k0 = kt * DBK;
    const double* pa = Ab + (long long)k0 * P.acs;
    double* sa = As + (buf * BM + ai0) * DSK + ak0;
#pragma unroll
    for (int q = 0; q < LA; ++q) {
      const bool ok = (m0 + ai0 + q * adi < P.m) && (k0 + ak0 + q * adk < P.k);
      cp_async8_(sa + q * (adi * DSK + adk), ok ? pa + q * astep : P.A, ok);
    }
    const double* pb = Bb + (long long)k0 * P.brs;
    double* sb = Bs + (buf * BN + bj0) * DSK + bk0;
#pragma unroll
    for (int q = 0; q < LB; ++q) {
      const bool ok = (n0 + bj0 + q * bdj < P.n) && (k0 + bk0 + q * bdk < P.k);
      cp_async8_(sb + q * (bdj * DSK + bdk), ok ? pb + q * bstep : P.B, ok);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  // DNS-stage ring, one barrier per k-tile: tile kt + DNS - 1 goes into the buffer of tile
  // kt - 1, which every warp has finished once it passes this iteration's barrier
  const int nk = (P.k + DBK - 1) / DBK;
#pragma unroll
  for (int st = 0; st < DNS - 1; ++st) {
    if (st < nk) issue(st, st);
    else asm volatile("cp.async.commit_group;\n" ::);
  }
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt % DNS;
    asm volatile("cp.async.wait_group %0;\n" ::"n"(DNS - 2));
    __syncthreads();
    if (kt + DNS - 1 < nk) issue(kt + DNS - 1, (kt + DNS - 1) % DNS);
    else asm volatile("cp.async.commit_group;\n" ::);
    const double* Aw = As + (buf * BM + wm + g) * DSK + t;
    const double* Bw = Bs + (buf * BN + wn + g) * DSK + t;
#pragma unroll
    for (int ks = 0; ks < DBK / 4; ++ks) {
      double a[MT], b[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) a[i] = Aw[i * 8 * DSK + ks * 4];
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = Bw[j * 8 * DSK + ks * 4];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma884_(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int gi = m0 + wm + i * 8 + g;
    if (gi >= P.m) continue;
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int gj = n0 + wn + j * 8 + 2 * t + e;
        if (gj >= P.n) continue;
        double* c = P.C + (long long)gi * P.crs + (long long)gj * P.ccs;
        const double v = P.alpha * acc[i][j][e];
        *c = (P.beta == 0.0) ? v : fma(P.beta, *c, v);
      }
  }
}

template <int MT, int NT, int MINB>
static void launch_dmma(const GemmProb* d, int maxm, int maxn, unsigned nb, cudaStream_t s) {
  constexpr int BM = 16 * MT, BN = 32 * NT;
  const size_t smem = (size_t)DNS * (BM + BN) * DSK * sizeof(double);
  // (set per launch: the attribute belongs to the current device's context)
  CUDA_CHECK(cudaFuncSetAttribute(bgemm_dmma_kernel<MT, NT, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid(ceil_div(maxn, BN), ceil_div(maxm, BM), nb);
  bgemm_dmma_kernel<MT, NT, MINB><<<grid, 256, smem, s>>>(d);
}

void bgemm(const std::vector<GemmProb>& probs_in, cudaStream_t s) {
  std::vector<GemmProb> probs;
  int maxm = 0, maxn = 0;
  for (const auto& p : probs_in) {
    if (p.m <= 0 || p.n <= 0) continue;
    probs.push_back(p);
    maxm = std::max(maxm, p.m);
    maxn = std::max(maxn, p.n);
  }
  if (probs.empty()) return;
  for (size_t b0 = 0; b0 < probs.size(); b0 += 65535) {
    std::vector<GemmProb> chunk(probs.begin() + b0,
                                probs.begin() + std::min(probs.size(), b0 + 65535));
    GemmProb* d = upload_probs(chunk, s);
    // FP64 tensor cores: 64 x 128 CTA tiles (two CTAs per SM) for the big factor GEMMs, 32 x 64
    // otherwise (measured: 64 x 128 beat 128 x 128 and 128 x 64 at config 3)
    if (maxm >= 256 && maxn >= 256) launch_dmma<4, 4, 2>(d, maxm, maxn, (unsigned)chunk.size(), s);
    else launch_dmma<4, 2, 2>(d, maxm, maxn, (unsigned)chunk.size(), s);
    LAUNCH_CHECK();
    free_probs(d, s);
  }
}

// ------------------------------------------------------------------ Cholesky
#define AT(P, i, j) (P).A[(long long)(i) * (P).rs + (long long)(j) * (P).cs]

__global__ void __launch_bounds__(256) bpotrf_kernel(const SqProb* __restrict__ probs, int* info) {
  const SqProb P = probs[blockIdx.x];
  const int n = P.n;
  extern __shared__ double ljrow[];
  __shared__ double dj;
  __shared__ int fail;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  if (tid == 0) fail = 0;
  for (int j = 0; j < n; ++j) {
    for (int p = tid; p < j; p += blockDim.x) ljrow[p] = AT(P, j, p);
    __syncthreads();
    for (int i = j + wid; i < n; i += nw) {
      double acc = 0.0;
      for (int p = lane; p < j; p += 32) acc = fma(AT(P, i, p), ljrow[p], acc);
      acc = warp_sum(acc);
      if (lane == 0) AT(P, i, j) -= acc;
    }
    __syncthreads();
    if (tid == 0) {
      const double d = AT(P, j, j);
      if (!(d > 0.0)) {
        fail = j + 1;
      } else {
        dj = sqrt(d);
        AT(P, j, j) = dj;
      }
    }
    __syncthreads();
    if (fail) break;
    for (int i = j + 1 + tid; i < n; i += blockDim.x) AT(P, i, j) /= dj;
    __syncthreads();
  }
  if (tid == 0 && info) info[blockIdx.x] = fail;
  if (fail) return;
  for (long long e = tid; e < (long long)n * n; e += blockDim.x) {
    const int i = (int)(e / n), j = (int)(e % n);
    if (j > i) AT(P, i, j) = 0.0;
  }
}

// Right-looking blocked Cholesky on tensor cores, one CTA (16 warps) per node.  Per panel of
// CNB = 16 columns (already updated by the previous panels): the panel rows are staged in
// shared memory, warp 0 factors the 16 x 16 diagonal block, every thread solves one row of
// L21 = A21 L11^-T (forward substitution), and the trailing lower triangle gets
// A22 -= L21 L21^T as 8 x 8 DMMA tiles (k = 16) read and written in place.  The first
// non-positive pivot stops the factorization (info = its index + 1), as bpotrf_kernel.
constexpr int CMAX = 1024, CMAX8 = 2304;

// CNB panel width, CPS its shared-memory row stride (= 4 mod 8: conflict-free fragments);
// <16, 20> up to CMAX rows, <8, 12> up to CMAX8 (large near-exact nodes)
template <int CNB, int CPS>
__global__ void __launch_bounds__(512, 1) bpotrf_tc_kernel(const SqProb* __restrict__ probs, int* info) {
  const SqProb P = probs[blockIdx.x];
  const int n = P.n, tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  extern __shared__ __align__(16) double csm[];
  double* pl = csm;                       // CMAX x CPS: panel rows (row-major)
  __shared__ int fail;
  if (tid == 0) fail = 0;
  for (int p0 = 0; p0 < n; p0 += CNB) {
    const int pb = min(CNB, n - p0), mr = n - p0;
    for (int e = tid; e < mr * CNB; e += 512) {
      const int i = e / CNB, j = e % CNB;
      pl[i * CPS + j] = (j < pb) ? AT(P, p0 + i, p0 + j) : 0.0;
    }
    __syncthreads();
    if (w == 0) {  // diagonal block: lane i holds row i
      for (int j = 0; j < pb; ++j) {
        double d = 0.0;
        if (lane == j) {
          d = pl[j * CPS + j];
          if (d > 0.0) pl[j * CPS + j] = d = sqrt(d);
        }
        d = __shfl_sync(0xffffffffu, d, j);
        if (!(d > 0.0)) {
          if (lane == 0) fail = p0 + j + 1;
          break;
        }
        if (lane > j && lane < pb) pl[lane * CPS + j] /= d;
        __syncwarp();
        if (lane > j && lane < pb) {
          const double l = pl[lane * CPS + j];
          for (int k = j + 1; k <= lane; ++k) pl[lane * CPS + k] = fma(-l, pl[k * CPS + j], pl[lane * CPS + k]);
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (fail) break;
    for (int i = pb + tid; i < mr; i += 512) {  // L21 row i: forward substitution against L11^T
      double* r = pl + i * CPS;
      for (int j = 0; j < pb; ++j) {
        double a = r[j];
        for (int k = 0; k < j; ++k) a = fma(-r[k], pl[j * CPS + k], a);
        r[j] = a / pl[j * CPS + j];
      }
    }
    __syncthreads();
    for (int e = tid; e < mr * CNB; e += 512) {  // write the panel back (lower part)
      const int i = e / CNB, j = e % CNB;
      if (j < pb && j <= i) AT(P, p0 + i, p0 + j) = pl[i * CPS + j];
    }
    // trailing: rows / columns pb .. mr-1 (panel-local); tiles (mi, ci), ci <= mi
    const int nt = (mr - pb + 7) / 8, ntile = nt * (nt + 1) / 2;
    constexpr int U = 4;  // tiles in flight per warp
    for (int base = w * U; base < ntile; base += 16 * U) {
      double d[U][2];
      int rr[U], cc[U], ra[U], rb[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int tI = base + u;
        int mi = (int)((sqrtf(8.0f * tI + 1.0f) - 1.0f) * 0.5f);
        while ((mi + 1) * (mi + 2) / 2 <= tI) ++mi;
        while (mi * (mi + 1) / 2 > tI) --mi;
        const int ci = tI - mi * (mi + 1) / 2;
        rr[u] = (tI < ntile) ? pb + mi * 8 + g : mr;
        cc[u] = pb + ci * 8 + 2 * t;
        ra[u] = pb + mi * 8 + g;
        rb[u] = pb + ci * 8 + g;
        d[u][0] = (rr[u] < mr && cc[u] < mr) ? AT(P, p0 + rr[u], p0 + cc[u]) : 0.0;
        d[u][1] = (rr[u] < mr && cc[u] + 1 < mr) ? AT(P, p0 + rr[u], p0 + cc[u] + 1) : 0.0;
      }
#pragma unroll
      for (int ks = 0; ks < CNB / 4; ++ks)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const double av = (ra[u] < mr) ? -pl[ra[u] * CPS + ks * 4 + t] : 0.0;
          const double bv = (rb[u] < mr) ? pl[rb[u] * CPS + ks * 4 + t] : 0.0;
          dmma884_(d[u][0], d[u][1], av, bv);
        }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (rr[u] < mr) {
          if (cc[u] < mr) AT(P, p0 + rr[u], p0 + cc[u]) = d[u][0];
          if (cc[u] + 1 < mr) AT(P, p0 + rr[u], p0 + cc[u] + 1) = d[u][1];
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0 && info) info[blockIdx.x] = fail;
  if (fail) return;
  for (long long e = tid; e < (long long)n * n; e += 512) {
    const int i = (int)(e / n), j = (int)(e % n);
    if (j > i) AT(P, i, j) = 0.0;
  }
}

void bpotrf(const std::vector<SqProb>& probs, int* d_info, cudaStream_t s) {
  if (probs.empty()) return;
  int maxn = 0;
  for (auto& p : probs) maxn = std::max(maxn, p.n);
  SqProb* d = upload_probs(probs, s);
  if (maxn <= CMAX8) {
    // (the panel width is chosen by the batch's largest node; bitwise P-invariance of the
    // sharded build therefore assumes all nodes of a level are on the same side of CMAX)
    if (maxn <= CMAX) {
      const size_t smem = (size_t)CMAX * 20 * sizeof(double);
      CUDA_CHECK(cudaFuncSetAttribute(bpotrf_tc_kernel<16, 20>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      bpotrf_tc_kernel<16, 20><<<(unsigned)probs.size(), 512, smem, s>>>(d, d_info);
    } else {
      const size_t smem = (size_t)CMAX8 * 12 * sizeof(double);
      CUDA_CHECK(cudaFuncSetAttribute(bpotrf_tc_kernel<8, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      bpotrf_tc_kernel<8, 12><<<(unsigned)probs.size(), 512, smem, s>>>(d, d_info);
    }
    LAUNCH_CHECK();
    free_probs(d, s);
    return;
  }
  size_t smem = (size_t)std::max(1, maxn) * sizeof(double);
  if (smem > 48 * 1024)
    CUDA_CHECK(cudaFuncSetAttribute(bpotrf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
  bpotrf_kernel<<<(unsigned)probs.size(), 256, smem, s>>>(d, d_info);
  LAUNCH_CHECK();
  free_probs(d, s);
}

// ------------------------------------------------------------------ TRSM
constexpr int TB = 32, TC = 16;

template <bool LOWER>
__global__ void __launch_bounds__(256) btrsm_kernel(const TrsmProb* __restrict__ probs) {
  const TrsmProb P = probs[blockIdx.y];
  const int c0 = blockIdx.x * TC;
  if (c0 >= P.nrhs || P.n == 0) return;
  const int nc = min(TC, P.nrhs - c0);
  __shared__ double Ts[TB][TB + 1];
  __shared__ double Xs[TB][TC + 1];
  __shared__ double Tp[TB][TB + 1];
  __shared__ double Xp[TB][TC + 1];
  const int tid = threadIdx.x, c = tid & 15, i0 = tid >> 4;  // rows i0 and i0 + 16
  const int n = P.n, nb = (n + TB - 1) / TB;
#define TT(i, j) P.T[(long long)(i) * P.trs + (long long)(j) * P.tcs]
#define XX(i, j) P.X[(long long)(i) * P.xrs + (long long)(j) * P.xcs]
  for (int bi = 0; bi < nb; ++bi) {
    int I0, I1;
    if (LOWER) { I0 = bi * TB; I1 = min(n, I0 + TB); }
    else { I1 = n - bi * TB; I0 = max(0, I1 - TB); }
    const int bs = I1 - I0;
    double acc0 = 0.0, acc1 = 0.0;
    // update with solved rows: lower -> [0, I0), upper -> [I1, n)
    const int pa = LOWER ? 0 : I1, pb = LOWER ? I0 : n;
    for (int p0 = pa; p0 < pb; p0 += TB) {
      const int pl = min(TB, pb - p0);
      for (int e = tid; e < TB * TB; e += 256) {
        const int ii = e / TB, pp = e % TB;
        Tp[ii][pp] = (ii < bs && pp < pl) ? TT(I0 + ii, p0 + pp) : 0.0;
      }
      for (int e = tid; e < TB * TC; e += 256) {
        const int pp = e / TC, cc = e % TC;
        Xp[pp][cc] = (pp < pl && cc < nc) ? XX(p0 + pp, c0 + cc) : 0.0;
      }
      __syncthreads();
#pragma unroll 8
      for (int pp = 0; pp < TB; ++pp) {
        acc0 = fma(Tp[i0][pp], Xp[pp][c], acc0);
        acc1 = fma(Tp[i0 + 16][pp], Xp[pp][c], acc1);
      }
      __syncthreads();
    }
    for (int e = tid; e < TB * TB; e += 256) {
      const int ii = e / TB, jj = e % TB;
      Ts[ii][jj] = (ii < bs && jj < bs) ? TT(I0 + ii, I0 + jj) : 0.0;
    }
    if (i0 < bs && c < nc) Xs[i0][c] = XX(I0 + i0, c0 + c) - acc0;
    if (i0 + 16 < bs && c < nc) Xs[i0 + 16][c] = XX(I0 + i0 + 16, c0 + c) - acc1;
    __syncthreads();
    // in-block substitution (column oriented)
    for (int t = 0; t < bs; ++t) {
      const int jj = LOWER ? t : bs - 1 - t;
      if (tid < nc) Xs[jj][tid] = Xs[jj][tid] / Ts[jj][jj];
      __syncthreads();
      for (int e = tid; e < TB * TC; e += 256) {
        const int ii = e / TC, cc = e % TC;
        const bool below = LOWER ? (ii > jj) : (ii < jj);
        if (below && ii < bs && cc < nc) Xs[ii][cc] -= Ts[ii][jj] * Xs[jj][cc];
      }
      __syncthreads();
    }
    if (i0 < bs && c < nc) XX(I0 + i0, c0 + c) = Xs[i0][c];
    if (i0 + 16 < bs && c < nc) XX(I0 + i0 + 16, c0 + c) = Xs[i0 + 16][c];
    __syncthreads();
  }
#undef TT
#undef XX
}

// Triangular solve on tensor cores: one CTA (8 warps) per (problem, 16 right-hand-side
// columns).  The 16 x 16 diagonal blocks are inverted first (lane c: column c of the block
// inverse, by substitution); then block by block (top down for lower, bottom up for upper):
// X_b = D_b^-1 X_b (DMMA, 2 x 2 tiles) and the not-yet-solved rows get X_i -= T_ib X_b (DMMA,
// k = 16), with X resident in shared memory and T fragments read through L1.
constexpr int SW_ = 16, SXS = 24, SDS = 20, SMAXN = 512;

// The 16 x 16 diagonal-block inverses of every problem, once (warp per block, lane c: column c
// by substitution), into dg (problem p at dg + doff[p], block bi at 256 bi, row-major 16 x 16).
template <bool LOWER>
__global__ void __launch_bounds__(256) trsm_dinv_kernel(const TrsmProb* __restrict__ probs,
                                                        const long long* __restrict__ doff, double* __restrict__ dg) {
  const TrsmProb P = probs[blockIdx.y];
  const int n = P.n, nb = (n + 15) / 16, lane = threadIdx.x & 31;
  const int bi = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (bi >= nb || lane >= 16) return;
  int r0, r1;
  if (LOWER) { r0 = bi * 16; r1 = min(n, r0 + 16); }
  else { r1 = n - bi * 16; r0 = max(0, r1 - 16); }
  const int bs = r1 - r0, c = lane;
#define TD(i, j) __ldg(P.T + (long long)(i) * P.trs + (long long)(j) * P.tcs)
  double z[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) z[j] = 0.0;
  if (c < bs) {
    if (LOWER) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j < c || j >= bs) continue;
        double a = (j == c) ? 1.0 : 0.0;
        for (int p = c; p < j; ++p) a = fma(-TD(r0 + j, r0 + p), z[p], a);
        z[j] = a / TD(r0 + j, r0 + j);
      }
    } else {
#pragma unroll
      for (int jj = 15; jj >= 0; --jj) {
        if (jj > c) continue;
        double a = (jj == c) ? 1.0 : 0.0;
        for (int p = jj + 1; p <= c; ++p) a = fma(-TD(r0 + jj, r0 + p), z[p], a);
        z[jj] = a / TD(r0 + jj, r0 + jj);
      }
    }
  }
#undef TD
  double* D = dg + doff[blockIdx.y] + (long long)bi * 256;
#pragma unroll
  for (int j = 0; j < 16; ++j) D[j * 16 + c] = z[j];
}

template <bool LOWER>
__global__ void __launch_bounds__(256) btrsm_tc_kernel(const TrsmProb* __restrict__ probs,
                                                        const long long* __restrict__ doff, const double* __restrict__ dg) {
  const TrsmProb P = probs[blockIdx.y];
  const int c0 = blockIdx.x * SW_;
  if (c0 >= P.nrhs || P.n == 0) return;
  const int n = P.n, nc = min(SW_, P.nrhs - c0), nb = (n + 15) / 16;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  extern __shared__ __align__(16) double tsm[];
  double* Xs = tsm;                               // n8 x SXS
  double* Di = tsm + (size_t)((n + 7) & ~7) * SXS;  // nb x 16 x SDS
#define TT(i, j) __ldg(P.T + (long long)(i) * P.trs + (long long)(j) * P.tcs)
#define XX(i, j) P.X[(long long)(i) * P.xrs + (long long)(j) * P.xcs]
  auto blk = [&](int bi, int& r0, int& r1) {
    if (LOWER) { r0 = bi * 16; r1 = min(n, r0 + 16); }
    else { r1 = n - bi * 16; r0 = max(0, r1 - 16); }
  };
  for (int e = tid; e < ((n + 7) & ~7) * SW_; e += 256) {
    const int i = e / SW_, c = e % SW_;
    Xs[i * SXS + c] = (i < n && c < nc) ? XX(i, c0 + c) : 0.0;
  }
  {  // diagonal block inverses (trsm_dinv_kernel), zero padded to 16 x 16
    const double* dsrc = dg + doff[blockIdx.y];
    for (int e = tid; e < nb * 256; e += 256) Di[(size_t)(e >> 8) * 16 * SDS + ((e >> 4) & 15) * SDS + (e & 15)] = dsrc[e];
  }
  __syncthreads();
  for (int bi = 0; bi < nb; ++bi) {
    int r0, r1;
    blk(bi, r0, r1);
    const int bs = r1 - r0;
    const double* D = Di + (size_t)bi * 16 * SDS;
    double y0 = 0.0, y1 = 0.0;
    const int mt = w & 1, nt = (w >> 1) & 1;
    if (w < 4) {  // X_b = D^-1 X_b, tile (mt, nt)
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const int k = ks * 4 + t;
        const double bv = (k < bs) ? Xs[(r0 + k) * SXS + nt * 8 + g] : 0.0;
        dmma884_(y0, y1, D[(mt * 8 + g) * SDS + k], bv);
      }
    }
    __syncthreads();
    if (w < 4 && mt * 8 + g < bs) {
      Xs[(r0 + mt * 8 + g) * SXS + nt * 8 + 2 * t] = y0;
      Xs[(r0 + mt * 8 + g) * SXS + nt * 8 + 2 * t + 1] = y1;
    }
    __syncthreads();
    // X_i -= T[i, r0:r1] X_b for the unsolved rows: lower [r1, n), upper [0, r0)
    const int u0 = LOWER ? r1 : 0, u1 = LOWER ? n : r0;
    double bf[2][4];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const int k = ks * 4 + t;
        bf[q][ks] = (k < bs) ? Xs[(r0 + k) * SXS + q * 8 + g] : 0.0;
      }
    const int nt8 = (u1 - u0 + 7) / 8;
    for (int mi = w; mi < nt8; mi += 8) {
      const int ra = u0 + mi * 8 + g;
      double af[4];
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const int k = ks * 4 + t;
        af[ks] = (ra < u1 && k < bs) ? -TT(ra, r0 + k) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        double* xr = Xs + ra * SXS + q * 8 + 2 * t;
        double d0 = (ra < u1) ? xr[0] : 0.0, d1 = (ra < u1) ? xr[1] : 0.0;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) dmma884_(d0, d1, af[ks], bf[q][ks]);
        if (ra < u1) { xr[0] = d0; xr[1] = d1; }
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < n * SW_; e += 256) {
    const int i = e / SW_, c = e % SW_;
    if (c < nc) XX(i, c0 + c) = Xs[i * SXS + c];
  }
#undef TT
#undef XX
}

void btrsm(const std::vector<TrsmProb>& probs_in, bool lower, cudaStream_t s) {
  std::vector<TrsmProb> probs;
  int maxr = 0, maxn = 0;
  for (auto& p : probs_in)
    if (p.n > 0 && p.nrhs > 0) { probs.push_back(p); maxr = std::max(maxr, p.nrhs); maxn = std::max(maxn, p.n); }
  if (probs.empty()) return;
  for (size_t b0 = 0; b0 < probs.size(); b0 += 65535) {
    std::vector<TrsmProb> chunk(probs.begin() + b0,
                                probs.begin() + std::min(probs.size(), b0 + 65535));
    TrsmProb* d = upload_probs(chunk, s);
    if (maxn <= SMAXN) {
      const size_t smem = ((size_t)((maxn + 7) & ~7) * SXS + (size_t)((maxn + 15) / 16) * 16 * SDS) * sizeof(double);
      dim3 grid(ceil_div(maxr, SW_), (unsigned)chunk.size());
      std::vector<long long> doff(chunk.size());
      long long tot = 0;
      for (size_t q = 0; q < chunk.size(); ++q) { doff[q] = tot; tot += (long long)((chunk[q].n + 15) / 16) * 256; }
      auto ddoff = upload(doff, s);
      DevBuf<double> dg((size_t)std::max<long long>(1, tot));
      dim3 gdi(ceil_div((maxn + 15) / 16, 8), (unsigned)chunk.size());
      if (lower) {
        trsm_dinv_kernel<true><<<gdi, 256, 0, s>>>(d, ddoff.p, dg.p);
        CUDA_CHECK(cudaFuncSetAttribute(btrsm_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        btrsm_tc_kernel<true><<<grid, 256, smem, s>>>(d, ddoff.p, dg.p);
      } else {
        trsm_dinv_kernel<false><<<gdi, 256, 0, s>>>(d, ddoff.p, dg.p);
        CUDA_CHECK(cudaFuncSetAttribute(btrsm_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        btrsm_tc_kernel<false><<<grid, 256, smem, s>>>(d, ddoff.p, dg.p);
      }
      LAUNCH_CHECK();
      free_probs(d, s);
      continue;
    }
    dim3 grid(ceil_div(maxr, TC), (unsigned)chunk.size());
    if (lower) btrsm_kernel<true><<<grid, 256, 0, s>>>(d);
    else btrsm_kernel<false><<<grid, 256, 0, s>>>(d);
    LAUNCH_CHECK();
    free_probs(d, s);
  }
}

// ------------------------------------------------------------------ Householder QR
// Blocked right-looking Householder QR, one CTA per node.  The (m - p0) x NB panel is
// factored in shared memory (dlarfg convention, identical reflectors to unblocked dgeqr2
// up to rounding); the trailing columns are updated with the compact-WY block reflector
// (W = V^T A, W = T^T W, A -= V W), reading the trailing matrix twice per panel instead of
// twice per column.  Each thread owns whole columns (coalesced row-major access).
// shared memory of the QR kernel: panel m x nb, trailing column block m x cb, W and T^T W (nb x cb)
inline size_t qr_smem(int m, int nb, int cb) {
  return ((size_t)m * nb + (size_t)m * cb + 2 * (size_t)nb * cb) * 8;
}

constexpr int QT = 512;  // threads of the QR kernel

template <int NB>
__global__ void __launch_bounds__(QT) bgeqrf_kernel(const QrProb* __restrict__ probs, int cb) {
  const QrProb P = probs[blockIdx.x];
  const int m = P.m, n = P.n, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  extern __shared__ double sm[];
  double* pan = sm;                 // (m) x NB panel, row-major stride NB
  double* ablk = pan + (size_t)m * NB;   // m x cb (cb: trailing-update column block)
  double* wsh = ablk + (size_t)m * cb;   // NB x cb
  double* w2sh = wsh + NB * cb;          // NB x cb
  __shared__ double T[NB][NB + 1];
  __shared__ double tau_s[NB];
  __shared__ double red[32];
#define QA(i, j) P.A[(long long)(i) * P.rs + (long long)(j) * P.cs]
  for (int p0 = 0; p0 < n; p0 += NB) {
    const int pb = min(NB, n - p0), mr = m - p0;
    for (int e = tid; e < mr * NB; e += QT) {
      const int i = e / NB, j = e % NB;
      pan[e] = (j < pb) ? QA(p0 + i, p0 + j) : 0.0;
    }
    __syncthreads();
    // factor the panel in shared memory
    for (int j = 0; j < pb; ++j) {
      double part = 0.0;
      for (int i = j + 1 + tid; i < mr; i += QT) { const double x = pan[i * NB + j]; part = fma(x, x, part); }
      const double xs = block_sum(part, red);
      const double alpha = pan[j * NB + j];
      double tau, scal, beta;
      if (xs == 0.0) { tau = 0.0; scal = 1.0; beta = alpha; }
      else {
        beta = -copysign(sqrt(alpha * alpha + xs), alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      if (tau != 0.0)
        for (int i = j + 1 + tid; i < mr; i += QT) pan[i * NB + j] *= scal;
      __syncthreads();
      if (tid == 0) { pan[j * NB + j] = beta; tau_s[j] = tau; }
      // apply H_j to panel columns c > j: warp per column
      if (tau != 0.0) {
        for (int c = j + 1 + wid; c < pb; c += QT / 32) {
          double w = 0.0;
          for (int i = j + lane; i < mr; i += 32) {
            const double vi = (i == j) ? 1.0 : pan[i * NB + j];
            w = fma(vi, pan[i * NB + c], w);
          }
          w = warp_sum(w) * tau;
          for (int i = j + lane; i < mr; i += 32) {
            const double vi = (i == j) ? 1.0 : pan[i * NB + j];
            pan[i * NB + c] = fma(-w, vi, pan[i * NB + c]);
          }
        }
      }
      __syncthreads();
    }
    // T (pb x pb upper): T_jj = tau_j, T[0:j, j] = -tau_j T[0:j,0:j] (V[:,0:j]^T v_j)
    for (int j = 0; j < pb; ++j) {
      // s_i = V[:, i]^T v_j for i < j  (warp per i)
      for (int i = wid; i < j; i += QT / 32) {
        double a = 0.0;
        for (int r = j + lane; r < mr; r += 32) {
          const double vi = (r == i) ? 1.0 : (r > i ? pan[r * NB + i] : 0.0);
          const double vj = (r == j) ? 1.0 : pan[r * NB + j];
          a = fma(vi, vj, a);
        }
        a = warp_sum(a);
        if (lane == 0) T[i][j] = a;   // temporarily holds s_i
      }
      __syncthreads();
      if (tid < j) {
        double a = 0.0;
        for (int q = tid; q < j; ++q) a = fma(T[tid][q], T[q][j], a);
        red[tid] = a;
      }
      __syncthreads();
      if (tid < j) T[tid][j] = -tau_s[j] * red[tid];
      if (tid == 0) T[j][j] = tau_s[j];
      for (int i = j + 1 + tid; i < NB; i += QT) T[i][j] = 0.0;
      __syncthreads();
    }
    // write the panel back (R on/above the diagonal, V below) and tau
    for (int e = tid; e < mr * pb; e += QT) {
      const int i = e / pb, j = e % pb;
      QA(p0 + i, p0 + j) = pan[i * NB + j];
    }
    if (tid < pb) P.tau[p0 + tid] = tau_s[tid];
    // trailing update: A[p0:, c] -= V T^T V^T A[p0:, c]  for c >= p0 + pb, in blocks of cb
    // columns staged through shared memory (coalesced global traffic, one read and one write
    // per panel).  Per column the arithmetic order is the plain one: w_j = sum_i v_ij a_i in
    // row order, w2 = T^T w, a_i -= sum_j v_ij w2_j in j order.
    for (int c0 = p0 + pb; c0 < n; c0 += cb) {
      const int nc = min(cb, n - c0);
      for (int e = tid; e < mr * nc; e += QT) {
        const int i = e / nc, c = e % nc;
        ablk[i * cb + c] = QA(p0 + i, c0 + c);
      }
      __syncthreads();
      for (int e = tid; e < NB * nc; e += QT) {  // W[j][c] = V[:, j]^T a_c
        const int j = e / nc, c = e % nc;
        double w = 0.0;
        if (j < pb) {
          for (int i = j; i < mr; ++i) {
            const double v = (i == j) ? 1.0 : pan[i * NB + j];
            w = fma(v, ablk[i * cb + c], w);
          }
        }
        wsh[j * cb + c] = w;
      }
      __syncthreads();
      for (int e = tid; e < NB * nc; e += QT) {  // W2 = T^T W (column c)
        const int j = e / nc, c = e % nc;
        double a = 0.0;
        for (int q = 0; q <= j; ++q) a = fma(T[q][j], wsh[q * cb + c], a);
        w2sh[j * cb + c] = a;
      }
      __syncthreads();
      for (int e = tid; e < mr * nc; e += QT) {  // a -= V W2
        const int i = e / nc, c = e % nc;
        double a = ablk[i * cb + c];
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          const double v = (i == j) ? 1.0 : ((i > j) ? pan[i * NB + j] : 0.0);
          a = fma(-v, w2sh[j * cb + c], a);
        }
        QA(p0 + i, c0 + c) = a;
      }
      __syncthreads();
    }
    __syncthreads();
  }
#undef QA
}

// Householder QR with tensor-core trailing updates, one CTA (16 warps) per node, m <= 16 * 32.
// Panels of NB = 16 columns: warp w keeps panel column w in registers (rows lane + 32 q);
// step j: warp j forms its reflector (dlarfg convention) and publishes v_j to shared memory,
// one CTA barrier, warps c > j apply H_j to their own column -- one barrier per column.  Then
// T (compact WY, NB x NB) from G = V^T V, and the trailing columns, in blocks of QCB = 16
// staged in shared memory, get A -= V (T^T (V^T A)) on DMMA: W = V^T A as 2 x 2 output tiles
// with the row range split in 4 quarters (16 warps), the quarters summed in a fixed order;
// the update D = A + V (-T^T W) as (m/8) x 2 tiles.  Arithmetic order depends on m and n only.
constexpr int QNB = 16, QCB = 16, QRPL = 16, QMAX = 32 * QRPL;
constexpr int QSP = 520;   // panel column stride (= 8 mod 32: conflict-free A-fragments of V W2)
constexpr int QSB = 24;    // trailing block row stride (= 24 mod 32: conflict-free B-fragments)

__global__ void __launch_bounds__(512, 1) bgeqrf_tc_kernel(const QrProb* __restrict__ probs) {
  const QrProb P = probs[blockIdx.x];
  const int m = P.m, n = P.n, tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  extern __shared__ __align__(16) double qsm[];
  double* pv = qsm;                         // QNB x QSP: v_j (unit diagonal, zeros above), local rows
  double* ab = pv + QNB * QSP;              // QMAX x QSB: trailing column block
  double* wp = ab + QMAX * QSB;             // 4 x QNB x QCB: W partials (row quarters)
  double* w2 = wp + 4 * QNB * QCB;          // QNB x QCB: -T^T W
  __shared__ double Tm[QNB][QNB + 1];
  __shared__ double Gm[QNB][QNB + 1];
  __shared__ double taus[QNB];
#define QA(i, j) P.A[(long long)(i) * P.rs + (long long)(j) * P.cs]
  for (int p0 = 0; p0 < n; p0 += QNB) {
    const int pb = min(QNB, n - p0), mr = m - p0;
    // ---- panel: warp w owns column p0 + w
    double x[QRPL];
    const bool own = w < pb;
#pragma unroll
    for (int q = 0; q < QRPL; ++q) {
      const int i = lane + 32 * q;
      x[q] = (own && i < mr) ? QA(p0 + i, p0 + w) : 0.0;
    }
    double rjj = 0.0;
    for (int j = 0; j < pb; ++j) {
      if (w == j) {
        double xs = 0.0;
#pragma unroll
        for (int q = 0; q < QRPL; ++q) {
          const int i = lane + 32 * q;
          if (i > j && i < mr) xs = fma(x[q], x[q], xs);
        }
        xs = warp_sum(xs);
        const double alpha = __shfl_sync(0xffffffffu, x[0], j);  // row j < QNB <= 32: q = 0
        double tau = 0.0, scal = 1.0, beta = alpha;
        if (xs != 0.0) {
          beta = -copysign(sqrt(alpha * alpha + xs), alpha);
          tau = (beta - alpha) / beta;
          scal = 1.0 / (alpha - beta);
        }
#pragma unroll
        for (int q = 0; q < QRPL; ++q) {
          const int i = lane + 32 * q;
          if (i < mr) {
            double v = 0.0;
            if (i == j) v = 1.0;
            else if (i > j) { if (tau != 0.0) x[q] *= scal; v = x[q]; }
            pv[j * QSP + i] = v;
          }
        }
        rjj = beta;
        if (lane == 0) taus[j] = tau;
      }
      __syncthreads();
      if (w > j && w < pb) {
        const double tau = taus[j];
        double d = 0.0;
#pragma unroll
        for (int q = 0; q < QRPL; ++q) {
          const int i = lane + 32 * q;
          if (i >= j && i < mr) d = fma(pv[j * QSP + i], x[q], d);
        }
        d = warp_sum(d) * tau;
#pragma unroll
        for (int q = 0; q < QRPL; ++q) {
          const int i = lane + 32 * q;
          if (i >= j && i < mr) x[q] = fma(-d, pv[j * QSP + i], x[q]);
        }
      }
    }
    // write the panel back: R above / on the diagonal, v below; zero-pad pv past pb and mr
    if (own) {
#pragma unroll
      for (int q = 0; q < QRPL; ++q) {
        const int i = lane + 32 * q;
        if (i < mr) QA(p0 + i, p0 + w) = (i == w) ? rjj : x[q];
      }
      if (lane == 0) P.tau[p0 + w] = taus[w];
    }
    for (int e = tid; e < QNB * QSP; e += 512) {
      const int j = e / QSP, i = e % QSP;
      if (j >= pb || i >= mr) pv[e] = 0.0;
    }
    __syncthreads();
    // ---- G = V^T V (upper), warp c: G[i][c], i <= c
    if (w < pb) {
      for (int i = 0; i <= w; ++i) {
        double d = 0.0;
#pragma unroll
        for (int q = 0; q < QRPL; ++q) {
          const int r = lane + 32 * q;
          if (r < mr) d = fma(pv[i * QSP + r], pv[w * QSP + r], d);
        }
        d = warp_sum(d);
        if (lane == 0) Gm[i][w] = d;
      }
    }
    __syncthreads();
    // ---- T (upper): T_jj = tau_j, T[0:j, j] = -tau_j T[0:j, 0:j] G[0:j, j]  (warp 0)
    if (w == 0) {
      for (int j = 0; j < QNB; ++j) {
        double a = 0.0;
        if (lane < j && j < pb)
          for (int p = lane; p < j; ++p) a = fma(Tm[lane][p], Gm[p][j], a);
        __syncwarp();
        if (lane < QNB) {
          if (j >= pb) Tm[lane][j] = 0.0;
          else if (lane < j) Tm[lane][j] = -taus[j] * a;
          else Tm[lane][j] = (lane == j) ? taus[j] : 0.0;
        }
        __syncwarp();
      }
    }
    __syncthreads();
    // ---- trailing columns in blocks of QCB; the next block's loads are issued into registers
    // before the current block's arithmetic (global latency hidden under the DMMAs)
    const int mr8 = (mr + 7) & ~7;
    const int quarter = ((mr8 / 4 + 3) / 4) * 4;   // k range per W-partial, multiple of 4
    constexpr int PF = QMAX * QCB / 512;            // prefetch registers per thread
    double nx[PF];
    auto fetch = [&](int c0) {
      const int nc = min(QCB, n - c0);
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        const int e = tid + 512 * q, i = e / QCB, c = e % QCB;
        nx[q] = (i < mr && c < nc) ? QA(p0 + i, c0 + c) : 0.0;
      }
    };
    auto stage = [&]() {
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        const int e = tid + 512 * q, i = e / QCB, c = e % QCB;
        if (i < mr8) ab[i * QSB + c] = nx[q];
      }
    };
    if (p0 + pb < n) { fetch(p0 + pb); stage(); }
    __syncthreads();
    for (int c0 = p0 + pb; c0 < n; c0 += QCB) {
      const int nc = min(QCB, n - c0);
      const bool more = c0 + QCB < n;
      if (more) fetch(c0 + QCB);
      {  // W partial: tile (mt, nt) = (w & 1, (w >> 1) & 1), rows quarter w >> 2
        const int mt = w & 1, nt = (w >> 1) & 1, qr = w >> 2;
        const int k0 = qr * quarter, k1 = min(mr8, k0 + quarter);
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
        int k = k0;
        for (; k + 8 <= k1; k += 8) {
          dmma884_(a0, a1, pv[(mt * 8 + g) * QSP + k + t], ab[(k + t) * QSB + nt * 8 + g]);
          dmma884_(b0, b1, pv[(mt * 8 + g) * QSP + k + 4 + t], ab[(k + 4 + t) * QSB + nt * 8 + g]);
        }
        for (; k < k1; k += 4)
          dmma884_(a0, a1, pv[(mt * 8 + g) * QSP + k + t], ab[(k + t) * QSB + nt * 8 + g]);
        double* dst = wp + qr * QNB * QCB + (mt * 8 + g) * QCB + nt * 8 + 2 * t;
        dst[0] = a0 + b0;
        dst[1] = a1 + b1;
      }
      __syncthreads();
      if (tid < QNB * QCB) {  // W = sum of quarters (fixed order); w2 = -T^T W
        const int j = tid / QCB, c = tid % QCB;
        double a = 0.0;
        for (int q = 0; q <= j; ++q) {
          const int o = q * QCB + c;
          const double wv = ((wp[o] + wp[QNB * QCB + o]) + wp[2 * QNB * QCB + o]) + wp[3 * QNB * QCB + o];
          a = fma(Tm[q][j], wv, a);
        }
        w2[j * QCB + c] = -a;
      }
      __syncthreads();
      {  // update: tiles (mi, ni), mi < mr8 / 8, ni < 2; warp w takes mi = w, w + 16, ...
        double bf[2][QNB / 4];
#pragma unroll
        for (int ni = 0; ni < 2; ++ni)
#pragma unroll
          for (int ks = 0; ks < QNB / 4; ++ks) bf[ni][ks] = w2[(ks * 4 + t) * QCB + ni * 8 + g];
        for (int mi = w; mi < mr8 / 8; mi += 16) {
          const int r = mi * 8 + g;
          double af[QNB / 4];
#pragma unroll
          for (int ks = 0; ks < QNB / 4; ++ks) af[ks] = pv[(ks * 4 + t) * QSP + mi * 8 + g];
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) {
            const int c = ni * 8 + 2 * t;
            double d0 = ab[r * QSB + c], d1 = ab[r * QSB + c + 1];
#pragma unroll
            for (int ks = 0; ks < QNB / 4; ++ks) dmma884_(d0, d1, af[ks], bf[ni][ks]);
            if (r < mr) {
              if (c < nc) QA(p0 + r, c0 + c) = d0;
              if (c + 1 < nc) QA(p0 + r, c0 + c + 1) = d1;
            }
          }
        }
      }
      __syncthreads();
      if (more) { stage(); __syncthreads(); }
    }
  }
#undef QA
}

void bgeqr2(const std::vector<QrProb>& probs, cudaStream_t s) {
  if (probs.empty()) return;
  int maxm = 0;
  for (auto& p : probs) maxm = std::max(maxm, p.m);
  QrProb* d = upload_probs(probs, s);
  if (maxm <= QMAX) {
    const size_t smem = ((size_t)QNB * QSP + (size_t)QMAX * QSB + 5 * QNB * QCB) * sizeof(double);
    CUDA_CHECK(cudaFuncSetAttribute(bgeqrf_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    bgeqrf_tc_kernel<<<(unsigned)probs.size(), 512, smem, s>>>(d);
    LAUNCH_CHECK();
    free_probs(d, s);
    return;
  }
  // panel width NB and trailing column block cb: the largest that fit 200 KB for the tallest problem
  auto launch = [&](auto kern, int nb) -> bool {
    int cb = 32;
    while (cb > 1 && qr_smem(std::max(1, maxm), nb, cb) > 200 * 1024) cb >>= 1;
    const size_t smem = qr_smem(std::max(1, maxm), nb, cb);
    if (smem > 200 * 1024) return false;
    if (smem > 48 * 1024)
      CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)probs.size(), QT, smem, s>>>(d, cb);
    return true;
  };
  if (launch(bgeqrf_kernel<16>, 16)) {}
  else if (launch(bgeqrf_kernel<8>, 8)) {}
  else if (launch(bgeqrf_kernel<4>, 4)) {}
  else throw Error(HSS_EINVAL, "bgeqr2: node too tall for the shared-memory panel");
  LAUNCH_CHECK();
  free_probs(d, s);
}

// ------------------------------------------------------------------ larft
// Compact-WY T (Q = H_1 ... H_n = I - V T V^T, H_i = I - tau_i v_i v_i^T) from S = V^T V by one
// triangular solve instead of LAPACK's column recurrence: with D = diag(tau) and U = striu(S),
// T^-1 = D^-1 + U, i.e. T = (I + D U)^-1 D — a unit upper-triangular system with the diagonal
// right-hand side D (no division by tau, so tau_i = 0 gives a zero column as in dlarft).  The
// solve runs on btrsm's DMMA kernel (16 CTAs per node for n = 256) rather than one CTA per node
// walking the n columns in order: the few-node top levels of the factor are latency-bound
// (by_solve); wide levels keep the recurrence (blarft_blk_kernel: one CTA per node, faster
// there).  The caller picks by GLOBAL tree level, so the choice does not depend on the shard.
// Blocked larft: block columns of LNB = 16.  With S = V^T V on input (in place), for block
// column J: the diagonal block T_JJ by the column recurrence (warp 0), Y = S[0:J, J] T_JJ,
// and T[0:J, J] = -T[0:J, 0:J] Y (Q = Q_1 Q_2: T = [T1, -T1 V1^T V2 T2; 0, T2]); the block
// columns before J are final when J starts.  Thread (i, c) owns output row i, column c.
constexpr int LNB = 16;

__global__ void __launch_bounds__(512) blarft_blk_kernel(const SqProb* __restrict__ probs,
                                                         const double* const* __restrict__ taus, int lmax) {
  const SqProb P = probs[blockIdx.x];
  const double* tau = taus[blockIdx.x];
  const int n = P.n, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  extern __shared__ __align__(16) double lsm[];
  double* Sb = lsm;                  // lmax x LNB: S[0:j1, J-block]
  double* Y = Sb + (size_t)lmax * LNB;  // lmax x LNB
  __shared__ double Tjj[LNB][LNB + 1];
  for (int j0 = 0; j0 < n; j0 += LNB) {
    const int jb = min(LNB, n - j0), j1 = j0 + jb;
    for (int e = tid; e < j1 * LNB; e += 512) {
      const int i = e / LNB, c = e % LNB;
      Sb[e] = (c < jb) ? AT(P, i, j0 + c) : 0.0;
    }
    __syncthreads();
    if (w == 0) {  // T_JJ: T[r][c] = -tau_c sum_{p=r}^{c-1} T[r][p] S[j0+p][j0+c]
      for (int c = 0; c < LNB; ++c) {
        double a = 0.0;
        if (lane < c && c < jb)
          for (int q = lane; q < c; ++q) a = fma(Tjj[lane][q], Sb[(j0 + q) * LNB + c], a);
        __syncwarp();
        if (lane < LNB) {
          if (c >= jb) Tjj[lane][c] = 0.0;
          else if (lane < c) Tjj[lane][c] = -tau[j0 + c] * a;
          else Tjj[lane][c] = (lane == c) ? tau[j0 + c] : 0.0;
        }
        __syncwarp();
      }
    }
    __syncthreads();
    for (int e = tid; e < j0 * LNB; e += 512) {  // Y = S[0:j0, J] T_JJ
      const int i = e / LNB, c = e % LNB;
      double a = 0.0;
      for (int q = 0; q <= c; ++q) a = fma(Sb[i * LNB + q], Tjj[q][c], a);
      Y[e] = a;
    }
    __syncthreads();
    for (int e = tid; e < j0 * LNB; e += 512) {  // T[i, J] = -T[i, i:j0] Y[i:j0, :]
      const int i = e / LNB, c = e % LNB;
      double a = 0.0;
      for (int p = i; p < j0; ++p) a = fma(AT(P, i, p), Y[p * LNB + c], a);
      if (c < jb) AT(P, i, j0 + c) = -a;
    }
    for (int e = tid; e < (n - j0) * LNB; e += 512) {  // diagonal block and zeros below it
      const int i = j0 + e / LNB, c = e % LNB;
      if (c < jb) AT(P, i, j0 + c) = (i < j1) ? Tjj[i - j0][c] : 0.0;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) larft_system_kernel(const SqProb* __restrict__ probs,
                                                            const double* const* __restrict__ taus,
                                                            double* const* __restrict__ xs) {
  const SqProb P = probs[blockIdx.x];
  const double* tau = taus[blockIdx.x];
  double* X = xs[blockIdx.x];
  const int n = P.n;
  for (long long e = threadIdx.x; e < (long long)n * n; e += blockDim.x) {
    const int i = (int)(e / n), j = (int)(e % n);
    const double sij = AT(P, i, j);
    AT(P, i, j) = (j > i) ? tau[i] * sij : (j == i ? 1.0 : 0.0);   // I + D U
    X[e] = (i == j) ? tau[i] : 0.0;                                  // D
  }
}

__global__ void __launch_bounds__(256) larft_store_kernel(const SqProb* __restrict__ probs,
                                                           double* const* __restrict__ xs) {
  const SqProb P = probs[blockIdx.x];
  const double* X = xs[blockIdx.x];
  const int n = P.n;
  for (long long e = threadIdx.x; e < (long long)n * n; e += blockDim.x) {
    const int i = (int)(e / n), j = (int)(e % n);
    AT(P, i, j) = (j >= i) ? X[e] : 0.0;
  }
}

void blarft(const std::vector<SqProb>& probs, const std::vector<const double*>& taus, bool by_solve,
            cudaStream_t s) {
  if (probs.empty()) return;
  int maxn = 0;
  for (auto& p : probs) maxn = std::max(maxn, p.n);
  const int lmax = (maxn + 15) & ~15;
  const size_t sm2 = (size_t)2 * lmax * LNB * sizeof(double);
  if (!by_solve && sm2 <= 226 * 1024) {  // the column recurrence, one CTA per node
    SqProb* d = upload_probs(probs, s);
    const double** dt = upload_probs(taus, s);
    CUDA_CHECK(cudaFuncSetAttribute(blarft_blk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
    blarft_blk_kernel<<<(unsigned)probs.size(), 512, sm2, s>>>(d, dt, lmax);
    LAUNCH_CHECK();
    free_probs(d, s);
    free_probs((void*)dt, s);
    return;
  }
  int64_t tot = 0;
  std::vector<int64_t> off(probs.size());
  for (size_t q = 0; q < probs.size(); ++q) { off[q] = tot; tot += (int64_t)probs[q].n * probs[q].n; }
  DevBuf<double> xbuf(std::max<int64_t>(1, tot));
  std::vector<double*> xp(probs.size());
  std::vector<TrsmProb> tp(probs.size());
  for (size_t q = 0; q < probs.size(); ++q) {
    const SqProb& P = probs[q];
    xp[q] = xbuf.p + off[q];
    tp[q] = {P.n, P.n, P.A, P.rs, P.cs, xp[q], (long long)P.n, 1};
  }
  SqProb* d = upload_probs(probs, s);
  const double** dt = upload_probs(taus, s);
  double** dx = upload_probs(xp, s);
  larft_system_kernel<<<(unsigned)probs.size(), 256, 0, s>>>(d, dt, dx);
  LAUNCH_CHECK();
  btrsm(tp, false, s);   // X := (I + D U)^-1 D
  larft_store_kernel<<<(unsigned)probs.size(), 256, 0, s>>>(d, dx);
  LAUNCH_CHECK();
  free_probs(d, s);
  free_probs((void*)dt, s);
  free_probs((void*)dx, s);
}

// ------------------------------------------------------------------ column-pivoted QR (H3)
constexpr int CP_THREADS = 512;

template <int MAXPL>
__global__ void __launch_bounds__(CP_THREADS) bcpqr_kernel(const CpqrProb* __restrict__ probs,
                                                           double rel_tol, double abs_tol,
                                                           int cap, int cpqr_prefetch) {
  const CpqrProb P = probs[blockIdx.x];
  const int rows = P.rows, s = P.s;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = CP_THREADS / 32;
  extern __shared__ double sm[];
  double* norm2 = sm;                       // rows
  double* v = norm2 + rows;                 // s
  int* piv = (int*)(v + s);                 // rows
  __shared__ double red[32];
  __shared__ double rv[32];
  __shared__ int ri[32];
  __shared__ int s_p;
  __shared__ int s_stop;
  double* W = P.W;
  // initial column norms (column c = W[c, 0:s], contiguous)
  for (int c = wid; c < rows; c += nw) {
    double a = 0.0;
    for (int i = lane; i < s; i += 32) { const double x = W[(long long)c * s + i]; a = fma(x, x, a); }
    a = warp_sum(a);
    if (lane == 0) norm2[c] = a;
  }
  for (int c = tid; c < rows; c += CP_THREADS) piv[c] = c;
  __syncthreads();
  const bool adaptive = P.kfixed < 0;
  int kmax = adaptive ? min(min(cap, rows), s) : min(min(P.kfixed, rows), s);
  double thr = 0.0;
  int k = 0;
  for (int j = 0; j < kmax; ++j) {
    if (P.forced) {  // fixed-skeleton mode: the imported column's current position
      const int want = P.forced[j];
      for (int c = j + tid; c < rows; c += CP_THREADS)
        if (piv[c] == want) s_p = c;
    } else {
    // argmax_{c >= j} norm2[c], ties -> lowest index
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int c = j + tid; c < rows; c += CP_THREADS) {
      const double x = norm2[c];
      if (x > bv) { bv = x; bi = c; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { rv[wid] = bv; ri[wid] = bi; }
    __syncthreads();
    if (tid == 0) {
      double b = rv[0];
      int ix = ri[0];
      for (int w = 1; w < nw; ++w)
        if (rv[w] > b || (rv[w] == b && ri[w] < ix)) { b = rv[w]; ix = ri[w]; }
      s_p = ix;
    }
    }
    __syncthreads();
    const int p = s_p;
    if (p != j) {  // swap columns j and p
      for (int i = tid; i < s; i += CP_THREADS) {
        const double a = W[(long long)j * s + i];
        W[(long long)j * s + i] = W[(long long)p * s + i];
        W[(long long)p * s + i] = a;
      }
      __syncthreads();
      if (tid == 0) {
        const double t = norm2[j]; norm2[j] = norm2[p]; norm2[p] = t;
        const int q = piv[j]; piv[j] = piv[p]; piv[p] = q;
      }
    }
    __syncthreads();
    // Householder of column j, rows j..s-1 (dlarfg)
    double part = 0.0;
    for (int i = j + 1 + tid; i < s; i += CP_THREADS) { const double x = W[(long long)j * s + i]; part = fma(x, x, part); }
    const double xs = block_sum(part, red);
    const double alpha = W[(long long)j * s + j];
    const double rjj = sqrt(alpha * alpha + xs);
    if (adaptive) {
      if (j == 0) thr = fmax(rel_tol * rjj, abs_tol * sqrt((double)s));
      if (!(rjj > thr)) break;
    }
    double tau, scal, beta;
    if (xs == 0.0) { tau = 0.0; scal = 0.0; beta = alpha; }
    else {
      beta = -copysign(rjj, alpha);
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    for (int i = j + 1 + tid; i < s; i += CP_THREADS) {
      const double x = (tau == 0.0) ? W[(long long)j * s + i] : W[(long long)j * s + i] * scal;
      v[i] = x;
      W[(long long)j * s + i] = x;
    }
    if (tid == 0) { v[j] = 1.0; W[(long long)j * s + j] = beta; }
    __syncthreads();
    // update columns c > j (warp per column, column held in registers) + exact trailing norms
    for (int c = j + 1 + wid; c < rows; c += nw) {
      double x[MAXPL];
      double* col = W + (long long)c * s;
      // L2 prefetch of this warp's next column (its DRAM latency overlaps this column's work)
      if (cpqr_prefetch && c + nw < rows && 16 * lane < s - j)
        asm volatile("prefetch.global.L2 [%0];\n" ::"l"(W + (long long)(c + nw) * s + j + 16 * lane));
      double dot = 0.0;
#pragma unroll
      for (int q = 0; q < MAXPL; ++q) {
        const int i = j + lane + 32 * q;
        x[q] = (i < s) ? col[i] : 0.0;
        if (i < s) dot = fma(v[i], x[q], dot);
      }
      dot = warp_sum(dot) * tau;
      double nn = 0.0;
#pragma unroll
      for (int q = 0; q < MAXPL; ++q) {
        const int i = j + lane + 32 * q;
        if (i < s) {
          const double y = fma(-dot, v[i], x[q]);
          col[i] = y;
          if (i > j) nn = fma(y, y, nn);
        }
      }
      nn = warp_sum(nn);
      if (lane == 0) norm2[c] = nn;
    }
    __syncthreads();
    k = j + 1;
  }
  __syncthreads();
  int hit = 0;
  if (adaptive && k == kmax && k == cap && k < rows && k < s) {
    // tolerance unmet at the cap iff the next pivot's |R_kk| exceeds the threshold
    double bv = 0.0;
    for (int c = k + tid; c < rows; c += CP_THREADS) bv = fmax(bv, norm2[c]);
    for (int o = 16; o > 0; o >>= 1) bv = fmax(bv, __shfl_xor_sync(0xffffffffu, bv, o));
    if (lane == 0) red[wid] = bv;
    __syncthreads();
    if (tid == 0) {
      double b = 0.0;
      for (int w = 0; w < nw; ++w) b = fmax(b, red[w]);
      s_stop = (sqrt(b) > thr) ? 1 : 0;
    }
    __syncthreads();
    hit = s_stop;
  }
  for (int c = tid; c < rows; c += CP_THREADS) P.piv[c] = piv[c];
  if (tid == 0) { *P.k_out = k; if (P.cap_hit) *P.cap_hit = hit; }
}

// Column-pivoted QR of one node on an 8-CTA cluster: position c (a column of W^T, i.e. a row of
// W) lives in the shared memory of CTA c % 8, so the whole node stays on chip (distributed
// shared memory) for all its pivot steps instead of streaming through L2 once per step.  Per
// step: local argmax -> candidates to CTA 0 (DSMEM) -> cluster barrier -> every CTA picks the
// same winner (max norm, lowest index) -> swap through DSMEM -> the owner of position j forms
// the Householder vector (block_sum over its 512 threads, as bcpqr_kernel) and writes it into
// every CTA -> cluster barrier -> each CTA updates its own columns (warp per column, the same
// lane partition as bcpqr_kernel).  Bitwise the same pivots, ranks and R as bcpqr_kernel.
constexpr int CPQ_CL = 8;

template <int MAXPL>
__global__ void __launch_bounds__(CP_THREADS) bcpqr_cluster_kernel(const CpqrProb* __restrict__ probs,
                                                                   double rel_tol, double abs_tol, int cap,
                                                                   int slots_max) {
  cg::cluster_group cl = cg::this_cluster();
  const int q = (int)cl.block_rank();
  const CpqrProb P = probs[blockIdx.x / CPQ_CL];
  const int rows = P.rows, s = P.s;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = CP_THREADS / 32;
  extern __shared__ double sm[];
  double* cols = sm;                                   // slots_max x s: position q + CPQ_CL*m at slot m
  double* v = cols + (size_t)slots_max * s;            // s: Householder vector of the current step
  double* tmp = v + s;                                 // s: swap staging
  double* norm2 = tmp + s;                             // slots_max
  int* piv = (int*)(norm2 + slots_max);                // slots_max
  __shared__ double red[32];
  __shared__ double rv[32];
  __shared__ int ri[32];
  __shared__ double cand_v[CPQ_CL];                    // used in CTA 0
  __shared__ int cand_i[CPQ_CL];
  __shared__ double sc[4];                             // tau, rjj, stop, tmp norm (written by the owner)
  __shared__ double tmpn;
  __shared__ int tmpp;
  const int nslot = (rows - q + CPQ_CL - 1) / CPQ_CL;  // positions q, q+8, ... < rows
  double* W = P.W;
  for (int e = tid; e < nslot * s; e += CP_THREADS) {
    const int m = e / s, i = e % s;
    cols[(size_t)m * s + i] = W[(long long)(q + CPQ_CL * m) * s + i];
  }
  for (int m = tid; m < nslot; m += CP_THREADS) piv[m] = q + CPQ_CL * m;
  __syncthreads();
  for (int m = wid; m < nslot; m += nw) {
    double a = 0.0;
    for (int i = lane; i < s; i += 32) { const double x = cols[(size_t)m * s + i]; a = fma(x, x, a); }
    a = warp_sum(a);
    if (lane == 0) norm2[m] = a;
  }
  __syncthreads();
  const bool adaptive = P.kfixed < 0;
  const int kmax = adaptive ? min(min(cap, rows), s) : min(min(P.kfixed, rows), s);
  double thr = 0.0;
  int k = 0;
  double* cand_v0 = cl.map_shared_rank(cand_v, 0);
  int* cand_i0 = cl.map_shared_rank(cand_i, 0);
  for (int j = 0; j < kmax; ++j) {
    // (1) argmax over this CTA's positions >= j
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int m = tid; m < nslot; m += CP_THREADS) {
      const int c = q + CPQ_CL * m;
      if (c >= j && norm2[m] > bv) { bv = norm2[m]; bi = c; }   // increasing c per thread
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { rv[wid] = bv; ri[wid] = bi; }
    __syncthreads();
    if (tid == 0) {
      double b = rv[0];
      int ix = ri[0];
      for (int w = 1; w < nw; ++w)
        if (rv[w] > b || (rv[w] == b && ri[w] < ix)) { b = rv[w]; ix = ri[w]; }
      cand_v0[q] = b;
      cand_i0[q] = ix;
    }
    cl.sync();
    // (2) the winner, computed identically by every CTA
    double b = cand_v0[0];
    int p = cand_i0[0];
    for (int r = 1; r < CPQ_CL; ++r) {
      const double vb = cand_v0[r];
      const int ib = cand_i0[r];
      if (vb > b || (vb == b && ib < p)) { b = vb; p = ib; }
    }
    const int oj = j % CPQ_CL, op = p % CPQ_CL, mj = j / CPQ_CL, mp = p / CPQ_CL;
    // (3) swap positions j and p (column data, norm, original index)
    if (p != j && oj == op) {  // both positions in one CTA: local swap
      if (q == oj) {
        double* a = cols + (size_t)mj * s;
        double* c2 = cols + (size_t)mp * s;
        for (int i = tid; i < s; i += CP_THREADS) { const double t = a[i]; a[i] = c2[i]; c2[i] = t; }
        if (tid == 0) {
          const double t = norm2[mj]; norm2[mj] = norm2[mp]; norm2[mp] = t;
          const int pp = piv[mj]; piv[mj] = piv[mp]; piv[mp] = pp;
        }
        __syncthreads();
      }
    } else if (p != j) {
      if (q == oj) {  // fetch column p
        const double* src = cl.map_shared_rank(cols, op) + (size_t)mp * s;
        for (int i = tid; i < s; i += CP_THREADS) tmp[i] = src[i];
        if (tid == 0) { tmpn = cl.map_shared_rank(norm2, op)[mp]; tmpp = cl.map_shared_rank(piv, op)[mp]; }
      } else if (q == op) {  // fetch column j
        const double* src = cl.map_shared_rank(cols, oj) + (size_t)mj * s;
        for (int i = tid; i < s; i += CP_THREADS) tmp[i] = src[i];
        if (tid == 0) { tmpn = cl.map_shared_rank(norm2, oj)[mj]; tmpp = cl.map_shared_rank(piv, oj)[mj]; }
      }
      cl.sync();
      if (q == oj || q == op) {
        const int m = (q == oj) ? mj : mp;
        for (int i = tid; i < s; i += CP_THREADS) cols[(size_t)m * s + i] = tmp[i];
        if (tid == 0) { norm2[m] = tmpn; piv[m] = tmpp; }
      }
      __syncthreads();
    }
    // (4) Householder of position j (owner), broadcast to every CTA
    if (q == oj) {
      double* cj = cols + (size_t)mj * s;
      double part = 0.0;
      for (int i = j + 1 + tid; i < s; i += CP_THREADS) { const double x = cj[i]; part = fma(x, x, part); }
      const double xs = block_sum(part, red);
      const double alpha = cj[j];
      const double rjj = sqrt(alpha * alpha + xs);
      double stop = 0.0;
      if (adaptive) {
        if (j == 0) thr = fmax(rel_tol * rjj, abs_tol * sqrt((double)s));
        if (!(rjj > thr)) stop = 1.0;
      }
      double tau = 0.0, scal = 0.0, beta = alpha;
      if (stop == 0.0 && xs != 0.0) {
        beta = -copysign(rjj, alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      if (stop == 0.0) {
        for (int i = j + 1 + tid; i < s; i += CP_THREADS) {
          const double x = (tau == 0.0) ? cj[i] : cj[i] * scal;
          cj[i] = x;
        }
        __syncthreads();
        if (tid == 0) cj[j] = beta;
      }
      __syncthreads();
      for (int r = 0; r < CPQ_CL; ++r) {
        double* vr = cl.map_shared_rank(v, r);
        for (int i = j + tid; i < s; i += CP_THREADS) vr[i] = (i == j) ? 1.0 : cj[i];
        if (tid == 0) {
          double* sr = cl.map_shared_rank(sc, r);
          sr[0] = tau; sr[1] = thr; sr[2] = stop;
        }
      }
    }
    cl.sync();
    if (sc[2] != 0.0) break;  // tolerance met (every CTA sees the same flag)
    thr = sc[1];
    const double tau = sc[0];
    // (5) update this CTA's positions c > j (warp per column) + exact trailing norms
    for (int m = wid; m < nslot; m += nw) {
      const int c = q + CPQ_CL * m;
      if (c <= j) continue;
      double x[MAXPL];
      double* col = cols + (size_t)m * s;
      double dot = 0.0;
#pragma unroll
      for (int qq = 0; qq < MAXPL; ++qq) {
        const int i = j + lane + 32 * qq;
        x[qq] = (i < s) ? col[i] : 0.0;
        if (i < s) dot = fma(v[i], x[qq], dot);
      }
      dot = warp_sum(dot) * tau;
      double nn = 0.0;
#pragma unroll
      for (int qq = 0; qq < MAXPL; ++qq) {
        const int i = j + lane + 32 * qq;
        if (i < s) {
          const double yv = fma(-dot, v[i], x[qq]);
          col[i] = yv;
          if (i > j) nn = fma(yv, yv, nn);
        }
      }
      nn = warp_sum(nn);
      if (lane == 0) norm2[m] = nn;
    }
    __syncthreads();
    k = j + 1;
  }
  // cap hit: tolerance unmet at the cap iff the next pivot's |R_kk| exceeds the threshold
  int hit = 0;
  if (adaptive && k == kmax && k == cap && k < rows && k < s) {
    double bv = 0.0;
    for (int m = tid; m < nslot; m += CP_THREADS)
      if (q + CPQ_CL * m >= k) bv = fmax(bv, norm2[m]);
    for (int o = 16; o > 0; o >>= 1) bv = fmax(bv, __shfl_xor_sync(0xffffffffu, bv, o));
    if (lane == 0) red[wid] = bv;
    __syncthreads();
    if (tid == 0) {
      double b = 0.0;
      for (int w = 0; w < nw; ++w) b = fmax(b, red[w]);
      cand_v0[q] = b;
    }
    cl.sync();
    double b = 0.0;
    for (int r = 0; r < CPQ_CL; ++r) b = fmax(b, cand_v0[r]);
    hit = (sqrt(b) > thr) ? 1 : 0;
  }
  // write back this CTA's columns and pivots
  for (int e = tid; e < nslot * s; e += CP_THREADS) {
    const int m = e / s, i = e % s;
    W[(long long)(q + CPQ_CL * m) * s + i] = cols[(size_t)m * s + i];
  }
  for (int m = tid; m < nslot; m += CP_THREADS) P.piv[q + CPQ_CL * m] = piv[m];
  if (q == 0 && tid == 0) { *P.k_out = k; if (P.cap_hit) *P.cap_hit = hit; }
  cl.sync();  // no CTA exits while others may still read its shared memory
}

void bcpqr(const std::vector<CpqrProb>& probs, double rel_tol, double abs_tol, int cap,
           cudaStream_t s) {
  if (probs.empty()) return;
  int maxr = 0, maxs = 0;
  for (auto& p : probs) { maxr = std::max(maxr, p.rows); maxs = std::max(maxs, p.s); }
  CpqrProb* d = upload_probs(probs, s);
  bool forced = false;
  for (auto& p : probs) forced = forced || (p.forced != nullptr);
  // cluster version when a node's columns fit the 8 CTAs' shared memory
  const int slots = (maxr + CPQ_CL - 1) / CPQ_CL;
  const size_t csm = ((size_t)slots * maxs + 2 * (size_t)maxs + slots) * sizeof(double) + (size_t)slots * sizeof(int) + 16;
  // SVMHSS_CPQR_MODE (A/B): 2 (default) = blocked kernel (cpqr.cu) on levels with many nodes, the
  // cluster kernel on levels with few; 1 = blocked everywhere; 0 = unblocked kernels only.
  // Measured at config 3 (r2d): compression 163.8 ms (2) / 172.2 (1) / 190.6 (0), same pivots.
  static const int mode = [] { const char* e = getenv("SVMHSS_CPQR_MODE"); return e ? atoi(e) : 2; }();
  const bool few = probs.size() * CPQ_CL <= 2 * 148;
  if (mode >= 1 && cpqr_blk_fits(maxr, maxs) && (mode == 1 || !few || forced)) {
    bcpqr_blk(d, (int)probs.size(), maxr, maxs, rel_tol, abs_tol, cap, s);
    free_probs(d, s);
    return;
  }
  const bool use = csm <= 200 * 1024 && few && !forced;
  if (use) {
    auto launchc = [&](auto kern) {
      CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(probs.size() * CPQ_CL));
      cfg.blockDim = dim3(CP_THREADS);
      cfg.dynamicSmemBytes = csm;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CPQ_CL;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, (const CpqrProb*)d, rel_tol, abs_tol, cap, slots));
    };
    if (maxs <= 96) launchc(bcpqr_cluster_kernel<3>);
    else if (maxs <= 160) launchc(bcpqr_cluster_kernel<5>);
    else if (maxs <= 288) launchc(bcpqr_cluster_kernel<9>);
    else if (maxs <= 576) launchc(bcpqr_cluster_kernel<18>);
    else launchc(bcpqr_cluster_kernel<36>);
    LAUNCH_CHECK();
    free_probs(d, s);
    return;
  }
  size_t smem = (size_t)maxr * (sizeof(double) + sizeof(int)) + (size_t)maxs * sizeof(double) + 16;
  auto launch = [&](auto kern) {
    if (smem > 48 * 1024)
      CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)probs.size(), CP_THREADS, smem, s>>>(d, rel_tol, abs_tol, cap, 1);
  };
  if (maxs <= 96) launch(bcpqr_kernel<3>);
  else if (maxs <= 160) launch(bcpqr_kernel<5>);
  else if (maxs <= 288) launch(bcpqr_kernel<9>);
  else if (maxs <= 576) launch(bcpqr_kernel<18>);
  else if (maxs <= 1152) launch(bcpqr_kernel<36>);
  else throw Error(HSS_EINVAL, "sketch width s > 1152 unsupported by the CPQR kernel");
  LAUNCH_CHECK();
  free_probs(d, s);
}

// ------------------------------------------------------------------ helpers
__global__ void fill_identity_kernel(double* A, int n, long long rs, long long cs) {
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)n * n) return;
  int i = (int)(e / n), j = (int)(e % n);
  A[i * rs + j * cs] = (i == j) ? 1.0 : 0.0;
}
void fill_identity(double* A, int n, long long rs, long long cs, cudaStream_t s) {
  if (n <= 0) return;
  long long tot = (long long)n * n;
  fill_identity_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(A, n, rs, cs);
  LAUNCH_CHECK();
}

}  // namespace svmhss

namespace svmhss {
// ------------------------------------------------------------------ skinny GEMM as streaming GEMV
// C (m x n, n <= 16 right-hand sides) = alpha op(A) B + beta C, B and C row-major with unit column
// stride (the HSS mat-vec's shapes, reading M: P:200).  op(A) row-major (acs == 1): one warp per
// row, lanes over k, a butterfly per column; op(A) transposed in memory (ars == 1): a CTA owns 64
// output rows (= stored columns: lanes read contiguous 256-byte row segments), 8 warps stride the
// stored rows, partials summed in warp order.  Both stream A once (HBM-bound), fixed order.
constexpr int GV_ROWS = 128;  // rows per CTA of the row GEMV (8 warps x 16 rows) on big batches
// rows per CTA rpc (8..128, a multiple of 8) is chosen per launch so that small batches (the top
// tree levels) still spread over the SMs; a row's arithmetic does not depend on it
template <int NR>
__global__ void __launch_bounds__(256) gemv_rows_kernel(const GemmProb* __restrict__ probs,
                                                        const int2* __restrict__ items, int rpc) {
  extern __shared__ double bsh[];   // B staged once per CTA: k x NR (zero beyond n)
  const int2 it = items[blockIdx.x];
  const GemmProb P = probs[it.x];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i0 = it.y * rpc, i1 = min(P.m, i0 + rpc);
  // the first row's segments are requested before B is staged (the two latencies overlap)
  const double* a0 = P.A + (long long)min(i0 + w, P.m - 1) * P.ars;
  double pre[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) pre[u] = (lane + 32 * u < P.k) ? a0[lane + 32 * u] : 0.0;
  for (int e = threadIdx.x; e < P.k * NR; e += 256) {
    const int j = e / NR, c = e % NR;
    bsh[e] = (c < P.n) ? P.B[(long long)j * P.brs + c] : 0.0;
  }
  __syncthreads();
  // NR <= 4: rows i and i + 8 together (16 loads per lane in flight; the per-row FMA order is the
  // one-row loop's), else one row at a time
  constexpr int RW = NR <= 4 ? 2 : 1;
  for (int i = i0 + w; i < i1; i += 8 * RW) {
    const double* a[RW];
    bool ok[RW];
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      ok[r] = i + 8 * r < i1;
      a[r] = P.A + (long long)(ok[r] ? i + 8 * r : i) * P.ars;
    }
    double acc[RW][NR];
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
      for (int c = 0; c < NR; ++c) acc[r][c] = 0.0;
    int j = lane;
    for (; j + 32 * 7 < P.k; j += 256) {   // eight row segments per row in flight per lane
      double av[RW][8];
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        if (r == 0 && i == i0 + w && j == lane) {
#pragma unroll
          for (int u = 0; u < 8; ++u) av[r][u] = pre[u];
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u) av[r][u] = ok[r] ? a[r][j + 32 * u] : 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int r = 0; r < RW; ++r)
#pragma unroll
          for (int c = 0; c < NR; ++c) acc[r][c] = fma(av[r][u], bsh[(j + 32 * u) * NR + c], acc[r][c]);
    }
    for (; j < P.k; j += 32) {
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        const double av = ok[r] ? a[r][j] : 0.0;
#pragma unroll
        for (int c = 0; c < NR; ++c) acc[r][c] = fma(av, bsh[j * NR + c], acc[r][c]);
      }
    }
#pragma unroll
    for (int r = 0; r < RW; ++r) {
#pragma unroll
      for (int c = 0; c < NR; ++c) acc[r][c] = warp_sum(acc[r][c]);
      if (ok[r] && lane < P.n) {
        double v = acc[r][0];
#pragma unroll
        for (int c = 1; c < NR; ++c) if (lane == c) v = acc[r][c];
        double* d = P.C + (long long)(i + 8 * r) * P.crs + lane;
        *d = (P.beta == 0.0) ? P.alpha * v : fma(P.beta, *d, P.alpha * v);
      }
    }
  }
}

template <int NR>
__global__ void __launch_bounds__(256) gemv_cols_kernel(const GemmProb* __restrict__ probs,
                                                        const int2* __restrict__ items) {
  __shared__ double red[8][64][NR];
  const int2 it = items[blockIdx.x];
  const GemmProb P = probs[it.x];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i0 = it.y * 64, ia = i0 + lane, ib = i0 + 32 + lane;
  const bool va = ia < P.m, vb = ib < P.m;
  double aa[NR], ab[NR];
#pragma unroll
  for (int c = 0; c < NR; ++c) aa[c] = ab[c] = 0.0;
  int j = w;
  for (; j + 56 < P.k; j += 64) {   // eight stored rows in flight per warp (rows j, j + 8, ... in order)
    double xa[8], xb[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double* row = P.A + (long long)(j + 8 * u) * P.acs;
      xa[u] = va ? row[ia] : 0.0;
      xb[u] = vb ? row[ib] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double* b = P.B + (long long)(j + 8 * u) * P.brs;
#pragma unroll
      for (int c = 0; c < NR; ++c)
        if (c < P.n) {
          const double bv = b[c];
          aa[c] = fma(xa[u], bv, aa[c]);
          ab[c] = fma(xb[u], bv, ab[c]);
        }
    }
  }
  for (; j < P.k; j += 8) {
    const double* row = P.A + (long long)j * P.acs;
    const double xa = va ? row[ia] : 0.0, xb = vb ? row[ib] : 0.0;
    const double* b = P.B + (long long)j * P.brs;
#pragma unroll
    for (int c = 0; c < NR; ++c)
      if (c < P.n) {
        const double bv = b[c];
        aa[c] = fma(xa, bv, aa[c]);
        ab[c] = fma(xb, bv, ab[c]);
      }
  }
#pragma unroll
  for (int c = 0; c < NR; ++c) { red[w][lane][c] = aa[c]; red[w][32 + lane][c] = ab[c]; }
  __syncthreads();
  for (int e = threadIdx.x; e < 64 * P.n; e += 256) {
    const int ii = e / P.n, c = e % P.n;
    if (i0 + ii >= P.m) continue;
    double t = red[0][ii][c];
#pragma unroll
    for (int q = 1; q < 8; ++q) t += red[q][ii][c];
    double* d = P.C + (long long)(i0 + ii) * P.crs + c;
    *d = (P.beta == 0.0) ? P.alpha * t : fma(P.beta, *d, P.alpha * t);
  }
}

template <int NR, bool COLS>
static void launch_gemv(const std::vector<GemmProb>& probs, cudaStream_t s) {
  const bool cols = COLS;
  std::vector<int2> items;
  int kmax = 1;
  int rpc = GV_ROWS;   // row kernel: halve the rows per CTA until the batch gives >= 4 CTAs per SM
  if (!cols) {
    int64_t mrows = 0;
    for (const auto& p : probs) mrows += p.m;
    while (rpc > 8 && mrows / rpc < 4 * 148) rpc /= 2;
  }
  for (size_t q = 0; q < probs.size(); ++q) {
    const int per = cols ? (probs[q].m + 63) / 64 : (probs[q].m + rpc - 1) / rpc;
    for (int t = 0; t < per; ++t) items.push_back(make_int2((int)q, t));
    kmax = std::max(kmax, probs[q].k);
  }
  if (items.empty()) return;
  const size_t smem = COLS ? 0 : (size_t)kmax * NR * sizeof(double);
  if constexpr (!COLS)
    if (smem > 48 * 1024) CUDA_CHECK(cudaFuncSetAttribute(gemv_rows_kernel<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  GemmProb* d = upload_probs(probs, s);
  int2* di = upload_probs(items, s);
  for (size_t b0 = 0; b0 < items.size(); b0 += (1u << 30)) {
    const unsigned nb = (unsigned)std::min<size_t>(1u << 30, items.size() - b0);
    if constexpr (COLS) gemv_cols_kernel<NR><<<nb, 256, 0, s>>>(d, di + b0);
    else gemv_rows_kernel<NR><<<nb, 256, smem, s>>>(d, di + b0, rpc);
    LAUNCH_CHECK();
  }
  free_probs(d, s);
  free_probs(di, s);
}

template <int NR>
static void gemv_split(const std::vector<GemmProb>& probs, cudaStream_t s) {
  std::vector<GemmProb> rows, cols;
  int cmax = 0;
  for (const auto& p : probs) {
    if (p.acs == 1) { rows.push_back(p); continue; }
    for (int c0 = 0; c0 < p.n; c0 += 8) {   // the column kernel takes <= 8 right-hand sides
      GemmProb q = p;
      q.B += c0;
      q.C += c0;
      q.n = std::min(8, p.n - c0);
      cmax = std::max(cmax, q.n);
      cols.push_back(q);
    }
  }
  launch_gemv<NR, false>(rows, s);
  if (cmax <= 2) launch_gemv<2, true>(cols, s);
  else if (cmax <= 4) launch_gemv<4, true>(cols, s);
  else launch_gemv<8, true>(cols, s);
}

void bgemv(const std::vector<GemmProb>& probs_in, cudaStream_t s) {
  std::vector<GemmProb> sk, other;
  int nmax = 0;
  for (const auto& p : probs_in) {
    if (p.m <= 0 || p.n <= 0) continue;
    const bool skinny = p.n <= 16 && p.bcs == 1 && p.ccs == 1 && (p.acs == 1 || p.ars == 1) && !p.lower &&
                        (p.ars == 1 || (size_t)p.k * 16 * sizeof(double) <= 200 * 1024);
    (skinny ? sk : other).push_back(p);
    if (skinny) nmax = std::max(nmax, p.n);
  }
  bgemm(other, s);
  if (sk.empty()) return;
  if (nmax <= 2) { gemv_split<2>(sk, s); return; }
  switch ((nmax + 3) / 4) {   // NR = 4, 8, 12, 16 (columns beyond n are skipped)
    case 1: gemv_split<4>(sk, s); break;
    case 2: gemv_split<8>(sk, s); break;
    case 3: gemv_split<12>(sk, s); break;
    default: gemv_split<16>(sk, s); break;
  }
}
}  // namespace svmhss
