// solve_dev.cuh — device functions of the ULV solve sweeps (ulv.cu).  Forward sweep t = M_t b (rows i < k -> the parent's input "up", rows >= k -> y_r);
// backward sweep x = M_t^T [x_s; y_r], both streaming the same stored M_t (no transposed copy):
//  - fwd_rows: one warp per row, lane-strided partial sums + butterfly;
//  - bwd_cols: a CTA of kBW warps owns kCW consecutive columns (lane l -> columns j0 + l and
//    j0 + 32 + l: fully coalesced row segments); warp w accumulates rows w, w + kBW, ... in
//    order; the kBW warp partials are summed in warp order.
// The summation order of every output element depends only on the node's shape.
#pragma once
#include "internal.cuh"

// rows in flight per warp in the backward column GEMV (A/B at config 3: 8 -> 1.405 ms per ADMM
// iteration, 4 -> 1.425, 16 -> 1.447)
#ifndef BWD_BQ
#define BWD_BQ 8
#endif

namespace svmhss {

// one row's lane-partial dot product: lane sums j = lane, lane + 32, ... in order
// QN loads per row in flight (lane-strided, 32 QN columns per pass); the per-element order
// (j = lane, lane + 32, ... sequentially) does not depend on RU or QN
template <int NR, int RU, int QN = 4>
__device__ __forceinline__ void row_partials(const double* const (&Mr)[RU], int R, const double* __restrict__ vsh,
                                             double (&acc)[RU][NR]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int u = 0; u < RU; ++u)
#pragma unroll
    for (int c = 0; c < NR; ++c) acc[u][c] = 0.0;
  int j = lane;
  for (; j + 32 * (QN - 1) < R; j += 32 * QN) {
    double m[RU][QN];
#pragma unroll
    for (int u = 0; u < RU; ++u)
#pragma unroll
      for (int q = 0; q < QN; ++q) m[u][q] = Mr[u][j + 32 * q];
#pragma unroll
    for (int u = 0; u < RU; ++u)
#pragma unroll
      for (int q = 0; q < QN; ++q)
#pragma unroll
        for (int c = 0; c < NR; ++c) acc[u][c] = fma(m[u][q], vsh[(j + 32 * q) * NR + c], acc[u][c]);
  }
  for (; j < R; j += 32) {
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      const double m0 = Mr[u][j];
#pragma unroll
      for (int c = 0; c < NR; ++c) acc[u][c] = fma(m0, vsh[j * NR + c], acc[u][c]);
    }
  }
}

template <int NR>
__device__ __forceinline__ void row_store(double (&acc)[NR], int i, int k, int64_t koff, int64_t yoff,
                                          double* __restrict__ out_up, double* __restrict__ out_yr) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int c = 0; c < NR; ++c) acc[c] = warp_sum(acc[c]);
  if (lane < NR) {
    double v = acc[0];
#pragma unroll
    for (int c = 1; c < NR; ++c) if (lane == c) v = acc[c];
    if (i < k) out_up[(koff + i) * NR + lane] = v;
    else out_yr[(yoff + i - k) * NR + lane] = v;
  }
}

// rows i0 + wid, i0 + wid + nw, ... < i1.  NR <= 2: one row per warp with all 16 loads per lane
// in flight (4 KB contiguous per round trip) plus an L2 prefetch of the warp's next row (A/B at
// config 3: 1.431 ms/iteration vs 1.543 with four rows x 4 loads and 1.501 with two rows x 4);
// NR > 2: two rows per warp (4 loads each).  The per-element order is the same either way.
template <int NR>
__device__ __forceinline__ void fwd_rows(const double* __restrict__ M, int R, const double* __restrict__ vsh,
                                         int i0, int i1, int wid, int nw, int k, int64_t koff, int64_t yoff,
                                         double* __restrict__ out_up, double* __restrict__ out_yr) {
  int i = i0 + wid;
  if constexpr (NR <= 2) {
    for (; i < i1; i += nw) {
      const double* Mr[1] = {M + (int64_t)i * R};
      if (i + nw < i1 && 16 * (threadIdx.x & 31) < R)
        asm volatile("prefetch.global.L2 [%0];\n" ::"l"(M + (int64_t)(i + nw) * R + 16 * (threadIdx.x & 31)));
      double acc[1][NR];
      row_partials<NR, 1, 16>(Mr, R, vsh, acc);
      row_store<NR>(acc[0], i, k, koff, yoff, out_up, out_yr);
    }
  } else {
    for (; i + nw < i1; i += 2 * nw) {
      const double* Mr[2] = {M + (int64_t)i * R, M + (int64_t)(i + nw) * R};
      double acc[2][NR];
      row_partials<NR, 2>(Mr, R, vsh, acc);
      row_store<NR>(acc[0], i, k, koff, yoff, out_up, out_yr);
      row_store<NR>(acc[1], i + nw, k, koff, yoff, out_up, out_yr);
    }
    if (i < i1) {
      const double* Mr[1] = {M + (int64_t)i * R};
      double acc[1][NR];
      row_partials<NR, 1>(Mr, R, vsh, acc);
      row_store<NR>(acc[0], i, k, koff, yoff, out_up, out_yr);
    }
  }
}

// fwd_rows for short rows (R <= 256, NR <= 2: the leaves): two rows per warp per pass, 8 loads
// each, so all loads of both rows are in flight at once (fwd_rows' one-row mode would leave half
// of its 16 lane loads idle).  Same per-row FMA order.
template <int NR>
__device__ __forceinline__ void fwd_rows_short(const double* __restrict__ M, int R, const double* __restrict__ vsh,
                                               int i0, int i1, int wid, int nw, int k, int64_t koff, int64_t yoff,
                                               double* __restrict__ out_up, double* __restrict__ out_yr) {
  int i = i0 + wid;
  for (; i + nw < i1; i += 2 * nw) {
    const double* Mr[2] = {M + (int64_t)i * R, M + (int64_t)(i + nw) * R};
    double acc[2][NR];
    row_partials<NR, 2, 8>(Mr, R, vsh, acc);
    row_store<NR>(acc[0], i, k, koff, yoff, out_up, out_yr);
    row_store<NR>(acc[1], i + nw, k, koff, yoff, out_up, out_yr);
  }
  if (i < i1) {
    const double* Mr[1] = {M + (int64_t)i * R};
    double acc[1][NR];
    row_partials<NR, 1, 8>(Mr, R, vsh, acc);
    row_store<NR>(acc[0], i, k, koff, yoff, out_up, out_yr);
  }
}

// x[j] for j in [j0, min(R, j0 + kCW)); ush = u (R x NR) in shared memory; red: kBW*kCW*NR
// doubles of shared scratch.  Must be called by all kBW*32 threads of the CTA.
// tig: the thread's index within its group of kBW*32 threads (several groups of one CTA may run
// different column chunks at once; every thread of the CTA must call this the same number of
// times).  idle: a group with no chunk (still takes part in the CTA barriers).
// first-batch preload for bwd_cols (rows wid + q kBW, q < BWD_BQ, of this thread's two columns),
// issued before a dependency wait; pass the arrays as pre_a / pre_b.
__device__ __forceinline__ void bwd_cols_preload(const double* __restrict__ M, int R, int j0, double* pa,
                                                 double* pb, int tig = -1) {
  if (tig < 0) tig = threadIdx.x;
  const int lane = tig & 31, wid = tig >> 5;
  const int ja = j0 + lane, jb = j0 + 32 + lane;
#pragma unroll
  for (int q = 0; q < BWD_BQ; ++q) {
    const int i = wid + q * kBW;
    const bool ok = (BWD_BQ - 1) * kBW < R;
    const double* Mr = M + (int64_t)i * R;
    pa[q] = (ok && ja < R) ? Mr[ja] : 0.0;
    pb[q] = (ok && jb < R) ? Mr[jb] : 0.0;
  }
}

template <int NR>
__device__ __forceinline__ void bwd_cols(const double* __restrict__ M, int R, const double* __restrict__ ush,
                                         int j0, double* __restrict__ red, double* __restrict__ out,
                                         int tig = -1, bool idle = false, const double* pre_a = nullptr,
                                         const double* pre_b = nullptr) {
  if (tig < 0) tig = threadIdx.x;
  const int lane = tig & 31, wid = tig >> 5;
  if (idle) {
    __syncthreads();
    __syncthreads();
    return;
  }
  const int ja = j0 + lane, jb = j0 + 32 + lane;
  const bool va = ja < R, vb = jb < R;
  double aa[NR], ab[NR];
#pragma unroll
  for (int c = 0; c < NR; ++c) aa[c] = ab[c] = 0.0;
  int i = wid;
  // BQ rows in flight per warp (16 loads / lane at BQ = 8); the per-column order (rows i, i + kBW,
  // ... sequentially) does not depend on BQ
  constexpr int BQ = BWD_BQ;
  if (pre_a) {  // the first batch was loaded by the caller (before its dependency wait)
    if ((BQ - 1) * kBW < R) {
#pragma unroll
      for (int q = 0; q < BQ; ++q)
#pragma unroll
        for (int c = 0; c < NR; ++c) {
          const double u = ush[(i + q * kBW) * NR + c];
          aa[c] = fma(pre_a[q], u, aa[c]);
          ab[c] = fma(pre_b[q], u, ab[c]);
        }
      i += BQ * kBW;
    }
  }
  for (; i + (BQ - 1) * kBW < R; i += BQ * kBW) {
    double ma[BQ], mb[BQ];
#pragma unroll
    for (int q = 0; q < BQ; ++q) {
      const double* Mr = M + (int64_t)(i + q * kBW) * R;
      ma[q] = va ? Mr[ja] : 0.0;
      mb[q] = vb ? Mr[jb] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < BQ; ++q)
#pragma unroll
      for (int c = 0; c < NR; ++c) {
        const double u = ush[(i + q * kBW) * NR + c];
        aa[c] = fma(ma[q], u, aa[c]);
        ab[c] = fma(mb[q], u, ab[c]);
      }
  }
  for (; i < R; i += kBW) {
    const double* Mr = M + (int64_t)i * R;
    const double ma = va ? Mr[ja] : 0.0, mb = vb ? Mr[jb] : 0.0;
#pragma unroll
    for (int c = 0; c < NR; ++c) {
      const double u = ush[i * NR + c];
      aa[c] = fma(ma, u, aa[c]);
      ab[c] = fma(mb, u, ab[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < NR; ++c) {
    red[(wid * kCW + lane) * NR + c] = aa[c];
    red[(wid * kCW + 32 + lane) * NR + c] = ab[c];
  }
  __syncthreads();
  for (int e = tig; e < kCW * NR; e += kBW * 32) {
    const int jj = e / NR, c = e % NR;
    if (j0 + jj < R) {
      double t = red[jj * NR + c];
#pragma unroll
      for (int w = 1; w < kBW; ++w) t += red[(w * kCW + jj) * NR + c];
      out[(int64_t)(j0 + jj) * NR + c] = t;
    }
  }
  __syncthreads();
}

}  // namespace svmhss
