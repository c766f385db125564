// cpqr.cu — column-pivoted Householder QR of Y_t^T with the AMB-10 rank rule (reading H3;
// P:184 [MR2854612] randomized interpolative decomposition), blocked as LAPACK's dgeqp3/dlaqps.
//
// One CTA per tree node.  A = W^T (s x rows; column c of A = row c of W, contiguous).  Panels of
// up to NB pivot steps; step j (panel column kk, panel start j0):
//   1. pivot p = argmax_{c >= j} vn1[c] (ties -> lowest position), or the imported skeleton's
//      j-th column (fixed-skeleton mode); swap columns j, p (W rows, F rows, norms, piv)
//   2. pending panel update of the pivot column only: a = A(j:, j) - V(j:, 0:kk) F(j, 0:kk)^T
//   3. Householder (dlarfg) of a: beta, tau, v; |R_jj| = |beta| decides the adaptive rank
//   4. F(c, kk) = tau A(j:, c)^T v + F(c, 0:kk) aux,  aux = -tau V(j:, 0:kk)^T v     (c > j)
//      -- one READ-ONLY pass over the trailing columns (A(j:, c) is as of the panel start)
//   5. row update A(j, c) -= V(j, 0:kk+1) F(c, 0:kk+1)^T   (rows < j+1 of column c are final)
//   6. norm downdate vn1[c] *= sqrt(1 - (A(j,c)/vn1[c])^2), or recompute after the panel when
//      cancellation makes it inaccurate (LAPACK's tol3z = sqrt(eps) test; the panel then ends)
// After a panel: A(j:, c) -= V(j:, 0:nb) F(c, 0:nb)^T for the trailing columns (one read+write
// pass per panel instead of one per pivot step as in unblocked Householder CPQR).
// Output (as the unblocked kernel): W column j (< k) holds R(0:j, j), beta at row j; columns
// c >= k hold R(0:k, c) in rows 0..k-1; piv[c] = original column at position c; k; cap hit.
// Pivots follow the same norm argmax as the oracle's LAPACK dgeqp3 (identical unless two
// candidates are within rounding of each other: AMB-12, checked bit-exact by the tests).
#include <cstdlib>
#include "dense.cuh"

namespace svmhss {

constexpr int CB_THREADS = 256, CB_WARPS = CB_THREADS / 32;

template <int MAXPL, int NB>
__global__ void __launch_bounds__(CB_THREADS, 3) bcpqr_blk_kernel(const CpqrProb* __restrict__ probs,
                                                                  double rel_tol, double abs_tol, int cap) {
  const CpqrProb P = probs[blockIdx.x];
  const int rows = P.rows, s = P.s;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  extern __shared__ double sm[];
  double* vn1 = sm;                          // rows: partial column norms (pivoting)
  double* vn2 = vn1 + rows;                  // rows: reference norms (downdate accuracy test)
  double* Fm = vn2 + rows;                   // rows x NB: F(c, q)
  double* Vp = Fm + (size_t)rows * NB;       // NB x s: panel reflectors, Vp[q*s + i] (i >= j0+q)
  int* piv = (int*)(Vp + (size_t)NB * s);    // rows: original column at each position
  int* pos = piv + rows;                     // rows: position of each original column
  int* flag = pos + rows;                    // rows: 1 = norm to be recomputed after the panel
  __shared__ double red[32];
  __shared__ double aux[NB];
  __shared__ int s_p, s_any;
  double* W = P.W;
  const double tol3z = 1.4901161193847656e-08;  // sqrt(eps), LAPACK dlaqps
  for (int c = wid; c < rows; c += CB_WARPS) {
    const double* col = W + (size_t)c * s;
    double a = 0.0;
    for (int i = lane; i < s; i += 32) { const double x = col[i]; a = fma(x, x, a); }
    a = warp_sum(a);
    if (lane == 0) { vn1[c] = sqrt(a); vn2[c] = vn1[c]; }
  }
  for (int c = tid; c < rows; c += CB_THREADS) { piv[c] = c; pos[c] = c; flag[c] = 0; }
  if (tid == 0) s_any = 0;
  __syncthreads();
  const bool adaptive = P.kfixed < 0;
  const int kmax = adaptive ? min(min(cap, rows), s) : min(min(P.kfixed, rows), s);
  double thr = 0.0;
  int j = 0;
  bool stop = false;
  while (j < kmax && !stop) {
    int kk = 0;
    while (true) {
      // ---- 1. pivot
      if (P.forced) {
        if (tid == 0) s_p = pos[P.forced[j]];
      } else {
        double bv = -1.0;
        int bi = 0x7fffffff;
        for (int c = j + tid; c < rows; c += CB_THREADS) {
          const double x = vn1[c];
          if (x > bv) { bv = x; bi = c; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
        }
        __shared__ double rv[CB_WARPS];
        __shared__ int ri[CB_WARPS];
        if (lane == 0) { rv[wid] = bv; ri[wid] = bi; }
        __syncthreads();
        if (tid == 0) {
          double b = rv[0];
          int ix = ri[0];
          for (int w = 1; w < CB_WARPS; ++w)
            if (rv[w] > b || (rv[w] == b && ri[w] < ix)) { b = rv[w]; ix = ri[w]; }
          s_p = ix;
        }
      }
      __syncthreads();
      const int p = s_p;
      if (p != j) {
        for (int i = tid; i < s; i += CB_THREADS) {
          const double a = W[(size_t)j * s + i];
          W[(size_t)j * s + i] = W[(size_t)p * s + i];
          W[(size_t)p * s + i] = a;
        }
        for (int q = tid; q < kk; q += CB_THREADS) {
          const double a = Fm[j * NB + q];
          Fm[j * NB + q] = Fm[p * NB + q];
          Fm[p * NB + q] = a;
        }
        if (tid == 0) {
          double t = vn1[j]; vn1[j] = vn1[p]; vn1[p] = t;
          t = vn2[j]; vn2[j] = vn2[p]; vn2[p] = t;
          const int a = piv[j], b = piv[p];
          piv[j] = b; piv[p] = a;
          pos[b] = j; pos[a] = p;
          const int f = flag[j]; flag[j] = flag[p]; flag[p] = f;
        }
      }
      __syncthreads();
      // ---- 2-3. pivot column with the pending panel update, Householder (dlarfg)
      double* vk = Vp + (size_t)kk * s;
      double part = 0.0;
      for (int i = j + tid; i < s; i += CB_THREADS) {
        double x = W[(size_t)j * s + i];
        for (int q = 0; q < kk; ++q) x = fma(-Vp[(size_t)q * s + i], Fm[j * NB + q], x);
        vk[i] = x;
        if (i > j) part = fma(x, x, part);
      }
      const double xs = block_sum(part, red);
      const double alpha = vk[j];
      const double rjj = sqrt(alpha * alpha + xs);
      if (adaptive) {
        if (j == 0) thr = fmax(rel_tol * rjj, abs_tol * sqrt((double)s));
        if (!(rjj > thr)) { stop = true; break; }
      }
      double tau, scal, beta;
      if (xs == 0.0) { tau = 0.0; scal = 1.0; beta = alpha; }
      else {
        beta = -copysign(rjj, alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      for (int i = j + 1 + tid; i < s; i += CB_THREADS) {
        const double v = vk[i] * scal;
        vk[i] = v;
        W[(size_t)j * s + i] = v;
      }
      __syncthreads();
      if (tid == 0) { vk[j] = 1.0; W[(size_t)j * s + j] = beta; }
      // ---- 4a. aux = -tau V(j:, 0:kk)^T v
      for (int q = wid; q < kk; q += CB_WARPS) {
        double a = 0.0;
        for (int i = j + lane; i < s; i += 32) {
          const double vi = (i == j) ? 1.0 : vk[i];
          a = fma(Vp[(size_t)q * s + i], vi, a);
        }
        a = warp_sum(a);
        if (lane == 0) aux[q] = -tau * a;
      }
      __syncthreads();
      // ---- 4b-6. read-only pass over the trailing columns (two columns per warp in flight)
      for (int c = j + 1 + wid; c < rows; c += 2 * CB_WARPS) {
        const int c2 = c + CB_WARPS;
        const bool has2 = c2 < rows;
        const double* col = W + (size_t)c * s;
        const double* col2 = W + (size_t)(has2 ? c2 : c) * s;
        double x1[MAXPL], x2[MAXPL];
#pragma unroll
        for (int q = 0; q < MAXPL; ++q) {
          const int i = j + lane + 32 * q;
          x1[q] = (i < s) ? col[i] : 0.0;
          x2[q] = (i < s && has2) ? col2[i] : 0.0;
        }
        double d1 = 0.0, d2 = 0.0;
#pragma unroll
        for (int q = 0; q < MAXPL; ++q) {
          const int i = j + lane + 32 * q;
          if (i < s) {
            const double vi = vk[i];
            d1 = fma(x1[q], vi, d1);
            d2 = fma(x2[q], vi, d2);
          }
        }
        // lane q < kk: the F and row-update corrections of panel column q
        double f1 = 0.0, f2 = 0.0, r1 = 0.0, r2 = 0.0;
        if (lane < kk) {
          const double a = aux[lane], vj = Vp[(size_t)lane * s + j];
          const double F1 = Fm[c * NB + lane];
          f1 = F1 * a;
          r1 = vj * F1;
          if (has2) {
            const double F2 = Fm[c2 * NB + lane];
            f2 = F2 * a;
            r2 = vj * F2;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          d1 += __shfl_xor_sync(0xffffffffu, d1, o);
          d2 += __shfl_xor_sync(0xffffffffu, d2, o);
          f1 += __shfl_xor_sync(0xffffffffu, f1, o);
          f2 += __shfl_xor_sync(0xffffffffu, f2, o);
          r1 += __shfl_xor_sync(0xffffffffu, r1, o);
          r2 += __shfl_xor_sync(0xffffffffu, r2, o);
        }
        if (lane == 0) {
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            if (u == 1 && !has2) break;
            const int cc = u ? c2 : c;
            const double F = fma(tau, u ? d2 : d1, u ? f2 : f1);
            Fm[cc * NB + kk] = F;
            const double a = (u ? x2[0] : x1[0]) - (u ? r2 : r1) - F;   // V(j, kk) = 1
            W[(size_t)cc * s + j] = a;
            const double n1 = vn1[cc];
            if (n1 != 0.0) {
              double t = fabs(a) / n1;
              t = fmax(0.0, (1.0 + t) * (1.0 - t));
              const double r = n1 / vn2[cc];
              if (t * r * r <= tol3z) { flag[cc] = 1; s_any = 1; }
              else vn1[cc] = n1 * sqrt(t);
            }
          }
        }
      }
      __syncthreads();
      ++kk;
      ++j;
      if (kk == NB || s_any || j >= kmax) break;
    }
    if (stop) break;
    // ---- panel end: trailing update A(j:, c) -= V(j:, 0:kk) F(c, 0:kk)^T (c >= j), and the
    // recomputed norms.  After the last pivot only the flagged norms matter (cap-hit test).
    const bool last = j >= kmax;
    if (last && !s_any) break;
    for (int c = j + wid; c < rows; c += CB_WARPS) {
      const bool fl = flag[c] != 0;
      if (last && !fl) continue;
      double f[NB];
#pragma unroll
      for (int q = 0; q < NB; ++q) f[q] = (q < kk) ? Fm[c * NB + q] : 0.0;
      double* col = W + (size_t)c * s;
      double nn = 0.0;
      for (int i = j + lane; i < s; i += 32) {
        double x = col[i];
#pragma unroll
        for (int q = 0; q < NB; ++q)
          if (q < kk) x = fma(-Vp[(size_t)q * s + i], f[q], x);
        if (!last) col[i] = x;
        nn = fma(x, x, nn);
      }
      if (fl) {
        nn = warp_sum(nn);
        if (lane == 0) { vn1[c] = sqrt(nn); vn2[c] = vn1[c]; flag[c] = 0; }
      }
    }
    __syncthreads();
    if (tid == 0) s_any = 0;
    __syncthreads();
    if (last) break;
  }
  const int k = j;
  int hit = 0;
  if (adaptive && !stop && k == kmax && k == cap && k < rows && k < s) {
    // tolerance unmet at the cap iff the next pivot's |R_kk| (its column norm) exceeds thr
    double bv = 0.0;
    for (int c = k + tid; c < rows; c += CB_THREADS) bv = fmax(bv, vn1[c]);
    for (int o = 16; o > 0; o >>= 1) bv = fmax(bv, __shfl_xor_sync(0xffffffffu, bv, o));
    if (lane == 0) red[wid] = bv;
    __syncthreads();
    if (tid == 0) {
      double b = 0.0;
      for (int w = 0; w < CB_WARPS; ++w) b = fmax(b, red[w]);
      s_p = (b > thr) ? 1 : 0;
    }
    __syncthreads();
    hit = s_p;
  }
  for (int c = tid; c < rows; c += CB_THREADS) P.piv[c] = piv[c];
  if (tid == 0) { *P.k_out = k; if (P.cap_hit) *P.cap_hit = hit; }
}

// panel width: 8 keeps the shared memory (F, V, norms) at ~63 KB for rows = 512, s = 272, so
// three CTAs share an SM and hide each other's per-step serial phases (SVMHSS_CPQR_NB=4 for A/B)
static int cpqr_nb() {
  static const int nb = [] { const char* e = getenv("SVMHSS_CPQR_NB"); return (e && atoi(e) == 4) ? 4 : 8; }();
  return nb;
}

size_t cpqr_blk_smem(int rows, int s) {
  const int nb = cpqr_nb();
  return ((size_t)2 * rows + (size_t)rows * nb + (size_t)nb * s) * sizeof(double) + (size_t)3 * rows * sizeof(int);
}

bool cpqr_blk_fits(int rows, int s) { return s <= 288 && cpqr_blk_smem(rows, s) <= 100 * 1024; }

void bcpqr_blk(const CpqrProb* d, int nprob, int maxr, int maxs, double rel_tol, double abs_tol, int cap,
               cudaStream_t s) {
  const size_t smem = cpqr_blk_smem(maxr, maxs);
  auto launch = [&](auto kern) {
    CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)nprob, CB_THREADS, smem, s>>>(d, rel_tol, abs_tol, cap);
  };
  if (cpqr_nb() == 4) {
    if (maxs <= 96) launch(bcpqr_blk_kernel<3, 4>);
    else if (maxs <= 160) launch(bcpqr_blk_kernel<5, 4>);
    else launch(bcpqr_blk_kernel<9, 4>);
  } else {
    if (maxs <= 96) launch(bcpqr_blk_kernel<3, 8>);
    else if (maxs <= 160) launch(bcpqr_blk_kernel<5, 8>);
    else launch(bcpqr_blk_kernel<9, 8>);
  }
  LAUNCH_CHECK();
}

}  // namespace svmhss
