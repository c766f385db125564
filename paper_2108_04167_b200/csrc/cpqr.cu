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

// VEC-wide global vectors of a column (VEC = 4: 256-bit loads, s = 0 mod 4; VEC = 2: 128-bit)
template <int VEC> struct Vec { double v[VEC]; };
template <int VEC>
__device__ __forceinline__ Vec<VEC> ldv(const double* p) {
  Vec<VEC> r;
  if constexpr (VEC == 4)
    asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3]) : "l"(p));
  else
    asm volatile("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.v[0]), "=d"(r.v[1]) : "l"(p));
  return r;
}
template <int VEC>
__device__ __forceinline__ void stv(double* p, const Vec<VEC>& r) {
  if constexpr (VEC == 4)
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(r.v[0]), "d"(r.v[1]), "d"(r.v[2]),
                 "d"(r.v[3]) : "memory");
  else
    asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(r.v[0]), "d"(r.v[1]) : "memory");
}

// Shared-memory layout (doubles, each part 32-byte aligned): vn1, vn2 (rows), F (NB x rows,
// F(c, q) at q*rows + c: lane-consecutive columns, conflict-free), V (NB x s), then piv, pos, flag.
__host__ __device__ inline int cb_al4(int x) { return (x + 3) & ~3; }

template <int NB, int VEC>
__global__ void __launch_bounds__(CB_THREADS, 3) bcpqr_blk_kernel(const CpqrProb* __restrict__ probs,
                                                                  double rel_tol, double abs_tol, int cap) {
  const CpqrProb P = probs[blockIdx.x];
  const int rows = P.rows, s = P.s;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int ra = cb_al4(rows);
  extern __shared__ __align__(32) double sm[];
  double* vn1 = sm;                          // partial column norms (pivoting)
  double* vn2 = vn1 + ra;                    // reference norms (downdate accuracy test)
  double* Fm = vn2 + ra;                     // NB x ra: F(c, q) at Fm[q*ra + c]
  double* Vp = Fm + (size_t)NB * ra;         // NB x s: panel reflectors, Vp[q*s + i] (i >= j0+q)
  int* piv = (int*)(Vp + (size_t)NB * s);    // original column at each position
  int* pos = piv + rows;                     // position of each original column
  int* flag = pos + rows;                    // 1 = norm to be recomputed after the panel
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
          const double a = Fm[q * ra + j];
          Fm[q * ra + j] = Fm[q * ra + p];
          Fm[q * ra + p] = a;
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
        for (int q = 0; q < kk; ++q) x = fma(-Vp[(size_t)q * s + i], Fm[q * ra + j], x);
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
      const int jal = j & ~(VEC - 1);
      for (int i = j + 1 + tid; i < s; i += CB_THREADS) {
        const double v = vk[i] * scal;
        vk[i] = v;
        W[(size_t)j * s + i] = v;
      }
      __syncthreads();
      if (tid == 0) { W[(size_t)j * s + j] = beta; vk[j] = 1.0; }
      if (tid > 0 && tid < VEC && jal + tid - 1 < j) vk[jal + tid - 1] = 0.0;  // masked lead-in of the vectors
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
      // ---- 4b-6. read-only pass: one trailing column per LANE (VEC-wide vector loads of its
      // rows jal.., v broadcast from shared memory), then its F entry, row update and norm
      const int ng = (rows - j - 1 + 31) >> 5;
      for (int g = wid; g < ng; g += CB_WARPS) {
        const int c = j + 1 + 32 * g + lane;
        if (c < rows) {
          const double* col = W + (size_t)c * s;
          double d[VEC];
#pragma unroll
          for (int e = 0; e < VEC; ++e) d[e] = 0.0;
          const Vec<VEC> x0 = ldv<VEC>(col + jal);
          double xj = x0.v[0];
#pragma unroll
          for (int e = 1; e < VEC; ++e) if (jal + e == j) xj = x0.v[e];
#pragma unroll
          for (int e = 0; e < VEC; ++e) d[e] = fma(x0.v[e], vk[jal + e], d[e]);
          int i = jal + VEC;
          for (; i + 4 * VEC <= s; i += 4 * VEC) {
            Vec<VEC> x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = ldv<VEC>(col + i + u * VEC);
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
              for (int e = 0; e < VEC; ++e) d[e] = fma(x[u].v[e], vk[i + u * VEC + e], d[e]);
          }
          for (; i < s; i += VEC) {
            const Vec<VEC> x1 = ldv<VEC>(col + i);
#pragma unroll
            for (int e = 0; e < VEC; ++e) d[e] = fma(x1.v[e], vk[i + e], d[e]);
          }
          double dot = d[0];
#pragma unroll
          for (int e = 1; e < VEC; ++e) dot += d[e];
          double fc = 0.0, rc = 0.0;
          for (int q = 0; q < kk; ++q) {
            const double Fq = Fm[q * ra + c];
            fc = fma(Fq, aux[q], fc);
            rc = fma(Vp[(size_t)q * s + j], Fq, rc);
          }
          const double Fv = fma(tau, dot, fc);
          Fm[kk * ra + c] = Fv;
          const double a = xj - rc - Fv;   // V(j, kk) = 1
          W[(size_t)c * s + j] = a;
          const double n1 = vn1[c];
          if (n1 != 0.0) {
            double t = fabs(a) / n1;
            t = fmax(0.0, (1.0 + t) * (1.0 - t));
            const double r = n1 / vn2[c];
            if (t * r * r <= tol3z) { flag[c] = 1; s_any = 1; }
            else vn1[c] = n1 * sqrt(t);
          }
        }
      }
      __syncthreads();
      ++kk;
      ++j;
      if (kk == NB || s_any || j >= kmax) break;
    }
    if (stop) break;
    // ---- panel end: trailing update A(j:, c) -= V(j:, 0:kk) F(c, 0:kk)^T (c >= j; one column per
    // lane, vector loads/stores), and the recomputed norms.  After the last pivot only the
    // flagged norms matter (cap-hit test).
    const bool last = j >= kmax;
    if (last && !s_any) break;
    const int jal = j & ~(VEC - 1);
    const int ng = (rows - j + 31) >> 5;
    for (int g = wid; g < ng; g += CB_WARPS) {
      const int c = j + 32 * g + lane;
      if (c >= rows) continue;
      const bool fl = flag[c] != 0;
      if (last && !fl) continue;
      double f[NB];
#pragma unroll
      for (int q = 0; q < NB; ++q) f[q] = (q < kk) ? Fm[q * ra + c] : 0.0;
      double* col = W + (size_t)c * s;
      double nn = 0.0;
      for (int i = jal; i < s; i += VEC) {
        Vec<VEC> x = ldv<VEC>(col + i);
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          if (i + e < j) continue;          // rows above j are final
          double y = x.v[e];
#pragma unroll
          for (int q = 0; q < NB; ++q)
            if (q < kk) y = fma(-Vp[(size_t)q * s + i + e], f[q], y);
          x.v[e] = y;
          nn = fma(y, y, nn);
        }
        if (!last) stv<VEC>(col + i, x);
      }
      if (fl) { vn1[c] = sqrt(nn); vn2[c] = vn1[c]; flag[c] = 0; }
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

// panel width 8 keeps the shared memory (F, V, norms) at ~63 KB for rows = 512, s = 272, so three
// CTAs share an SM and hide each other's per-step serial phases
constexpr int kCpqrNB = 8;

size_t cpqr_blk_smem(int rows, int s) {
  return ((size_t)(2 + kCpqrNB) * cb_al4(rows) + (size_t)kCpqrNB * s) * sizeof(double) +
         (size_t)3 * rows * sizeof(int);
}

bool cpqr_blk_fits(int rows, int s) { return s <= 1152 && s % 2 == 0 && cpqr_blk_smem(rows, s) <= 100 * 1024; }

void bcpqr_blk(const CpqrProb* d, int nprob, int maxr, int maxs, double rel_tol, double abs_tol, int cap,
               cudaStream_t s) {
  const size_t smem = cpqr_blk_smem(maxr, maxs);
  auto launch = [&](auto kern) {
    CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)nprob, CB_THREADS, smem, s>>>(d, rel_tol, abs_tol, cap);
  };
  // every node of a batch has the same s (the level's sample width)
  if (maxs % 4 == 0) launch(bcpqr_blk_kernel<kCpqrNB, 4>);
  else launch(bcpqr_blk_kernel<kCpqrNB, 2>);
  LAUNCH_CHECK();
}

}  // namespace svmhss
