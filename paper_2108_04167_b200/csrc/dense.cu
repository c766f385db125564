// dense.cu — batched small dense fp64 kernels (one problem = one HSS tree node).
//
//  bgemm   : smem-tiled DFMA GEMM with arbitrary strides (sibling updates H4, Omega' = U^T Omega^,
//            R_a B R_b^T, Q^T D Q, the explicit solve operators of the ULV).
//  bpotrf  : left-looking Cholesky, one CTA per node (U: Dc_rr = L_r L_r^T; root).
//  btrsm   : blocked triangular solve with many right-hand sides (T = R11^-1 R12 in H3;
//            L_sr, G_r = L_r^-1 Q_r^T in U).
//  bgeqr2  : Householder QR (LAPACK dlarfg convention) of Ucur (U).
//  blarft  : compact-WY T factor (Q = I - V T V^T).
//  bcpqr   : column-pivoted Householder QR of Y^T with the AMB-10 rank rule (H3): exact
//            trailing column norms recomputed in the update pass; argmax ties -> lowest index.
#include "dense.cuh"

namespace svmhss {

template <typename P>
static P* upload_probs(const std::vector<P>& v, cudaStream_t s) {
  P* d = nullptr;
  CUDA_CHECK(cudaMallocAsync((void**)&d, v.size() * sizeof(P), s));
  CUDA_CHECK(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(P), cudaMemcpyHostToDevice, s));
  return d;
}
static void free_probs(void* d, cudaStream_t s) { CUDA_CHECK(cudaFreeAsync(d, s)); }

// ------------------------------------------------------------------ GEMM
constexpr int GBM = 64, GBN = 64, GBK = 16;

__global__ void __launch_bounds__(256) bgemm_kernel(const GemmProb* __restrict__ probs) {
  const GemmProb P = probs[blockIdx.z];
  const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * GBN;
  if (m0 >= P.m || n0 >= P.n) return;
  __shared__ double As[GBK][GBM + 1];
  __shared__ double Bs[GBK][GBN + 1];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  const bool a_rowmajor = (P.acs == 1), b_rowmajor = (P.bcs == 1);
  for (int k0 = 0; k0 < P.k; k0 += GBK) {
    for (int e = tid; e < GBM * GBK; e += 256) {
      int i, kk;
      if (a_rowmajor) { i = e / GBK; kk = e % GBK; } else { kk = e / GBM; i = e % GBM; }
      const int gi = m0 + i, gk = k0 + kk;
      As[kk][i] = (gi < P.m && gk < P.k) ? P.A[(long long)gi * P.ars + (long long)gk * P.acs] : 0.0;
    }
    for (int e = tid; e < GBN * GBK; e += 256) {
      int j, kk;
      if (b_rowmajor) { kk = e / GBN; j = e % GBN; } else { j = e / GBK; kk = e % GBK; }
      const int gj = n0 + j, gk = k0 + kk;
      Bs[kk][j] = (gj < P.n && gk < P.k) ? P.B[(long long)gk * P.brs + (long long)gj * P.bcs] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GBK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gi = m0 + ty + 16 * i;
    if (gi >= P.m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gj = n0 + tx + 16 * j;
      if (gj >= P.n) continue;
      double* c = P.C + (long long)gi * P.crs + (long long)gj * P.ccs;
      const double v = P.alpha * acc[i][j];
      *c = (P.beta == 0.0) ? v : fma(P.beta, *c, v);
    }
  }
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
    dim3 grid(ceil_div(maxn, GBN), ceil_div(maxm, GBM), (unsigned)chunk.size());
    bgemm_kernel<<<grid, 256, 0, s>>>(d);
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

void bpotrf(const std::vector<SqProb>& probs, int* d_info, cudaStream_t s) {
  if (probs.empty()) return;
  int maxn = 0;
  for (auto& p : probs) maxn = std::max(maxn, p.n);
  SqProb* d = upload_probs(probs, s);
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

void btrsm(const std::vector<TrsmProb>& probs_in, bool lower, cudaStream_t s) {
  std::vector<TrsmProb> probs;
  int maxr = 0;
  for (auto& p : probs_in)
    if (p.n > 0 && p.nrhs > 0) { probs.push_back(p); maxr = std::max(maxr, p.nrhs); }
  if (probs.empty()) return;
  for (size_t b0 = 0; b0 < probs.size(); b0 += 65535) {
    std::vector<TrsmProb> chunk(probs.begin() + b0,
                                probs.begin() + std::min(probs.size(), b0 + 65535));
    TrsmProb* d = upload_probs(chunk, s);
    dim3 grid(ceil_div(maxr, TC), (unsigned)chunk.size());
    if (lower) btrsm_kernel<true><<<grid, 256, 0, s>>>(d);
    else btrsm_kernel<false><<<grid, 256, 0, s>>>(d);
    LAUNCH_CHECK();
    free_probs(d, s);
  }
}

// ------------------------------------------------------------------ Householder QR
__global__ void __launch_bounds__(256) bgeqr2_kernel(const QrProb* __restrict__ probs) {
  const QrProb P = probs[blockIdx.x];
  const int m = P.m, n = P.n, tid = threadIdx.x;
  extern __shared__ double v[];   // m doubles
  __shared__ double red[32];
  __shared__ double s_tau;
#define QA(i, j) P.A[(long long)(i) * P.rs + (long long)(j) * P.cs]
  for (int j = 0; j < n; ++j) {
    double part = 0.0;
    for (int i = j + 1 + tid; i < m; i += blockDim.x) { const double x = QA(i, j); part = fma(x, x, part); }
    const double xs = block_sum(part, red);
    const double alpha = QA(j, j);
    double tau, scal, beta;
    if (xs == 0.0) { tau = 0.0; scal = 0.0; beta = alpha; }
    else {
      beta = -copysign(sqrt(alpha * alpha + xs), alpha);
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    if (tid == 0) { s_tau = tau; v[j] = 1.0; }
    for (int i = j + 1 + tid; i < m; i += blockDim.x) {
      const double x = (tau == 0.0) ? QA(i, j) : QA(i, j) * scal;
      v[i] = x;
      QA(i, j) = x;
    }
    __syncthreads();
    if (tid == 0) { QA(j, j) = beta; P.tau[j] = tau; }
    if (tau != 0.0) {
      for (int c = j + 1 + tid; c < n; c += blockDim.x) {
        double w = 0.0;
        for (int i = j; i < m; ++i) w = fma(v[i], QA(i, c), w);
        w *= tau;
        for (int i = j; i < m; ++i) QA(i, c) = fma(-w, v[i], QA(i, c));
      }
    }
    __syncthreads();
  }
#undef QA
}

void bgeqr2(const std::vector<QrProb>& probs, cudaStream_t s) {
  if (probs.empty()) return;
  int maxm = 0;
  for (auto& p : probs) maxm = std::max(maxm, p.m);
  QrProb* d = upload_probs(probs, s);
  size_t smem = (size_t)std::max(1, maxm) * sizeof(double);
  if (smem > 48 * 1024)
    CUDA_CHECK(cudaFuncSetAttribute(bgeqr2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
  bgeqr2_kernel<<<(unsigned)probs.size(), 256, smem, s>>>(d);
  LAUNCH_CHECK();
  free_probs(d, s);
}

// ------------------------------------------------------------------ larft
__global__ void __launch_bounds__(256) blarft_kernel(const SqProb* __restrict__ probs,
                                                     const double* const* __restrict__ taus) {
  const SqProb P = probs[blockIdx.x];
  const double* tau = taus[blockIdx.x];
  const int n = P.n, tid = threadIdx.x;
  extern __shared__ double scol[];   // n doubles: S[0:j, j]
  for (int j = 0; j < n; ++j) {
    for (int p = tid; p < j; p += blockDim.x) scol[p] = AT(P, p, j);
    __syncthreads();
    const double tj = tau[j];
    for (int i = tid; i < j; i += blockDim.x) {
      double acc = 0.0;
      for (int p = i; p < j; ++p) acc = fma(AT(P, i, p), scol[p], acc);
      AT(P, i, j) = -tj * acc;
    }
    if (tid == 0) AT(P, j, j) = tj;
    __syncthreads();
  }
  for (long long e = tid; e < (long long)n * n; e += blockDim.x) {
    const int i = (int)(e / n), j = (int)(e % n);
    if (i > j) AT(P, i, j) = 0.0;
  }
}

void blarft(const std::vector<SqProb>& probs, const std::vector<const double*>& taus,
            cudaStream_t s) {
  if (probs.empty()) return;
  int maxn = 0;
  for (auto& p : probs) maxn = std::max(maxn, p.n);
  SqProb* d = upload_probs(probs, s);
  const double** dt = upload_probs(taus, s);
  size_t smem = (size_t)std::max(1, maxn) * sizeof(double);
  if (smem > 48 * 1024)
    CUDA_CHECK(cudaFuncSetAttribute(blarft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
  blarft_kernel<<<(unsigned)probs.size(), 256, smem, s>>>(d, dt);
  LAUNCH_CHECK();
  free_probs(d, s);
  free_probs((void*)dt, s);
}

// ------------------------------------------------------------------ column-pivoted QR (H3)
constexpr int CP_THREADS = 512;

template <int MAXPL>
__global__ void __launch_bounds__(CP_THREADS) bcpqr_kernel(const CpqrProb* __restrict__ probs,
                                                           double rel_tol, double abs_tol,
                                                           int cap) {
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

void bcpqr(const std::vector<CpqrProb>& probs, double rel_tol, double abs_tol, int cap,
           cudaStream_t s) {
  if (probs.empty()) return;
  int maxr = 0, maxs = 0;
  for (auto& p : probs) { maxr = std::max(maxr, p.rows); maxs = std::max(maxs, p.s); }
  CpqrProb* d = upload_probs(probs, s);
  size_t smem = (size_t)maxr * (sizeof(double) + sizeof(int)) + (size_t)maxs * sizeof(double) + 16;
  auto launch = [&](auto kern) {
    if (smem > 48 * 1024)
      CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)probs.size(), CP_THREADS, smem, s>>>(d, rel_tol, abs_tol, cap);
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
