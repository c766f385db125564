// admm.cu — closed-form ADMM for the SVM dual (Alg. 2; Alg. 3 lines 4-13,
// P:211-221 with reading AMB-1), the averaged bias (AMB-2, AMB-3), the
// objective f~ of Eq. (8), and the label assignment.
//
// Per iteration (one CUDA graph replay; no host involvement):
//   ULV forward sweep (levels L..0) -> backward sweep (0..L)            v = K_b^-1 (Y q)
//   epilogue, per point i and problem c (all nC problems = nC right-hand sides):
//     x = y_i v_i - (w^T q / w1) w_i;  z = clip(x - mu/beta, 0, C_c);  mu -= beta (x - z)
//     q' = 1 + mu + beta z;  next right-hand side y_i q'; per-block partial w^T q'
//   fixed-order reduction of the partials -> w^T q' for the next iteration.
#include "solve_dev.cuh"

namespace svmhss {

// The per-point ADMM update (A2-A3, P:164-166 with AMB-1) for problem c:
//   x = y v - (w^T q / w1) w;  z = clip(x - mu/beta, 0, C);  mu -= beta (x - z)
//   q' = 1 + mu + beta z;  next right-hand side y q'.   Returns w_i q'_i.
// x of pass-through leaves is read straight from level L-1's solution and their next
// right-hand side written straight into level L-1's input (ptmap), fusing the leaf level of
// both sweeps into the epilogue.
struct EpiArgs {
  const double *y, *w, *Cv, *swq;
  double w1, beta;
  const double *xL, *xL1;
  const int64_t* ptmap;
  double *z, *mu, *bL, *bL1;
  int nC;
};
// One point's update with every rounding spelled out (no compiler FMA contraction choices), so
// the epilogue kernel and the fused leaf kernel produce bitwise the same values.
__device__ __forceinline__ double admm_update(double vi, double yi, double wi, double m, double coef, double C,
                                              double beta, double& zn, double& mn, double& rhs) {
  const double x = __fma_rn(yi, vi, -__dmul_rn(coef, wi));      // x = y v - (w^T q / w1) w
  zn = fmin(fmax(__dsub_rn(x, __ddiv_rn(m, beta)), 0.0), C);    // z = clip(x - mu / beta, 0, C)
  mn = __fma_rn(-beta, __dsub_rn(x, zn), m);                    // mu - beta (x - z)
  const double qn = __fma_rn(beta, zn, __dadd_rn(1.0, mn));     // q' = 1 + mu + beta z
  rhs = __dmul_rn(yi, qn);                                      // next right-hand side y q'
  return __dmul_rn(wi, qn);                                     // w_i q'_i
}
__device__ __forceinline__ double epi_point(const EpiArgs& A, int64_t i, int c) {
  const double coef = __ddiv_rn(A.swq[c], A.w1), C = A.Cv[c];
  const int nC = A.nC;
  const int64_t e = i * nC + c;
  const int64_t q = A.ptmap ? A.ptmap[i] : -1;
  const double vi = (q >= 0) ? A.xL1[q * nC + c] : A.xL[e];
  double zn, mn, rhs;
  const double r = admm_update(vi, A.y[i], A.w[i], A.mu[e], coef, C, A.beta, zn, mn, rhs);
  A.z[e] = zn;
  A.mu[e] = mn;
  if (q >= 0) A.bL1[q * nC + c] = rhs;
  else A.bL[e] = rhs;
  return r;
}
// A leaf's w^T q' partial is defined chunk-wise (both epilogue kernels below): chunks of 32
// consecutive points from the leaf's start, each summed by a warp butterfly, then the chunk sums
// added in order.  One warp updates one chunk and returns its sums (lane c holds problem c).
__device__ __forceinline__ double epi_chunk(const EpiArgs& A, int64_t p0, int cnt) {
  const int lane = threadIdx.x & 31;
  double mine = 0.0;
  for (int c = 0; c < A.nC; ++c) {
    const double v = (lane < cnt) ? epi_point(A, p0 + lane, c) : 0.0;
    const double t = warp_sum(v);
    if (lane == c) mine = t;
  }
  return mine;
}

// One block per leaf (leaf list, or all of this rank's leaves when `leaves` is NULL).  With
// `counter`, the last block to finish reduces the leaf partials up the subtree -> out (so the
// reduction adds no launch).
__global__ void __launch_bounds__(256) admm_epilogue_kernel(EpiArgs A, const int64_t* __restrict__ leaf_lo,
                                                            const int* __restrict__ leaves, int nleaf_all,
                                                            double* __restrict__ part, double* __restrict__ out,
                                                            unsigned* __restrict__ counter, int smem_tree) {
  extern __shared__ double cs[];  // chunk sums: nch x nC (last block: the leaf-partial tree)
  pdl_trigger();
  pdl_wait();
  const int leaf = leaves ? leaves[blockIdx.x] : (int)blockIdx.x;
  const int64_t i0 = leaf_lo[leaf], i1 = leaf_lo[leaf + 1];
  const int nch = (int)((i1 - i0 + 31) / 32);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int ch = wid; ch < nch; ch += 8) {
    const int64_t p0 = i0 + 32LL * ch;
    const double t = epi_chunk(A, p0, (int)((i1 - p0) < 32 ? (i1 - p0) : 32));
    if (lane < A.nC) cs[ch * A.nC + lane] = t;
  }
  __syncthreads();
  if (threadIdx.x < A.nC) {
    double t = 0.0;
    for (int ch = 0; ch < nch; ++ch) t += cs[ch * A.nC + threadIdx.x];
    part[(int64_t)leaf * A.nC + threadIdx.x] = t;
  }
  if (counter) {
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (smem_tree) {
      // the same pairwise tree (part[i] += part[i + st], i = 0 mod 2 st), one column at a time in
      // shared memory (the chunk-sum scratch is free now): ~11 steps of smem latency, not L2
      for (int c = 0; c < A.nC; ++c) {
        for (int i = threadIdx.x; i < nleaf_all; i += blockDim.x) cs[i] = __ldcg(part + (int64_t)i * A.nC + c);
        __syncthreads();
        for (int st = 1; st < nleaf_all; st <<= 1) {
          for (int i = threadIdx.x * 2 * st; i + st < nleaf_all; i += blockDim.x * 2 * st) cs[i] += cs[i + st];
          __syncthreads();
        }
        if (threadIdx.x == 0) { out[c] = cs[0]; part[c] = cs[0]; }
        __syncthreads();
      }
    } else {
      // same pairwise tree as the shared-memory path (i + st < n bound: any leaf count)
      for (int st = 1; st < nleaf_all; st <<= 1) {
        const int npair = (nleaf_all + 2 * st - 1) / (2 * st);
        for (int e = threadIdx.x; e < npair * A.nC; e += blockDim.x) {
          const int i = (e / A.nC) * 2 * st, c = e % A.nC;
          if (i + st < nleaf_all) part[(int64_t)i * A.nC + c] += part[(int64_t)(i + st) * A.nC + c];
        }
        __syncthreads();
      }
      for (int c = threadIdx.x; c < A.nC; c += blockDim.x) out[c] = part[c];
    }
    if (threadIdx.x == 0) *counter = 0u;
  }
}

// ---- the leaf level of both sweeps fused with the epilogue (one CTA per leaf; the leaves with
// their own transform first, the pass-through leaves after):
//   leaf t with M_t:  x_t = M_t^T [x_s; y_r]  ->  ADMM update of its points (next right-hand side
//                     b_t kept in shared memory)  ->  t' = M_t b_t: up -> level L-1 input, y_r
//                     (the next iteration's level-L forward sweep)
//   pass-through leaf: the ADMM update reading x from level L-1's solution, writing the next
//                     right-hand side into level L-1's input
// bwd_cols / fwd_rows are the level kernels' device functions and the point update is
// epi_point's formula in the same order, so the results are bitwise those of the unfused
// ulv_bwd_kernel -> admm_epilogue_kernel -> ulv_fwd_kernel sequence.
constexpr int kLeafThreads = 512, kLeafGroups = kLeafThreads / (kBW * 32);
constexpr int kLeafWarps = kLeafThreads / 32;

// ADMM update (epi_point's formula, same order) of one leaf's points by warps [w0, w0 + nw): chunk
// ch (32 points) by warp w0 + ch mod nw; chunk sums (lane c: problem c) into cs[ch * NR + c].
// x from xv (the leaf's own transform, shared memory) or level L-1's solution (pass-through);
// the next right-hand side into rhs_sm (shared) or level L-1's input (pass-through).
template <int NR>
__device__ __forceinline__ void leaf_update(const EpiArgs& A, const SolveNode& N, int64_t i0, int npt, int w0, int nw,
                                            const double* __restrict__ xs_in, const double* xv,
                                            double* __restrict__ fin_up, double* rhs_sm, double* cs) {
  const int lane = threadIdx.x & 31, wid = (threadIdx.x >> 5) - w0;
  const int nch = (npt + 31) / 32;
  for (int ch = wid; ch < nch; ch += nw) {
    const int ii = 32 * ch + lane;
    const int64_t p = i0 + ii;
    const bool valid = ii < npt;
    double mine = 0.0;
#pragma unroll
    for (int c = 0; c < NR; ++c) {
      double v = 0.0;
      if (valid) {
        const double coef = __ddiv_rn(A.swq[c], A.w1), C = A.Cv[c];
        const int64_t e = p * NR + c;
        const double vi = N.pt ? xs_in[(N.koff + ii) * NR + c] : xv[ii * NR + c];
        double zn, mn, rhs;
        v = admm_update(vi, A.y[p], A.w[p], A.mu[e], coef, C, A.beta, zn, mn, rhs);
        A.z[e] = zn;
        A.mu[e] = mn;
        if (N.pt) fin_up[(N.koff + ii) * NR + c] = rhs;
        else rhs_sm[ii * NR + c] = rhs;
      }
      const double t = warp_sum(v);
      if (lane == c) mine = t;
    }
    if (lane < NR) cs[ch * NR + lane] = mine;
  }
}

// work[b] = {leaf a, leaf b}: a leaf with its own transform alone ({a, -1}, all warps), or one or
// two pass-through leaves (half of the warps each) -- pass-through leaves are only an ADMM update,
// so two per CTA halve the number of short CTAs.
template <int NR>
__global__ void __launch_bounds__(kLeafThreads, 2) admm_leaf_kernel(EpiArgs A, const SolveNode* __restrict__ nodes,
                                                                 const int2* __restrict__ work,
                                                                 const int64_t* __restrict__ leaf_lo, int nleaf_all,
                                                                 const double* __restrict__ M,
                                                                 const double* __restrict__ xs_in,
                                                                 double* __restrict__ yr, double* __restrict__ fin_up,
                                                                 double* __restrict__ part, double* __restrict__ out,
                                                                 unsigned* __restrict__ counter, int smem_tree,
                                                                 int maxR, int maxch) {
  extern __shared__ double sm[];
  pdl_trigger();
  // static data first (work list, node descriptor, the first batch of the leaf's M columns),
  // then the wait for the previous kernel (programmatic dependent launch)
  const int2 wk = work[blockIdx.x];
  const int leaf = wk.x;
  const SolveNode N = nodes[leaf];
  const int64_t i0 = leaf_lo[leaf], i1 = leaf_lo[leaf + 1];
  const int npt = (int)(i1 - i0);
  const int tid = threadIdx.x;
  double pa[BWD_BQ], pb[BWD_BQ];
  if (!N.pt && (tid / (kBW * 32)) * kCW < N.R)
    bwd_cols_preload(M + N.moff, N.R, (tid / (kBW * 32)) * kCW, pa, pb, tid % (kBW * 32));
  pdl_wait();
  double* ush = sm;                          // maxR x NR: [x_s; y_r], then the next rhs
  double* xv = ush + (size_t)maxR * NR;      // maxR x NR: x of the leaf's points
  double* red = xv + (size_t)maxR * NR;      // groups x kBW x kCW x NR
  double* cs = red + (size_t)kLeafGroups * kBW * kCW * NR; // chunk sums (2 x maxch x NR; last block: the tree)
  if (!N.pt) {
    const int R = N.R, kn = N.k * NR;
    for (int e = tid; e < R * NR; e += kLeafThreads) ush[e] = (e < kn) ? xs_in[N.koff * NR + e] : yr[(N.yoff - N.k) * NR + e];
    __syncthreads();
    // the column chunks in parallel, one group of kBW warps per chunk
    const int grp = tid / (kBW * 32), tig = tid % (kBW * 32);
    const int nrounds = ((R + kCW - 1) / kCW + kLeafGroups - 1) / kLeafGroups;  // uniform over the CTA
    for (int rd = 0; rd < nrounds; ++rd) {
      const int j0 = (rd * kLeafGroups + grp) * kCW;
      bwd_cols<NR>(M + N.moff, R, ush, j0, red + (size_t)grp * kBW * kCW * NR, xv, tig, j0 >= R,
                   rd == 0 ? pa : nullptr, rd == 0 ? pb : nullptr);
    }
    leaf_update<NR>(A, N, i0, npt, 0, kLeafWarps, xs_in, xv, fin_up, ush, cs);
    __syncthreads();
    if (tid < NR) {
      double t = 0.0;
      for (int ch = 0; ch < (npt + 31) / 32; ++ch) t += cs[ch * NR + tid];
      part[(int64_t)leaf * NR + tid] = t;
    }
    if (NR <= 2 && N.R <= 256)
      fwd_rows_short<NR>(M + N.moff, N.R, ush, 0, N.R, tid >> 5, kLeafWarps, N.k, N.koff, N.yoff, fin_up, yr);
    else
      fwd_rows<NR>(M + N.moff, N.R, ush, 0, N.R, tid >> 5, kLeafWarps, N.k, N.koff, N.yoff, fin_up, yr);
  } else {
    const int half = (tid >> 5) >= kLeafWarps / 2;
    const int lf = half ? wk.y : leaf;
    if (lf >= 0) {
      const SolveNode Nh = half ? nodes[lf] : N;
      const int64_t j0 = leaf_lo[lf];
      leaf_update<NR>(A, Nh, j0, (int)(leaf_lo[lf + 1] - j0), half * (kLeafWarps / 2), kLeafWarps / 2, xs_in,
                      nullptr, fin_up, nullptr, cs + (size_t)half * maxch * NR);
    }
    __syncthreads();
    if (tid < 2 * NR) {
      const int h = tid / NR, c = tid % NR;
      const int lh = h ? wk.y : leaf;
      if (lh >= 0) {
        const int nc = (int)((leaf_lo[lh + 1] - leaf_lo[lh] + 31) / 32);
        double t = 0.0;
        for (int ch = 0; ch < nc; ++ch) t += cs[((size_t)h * maxch + ch) * NR + c];
        part[(int64_t)lh * NR + c] = t;
      }
    }
  }
  // the last block to finish reduces the leaf partials up the subtree (as admm_epilogue_kernel)
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (tid == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (smem_tree) {
    for (int c = 0; c < NR; ++c) {
      for (int i = tid; i < nleaf_all; i += kLeafThreads) cs[i] = __ldcg(part + (int64_t)i * NR + c);
      __syncthreads();
      for (int st = 1; st < nleaf_all; st <<= 1) {
        for (int i = tid * 2 * st; i + st < nleaf_all; i += kLeafThreads * 2 * st) cs[i] += cs[i + st];
        __syncthreads();
      }
      if (tid == 0) { out[c] = cs[0]; part[c] = cs[0]; }
      __syncthreads();
    }
  } else {
    for (int st = 1; st < nleaf_all; st <<= 1) {
      const int npair = (nleaf_all + 2 * st - 1) / (2 * st);
      for (int e = tid; e < npair * NR; e += kLeafThreads) {
        const int i = (e / NR) * 2 * st, c = e % NR;
        if (i + st < nleaf_all) part[(int64_t)i * NR + c] += __ldcg(part + (int64_t)(i + st) * NR + c);
      }
      __syncthreads();
    }
    for (int c = tid; c < NR; c += kLeafThreads) out[c] = part[c];
  }
  if (tid == 0) *counter = 0u;
}

static void leaf_dispatch(int NR, dim3 grid, size_t smem, cudaStream_t s, const EpiArgs& A, const SolveNode* nodes,
                          const int2* order, const int64_t* leaf_lo, int nleaf, const double* M, const double* xs_in,
                          double* yr, double* fin_up, double* part, double* out, unsigned* counter, int smem_tree,
                          int maxR, int maxch) {
  switch (NR) {
#define LC(k)                                                                                                     \
  case k:                                                                                                         \
    if (smem > 48 * 1024)                                                                                         \
      CUDA_CHECK(cudaFuncSetAttribute(admm_leaf_kernel<k>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    launch_pdl(admm_leaf_kernel<k>, grid, dim3(kLeafThreads), smem, s, A, nodes, order, leaf_lo, nleaf, M, xs_in, yr, fin_up, \
               part, out, counter, smem_tree, maxR, maxch);                                                       \
    break;
    LC(1) LC(2) LC(3) LC(4) LC(5) LC(6) LC(7) LC(8)
#undef LC
    default: throw Error(HSS_EINVAL, "admm: nC must be 1..8");
  }
  g_launches.fetch_add(1);
}

// Per-leaf partials of column sums: out[leaf*ncols + c] = sum_{i in leaf} f(i, c)
//   mode 0: A[i*ncols + c]   mode 1: A[i*ncols + c] * B[i*ncols + c]
__global__ void leaf_colsum_kernel(const int64_t* __restrict__ leaf_lo, int ncols, const double* __restrict__ A,
                                   int mode, const double* __restrict__ B, double* __restrict__ part) {
  __shared__ double red[32];
  const int64_t i0 = leaf_lo[blockIdx.x], i1 = leaf_lo[blockIdx.x + 1];
  for (int c = 0; c < ncols; ++c) {
    double a = 0.0;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
      const double x = A[i * ncols + c];
      a += (mode == 0) ? x : x * B[i * ncols + c];
    }
    const double t = block_sum(a, red);
    if (threadIdx.x == 0) part[(int64_t)blockIdx.x * ncols + c] = t;
  }
}

__global__ void label_check_kernel(const double* __restrict__ y, int64_t n, int* bad) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && !(y[i] == 1.0 || y[i] == -1.0)) atomicAdd(bad, 1);
}

__global__ void fill_kernel(double* a, int64_t n, double v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}

// initial right-hand side y q0 = y (q0 = e), written where the fused leaf I/O expects it
__global__ void init_rhs_kernel(const double* __restrict__ y, int64_t n, int nC, const int64_t* __restrict__ ptmap,
                                double* __restrict__ bL, double* __restrict__ bL1) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * nC) return;
  const int64_t i = e / nC;
  const int c = (int)(e % nC);
  const int64_t q = ptmap ? ptmap[i] : -1;
  if (q >= 0) bL1[q * nC + c] = y[i];
  else bL[e] = y[i];
}

__global__ void mul_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                           double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] * b[i];
}

// per-leaf margin-set counts: part[leaf*2nC + 2c] = #{eps < z < C-eps}, [+1] = #{z > eps}
__global__ void margin_count_kernel(const int64_t* __restrict__ leaf_lo, int nC, const double* __restrict__ z,
                                    const double* __restrict__ Cv, double eps_rel, double* __restrict__ part) {
  __shared__ double red[32];
  const int64_t i0 = leaf_lo[blockIdx.x], i1 = leaf_lo[blockIdx.x + 1];
  for (int c = 0; c < nC; ++c) {
    const double C = Cv[c], eps = eps_rel * C;
    double a = 0.0, b = 0.0;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
      const double zi = z[i * nC + c];
      a += (zi > eps && zi < C - eps) ? 1.0 : 0.0;
      b += (zi > eps) ? 1.0 : 0.0;
    }
    const double ta = block_sum(a, red);
    const double tb = block_sum(b, red);
    if (threadIdx.x == 0) { part[(int64_t)blockIdx.x * 2 * nC + 2 * c] = ta; part[(int64_t)blockIdx.x * 2 * nC + 2 * c + 1] = tb; }
  }
}

// V[:, 2c] = indicator of the chosen margin set, V[:, 2c+1] = z_y = y z
__global__ void bias_rhs_kernel(int64_t n, int nC, const double* __restrict__ z,
                                const double* __restrict__ y, const double* __restrict__ Cv,
                                const int* __restrict__ mode, double eps_rel, double* __restrict__ V) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * nC) return;
  const int64_t i = e / nC;
  const int c = (int)(e % nC);
  const double C = Cv[c], eps = eps_rel * C, zi = z[e];
  double ind = 0.0;
  if (mode[c] == 0) ind = (zi > eps && zi < C - eps) ? 1.0 : 0.0;
  else if (mode[c] == 1) ind = (zi > eps) ? 1.0 : 0.0;
  V[i * 2 * nC + 2 * c] = ind;
  V[i * 2 * nC + 2 * c + 1] = y[i] * zi;
}

// per-leaf sums: part[leaf*4nC + 4c + 0] = sum_M y, +1 = z_y . (K~ e_M), +2 = z_y . (K~ z_y),
// +3 = sum z
__global__ void bias_sums_kernel(const int64_t* __restrict__ leaf_lo, int nC, const double* __restrict__ V,
                                 const double* __restrict__ KV, const double* __restrict__ y,
                                 const double* __restrict__ z, double* __restrict__ part) {
  __shared__ double red[32];
  const int64_t i0 = leaf_lo[blockIdx.x], i1 = leaf_lo[blockIdx.x + 1];
  for (int c = 0; c < nC; ++c) {
    double a = 0, b = 0, d = 0, f = 0;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
      const double ind = V[i * 2 * nC + 2 * c], zy = V[i * 2 * nC + 2 * c + 1];
      a += ind * y[i];
      b += zy * KV[i * 2 * nC + 2 * c];
      d += zy * KV[i * 2 * nC + 2 * c + 1];
      f += z[i * nC + c];
    }
    a = block_sum(a, red); b = block_sum(b, red); d = block_sum(d, red); f = block_sum(f, red);
    if (threadIdx.x == 0) {
      double* o = part + (int64_t)blockIdx.x * 4 * nC + 4 * c;
      o[0] = a; o[1] = b; o[2] = d; o[3] = f;
    }
  }
}

// y_orig: device labels (original order, all n).  z_out / mu_out: device, original order,
// n x nC (every rank gets the full vectors).
AdmmResult admm_train_impl(const ULVImpl& F, const double* y_orig, const std::vector<double>& Cs,
                           int max_it, const admm_opts* opt, double* z_out, double* mu_out,
                           double* bias_out, double* obj_out, cudaStream_t s) {
  const HSSImpl& H = *F.H;
  const Shard& sh = H.sh;
  const int64_t N = H.n, n = H.nloc();
  const int L = H.L, nC = (int)Cs.size(), nleaf = H.nleaf_loc();
  const double beta = F.beta;
  AdmmResult R{};
  {
    DevBuf<int> bad(1);
    CUDA_CHECK(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
    label_check_kernel<<<ceil_div(N, 256), 256, 0, s>>>(y_orig, N, bad.p);
    LAUNCH_CHECK();
    int hb = 0;
    d2h(&hb, bad.p, 1, s);
    CUDA_CHECK(cudaStreamSynchronize(s));
    require(hb == 0, "admm_svm_train: labels must be exactly +1 or -1");
  }
  DevBuf<double> y(n), w(n), z((size_t)n * nC), mu((size_t)n * nC), dC(nC), swq(nC), subwq(nC);
  DevBuf<double> part((size_t)std::max(1, nleaf) * std::max(4 * nC, 2));
  gather_rows(y_orig, H.perm.p + H.lo_g, n, 1, y.p, s);
  h2d(dC.p, Cs.data(), nC, s);
  // ---- precompute (A0): v = K_b^-1 e; w = Y v; w1 = e^T v (cluster-tree-ordered sums)
  EventTimer tpre(s);
  double w1 = 0.0, wte = 0.0;
  {
    SolveWS ws1;
    solve_ws_alloc(F, 1, ws1);
    fill_kernel<<<ceil_div(std::max<int64_t>(1, n), 256), 256, 0, s>>>(ws1.fin[L], n, 1.0);
    LAUNCH_CHECK();
    ulv_solve_tree(F, ws1, s);
    mul_kernel<<<ceil_div(std::max<int64_t>(1, n), 256), 256, 0, s>>>(y.p, ws1.xout[L], n, w.p);
    LAUNCH_CHECK();
    leaf_colsum_kernel<<<nleaf, 256, 0, s>>>(H.leaf_lo.p, 1, ws1.xout[L], 0, nullptr, part.p);
    LAUNCH_CHECK();
    tree_reduce_all(H, part.p, 1, &w1, s);
  }
  R.ms_pre = tpre.stop_ms();
  static const bool fault_w1 = [] { const char* e = getenv("SVMHSS_FAULT_W1"); return e && e[0] == '1'; }();
  if (fault_w1) w1 = -w1;  // test hook (include/svmhss.h): exercises the HSS_EW1 path
  R.w1 = w1;
  if (!(w1 > 0.0)) throw Error(HSS_EW1, "w1 = e^T (K~+beta I)^-1 e = " + std::to_string(w1) + " <= 0");
  // ---- state: x0 = z0 = mu0 = 0 (AMB-6); q0 = e
  const bool fused = L >= 1 && F.nleafpt > 0;
  SolveWS ws;
  ws.nextra = nC;
  solve_ws_alloc(F, nC, ws);
  ws.fused_leaf_io = fused;
  DevBuf<double> allwq((size_t)sh.P * nC);
  if (sh.on()) { ws.extra = subwq.p; ws.extra_all = allwq.p; ws.extra_top = swq.p; }
  double* bL = ws.fin[L];
  double* bL1 = fused ? ws.fin[L - 1] : nullptr;
  const double* xL = ws.xout[L];
  const double* xL1 = fused ? ws.xout[L - 1] : nullptr;
  const int64_t* ptm = fused ? F.ptmap.p : nullptr;
  CUDA_CHECK(cudaMemsetAsync(z.p, 0, (size_t)n * nC * 8, s));
  CUDA_CHECK(cudaMemsetAsync(mu.p, 0, (size_t)n * nC * 8, s));
  init_rhs_kernel<<<ceil_div(std::max<int64_t>(1, n * nC), 256), 256, 0, s>>>(y.p, n, nC, ptm, bL, bL1);
  LAUNCH_CHECK();
  {
    // w^T q0 = w^T e: this rank's subtree partial (exchanged in the first iteration) and total
    DevBuf<double> sub(1);
    leaf_colsum_kernel<<<nleaf, 256, 0, s>>>(H.leaf_lo.p, 1, w.p, 0, nullptr, part.p);
    LAUNCH_CHECK();
    tree_reduce_local(H, part.p, 1, sub.p, s);
    leaf_colsum_kernel<<<nleaf, 256, 0, s>>>(H.leaf_lo.p, 1, w.p, 0, nullptr, part.p);
    LAUNCH_CHECK();
    tree_reduce_all(H, part.p, 1, &wte, s);
    for (int c = 0; c < nC; ++c) {
      CUDA_CHECK(cudaMemcpyAsync(subwq.p + c, sub.p, 8, cudaMemcpyDeviceToDevice, s));
      h2d(swq.p + c, &wte, 1, s);
    }
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  DevBuf<unsigned> counter(1);
  CUDA_CHECK(cudaMemsetAsync(counter.p, 0, sizeof(unsigned), s));
  double* epi_out = sh.on() ? subwq.p : swq.p;
  EpiArgs EA{y.p, w.p, dC.p, swq.p, w1, beta, xL, xL1, ptm, z.p, mu.p, bL, bL1, nC};
  int maxleaf = 1;
  for (int i = sh.first(L); i < sh.last(L); ++i) maxleaf = std::max<int>(maxleaf, (int)(H.lv[L][i].hi - H.lv[L][i].lo));
  size_t epi_smem = (size_t)((maxleaf + 31) / 32) * nC * sizeof(double);
  const int smem_tree = ((size_t)nleaf * sizeof(double) <= 200 * 1024) ? 1 : 0;
  if (smem_tree) epi_smem = std::max(epi_smem, (size_t)nleaf * sizeof(double));
  if (epi_smem > 48 * 1024)
    CUDA_CHECK(cudaFuncSetAttribute(admm_epilogue_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)epi_smem));
  // leaf level fused with the epilogue (admm_leaf_kernel): needs the leaves strictly below the
  // exchanged level; bitwise the same as the unfused sequence (SVMHSS_LEAF_FUSE=0 runs that)
  static const bool leaf_fuse_env = [] { const char* e = getenv("SVMHSS_LEAF_FUSE"); return !(e && e[0] == '0'); }();
  const bool leaf_fuse = fused && leaf_fuse_env && L > sh.lg && !F.lv[L].allpt;
  DevBuf<int2> lorder;
  size_t leaf_smem = 0;
  int maxRL = 1, nleafw = 0;
  const int maxch = (maxleaf + 31) / 32;
  if (leaf_fuse) {
    std::vector<int2> ord;
    std::vector<int> pts;
    for (int i = sh.first(L); i < sh.last(L); ++i) {
      if (!H.lv[L][i].pt) ord.push_back(make_int2(i - sh.first(L), -1));
      else pts.push_back(i - sh.first(L));
    }
    for (size_t q = 0; q < pts.size(); q += 2)
      ord.push_back(make_int2(pts[q], q + 1 < pts.size() ? pts[q + 1] : -1));
    nleafw = (int)ord.size();
    lorder = upload(ord, s);
    maxRL = std::max(1, F.lv[L].maxR);
    leaf_smem = ((size_t)2 * maxRL * nC + (size_t)kLeafGroups * kBW * kCW * nC +
                 std::max((size_t)2 * maxch * nC, smem_tree ? (size_t)nleaf : 0)) * sizeof(double);
    // prologue: the level-L forward sweep of iteration 1 (the loop body's leaf kernel produces it
    // for the next iteration)
    ulv_solve_steps(F, ws, {SolveStep{SolveStep::FWD, L, L}}, s);
  }
  auto iteration = [&](cudaStream_t st) {
    if (leaf_fuse) {
      ulv_solve_steps(F, ws, {SolveStep{SolveStep::FWD, L - 1, 0}, SolveStep{SolveStep::BWD, 0, L - 1}}, st);
      leaf_dispatch(nC, dim3(nleafw), leaf_smem, st, EA, F.lv[L].nodes.p, lorder.p, H.leaf_lo.p, nleaf, F.lv[L].M.p,
                    ws.xout[L - 1], ws.yr[L], ws.fin[L - 1], part.p, epi_out, counter.p, smem_tree, maxRL, maxch);
      return;
    }
    ulv_solve_tree(F, ws, st);
    launch_pdl(admm_epilogue_kernel, dim3(nleaf), dim3(256), epi_smem, st, EA, H.leaf_lo.p, (const int*)nullptr,
               nleaf, part.p, epi_out, counter.p, smem_tree);
  };
  // one iteration as a CUDA graph (needs a capturable exchange when sharded); without traces,
  // also a graph of `gb` consecutive iterations, so the programmatic (PDL) edges continue from one
  // iteration into the next instead of draining at every graph launch
  cudaGraphExec_t gexec = nullptr, gexecB = nullptr;
  const bool use_graph = !sh.on() || sh.comm->capturable();
  const int te = (opt && opt->trace_every > 0) ? opt->trace_every : 0;
  static const int gb_env = [] { const char* e = getenv("SVMHSS_GRAPH_ITERS"); return e ? std::max(1, atoi(e)) : 4; }();
  const int gb = (use_graph && !te && max_it >= 2 * gb_env) ? gb_env : 1;
  const long long g0 = g_launches.load();  // launches are counted per executed iteration below
  auto capture = [&](int iters, cudaGraphExec_t* out) {
    cudaStream_t cs;
    CUDA_CHECK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t graph = nullptr;
    CUDA_CHECK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    for (int q = 0; q < iters; ++q) iteration(cs);
    CUDA_CHECK(cudaStreamEndCapture(cs, &graph));
    CUDA_CHECK(cudaGraphInstantiate(out, graph, 0));
    CUDA_CHECK(cudaGraphDestroy(graph));
    CUDA_CHECK(cudaStreamDestroy(cs));
  };
  if (use_graph) {
    capture(1, &gexec);
    R.graph = 1;
    R.launches = g_launches.load() - g0;
    if (gb > 1) capture(gb, &gexecB);
    g_launches.store(g0);
  }
  DevBuf<double> full((te && (opt->trace_z || opt->trace_mu)) ? (size_t)N * nC : 0);
  EventTimer tloop(s);
  int tcount = 0;
  for (int it = 1; it <= max_it; ++it) {
    const long long gi = g_launches.load();
    if (gexecB && it + gb - 1 <= max_it) {
      CUDA_CHECK(cudaGraphLaunch(gexecB, s));
      g_launches.store(gi + (long long)gb * R.launches);
      it += gb - 1;
      continue;
    }
    if (use_graph) {
      CUDA_CHECK(cudaGraphLaunch(gexec, s));
      g_launches.store(gi + R.launches);
    } else {
      iteration(s);
      R.launches = g_launches.load() - gi;
    }
    if (te && (it % te == 0 || it == max_it)) {
      if (opt->trace_z) {
        gather_points(H, z.p, nC, full.p, s);
        scatter_rows(full.p, H.perm.p, N, nC, opt->trace_z + (int64_t)tcount * N * nC, s);
      }
      if (opt->trace_mu) {
        gather_points(H, mu.p, nC, full.p, s);
        scatter_rows(full.p, H.perm.p, N, nC, opt->trace_mu + (int64_t)tcount * N * nC, s);
      }
      ++tcount;
    }
  }
  R.ms_loop = tloop.stop_ms();
  if (gexec) cudaGraphExecDestroy(gexec);
  if (gexecB) cudaGraphExecDestroy(gexecB);
  {
    DevBuf<double> zf((size_t)N * nC);
    gather_points(H, z.p, nC, zf.p, s);
    scatter_rows(zf.p, H.perm.p, N, nC, z_out, s);
    if (mu_out) {
      gather_points(H, mu.p, nC, zf.p, s);
      scatter_rows(zf.p, H.perm.p, N, nC, mu_out, s);
    }
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  // ---- bias + objective (one HSS mat-vec with 2 nC columns)
  if (bias_out || obj_out) {
    EventTimer tb(s);
    const double eps_rel = (opt && opt->margin_eps_rel > 0) ? opt->margin_eps_rel : 1e-8;
    margin_count_kernel<<<nleaf, 256, 0, s>>>(H.leaf_lo.p, nC, z.p, dC.p, eps_rel, part.p);
    LAUNCH_CHECK();
    std::vector<double> hc(2 * nC);
    tree_reduce_all(H, part.p, 2 * nC, hc.data(), s);
    std::vector<int> mode(nC);
    std::vector<double> msize(nC);
    for (int c = 0; c < nC; ++c) {
      if (hc[2 * c] > 0) { mode[c] = 0; msize[c] = hc[2 * c]; }
      else if (hc[2 * c + 1] > 0) { mode[c] = 1; msize[c] = hc[2 * c + 1]; }
      else { mode[c] = 2; msize[c] = 0; }
    }
    auto dmode = upload(mode, s);
    DevBuf<double> V((size_t)std::max<int64_t>(1, n) * 2 * nC), KV((size_t)std::max<int64_t>(1, n) * 2 * nC);
    bias_rhs_kernel<<<ceil_div(std::max<int64_t>(1, n * nC), 256), 256, 0, s>>>(n, nC, z.p, y.p, dC.p, dmode.p,
                                                                                eps_rel, V.p);
    LAUNCH_CHECK();
    hss_matvec_tree(H, V.p, KV.p, 2 * nC, s);
    bias_sums_kernel<<<nleaf, 256, 0, s>>>(H.leaf_lo.p, nC, V.p, KV.p, y.p, z.p, part.p);
    LAUNCH_CHECK();
    std::vector<double> hs(4 * nC);
    tree_reduce_all(H, part.p, 4 * nC, hs.data(), s);
    for (int c = 0; c < nC; ++c) {
      if (bias_out) bias_out[c] = (msize[c] > 0) ? (hs[4 * c] - hs[4 * c + 1]) / msize[c] : 0.0;
      if (obj_out) obj_out[c] = 0.5 * hs[4 * c + 2] - hs[4 * c + 3];
    }
    R.ms_bias = tb.stop_ms();
  }
  CUDA_CHECK(cudaStreamSynchronize(s));
  return R;
}

// ------------------------------------------------------------------ prediction (K8)
__global__ void predict_finish_kernel(const double* __restrict__ S, int64_t m, int nC, int lds,
                                      const double* __restrict__ bias, double* __restrict__ dv,
                                      int8_t* __restrict__ lab) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m * nC) return;
  const int64_t t = e / nC;
  const int c = (int)(e % nC);
  const double d = S[t * lds + c] + bias[c];
  if (dv) dv[e] = d;
  if (lab) lab[e] = (d >= 0.0) ? (int8_t)1 : (int8_t)-1;
}

// coefficients z_y = y o z, padded to ld columns: out[i*ld + c] = y_i z[i*nC + c] (c < nC)
__global__ void coef_kernel(const double* __restrict__ y, const double* __restrict__ z, int64_t n, int nC, int ld,
                            double* __restrict__ out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * ld) return;
  const int64_t i = e / ld;
  const int c = (int)(e % ld);
  out[e] = (c < nC) ? y[i] * z[i * nC + c] : 0.0;
}

__global__ void pad_coef16_kernel(const double* __restrict__ coef, int64_t n, int ld, double* __restrict__ out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * 16) return;
  const int64_t i = e / 16;
  const int c = (int)(e % 16);
  out[e] = (c < ld) ? coef[i * ld + c] : 0.0;
}

__global__ void copy_cols_kernel(const double* __restrict__ src, int64_t m, int lds, int ldd, double* __restrict__ dst) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m * ldd) return;
  dst[e] = src[(e / ldd) * lds + e % ldd];
}

// dv / labels of test rows [0, m) (this rank's share when sharded: the caller offsets Ftest)
static void predict_rows(const double* Ftr, const double* nutr, const double* coef, int64_t n, int r, int rp,
                         int SA, int ld, const double* Ftrain, double h, const double* bias_dev, int nC,
                         const double* Ftest, int64_t m, double* dv, int8_t* lab, cudaStream_t s) {
  if (m <= 0) return;
  DevBuf<double> Fte((size_t)m * SA), nute(m + kNormPad), S((size_t)m * ld);
  pad_rows(Ftest, m, r, SA, Fte.p, s);
  row_norms(Fte.p, m, SA, nute.p, s);
  if (rp <= 128) {
    predict_sums(Fte.p, nute.p, m, Ftr, nutr, coef, n, rp, SA, ld, -1.0 / (2.0 * h * h), S.p, s);
  } else {
    // wide features (r > 128): the sketch kernel's shared-memory tiling (rows at stride rp),
    // with the coefficients as a 16-column right-hand side
    DevBuf<double> Ftr2((size_t)n * rp), Fte2((size_t)m * rp), W16((size_t)n * 16 + 2), S16((size_t)m * 16);
    pad_rows(Ftrain, n, r, rp, Ftr2.p, s);
    pad_rows(Ftest, m, r, rp, Fte2.p, s);
    pad_coef16_kernel<<<ceil_div(n * 16, 256), 256, 0, s>>>(coef, n, ld, W16.p);
    LAUNCH_CHECK();
    KmmArgs a{};
    a.Fa = Fte2.p; a.nua = nute.p; a.na = m;
    a.Fb = Ftr2.p; a.nub = nutr; a.nb = n;
    a.rp = rp; a.W = W16.p; a.ldw = 16; a.ncols = 16; a.S = S16.p; a.lds = 16;
    a.neg_inv_2h2 = -1.0 / (2.0 * h * h);
    a.same_set = 0; a.leaf_a = nullptr; a.leaf_b = nullptr;
    kernel_matmul(a, s);
    copy_cols_kernel<<<ceil_div(m * ld, 256), 256, 0, s>>>(S16.p, m, 16, ld, S.p);
    LAUNCH_CHECK();
  }
  predict_finish_kernel<<<ceil_div(m * nC, 256), 256, 0, s>>>(S.p, m, nC, ld, bias_dev, dv, lab);
  LAUNCH_CHECK();
}

__global__ void labels_kernel(const double* __restrict__ dv, int64_t e_tot, int8_t* __restrict__ lab) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < e_tot) lab[e] = (dv[e] >= 0.0) ? (int8_t)1 : (int8_t)-1;
}

void predict_impl(const double* Ftrain, const double* y, const double* z, int64_t n, int r, double h,
                  const double* bias_host, int nC, const double* Ftest, int64_t m, double* dv,
                  int8_t* lab, Comm* comm, cudaStream_t s) {
  const int rp = (r + 3) / 4 * 4;
  const int SA = predict_stride(rp);
  const int ld = nC <= 1 ? 1 : nC <= 2 ? 2 : nC <= 4 ? 4 : nC <= 8 ? 8 : 16;
  DevBuf<double> Ftr((size_t)n * SA), nutr(n + kNormPad), W((size_t)n * ld + 2), b(nC);
  pad_rows(Ftrain, n, r, SA, Ftr.p, s);
  row_norms(Ftr.p, n, SA, nutr.p, s);
  CUDA_CHECK(cudaMemsetAsync(W.p + (size_t)n * ld, 0, 2 * sizeof(double), s));
  coef_kernel<<<ceil_div(n * ld, 256), 256, 0, s>>>(y, z, n, nC, ld, W.p);
  LAUNCH_CHECK();
  h2d(b.p, bias_host, nC, s);
  const int P = comm ? comm->size : 1;
  if (P == 1) {
    predict_rows(Ftr.p, nutr.p, W.p, n, r, rp, SA, ld, Ftrain, h, b.p, nC, Ftest, m, dv, lab, s);
    CUDA_CHECK(cudaStreamSynchronize(s));
    return;
  }
  // test points sharded: rank g takes [m g / P, m (g+1) / P); one allgather of the decision values
  auto lo = [&](int g) { return (int64_t)((__int128)m * g / P); };
  int64_t slot_rows = 0;
  for (int g = 0; g < P; ++g) slot_rows = std::max(slot_rows, lo(g + 1) - lo(g));
  const int64_t slot = std::max<int64_t>(1, slot_rows * nC);
  const int64_t l0 = lo(comm->rank), cnt = lo(comm->rank + 1) - l0;
  DevBuf<double> send(slot), recv(slot * P), dfull(dv ? 0 : (size_t)m * nC);
  predict_rows(Ftr.p, nutr.p, W.p, n, r, rp, SA, ld, Ftrain, h, b.p, nC, Ftest + l0 * r, cnt, send.p, nullptr, s);
  comm->allgather(send.p, recv.p, slot * sizeof(double), s);
  double* out = dv ? dv : dfull.p;
  for (int g = 0; g < P; ++g) {
    const int64_t c = lo(g + 1) - lo(g);
    if (c > 0)
      CUDA_CHECK(cudaMemcpyAsync(out + lo(g) * nC, recv.p + g * slot, (size_t)c * nC * sizeof(double),
                                 cudaMemcpyDeviceToDevice, s));
  }
  if (lab) {
    labels_kernel<<<ceil_div(m * nC, 256), 256, 0, s>>>(out, m * nC, lab);
    LAUNCH_CHECK();
  }
  CUDA_CHECK(cudaStreamSynchronize(s));
}

}  // namespace svmhss
