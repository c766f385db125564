// tiles.cu — kernel-block generation and the fused sketch product (H1/H2).
//
// kmm_kernel: S = K(Fa, Fb) W with K_ij = exp(-max(0, nu_i + nu_j - 2 f_i.f_j) / (2h^2))
// (AMB-4).  Per CTA: a 64-row tile of Fa and a 16*NT-column chunk of W, sweeping
// the Fb points in BJ-point steps:
//   (1) distance tile 64 x BJ on FP64 tensor cores (DMMA m8n8k4: the dot products f_i.f_j),
//   (2) exp + mask -> E tile in shared memory,
//   (3) S_acc(64 x 16NT) += E(64 x BJ) W(BJ x 16NT) on DMMA, accumulators in registers.
// Fb / nu_b / W tiles stream through a 2-stage cp.async pipeline; K is never stored.
// Shared-memory row strides are = 4 (mod 16) doubles so every DMMA fragment load is
// bank-conflict free.
#include "internal.cuh"

namespace svmhss {

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool pred) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

static inline int pad_stride(int x) {  // smallest S >= x with S % 16 == 4
  int S = x;
  while (S % 16 != 4) ++S;
  return S;
}

constexpr int KBM = 64;

template <int BJ, int NT>
__global__ void __launch_bounds__(256, 1) kmm_kernel(KmmArgs a, int SA) {
  constexpr int NCH = 16 * NT, SW = NCH + 4, SE = BJ + 4, HALF = NCH / 2;
  extern __shared__ __align__(16) double smem[];
  double* Fa_s = smem;
  double* nua_s = Fa_s + KBM * SA;
  double* E_s = nua_s + KBM;
  double* st0 = E_s + KBM * SE;
  const int stage_d = BJ * SA + BJ + BJ * SW;
  int* leafb_s = (int*)(st0 + 2 * stage_d);

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  const int64_t row0 = (int64_t)blockIdx.x * KBM;
  const int col0 = blockIdx.y * NCH;
  const int rp = a.rp;

  // A tile (Fa rows) and norms
  for (int e = tid; e < KBM * rp; e += 256) {
    const int i = e / rp, f = e % rp;
    const int64_t gi = row0 + i;
    Fa_s[i * SA + f] = (gi < a.na) ? a.Fa[gi * rp + f] : 0.0;
  }
  for (int i = tid; i < KBM; i += 256) {
    const int64_t gi = row0 + i;
    nua_s[i] = (gi < a.na) ? a.nua[gi] : 0.0;
  }
  const int64_t my_row = row0 + w * 8 + g;
  const int my_leaf = (a.leaf_a && my_row < a.na) ? a.leaf_a[my_row] : -1;
  int tile_leaf = -2;
  if (a.leaf_a) {
    const int64_t last = min(row0 + KBM, a.na) - 1;
    const int la = a.leaf_a[row0], lb = a.leaf_a[last];
    tile_leaf = (la == lb) ? la : -2;
  }

  double acc[2][NT][2];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

  const int64_t nsteps = (a.nb + BJ - 1) / BJ;
  auto issue = [&](int64_t js) {
    double* st = st0 + (js & 1) * stage_d;
    double* Fb_s = st;
    double* nub_s = st + BJ * SA;
    double* W_s = nub_s + BJ;
    const int64_t j0 = js * BJ;
    const int cpr = rp / 2;  // 16B chunks per feature row
    for (int e = tid; e < BJ * cpr; e += 256) {
      const int jj = e / cpr, c = e % cpr;
      const int64_t gj = j0 + jj;
      const bool ok = gj < a.nb;
      cp_async16(Fb_s + jj * SA + 2 * c, ok ? (const void*)(a.Fb + gj * rp + 2 * c) : (const void*)a.Fb, ok);
    }
    for (int e = tid; e < BJ; e += 256) {
      const int64_t gj = j0 + e;
      const bool ok = gj < a.nb;
      cp_async8(nub_s + e, ok ? (const void*)(a.nub + gj) : (const void*)a.nub, ok);
    }
    constexpr int cpw = NCH / 2;
    for (int e = tid; e < BJ * cpw; e += 256) {
      const int jj = e / cpw, c = e % cpw;
      const int64_t gj = j0 + jj;
      const int gc = col0 + 2 * c;
      const bool ok = gj < a.nb && gc < a.ncols;
      cp_async16(W_s + jj * SW + 2 * c, ok ? (const void*)(a.W + gj * a.ldw + gc) : (const void*)a.W, ok);
    }
    if (a.leaf_b) {
      int* lb = leafb_s + (js & 1) * BJ;
      for (int e = tid; e < BJ; e += 256) {
        const int64_t gj = j0 + e;
        const bool ok = gj < a.nb;
        cp_async4(lb + e, ok ? (const void*)(a.leaf_b + gj) : (const void*)a.leaf_b, ok);
      }
    }
  };

  issue(0);
  cp_async_commit();
  for (int64_t js = 0; js < nsteps; ++js) {
    if (js + 1 < nsteps) { issue(js + 1); cp_async_commit(); cp_async_wait<1>(); }
    else { cp_async_wait<0>(); }
    __syncthreads();
    const double* st = st0 + (js & 1) * stage_d;
    const double* Fb_s = st;
    double* nub_s = (double*)(st + BJ * SA);
    const double* W_s = nub_s + BJ;
    int* lb = leafb_s + (js & 1) * BJ;
    const int64_t j0 = js * BJ;
    const int jvalid = (int)min((int64_t)BJ, a.nb - j0);
    bool skip = false;
    if (a.leaf_b && tile_leaf >= 0) skip = (lb[0] == tile_leaf && lb[jvalid - 1] == tile_leaf);
    if (!skip) {
      // (1) distances for m-tile w, BJ/8 n-tiles
      double dacc[BJ / 8][2];
#pragma unroll
      for (int nt = 0; nt < BJ / 8; ++nt) dacc[nt][0] = dacc[nt][1] = 0.0;
      for (int kk = 0; kk < rp / 4; ++kk) {
        const double av = Fa_s[(w * 8 + g) * SA + kk * 4 + t];
#pragma unroll
        for (int nt = 0; nt < BJ / 8; ++nt) {
          const double bv = Fb_s[(nt * 8 + g) * SA + kk * 4 + t];
          dmma884(dacc[nt][0], dacc[nt][1], av, bv);
        }
      }
      // (2) exp + masks -> E
      const double nui = nua_s[w * 8 + g];
#pragma unroll
      for (int nt = 0; nt < BJ / 8; ++nt) {
        double ev[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int jj = nt * 8 + 2 * t + e;
          const int64_t gj = j0 + jj;
          double d2 = nui + nub_s[jj] - 2.0 * dacc[nt][e];
          d2 = fmax(d2, 0.0);
          double v = exp(d2 * a.neg_inv_2h2);
          if (a.same_set && gj == my_row) v = 1.0;
          if (a.leaf_b && lb[jj] == my_leaf) v = 0.0;
          if (jj >= jvalid || my_row >= a.na) v = 0.0;
          ev[e] = v;
        }
        *reinterpret_cast<double2*>(&E_s[(w * 8 + g) * SE + nt * 8 + 2 * t]) = make_double2(ev[0], ev[1]);
      }
      __syncthreads();
      // (3) S_acc += E W
      const int wm = w & 3, wn = w >> 2;
#pragma unroll
      for (int kk = 0; kk < BJ / 4; ++kk) {
        const double a0 = E_s[(wm * 16 + g) * SE + kk * 4 + t];
        const double a1 = E_s[(wm * 16 + 8 + g) * SE + kk * 4 + t];
        const double* wrow = W_s + (kk * 4 + t) * SW + wn * HALF + g;
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) {
          const double bv = wrow[ni * 8];
          dmma884(acc[0][ni][0], acc[0][ni][1], a0, bv);
          dmma884(acc[1][ni][0], acc[1][ni][1], a1, bv);
        }
      }
    }
    __syncthreads();
  }
  // epilogue
  const int wm = w & 3, wn = w >> 2;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi) {
    const int64_t gi = row0 + wm * 16 + mi * 8 + g;
    if (gi >= a.na) continue;
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      const int gc = col0 + wn * HALF + ni * 8 + 2 * t;
      if (gc < a.ncols) {
        double* dst = a.S + gi * a.lds + gc;
        if (gc + 1 < a.ncols) {
          dst[0] = acc[mi][ni][0];
          dst[1] = acc[mi][ni][1];
        } else {
          dst[0] = acc[mi][ni][0];
        }
      }
    }
  }
}

static size_t kmm_smem(int BJ, int NT, int SA) {
  const int NCH = 16 * NT, SW = NCH + 4, SE = BJ + 4;
  return 8 * (size_t)(KBM * SA + KBM + KBM * SE + 2 * (BJ * SA + BJ + BJ * SW)) + 2 * BJ * 4;
}

static int pick_nt(int ncols) {
  if (ncols <= 16) return 1;
  if (ncols <= 80) return 5;
  if (ncols <= 144) return 9;
  return 17;
}

int kmm_chunk_cols(int rp, int ncols) { (void)rp; return 16 * pick_nt(ncols); }

template <int BJ, int NT>
static void launch_kmm(const KmmArgs& a, int SA, cudaStream_t s) {
  const size_t smem = kmm_smem(BJ, NT, SA);
  CUDA_CHECK(cudaFuncSetAttribute(kmm_kernel<BJ, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  dim3 grid((unsigned)((a.na + KBM - 1) / KBM), (unsigned)ceil_div(a.ncols, 16 * NT));
  kmm_kernel<BJ, NT><<<grid, 256, smem, s>>>(a, SA);
  LAUNCH_CHECK();
}

void kernel_matmul(const KmmArgs& a, cudaStream_t s) {
  if (a.na <= 0 || a.ncols <= 0) return;
  require(a.rp % 4 == 0, "kernel_matmul: rp must be a multiple of 4");
  require(a.ldw % 2 == 0 && a.ncols % 2 == 0, "kernel_matmul: W columns / ld must be even");
  if (a.nb <= 0) {  // nothing to accumulate: zero output
    CUDA_CHECK(cudaMemset2DAsync(a.S, a.lds * 8, 0, a.ncols * 8, a.na, s));
    return;
  }
  const int SA = pad_stride(a.rp);
  const int NT = pick_nt(a.ncols);
  const size_t lim = 227 * 1024;
  const int BJ = (kmm_smem(32, NT, SA) <= lim) ? 32 : 16;
  require(kmm_smem(BJ, NT, SA) <= lim, "kernel_matmul: feature dimension too large for shared memory");
#define KMM_CASE(bj, nt) if (BJ == bj && NT == nt) { launch_kmm<bj, nt>(a, SA, s); return; }
  KMM_CASE(32, 1) KMM_CASE(32, 5) KMM_CASE(32, 9) KMM_CASE(32, 17)
  KMM_CASE(16, 1) KMM_CASE(16, 5) KMM_CASE(16, 9) KMM_CASE(16, 17)
#undef KMM_CASE
  throw Error(HSS_EINVAL, "kernel_matmul: no kernel configuration");
}

// ------------------------------------------------------------------ Omega (R1-R3)
__global__ void omega_kernel(uint64_t key, const int64_t* __restrict__ idx, int64_t rows, int s,
                             double* __restrict__ out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= rows * s) return;
  const int64_t i = e / s;
  const int j = (int)(e % s);
  out[e] = counter_gaussian(key, (uint64_t)idx[i], (uint64_t)j);
}

void omega_rows(uint64_t seed, const int64_t* idx, int64_t rows, int s, double* out,
                cudaStream_t st) {
  if (rows <= 0 || s <= 0) return;
  const int64_t tot = rows * s;
  omega_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(splitmix64(seed), idx, rows, s, out);
  LAUNCH_CHECK();
}

// ------------------------------------------------------------------ direct kernel blocks
__global__ void kblock_kernel(const double* __restrict__ F, int rp, int r, double two_h2,
                              const KblkProb* __restrict__ probs) {
  const KblkProb P = probs[blockIdx.z];
  const int i0 = blockIdx.y * 16, j0 = blockIdx.x * 16;
  if (i0 >= P.na || j0 >= P.nb) return;
  extern __shared__ double sh[];
  double* As = sh;            // 16 x r
  double* Bs = sh + 16 * r;   // 16 x r
  __shared__ int64_t ia_s[16], ib_s[16];
  const int tid = threadIdx.y * 16 + threadIdx.x;
  if (tid < 16) {
    const int i = i0 + tid;
    ia_s[tid] = (i < P.na) ? (P.ia ? P.ia[i] : P.a0 + i) : -1;
  } else if (tid < 32) {
    const int j = j0 + tid - 16;
    ib_s[tid - 16] = (j < P.nb) ? (P.ib ? P.ib[j] : P.b0 + j) : -1;
  }
  __syncthreads();
  for (int e = tid; e < 16 * r; e += 256) {
    const int q = e / r, f = e % r;
    As[e] = ia_s[q] >= 0 ? F[ia_s[q] * rp + f] : 0.0;
    Bs[e] = ib_s[q] >= 0 ? F[ib_s[q] * rp + f] : 0.0;
  }
  __syncthreads();
  const int ti = threadIdx.y, tj = threadIdx.x;
  const int i = i0 + ti, j = j0 + tj;
  if (i >= P.na || j >= P.nb) return;
  double d2 = 0.0;
  for (int f = 0; f < r; ++f) {
    const double d = As[ti * r + f] - Bs[tj * r + f];
    d2 = fma(d, d, d2);
  }
  double v = exp(-d2 / two_h2);
  if (ia_s[ti] == ib_s[tj]) v = 1.0 + P.diag_add;
  P.out[(long long)i * P.ld + j] = v;
}

void kernel_blocks(const double* F, int rp, int r, double h, const std::vector<KblkProb>& probs_in,
                   cudaStream_t s) {
  std::vector<KblkProb> probs;
  int mr = 0, mc = 0;
  for (auto& p : probs_in)
    if (p.na > 0 && p.nb > 0) { probs.push_back(p); mr = std::max(mr, p.na); mc = std::max(mc, p.nb); }
  if (probs.empty()) return;
  const double two_h2 = 2.0 * h * h;
  for (size_t b0 = 0; b0 < probs.size(); b0 += 65535) {
    std::vector<KblkProb> chunk(probs.begin() + b0, probs.begin() + std::min(probs.size(), b0 + 65535));
    KblkProb* d = nullptr;
    CUDA_CHECK(cudaMallocAsync((void**)&d, chunk.size() * sizeof(KblkProb), s));
    CUDA_CHECK(cudaMemcpyAsync(d, chunk.data(), chunk.size() * sizeof(KblkProb), cudaMemcpyHostToDevice, s));
    dim3 grid(ceil_div(mc, 16), ceil_div(mr, 16), (unsigned)chunk.size());
    size_t smem = 2 * 16 * (size_t)r * sizeof(double);
    if (smem > 48 * 1024)
      CUDA_CHECK(cudaFuncSetAttribute(kblock_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kblock_kernel<<<grid, dim3(16, 16), smem, s>>>(F, rp, r, two_h2, d);
    LAUNCH_CHECK();
    CUDA_CHECK(cudaFreeAsync(d, s));
  }
}

// ------------------------------------------------------------------ small helpers
__global__ void pad_rows_kernel(const double* __restrict__ F, int64_t n, int r, int rp, double* out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * rp) return;
  const int64_t i = e / rp;
  const int f = (int)(e % rp);
  out[e] = (f < r) ? F[i * r + f] : 0.0;
}
void pad_rows(const double* F, int64_t n, int r, int rp, double* out, cudaStream_t s) {
  const int64_t tot = n * rp;
  if (tot <= 0) return;
  pad_rows_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(F, n, r, rp, out);
  LAUNCH_CHECK();
}

__global__ void row_norms_kernel(const double* __restrict__ F, int64_t n, int rp, double* nu) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double a = 0.0;
  for (int f = 0; f < rp; ++f) { const double x = F[i * rp + f]; a = fma(x, x, a); }
  nu[i] = a;
}
void row_norms(const double* F, int64_t n, int rp, double* nu, cudaStream_t s) {
  if (n <= 0) return;
  row_norms_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(F, n, rp, nu);
  LAUNCH_CHECK();
}

__global__ void bcopy_kernel(const CopyProb* __restrict__ probs) {
  const CopyProb P = probs[blockIdx.y];
  const int64_t tot = (int64_t)P.rows * P.cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / P.cols, j = e % P.cols;
    const double v = P.src[i * P.srs + j];
    double* d = P.dst + i * P.drs + j;
    *d = P.accumulate ? *d + v : v;
  }
}
void bcopy(const std::vector<CopyProb>& probs_in, cudaStream_t s) {
  std::vector<CopyProb> probs;
  int64_t mx = 0;
  for (auto& p : probs_in)
    if (p.rows > 0 && p.cols > 0) { probs.push_back(p); mx = std::max(mx, (int64_t)p.rows * p.cols); }
  if (probs.empty()) return;
  for (size_t b0 = 0; b0 < probs.size(); b0 += 65535) {
    std::vector<CopyProb> chunk(probs.begin() + b0, probs.begin() + std::min(probs.size(), b0 + 65535));
    CopyProb* d = nullptr;
    CUDA_CHECK(cudaMallocAsync((void**)&d, chunk.size() * sizeof(CopyProb), s));
    CUDA_CHECK(cudaMemcpyAsync(d, chunk.data(), chunk.size() * sizeof(CopyProb), cudaMemcpyHostToDevice, s));
    dim3 grid((unsigned)std::min<int64_t>(1024, (mx + 255) / 256), (unsigned)chunk.size());
    bcopy_kernel<<<grid, 256, 0, s>>>(d);
    LAUNCH_CHECK();
    CUDA_CHECK(cudaFreeAsync(d, s));
  }
}

__global__ void gather_rows_kernel(const double* __restrict__ src, const int64_t* __restrict__ idx,
                                   int64_t rows, int cols, double* __restrict__ dst, int scatter) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  const int64_t i = e / cols;
  const int c = (int)(e % cols);
  if (scatter) dst[idx[i] * cols + c] = src[e];
  else dst[e] = src[idx[i] * cols + c];
}
void gather_rows(const double* src, const int64_t* idx, int64_t rows, int cols, double* dst,
                 cudaStream_t s) {
  const int64_t tot = rows * cols;
  if (tot <= 0) return;
  gather_rows_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(src, idx, rows, cols, dst, 0);
  LAUNCH_CHECK();
}
void scatter_rows(const double* src, const int64_t* idx, int64_t rows, int cols, double* dst,
                  cudaStream_t s) {
  const int64_t tot = rows * cols;
  if (tot <= 0) return;
  gather_rows_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(src, idx, rows, cols, dst, 1);
  LAUNCH_CHECK();
}

}  // namespace svmhss
