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

// exp(x) for the Gaussian kernel entries (x = -d2 / (2h^2) <= 0), table-driven: x = (64 m + j)
// ln2/64 + r with |r| <= ln2/128 (Cody-Waite split of ln2/64), exp(x) = 2^m 2^(j/64) e^r,
// 2^(j/64) from a 64-entry table in shared memory (correctly rounded constants,
// scripts/gen_exp_table.py), e^r by a degree-5 Taylor polynomial (truncation < r^6/720 < 4e-17),
// 2^m as two exact power-of-two factors (gradual underflow; 0 below -745).  13 FP64 operations
// per entry instead of the 20 of a degree-13 polynomial on |r| <= ln2/2 (the FP64 pipe also
// runs the DMMAs of the sketch and prediction kernels).  <= 2 ulp against the correctly rounded
// exp (tests/test_gpu_parity.py pins the sketch at 1e-12, tests/test_gpu_predict.py at 1e-12).
__constant__ double c_exp2_64[64] = {
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0,
    0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0,
    0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0,
    0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0, 0x1.2d285a6e4030bp+0,
    0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0,
    0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0,
    0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0,
    0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0, 0x1.6247eb03a5585p+0, 0x1.6623882552225p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0,
    0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0,
    0x1.9c49182a3f090p+0, 0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0,
    0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0,
    0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0,
    0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0,
};

__device__ __forceinline__ void exp_table_load(double* t) {
  for (int e = threadIdx.x; e < 64; e += blockDim.x) t[e] = c_exp2_64[e];
}
__device__ __forceinline__ double exp_kernel(double x, const double* __restrict__ tab) {
  x = fmax(x, -1100.0);
  const double kShift = 6755399441055744.0;  // 1.5 * 2^52: t's low word holds round(64 x / ln2)
  const double t = fma(x, 0x1.71547652b82fep+6, kShift);
  const double n = t - kShift;
  const int ni = __double2loint(t);
  double r = fma(n, -0x1.62e42fefa0000p-7, x);
  r = fma(n, -0x1.cf79abc9e3b3ap-46, r);
  double p = 1.0 / 120.0;
  p = fma(p, r, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const double tj = tab[ni & 63];
  const int m = ni >> 6;                       // floor(n / 64)
  const int h1 = m >> 1, h2 = m - h1;          // 2^m = 2^h1 * 2^h2, each a normal number
  return ((tj * p) * __hiloint2double((h1 + 1023) << 20, 0)) * __hiloint2double((h2 + 1023) << 20, 0);
}

// --- mbarrier / bulk-copy (TMA) helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// 16 warps (4 per SM sub-partition, so DMMA latency and the exp dependency chains of one
// warp hide under the others).  Warp w: m-tile mt = w & 7 (rows mt*8..mt*8+7) and column half
// hf = w >> 3.  Per j-step of BJ = 32 points:
//   (1) distance DMMAs for (mt, its 16 of the BJ columns) -> exp/mask -> E tile in smem,
//       then a 64-thread named barrier with the partner warp of the same m-tile;
//   (2) sketch DMMAs S_acc(8 rows x 8*NT cols) += E(8 x BJ) W(BJ x 8*NT cols).
// Operands arrive by TMA bulk copies (cp.async.bulk, one row per copy into padded smem rows)
// into a 2-stage ring completed on mbarriers; one CTA barrier per step guards buffer reuse.
// Persistent, wave-synchronous schedule: gridDim.x CTAs (one per SM) walk the 64-row tiles
// tile = blockIdx.x + it * gridDim.x, and a grid barrier after every tile keeps the whole wave
// on the same j-step of the (tile-independent) operand stream, so each W / Fb tile is read from
// HBM about once per wave and served from L2 to the other CTAs (the unsynchronised grid read
// Omega ~50x more often than this).  The operand ring runs continuously across tiles (global
// step counter G): the prefetch of a tile's first step overlaps the previous tile's epilogue.
// Requires co-residency of the grid: launched cooperatively.
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <int BJ, int NT>
__global__ void __launch_bounds__(512, 1) kmm_kernel(KmmArgs a, int SA, unsigned* gbar,
                                                     unsigned long long* probe) {
  const unsigned long long t_start = probe ? gtimer() : 0ull;
  unsigned long long t_wait = 0ull;
  constexpr int NCH = 16 * NT, SW = NCH + 4, SE = BJ + 4, HQ = BJ / 16;  // n-tiles of distance per warp
  extern __shared__ __align__(128) double smem[];
  double* Fa_s = smem;                       // 64 x SA
  double* nua_s = Fa_s + KBM * SA;           // 64
  double* E_s = nua_s + KBM;                 // 64 x SE
  double* wbuf = E_s + KBM * SE;             // 2 x BJ x SW
  double* fbuf = wbuf + 2 * BJ * SW;         // 2 x (BJ x SA + BJ)
  int* lbuf = (int*)(fbuf + 2 * (BJ * SA + BJ));  // 2 x BJ
  __shared__ __align__(8) uint64_t full[2];   // stage filled (TMA transaction count)
  __shared__ __align__(8) uint64_t empty[2];  // stage released by all 16 warps
  __shared__ double exp_t[64];
  exp_table_load(exp_t);

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  const int mt = w & 7, hf = w >> 3;
  const int col0 = blockIdx.y * NCH;
  const int rp = a.rp;
  const int ncl = min(NCH, a.ncols - col0);  // valid columns of this chunk (even)
  const int64_t nsteps = (a.nb + BJ - 1) / BJ;
  const int64_t ntiles = (a.na + KBM - 1) / KBM;
  const int64_t niter = (ntiles + gridDim.x - 1) / gridDim.x;

  for (int e = tid; e < 2 * BJ * SW + 2 * (BJ * SA + BJ); e += 512) wbuf[e] = 0.0;
  for (int e = tid; e < 2 * BJ; e += 512) lbuf[e] = -3;
  if (tid == 0) {
    mbar_init(&full[0], 1); mbar_init(&full[1], 1);
    mbar_init(&empty[0], 16); mbar_init(&empty[1], 16);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();

  auto issue = [&](int64_t G) {  // warp 0: one bulk copy per row; global step G -> j-step G mod nsteps
    const int b = (int)(G & 1);
    const int64_t j = G % nsteps;
    double* W_s = wbuf + b * BJ * SW;
    double* Fb_s = fbuf + b * (BJ * SA + BJ);
    double* nub_s = Fb_s + BJ * SA;
    int* lb = lbuf + b * BJ;
    const int64_t j0 = j * BJ;
    const int jv = (int)min((int64_t)BJ, a.nb - j0);
    const unsigned nb8 = (unsigned)(((jv * 8) + 15) & ~15), lb4 = (unsigned)(((jv * 4) + 15) & ~15);
    if (lane == 0)
      mbar_expect_tx(&full[b], (unsigned)jv * (rp * 8 + ncl * 8) + nb8 + (a.leaf_b ? lb4 : 0u));
    __syncwarp();
    for (int jj = lane; jj < jv; jj += 32) {
      bulk_g2s(W_s + jj * SW, a.W + (j0 + jj) * a.ldw + col0, ncl * 8, &full[b]);
      bulk_g2s(Fb_s + jj * SA, a.Fb + (j0 + jj) * rp, rp * 8, &full[b]);
    }
    if (lane == 0) {
      bulk_g2s(nub_s, a.nub + j0, nb8, &full[b]);
      if (a.leaf_b) bulk_g2s(lb, a.leaf_b + j0, lb4, &full[b]);
    }
  };

  const int64_t total = niter * nsteps;  // every CTA runs the same number of steps (idle tiles too)
  int64_t G = 0;
  if (w == 0) issue(0);
  for (int64_t it = 0; it < niter; ++it) {
    const int64_t tile = blockIdx.x + it * gridDim.x;
    const bool active = tile < ntiles;
    const int64_t row0 = tile * KBM;
    for (int e = tid; e < KBM * rp; e += 512) {
      const int i = e / rp, f = e % rp;
      const int64_t gi = row0 + i;
      Fa_s[i * SA + f] = (active && gi < a.na) ? a.Fa[gi * rp + f] : 0.0;
    }
    for (int i = tid; i < KBM; i += 512) {
      const int64_t gi = row0 + i;
      nua_s[i] = (active && gi < a.na) ? a.nua[gi] : 0.0;
    }
    __syncthreads();
    const int64_t my_row = row0 + mt * 8 + g;
    const bool row_ok = active && my_row < a.na;
    const int my_leaf = (a.leaf_a && row_ok) ? a.leaf_a[my_row] : -1;
    const double nui = nua_s[mt * 8 + g];
    const double* Fa_w = Fa_s + (mt * 8 + g) * SA + t;
    const double* E_w = E_s + (mt * 8 + g) * SE + t;

    double acc[NT][2];
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) acc[ni][0] = acc[ni][1] = 0.0;
    for (int64_t js = 0; js < nsteps; ++js, ++G) {
      const int b = (int)(G & 1);
      mbar_wait(&full[b], (unsigned)((G >> 1) & 1));
      if (w == 0 && G + 1 < total) {
        // the other stage held step G-1: refill it once all 16 warps released it
        if (G >= 1) mbar_wait(&empty[b ^ 1], (unsigned)(((G - 1) >> 1) & 1));
        issue(G + 1);
      }
      const double* W_s = wbuf + b * BJ * SW;
      const double* Fb_s = fbuf + b * (BJ * SA + BJ);
      const double* nub_s = Fb_s + BJ * SA;
      const int* lb = lbuf + b * BJ;
      const int64_t j0 = js * BJ;
      const int jvalid = (int)min((int64_t)BJ, a.nb - j0);
      if (!active) {  // idle tile: keep the ring in step
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[b]);
        continue;
      }
      // (1) distances: rows mt*8.., columns hf*BJ/2 + [0, BJ/2)
      double dacc[HQ][2];
#pragma unroll
      for (int q = 0; q < HQ; ++q) dacc[q][0] = dacc[q][1] = 0.0;
      const double* Fb_w = Fb_s + (hf * (BJ / 2) + g) * SA + t;
      {
        // two interleaved partial sums per tile: 2*HQ independent DMMA chains of rp/8 steps
        double dacc2[HQ][2];
#pragma unroll
        for (int q = 0; q < HQ; ++q) dacc2[q][0] = dacc2[q][1] = 0.0;
        int kk = 0;
        for (; kk + 1 < rp / 4; kk += 2) {
          const double av0 = Fa_w[kk * 4], av1 = Fa_w[kk * 4 + 4];
#pragma unroll
          for (int q = 0; q < HQ; ++q) {
            dmma884(dacc[q][0], dacc[q][1], av0, Fb_w[q * 8 * SA + kk * 4]);
            dmma884(dacc2[q][0], dacc2[q][1], av1, Fb_w[q * 8 * SA + kk * 4 + 4]);
          }
        }
        if (kk < rp / 4) {
          const double av = Fa_w[kk * 4];
#pragma unroll
          for (int q = 0; q < HQ; ++q) dmma884(dacc[q][0], dacc[q][1], av, Fb_w[q * 8 * SA + kk * 4]);
        }
#pragma unroll
        for (int q = 0; q < HQ; ++q) { dacc[q][0] += dacc2[q][0]; dacc[q][1] += dacc2[q][1]; }
      }
      // the partner warp (same m-tile) has finished reading E_s of the previous step
      asm volatile("bar.sync %0, 64;\n" ::"r"(1 + mt) : "memory");
#pragma unroll
      for (int q = 0; q < HQ; ++q) {
        double ev[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int jj = hf * (BJ / 2) + q * 8 + 2 * t + e;
          double d2 = fmax(nui + nub_s[jj] - 2.0 * dacc[q][e], 0.0);
          double v = exp_kernel(d2 * a.neg_inv_2h2, exp_t);
          if (a.same_set && j0 + jj == my_row + a.diag_off) v = 1.0;
          if (a.leaf_b && lb[jj] == my_leaf) v = 0.0;
          if (jj >= jvalid || !row_ok) v = 0.0;
          ev[e] = v;
        }
        *reinterpret_cast<double2*>(&E_s[(mt * 8 + g) * SE + hf * (BJ / 2) + q * 8 + 2 * t]) =
            make_double2(ev[0], ev[1]);
      }
      asm volatile("bar.sync %0, 64;\n" ::"r"(1 + mt) : "memory");  // partner warps w, w^8
      // (2) sketch: columns hf*8*NT .. + 8*NT
      const double* W_w = W_s + t * SW + hf * (8 * NT) + g;
#pragma unroll
      for (int kk = 0; kk < BJ / 4; ++kk) {
        const double av = E_w[kk * 4];
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) dmma884(acc[ni][0], acc[ni][1], av, W_w[kk * 4 * SW + ni * 8]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[b]);  // this warp is done with stage b
    }
    // epilogue
    if (row_ok) {
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) {
        const int gc = col0 + hf * (8 * NT) + ni * 8 + 2 * t;
        if (gc < a.ncols) {
          double* dst = a.S + my_row * a.lds + gc;
          dst[0] = acc[ni][0];
          if (gc + 1 < a.ncols) dst[1] = acc[ni][1];
        }
      }
    }
    // wave barrier (grid-wide, per column chunk): nobody starts tile it+1 before all finished it
    if (it + 1 < niter) {
      __syncthreads();
      if (tid == 0) {
        const unsigned long long t0 = probe ? gtimer() : 0ull;
        unsigned* bar = gbar + blockIdx.y;
        __threadfence();
        atomicAdd(bar, 1u);
        const unsigned target = (unsigned)((it + 1) * gridDim.x);
        while (atomicAdd(bar, 0u) < target) __nanosleep(200);
        if (probe) t_wait += gtimer() - t0;
      }
      __syncthreads();
    }
  }
  if (probe && tid == 0) {  // diagnostics (SVMHSS_KMM_PROBE=1): barrier wait and total time per CTA
    const int b = blockIdx.y * gridDim.x + blockIdx.x;
    probe[2 * b] = t_wait;
    probe[2 * b + 1] = gtimer() - t_start;
  }
}

static size_t kmm_smem(int BJ, int NT, int SA) {
  const int NCH = 16 * NT, SW = NCH + 4, SE = BJ + 4;
  return 8 * (size_t)(KBM * SA + KBM + KBM * SE + 2 * BJ * SW + 2 * (BJ * SA + BJ)) + 2 * BJ * 4;
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
  int dev = 0, nsm = 0, per_sm = 0;
  CUDA_CHECK(cudaGetDevice(&dev));
  CUDA_CHECK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kmm_kernel<BJ, NT>, 512, smem));
  const int nchunk = ceil_div(a.ncols, 16 * NT);
  const int64_t ntiles = (a.na + KBM - 1) / KBM;
  // co-resident grid: every column chunk gets (SMs * per_sm) / nchunk persistent CTAs
  const int64_t slots = std::max<int64_t>(1, ((int64_t)nsm * std::max(1, per_sm)) / nchunk);
  const unsigned gx = (unsigned)std::max<int64_t>(1, std::min(ntiles, slots));
  DevBuf<unsigned> gbar(nchunk);
  CUDA_CHECK(cudaMemsetAsync(gbar.p, 0, nchunk * sizeof(unsigned), s));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(gx, (unsigned)nchunk);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  static const bool probe_on = [] { const char* e = getenv("SVMHSS_KMM_PROBE"); return e && e[0] == '1'; }();
  const int nb = (int)gx * nchunk;
  DevBuf<unsigned long long> probe(probe_on ? 2 * (size_t)nb : 0);
  CUDA_CHECK(cudaLaunchKernelEx(&cfg, kmm_kernel<BJ, NT>, a, SA, gbar.p, probe_on ? probe.p : (unsigned long long*)nullptr));
  LAUNCH_CHECK();
  if (probe_on) {
    std::vector<unsigned long long> h(2 * (size_t)nb);
    d2h(h.data(), probe.p, h.size(), s);
    CUDA_CHECK(cudaStreamSynchronize(s));
    double w = 0, tmax = 0, wmax = 0;
    for (int b = 0; b < nb; ++b) { w += h[2 * b]; tmax = std::max(tmax, (double)h[2 * b + 1]); wmax = std::max(wmax, (double)h[2 * b]); }
    fprintf(stderr, "[kmm probe] na=%lld nb=%lld grid=%dx%d: mean barrier wait %.3f ms (max %.3f) of %.3f ms\n",
            (long long)a.na, (long long)a.nb, (int)gx, nchunk, w / nb / 1e6, wmax / 1e6, tmax / 1e6);
  }
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
  // narrow right-hand sides (prediction: 16 columns): 64-point steps, so each warp runs 4
  // distance tiles (8 independent DMMA chains) per step and the per-step barriers amortise
  const int BJ = (NT <= 5 && kmm_smem(64, NT, SA) <= lim) ? 64 : (kmm_smem(32, NT, SA) <= lim) ? 32 : 16;
  require(kmm_smem(BJ, NT, SA) <= lim, "kernel_matmul: feature dimension too large for shared memory");
#define KMM_CASE(bj, nt) if (BJ == bj && NT == nt) { launch_kmm<bj, nt>(a, SA, s); return; }
  KMM_CASE(64, 1) KMM_CASE(64, 5)
  KMM_CASE(32, 1) KMM_CASE(32, 5) KMM_CASE(32, 9) KMM_CASE(32, 17)
  KMM_CASE(16, 1) KMM_CASE(16, 5) KMM_CASE(16, 9) KMM_CASE(16, 17)
#undef KMM_CASE
  throw Error(HSS_EINVAL, "kernel_matmul: no kernel configuration");
}

// ------------------------------------------------------------------ prediction (a11)
// dv_t = sum_i coef_i K(f_i, t) for nC <= 16 coefficient columns.  One CTA = 128 test
// points (16 warps x one 8-row m-tile); the warp keeps its rows' A-fragments in registers for the
// whole sweep, so a step needs only the B-fragments of the 64 training points.  Per step:
// distance tile 8 x 64 on DMMA (8 independent chains of rp/4), exp, and the coefficient-weighted
// sums accumulated in registers (a GEMV: no second DMMA, no shared-memory exchange).  Training
// tiles (features with row stride PSA = 4 mod 16, norms, coefficients) stream through a
// 3-stage TMA bulk-copy ring.  Per-thread sums run in training-point order; the 4 lanes of a
// row are combined by a fixed butterfly.
constexpr int PBJ = 64, PST = 3;

// NKM: register A-fragments per thread (rp <= 4 NKM); NW warps per CTA (rows = 8 NW).
template <int NC, int NKM, int NW>
__global__ void __launch_bounds__(NW * 32, 1) predict_kernel(const double* __restrict__ Fa, const double* __restrict__ nua,
                                                         int64_t na, const double* __restrict__ Fb,
                                                         const double* __restrict__ nub, const double* __restrict__ coef,
                                                         int64_t nb, int rp, int SA, double neg_inv_2h2,
                                                         double* __restrict__ S, int nst) {
  extern __shared__ __align__(128) double psm[];
  const int cpad = (PBJ * NC + 1) & ~1;
  const int stage_d = PBJ * SA + PBJ + cpad;          // doubles per stage (16-byte multiples)
  __shared__ __align__(8) uint64_t full[PST];
  __shared__ __align__(8) uint64_t empty[PST];
  __shared__ double exp_t[64];
  exp_table_load(exp_t);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  const int64_t row0 = (int64_t)blockIdx.x * (8 * NW);
  const int64_t nsteps = (nb + PBJ - 1) / PBJ;
  if (tid == 0) {
    for (int b = 0; b < nst; ++b) { mbar_init(&full[b], 1); mbar_init(&empty[b], NW); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t js) {
    const int b = (int)(js % nst);
    double* Fs = psm + (size_t)b * stage_d;
    double* ns = Fs + PBJ * SA;
    double* cs = ns + PBJ;
    const int64_t j0 = js * PBJ;
    const int jv = (int)min((int64_t)PBJ, nb - j0);
    const unsigned fb = (unsigned)jv * SA * 8, nbv = (unsigned)((jv * 8 + 15) & ~15),
                   cb = (unsigned)((jv * NC * 8 + 15) & ~15);
    mbar_expect_tx(&full[b], fb + nbv + cb);
    bulk_g2s(Fs, Fb + j0 * SA, fb, &full[b]);
    bulk_g2s(ns, nub + j0, nbv, &full[b]);
    bulk_g2s(cs, coef + j0 * NC, cb, &full[b]);
  };
  if (tid == 0)
    for (int64_t js = 0; js < min((int64_t)nst, nsteps); ++js) issue(js);
  // this warp's rows: A-fragments (row g, k = 4 kk + t) in registers for the whole sweep
  const int64_t my_row = row0 + w * 8 + g;
  const bool row_ok = my_row < na;
  double fa[NKM];
#pragma unroll
  for (int kk = 0; kk < NKM; ++kk)
    fa[kk] = (row_ok && 4 * kk < rp) ? Fa[my_row * SA + 4 * kk + t] : 0.0;
  const double nui = row_ok ? nua[my_row] : 0.0;
  double acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0.0;
  const int nk = rp / 4;
  for (int64_t js = 0; js < nsteps; ++js) {
    const int b = (int)(js % nst);
    mbar_wait(&full[b], (unsigned)((js / nst) & 1));
    // refill the stage of step js-1 (released by every warp by now, in the common case)
    if (tid == 0 && js >= 1 && js - 1 + nst < nsteps) {
      const int pb = (int)((js - 1) % nst);
      mbar_wait(&empty[pb], (unsigned)(((js - 1) / nst) & 1));
      issue(js - 1 + nst);
    }
    const double* Fs = psm + (size_t)b * stage_d;
    const double* ns = Fs + PBJ * SA;
    const double* cs = ns + PBJ;
    const int jv = (int)min((int64_t)PBJ, nb - js * PBJ);
    double d[8][2];
#pragma unroll
    for (int q = 0; q < 8; ++q) d[q][0] = d[q][1] = 0.0;
    const double* Fw = Fs + g * SA + t;
#pragma unroll
    for (int kk = 0; kk < NKM; ++kk) {
      if (kk < nk) {
#pragma unroll
        for (int q = 0; q < 8; ++q) dmma884(d[q][0], d[q][1], fa[kk], Fw[q * 8 * SA + 4 * kk]);
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int jj = q * 8 + 2 * t + e;
        const double d2 = fmax(nui + ns[jj] - 2.0 * d[q][e], 0.0);
        double v = exp_kernel(d2 * neg_inv_2h2, exp_t);
        if (jj >= jv) v = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c] = fma(v, cs[jj * NC + c], acc[c]);
      }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[b]);
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], 1);
    acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], 2);
  }
  if (row_ok && t == 0)
#pragma unroll
    for (int c = 0; c < NC; ++c) S[my_row * NC + c] = acc[c];
}

int predict_stride(int rp) { return pad_stride(rp); }

template <int NC, int NKM, int NW>
static void launch_predict(const double* Fa, const double* nua, int64_t na, const double* Fb, const double* nub,
                           const double* coef, int64_t nb, int rp, int SA, double c, double* S, cudaStream_t s) {
  const size_t stage = (size_t)(PBJ * SA + PBJ + ((PBJ * NC + 1) & ~1)) * sizeof(double);
  const int nst = (PST * stage <= 220 * 1024) ? PST : 2;   // 3-stage ring, 2 for wide features
  const size_t smem = nst * stage;
  require(smem <= 220 * 1024, "predict: feature dimension too large for shared memory");
  CUDA_CHECK(cudaFuncSetAttribute(predict_kernel<NC, NKM, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const unsigned grid = (unsigned)((na + 8 * NW - 1) / (8 * NW));
  predict_kernel<NC, NKM, NW><<<grid, NW * 32, smem, s>>>(Fa, nua, na, Fb, nub, coef, nb, rp, SA, c, S, nst);
  LAUNCH_CHECK();
}

void predict_sums(const double* Fa, const double* nua, int64_t na, const double* Fb, const double* nub,
                  const double* coef, int64_t nb, int rp, int SA, int NC, double neg_inv_2h2, double* S,
                  cudaStream_t s) {
  if (na <= 0) return;
  require(rp % 4 == 0 && rp <= 128, "predict: padded feature count must be a multiple of 4 and <= 128");
#define PRED_CASE(nc)                                                                                       \
  if (NC == nc) {                                                                                          \
    if (rp <= 32) launch_predict<nc, 8, 16>(Fa, nua, na, Fb, nub, coef, nb, rp, SA, neg_inv_2h2, S, s);     \
    else if (rp <= 64) launch_predict<nc, 16, 16>(Fa, nua, na, Fb, nub, coef, nb, rp, SA, neg_inv_2h2, S, s); \
    else launch_predict<nc, 32, 8>(Fa, nua, na, Fb, nub, coef, nb, rp, SA, neg_inv_2h2, S, s);              \
    return;                                                                                                \
  }
  PRED_CASE(1) PRED_CASE(2) PRED_CASE(4) PRED_CASE(8) PRED_CASE(16)
#undef PRED_CASE
  throw Error(HSS_EINVAL, "predict: NC must be 1, 2, 4, 8 or 16");
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
// 64 x 64 entries per CTA, 4 x 4 per thread (rows ty + 16a, columns tx + 16b): the gathered
// feature rows staged in shared memory (32 features at a time, odd row stride: conflict-free
// column reads), each
// entry d2 = sum_f (a_f - b_f)^2 by fma in feature order, then exp(-d2 / 2h^2) -- the per-entry
// arithmetic of the direct-difference definition (AMB-4), unchanged by the register blocking.
constexpr int KBT = 64, KBF = 32, KBS = KBF + 1;  // features staged KBF at a time, odd stride
__global__ void __launch_bounds__(256) kblock_kernel(const double* __restrict__ F, int rp, int r, double two_h2,
                                                     const KblkProb* __restrict__ probs) {
  const KblkProb P = probs[blockIdx.z];
  const int i0 = blockIdx.y * KBT, j0 = blockIdx.x * KBT;
  if (i0 >= P.na || j0 >= P.nb) return;
  __shared__ double As[KBT * KBS], Bs[KBT * KBS];
  __shared__ int64_t ia_s[KBT], ib_s[KBT];
  const int tid = threadIdx.y * 16 + threadIdx.x;
  if (tid < KBT) {
    const int i = i0 + tid;
    ia_s[tid] = (i < P.na) ? (P.ia ? P.ia[i] : P.a0 + i) : -1;
  } else if (tid < 2 * KBT) {
    const int j = j0 + tid - KBT;
    ib_s[tid - KBT] = (j < P.nb) ? (P.ib ? P.ib[j] : P.b0 + j) : -1;
  }
  const int ty = threadIdx.y, tx = threadIdx.x;
  double d2[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) d2[a][b] = 0.0;
  for (int f0 = 0; f0 < r; f0 += KBF) {
    const int nf = min(KBF, r - f0);
    __syncthreads();
    for (int e = tid; e < KBT * nf; e += 256) {
      const int q = e / nf, f = e % nf;
      As[q * KBS + f] = ia_s[q] >= 0 ? F[ia_s[q] * rp + f0 + f] : 0.0;
      Bs[q * KBS + f] = ib_s[q] >= 0 ? F[ib_s[q] * rp + f0 + f] : 0.0;
    }
    __syncthreads();
    for (int f = 0; f < nf; ++f) {
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[(ty + 16 * a) * KBS + f];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = Bs[(tx + 16 * b) * KBS + f];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const double d = av[a] - bv[b];
          d2[a][b] = fma(d, d, d2[a][b]);
        }
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int il = ty + 16 * a, i = i0 + il;
    if (i >= P.na) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int jl = tx + 16 * b, j = j0 + jl;
      if (j >= P.nb) continue;
      double v = exp(-d2[a][b] / two_h2);
      if (ia_s[il] == ib_s[jl]) v = 1.0 + P.diag_add;
      P.out[(long long)i * P.ld + j] = v;
    }
  }
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
    lib_malloc((void**)&d, chunk.size() * sizeof(KblkProb), s);
    CUDA_CHECK(cudaMemcpyAsync(d, chunk.data(), chunk.size() * sizeof(KblkProb), cudaMemcpyHostToDevice, s));
    dim3 grid(ceil_div(mc, KBT), ceil_div(mr, KBT), (unsigned)chunk.size());
    kblock_kernel<<<grid, dim3(16, 16), 0, s>>>(F, rp, r, two_h2, d);
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
  if (P.accumulate == 2) {  // transpose through 32 x 33 shared tiles (coalesced both ways)
    __shared__ double tile[32][33];
    const int tr = (P.rows + 31) / 32, tc = (P.cols + 31) / 32;
    for (int t = blockIdx.x; t < tr * tc; t += gridDim.x) {
      const int i0 = (t / tc) * 32, j0 = (t % tc) * 32;
      for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
        const int ii = e / 32, jj = e % 32;
        if (i0 + ii < P.rows && j0 + jj < P.cols) tile[ii][jj] = P.src[(int64_t)(i0 + ii) * P.srs + j0 + jj];
      }
      __syncthreads();
      for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
        const int jj = e / 32, ii = e % 32;
        if (i0 + ii < P.rows && j0 + jj < P.cols) P.dst[(int64_t)(j0 + jj) * P.drs + i0 + ii] = tile[ii][jj];
      }
      __syncthreads();
    }
    return;
  }
  const int64_t tot = (int64_t)P.rows * P.cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / P.cols, j = e % P.cols;
    if (P.accumulate == 3) {
      P.dst[i * P.drs + j] = (j <= i) ? P.src[i * P.srs + j] : P.src[j * P.srs + i];
      continue;
    }
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
    lib_malloc((void**)&d, chunk.size() * sizeof(CopyProb), s);
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
