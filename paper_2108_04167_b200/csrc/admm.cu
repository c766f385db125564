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
#include "internal.cuh"

namespace svmhss {

constexpr int EPI_BLOCKS = 1024;

__global__ void __launch_bounds__(256) admm_epilogue_kernel(
    int64_t n, int nC, const double* __restrict__ y, const double* __restrict__ w, double w1,
    double beta, const double* __restrict__ Cv, const double* __restrict__ swq,
    const double* __restrict__ v, double* __restrict__ z, double* __restrict__ mu,
    double* __restrict__ bnext, double* __restrict__ part) {
  __shared__ double red[32];
  for (int c = 0; c < nC; ++c) {
    const double coef = swq[c] / w1, C = Cv[c];
    double pw = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t e = i * nC + c;
      const double yi = y[i], wi = w[i];
      const double x = yi * v[e] - coef * wi;
      const double m = mu[e];
      const double zn = fmin(fmax(x - m / beta, 0.0), C);
      const double mn = m - beta * (x - zn);
      z[e] = zn;
      mu[e] = mn;
      const double q = 1.0 + mn + beta * zn;
      bnext[e] = yi * q;
      pw = fma(wi, q, pw);
    }
    const double t = block_sum(pw, red);
    if (threadIdx.x == 0) part[(int64_t)blockIdx.x * nC + c] = t;
  }
}

// out[c] = sum_b part[b*nC + c]   (fixed order)
__global__ void reduce_partials_kernel(const double* __restrict__ part, int nb, int nC,
                                       double* __restrict__ out) {
  __shared__ double red[32];
  for (int c = 0; c < nC; ++c) {
    double a = 0.0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) a += part[(int64_t)b * nC + c];
    const double t = block_sum(a, red);
    if (threadIdx.x == 0) out[c] = t;
  }
}

// per-column fixed-order sums of f(i, c) for a few reductions used by precompute / bias
__global__ void colsum_kernel(int64_t n, int ncols, const double* __restrict__ A, int mode,
                              const double* __restrict__ B, double* __restrict__ out) {
  __shared__ double red[32];
  const int c = blockIdx.x;
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double x = A[i * ncols + c];
    a += (mode == 0) ? x : x * B[i * ncols + c];
  }
  const double t = block_sum(a, red);
  if (threadIdx.x == 0) out[c] = t;
}

__global__ void label_check_kernel(const double* __restrict__ y, int64_t n, int* bad) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && !(y[i] == 1.0 || y[i] == -1.0)) atomicAdd(bad, 1);
}

__global__ void fill_kernel(double* a, int64_t n, double v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}

__global__ void init_rhs_kernel(const double* __restrict__ y, int64_t n, int nC, double* __restrict__ b) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < n * nC) b[e] = y[e / nC];
}

__global__ void mul_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                           double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] * b[i];
}

// margin-set counts per c: cnt[2c] = #{eps < z < C-eps}, cnt[2c+1] = #{z > eps}
__global__ void margin_count_kernel(int64_t n, int nC, const double* __restrict__ z,
                                    const double* __restrict__ Cv, double eps_rel,
                                    double* __restrict__ cnt) {
  __shared__ double red[32];
  const int c = blockIdx.x;
  const double C = Cv[c], eps = eps_rel * C;
  double a = 0.0, b = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double zi = z[i * nC + c];
    a += (zi > eps && zi < C - eps) ? 1.0 : 0.0;
    b += (zi > eps) ? 1.0 : 0.0;
  }
  const double ta = block_sum(a, red);
  const double tb = block_sum(b, red);
  if (threadIdx.x == 0) { cnt[2 * c] = ta; cnt[2 * c + 1] = tb; }
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

// sums per c: s[4c+0] = sum_M y, s[4c+1] = z_y . (K~ e_M), s[4c+2] = z_y . (K~ z_y), s[4c+3] = sum z
__global__ void bias_sums_kernel(int64_t n, int nC, const double* __restrict__ V,
                                 const double* __restrict__ KV, const double* __restrict__ y,
                                 const double* __restrict__ z, double* __restrict__ out) {
  __shared__ double red[32];
  const int c = blockIdx.x;
  double a = 0, b = 0, d = 0, f = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double ind = V[i * 2 * nC + 2 * c], zy = V[i * 2 * nC + 2 * c + 1];
    a += ind * y[i];
    b += zy * KV[i * 2 * nC + 2 * c];
    d += zy * KV[i * 2 * nC + 2 * c + 1];
    f += z[i * nC + c];
  }
  a = block_sum(a, red); b = block_sum(b, red); d = block_sum(d, red); f = block_sum(f, red);
  if (threadIdx.x == 0) { out[4 * c] = a; out[4 * c + 1] = b; out[4 * c + 2] = d; out[4 * c + 3] = f; }
}

// y_orig: device labels (original order).  z_out / mu_out: device, original order, n x nC.
AdmmResult admm_train_impl(const ULVImpl& F, const double* y_orig, const std::vector<double>& Cs,
                           int max_it, const admm_opts* opt, double* z_out, double* mu_out,
                           double* bias_out, double* obj_out, cudaStream_t s) {
  const HSSImpl& H = *F.H;
  const int64_t n = H.n;
  const int nC = (int)Cs.size();
  const double beta = F.beta;
  AdmmResult R{};
  {
    DevBuf<int> bad(1);
    CUDA_CHECK(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
    label_check_kernel<<<ceil_div(n, 256), 256, 0, s>>>(y_orig, n, bad.p);
    LAUNCH_CHECK();
    int hb = 0;
    d2h(&hb, bad.p, 1, s);
    CUDA_CHECK(cudaStreamSynchronize(s));
    require(hb == 0, "admm_svm_train: labels must be exactly +1 or -1");
  }
  DevBuf<double> y(n), w(n), z((size_t)n * nC), mu((size_t)n * nC), dC(nC), swq(nC);
  gather_rows(y_orig, H.perm.p, n, 1, y.p, s);
  h2d(dC.p, Cs.data(), nC, s);
  // ---- precompute (A0): v = K_b^-1 e; w = Y v; w1 = e^T v
  EventTimer tpre(s);
  double w1 = 0.0;
  {
    SolveWS ws1;
    solve_ws_alloc(F, 1, ws1);
    fill_kernel<<<ceil_div(n, 256), 256, 0, s>>>(ws1.fin[H.L], n, 1.0);
    LAUNCH_CHECK();
    ulv_solve_tree(F, ws1, s);
    mul_kernel<<<ceil_div(n, 256), 256, 0, s>>>(y.p, ws1.xout[H.L], n, w.p);
    LAUNCH_CHECK();
    DevBuf<double> t(1);
    colsum_kernel<<<1, 256, 0, s>>>(n, 1, ws1.xout[H.L], 0, nullptr, t.p);
    LAUNCH_CHECK();
    d2h(&w1, t.p, 1, s);
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  R.ms_pre = tpre.stop_ms();
  R.w1 = w1;
  if (!(w1 > 0.0)) throw Error(HSS_EW1, "w1 = e^T (K~+beta I)^-1 e = " + std::to_string(w1) + " <= 0");
  // ---- state
  SolveWS ws;
  solve_ws_alloc(F, nC, ws);
  double* bvec = ws.fin[H.L];
  const double* xvec = ws.xout[H.L];
  CUDA_CHECK(cudaMemsetAsync(z.p, 0, (size_t)n * nC * 8, s));
  CUDA_CHECK(cudaMemsetAsync(mu.p, 0, (size_t)n * nC * 8, s));
  init_rhs_kernel<<<ceil_div(n * nC, 256), 256, 0, s>>>(y.p, n, nC, bvec);  // q0 = e
  LAUNCH_CHECK();
  {
    DevBuf<double> t(1);
    colsum_kernel<<<1, 256, 0, s>>>(n, 1, w.p, 0, nullptr, t.p);  // w^T e
    LAUNCH_CHECK();
    for (int c = 0; c < nC; ++c)
      CUDA_CHECK(cudaMemcpyAsync(swq.p + c, t.p, 8, cudaMemcpyDeviceToDevice, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  const int eb = (int)std::min<int64_t>(EPI_BLOCKS, std::max<int64_t>(1, (n + 255) / 256));
  DevBuf<double> part((size_t)eb * nC);
  auto iteration = [&](cudaStream_t st) {
    ulv_solve_tree(F, ws, st);
    admm_epilogue_kernel<<<eb, 256, 0, st>>>(n, nC, y.p, w.p, w1, beta, dC.p, swq.p, xvec,
                                             z.p, mu.p, bvec, part.p);
    reduce_partials_kernel<<<1, 256, 0, st>>>(part.p, eb, nC, swq.p);
  };
  R.launches = ulv_solve_launches(F) + 2;
  // capture one iteration as a CUDA graph
  cudaGraphExec_t gexec = nullptr;
  {
    cudaStream_t cs;
    CUDA_CHECK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t graph = nullptr;
    CUDA_CHECK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    iteration(cs);
    CUDA_CHECK(cudaStreamEndCapture(cs, &graph));
    CUDA_CHECK(cudaGraphInstantiate(&gexec, graph, 0));
    CUDA_CHECK(cudaGraphDestroy(graph));
    CUDA_CHECK(cudaStreamDestroy(cs));
    R.graph = 1;
  }
  const int te = (opt && opt->trace_every > 0) ? opt->trace_every : 0;
  EventTimer tloop(s);
  int tcount = 0;
  for (int it = 1; it <= max_it; ++it) {
    CUDA_CHECK(cudaGraphLaunch(gexec, s));
    if (te && (it % te == 0 || it == max_it)) {
      if (opt->trace_z) scatter_rows(z.p, H.perm.p, n, nC, opt->trace_z + (int64_t)tcount * n * nC, s);
      if (opt->trace_mu) scatter_rows(mu.p, H.perm.p, n, nC, opt->trace_mu + (int64_t)tcount * n * nC, s);
      ++tcount;
    }
  }
  R.ms_loop = tloop.stop_ms();
  // graph replays are not seen by LAUNCH_CHECK: account for them (capture counted one iteration)
  g_launches.fetch_add((long long)(max_it - 1) * R.launches);
  cudaGraphExecDestroy(gexec);
  scatter_rows(z.p, H.perm.p, n, nC, z_out, s);
  if (mu_out) scatter_rows(mu.p, H.perm.p, n, nC, mu_out, s);
  // ---- bias + objective (one HSS mat-vec with 2 nC columns)
  if (bias_out || obj_out) {
    EventTimer tb(s);
    const double eps_rel = (opt && opt->margin_eps_rel > 0) ? opt->margin_eps_rel : 1e-8;
    DevBuf<double> cnt(2 * nC);
    margin_count_kernel<<<nC, 256, 0, s>>>(n, nC, z.p, dC.p, eps_rel, cnt.p);
    LAUNCH_CHECK();
    std::vector<double> hc(2 * nC);
    d2h(hc.data(), cnt.p, 2 * nC, s);
    CUDA_CHECK(cudaStreamSynchronize(s));
    std::vector<int> mode(nC);
    std::vector<double> msize(nC);
    for (int c = 0; c < nC; ++c) {
      if (hc[2 * c] > 0) { mode[c] = 0; msize[c] = hc[2 * c]; }
      else if (hc[2 * c + 1] > 0) { mode[c] = 1; msize[c] = hc[2 * c + 1]; }
      else { mode[c] = 2; msize[c] = 0; }
    }
    auto dmode = upload(mode, s);
    DevBuf<double> V((size_t)n * 2 * nC), KV((size_t)n * 2 * nC), sums(4 * nC);
    bias_rhs_kernel<<<ceil_div(n * nC, 256), 256, 0, s>>>(n, nC, z.p, y.p, dC.p, dmode.p, eps_rel, V.p);
    LAUNCH_CHECK();
    hss_matvec_tree(H, V.p, KV.p, 2 * nC, s);
    bias_sums_kernel<<<nC, 256, 0, s>>>(n, nC, V.p, KV.p, y.p, z.p, sums.p);
    LAUNCH_CHECK();
    std::vector<double> hs(4 * nC);
    d2h(hs.data(), sums.p, 4 * nC, s);
    CUDA_CHECK(cudaStreamSynchronize(s));
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

__global__ void pad_coef_kernel(const double* __restrict__ coef, int64_t n, int nC, int ld,
                                double* __restrict__ out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * ld) return;
  const int64_t i = e / ld;
  const int c = (int)(e % ld);
  out[e] = (c < nC) ? coef[i * nC + c] : 0.0;
}

void predict_impl(const double* Ftrain, const double* coef, int64_t n, int r, double h,
                  const double* bias_host, int nC, const double* Ftest, int64_t m, double* dv,
                  int8_t* lab, cudaStream_t s) {
  const int rp = (r + 3) / 4 * 4;
  const int ld = 16;
  DevBuf<double> Ftr((size_t)n * rp), Fte((size_t)std::max<int64_t>(1, m) * rp), nutr(n + kNormPad),
      nute(std::max<int64_t>(1, m) + kNormPad), W((size_t)n * ld), S((size_t)std::max<int64_t>(1, m) * ld), b(nC);
  pad_rows(Ftrain, n, r, rp, Ftr.p, s);
  pad_rows(Ftest, m, r, rp, Fte.p, s);
  row_norms(Ftr.p, n, rp, nutr.p, s);
  row_norms(Fte.p, m, rp, nute.p, s);
  pad_coef_kernel<<<ceil_div(n * ld, 256), 256, 0, s>>>(coef, n, nC, ld, W.p);
  LAUNCH_CHECK();
  KmmArgs a{};
  a.Fa = Fte.p; a.nua = nute.p; a.na = m;
  a.Fb = Ftr.p; a.nub = nutr.p; a.nb = n;
  a.rp = rp; a.W = W.p; a.ldw = ld; a.ncols = ld; a.S = S.p; a.lds = ld;
  a.neg_inv_2h2 = -1.0 / (2.0 * h * h);
  a.same_set = 0; a.leaf_a = nullptr; a.leaf_b = nullptr;
  kernel_matmul(a, s);
  h2d(b.p, bias_host, nC, s);
  predict_finish_kernel<<<ceil_div(m * nC, 256), 256, 0, s>>>(S.p, m, nC, ld, b.p, dv, lab);
  LAUNCH_CHECK();
  CUDA_CHECK(cudaStreamSynchronize(s));
}

}  // namespace svmhss
