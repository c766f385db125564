// ulv.cu — symmetric ULV factorization of K~ + beta I (readings U, AMB-14)
// and the ULV solve (readings S) as per-level batched GEMV sweeps.
//
// Factorization, per node t (bottom-up, all nodes of a level batched):
//   Dcur = D_t + beta I (leaf) | [[Dh_a, R_a B R_b^T], [., Dh_b]] (internal)
//   Ucur = U_t (leaf)          | diag(R_a, R_b) U_t (internal)
//   Householder QR  Q^T Ucur = [R; 0]   (compact WY: Q = I - V T V^T)
//   Dc = Q^T Dcur Q = Dcur - Z V^T - V Z^T,  Z = Dcur V T - 1/2 V T^T (V^T Dcur V) T
//   L_r = chol(Dc_rr);  L_sr = Dc_sr L_r^-T;  Dh_t = Dc_ss - L_sr L_sr^T
// B200 design: instead of keeping (V, T, L_r, L_sr) and doing two
// triangular solves per node per sweep, we store the node's solve operator explicitly,
//   M_t = [[I, -L_sr L_r^-1], [0, L_r^-1]] Q^T = [ Q_s^T - L_sr G_r ; G_r ],  G_r = L_r^-1 Q_r^T
// (rows x rows), so the forward sweep is t = M_t b (up = t[:k], y_r = t[k:]) and the backward
// sweep is x = M_t^T [x_s; y_r]: one dense GEMV each way, streaming M_t from HBM once per
// sweep.  Root: M_0 = L^-1 of its Cholesky factor (k = 0).  Pass-through nodes: M = I.
#include "internal.cuh"

namespace svmhss {

__global__ void leaf_dcur_kernel(const double* __restrict__ D, const int64_t* __restrict__ doff,
                                 const int64_t* __restrict__ coff, const int* __restrict__ R,
                                 double beta, double* __restrict__ Dcur) {
  const int nd = blockIdx.x;
  const int n = R[nd];
  const double* src = D + doff[nd];
  double* dst = Dcur + coff[nd];
  for (int64_t e = threadIdx.x; e < (int64_t)n * n; e += blockDim.x) {
    const int i = (int)(e / n), j = (int)(e % n);
    dst[e] = src[e] + (i == j ? beta : 0.0);
  }
}

struct PackDesc { int64_t src, dst; int R, k, mode, pad; };
// mode 0: extract R (k x k upper of A (R x k)) ; mode 1: extract V (unit lower trapezoidal R x k)
// mode 2: identity (R x R) ; mode 3: blockdiag(Ra, Rb) with Ra at src (ka = k) and Rb at dst2
__global__ void pack_kernel(const double* __restrict__ A, const PackDesc* __restrict__ pd,
                            double* __restrict__ out) {
  const PackDesc P = pd[blockIdx.x];
  if (P.mode == 0) {
    for (int64_t e = threadIdx.x; e < (int64_t)P.k * P.k; e += blockDim.x) {
      const int i = (int)(e / P.k), j = (int)(e % P.k);
      out[P.dst + e] = (j >= i) ? A[P.src + (int64_t)i * P.k + j] : 0.0;
    }
  } else if (P.mode == 1) {
    for (int64_t e = threadIdx.x; e < (int64_t)P.R * P.k; e += blockDim.x) {
      const int i = (int)(e / P.k), j = (int)(e % P.k);
      out[P.dst + e] = (i > j) ? A[P.src + e] : (i == j ? 1.0 : 0.0);
    }
  } else {
    for (int64_t e = threadIdx.x; e < (int64_t)P.R * P.R; e += blockDim.x) {
      const int i = (int)(e / P.R), j = (int)(e % P.R);
      out[P.dst + e] = (i == j) ? 1.0 : 0.0;
    }
  }
}

// batched square transpose: out[off + j*R + i] = A[off + i*R + j] (same offsets as A)
__global__ void btranspose_kernel(const SqProb* __restrict__ probs, const double* __restrict__ base,
                                  double* __restrict__ out) {
  const SqProb P = probs[blockIdx.z];
  const int n = P.n;
  const int64_t off = P.A - base;
  __shared__ double tile[32][33];
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  if (i0 >= n || j0 >= n) return;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int i = i0 + r, j = j0 + threadIdx.x;
    tile[r][threadIdx.x] = (i < n && j < n) ? P.A[(int64_t)i * n + j] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int j = j0 + r, i = i0 + threadIdx.x;
    if (i < n && j < n) out[off + (int64_t)j * n + i] = tile[threadIdx.x][r];
  }
}

void btranspose(const std::vector<SqProb>& probs, const double* base, double* out, cudaStream_t s) {
  if (probs.empty()) return;
  int mx = 0;
  for (auto& p : probs) mx = std::max(mx, p.n);
  auto d = upload(probs, s);
  dim3 grid(ceil_div(mx, 32), ceil_div(mx, 32), (unsigned)probs.size());
  btranspose_kernel<<<grid, dim3(32, 8), 0, s>>>(d.p, base, out);
  LAUNCH_CHECK();
  CUDA_CHECK(cudaStreamSynchronize(s));
}

static void run_pack(const double* A, const std::vector<PackDesc>& pd, double* out, cudaStream_t s) {
  if (pd.empty()) return;
  auto d = upload(pd, s);
  pack_kernel<<<(unsigned)pd.size(), 256, 0, s>>>(A, d.p, out);
  LAUNCH_CHECK();
  CUDA_CHECK(cudaStreamSynchronize(s));
}

static void check_info(const DevBuf<int>& info, const std::vector<int>& ids, cudaStream_t s) {
  if (ids.empty()) return;
  std::vector<int> h(ids.size());
  d2h(h.data(), info.p, ids.size(), s);
  CUDA_CHECK(cudaStreamSynchronize(s));
  for (size_t i = 0; i < ids.size(); ++i)
    if (h[i] != 0)
      throw Error(HSS_ENOTSPD, "K~ + beta I not SPD: Cholesky breakdown at node " +
                                   std::to_string(ids[i]) + " (pivot " + std::to_string(h[i] - 1) +
                                   "); increase beta (AMB-9)");
}

void ulv_factor_impl(ULVImpl& F, cudaStream_t s) {
  HSSImpl& H = *F.H;
  const int L = H.L;
  const double beta = F.beta;
  F.lv.clear();
  F.lv.resize(L + 1);
  EventTimer tm(s);
  // per-node reduced blocks passed to the parent: Dh (k x k), Rm (k x k)
  DevBuf<double> DhC, RmC;           // child level
  std::vector<int64_t> dhoffC;       // offsets (doubles), per child node (k*k packing)
  int64_t total_bytes = 0;
  for (int l = L; l >= 0; --l) {
    const bool leaf = (l == L);
    auto& hv = H.lv[l];
    const int nn = (int)hv.size();
    std::vector<int> R(nn), K(nn), PT(nn);
    for (int i = 0; i < nn; ++i) {
      R[i] = (l == 0) ? ((L == 0) ? (int)H.n : hv[i].rows) : hv[i].rows;
      K[i] = (l == 0) ? 0 : hv[i].k;
      PT[i] = (l == 0) ? 0 : (hv[i].pt ? 1 : 0);
    }
    // ---- assemble Dcur
    std::vector<int64_t> coff(nn);
    int64_t sumR2 = 0;
    for (int i = 0; i < nn; ++i) { coff[i] = sumR2; sumR2 += (int64_t)R[i] * R[i]; }
    DevBuf<double> Dcur(std::max<int64_t>(1, sumR2));
    if (leaf) {
      std::vector<int64_t> doff(nn);
      for (int i = 0; i < nn; ++i) doff[i] = hv[i].doff;
      auto d_doff = upload(doff, s), d_coff = upload(coff, s);
      auto d_R = upload(R, s);
      leaf_dcur_kernel<<<nn, 256, 0, s>>>(H.D.p, d_doff.p, d_coff.p, d_R.p, beta, Dcur.p);
      LAUNCH_CHECK();
      CUDA_CHECK(cudaStreamSynchronize(s));
    } else {
      auto& cv = H.lv[l + 1];
      std::vector<CopyProb> cp;
      std::vector<GemmProb> g1, g2;
      int64_t sumT = 0;
      std::vector<int64_t> toff(nn);
      for (int i = 0; i < nn; ++i) { toff[i] = sumT; sumT += (int64_t)cv[2 * i].k * cv[2 * i + 1].k; }
      DevBuf<double> tmp(std::max<int64_t>(1, sumT));
      for (int i = 0; i < nn; ++i) {
        const int ka = cv[2 * i].k, kb = cv[2 * i + 1].k, Rn = R[i];
        double* Dc = Dcur.p + coff[i];
        const double* Dha = DhC.p + dhoffC[2 * i];
        const double* Dhb = DhC.p + dhoffC[2 * i + 1];
        const double* Ra = RmC.p + dhoffC[2 * i];
        const double* Rb = RmC.p + dhoffC[2 * i + 1];
        const double* Bp = H.B[l].p + hv[i].boff;
        cp.push_back({ka, ka, Dha, ka, Dc, Rn, 0});
        cp.push_back({kb, kb, Dhb, kb, Dc + (int64_t)ka * Rn + ka, Rn, 0});
        if (ka > 0 && kb > 0) {
          g1.push_back({ka, kb, ka, Ra, ka, 1, Bp, kb, 1, tmp.p + toff[i], kb, 1, 1.0, 0.0});
          // off = tmp R_b^T -> upper-right block, and its transpose -> lower-left block
          g2.push_back({ka, kb, kb, tmp.p + toff[i], kb, 1, Rb, 1, kb, Dc + ka, Rn, 1, 1.0, 0.0});
          g2.push_back({ka, kb, kb, tmp.p + toff[i], kb, 1, Rb, 1, kb, Dc + (int64_t)ka * Rn, 1, Rn, 1.0, 0.0});
        }
      }
      bcopy(cp, s);
      bgemm(g1, s);
      bgemm(g2, s);
      CUDA_CHECK(cudaStreamSynchronize(s));
    }
    // ---- root: Cholesky + M_0 = L^-1
    auto& F_l = F.lv[l];
    F_l.nnodes = nn;
    if (l == 0) {
      const int Rn = R[0];
      DevBuf<int> info(1);
      bpotrf({{Rn, Dcur.p, Rn, 1}}, info.p, s);
      check_info(info, {0}, s);
      F_l.M.alloc((size_t)Rn * Rn);
      fill_identity(F_l.M.p, Rn, Rn, 1, s);
      btrsm({{Rn, Rn, Dcur.p, Rn, 1, F_l.M.p, Rn, 1}}, true, s);
      std::vector<SolveNode> sn = {{Rn, 0, 0, 0, 0, 0, 0, 0}};
      F_l.nodes = upload(sn, s);
      F_l.sumR = Rn; F_l.sumK = 0; F_l.sumY = Rn; F_l.maxR = Rn; F_l.allpt = 0;
      total_bytes += 8LL * Rn * Rn;
      CUDA_CHECK(cudaStreamSynchronize(s));
      break;
    }
    // ---- Ucur
    std::vector<int64_t> uoff(nn), koff2(nn);
    int64_t sumRK = 0, sumK = 0, sumK2 = 0;
    for (int i = 0; i < nn; ++i) {
      uoff[i] = sumRK;
      if (!PT[i]) sumRK += (int64_t)R[i] * K[i];
      koff2[i] = sumK2;
      sumK2 += (int64_t)K[i] * K[i];
      sumK += K[i];
    }
    DevBuf<double> Ucur(std::max<int64_t>(1, sumRK));
    {
      std::vector<CopyProb> cp;
      std::vector<GemmProb> gp;
      for (int i = 0; i < nn; ++i) {
        if (PT[i] || K[i] == 0) continue;
        const double* Ut = H.U[l].p + hv[i].uoff;
        if (leaf) {
          cp.push_back({R[i], K[i], Ut, K[i], Ucur.p + uoff[i], K[i], 0});
        } else {
          auto& cv = H.lv[l + 1];
          const int ka = cv[2 * i].k, kb = cv[2 * i + 1].k;
          const double* Ra = RmC.p + dhoffC[2 * i];
          const double* Rb = RmC.p + dhoffC[2 * i + 1];
          gp.push_back({ka, K[i], ka, Ra, ka, 1, Ut, K[i], 1, Ucur.p + uoff[i], K[i], 1, 1.0, 0.0});
          gp.push_back({kb, K[i], kb, Rb, kb, 1, Ut + (int64_t)ka * K[i], K[i], 1,
                        Ucur.p + uoff[i] + (int64_t)ka * K[i], K[i], 1, 1.0, 0.0});
        }
      }
      bcopy(cp, s);
      bgemm(gp, s);
    }
    // outputs of this level for the parent
    DevBuf<double> DhP(std::max<int64_t>(1, sumK2)), RmP(std::max<int64_t>(1, sumK2));
    // pass-through nodes: Dh = Dcur, Rm = I (leaf) or diag(R_a, R_b)
    {
      std::vector<CopyProb> cp;
      std::vector<PackDesc> pd;
      for (int i = 0; i < nn; ++i) {
        if (!PT[i]) continue;
        cp.push_back({R[i], R[i], Dcur.p + coff[i], R[i], DhP.p + koff2[i], K[i], 0});
        if (leaf) {
          pd.push_back({0, koff2[i], K[i], K[i], 2, 0});
        } else {
          auto& cv = H.lv[l + 1];
          const int ka = cv[2 * i].k, kb = cv[2 * i + 1].k;
          CUDA_CHECK(cudaMemsetAsync(RmP.p + koff2[i], 0, (size_t)K[i] * K[i] * 8, s));
          cp.push_back({ka, ka, RmC.p + dhoffC[2 * i], ka, RmP.p + koff2[i], K[i], 0});
          cp.push_back({kb, kb, RmC.p + dhoffC[2 * i + 1], kb, RmP.p + koff2[i] + (int64_t)ka * K[i] + ka, K[i], 0});
        }
      }
      bcopy(cp, s);
      run_pack(nullptr, pd, RmP.p, s);
    }
    // non-pass-through nodes
    std::vector<int> np;
    for (int i = 0; i < nn; ++i) if (!PT[i] && K[i] > 0 && R[i] > K[i]) np.push_back(i);
    // nodes with k == 0 (rank 0, not pass-through): everything eliminated, no coupling
    std::vector<int> nz;
    for (int i = 0; i < nn; ++i) if (!PT[i] && K[i] == 0) nz.push_back(i);
    // M storage
    std::vector<int64_t> moff(nn, 0), yoff(nn, 0);
    int64_t sumM = 0, sumY = 0, sumRall = 0;
    for (int i = 0; i < nn; ++i) {
      moff[i] = sumM;
      if (!PT[i]) sumM += (int64_t)R[i] * R[i];
      yoff[i] = sumY;
      sumY += R[i] - K[i];
      sumRall += R[i];
    }
    F_l.M.alloc(std::max<int64_t>(1, sumM));
    total_bytes += 8 * sumM;
    if (!np.empty() || !nz.empty()) {
      std::vector<int64_t> vo(nn), to(nn);
      int64_t sRK = 0, sKK = 0;
      for (int i : np) { vo[i] = sRK; sRK += (int64_t)R[i] * K[i]; to[i] = sKK; sKK += (int64_t)K[i] * K[i]; }
      DevBuf<double> tau(std::max<int64_t>(1, sumK)), V(std::max<int64_t>(1, sRK)), T(std::max<int64_t>(1, sKK)),
          Wt(std::max<int64_t>(1, sRK)), Z(std::max<int64_t>(1, sRK)), Mk(std::max<int64_t>(1, sKK)),
          X1(std::max<int64_t>(1, sKK)), X2(std::max<int64_t>(1, sKK));
      std::vector<int64_t> tauoff(nn);
      { int64_t o = 0; for (int i = 0; i < nn; ++i) { tauoff[i] = o; o += K[i]; } }
      // QR of Ucur
      std::vector<QrProb> qp;
      for (int i : np) qp.push_back({R[i], K[i], Ucur.p + uoff[i], K[i], 1, tau.p + tauoff[i]});
      bgeqr2(qp, s);
      std::vector<PackDesc> pR, pV;
      for (int i : np) {
        pR.push_back({uoff[i], koff2[i], R[i], K[i], 0, 0});
        pV.push_back({uoff[i], vo[i], R[i], K[i], 1, 0});
      }
      run_pack(Ucur.p, pR, RmP.p, s);
      run_pack(Ucur.p, pV, V.p, s);
      // T = larft(V^T V, tau)
      std::vector<GemmProb> g;
      for (int i : np) g.push_back({K[i], K[i], R[i], V.p + vo[i], 1, K[i], V.p + vo[i], K[i], 1, T.p + to[i], K[i], 1, 1.0, 0.0});
      bgemm(g, s);
      std::vector<SqProb> tp;
      std::vector<const double*> taus;
      for (int i : np) { tp.push_back({K[i], T.p + to[i], K[i], 1}); taus.push_back(tau.p + tauoff[i]); }
      blarft(tp, taus, s);
      // W = Dcur V ; Mk = V^T W ; X1 = Mk T ; X2 = T^T X1 ; Z = W T - 1/2 V X2
      g.clear();
      for (int i : np) g.push_back({R[i], K[i], R[i], Dcur.p + coff[i], R[i], 1, V.p + vo[i], K[i], 1, Wt.p + vo[i], K[i], 1, 1.0, 0.0});
      bgemm(g, s);
      g.clear();
      for (int i : np) g.push_back({K[i], K[i], R[i], V.p + vo[i], 1, K[i], Wt.p + vo[i], K[i], 1, Mk.p + to[i], K[i], 1, 1.0, 0.0});
      for (int i : np) g.push_back({R[i], K[i], K[i], Wt.p + vo[i], K[i], 1, T.p + to[i], K[i], 1, Z.p + vo[i], K[i], 1, 1.0, 0.0});
      bgemm(g, s);
      g.clear();
      for (int i : np) g.push_back({K[i], K[i], K[i], Mk.p + to[i], K[i], 1, T.p + to[i], K[i], 1, X1.p + to[i], K[i], 1, 1.0, 0.0});
      bgemm(g, s);
      g.clear();
      for (int i : np) g.push_back({K[i], K[i], K[i], T.p + to[i], 1, K[i], X1.p + to[i], K[i], 1, X2.p + to[i], K[i], 1, 1.0, 0.0});
      bgemm(g, s);
      g.clear();
      for (int i : np) g.push_back({R[i], K[i], K[i], V.p + vo[i], K[i], 1, X2.p + to[i], K[i], 1, Z.p + vo[i], K[i], 1, -0.5, 1.0});
      bgemm(g, s);
      // Dc = Dcur - Z V^T - V Z^T
      g.clear();
      for (int i : np) g.push_back({R[i], R[i], K[i], Z.p + vo[i], K[i], 1, V.p + vo[i], 1, K[i], Dcur.p + coff[i], R[i], 1, -1.0, 1.0});
      bgemm(g, s);
      g.clear();
      for (int i : np) g.push_back({R[i], R[i], K[i], V.p + vo[i], K[i], 1, Z.p + vo[i], 1, K[i], Dcur.p + coff[i], R[i], 1, -1.0, 1.0});
      bgemm(g, s);
      // L_r = chol(Dc_rr)   (also nodes with k == 0: whole block)
      std::vector<SqProb> cp2;
      std::vector<int> ids;
      for (int i : np) { cp2.push_back({R[i] - K[i], Dcur.p + coff[i] + (int64_t)K[i] * R[i] + K[i], R[i], 1}); ids.push_back(H.node_id(l, i)); }
      for (int i : nz) { cp2.push_back({R[i], Dcur.p + coff[i], R[i], 1}); ids.push_back(H.node_id(l, i)); }
      DevBuf<int> info(std::max<size_t>(1, cp2.size()));
      bpotrf(cp2, info.p, s);
      check_info(info, ids, s);
      // L_sr^T = L_r^-1 Dc_rs  (in place, rows k.., cols 0..k)
      std::vector<TrsmProb> tr;
      for (int i : np)
        tr.push_back({R[i] - K[i], K[i], Dcur.p + coff[i] + (int64_t)K[i] * R[i] + K[i], R[i], 1,
                      Dcur.p + coff[i] + (int64_t)K[i] * R[i], R[i], 1});
      btrsm(tr, true, s);
      // Dh = Dc_ss - L_sr L_sr^T
      std::vector<CopyProb> cpy;
      for (int i : np) cpy.push_back({K[i], K[i], Dcur.p + coff[i], R[i], DhP.p + koff2[i], K[i], 0});
      bcopy(cpy, s);
      g.clear();
      for (int i : np) {
        const double* Lt = Dcur.p + coff[i] + (int64_t)K[i] * R[i];  // (R-k) x k, ld R: L_sr^T
        g.push_back({K[i], K[i], R[i] - K[i], Lt, 1, R[i], Lt, R[i], 1, DhP.p + koff2[i], K[i], 1, -1.0, 1.0});
      }
      bgemm(g, s);
      // M = Q^T = I - V T^T V^T  ; G_r = L_r^-1 M[k:, :] ; M[:k, :] -= L_sr G_r
      std::vector<PackDesc> pI;
      for (int i : np) pI.push_back({0, moff[i], R[i], K[i], 2, 0});
      for (int i : nz) pI.push_back({0, moff[i], R[i], K[i], 2, 0});
      run_pack(nullptr, pI, F_l.M.p, s);
      g.clear();
      for (int i : np) g.push_back({R[i], K[i], K[i], V.p + vo[i], K[i], 1, T.p + to[i], 1, K[i], Wt.p + vo[i], K[i], 1, 1.0, 0.0});
      bgemm(g, s);  // Wt := V T^T (reuse)
      g.clear();
      for (int i : np) g.push_back({R[i], R[i], K[i], Wt.p + vo[i], K[i], 1, V.p + vo[i], 1, K[i], F_l.M.p + moff[i], R[i], 1, -1.0, 1.0});
      bgemm(g, s);
      tr.clear();
      for (int i : np)
        tr.push_back({R[i] - K[i], R[i], Dcur.p + coff[i] + (int64_t)K[i] * R[i] + K[i], R[i], 1,
                      F_l.M.p + moff[i] + (int64_t)K[i] * R[i], R[i], 1});
      for (int i : nz) tr.push_back({R[i], R[i], Dcur.p + coff[i], R[i], 1, F_l.M.p + moff[i], R[i], 1});
      btrsm(tr, true, s);
      g.clear();
      for (int i : np) {
        const double* Lt = Dcur.p + coff[i] + (int64_t)K[i] * R[i];
        g.push_back({K[i], R[i], R[i] - K[i], Lt, 1, R[i], F_l.M.p + moff[i] + (int64_t)K[i] * R[i], R[i], 1,
                     F_l.M.p + moff[i], R[i], 1, -1.0, 1.0});
      }
      bgemm(g, s);
      CUDA_CHECK(cudaStreamSynchronize(s));
    }
    // solve descriptors
    std::vector<SolveNode> sn(nn);
    std::vector<SolveWork> fw, bw;
    int maxR = 0, allpt = 1;
    for (int i = 0; i < nn; ++i) {
      sn[i] = {R[i], K[i], PT[i], 0, moff[i], leaf ? hv[i].lo : hv[i].roff, hv[i].koff, yoff[i]};
      maxR = std::max(maxR, R[i]);
      if (!PT[i]) allpt = 0;
    }
    F_l.nodes = upload(sn, s);
    F_l.sumR = sumRall; F_l.sumK = sumK; F_l.sumY = sumY; F_l.maxR = maxR; F_l.allpt = allpt;
    // next level inputs
    DhC = std::move(DhP);
    RmC = std::move(RmP);
    dhoffC = koff2;
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  // transposed copies M^T (backward sweep = row GEMV too) and work lists
  for (int l = 0; l <= L; ++l) {
    auto& F_l = F.lv[l];
    std::vector<SolveNode> sn(F_l.nnodes);
    d2h(sn.data(), F_l.nodes.p, sn.size(), s);
    CUDA_CHECK(cudaStreamSynchronize(s));
    F_l.MT.alloc(std::max<size_t>(1, F_l.M.n));
    std::vector<SqProb> tp;
    for (auto& nd : sn)
      if (!nd.pt) tp.push_back({nd.R, F_l.M.p + nd.moff, nd.R, 1});
    btranspose(tp, F_l.M.p, F_l.MT.p, s);
    // rows per CTA: enough CTAs to fill the chip (>= ~8 per SM), at most 32
    int64_t rows = 0;
    for (auto& nd : sn) if (!(l == L && nd.pt)) rows += nd.R;
    int ch = 32;
    while (ch > 8 && rows / ch < 148 * 8) ch /= 2;
    F_l.ch = ch;
    std::vector<SolveWork> wk;
    for (int i = 0; i < F_l.nnodes; ++i) {
      if (l == L && sn[i].pt) continue;  // pass-through leaves: handled by leaf_pt_copy
      for (int c = 0; c < ceil_div(sn[i].R, ch); ++c) wk.push_back({i, c});
    }
    F_l.work = upload(wk, s);
    F_l.nwork = (int)wk.size();
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  // pass-through leaves: tree position -> index in level L-1's vectors
  {
    std::vector<int64_t> pm(H.n, -1);
    int npt = 0;
    if (L >= 1)
      for (auto& nd : H.lv[L])
        if (nd.pt) {
          ++npt;
          for (int64_t p2 = nd.lo; p2 < nd.hi; ++p2) pm[p2] = nd.koff + (p2 - nd.lo);
        }
    F.nleafpt = npt;
    F.ptmap = upload(pm, s);
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  F.st.beta = beta;
  F.st.factor_bytes = total_bytes;
  F.st.ms_factor = tm.stop_ms();
}

// ------------------------------------------------------------------ solve sweeps
// One row-GEMV kernel serves both sweeps: forward t = M_t b (rows i < k -> parent's up,
// i >= k -> y_r), backward x = M_t^T [x_s; y_r] read from the stored transpose (rows j ->
// x).  A CTA handles `ch` consecutive rows of one node (ch chosen per level so small levels
// still spread over the chip); each warp streams its rows with 4 independent loads per lane
// in flight and reduces with shuffles (fixed order).
template <int NR>
__global__ void __launch_bounds__(256) ulv_gemv_kernel(const SolveNode* __restrict__ nodes,
                                                       const SolveWork* __restrict__ work, int ch,
                                                       const double* __restrict__ M, int bwd,
                                                       const double* __restrict__ in_a,
                                                       const double* __restrict__ in_b,
                                                       double* __restrict__ out_a,
                                                       double* __restrict__ out_b) {
  const SolveWork wk = work[blockIdx.x];
  const SolveNode N = nodes[wk.node];
  const int R = N.R, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  extern __shared__ double vsh[];  // R * NR
  const int i0 = wk.chunk * ch, i1 = min(R, i0 + ch);
  if (N.pt) {  // identity operator
    const int64_t src = bwd ? N.koff : N.roff, dst = bwd ? N.roff : N.koff;
    for (int e = tid; e < (i1 - i0) * NR; e += 256)
      out_a[(dst + i0) * NR + e] = in_a[(src + i0) * NR + e];
    return;
  }
  if (!bwd) {
    for (int e = tid; e < R * NR; e += 256) vsh[e] = in_a[N.roff * NR + e];
  } else {
    const int kn = N.k * NR;
    for (int e = tid; e < R * NR; e += 256)
      vsh[e] = (e < kn) ? in_a[N.koff * NR + e] : in_b[(N.yoff - N.k) * NR + e];
  }
  __syncthreads();
  for (int i = i0 + wid; i < i1; i += 8) {
    const double* Mr = M + N.moff + (int64_t)i * R;
    double acc[NR];
#pragma unroll
    for (int c = 0; c < NR; ++c) acc[c] = 0.0;
    int j = lane;
    for (; j + 96 < R; j += 128) {
      const double m0 = Mr[j], m1 = Mr[j + 32], m2 = Mr[j + 64], m3 = Mr[j + 96];
#pragma unroll
      for (int c = 0; c < NR; ++c) {
        acc[c] = fma(m0, vsh[j * NR + c], acc[c]);
        acc[c] = fma(m1, vsh[(j + 32) * NR + c], acc[c]);
        acc[c] = fma(m2, vsh[(j + 64) * NR + c], acc[c]);
        acc[c] = fma(m3, vsh[(j + 96) * NR + c], acc[c]);
      }
    }
    for (; j < R; j += 32) {
      const double m0 = Mr[j];
#pragma unroll
      for (int c = 0; c < NR; ++c) acc[c] = fma(m0, vsh[j * NR + c], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < NR; ++c) acc[c] = warp_sum(acc[c]);
    if (lane < NR) {
      double v = acc[0];
#pragma unroll
      for (int c = 1; c < NR; ++c) if (lane == c) v = acc[c];
      if (bwd) out_a[(N.roff + i) * NR + lane] = v;
      else if (i < N.k) out_a[(N.koff + i) * NR + lane] = v;
      else out_b[(N.yoff + i - N.k) * NR + lane] = v;
    }
  }
}

// pass-through leaves: fwd  fin_{L-1}[map[p]] = fin_L[p];  bwd  xout_L[p] = xout_{L-1}[map[p]]
template <int NR>
__global__ void leaf_pt_copy_kernel(const int64_t* __restrict__ map, int64_t n, int bwd,
                                    const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * NR) return;
  const int64_t p = e / NR;
  const int c = (int)(e % NR);
  const int64_t q = map[p];
  if (q < 0) return;
  if (bwd) dst[p * NR + c] = src[q * NR + c];
  else dst[q * NR + c] = src[p * NR + c];
}

void solve_ws_alloc(const ULVImpl& F, int nrhs, SolveWS& ws) {
  const HSSImpl& H = *F.H;
  const int L = H.L;
  ws.nrhs = nrhs;
  ws.own.clear();
  ws.fin.assign(L + 1, nullptr);
  ws.yr.assign(L + 1, nullptr);
  ws.xout.assign(L + 1, nullptr);
  auto mk = [&](int64_t rows) {
    ws.own.emplace_back(std::max<int64_t>(1, rows) * nrhs);
    return ws.own.back().p;
  };
  ws.own.reserve(3 * (L + 1) + 2);
  ws.fin[L] = mk(H.n);
  for (int l = L; l >= 1; --l) ws.fin[l - 1] = F.lv[l].allpt ? ws.fin[l] : mk(F.lv[l].sumK);
  for (int l = 0; l <= L; ++l) if (!F.lv[l].allpt) ws.yr[l] = mk(F.lv[l].sumY);
  ws.xout[0] = mk(F.lv[0].sumR);
  for (int l = 1; l <= L; ++l) ws.xout[l] = F.lv[l].allpt ? ws.xout[l - 1] : mk(F.lv[l].sumR);
}

template <int NR>
static void solve_impl(const ULVImpl& F, SolveWS& ws, cudaStream_t s) {
  const int L = F.H->L;
  const int64_t n = F.H->n;
  for (int l = L; l >= 0; --l) {
    const auto& lv = F.lv[l];
    if (lv.allpt) continue;
    if (l == L && F.nleafpt > 0) {
      leaf_pt_copy_kernel<NR><<<ceil_div(n * NR, 256), 256, 0, s>>>(F.ptmap.p, n, 0, ws.fin[L], ws.fin[L - 1]);
    }
    if (lv.nwork == 0) continue;
    const size_t sm = (size_t)lv.maxR * NR * sizeof(double);
    ulv_gemv_kernel<NR><<<lv.nwork, 256, sm, s>>>(lv.nodes.p, lv.work.p, lv.ch, lv.M.p, 0, ws.fin[l], nullptr,
                                                  l > 0 ? ws.fin[l - 1] : nullptr, ws.yr[l]);
  }
  for (int l = 0; l <= L; ++l) {
    const auto& lv = F.lv[l];
    if (lv.allpt) continue;
    if (lv.nwork > 0) {
      const size_t sm = (size_t)lv.maxR * NR * sizeof(double);
      ulv_gemv_kernel<NR><<<lv.nwork, 256, sm, s>>>(lv.nodes.p, lv.work.p, lv.ch, lv.MT.p, 1,
                                                    l > 0 ? ws.xout[l - 1] : nullptr, ws.yr[l], ws.xout[l], nullptr);
    }
    if (l == L && F.nleafpt > 0) {
      leaf_pt_copy_kernel<NR><<<ceil_div(n * NR, 256), 256, 0, s>>>(F.ptmap.p, n, 1, ws.xout[L - 1], ws.xout[L]);
    }
  }
}

template <int NR>
static void set_smem_attrs(size_t sm) {
  CUDA_CHECK(cudaFuncSetAttribute(ulv_gemv_kernel<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
}

void ulv_solve_tree(const ULVImpl& F, SolveWS& ws, cudaStream_t s) {
  int maxR = 0;
  for (auto& lv : F.lv) maxR = std::max(maxR, lv.maxR);
  const size_t sm = (size_t)maxR * ws.nrhs * sizeof(double);
  require(sm <= 227 * 1024, "ulv_solve: node too large for the shared-memory vector");
  switch (ws.nrhs) {
#define NRC(k) case k: if (sm > 48 * 1024) set_smem_attrs<k>(sm); solve_impl<k>(F, ws, s); break;
    NRC(1) NRC(2) NRC(3) NRC(4) NRC(5) NRC(6) NRC(7) NRC(8)
#undef NRC
    default: throw Error(HSS_EINVAL, "ulv_solve: nrhs must be 1..8");
  }
  LAUNCH_CHECK();
}

int ulv_solve_launches(const ULVImpl& F) {
  int c = 0;
  for (auto& lv : F.lv) if (!lv.allpt) c += (lv.nwork > 0) ? 2 : 0;
  if (F.nleafpt > 0 && !F.lv[F.H->L].allpt) c += 2;
  return c;
}

}  // namespace svmhss
