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
  // work lists (fwd: 32-row chunks; bwd: 64-column chunks)
  for (int l = 0; l <= L; ++l) {
    auto& F_l = F.lv[l];
    std::vector<SolveNode> sn(F_l.nnodes);
    d2h(sn.data(), F_l.nodes.p, sn.size(), s);
    CUDA_CHECK(cudaStreamSynchronize(s));
    std::vector<SolveWork> fw, bw;
    for (int i = 0; i < F_l.nnodes; ++i) {
      for (int c = 0; c < ceil_div(sn[i].R, 32); ++c) fw.push_back({i, c});
      for (int c = 0; c < ceil_div(sn[i].R, 64); ++c) bw.push_back({i, c});
    }
    F_l.fwd_work = upload(fw, s);
    F_l.bwd_work = upload(bw, s);
    F_l.nfwd = (int)fw.size();
    F_l.nbwd = (int)bw.size();
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  F.st.beta = beta;
  F.st.factor_bytes = total_bytes;
  F.st.ms_factor = tm.stop_ms();
}

// ------------------------------------------------------------------ solve sweeps
template <int NR>
__global__ void __launch_bounds__(256) ulv_fwd_kernel(const SolveNode* __restrict__ nodes,
                                                      const SolveWork* __restrict__ work,
                                                      const double* __restrict__ M,
                                                      const double* __restrict__ fin,
                                                      double* __restrict__ fout,
                                                      double* __restrict__ yr) {
  const SolveWork wk = work[blockIdx.x];
  const SolveNode N = nodes[wk.node];
  const int R = N.R, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  extern __shared__ double bsh[];  // R * NR
  const double* b = fin + N.roff * NR;
  const int i0 = wk.chunk * 32;
  if (N.pt) {
    for (int e = tid; e < 32 * NR; e += 256) {
      const int i = i0 + e / NR;
      if (i < R) fout[(N.koff + i) * NR + e % NR] = b[(int64_t)i0 * NR + e];
    }
    return;
  }
  for (int e = tid; e < R * NR; e += 256) bsh[e] = b[e];
  __syncthreads();
  const int ib = i0 + wid * 4;
  double acc[4][NR];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int c = 0; c < NR; ++c) acc[q][c] = 0.0;
  const double* Mr = M + N.moff + (int64_t)ib * R;
  const int nq = min(4, R - ib);
  if (nq == 4) {
    for (int j = lane; j < R; j += 32) {
      const double m0 = Mr[j], m1 = Mr[R + j], m2 = Mr[2 * R + j], m3 = Mr[3 * R + j];
#pragma unroll
      for (int c = 0; c < NR; ++c) {
        const double bv = bsh[j * NR + c];
        acc[0][c] = fma(m0, bv, acc[0][c]);
        acc[1][c] = fma(m1, bv, acc[1][c]);
        acc[2][c] = fma(m2, bv, acc[2][c]);
        acc[3][c] = fma(m3, bv, acc[3][c]);
      }
    }
  } else {
    for (int q = 0; q < nq; ++q)
      for (int j = lane; j < R; j += 32) {
        const double m = Mr[(int64_t)q * R + j];
#pragma unroll
        for (int c = 0; c < NR; ++c) acc[q][c] = fma(m, bsh[j * NR + c], acc[q][c]);
      }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
#pragma unroll
    for (int c = 0; c < NR; ++c) acc[q][c] = warp_sum(acc[q][c]);
    const int i = ib + q;
    if (lane < NR && q < nq) {
      double v = acc[q][0];
#pragma unroll
      for (int c = 1; c < NR; ++c) if (lane == c) v = acc[q][c];
      if (i < N.k) fout[(N.koff + i) * NR + lane] = v;
      else yr[(N.yoff + i - N.k) * NR + lane] = v;
    }
  }
}

template <int NR>
__global__ void __launch_bounds__(256) ulv_bwd_kernel(const SolveNode* __restrict__ nodes,
                                                      const SolveWork* __restrict__ work,
                                                      const double* __restrict__ M,
                                                      const double* __restrict__ xin,
                                                      const double* __restrict__ yr,
                                                      double* __restrict__ xout) {
  const SolveWork wk = work[blockIdx.x];
  const SolveNode N = nodes[wk.node];
  const int R = N.R, tid = threadIdx.x, tx = tid & 63, ty = tid >> 6;
  extern __shared__ double u[];  // R * NR
  __shared__ double red[4][64][NR];
  const int j0 = wk.chunk * 64;
  if (N.pt) {
    for (int e = tid; e < 64 * NR; e += 256) {
      const int j = j0 + e / NR;
      if (j < R) xout[(N.roff + j) * NR + e % NR] = xin[(N.koff + j0) * NR + e];
    }
    return;
  }
  for (int e = tid; e < R * NR; e += 256) {
    const int i = e / NR;
    u[e] = (i < N.k) ? xin[N.koff * NR + e] : yr[(N.yoff - N.k) * NR + e];
  }
  __syncthreads();
  const int j = j0 + tx;
  double acc[NR];
#pragma unroll
  for (int c = 0; c < NR; ++c) acc[c] = 0.0;
  if (j < R) {
    const double* Mc = M + N.moff + j;
    int i = ty;
    for (; i + 12 < R; i += 16) {
      const double m0 = Mc[(int64_t)i * R], m1 = Mc[(int64_t)(i + 4) * R];
      const double m2 = Mc[(int64_t)(i + 8) * R], m3 = Mc[(int64_t)(i + 12) * R];
#pragma unroll
      for (int c = 0; c < NR; ++c) {
        acc[c] = fma(m0, u[i * NR + c], acc[c]);
        acc[c] = fma(m1, u[(i + 4) * NR + c], acc[c]);
        acc[c] = fma(m2, u[(i + 8) * NR + c], acc[c]);
        acc[c] = fma(m3, u[(i + 12) * NR + c], acc[c]);
      }
    }
    for (; i < R; i += 4) {
      const double m = Mc[(int64_t)i * R];
#pragma unroll
      for (int c = 0; c < NR; ++c) acc[c] = fma(m, u[i * NR + c], acc[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < NR; ++c) red[ty][tx][c] = acc[c];
  __syncthreads();
  if (ty == 0 && j < R) {
#pragma unroll
    for (int c = 0; c < NR; ++c) {
      const double v = ((red[0][tx][c] + red[1][tx][c]) + red[2][tx][c]) + red[3][tx][c];
      xout[(N.roff + j) * NR + c] = v;
    }
  }
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
  for (int l = L; l >= 0; --l) {
    const auto& lv = F.lv[l];
    if (lv.allpt) continue;
    const size_t sm = (size_t)lv.maxR * NR * sizeof(double);
    ulv_fwd_kernel<NR><<<lv.nfwd, 256, sm, s>>>(lv.nodes.p, lv.fwd_work.p, lv.M.p, ws.fin[l],
                                                l > 0 ? ws.fin[l - 1] : nullptr, ws.yr[l]);
  }
  for (int l = 0; l <= L; ++l) {
    const auto& lv = F.lv[l];
    if (lv.allpt) continue;
    const size_t sm = (size_t)lv.maxR * NR * sizeof(double);
    ulv_bwd_kernel<NR><<<lv.nbwd, 256, sm, s>>>(lv.nodes.p, lv.bwd_work.p, lv.M.p,
                                                l > 0 ? ws.xout[l - 1] : nullptr, ws.yr[l], ws.xout[l]);
  }
}

template <int NR>
static void set_smem_attrs(size_t sm) {
  CUDA_CHECK(cudaFuncSetAttribute(ulv_fwd_kernel<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  CUDA_CHECK(cudaFuncSetAttribute(ulv_bwd_kernel<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
}

void ulv_solve_tree(const ULVImpl& F, SolveWS& ws, cudaStream_t s) {
  int maxR = 0;
  for (auto& lv : F.lv) maxR = std::max(maxR, lv.maxR);
  const size_t sm = (size_t)maxR * ws.nrhs * sizeof(double);
  require(sm + 4 * 64 * ws.nrhs * 8 <= 227 * 1024, "ulv_solve: node too large for the shared-memory vector");
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
  for (auto& lv : F.lv) if (!lv.allpt) c += 2;
  return c;
}

}  // namespace svmhss
