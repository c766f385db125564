// ulv.cu — symmetric ULV factorization of K~ + beta I (readings U, AMB-14)
// and the ULV solve (readings S) as per-level batched GEMV sweeps.
//
// Factorization, per node t (bottom-up, all nodes of a level batched):
//   Dcur = D_t + beta I (leaf) | [[Dh_a, R_a B R_b^T], [., Dh_b]] (internal)
//   Ucur = U_t (leaf)          | diag(R_a, R_b) U_t (internal)
//   Householder QR  Q^T Ucur = [R; 0]   (compact WY: Q = I - V T V^T)
//   Dc = Q^T Dcur Q = M Dcur M^T with M = Q^T formed explicitly
//   L_r = chol(Dc_rr);  L_sr = Dc_sr L_r^-T;  Dh_t = Dc_ss - L_sr L_sr^T
// B200 design: instead of keeping (V, T, L_r, L_sr) and doing two
// triangular solves per node per sweep, we store the node's solve operator explicitly,
//   M_t = [[I, -L_sr L_r^-1], [0, L_r^-1]] Q^T = [ Q_s^T - L_sr G_r ; G_r ],  G_r = L_r^-1 Q_r^T
// (rows x rows), so the forward sweep is t = M_t b (up = t[:k], y_r = t[k:]) and the backward
// sweep is x = M_t^T [x_s; y_r]: one dense GEMV each way, streaming M_t from HBM once per
// sweep.  Root: M_0 = L^-1 of its Cholesky factor (k = 0).  Pass-through nodes: M = I.
#include "solve_dev.cuh"

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
// grid (row blocks of 8, problems): each CTA writes 8 rows of one problem (coalesced columns)
__global__ void pack_kernel(const double* __restrict__ A, const PackDesc* __restrict__ pd,
                            double* __restrict__ out) {
  const PackDesc P = pd[blockIdx.y];
  const int rows = (P.mode == 0) ? P.k : P.R, cols = (P.mode == 2) ? P.R : P.k;
  const int i0 = blockIdx.x * 8;
  if (i0 >= rows) return;
  for (int e = threadIdx.x; e < 8 * cols; e += blockDim.x) {
    const int i = i0 + e / cols, j = e % cols;
    if (i >= rows) break;
    const int64_t o = (int64_t)i * cols + j;
    double v;
    if (P.mode == 0) v = (j >= i) ? A[P.src + o] : 0.0;
    else if (P.mode == 1) v = (i > j) ? A[P.src + o] : (i == j ? 1.0 : 0.0);
    else v = (i == j) ? 1.0 : 0.0;
    out[P.dst + o] = v;
  }
}

static void run_pack(const double* A, const std::vector<PackDesc>& pd, double* out, cudaStream_t s) {
  if (pd.empty()) return;
  int maxrows = 1;
  for (auto& q : pd) maxrows = std::max(maxrows, q.mode == 0 ? q.k : q.R);
  auto d = upload(pd, s);
  for (size_t b0 = 0; b0 < pd.size(); b0 += 65535) {
    const unsigned nb = (unsigned)std::min<size_t>(65535, pd.size() - b0);
    pack_kernel<<<dim3((unsigned)ceil_div(maxrows, 8), nb), 256, 0, s>>>(A, d.p + b0, out);
    LAUNCH_CHECK();
  }
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
  const Shard& sh = H.sh;
  // per-node reduced blocks passed to the parent: Dh (k x k), Rm (k x k)
  DevBuf<double> DhC, RmC;           // child level
  std::vector<int64_t> dhoffC;       // offsets (doubles) by the child's BFS index (k*k packing)
  int64_t total_bytes = 0;
  // algorithmic flops (per non-pass-through node of R rows and rank k):
  // 2Rk^2 + 8R^2k + (R-k)^3/3 + k(R-k)^2 + k^2(R-k) + 4k^3; root: R^3/3
  double total_flops = 0.0;
  PhaseTrace ptr_("ulv_factor", s);
  for (int l = L; l >= 0; --l) {
    ptr_.mark("L" + std::to_string(l) + " begin");
    const bool leaf = (l == L);
    const int f0 = sh.first(l);
    // this rank's nodes of level l, re-based to 0 (hv[i] = H.lv[l][f0 + i])
    NodeInfo* hv = H.lv[l].data() + f0;
    const int nn = sh.last(l) - f0;
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
      const NodeInfo* cv = H.lv[l + 1].data() + 2 * f0;  // children of hv[i]: cv[2i], cv[2i+1]
      const int64_t* dho = dhoffC.data() + 2 * f0;
      std::vector<CopyProb> cp, tp;
      std::vector<GemmProb> g1, g2;
      int64_t sumT = 0;
      std::vector<int64_t> toff(nn);
      for (int i = 0; i < nn; ++i) { toff[i] = sumT; sumT += (int64_t)cv[2 * i].k * cv[2 * i + 1].k; }
      DevBuf<double> tmp(std::max<int64_t>(1, sumT));
      for (int i = 0; i < nn; ++i) {
        const int ka = cv[2 * i].k, kb = cv[2 * i + 1].k, Rn = R[i];
        double* Dc = Dcur.p + coff[i];
        const double* Dha = DhC.p + dho[2 * i];
        const double* Dhb = DhC.p + dho[2 * i + 1];
        const double* Ra = RmC.p + dho[2 * i];
        const double* Rb = RmC.p + dho[2 * i + 1];
        const double* Bp = H.B[l].p + hv[i].boff;
        cp.push_back({ka, ka, Dha, ka, Dc, Rn, 0});
        cp.push_back({kb, kb, Dhb, kb, Dc + (int64_t)ka * Rn + ka, Rn, 0});
        if (ka > 0 && kb > 0) {
          g1.push_back({ka, kb, ka, Ra, ka, 1, Bp, kb, 1, tmp.p + toff[i], kb, 1, 1.0, 0.0});
          // off = tmp R_b^T -> upper-right block; its transpose -> lower-left block (copy)
          g2.push_back({ka, kb, kb, tmp.p + toff[i], kb, 1, Rb, 1, kb, Dc + ka, Rn, 1, 1.0, 0.0});
          tp.push_back({ka, kb, Dc + ka, Rn, Dc + (int64_t)ka * Rn, Rn, 2});
        }
      }
      bcopy(cp, s);
      bgemm(g1, s);
      bgemm(g2, s);
      bcopy(tp, s);
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
      total_flops += (double)Rn * Rn * Rn / 3.0;
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
          const NodeInfo* cv = H.lv[l + 1].data() + 2 * f0;
          const int64_t* dho = dhoffC.data() + 2 * f0;
          const int ka = cv[2 * i].k, kb = cv[2 * i + 1].k;
          const double* Ra = RmC.p + dho[2 * i];
          const double* Rb = RmC.p + dho[2 * i + 1];
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
          const NodeInfo* cv = H.lv[l + 1].data() + 2 * f0;
          const int64_t* dho = dhoffC.data() + 2 * f0;
          const int ka = cv[2 * i].k, kb = cv[2 * i + 1].k;
          CUDA_CHECK(cudaMemsetAsync(RmP.p + koff2[i], 0, (size_t)K[i] * K[i] * 8, s));
          cp.push_back({ka, ka, RmC.p + dho[2 * i], ka, RmP.p + koff2[i], K[i], 0});
          cp.push_back({kb, kb, RmC.p + dho[2 * i + 1], kb, RmP.p + koff2[i] + (int64_t)ka * K[i] + ka, K[i], 0});
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
    for (int i = 0; i < nn; ++i) {
      if (PT[i]) continue;
      const double r = R[i], k = K[i], e = r - k;
      total_flops += 2 * r * k * k + 8 * r * r * k + e * e * e / 3 + k * e * e + k * k * e + 4 * k * k * k;
    }
    if (!np.empty() || !nz.empty()) {
      std::vector<int64_t> vo(nn), to(nn);
      int64_t sRK = 0, sKK = 0;
      for (int i : np) { vo[i] = sRK; sRK += (int64_t)R[i] * K[i]; to[i] = sKK; sKK += (int64_t)K[i] * K[i]; }
      DevBuf<double> tau(std::max<int64_t>(1, sumK)), V(std::max<int64_t>(1, sRK)), T(std::max<int64_t>(1, sKK)),
          Wt(std::max<int64_t>(1, sRK));
      std::vector<int64_t> tauoff(nn);
      { int64_t o = 0; for (int i = 0; i < nn; ++i) { tauoff[i] = o; o += K[i]; } }
      ptr_.mark("  assembled");
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
      ptr_.mark("  qr+pack");
      // T = larft(V^T V, tau)
      std::vector<GemmProb> g;
      for (int i : np) g.push_back({K[i], K[i], R[i], V.p + vo[i], 1, K[i], V.p + vo[i], K[i], 1, T.p + to[i], K[i], 1, 1.0, 0.0});
      bgemm(g, s);
      std::vector<SqProb> tp;
      std::vector<const double*> taus;
      for (int i : np) { tp.push_back({K[i], T.p + to[i], K[i], 1}); taus.push_back(tau.p + tauoff[i]); }
      blarft(tp, taus, l <= kLarftSolveMaxLevel, s);
      // Q^T D Q: M = Q^T = I - (V T^T) V^T is formed first (needed for the solve operator
      // anyway), then Y = D M^T and D' = M Y (two R x R x R GEMMs; 13% fewer flops than the
      // compact-WY form D - Z V^T - V Z^T and fewer, larger launches).
      {
        std::vector<PackDesc> pI0;
        for (int i : np) pI0.push_back({0, moff[i], R[i], K[i], 2, 0});
        run_pack(nullptr, pI0, F_l.M.p, s);
        g.clear();
        for (int i : np) g.push_back({R[i], K[i], K[i], V.p + vo[i], K[i], 1, T.p + to[i], 1, K[i], Wt.p + vo[i], K[i], 1, 1.0, 0.0});
        bgemm(g, s);  // Wt := V T^T
        g.clear();
        for (int i : np) g.push_back({R[i], R[i], K[i], Wt.p + vo[i], K[i], 1, V.p + vo[i], 1, K[i], F_l.M.p + moff[i], R[i], 1, -1.0, 1.0});
        bgemm(g, s);  // M = I - Wt V^T = Q^T
        int64_t sumR2np = 0;
        std::vector<int64_t> yo(nn, 0);
        for (int i : np) { yo[i] = sumR2np; sumR2np += (int64_t)R[i] * R[i]; }
        DevBuf<double> Yq(std::max<int64_t>(1, sumR2np));
        g.clear();
        for (int i : np) g.push_back({R[i], R[i], R[i], Dcur.p + coff[i], R[i], 1, F_l.M.p + moff[i], 1, R[i], Yq.p + yo[i], R[i], 1, 1.0, 0.0});
        bgemm(g, s);  // Y = D M^T
        g.clear();
        for (int i : np) g.push_back({R[i], R[i], R[i], F_l.M.p + moff[i], R[i], 1, Yq.p + yo[i], R[i], 1, Dcur.p + coff[i], R[i], 1, 1.0, 0.0, 1});
        bgemm(g, s);  // D' = M Y = Q^T D Q, symmetric: the lower-triangle tiles only (L_r, L_sr, D^ read it)
      }
      ptr_.mark("  wy QtDQ");
      // L_r = chol(Dc_rr)   (also nodes with k == 0: whole block)
      std::vector<SqProb> cp2;
      std::vector<int> ids;
      for (int i : np) { cp2.push_back({R[i] - K[i], Dcur.p + coff[i] + (int64_t)K[i] * R[i] + K[i], R[i], 1}); ids.push_back(H.node_id(l, f0 + i)); }
      for (int i : nz) { cp2.push_back({R[i], Dcur.p + coff[i], R[i], 1}); ids.push_back(H.node_id(l, f0 + i)); }
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
      std::vector<CopyProb> cpy;   // D^ starts from the symmetric Dc_ss (from its lower triangle)
      for (int i : np) cpy.push_back({K[i], K[i], Dcur.p + coff[i], R[i], DhP.p + koff2[i], K[i], 3});
      bcopy(cpy, s);
      g.clear();
      for (int i : np) {
        const double* Lt = Dcur.p + coff[i] + (int64_t)K[i] * R[i];  // (R-k) x k, ld R: L_sr^T
        g.push_back({K[i], K[i], R[i] - K[i], Lt, 1, R[i], Lt, R[i], 1, DhP.p + koff2[i], K[i], 1, -1.0, 1.0});
      }
      bgemm(g, s);
      ptr_.mark("  potrf/trsm/Dh");
      // G_r = L_r^-1 M[k:, :] ; M[:k, :] -= L_sr G_r   (k == 0 nodes: M = L^-1)
      std::vector<PackDesc> pI;
      for (int i : nz) pI.push_back({0, moff[i], R[i], K[i], 2, 0});
      run_pack(nullptr, pI, F_l.M.p, s);
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
    // solve descriptors (leaf rows: this rank's local point positions)
    std::vector<SolveNode> sn(nn);
    int maxR = 0, allpt = 1;
    for (int i = 0; i < nn; ++i) {
      sn[i] = {R[i], K[i], PT[i], 0, moff[i], leaf ? hv[i].lo - H.lo_g : hv[i].roff, hv[i].koff, yoff[i]};
      maxR = std::max(maxR, R[i]);
      if (!PT[i]) allpt = 0;
    }
    if (sh.on() && l == sh.lg) allpt = 0;  // the exchanged level always has its own buffers
    F_l.nodes = upload(sn, s);
    F_l.sumR = sumRall; F_l.sumK = level_sumk(H, l); F_l.sumY = sumY; F_l.maxR = maxR; F_l.allpt = allpt;
    // next level inputs (offsets by BFS index of this level)
    dhoffC.assign(H.lv[l].size(), -1);
    for (int i = 0; i < nn; ++i) dhoffC[f0 + i] = koff2[i];
    if (sh.on() && l == sh.lg) {
      // exchange the subtree roots' reduced blocks (Dh, Rm: k x k each) -> every rank
      const int km = H.kmax_lg;
      const int64_t slot = std::max<int64_t>(1, 2LL * km * km);
      DevBuf<double> send(slot), recv(slot * sh.P);
      const int ko = K[0];
      if (ko > 0) {
        CUDA_CHECK(cudaMemcpyAsync(send.p, DhP.p, (size_t)ko * ko * 8, cudaMemcpyDeviceToDevice, s));
        CUDA_CHECK(cudaMemcpyAsync(send.p + (int64_t)km * km, RmP.p, (size_t)ko * ko * 8, cudaMemcpyDeviceToDevice, s));
      }
      sh.comm->allgather(send.p, recv.p, slot * 8, s);
      int64_t tot = 0;
      for (int p = 0; p < sh.P; ++p) { dhoffC[p] = tot; tot += (int64_t)H.lv[l][p].k * H.lv[l][p].k; }
      DevBuf<double> Dall(std::max<int64_t>(1, tot)), Rall(std::max<int64_t>(1, tot));
      for (int p = 0; p < sh.P; ++p) {
        const int64_t kk = (int64_t)H.lv[l][p].k * H.lv[l][p].k;
        if (!kk) continue;
        CUDA_CHECK(cudaMemcpyAsync(Dall.p + dhoffC[p], recv.p + p * slot, kk * 8, cudaMemcpyDeviceToDevice, s));
        CUDA_CHECK(cudaMemcpyAsync(Rall.p + dhoffC[p], recv.p + p * slot + (int64_t)km * km, kk * 8,
                                   cudaMemcpyDeviceToDevice, s));
      }
      CUDA_CHECK(cudaStreamSynchronize(s));
      DhP = std::move(Dall);
      RmP = std::move(Rall);
    }
    DhC = std::move(DhP);
    RmC = std::move(RmP);
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  ptr_.mark("levels done");
  // work lists: forward = (node, chunk of `ch` rows), backward = (node, chunk of kCW columns)
  for (int l = 0; l <= L; ++l) {
    auto& F_l = F.lv[l];
    std::vector<SolveNode> sn(F_l.nnodes);
    d2h(sn.data(), F_l.nodes.p, sn.size(), s);
    CUDA_CHECK(cudaStreamSynchronize(s));
    // rows per CTA: enough CTAs to fill the chip (>= ~8 per SM)
    int64_t rows = 0;
    for (auto& nd : sn) if (!(l == L && nd.pt)) rows += nd.R;
    // rows per forward CTA, at most 64 (A/B with the mode-5 forward GEMV at config 3: 1.406 ms per
    // iteration vs 1.426 with 32 and 1.41-1.42 with 128; the per-row arithmetic does not depend on it)
    static const int chmax = [] { const char* e = getenv("SVMHSS_FWD_CH"); return e ? atoi(e) : 64; }();
    int ch = chmax;
    while (ch > 8 && rows / ch < 148 * 8) ch /= 2;
    F_l.ch = ch;
    std::vector<SolveWork> wk, bk;
    F_l.split = (l <= kSplitMaxLevel && l < L - 1) ? 1 : 0;
    for (int i = 0; i < F_l.nnodes; ++i) {
      if (l == L && sn[i].pt) continue;  // pass-through leaves: handled by leaf_pt_copy
      for (int c = 0; c < ceil_div(sn[i].R, ch); ++c) wk.push_back({i, c});
      const int nb = ceil_div(sn[i].R, kCW) * (F_l.split ? ceil_div(sn[i].R, kRB) : 1);
      for (int c = 0; c < nb; ++c) bk.push_back({i, c});
    }
    F_l.work = upload(wk, s);
    F_l.nwork = (int)wk.size();
    F_l.bwork = upload(bk, s);
    F_l.nbwork = (int)bk.size();
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  // pass-through leaves: local point position -> index in level L-1's vectors
  {
    std::vector<int64_t> pm(std::max<int64_t>(1, H.nloc()), -1);
    int npt = 0;
    if (L >= 1)
      for (int i = sh.first(L); i < sh.last(L); ++i) {
        const auto& nd = H.lv[L][i];
        if (nd.pt) {
          ++npt;
          for (int64_t p2 = nd.lo; p2 < nd.hi; ++p2) pm[p2 - H.lo_g] = nd.koff + (p2 - nd.lo);
        }
      }
    F.nleafpt = npt;
    F.ptmap = upload(pm, s);
    CUDA_CHECK(cudaStreamSynchronize(s));
  }
  F.st.beta = beta;
  F.st.factor_bytes = total_bytes;
  F.st.factor_flops = total_flops;
  F.st.ms_factor = tm.stop_ms();
}

// ------------------------------------------------------------------ solve sweeps
// (device functions fwd_rows / bwd_cols: solve_dev.cuh).  A forward work item = (node, chunk
// of `ch` rows) of t = M_t b; all threads of the CTA take part.
template <int NR>
__device__ __forceinline__ void fwd_item(const SolveNode* __restrict__ nodes, SolveWork wk, int ch,
                                         const double* __restrict__ M, const double* __restrict__ in,
                                         double* __restrict__ out_up, double* __restrict__ out_yr, double* vsh) {
  const SolveNode N = nodes[wk.node];
  const int R = N.R, tid = threadIdx.x;
  const int i0 = wk.chunk * ch, i1 = min(R, i0 + ch);
  if (N.pt) {  // identity operator
    pdl_wait();
    for (int e = tid; e < (i1 - i0) * NR; e += 256) out_up[(N.koff + i0) * NR + e] = in[(N.roff + i0) * NR + e];
  } else if (NR <= 2 && R <= 512 && i1 - i0 <= 8) {
    // one row per warp (small chunks: the top levels): the row's 16 loads (M is static) are issued
    // BEFORE the wait for the previous level (programmatic dependent launch), so they overlap its
    // tail; then the input vector is staged.  Same per-row FMA order as fwd_rows.
    const int lane = tid & 31, i = i0 + (tid >> 5);
    const double* Mr = M + N.moff + (int64_t)i * R;
    double m[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) m[q] = (i < i1 && lane + 32 * q < R) ? Mr[lane + 32 * q] : 0.0;
    pdl_wait();
    for (int e = tid; e < R * NR; e += 256) vsh[e] = in[N.roff * NR + e];
    __syncthreads();
    if (i < i1) {
      double acc[NR];
#pragma unroll
      for (int c = 0; c < NR; ++c) acc[c] = 0.0;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int j = lane + 32 * q;
        if (j < R) {
#pragma unroll
          for (int c = 0; c < NR; ++c) acc[c] = fma(m[q], vsh[j * NR + c], acc[c]);
        }
      }
      row_store<NR>(acc, i, N.k, N.koff, N.yoff, out_up, out_yr);
    }
  } else if (NR <= 2 && R <= 512) {
    // this warp's first row loaded before the wait for the previous level (as above), the rest
    // by fwd_rows; the per-row FMA order is fwd_rows' (j = lane, lane + 32, ...)
    const int lane = tid & 31, wid = tid >> 5, i = i0 + wid;
    const double* Mr = M + N.moff + (int64_t)i * R;
    double m[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) m[q] = (i < i1 && lane + 32 * q < R) ? Mr[lane + 32 * q] : 0.0;
    pdl_wait();
    for (int e = tid; e < R * NR; e += 256) vsh[e] = in[N.roff * NR + e];
    __syncthreads();
    if (i < i1) {
      double acc[NR];
#pragma unroll
      for (int c = 0; c < NR; ++c) acc[c] = 0.0;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int j = lane + 32 * q;
        if (j < R) {
#pragma unroll
          for (int c = 0; c < NR; ++c) acc[c] = fma(m[q], vsh[j * NR + c], acc[c]);
        }
      }
      row_store<NR>(acc, i, N.k, N.koff, N.yoff, out_up, out_yr);
    }
    fwd_rows<NR>(M + N.moff, R, vsh, i0 + 8, i1, wid, 8, N.k, N.koff, N.yoff, out_up, out_yr);
  } else {
    pdl_wait();
    for (int e = tid; e < R * NR; e += 256) vsh[e] = in[N.roff * NR + e];
    __syncthreads();
    fwd_rows<NR>(M + N.moff, R, vsh, i0, i1, tid >> 5, 8, N.k, N.koff, N.yoff, out_up, out_yr);
  }
  __syncthreads();
}

template <int NR>
__global__ void __launch_bounds__(256) ulv_fwd_kernel(const SolveNode* __restrict__ nodes,
                                                      const SolveWork* __restrict__ work, int ch,
                                                      const double* __restrict__ M,
                                                      const double* __restrict__ in,
                                                      double* __restrict__ out_up,
                                                      double* __restrict__ out_yr) {
  extern __shared__ double vsh[];  // R * NR
  pdl_trigger();
  fwd_item<NR>(nodes, work[blockIdx.x], ch, M, in, out_up, out_yr, vsh);  // waits (pdl_wait) inside
}

template <int NR>
__global__ void __launch_bounds__(kBW * 32) ulv_bwd_kernel(const SolveNode* __restrict__ nodes,
                                                           const SolveWork* __restrict__ work,
                                                           const double* __restrict__ M,
                                                           const double* __restrict__ in_s,
                                                           const double* __restrict__ in_r,
                                                           double* __restrict__ out) {
  pdl_trigger();
  const SolveWork wk = work[blockIdx.x];
  const SolveNode N = nodes[wk.node];
  const int R = N.R, tid = threadIdx.x;
  const int j0 = wk.chunk * kCW;
  if (N.pt) {  // identity operator
    pdl_wait();
    const int j1 = min(R, j0 + kCW);
    for (int e = tid; e < (j1 - j0) * NR; e += kBW * 32) out[(N.roff + j0) * NR + e] = in_s[(N.koff + j0) * NR + e];
    return;
  }
  extern __shared__ double sm[];  // u: R * NR, then red: kBW * kCW * NR
  double* ush = sm;
  double* red = sm + R * NR;
  // the first batch of M rows (static) before the wait for the previous level
  double pa[BWD_BQ], pb[BWD_BQ];
  bwd_cols_preload(M + N.moff, R, j0, pa, pb);
  pdl_wait();
  const int kn = N.k * NR;
  for (int e = tid; e < R * NR; e += kBW * 32) ush[e] = (e < kn) ? in_s[N.koff * NR + e] : in_r[(N.yoff - N.k) * NR + e];
  __syncthreads();
  bwd_cols<NR>(M + N.moff, R, ush, j0, red, out + N.roff * NR, -1, false, pa, pb);
}

// Backward sweep of a small level (few nodes: latency-bound): the rows are split too.  Work item
// = (node, column chunk cc, row chunk rc of kRB rows); each CTA sums its rows (warp w: rows
// i0 + w, i0 + w + kBW, ... in order; warps in order) into a partial slab, and the last CTA of
// (node, cc) adds the row-chunk partials in rc order.  Used for levels l <= kSplitMaxLevel
// (l < L-1), a rule of the global tree, so results stay P-invariant.
template <int NR>
__device__ __forceinline__ void bwd_split_item(const SolveNode* __restrict__ nodes, SolveWork wk, int item,
                                               const double* __restrict__ M, const double* __restrict__ in_s,
                                               const double* __restrict__ in_r, double* __restrict__ out,
                                               double* __restrict__ part, unsigned* __restrict__ cnt) {
  const SolveNode N = nodes[wk.node];
  const int R = N.R, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nrc = (R + kRB - 1) / kRB, cc = wk.chunk / nrc, rc = wk.chunk % nrc;
  const int j0 = cc * kCW, i0 = rc * kRB, i1 = min(R, i0 + kRB);
  if (N.pt) {  // identity operator (row chunk 0 copies)
    pdl_wait();
    if (rc == 0) {
      const int j1 = min(R, j0 + kCW);
      for (int e = tid; e < (j1 - j0) * NR; e += kBW * 32) out[(N.roff + j0) * NR + e] = in_s[(N.koff + j0) * NR + e];
    }
    __syncthreads();
    return;
  }
  __shared__ double ush[kRB * NR];
  __shared__ double red[kBW * kCW * NR];
  const int ja = j0 + lane, jb = j0 + 32 + lane;
  const bool va = ja < R, vb = jb < R;
  const double* Mn = M + N.moff;
  double aa[NR], ab[NR];
#pragma unroll
  for (int c = 0; c < NR; ++c) aa[c] = ab[c] = 0.0;
  {  // this warp's rows i0 + wid + q*kBW (q < kRB/kBW): all loads in flight, then FMAs in row order
    constexpr int NQ = kRB / kBW;
    double ma[NQ], mb[NQ];
    // M (static) first, BEFORE the wait for the previous level: its loads overlap that level's
    // tail, the input-vector load and the barrier below
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int i = i0 + wid + q * kBW;
      const double* Mr = Mn + (int64_t)i * R;
      ma[q] = (i < i1 && va) ? Mr[ja] : 0.0;
      mb[q] = (i < i1 && vb) ? Mr[jb] : 0.0;
    }
    pdl_wait();
    for (int e = tid; e < (i1 - i0) * NR; e += kBW * 32) {
      const int i = i0 + e / NR, c = e % NR;
      ush[e] = (i < N.k) ? in_s[(N.koff + i) * NR + c] : in_r[(N.yoff + i - N.k) * NR + c];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int i = i0 + wid + q * kBW;
      if (i < i1) {
#pragma unroll
        for (int c = 0; c < NR; ++c) {
          const double u = ush[(i - i0) * NR + c];
          aa[c] = fma(ma[q], u, aa[c]);
          ab[c] = fma(mb[q], u, ab[c]);
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < NR; ++c) {
    red[(wid * kCW + lane) * NR + c] = aa[c];
    red[(wid * kCW + 32 + lane) * NR + c] = ab[c];
  }
  __syncthreads();
  double* my = part + (int64_t)item * kCW * NR;
  for (int e = tid; e < kCW * NR; e += kBW * 32) {
    double t = red[e];
#pragma unroll
    for (int w = 1; w < kBW; ++w) t += red[w * kCW * NR + e];
    my[e] = t;
  }
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  const int g = item - rc;  // first work item of (node, cc)
  if (tid == 0) last = (atomicAdd(&cnt[g], 1u) == (unsigned)(nrc - 1));
  __syncthreads();
  if (last) {
    __threadfence();
    for (int e = tid; e < kCW * NR; e += kBW * 32) {
      const int jj = e / NR;
      if (j0 + jj >= R) continue;
      double t = 0.0;
      for (int q = 0; q < nrc; ++q) t += part[((int64_t)(g + q) * kCW) * NR + e];
      out[(N.roff + j0) * NR + e] = t;
    }
    if (tid == 0) cnt[g] = 0u;
  }
  __syncthreads();
}

template <int NR>
__global__ void __launch_bounds__(kBW * 32) ulv_bwd_split_kernel(const SolveNode* __restrict__ nodes,
                                                                 const SolveWork* __restrict__ work,
                                                                 const double* __restrict__ M,
                                                                 const double* __restrict__ in_s,
                                                                 const double* __restrict__ in_r,
                                                                 double* __restrict__ out,
                                                                 double* __restrict__ part,
                                                                 unsigned* __restrict__ cnt) {
  pdl_trigger();
  bwd_split_item<NR>(nodes, work[blockIdx.x], blockIdx.x, M, in_s, in_r, out, part, cnt);  // waits inside
}

// pass-through leaves: fwd  fin_{L-1}[map[p]] = fin_L[p];  bwd  xout_L[p] = xout_{L-1}[map[p]]
template <int NR>
__global__ void leaf_pt_copy_kernel(const int64_t* __restrict__ map, int64_t n, int bwd,
                                    const double* __restrict__ src, double* __restrict__ dst) {
  pdl_trigger();
  pdl_wait();
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
  ws.own.reserve(4 * (L + 1) + 2);
  ws.cnt_own.reserve(L + 1);
  ws.fin[L] = mk(H.nloc());
  if (H.sh.on()) exch_ws_alloc(H, nrhs, ws.nextra, ws.xw);
  for (int l = L; l >= 1; --l) ws.fin[l - 1] = F.lv[l].allpt ? ws.fin[l] : mk(F.lv[l].sumK);
  for (int l = 0; l <= L; ++l) if (!F.lv[l].allpt) ws.yr[l] = mk(F.lv[l].sumY);
  ws.xout[0] = mk(F.lv[0].sumR);
  for (int l = 1; l <= L; ++l) ws.xout[l] = F.lv[l].allpt ? ws.xout[l - 1] : mk(F.lv[l].sumR);
  ws.bpart.assign(L + 1, nullptr);
  ws.bcnt.assign(L + 1, nullptr);
  for (int l = 0; l <= L; ++l)
    if (F.lv[l].split && F.lv[l].nbwork > 0) {
      ws.bpart[l] = mk((int64_t)F.lv[l].nbwork * kCW);
      ws.cnt_own.emplace_back(F.lv[l].nbwork);
      CUDA_CHECK(cudaMemsetAsync(ws.cnt_own.back().p, 0, F.lv[l].nbwork * sizeof(unsigned), g_alloc_stream));
      ws.bcnt[l] = ws.cnt_own.back().p;
    }
}

template <int NR>
static void fwd_level(const ULVImpl& F, SolveWS& ws, int l, const SolveWork* work, int nwork, cudaStream_t s) {
  const auto& lv = F.lv[l];
  if (nwork <= 0) return;
  const size_t sm = (size_t)lv.maxR * NR * sizeof(double);
  launch_pdl(ulv_fwd_kernel<NR>, dim3(nwork), dim3(256), sm, s, lv.nodes.p, work, lv.ch, lv.M.p, ws.fin[l],
             l > 0 ? ws.fin[l - 1] : nullptr, ws.yr[l]);
  g_launches.fetch_add(1);
}

template <int NR>
static void bwd_level(const ULVImpl& F, SolveWS& ws, int l, const SolveWork* work, int nwork, cudaStream_t s) {
  const auto& lv = F.lv[l];
  if (nwork <= 0) return;
  if (lv.split) {
    launch_pdl(ulv_bwd_split_kernel<NR>, dim3(nwork), dim3(kBW * 32), 0, s, lv.nodes.p, work, lv.M.p,
               l > 0 ? ws.xout[l - 1] : nullptr, ws.yr[l], ws.xout[l], ws.bpart[l], ws.bcnt[l]);
    g_launches.fetch_add(1);
    return;
  }
  const size_t sm = ((size_t)lv.maxR + (size_t)kBW * kCW) * NR * sizeof(double);
  launch_pdl(ulv_bwd_kernel<NR>, dim3(nwork), dim3(kBW * 32), sm, s, lv.nodes.p, work, lv.M.p,
             l > 0 ? ws.xout[l - 1] : nullptr, ws.yr[l], ws.xout[l]);
  g_launches.fetch_add(1);
}

template <int NR>
static void exchange_step(const ULVImpl& F, SolveWS& ws, cudaStream_t s) {
  const HSSImpl& H = *F.H;
  // subtree roots' reduced right-hand sides (+ the caller's per-rank extra) -> every rank
  exchange_lg(H, ws.xw, ws.fin[H.sh.lg - 1], ws.extra, ws.extra_all, s);
  if (ws.extra && ws.extra_top) tree_reduce_top(H.sh.P, ws.extra_all, ws.nextra, ws.extra_top, s);
}

template <int NR>
static void run_step(const ULVImpl& F, SolveWS& ws, const SolveStep& st, cudaStream_t s) {
  const HSSImpl& H = *F.H;
  const int L = H.L;
  const int64_t n = H.nloc();
  switch (st.kind) {
    case SolveStep::FWD:  // levels a down to b (a >= b); the exchange after level lg unless told not to
      for (int l = st.a; l >= st.b; --l) {
        const auto& lv = F.lv[l];
        if (!lv.allpt) {
          if (l == L && F.nleafpt > 0 && !ws.fused_leaf_io) {
            launch_pdl(leaf_pt_copy_kernel<NR>, dim3(ceil_div(n * NR, 256)), dim3(256), 0, s, F.ptmap.p, n, 0,
                       ws.fin[L], ws.fin[L - 1]);
            g_launches.fetch_add(1);
          }
          fwd_level<NR>(F, ws, l, lv.work.p, lv.nwork, s);
        }
        if (H.sh.on() && l == H.sh.lg && !st.no_exchange) exchange_step<NR>(F, ws, s);
      }
      break;
    case SolveStep::BWD:  // levels a up to b (a <= b)
      for (int l = st.a; l <= st.b; ++l) {
        const auto& lv = F.lv[l];
        if (lv.allpt) continue;
        bwd_level<NR>(F, ws, l, lv.bwork.p, lv.nbwork, s);
        if (l == L && F.nleafpt > 0 && !ws.fused_leaf_io) {
          launch_pdl(leaf_pt_copy_kernel<NR>, dim3(ceil_div(n * NR, 256)), dim3(256), 0, s, F.ptmap.p, n, 1,
                     ws.xout[L - 1], ws.xout[L]);
          g_launches.fetch_add(1);
        }
      }
      break;
    case SolveStep::EXCHANGE: if (H.sh.on()) exchange_step<NR>(F, ws, s); break;
  }
}

template <int NR>
static void set_smem_attrs(size_t fwd, size_t bwd) {
  CUDA_CHECK(cudaFuncSetAttribute(ulv_fwd_kernel<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fwd));
  CUDA_CHECK(cudaFuncSetAttribute(ulv_bwd_kernel<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bwd));
}

void ulv_solve_steps(const ULVImpl& F, SolveWS& ws, const std::vector<SolveStep>& steps, cudaStream_t s) {
  int maxR = 0;
  for (auto& lv : F.lv) maxR = std::max(maxR, lv.maxR);
  const size_t smf = (size_t)maxR * ws.nrhs * sizeof(double);
  const size_t smb = ((size_t)maxR + (size_t)kBW * kCW) * ws.nrhs * sizeof(double);
  require(smb <= 227 * 1024, "ulv_solve: node too large for the shared-memory vector");
  switch (ws.nrhs) {
#define NRC(k)                                            \
  case k:                                                 \
    if (smb > 48 * 1024) set_smem_attrs<k>(smf, smb);     \
    for (const auto& st : steps) run_step<k>(F, ws, st, s); \
    break;
    NRC(1) NRC(2) NRC(3) NRC(4) NRC(5) NRC(6) NRC(7) NRC(8)
#undef NRC
    default: throw Error(HSS_EINVAL, "ulv_solve: nrhs must be 1..8");
  }
  CUDA_CHECK(cudaGetLastError());
}

void ulv_solve_tree(const ULVImpl& F, SolveWS& ws, cudaStream_t s) {
  const int L = F.H->L;
  ulv_solve_steps(F, ws, {SolveStep{SolveStep::FWD, L, 0}, SolveStep{SolveStep::BWD, 0, L}}, s);
}


}  // namespace svmhss
