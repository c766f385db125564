// hss.cu — randomized ID-based HSS compression on the GPU (readings H1-H5; P:180-187,
// Alg. 3 line 1 at P:208) and the HSS mat-vec (reading M).
//
// Data layout (all device, fp64, level-major; nodes of a level in BFS order):
//   Fp (n x rp), nu (n)           permuted, zero-padded features and squared norms
//   Y_l, Omega^_l  (sum rows x s) per-node sketch rows, row-packed: node t at roff_t
//   J_l (sum k)                   skeleton tree positions, k-packed: node t at koff_t
//   U_l (sum rows*k)              interpolation bases P[I; T^T], row-major rows x k
//   B_l (parents at level l)      k_left x k_right kernel blocks at skeleton points
//   D   (leaves)                  m_t x m_t diagonal blocks
// Because children are consecutive in BFS order, the k-packed outputs of level l are exactly
// the row-packed inputs of level l-1 (rows of a parent = [J_left; J_right]), so no copies
// are needed to assemble a parent's Y, Omega^ and active rows.
#include "internal.cuh"

namespace svmhss {

__global__ void iperm_kernel(const int64_t* __restrict__ perm, int64_t n, int64_t* __restrict__ ip) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) ip[perm[i]] = i;
}
__global__ void iota_kernel64(int64_t* a, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}

struct SelNode { int64_t roff, koff, uoff; int rows, k, pt, pad; };

// U scatter: U[piv[c]][j] = (c < k) ? delta_cj : T[j][c-k]  (T stored in W[(roff+c)*s + j])
__global__ void scatter_u_kernel(const SelNode* __restrict__ nd, const int* __restrict__ piv,
                                 const double* __restrict__ W, int s, double* __restrict__ U) {
  const SelNode N = nd[blockIdx.x];
  if (N.pt) return;
  const int64_t tot = (int64_t)N.rows * N.k;
  for (int64_t e = threadIdx.x; e < tot; e += blockDim.x) {
    const int c = (int)(e / N.k), j = (int)(e % N.k);
    const int prow = piv[N.roff + c];
    const double v = (c < N.k) ? (c == j ? 1.0 : 0.0) : W[(N.roff + c) * s + j];
    U[N.uoff + (int64_t)prow * N.k + j] = v;
  }
}

// skeleton selection: J, Y_sk (and Omega' for pass-through nodes)
__global__ void select_kernel(const SelNode* __restrict__ nd, const int* __restrict__ piv,
                              const int64_t* __restrict__ act, const double* __restrict__ Y,
                              const double* __restrict__ Om, int s, int64_t* __restrict__ J,
                              double* __restrict__ Ysk, double* __restrict__ Omp) {
  const SelNode N = nd[blockIdx.x];
  const int64_t tot = (int64_t)N.k * s;
  for (int64_t e = threadIdx.x; e < tot; e += blockDim.x) {
    const int j = (int)(e / s), c = (int)(e % s);
    const int sel = N.pt ? j : piv[N.roff + j];
    Ysk[(N.koff + j) * s + c] = Y[(N.roff + sel) * s + c];
    if (N.pt) Omp[(N.koff + j) * s + c] = Om[(N.roff + j) * s + c];
    if (c == 0) J[N.koff + j] = act[N.roff + sel];
  }
}

void hss_build_impl(HSSImpl& H, const double* F, int64_t n, int r, double h, const hss_opts& o,
                    cudaStream_t s) {
  H.n = n;
  H.r = r;
  H.rp = (r + 3) / 4 * 4;
  H.h = h;
  H.m = o.leaf_size;
  H.s = o.max_rank + o.oversample;
  H.L = num_levels(n, H.m);
  const int rp = H.rp, S = H.s, L = H.L;
  std::vector<std::vector<std::pair<int64_t, int64_t>>> rg;
  node_ranges(n, L, rg);
  H.lv.assign(L + 1, {});
  for (int l = 0; l <= L; ++l) {
    H.lv[l].resize(rg[l].size());
    for (size_t i = 0; i < rg[l].size(); ++i) { H.lv[l][i].lo = rg[l][i].first; H.lv[l][i].hi = rg[l][i].second; }
  }
  H.st = hss_stats{};
  H.st.n = n; H.st.r = r; H.st.L = L; H.st.s = S; H.st.leaf_size = H.m;

  // ---- T1-T4: tree
  {
    EventTimer tm(s);
    DevBuf<double> Fpad((size_t)n * rp);
    pad_rows(F, n, r, rp, Fpad.p, s);
    H.perm.alloc(n);
    H.Fp.alloc((size_t)n * rp);
    build_tree(Fpad.p, n, r, rp, H.m, o.tree_seed, H.perm.p, H.Fp.p, s);
    H.nu.alloc(n + kNormPad);
    row_norms(H.Fp.p, n, rp, H.nu.p, s);
    H.iperm.alloc(n);
    iperm_kernel<<<ceil_div(n, 256), 256, 0, s>>>(H.perm.p, n, H.iperm.p);
    LAUNCH_CHECK();
    std::vector<int> lof(n);
    for (size_t i = 0; i < rg[L].size(); ++i)
      for (int64_t p = rg[L][i].first; p < rg[L][i].second; ++p) lof[p] = (int)i;
    lof.resize(n + kLeafPad, -3);
    H.leaf_of = upload(lof, s);
    H.st.ms_tree = tm.stop_ms();
  }
  // ---- leaves: D_t = K(I_t, I_t) (H2)
  {
    auto& lvL = H.lv[L];
    std::vector<KblkProb> kp;
    int64_t off = 0;
    for (auto& nd : lvL) {
      nd.doff = off;
      const int mloc = (int)(nd.hi - nd.lo);
      kp.push_back({mloc, mloc, nullptr, nd.lo, nullptr, nd.lo, nullptr, mloc, 0.0});
      off += (int64_t)mloc * mloc;
    }
    H.D.alloc(off);
    for (size_t i = 0; i < lvL.size(); ++i) kp[i].out = H.D.p + lvL[i].doff;
    kernel_blocks(H.Fp.p, rp, r, h, kp, s);
  }
  H.U.clear(); H.J.clear(); H.B.clear();
  H.U.resize(L + 1); H.J.resize(L + 1); H.B.resize(L + 1);
  if (L == 0) {
    H.lv[0][0].rows = (int)n;
    H.st.generator_bytes = (int64_t)H.D.bytes();
    CUDA_CHECK(cudaStreamSynchronize(s));
    return;
  }
  // ---- R1-R3: Omega_p, H1: masked sketch (diagonal leaf blocks excluded -> Y_leaf directly)
  DevBuf<double> Om((size_t)n * S), Y((size_t)n * S);
  {
    EventTimer tm(s);
    omega_rows(o.omega_seed, H.perm.p, n, S, Om.p, s);
    H.st.ms_omega = tm.stop_ms();
  }
  {
    EventTimer tm(s);
    KmmArgs a{};
    a.Fa = H.Fp.p; a.nua = H.nu.p; a.na = n;
    a.Fb = H.Fp.p; a.nub = H.nu.p; a.nb = n;
    a.rp = rp; a.W = Om.p; a.ldw = S; a.ncols = S; a.S = Y.p; a.lds = S;
    a.neg_inv_2h2 = -1.0 / (2.0 * h * h);
    a.same_set = 1;
    a.leaf_a = H.leaf_of.p; a.leaf_b = H.leaf_of.p;
    kernel_matmul(a, s);
    H.st.ms_sketch = tm.stop_ms();
  }
  EventTimer tmc(s);
  DevBuf<int64_t> act0(n);
  iota_kernel64<<<ceil_div(n, 256), 256, 0, s>>>(act0.p, n);
  LAUNCH_CHECK();
  const int64_t* act = act0.p;
  DevBuf<double> Ycur = std::move(Y), Omcur = std::move(Om);
  const int nnodes_all = (1 << (L + 1)) - 1;
  int cap_hits = 0, maxk = 0, npt = 0;
  for (int l = L; l >= 1; --l) {
    auto& lv = H.lv[l];
    const int nn = (int)lv.size();
    int64_t sumR = 0;
    for (int i = 0; i < nn; ++i) {
      auto& nd = lv[i];
      if (l == L) nd.rows = (int)(nd.hi - nd.lo);
      else nd.rows = H.lv[l + 1][2 * i].k + H.lv[l + 1][2 * i + 1].k;
      nd.roff = sumR;
      sumR += nd.rows;
    }
    // ranks: fixed (known) or adaptive (CPQR decides)
    std::vector<int> kfix(nn, -1);
    if (o.ranks) {
      for (int i = 0; i < nn; ++i) {
        const int t = H.node_id(l, i);
        (void)nnodes_all;
        kfix[i] = std::max(0, std::min(std::min(o.ranks[t], lv[i].rows), S));
      }
    }
    DevBuf<double> Wk((size_t)sumR * S);
    CUDA_CHECK(cudaMemcpyAsync(Wk.p, Ycur.p, (size_t)sumR * S * sizeof(double), cudaMemcpyDeviceToDevice, s));
    DevBuf<int> piv(std::max<int64_t>(1, sumR)), kd(nn), ch(nn);
    CUDA_CHECK(cudaMemsetAsync(ch.p, 0, nn * sizeof(int), s));
    std::vector<CpqrProb> cp;
    for (int i = 0; i < nn; ++i) {
      auto& nd = lv[i];
      if (kfix[i] >= 0 && kfix[i] == nd.rows) continue;  // known pass-through
      if (nd.rows == 0) continue;
      cp.push_back({nd.rows, S, Wk.p + nd.roff * S, piv.p + nd.roff, kfix[i], kd.p + i, ch.p + i});
    }
    bcpqr(cp, o.rel_tol, o.abs_tol, o.max_rank, s);
    std::vector<int> kh(nn, 0), chh(nn, 0);
    d2h(kh.data(), kd.p, nn, s);
    d2h(chh.data(), ch.p, nn, s);
    CUDA_CHECK(cudaStreamSynchronize(s));
    int64_t sumK = 0, sumU = 0;
    for (int i = 0; i < nn; ++i) {
      auto& nd = lv[i];
      if ((kfix[i] >= 0 && kfix[i] == nd.rows) || nd.rows == 0) nd.k = nd.rows;
      else nd.k = kh[i];
      nd.pt = (nd.k == nd.rows);
      nd.cap_hit = chh[i];
      cap_hits += chh[i];
      maxk = std::max(maxk, nd.k);
      npt += nd.pt ? 1 : 0;
      nd.koff = sumK;
      sumK += nd.k;
      nd.uoff = sumU;
      if (!nd.pt) sumU += (int64_t)nd.rows * nd.k;
    }
    // T = R11^-1 R12 (upper triangular solve, in place in Wk)
    std::vector<TrsmProb> tp;
    for (auto& nd : lv)
      if (!nd.pt && nd.k > 0 && nd.rows > nd.k)
        tp.push_back({nd.k, nd.rows - nd.k, Wk.p + nd.roff * S, 1, S, Wk.p + (nd.roff + nd.k) * S, 1, S});
    btrsm(tp, false, s);
    H.U[l].alloc(std::max<int64_t>(1, sumU));
    H.J[l].alloc(std::max<int64_t>(1, sumK));
    DevBuf<double> Ysk((size_t)std::max<int64_t>(1, sumK) * S), Omp((size_t)std::max<int64_t>(1, sumK) * S);
    std::vector<SelNode> sn(nn);
    for (int i = 0; i < nn; ++i) sn[i] = {lv[i].roff, lv[i].koff, lv[i].uoff, lv[i].rows, lv[i].k, lv[i].pt ? 1 : 0, 0};
    auto dsn = upload(sn, s);
    scatter_u_kernel<<<nn, 256, 0, s>>>(dsn.p, piv.p, Wk.p, S, H.U[l].p);
    LAUNCH_CHECK();
    select_kernel<<<nn, 256, 0, s>>>(dsn.p, piv.p, act, Ycur.p, Omcur.p, S, H.J[l].p, Ysk.p, Omp.p);
    LAUNCH_CHECK();
    // Omega'_t = U_t^T Omega^_t
    std::vector<GemmProb> gp;
    for (auto& nd : lv)
      if (!nd.pt && nd.k > 0)
        gp.push_back({nd.k, S, nd.rows, H.U[l].p + nd.uoff, 1, nd.k, Omcur.p + nd.roff * S, S, 1,
                      Omp.p + nd.koff * S, S, 1, 1.0, 0.0});
    bgemm(gp, s);
    // parents at level l-1: B = K(J_a, J_b); sibling update of Y_sk (H4)
    auto& pv = H.lv[l - 1];
    int64_t sumB = 0;
    for (size_t p = 0; p < pv.size(); ++p) {
      pv[p].boff = sumB;
      sumB += (int64_t)lv[2 * p].k * lv[2 * p + 1].k;
    }
    H.B[l - 1].alloc(std::max<int64_t>(1, sumB));
    std::vector<KblkProb> kb;
    for (size_t p = 0; p < pv.size(); ++p) {
      auto &a = lv[2 * p], &b = lv[2 * p + 1];
      kb.push_back({a.k, b.k, H.J[l].p + a.koff, 0, H.J[l].p + b.koff, 0, H.B[l - 1].p + pv[p].boff, b.k, 0.0});
    }
    kernel_blocks(H.Fp.p, rp, r, h, kb, s);
    if (l - 1 >= 1) {
      std::vector<GemmProb> up;
      for (size_t p = 0; p < pv.size(); ++p) {
        auto &a = lv[2 * p], &b = lv[2 * p + 1];
        const double* Bp = H.B[l - 1].p + pv[p].boff;
        if (a.k > 0 && b.k > 0) {
          up.push_back({a.k, S, b.k, Bp, b.k, 1, Omp.p + b.koff * S, S, 1, Ysk.p + a.koff * S, S, 1, -1.0, 1.0});
          up.push_back({b.k, S, a.k, Bp, 1, b.k, Omp.p + a.koff * S, S, 1, Ysk.p + b.koff * S, S, 1, -1.0, 1.0});
        }
      }
      bgemm(up, s);
    }
    CUDA_CHECK(cudaStreamSynchronize(s));  // host-side descriptors / Wk lifetime
    act = H.J[l].p;
    Ycur = std::move(Ysk);
    Omcur = std::move(Omp);
  }
  H.lv[0][0].rows = H.lv[1][0].k + H.lv[1][1].k;
  H.st.ms_compress = tmc.stop_ms();
  H.st.cap_hits = cap_hits;
  H.st.max_rank_used = maxk;
  H.st.passthrough = npt;
  int64_t gb = (int64_t)H.D.bytes();
  for (int l = 0; l <= L; ++l) {
    for (auto& nd : H.lv[l]) if (l >= 1 && !nd.pt) gb += 8LL * nd.rows * nd.k;
    if (l < L)
      for (size_t p = 0; p < H.lv[l].size(); ++p)
        gb += 8LL * H.lv[l + 1][2 * p].k * H.lv[l + 1][2 * p + 1].k;
  }
  H.st.generator_bytes = gb;
  CUDA_CHECK(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------------ mat-vec (M)
void hss_matvec_tree(const HSSImpl& H, const double* V, double* out, int nrhs, cudaStream_t s) {
  const int L = H.L;
  if (L == 0) {
    const int n = (int)H.n;
    bgemm({{n, nrhs, n, H.D.p, n, 1, V, nrhs, 1, out, nrhs, 1, 1.0, 0.0}}, s);
    return;
  }
  std::vector<DevBuf<double>> up(L + 1), dn(L + 1);
  for (int l = 1; l <= L; ++l) {
    int64_t sk = 0;
    for (auto& nd : H.lv[l]) sk += nd.k;
    up[l].alloc(std::max<int64_t>(1, sk) * nrhs);
    dn[l].alloc(std::max<int64_t>(1, sk) * nrhs);
  }
  // upward: up_t = U_t^T [V(I_t) | up_children]
  for (int l = L; l >= 1; --l) {
    const double* in = (l == L) ? V : up[l + 1].p;
    std::vector<GemmProb> gp;
    std::vector<CopyProb> cp;
    for (auto& nd : H.lv[l]) {
      const int64_t ro = (l == L) ? nd.lo : nd.roff;
      if (nd.pt) cp.push_back({nd.rows, nrhs, in + ro * nrhs, nrhs, up[l].p + nd.koff * nrhs, nrhs, 0});
      else if (nd.k > 0)
        gp.push_back({nd.k, nrhs, nd.rows, H.U[l].p + nd.uoff, 1, nd.k, in + ro * nrhs, nrhs, 1,
                      up[l].p + nd.koff * nrhs, nrhs, 1, 1.0, 0.0});
    }
    bcopy(cp, s);
    bgemm(gp, s);
  }
  // downward: children of t get U_t g_t (split) + sibling couplings B up_sibling
  for (int l = 0; l < L; ++l) {
    auto& pv = H.lv[l];
    auto& cv = H.lv[l + 1];
    std::vector<GemmProb> gp;
    std::vector<CopyProb> cp;
    for (size_t p = 0; p < pv.size(); ++p) {
      auto& nd = pv[p];
      auto &a = cv[2 * p], &b = cv[2 * p + 1];
      double* dst = dn[l + 1].p + a.koff * nrhs;  // a.koff .. b.koff + b.k contiguous
      const int rows = a.k + b.k;
      if (l == 0) {
        CUDA_CHECK(cudaMemsetAsync(dst, 0, (size_t)rows * nrhs * sizeof(double), s));
      } else if (nd.pt) {
        cp.push_back({rows, nrhs, dn[l].p + nd.koff * nrhs, nrhs, dst, nrhs, 0});
      } else if (nd.k > 0) {
        gp.push_back({rows, nrhs, nd.k, H.U[l].p + nd.uoff, nd.k, 1, dn[l].p + nd.koff * nrhs, nrhs, 1,
                      dst, nrhs, 1, 1.0, 0.0});
      } else {
        CUDA_CHECK(cudaMemsetAsync(dst, 0, (size_t)rows * nrhs * sizeof(double), s));
      }
    }
    bcopy(cp, s);
    bgemm(gp, s);
    std::vector<GemmProb> g2;
    for (size_t p = 0; p < pv.size(); ++p) {
      auto &a = cv[2 * p], &b = cv[2 * p + 1];
      const double* Bp = H.B[l].p + pv[p].boff;
      if (a.k > 0 && b.k > 0) {
        g2.push_back({a.k, nrhs, b.k, Bp, b.k, 1, up[l + 1].p + b.koff * nrhs, nrhs, 1,
                      dn[l + 1].p + a.koff * nrhs, nrhs, 1, 1.0, 1.0});
        g2.push_back({b.k, nrhs, a.k, Bp, 1, b.k, up[l + 1].p + a.koff * nrhs, nrhs, 1,
                      dn[l + 1].p + b.koff * nrhs, nrhs, 1, 1.0, 1.0});
      }
    }
    bgemm(g2, s);
  }
  // leaves: out = D V + U g
  std::vector<GemmProb> gp;
  std::vector<CopyProb> cp;
  for (auto& nd : H.lv[L]) {
    const int mloc = (int)(nd.hi - nd.lo);
    gp.push_back({mloc, nrhs, mloc, H.D.p + nd.doff, mloc, 1, V + nd.lo * nrhs, nrhs, 1,
                  out + nd.lo * nrhs, nrhs, 1, 1.0, 0.0});
  }
  bgemm(gp, s);
  gp.clear();
  for (auto& nd : H.lv[L]) {
    if (nd.pt) cp.push_back({nd.rows, nrhs, dn[L].p + nd.koff * nrhs, nrhs, out + nd.lo * nrhs, nrhs, 1});
    else if (nd.k > 0)
      gp.push_back({nd.rows, nrhs, nd.k, H.U[L].p + nd.uoff, nd.k, 1, dn[L].p + nd.koff * nrhs, nrhs, 1,
                    out + nd.lo * nrhs, nrhs, 1, 1.0, 1.0});
  }
  bcopy(cp, s);
  bgemm(gp, s);
  CUDA_CHECK(cudaStreamSynchronize(s));
}

}  // namespace svmhss
