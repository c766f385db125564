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
#include <cstring>
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

// Pass-through certificate for a node whose rank could be all of its rows (adaptive rank rule,
// AMB-10): G = Y Y^T (rows x rows, Y = the node's sample block, rows x s).  The CPQR threshold is
// thr = max(rel_tol |R_11|, abs_tol sqrt(s)) with |R_11| = the largest column norm of Y^T =
// sqrt(max_i G_ii).  Every |R_jj| of a QR of Y^T is >= sigma_min(Y^T) (R triangular: |R_jj| are its
// eigenvalues), so if G - (1.01 thr)^2 I has a Cholesky factor, every |R_jj| > thr and the rank
// rule gives k = rows: the node is pass-through without running the CPQR (the 1% margin covers
// the rounding of G and of the CPQR's |R_jj|).  Nodes that fail the test take the CPQR as usual.
__global__ void cert_shift_kernel(double* __restrict__ G, const int64_t* __restrict__ goff,
                                  const int* __restrict__ rows, double rel_tol, double abs_tol, int s) {
  const int q = blockIdx.x;
  const int R = rows[q];
  double* g = G + goff[q];
  __shared__ double red[32];
  double m = 0.0;
  for (int i = threadIdx.x; i < R; i += blockDim.x) m = fmax(m, g[(int64_t)i * R + i]);
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) b = fmax(b, red[w]);
    red[0] = b;
  }
  __syncthreads();
  const double thr = fmax(rel_tol * sqrt(red[0]), abs_tol * sqrt((double)s));
  const double sh = (1.01 * thr) * (1.01 * thr);
  for (int i = threadIdx.x; i < R; i += blockDim.x) g[(int64_t)i * R + i] -= sh;
}

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
    if (Y) {
      Ysk[(N.koff + j) * s + c] = Y[(N.roff + sel) * s + c];
      if (N.pt) Omp[(N.koff + j) * s + c] = Om[(N.roff + j) * s + c];
    }
    if (c == 0) J[N.koff + j] = act[N.roff + sel];
  }
}

__global__ void iota_off_kernel64(int64_t* a, int64_t n, int64_t off) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = off + i;
}

// Build-time exchange record of one rank's subtree root (level lg), followed in the slot by
// J (S int64), Y_sk (S x S) and Omega' (S x S).
struct RootRec {
  int64_t k, rows, pt, cap_hit;
  int64_t sub_cap_hits, sub_pt, sub_maxk, sub_bytes;  // this rank's subtree (levels >= lg)
};

// N4 (SPD-preserving compression): for every non-pass-through node t of level l
// this rank holds, U_t = K(A_t, J_t) (K(J_t, J_t) + eps I)^-1 (rows x k, row-major), with the
// skeleton J_t already selected (select_kernel).  K(A_t, J_t) is written straight into U_t's
// storage; read as a k x rows matrix with unit row stride it is K(J_t, A_t) (K symmetric), so
// two triangular solves with the Cholesky factor L of G = K(J_t, J_t) + eps I (L then L^T, a
// stride swap) turn it into G^-1 K(J_t, A_t) = U_t^T in place, i.e. U_t row-major.
static void spd_interp_level(HSSImpl& H, int l, const int64_t* act, double eps, cudaStream_t s) {
  auto& lv = H.lv[l];
  const int f = H.sh.first(l), e = H.sh.last(l);
  std::vector<int> ids;
  std::vector<int64_t> goff;
  int64_t gtot = 0;
  for (int i = f; i < e; ++i) {
    const auto& nd = lv[i];
    if (nd.pt || nd.k == 0) continue;
    ids.push_back(i);
    goff.push_back(gtot);
    gtot += (int64_t)nd.k * nd.k;
  }
  if (ids.empty()) return;
  DevBuf<double> G(gtot);
  std::vector<KblkProb> kp;
  for (size_t q = 0; q < ids.size(); ++q) {
    const auto& nd = lv[ids[q]];
    const int64_t* J = H.J[l].p + nd.koff;
    kp.push_back({nd.rows, nd.k, act + nd.roff, 0, J, 0, H.U[l].p + nd.uoff, nd.k, 0.0});
    kp.push_back({nd.k, nd.k, J, 0, J, 0, G.p + goff[q], nd.k, eps});
  }
  kernel_blocks(H.Fp.p, H.rp, H.r, H.h, kp, s);
  std::vector<SqProb> pp;
  for (size_t q = 0; q < ids.size(); ++q) pp.push_back({lv[ids[q]].k, G.p + goff[q], lv[ids[q]].k, 1});
  DevBuf<int> info(ids.size());
  bpotrf(pp, info.p, s);
  std::vector<int> hi(ids.size());
  d2h(hi.data(), info.p, ids.size(), s);
  CUDA_CHECK(cudaStreamSynchronize(s));
  for (size_t q = 0; q < ids.size(); ++q)
    if (hi[q] != 0)
      throw Error(HSS_ENOTSPD, "hss_build (interp=spd): K(J,J) + spd_eps I not SPD at node " +
                                   std::to_string(H.node_id(l, ids[q])) + " (pivot " + std::to_string(hi[q] - 1) +
                                   "); raise spd_eps");
  std::vector<TrsmProb> lo, up;
  for (size_t q = 0; q < ids.size(); ++q) {
    const auto& nd = lv[ids[q]];
    double* X = H.U[l].p + nd.uoff;
    lo.push_back({nd.k, nd.rows, G.p + goff[q], nd.k, 1, X, 1, nd.k});
    up.push_back({nd.k, nd.rows, G.p + goff[q], 1, nd.k, X, 1, nd.k});
  }
  btrsm(lo, true, s);
  btrsm(up, false, s);
}

void hss_build_impl(HSSImpl& H, const double* F, int64_t n, int r, double h, const hss_opts& o,
                    std::shared_ptr<Comm> comm, cudaStream_t s, int s_cols) {
  H.n = n;
  H.r = r;
  H.rp = (r + 3) / 4 * 4;
  H.h = h;
  H.m = o.leaf_size;
  H.s = s_cols > 0 ? s_cols : o.max_rank + o.oversample;
  H.L = num_levels(n, H.m);
  const int rp = H.rp, S = H.s, L = H.L;
  // ---- shard plan: rank g owns node g of level lg = log2 P
  Shard& sh = H.sh;
  sh.comm = comm;
  sh.P = comm ? comm->size : 1;
  sh.g = comm ? comm->rank : 0;
  sh.lg = 0;
  while ((1 << sh.lg) < sh.P) ++sh.lg;
  require((1 << sh.lg) == sh.P, "hss_build: the number of ranks must be a power of two");
  require(sh.lg <= L, "hss_build: more ranks than leaves (need P <= 2^L, L = ceil(log2(n/leaf_size)))");
  const int lg = sh.lg;
  std::vector<std::vector<std::pair<int64_t, int64_t>>> rg;
  node_ranges(n, L, rg);
  H.lv.assign(L + 1, {});
  for (int l = 0; l <= L; ++l) {
    H.lv[l].resize(rg[l].size());
    for (size_t i = 0; i < rg[l].size(); ++i) { H.lv[l][i].lo = rg[l][i].first; H.lv[l][i].hi = rg[l][i].second; }
  }
  H.lo_g = rg[lg][sh.g].first;
  H.hi_g = rg[lg][sh.g].second;
  {
    std::vector<int64_t> lo(sh.P), cnt(sh.P);
    H.nmax_g = 0;
    for (int p = 0; p < sh.P; ++p) {
      lo[p] = rg[lg][p].first;
      cnt[p] = rg[lg][p].second - rg[lg][p].first;
      H.nmax_g = std::max(H.nmax_g, cnt[p]);
    }
    H.rank_lo = upload(lo, s);
    H.rank_cnt = upload(cnt, s);
  }
  const int64_t nl = H.nloc();
  H.st = hss_stats{};
  H.st.n = n; H.st.r = r; H.st.L = L; H.st.s = S; H.st.leaf_size = H.m;

  // ---- T1-T4: tree (every rank builds the whole tree: deterministic, identical)
  const bool ann = o.sampling == HSS_SAMPLING_ANN;
  DevBuf<double> Fpad((size_t)n * rp);
  {
    EventTimer tm(s);
    pad_rows(F, n, r, rp, Fpad.p, s);
    H.Fp.alloc((size_t)n * rp);
    if (o.perm) {  // imported tree (parity mode): the permutation only, ranges stay T1's split
      std::vector<int64_t> pv(o.perm, o.perm + n);
      std::vector<char> seen(n, 0);
      for (int64_t v : pv) {
        require(v >= 0 && v < n && !seen[v], "hss_build: opts.perm is not a permutation of 0..n-1");
        seen[v] = 1;
      }
      H.perm = upload(pv, s);
      gather_rows(Fpad.p, H.perm.p, n, rp, H.Fp.p, s);
      CUDA_CHECK(cudaStreamSynchronize(s));
    } else {
      H.perm.alloc(n);
      build_tree(Fpad.p, n, r, rp, H.m, o.tree_seed, H.perm.p, H.Fp.p, s);
    }
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
    // per-leaf local offsets of this rank's leaves (cluster-tree-ordered reductions)
    std::vector<int64_t> llo;
    for (int i = sh.first(L); i < sh.last(L); ++i) llo.push_back(rg[L][i].first - H.lo_g);
    llo.push_back(nl);
    H.leaf_lo = upload(llo, s);
    H.st.ms_tree = tm.stop_ms();
  }
  // ---- leaves this rank holds: D_t = K(I_t, I_t) (H2)
  {
    auto& lvL = H.lv[L];
    std::vector<KblkProb> kp;
    int64_t off = 0;
    for (int i = sh.first(L); i < sh.last(L); ++i) {
      auto& nd = lvL[i];
      nd.doff = off;
      const int mloc = (int)(nd.hi - nd.lo);
      kp.push_back({mloc, mloc, nullptr, nd.lo, nullptr, nd.lo, nullptr, mloc, 0.0});
      off += (int64_t)mloc * mloc;
    }
    H.D.alloc(off);
    for (size_t q = 0; q < kp.size(); ++q) kp[q].out = H.D.p + lvL[sh.first(L) + q].doff;
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
  // ---- R1-R3: Omega_p (all n rows: the sketch's right-hand matrix), H1: this rank's rows of
  // the masked sketch (diagonal leaf blocks excluded -> Y_leaf directly)
  DevBuf<double> Om(ann ? 0 : (size_t)n * S), Y(ann ? 0 : (size_t)std::max<int64_t>(1, nl) * S);
  // HSS-ANN (N1): neighbour lists of all points, re-indexed by tree position
  const int kap = ann ? o.ann_neighbors : 0;
  DevBuf<int64_t> ann_pos(ann ? (size_t)n * kap : 0);
  DevBuf<double> ann_dp(ann ? (size_t)n * kap : 0);
  if (ann) {
    EventTimer tm(s);
    DevBuf<int64_t> aidx((size_t)n * kap);
    DevBuf<double> ad((size_t)n * kap);
    ann_build(Fpad.p, n, r, rp, kap, o.ann_trees, o.ann_leaf, o.ann_seed, aidx.p, ad.p, s);
    ann_to_tree(H, kap, aidx.p, ad.p, ann_pos.p, ann_dp.p, s);
    CUDA_CHECK(cudaStreamSynchronize(s));
    H.st.ms_sketch = tm.stop_ms();
  } else {
    EventTimer tm(s);
    omega_rows(o.omega_seed, H.perm.p, n, S, Om.p, s);
    H.st.ms_omega = tm.stop_ms();
  }
  Fpad.release();
  if (!ann) {
    EventTimer tm(s);
    KmmArgs a{};
    a.Fa = H.Fp.p + H.lo_g * rp; a.nua = H.nu.p + H.lo_g; a.na = nl;
    a.Fb = H.Fp.p; a.nub = H.nu.p; a.nb = n;
    a.rp = rp; a.W = Om.p; a.ldw = S; a.ncols = S; a.S = Y.p; a.lds = S;
    a.neg_inv_2h2 = -1.0 / (2.0 * h * h);
    a.same_set = 1;
    a.diag_off = H.lo_g;
    a.leaf_a = H.leaf_of.p + H.lo_g; a.leaf_b = H.leaf_of.p;
    kernel_matmul(a, s);
    H.st.ms_sketch = tm.stop_ms();
  }
  // fixed-skeleton import (AMB-12 diagnostic): every node's rank from `ranks` (as kfix below),
  // its skeleton from the hss_info layout (levels 1..L, BFS order), its active rows = its points
  // (leaves) or its children's imported skeletons; the CPQR takes the local indices as pivots.
  std::vector<std::vector<int>> kall, rall;            // per level, per node (all nodes)
  std::vector<std::vector<int64_t>> soff;              // offset of node's skeleton in o.skeletons
  if (o.skeletons) {
    require(o.ranks != nullptr, "hss_build: opts.skeletons needs opts.ranks");
    require(!ann && o.adaptive_s0 <= 0, "hss_build: opts.skeletons needs sketch sampling, fixed s");
    kall.assign(L + 1, {}); rall.assign(L + 1, {}); soff.assign(L + 1, {});
    for (int l = L; l >= 1; --l) {
      const int cnt = (int)H.lv[l].size();
      kall[l].resize(cnt); rall[l].resize(cnt);
      for (int i = 0; i < cnt; ++i) {
        const int rows = (l == L) ? (int)(H.lv[l][i].hi - H.lv[l][i].lo) : kall[l + 1][2 * i] + kall[l + 1][2 * i + 1];
        rall[l][i] = rows;
        kall[l][i] = std::max(0, std::min(std::min(o.ranks[H.node_id(l, i)], rows), S));
      }
    }
    int64_t off = 0;
    for (int l = 1; l <= L; ++l) {
      soff[l].resize(H.lv[l].size());
      for (size_t i = 0; i < H.lv[l].size(); ++i) { soff[l][i] = off; off += kall[l][i]; }
    }
  }
  auto imported_forced = [&](int l, int i, std::vector<int>& out) {
    // local pivot indices of node (l, i): positions of its imported skeleton in its active rows
    std::vector<int64_t> act;
    if (l == L) {
      for (int64_t p = H.lv[l][i].lo; p < H.lv[l][i].hi; ++p) act.push_back(p);
    } else {
      for (int c = 2 * i; c <= 2 * i + 1; ++c)
        act.insert(act.end(), o.skeletons + soff[l + 1][c], o.skeletons + soff[l + 1][c] + kall[l + 1][c]);
    }
    std::vector<int> used(act.size(), 0);
    const int64_t* J = o.skeletons + soff[l][i];
    const bool pt = kall[l][i] == rall[l][i];
    out.clear();
    for (int q = 0; q < kall[l][i]; ++q) {
      int at = -1;
      for (size_t a = 0; a < act.size(); ++a)
        if (act[a] == J[q]) { at = (int)a; break; }
      require(at >= 0 && !used[at], "hss_build: imported skeleton of node " + std::to_string(H.node_id(l, i)) +
                                        " is not a set of distinct active rows");
      require(!pt || at == q, "hss_build: imported skeleton of pass-through node " +
                                  std::to_string(H.node_id(l, i)) + " must be its active rows in order");
      used[at] = 1;
      out.push_back(at);
    }
  };
  EventTimer tmc(s);
  DevBuf<int64_t> act0(std::max<int64_t>(1, nl));
  iota_off_kernel64<<<ceil_div(std::max<int64_t>(1, nl), 256), 256, 0, s>>>(act0.p, nl, H.lo_g);
  LAUNCH_CHECK();
  const int64_t* act = act0.p;
  DevBuf<double> Ycur = std::move(Y), Omhold;
  const double* omcur = ann ? nullptr : Om.p + H.lo_g * S;  // Omega^ of the leaves = this rank's rows
  int cap_hits = 0, maxk = 0, npt = 0;        // levels < lg (replicated) counted once
  int64_t sub_bytes = (int64_t)H.D.bytes(), top_bytes = 0;
  int sub_cap = 0, sub_pt = 0, sub_maxk = 0;  // this rank's subtree (levels >= lg)
  PhaseTrace ptr_("hss_compress", s);
  for (int l = L; l >= 1; --l) {
    ptr_.mark("L" + std::to_string(l) + " begin");
    auto& lv = H.lv[l];
    const int f = sh.first(l), e = sh.last(l), nn = e - f;
    int64_t sumR = 0;
    for (int i = f; i < e; ++i) {
      auto& nd = lv[i];
      if (l == L) nd.rows = (int)(nd.hi - nd.lo);
      else nd.rows = H.lv[l + 1][2 * i].k + H.lv[l + 1][2 * i + 1].k;
      nd.roff = sumR;
      sumR += nd.rows;
    }
    // ranks: fixed (known) or adaptive (CPQR decides)
    std::vector<int> kfix(nn, -1);
    if (o.ranks)
      for (int q = 0; q < nn; ++q)
        kfix[q] = std::max(0, std::min(std::min(o.ranks[H.node_id(l, f + q)], lv[f + q].rows), S));
    DevBuf<double> Wk((size_t)std::max<int64_t>(1, sumR) * S);
    if (ann) {  // N2-N3: Y_t = K(A_t, C_t) on the sampled columns
      DevBuf<int64_t> Cs((size_t)std::max(1, nn) * S);
      ann_sample_level(H, l, act, ann_pos.p, ann_dp.p, kap, o.ann_seed, Cs.p, s);
      ann_y_level(H, l, act, Cs.p, Wk.p, s);
    } else {
      CUDA_CHECK(cudaMemcpyAsync(Wk.p, Ycur.p, (size_t)sumR * S * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    DevBuf<int> piv(std::max<int64_t>(1, sumR)), kd(nn), ch(nn);
    CUDA_CHECK(cudaMemsetAsync(ch.p, 0, nn * sizeof(int), s));
    std::vector<int> fh;                       // imported pivots of this level's nodes
    std::vector<int64_t> foff(nn, -1);
    if (o.skeletons) {
      std::vector<int> one;
      for (int q = 0; q < nn; ++q) {
        imported_forced(l, f + q, one);
        require(kall[l][f + q] == std::max(0, kfix[q]) && rall[l][f + q] == lv[f + q].rows,
                "hss_build: imported skeletons inconsistent with the ranks");
        foff[q] = (int64_t)fh.size();
        fh.insert(fh.end(), one.begin(), one.end());
      }
    }
    auto dforced = upload(fh, s);
    // pass-through certificates (cert_shift_kernel): adaptive nodes whose rank could be all rows
    std::vector<char> cert(nn, 0);
    if (!o.ranks && !ann) {
      std::vector<int> cq, crow;
      std::vector<int64_t> goff;
      int64_t gtot = 0;
      for (int q = 0; q < nn; ++q) {
        const auto& nd = lv[f + q];
        if (nd.rows == 0 || nd.rows > std::min(o.max_rank, S) || nd.rows > 512) continue;
        cq.push_back(q); crow.push_back(nd.rows); goff.push_back(gtot);
        gtot += (int64_t)nd.rows * nd.rows;
      }
      if (!cq.empty()) {
        DevBuf<double> G(gtot);
        std::vector<GemmProb> gp;
        for (size_t u = 0; u < cq.size(); ++u) {
          const auto& nd = lv[f + cq[u]];
          const double* Y = Wk.p + nd.roff * S;
          gp.push_back({nd.rows, nd.rows, S, Y, S, 1, Y, 1, S, G.p + goff[u], nd.rows, 1, 1.0, 0.0});
        }
        bgemm(gp, s);
        auto dgo = upload(goff, s);
        auto drw = upload(crow, s);
        cert_shift_kernel<<<(unsigned)cq.size(), 256, 0, s>>>(G.p, dgo.p, drw.p, o.rel_tol, o.abs_tol, S);
        LAUNCH_CHECK();
        std::vector<SqProb> pp;
        for (size_t u = 0; u < cq.size(); ++u) pp.push_back({crow[u], G.p + goff[u], crow[u], 1});
        DevBuf<int> info(cq.size());
        bpotrf(pp, info.p, s);
        std::vector<int> hi(cq.size());
        d2h(hi.data(), info.p, cq.size(), s);
        CUDA_CHECK(cudaStreamSynchronize(s));
        for (size_t u = 0; u < cq.size(); ++u) cert[cq[u]] = (hi[u] == 0) ? 1 : 0;
      }
    }
    std::vector<CpqrProb> cp;
    for (int q = 0; q < nn; ++q) {
      auto& nd = lv[f + q];
      if (kfix[q] >= 0 && kfix[q] == nd.rows) continue;  // known pass-through
      if (cert[q]) continue;                             // certified pass-through
      if (nd.rows == 0) continue;
      cp.push_back({nd.rows, S, Wk.p + nd.roff * S, piv.p + nd.roff, kfix[q], kd.p + q, ch.p + q,
                    o.skeletons ? dforced.p + foff[q] : nullptr});
    }
    ptr_.mark("  Y ready");
    bcpqr(cp, o.rel_tol, o.abs_tol, o.max_rank, s);
    ptr_.mark("  cpqr");
    std::vector<int> kh(nn, 0), chh(nn, 0);
    d2h(kh.data(), kd.p, nn, s);
    d2h(chh.data(), ch.p, nn, s);
    CUDA_CHECK(cudaStreamSynchronize(s));
    int64_t sumK = 0, sumU = 0;
    for (int q = 0; q < nn; ++q) {
      auto& nd = lv[f + q];
      if ((kfix[q] >= 0 && kfix[q] == nd.rows) || nd.rows == 0 || cert[q]) { nd.k = nd.rows; chh[q] = 0; }
      else nd.k = kh[q];
      nd.pt = (nd.k == nd.rows);
      nd.cap_hit = chh[q];
      if (l >= lg) {
        sub_cap += chh[q]; sub_maxk = std::max(sub_maxk, nd.k); sub_pt += nd.pt ? 1 : 0;
        if (!nd.pt) sub_bytes += 8LL * nd.rows * nd.k;
      } else {
        cap_hits += chh[q]; maxk = std::max(maxk, nd.k); npt += nd.pt ? 1 : 0;
        if (!nd.pt) top_bytes += 8LL * nd.rows * nd.k;
      }
      nd.koff = sumK;
      sumK += nd.k;
      nd.uoff = sumU;
      if (!nd.pt) sumU += (int64_t)nd.rows * nd.k;
    }
    // T = R11^-1 R12 (upper triangular solve, in place in Wk)
    std::vector<TrsmProb> tp;
    for (int i = f; i < e; ++i) {
      auto& nd = lv[i];
      if (!nd.pt && nd.k > 0 && nd.rows > nd.k)
        tp.push_back({nd.k, nd.rows - nd.k, Wk.p + nd.roff * S, 1, S, Wk.p + (nd.roff + nd.k) * S, 1, S});
    }
    const bool spd = o.interp == HSS_INTERP_SPD;
    if (!spd) btrsm(tp, false, s);
    H.U[l].alloc(std::max<int64_t>(1, sumU));
    H.J[l].alloc(std::max<int64_t>(1, sumK));
    DevBuf<double> Ysk(ann ? 1 : (size_t)std::max<int64_t>(1, sumK) * S), Omp(ann ? 1 : (size_t)std::max<int64_t>(1, sumK) * S);
    std::vector<SelNode> sn(nn);
    for (int q = 0; q < nn; ++q) {
      auto& nd = lv[f + q];
      sn[q] = {nd.roff, nd.koff, nd.uoff, nd.rows, nd.k, nd.pt ? 1 : 0, 0};
    }
    auto dsn = upload(sn, s);
    if (!spd) {
      scatter_u_kernel<<<nn, 256, 0, s>>>(dsn.p, piv.p, Wk.p, S, H.U[l].p);
      LAUNCH_CHECK();
    }
    select_kernel<<<nn, 256, 0, s>>>(dsn.p, piv.p, act, ann ? nullptr : Ycur.p, omcur, S, H.J[l].p, Ysk.p, Omp.p);
    LAUNCH_CHECK();
    if (spd) spd_interp_level(H, l, act, o.spd_eps, s);
    // Omega'_t = U_t^T Omega^_t
    std::vector<GemmProb> gp;
    for (int i = f; i < e && !ann; ++i) {
      auto& nd = lv[i];
      if (!nd.pt && nd.k > 0)
        gp.push_back({nd.k, S, nd.rows, H.U[l].p + nd.uoff, 1, nd.k, omcur + nd.roff * S, S, 1,
                      Omp.p + nd.koff * S, S, 1, 1.0, 0.0});
    }
    bgemm(gp, s);
    if (l == lg && sh.on()) {
      // ---- exchange the subtree roots: k, J, Y_sk, Omega' of every rank's level-lg node
      const auto& own = lv[sh.g];
      const int64_t hdr = (sizeof(RootRec) + 7) / 8, slot = hdr + S + 2LL * S * S;
      DevBuf<double> send(slot), recv(slot * sh.P);
      RootRec rec{own.k, own.rows, own.pt ? 1 : 0, own.cap_hit, sub_cap, sub_pt, sub_maxk, sub_bytes};
      std::vector<double> hh(hdr, 0.0);
      std::memcpy(hh.data(), &rec, sizeof(rec));
      h2d(send.p, hh.data(), hdr, s);
      if (own.k > 0) CUDA_CHECK(cudaMemcpyAsync(send.p + hdr, H.J[l].p, own.k * 8, cudaMemcpyDeviceToDevice, s));
      if (own.k > 0 && !ann) {
        CUDA_CHECK(cudaMemcpyAsync(send.p + hdr + S, Ysk.p, (size_t)own.k * S * 8, cudaMemcpyDeviceToDevice, s));
        CUDA_CHECK(cudaMemcpyAsync(send.p + hdr + S + (int64_t)S * S, Omp.p, (size_t)own.k * S * 8,
                                   cudaMemcpyDeviceToDevice, s));
      }
      sh.comm->allgather(send.p, recv.p, slot * 8, s);
      std::vector<double> hr((size_t)sh.P * hdr);
      for (int p = 0; p < sh.P; ++p) d2h(hr.data() + (size_t)p * hdr, recv.p + p * slot, hdr, s);
      CUDA_CHECK(cudaStreamSynchronize(s));
      int64_t gK = 0;
      std::vector<int64_t> koffs(sh.P), ks(sh.P);
      sub_cap = sub_pt = sub_maxk = 0;
      int64_t all_sub_bytes = 0;
      for (int p = 0; p < sh.P; ++p) {
        RootRec rp_;
        std::memcpy(&rp_, hr.data() + (size_t)p * hdr, sizeof(rp_));
        auto& nd = lv[p];
        nd.k = (int)rp_.k; nd.rows = (int)rp_.rows; nd.pt = rp_.pt != 0; nd.cap_hit = (int)rp_.cap_hit;
        nd.koff = gK;
        koffs[p] = gK; ks[p] = nd.k;
        gK += nd.k;
        sub_cap += (int)rp_.sub_cap_hits; sub_pt += (int)rp_.sub_pt;
        sub_maxk = std::max<int>(sub_maxk, (int)rp_.sub_maxk);
        all_sub_bytes += rp_.sub_bytes;
        H.kmax_lg = std::max(H.kmax_lg, nd.k);
      }
      sub_bytes = all_sub_bytes;
      H.lg_koff = upload(koffs, s);
      H.lg_k = upload(ks, s);
      DevBuf<int64_t> Jall(std::max<int64_t>(1, gK));
      DevBuf<double> Yall(ann ? 1 : (size_t)std::max<int64_t>(1, gK) * S), Oall(ann ? 1 : (size_t)std::max<int64_t>(1, gK) * S);
      for (int p = 0; p < sh.P; ++p) {
        const int64_t k = ks[p];
        if (!k) continue;
        const double* src = recv.p + p * slot;
        CUDA_CHECK(cudaMemcpyAsync(Jall.p + koffs[p], src + hdr, k * 8, cudaMemcpyDeviceToDevice, s));
        if (ann) continue;
        CUDA_CHECK(cudaMemcpyAsync(Yall.p + koffs[p] * S, src + hdr + S, (size_t)k * S * 8, cudaMemcpyDeviceToDevice, s));
        CUDA_CHECK(cudaMemcpyAsync(Oall.p + koffs[p] * S, src + hdr + S + (int64_t)S * S, (size_t)k * S * 8,
                                   cudaMemcpyDeviceToDevice, s));
      }
      CUDA_CHECK(cudaStreamSynchronize(s));
      H.J[l] = std::move(Jall);
      Ysk = std::move(Yall);
      Omp = std::move(Oall);
    }
    // parents at level l-1: B = K(J_a, J_b); sibling update of Y_sk (H4)
    auto& pv = H.lv[l - 1];
    const int pf = sh.first(l - 1), pe = sh.last(l - 1);
    int64_t sumB = 0;
    for (int p = pf; p < pe; ++p) {
      pv[p].boff = sumB;
      const int64_t bb = (int64_t)lv[2 * p].k * lv[2 * p + 1].k;
      sumB += bb;
      if (l - 1 >= lg) sub_bytes += 8 * bb;
      else top_bytes += 8 * bb;
    }
    H.B[l - 1].alloc(std::max<int64_t>(1, sumB));
    std::vector<KblkProb> kb;
    for (int p = pf; p < pe; ++p) {
      auto &a = lv[2 * p], &b = lv[2 * p + 1];
      kb.push_back({a.k, b.k, H.J[l].p + a.koff, 0, H.J[l].p + b.koff, 0, H.B[l - 1].p + pv[p].boff, b.k, 0.0});
    }
    kernel_blocks(H.Fp.p, rp, r, h, kb, s);
    if (l - 1 >= 1 && !ann) {
      std::vector<GemmProb> up;
      for (int p = pf; p < pe; ++p) {
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
    Omhold = std::move(Omp);
    omcur = Omhold.p;
    if (l == L && !ann) Om.release();
  }
  H.lv[0][0].rows = H.lv[1][0].k + H.lv[1][1].k;
  H.st.ms_compress = tmc.stop_ms();
  H.st.cap_hits = cap_hits + sub_cap;
  H.st.max_rank_used = std::max(maxk, sub_maxk);
  H.st.passthrough = npt + sub_pt;
  H.st.generator_bytes = sub_bytes + top_bytes;
  CUDA_CHECK(cudaStreamSynchronize(s));
}

// N2b: does some node of this build have its rank at the sample budget (k > s - p) while
// min(cap, rows) allowed more?  Global over ranks (an allgather of one flag).
bool hss_unconverged(const HSSImpl& H, int p, int cap) {
  int bad = 0;
  for (int l = 1; l <= H.L && !bad; ++l)
    for (int i = H.sh.first(l); i < H.sh.last(l); ++i) {
      const auto& nd = H.lv[l][i];
      if (nd.k > H.s - p && nd.k < std::min(cap, nd.rows)) { bad = 1; break; }
    }
  if (H.sh.on()) {
    DevBuf<int> one(1), all(H.sh.P);
    CUDA_CHECK(cudaMemcpy(one.p, &bad, sizeof(int), cudaMemcpyHostToDevice));
    H.sh.comm->allgather(one.p, all.p, sizeof(int), g_alloc_stream);
    std::vector<int> h(H.sh.P);
    d2h(h.data(), all.p, H.sh.P, g_alloc_stream);
    CUDA_CHECK(cudaStreamSynchronize(g_alloc_stream));
    bad = 0;
    for (int v : h) bad |= v;
  }
  return bad != 0;
}

// ------------------------------------------------------------------ mat-vec (M)
// Sum of k over the nodes of level l this rank holds k-packed vectors for (all P nodes at the
// exchanged level lg when sharded).
int64_t level_sumk(const HSSImpl& H, int l) {
  int f = H.sh.first(l), e = H.sh.last(l);
  if (H.sh.on() && l == H.sh.lg) { f = 0; e = H.sh.P; }
  int64_t sk = 0;
  for (int i = f; i < e; ++i) sk += H.lv[l][i].k;
  return sk;
}

void hss_matvec_tree(const HSSImpl& H, const double* V, double* out, int nrhs, cudaStream_t s) {
  const int L = H.L;
  const Shard& sh = H.sh;
  if (L == 0) {
    const int n = (int)H.n;
    bgemv({{n, nrhs, n, H.D.p, n, 1, V, nrhs, 1, out, nrhs, 1, 1.0, 0.0}}, s);
    return;
  }
  std::vector<DevBuf<double>> up(L + 1), dn(L + 1);
  for (int l = 1; l <= L; ++l) {
    const int64_t sk = level_sumk(H, l);
    up[l].alloc(std::max<int64_t>(1, sk) * nrhs);
    dn[l].alloc(std::max<int64_t>(1, sk) * nrhs);
  }
  ExchWS xw;
  if (sh.on()) exch_ws_alloc(H, nrhs, 0, xw);
  // upward: up_t = U_t^T [V(I_t) | up_children]
  for (int l = L; l >= 1; --l) {
    const double* in = (l == L) ? V : up[l + 1].p;
    std::vector<GemmProb> gp;
    std::vector<CopyProb> cp;
    for (int i = sh.first(l); i < sh.last(l); ++i) {
      const auto& nd = H.lv[l][i];
      const int64_t ro = (l == L) ? nd.lo - H.lo_g : nd.roff;
      if (nd.pt) cp.push_back({nd.rows, nrhs, in + ro * nrhs, nrhs, up[l].p + nd.koff * nrhs, nrhs, 0});
      else if (nd.k > 0)
        gp.push_back({nd.k, nrhs, nd.rows, H.U[l].p + nd.uoff, 1, nd.k, in + ro * nrhs, nrhs, 1,
                      up[l].p + nd.koff * nrhs, nrhs, 1, 1.0, 0.0});
    }
    bcopy(cp, s);
    bgemv(gp, s);
    if (l == sh.lg && sh.on()) exchange_lg(H, xw, up[l].p, nullptr, nullptr, s);
  }
  // downward: children of t get U_t g_t (split) + sibling couplings B up_sibling
  for (int l = 0; l < L; ++l) {
    auto& pv = H.lv[l];
    auto& cv = H.lv[l + 1];
    std::vector<GemmProb> gp;
    std::vector<CopyProb> cp;
    for (int p = sh.first(l); p < sh.last(l); ++p) {
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
    bgemv(gp, s);
    std::vector<GemmProb> g2;
    for (int p = sh.first(l); p < sh.last(l); ++p) {
      auto &a = cv[2 * p], &b = cv[2 * p + 1];
      const double* Bp = H.B[l].p + pv[p].boff;
      if (a.k > 0 && b.k > 0) {
        g2.push_back({a.k, nrhs, b.k, Bp, b.k, 1, up[l + 1].p + b.koff * nrhs, nrhs, 1,
                      dn[l + 1].p + a.koff * nrhs, nrhs, 1, 1.0, 1.0});
        g2.push_back({b.k, nrhs, a.k, Bp, 1, b.k, up[l + 1].p + a.koff * nrhs, nrhs, 1,
                      dn[l + 1].p + b.koff * nrhs, nrhs, 1, 1.0, 1.0});
      }
    }
    bgemv(g2, s);
  }
  // leaves: out = D V + U g
  std::vector<GemmProb> gp;
  std::vector<CopyProb> cp;
  for (int i = sh.first(L); i < sh.last(L); ++i) {
    const auto& nd = H.lv[L][i];
    const int mloc = (int)(nd.hi - nd.lo);
    const int64_t lo = nd.lo - H.lo_g;
    gp.push_back({mloc, nrhs, mloc, H.D.p + nd.doff, mloc, 1, V + lo * nrhs, nrhs, 1,
                  out + lo * nrhs, nrhs, 1, 1.0, 0.0});
  }
  bgemv(gp, s);
  gp.clear();
  for (int i = sh.first(L); i < sh.last(L); ++i) {
    const auto& nd = H.lv[L][i];
    const int64_t lo = nd.lo - H.lo_g;
    if (nd.pt) cp.push_back({nd.rows, nrhs, dn[L].p + nd.koff * nrhs, nrhs, out + lo * nrhs, nrhs, 1});
    else if (nd.k > 0)
      gp.push_back({nd.rows, nrhs, nd.k, H.U[L].p + nd.uoff, nd.k, 1, dn[L].p + nd.koff * nrhs, nrhs, 1,
                    out + lo * nrhs, nrhs, 1, 1.0, 1.0});
  }
  bcopy(cp, s);
  bgemv(gp, s);
  CUDA_CHECK(cudaStreamSynchronize(s));
}

}  // namespace svmhss
