// internal.cuh — internal structures of libsvmhss (not part of the C-ABI).
#pragma once
#include <atomic>
#include <memory>
#include "common.cuh"
#include "comm.cuh"
#include "dense.cuh"

namespace svmhss {

// ---------------------------------------------------------------- kernel tiles (tiles.cu)
struct KmmArgs {
  const double* Fa; const double* nua; int64_t na;  // row points, rp-padded (stride rp)
  const double* Fb; const double* nub; int64_t nb;  // column points
  int rp;                                           // padded feature count (multiple of 4)
  const double* W; int64_t ldw; int ncols;          // nb x ncols right-hand matrix
  double* S; int64_t lds;                           // na x ncols output
  double neg_inv_2h2;                               // -1 / (2 h^2)
  int same_set;                                     // K_ii = 1 exactly (Fa rows are Fb rows)
  int64_t diag_off;                                 // same_set: Fa row i is Fb row diag_off + i
  const int* leaf_a; const int* leaf_b;             // nullable: zero pairs in the same leaf
  // NOTE: nub and leaf_b are read by 16-byte bulk copies: allocate them with >= 2 doubles /
  // 4 ints of padding past the end (kNormPad / kLeafPad).
};
constexpr int kNormPad = 2, kLeafPad = 4;
// S = K(Fa, Fb) W via DMMA distance GEMM -> exp -> DMMA GEMM (H1).
void kernel_matmul(const KmmArgs& a, cudaStream_t s);
// Prediction sums S (na x NC) = K(Fa, Fb) coef (a11): Fa / Fb with row stride SA =
// predict_stride(rp) (zero padded), nub and coef (nb x NC) with >= 2 doubles of padding.
int predict_stride(int rp);
void predict_sums(const double* Fa, const double* nua, int64_t na, const double* Fb, const double* nub,
                  const double* coef, int64_t nb, int rp, int SA, int NC, double neg_inv_2h2, double* S,
                  cudaStream_t s);
// Which kernel_matmul configuration serves (rp, ncols); for reporting.
int kmm_chunk_cols(int rp, int ncols);

// Omega rows for original indices idx (R1-R3), out rows x s (ld = s).
void omega_rows(uint64_t seed, const int64_t* idx, int64_t rows, int s, double* out,
                cudaStream_t st);

struct KblkProb {  // out[i*ld + j] = K(F[ia ? ia[i] : a0+i], F[ib ? ib[j] : b0+j])
  int na, nb;
  const int64_t* ia; int64_t a0;
  const int64_t* ib; int64_t b0;
  double* out; long long ld;
  double diag_add;  // added where (row point == column point), e.g. beta for D + beta I
};
// Direct-difference Gaussian kernel blocks over points of F (n x rp, stride rp, r used).
void kernel_blocks(const double* F, int rp, int r, double h, const std::vector<KblkProb>& probs,
                   cudaStream_t s);
// Pad F (n x r) to Fp (n x rp) and compute nu = ||f||^2 of the padded rows.
void pad_rows(const double* F, int64_t n, int r, int rp, double* out, cudaStream_t s);
void row_norms(const double* F, int64_t n, int rp, double* nu, cudaStream_t s);

struct CopyProb {  // rows x cols: mode 0 dst[i*drs + j] = src[i*srs + j]; 1: +=; 2: transposed,
                   // dst[j*drs + i] = src[i*srs + j]; 3 (square): symmetric from the lower triangle,
                   // dst[i*drs + j] = src[max(i,j)*srs + min(i,j)]
  int rows, cols;
  const double* src; long long srs;
  double* dst; long long drs;
  int accumulate;
};
void bcopy(const std::vector<CopyProb>& probs, cudaStream_t s);

// ---------------------------------------------------------------- stable radix sort (sort.cu)
// (key, value) pairs sorted stably by key bits [begin_bit, end_bit); bits above end_bit must be 0.
void radix_sort_pairs(const uint64_t* kin, uint64_t* kout, const int* vin, int* vout, int64_t n, int begin_bit,
                      int end_bit, cudaStream_t s);
void radix_sort_pairs(const unsigned* kin, unsigned* kout, const int* vin, int* vout, int64_t n, int begin_bit,
                      int end_bit, cudaStream_t s);
void radix_sort_pairs(const uint64_t* kin, uint64_t* kout, const uint64_t* vin, uint64_t* vout, int64_t n,
                      int begin_bit, int end_bit, cudaStream_t s);
void radix_sort_pairs(const unsigned* kin, unsigned* kout, const uint64_t* vin, uint64_t* vout, int64_t n,
                      int begin_bit, int end_bit, cudaStream_t s);
void radix_sort_pairs(const uint64_t* kin, uint64_t* kout, const double* vin, double* vout, int64_t n,
                      int begin_bit, int end_bit, cudaStream_t s);

// ---------------------------------------------------------------- tree (tree.cu)
// T1-T4 on the GPU. F: n x rp (padded, device). Outputs perm (n int64, device) and the
// permuted features Fp (n x rp) / norms nu.
// rp_tree_index >= 0: random-projection tree of HSS-ANN (reading N1; tree_seed = ann seed)
// instead of the PCA tree.
void build_tree(const double* Fpad, int64_t n, int r, int rp, int m, uint64_t tree_seed,
                int64_t* perm, double* Fp_out, cudaStream_t s, int rp_tree_index = -1);
int num_levels(int64_t n, int m);
void node_ranges(int64_t n, int L, std::vector<std::vector<std::pair<int64_t, int64_t>>>& out);

// ---------------------------------------------------------------- HSS
struct NodeInfo {
  int64_t lo = 0, hi = 0;  // tree positions
  int rows = 0, k = 0;     // active rows, rank
  bool pt = false;         // pass-through (k == rows)
  int cap_hit = 0;
  int64_t roff = 0;        // offset (rows) in level row-packed arrays
  int64_t koff = 0;        // offset (k) in level k-packed arrays
  int64_t uoff = 0;        // offset (doubles) of U_t in the level U buffer
  int64_t boff = 0;        // offset (doubles) of B_t (parents) in the level B buffer
  int64_t doff = 0;        // offset (doubles) of D_t (leaves)
};

// Subtree sharding plan: rank g of P (a power of two) owns node g of level
// lg = log2 P and its descendants; levels < lg are replicated.  At level l this rank
// processes BFS indices [first(l), last(l)).  Level-lg nodes of every rank become known
// after the build's exchange (k, skeletons, k-packed offsets: "global" packing at level lg).
struct Shard {
  std::shared_ptr<Comm> comm;
  int P = 1, g = 0, lg = 0;
  int first(int l) const { return l < lg ? 0 : (g << (l - lg)); }
  int last(int l) const { return l < lg ? (1 << l) : ((g + 1) << (l - lg)); }
  bool on() const { return P > 1; }
};

struct HSSImpl {
  std::atomic<int> refs{1};
  int64_t n = 0;
  int r = 0, rp = 0, L = 0, s = 0, m = 0;
  double h = 1.0;
  Shard sh;
  int64_t lo_g = 0, hi_g = 0;             // this rank's tree positions [lo_g, hi_g)
  int64_t nmax_g = 0;                     // max over ranks of hi_g - lo_g (exchange slots)
  int kmax_lg = 0;                        // max over level-lg nodes of k (exchange slots)
  DevBuf<int64_t> lg_koff, lg_k;          // level-lg nodes: global k-packed offset and k
  DevBuf<int64_t> rank_lo, rank_cnt;      // per rank: first tree position and count
  DevBuf<int64_t> leaf_lo;                // this rank's leaves: local first point (+ end)
  int nleaf_loc() const { return sh.last(L) - sh.first(L); }
  int64_t nloc() const { return hi_g - lo_g; }
  std::vector<std::vector<NodeInfo>> lv;  // lv[l][i], l = 0..L
  DevBuf<double> Fp, nu;
  DevBuf<int64_t> perm, iperm;
  DevBuf<int> leaf_of;
  DevBuf<double> D;                        // leaves (root if L == 0)
  std::vector<DevBuf<double>> U;           // per level
  std::vector<DevBuf<int64_t>> J;          // per level, k-packed tree positions
  std::vector<DevBuf<double>> B;           // per level (parents)
  hss_stats st{};
  int node_id(int l, int i) const { return (1 << l) - 1 + i; }
};

// s_cols > 0: sketch with s_cols columns instead of max_rank + oversample (adaptive sampling)
void hss_build_impl(HSSImpl& H, const double* F, int64_t n, int r, double h,
                    const hss_opts& o, std::shared_ptr<Comm> comm, cudaStream_t s, int s_cols = -1);
bool hss_unconverged(const HSSImpl& H, int p, int cap);
// K~ V in TREE order on this rank's points: V/out nloc x nrhs point-major (device),
// rows [lo_g, hi_g) of the tree order.
void hss_matvec_tree(const HSSImpl& H, const double* V, double* out, int nrhs, cudaStream_t s);
int64_t level_sumk(const HSSImpl& H, int l);

// ---------------------------------------------------------------- HSS-ANN (ann.cu; N1-N3)
// ANN lists of all n points (ORIGINAL order in and out): idx n x kappa original indices, d the
// squared distances; -1 / +inf padding.
void ann_build(const double* Fpad, int64_t n, int r, int rp, int kappa, int trees, int leaf, uint64_t seed,
               int64_t* idx_out, double* d_out, cudaStream_t s);
void ann_to_tree(const HSSImpl& H, int kappa, const int64_t* idx, const double* d, int64_t* pos, double* dp,
                 cudaStream_t s);
// sampled columns C (this rank's nodes of level l, nn x s, sorted tree positions, -1 padded)
void ann_sample_level(const HSSImpl& H, int l, const int64_t* act, const int64_t* ann_pos, const double* ann_d,
                      int kappa, uint64_t seed, int64_t* C, cudaStream_t s);
// Y_t = K(A_t, C_t) into the level's row-packed W (rows x s per node)
void ann_y_level(const HSSImpl& H, int l, const int64_t* act, const int64_t* C, double* W, cudaStream_t s);

// ---------------------------------------------------------------- sharded exchanges
// Workspace of the per-iteration level-lg exchange (allocated once: graph-capturable).
struct ExchWS {
  int ncols = 0, nextra = 0;
  int64_t slot = 0;              // doubles per rank slot: kmax_lg * ncols + nextra
  DevBuf<double> send, recv;     // slot, P * slot (ncclAllGather / host backends)
  std::shared_ptr<Comm> comm;    // device-API backend: the symmetric window below (N3)
  DevWindow win;
  ExchWS() {}
  ExchWS(const ExchWS&) = delete;
  ExchWS& operator=(const ExchWS&) = delete;
  ~ExchWS() { if (comm && win.win) comm->window_free(win); }
};
void exch_ws_alloc(const HSSImpl& H, int ncols, int nextra, ExchWS& ws);
// buf: level-lg k-packed vector (global offsets, ncols per row) in which only this rank's
// node is valid; fills every rank's node.  extra (nextra doubles, nullable) is appended to
// the slot and gathered to extra_out (P x nextra, rank-major).  No-op when P == 1 except
// copying extra to extra_out.
void exchange_lg(const HSSImpl& H, ExchWS& ws, double* buf, const double* extra,
                 double* extra_out, cudaStream_t s);
// local point vector (nloc x ncols, tree order) -> full tree-order vector (n x ncols) on
// every rank.
void gather_points(const HSSImpl& H, const double* loc, int ncols, double* full, cudaStream_t s);

// Fixed-order reductions that follow the cluster tree (bitwise P-invariant): `part` holds
// one partial per leaf this rank holds (nleaf_loc x ncols); reduce pairwise up to the
// subtree root (this rank) and, after an exchange of the P subtree-root values, pairwise over
// the top levels.  tree_reduce_local writes ncols values to `out`; tree_reduce_top reduces
// P x ncols rank-major values to ncols.
void tree_reduce_local(const HSSImpl& H, double* part, int ncols, double* out, cudaStream_t s);
void tree_reduce_top(int P, const double* in, int ncols, double* out, cudaStream_t s);
// Host convenience: full reduction of per-leaf partials to ncols host values.
void tree_reduce_all(const HSSImpl& H, double* part, int ncols, double* host_out, cudaStream_t s);

// ---------------------------------------------------------------- ULV
struct SolveNode {
  int R, k, pt, pad;
  int64_t moff;  // offset (doubles) of M_t in the level M buffer
  int64_t roff;  // offset (rows) in this level's row-packed vectors
  int64_t koff;  // offset (rows) in the parent level's row-packed vectors (= k-packed here)
  int64_t yoff;  // offset (rows) in this level's yr vectors
};
struct SolveWork { int node, chunk; };

constexpr int kCW = 64;  // backward sweep: columns per CTA
constexpr int kBW = 8;   // backward sweep: warps per CTA
constexpr int kSplitMaxLevel = 4;  // bwd row split for levels l <= 4 (l < L-1): <= 16 nodes (A/B at cfg 3: 4 best of -1..7)
constexpr int kLarftSolveMaxLevel = 7;  // factor: T by the triangular solve on levels l <= 7 (<= 128 nodes; A/B at cfg 3: 1.02 -> 0.53 ms per single-node level, slower from 256 nodes)
constexpr int kRB = 64;            // bwd row split: rows per chunk
struct ULVLevel {
  int nnodes = 0, maxR = 0, allpt = 1;
  int64_t sumR = 0, sumK = 0, sumY = 0;
  DevBuf<double> M;              // per-node solve operators (row-major R x R)
  DevBuf<SolveNode> nodes;
  DevBuf<SolveWork> work;        // fwd: (node, chunk of `ch` rows); leaf level: non-pass-through only
  DevBuf<SolveWork> bwork;       // bwd: (node, chunk of kCW columns [x row chunks if split])
  int nwork = 0, nbwork = 0, ch = 32;
  int split = 0;                 // bwd rows split into kRB-row chunks (small top levels)
};

struct ULVImpl {
  std::atomic<int> refs{1};
  HSSImpl* H = nullptr;
  double beta = 0.0;
  std::vector<ULVLevel> lv;   // 0..L (0 = root)
  DevBuf<int64_t> ptmap;      // tree position -> level L-1 vector index for pass-through leaves
  int nleafpt = 0;
  ulv_stats st{};
};

void ulv_factor_impl(ULVImpl& F, cudaStream_t s);

// Solve workspace for nrhs right-hand sides (tree order in/out, this rank's points).
struct SolveWS {
  int nrhs = 0;
  std::vector<double*> fin, yr, xout;  // per level (levels that are all pass-through alias)
  std::vector<double*> bpart;          // split bwd levels: row-chunk partials
  std::vector<unsigned*> bcnt;         // split bwd levels: per (node, column chunk) counters
  std::vector<DevBuf<double>> own;
  std::vector<DevBuf<unsigned>> cnt_own;
  // sharded: the level-lg exchange; `extra` (nextra doubles per rank, set nextra before
  // solve_ws_alloc) rides along, gathered to extra_all (P x nextra) and, if extra_top is set,
  // tree-reduced over the ranks into extra_top.
  ExchWS xw;
  int nextra = 0;
  const double* extra = nullptr;
  double* extra_all = nullptr;
  double* extra_top = nullptr;
  // ADMM: the caller reads x of pass-through leaves from xout[L-1] and writes their next
  // right-hand side into fin[L-1] itself (via ptmap), so the two leaf copies are skipped.
  bool fused_leaf_io = false;
};
void solve_ws_alloc(const ULVImpl& F, int nrhs, SolveWS& ws);
// x_tree = (K~+beta I)^-1 b_tree.  b is read from ws.fin[L] and x written to ws.xout[L].
void ulv_solve_tree(const ULVImpl& F, SolveWS& ws, cudaStream_t s);
// Pieces of the solve (sweeps over level ranges, the sharded exchange).
struct SolveStep {
  enum Kind { FWD, BWD, EXCHANGE };
  int kind = FWD, a = 0, b = 0;
  bool no_exchange = false;
};
void ulv_solve_steps(const ULVImpl& F, SolveWS& ws, const std::vector<SolveStep>& steps, cudaStream_t s);


// ---------------------------------------------------------------- ADMM / predict (admm.cu)
struct AdmmResult { double w1; double ms_pre, ms_loop, ms_bias; int graph; int64_t launches; };
AdmmResult admm_train_impl(const ULVImpl& F, const double* y_orig, const std::vector<double>& Cs,
                           int max_it, const admm_opts* opt, double* z_out, double* mu_out,
                           double* bias_out, double* obj_out, cudaStream_t s);
// a11: coefficients y o z formed on the device; comm (nullable) shards the
// test points (one allgather of the decision values).
void predict_impl(const double* Ftrain, const double* y, const double* z, int64_t n, int r, double h,
                  const double* bias_host, int nC, const double* Ftest, int64_t m, double* dv,
                  int8_t* lab, Comm* comm, cudaStream_t s);

// ---------------------------------------------------------------- permutation helpers
void gather_rows(const double* src, const int64_t* idx, int64_t rows, int cols, double* dst,
                 cudaStream_t s);   // dst[i] = src[idx[i]]
void scatter_rows(const double* src, const int64_t* idx, int64_t rows, int cols, double* dst,
                  cudaStream_t s);  // dst[idx[i]] = src[i]

}  // namespace svmhss
