// internal.cuh — internal structures of libsvmhss (not part of the C-ABI).
#pragma once
#include <atomic>
#include <memory>
#include "common.cuh"
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
  int same_set;                                     // K_ii = 1 exactly (Fa == Fb)
  const int* leaf_a; const int* leaf_b;             // nullable: zero pairs in the same leaf
  // NOTE: nub and leaf_b are read by 16-byte bulk copies: allocate them with >= 2 doubles /
  // 4 ints of padding past the end (kNormPad / kLeafPad).
};
constexpr int kNormPad = 2, kLeafPad = 4;
// S = K(Fa, Fb) W via DMMA distance GEMM -> exp -> DMMA GEMM (H1).
void kernel_matmul(const KmmArgs& a, cudaStream_t s);
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

struct CopyProb {  // dst[i*drs + j] (+)= src[i*srs + j], rows x cols
  int rows, cols;
  const double* src; long long srs;
  double* dst; long long drs;
  int accumulate;
};
void bcopy(const std::vector<CopyProb>& probs, cudaStream_t s);

// ---------------------------------------------------------------- tree (tree.cu)
// T1-T4 on the GPU. F: n x rp (padded, device). Outputs perm (n int64, device) and the
// permuted features Fp (n x rp) / norms nu.
void build_tree(const double* Fpad, int64_t n, int r, int rp, int m, uint64_t tree_seed,
                int64_t* perm, double* Fp_out, cudaStream_t s);
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

struct HSSImpl {
  std::atomic<int> refs{1};
  int64_t n = 0;
  int r = 0, rp = 0, L = 0, s = 0, m = 0;
  double h = 1.0;
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

void hss_build_impl(HSSImpl& H, const double* F, int64_t n, int r, double h,
                    const hss_opts& o, cudaStream_t s);
// K~ V in TREE order, V/out n x nrhs point-major (device).
void hss_matvec_tree(const HSSImpl& H, const double* V, double* out, int nrhs, cudaStream_t s);

// ---------------------------------------------------------------- ULV
struct SolveNode {
  int R, k, pt, pad;
  int64_t moff;  // offset (doubles) of M_t in the level M buffer
  int64_t roff;  // offset (rows) in this level's row-packed vectors
  int64_t koff;  // offset (rows) in the parent level's row-packed vectors (= k-packed here)
  int64_t yoff;  // offset (rows) in this level's yr vectors
};
struct SolveWork { int node, chunk; };

struct ULVLevel {
  int nnodes = 0, maxR = 0, allpt = 1;
  int64_t sumR = 0, sumK = 0, sumY = 0;
  DevBuf<double> M, MT;          // per-node solve operators and their transposes
  DevBuf<SolveNode> nodes;
  DevBuf<SolveWork> work;        // (node, chunk of `ch` rows); leaf level: non-pass-through only
  int nwork = 0, ch = 32;
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
void btranspose(const std::vector<SqProb>& probs, const double* base, double* out, cudaStream_t s);

// Solve workspace for nrhs right-hand sides (tree order in/out).
struct SolveWS {
  int nrhs = 0;
  std::vector<double*> fin, yr, xout;  // per level (levels that are all pass-through alias)
  std::vector<DevBuf<double>> own;
};
void solve_ws_alloc(const ULVImpl& F, int nrhs, SolveWS& ws);
// x_tree = (K~+beta I)^-1 b_tree.  b is read from ws.fin[L] and x written to ws.xout[L].
void ulv_solve_tree(const ULVImpl& F, SolveWS& ws, cudaStream_t s);
// number of kernel launches of ulv_solve_tree
int ulv_solve_launches(const ULVImpl& F);

// ---------------------------------------------------------------- ADMM / predict (admm.cu)
struct AdmmResult { double w1; double ms_pre, ms_loop, ms_bias; int graph; int64_t launches; };
AdmmResult admm_train_impl(const ULVImpl& F, const double* y_orig, const std::vector<double>& Cs,
                           int max_it, const admm_opts* opt, double* z_out, double* mu_out,
                           double* bias_out, double* obj_out, cudaStream_t s);
void predict_impl(const double* Ftrain, const double* coef, int64_t n, int r, double h,
                  const double* bias_host, int nC, const double* Ftest, int64_t m, double* dv,
                  int8_t* lab, cudaStream_t s);

// ---------------------------------------------------------------- permutation helpers
void gather_rows(const double* src, const int64_t* idx, int64_t rows, int cols, double* dst,
                 cudaStream_t s);   // dst[i] = src[idx[i]]
void scatter_rows(const double* src, const int64_t* idx, int64_t rows, int cols, double* dst,
                  cudaStream_t s);  // dst[idx[i]] = src[i]

}  // namespace svmhss
