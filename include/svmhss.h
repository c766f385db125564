/*
 * svmhss.h — C-ABI of libsvmhss.so: the B200 (sm_100a) hot path of
 * "ADMM + HSS kernel approximations for large-scale nonlinear SVMs" (arXiv 2108.04167).
 *
 * Citations: P:n = PAPER.md line n.  Step labels (T*, R*, H*, U*, S*, A*, AMB-*) are the
 * readings listed in DESIGN.md ("Readings of the paper").
 *
 * Common conventions (every entry point):
 *  - Array pointers are DEVICE pointers on the current CUDA device, fp64 unless noted,
 *    except the *_host entry points, whose pointers are HOST pointers.
 *  - User-visible per-point vectors are in ORIGINAL point order; internally the library
 *    works in tree (permuted) order.  Multi-column vectors are point-major:
 *    v[i*ncols + c].
 *  - Calls are ordered on `stream` (a cudaStream_t passed as void*; NULL = legacy default
 *    stream).  Functions that must read sizes back (build, factor, train) synchronize
 *    `stream` before returning.
 *  - Return 0 (HSS_OK) on success, a negative HSS_E* code on error; a human-readable
 *    message is available from hss_last_error() (thread-local).  On error no output
 *    buffer is guaranteed to be written and no handle is returned.
 *  - Ownership: handles own their device memory.  The caller owns every input and
 *    output buffer.  A ulv_t keeps its hss_t alive (reference counted), so the two can
 *    be freed in any order.
 *  - Determinism: identical inputs and options give bitwise-identical outputs (fixed
 *    reduction orders, no floating-point atomics).
 *  - No CPU fallback exists: without a usable CUDA device every call returns HSS_ECUDA.
 */
#ifndef SVMHSS_H
#define SVMHSS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  HSS_OK = 0,
  HSS_EINVAL = -1,   /* invalid argument (sizes, h <= 0, beta <= 0, C <= 0, labels not +-1, ...) */
  HSS_ENOMEM = -2,   /* device allocation failed */
  HSS_ECUDA = -3,    /* CUDA runtime / launch error, or no device */
  HSS_ENCCL = -4,    /* reserved for the multi-GPU communicator */
  HSS_ENOTSPD = -5,  /* K~ + beta I not SPD: Cholesky breakdown; node id in the message (AMB-14) */
  HSS_EW1 = -6       /* w1 = e^T (K~+beta I)^-1 e <= 0 */
};

typedef struct hss_s* hss_t;  /* compressed kernel K~ */
typedef struct ulv_s* ulv_t;  /* ULV factorization of K~ + beta I */
typedef struct hss_comm_s* hss_comm_t;  /* subtree-sharding communicator */

/* ---- multi-GPU subtree sharding ----
 * With a communicator of P ranks (P a power of two, P <= 2^L), rank g owns node g of tree
 * level lg = log2(P) — a contiguous range of tree positions — and all of its descendants.
 * Levels below lg are computed only by their owner; levels above lg redundantly by every
 * rank.  The only device<->device traffic is one allgather of fixed-size rank slots:
 * subtree-root skeleton data (build), reduced Schur blocks (factor), and per ADMM iteration
 * the reduced right-hand side plus the partial w^T q (the paper's method is sequential,
 * P:351; this partitioning is ours).  Node-level work and every reduction follow the cluster
 * tree, so results are bitwise identical for every P.  Every rank passes the same full
 * inputs (F, y: all n points, original order) and receives the same full outputs.
 *
 * hss_allgather_fn: host backend callback.  send: `bytes` HOST bytes of this rank; recv:
 * nranks * bytes HOST bytes, rank-major.  Return 0 on success (non-zero -> HSS_ENCCL).
 * The host backend synchronizes the stream at every exchange (not graph-capturable); it
 * lets P ranks run as P processes sharing fewer GPUs (no kernel ever waits on a peer).
 * The NCCL backend (libnccl.so.2 loaded at run time) exchanges device buffers with
 * ncclAllGather, stream-ordered and captured in the ADMM iteration's CUDA graph.
 * Errors: HSS_EINVAL (nranks < 1, rank out of range, NULL fn), HSS_ENCCL (NCCL missing or
 * failing).  hss_comm_free may be called while handles built with the comm are alive
 * (they keep it alive). */
typedef int (*hss_allgather_fn)(void* ctx, const void* send, void* recv, size_t bytes);
int hss_comm_nccl_id(void* unique_id_out /* 128 HOST bytes, rank 0 then broadcasts */);
int hss_comm_init_nccl(int32_t nranks, int32_t rank, const void* unique_id, hss_comm_t* out);
int hss_comm_init_host(int32_t nranks, int32_t rank, hss_allgather_fn fn, void* ctx,
                       hss_comm_t* out);
void hss_comm_free(hss_comm_t comm);
/* in-kernel exchange: with NCCL >= 2.28 and every rank an LSA (NVLink load/store)
 * peer, the NCCL communicator creates a device communicator (ncclDevCommCreate, one LSA barrier)
 * and the per-iteration level-lg exchange becomes ONE kernel (inside the ADMM iteration's CUDA
 * graph): the rank's slot is stored straight into every peer's symmetric window
 * (ncclCommWindowRegister over ncclMemAlloc memory, two halves used on alternate calls), one LSA
 * barrier, and every slot is unpacked from the local window.  Otherwise (older NCCL, ranks
 * not all NVLink peers, or SVMHSS_NCCL_DEVICE=0) ncclAllGather.  Results are bitwise the same.
 * hss_comm_info reports nranks / rank / whether the device API is in use (each nullable). */
int hss_comm_info(hss_comm_t comm, int32_t* nranks, int32_t* rank, int32_t* device_api);
/* Debug: one exchange of `count` doubles per rank through the communicator's per-iteration path
 * (device API when in use, else allgather); recv: nranks * count device doubles, rank-major.
 * Window allocation is collective: every rank must call it. */
int hss_comm_exchange_test(hss_comm_t comm, const double* send, int64_t count, double* recv, void* stream);

/* Build options (P:184-187 and readings T1-T4, R1-R3, H1-H5, AMB-10, AMB-11). */
typedef struct {
  int32_t leaf_size;       /* m >= 1: leaf size; tree depth L = ceil(log2(n/m)) (T1) */
  double rel_tol;          /* AMB-10 rank rule: |R_jj| > max(rel_tol |R_11|, abs_tol sqrt(s)) */
  double abs_tol;
  int32_t max_rank;        /* k_max >= 1: rank cap */
  int32_t oversample;      /* p >= 0: sketch columns s = max_rank + p (AMB-18) */
  uint64_t omega_seed;     /* R1-R3 key for Omega (keyed by ORIGINAL index, column) */
  uint64_t tree_seed;      /* R1-R3 key for the power-iteration start vectors (T2) */
  const int32_t* ranks;    /* HOST pointer, nullable.  Fixed-rank mode: one rank per node in
                              level-major BFS order (2^(L+1)-1 entries; root ignored); the
                              node's rank is min(ranks[t], rows_t, s).  NULL = adaptive. */
  hss_comm_t comm;         /* nullable: single GPU.  Else subtree sharding over comm's ranks;
                              the factorization and ADMM inherit it from the hss_t. */
  /* Column sampling of the compression:
   *  HSS_SAMPLING_SKETCH (0): randomized sketch S = K Omega of all columns (H1-H5);
   *  HSS_SAMPLING_ANN (1): HSS-ANN (readings N1-N3): per node, Y = K(A_t, C_t) on
   *    s sampled columns chosen from the active rows' approximate nearest neighbours
   *    (ann_trees random-projection trees of leaf size ann_leaf <= 256, ann_neighbors per
   *    point, ann_trees * ann_neighbors <= 256, ann_leaf * r * 8 <= 227 KB), random-filled
   *    from ann_seed; omega_seed is unused. */
  int32_t sampling;
  int32_t ann_neighbors, ann_trees, ann_leaf;
  uint64_t ann_seed;
  /* Adaptive randomized sampling (readings N2a-c; sketch sampling only):
   * adaptive_s0 > 0 starts with s = min(adaptive_s0, max_rank + oversample) columns of Omega and,
   * while some node's rank k > s - oversample with k < min(max_rank, rows), rebuilds with
   * s += adaptive_ds (> 0), up to max_rank + oversample.  0 = fixed s = max_rank + oversample. */
  int32_t adaptive_s0, adaptive_ds;
  /* Parity imports (sketch sampling, no adaptive rounds):
   * perm: HOST pointer, nullable.  n int64 tree position -> original index (a bijection of
   *   0..n-1, e.g. the oracle's T1-T4 output); replaces the tree construction (T1-T4).  Node
   *   ranges stay the uniform split of T1.  HSS_EINVAL if it is not a permutation.
   * skeletons: HOST pointer, nullable; needs `ranks`.  Fixed-skeleton diagnostic mode (AMB-12):
   *   the skeleton J_t of every non-root node, in hss_info's skel_out layout (levels 1..L,
   *   nodes in BFS order, k_t tree positions each, in pivot order).  The CPQR of Y_t^T then
   *   takes these columns as its first k_t pivots, in this order, instead of the norm argmax;
   *   U_t = P[I; (R11^-1 R12)^T] as usual.  Every J_t must be k_t distinct active rows of t
   *   (its points at the leaves, its children's skeletons above), else HSS_EINVAL. */
  const int64_t* perm;
  const int64_t* skeletons;
  /* Interpolation of the compression (SPD-preserving compression; DESIGN.md
   * "N4"):
   *  HSS_INTERP_ID (0): the paper's interpolative decomposition (H3): U_t = P[I; T^T],
   *    T = R11^-1 R12 of the CPQR of Y_t^T.  K~ can be indefinite once ranks are capped, so
   *    beta must exceed -lambda_min(K~) (AMB-9 calibration).
   *  HSS_INTERP_SPD (1): the same skeletons J_t (same CPQR, rank rule, imports), but
   *    U_t = K(A_t, J_t) (K(J_t, J_t) + spd_eps I)^-1 (kernel interpolation onto the skeleton;
   *    A_t = the node's active rows), by a Cholesky factor of K(J_t,J_t) + spd_eps I and two
   *    triangular solves.  K~ is then positive semidefinite for every rank choice, so
   *    K~ + beta I is SPD for every beta > 0 (the paper's beta schedule, applies).
   *    spd_eps >= 0 (relative to K_ii = 1; 1e-12 recommended).  HSS_ENOTSPD (naming the node)
   *    if a K(J_t,J_t) + spd_eps I has no Cholesky factor (e.g. repeated points, spd_eps = 0). */
  int32_t interp;
  double spd_eps;
} hss_opts;
enum { HSS_SAMPLING_SKETCH = 0, HSS_SAMPLING_ANN = 1 };
enum { HSS_INTERP_ID = 0, HSS_INTERP_SPD = 1 };

/* Build statistics (D6 / P:366-367 "Compression", "Memory"). */
typedef struct {
  int64_t n;
  int32_t r, L, s, leaf_size;
  int32_t max_rank_used;   /* max over nodes of k_t */
  int32_t cap_hits;        /* nodes where the tolerance was unmet at the cap (warning) */
  int32_t passthrough;     /* nodes with k_t == rows_t */
  int64_t generator_bytes; /* bytes of D, U, B (fp64) */
  double ms_tree, ms_omega, ms_sketch, ms_compress; /* phase device times (CUDA events) */
  int32_t s_used, sample_rounds;   /* sketch columns of the final build, builds (adaptive: >= 1) */
} hss_stats;

typedef struct {
  double beta;
  int64_t factor_bytes;    /* bytes of the per-node solve operators M_t */
  double ms_factor;
  double factor_flops;     /* algorithmic flops of this rank's nodes (SURVEY §8(d) a7 count) */
} ulv_stats;

/* ---- build: tree + Omega + sketch + per-level ID compression (Alg.3 l.1) ----
 * F: n x r row-major features (device).  h > 0 kernel width.
 * Returns HSS_EINVAL if n < 1, r < 1, h <= 0, leaf_size < 1, max_rank < 1, oversample < 0,
 * or s = max_rank + oversample > 2^20 (RNG column field, R1).
 * Memory: device buffers come from the library's OWN stream-ordered pool on the current device
 * (cudaMemPoolCreate; never the device's default pool, so torch's allocator is not affected).
 * The pool keeps freed memory reserved while any hss_t / ulv_t of the device is alive and is
 * trimmed to zero when the last one is freed (unless SVMHSS_POOL_KEEP=1; hss_pool_trim releases).  Before the first build of a given size the pool
 * is grown once to about 24 n (s + r) 8 bytes (at most half the free memory;
 * SVMHSS_POOL_RESERVE_GB overrides, 0 disables) so later phases do not map memory mid-call. */
int hss_build(const double* F, int64_t n, int32_t r, double h, const hss_opts* opt,
              void* stream, hss_t* out);

/* Stats and the tree/rank/skeleton export used by the parity tests.
 * perm_out: n int64 (tree position -> original index), nullable.
 * ranks_out: 2^(L+1)-1 int32 (level-major BFS, root = -1), nullable.  Sharded: nodes held
 *   by another rank (below level lg, outside this rank's subtree) are -2.
 * skel_out: sum_t k_t int64 tree positions, nodes in BFS order, nullable (sharded: only the
 *   nodes this rank holds contribute).  HOST pointers.
 * Stats (cap_hits, passthrough, max_rank_used, generator_bytes) are global over all ranks. */
int hss_info(hss_t H, hss_stats* st, int64_t* perm_out, int32_t* ranks_out, int64_t* skel_out);

/* out = K~ v (reading M: up/down sweeps); v, out: n x nrhs, original order. */
int hss_matvec(hss_t H, const double* v, double* out, int32_t nrhs, void* stream);

/* ---- ULV factorization of K~ + beta I (readings U) ----
 * beta > 0.  HSS_ENOTSPD if a Cholesky breaks down (message names the node). */
int hss_ulv_factor(hss_t H, double beta, void* stream, ulv_t* out);
int ulv_info(ulv_t U, ulv_stats* st);

/* x = (K~ + beta I)^-1 b (readings S); b, x: n x nrhs, original order; may alias.
 * nrhs >= 1 (the sweep kernels take up to 8 columns at a time; more run in groups of 8). */
int ulv_solve(ulv_t U, const double* b, double* x, int32_t nrhs, void* stream);

/* ---- ADMM training (Alg. 2; Alg. 3 lines 4-13; AMB-1) ----
 * y: n labels, exactly +-1.0 (original order).  C: nC box bounds > 0 (HOST pointer), nC >= 1.
 * The nC problems advance together as nC right-hand sides of one solve per iteration
 * (factorization reused across C); nC > 8 runs in groups of 8 (the sweep kernels'
 * widest right-hand side), each group an independent ADMM over its C values.
 * HSS_EW1 if w1 = e^T (K~+beta I)^-1 e <= 0.  Test hook: with the environment variable
 * SVMHSS_FAULT_W1=1 the computed w1 is negated before that check (the error path is otherwise
 * unreachable once the factorization succeeded: a successful ULV makes K~+beta I SPD).  max_it >= 1 iterations exactly.
 * Outputs (device, n x nC point-major, original order): z_out (required), mu_out (nullable).
 * bias_out, obj_out: nC HOST doubles, nullable: bias per AMB-2/AMB-3 via one HSS mat-vec
 * (P:196-200), objective f~(z) of Eq. (8).
 * trace: nullable; if trace_every > 0, z and mu after every trace_every-th iteration (and
 * the last) are written to trace_z / trace_mu (device, ntrace x n x nC, original order,
 * ntrace = ceil(max_it / trace_every)). */
typedef struct {
  int32_t trace_every;
  double* trace_z;
  double* trace_mu;
  double margin_eps_rel;   /* AMB-3 epsilon / C; <= 0 selects the default 1e-8 */
} admm_opts;

typedef struct {
  double w1;               /* e^T (K~+beta I)^-1 e */
  double ms_precompute, ms_loop, ms_bias;
  int32_t iterations, graph;  /* graph = 1 if the loop ran as a CUDA graph */
  int64_t kernel_launches_per_iter;
} admm_stats;

int admm_svm_train(ulv_t U, const double* y, const double* C, int32_t nC, int32_t max_it,
                   const admm_opts* opt, double* z_out, double* mu_out, double* bias_out,
                   double* obj_out, admm_stats* st, void* stream);

/* ---- prediction (Alg. 3; AMB-15, AMB-19: exact kernel) ----
 * dv[t*nC + c] = sum_i y_i z[i*nC + c] K(Ftrain_i, Ftest_t) + bias[c]; label = +1 if dv >= 0.
 * The coefficients z_y = y o z are formed inside the library.
 * Ftrain: n x r, Ftest: m x r row-major (device); y: n labels (device); z: n x nC (device,
 * admm_svm_train's z_out); bias: nC HOST doubles.  dv_out: m x nC device (nullable);
 * label_out: m x nC int8 device (nullable).  1 <= nC <= 16.
 * comm: nullable.  With a communicator of P ranks every rank passes the same full inputs; rank
 * g evaluates test points [floor(m g / P), floor(m (g+1) / P)) and one allgather of the decision
 * values gives every rank the full dv_out / label_out (bitwise the same as P = 1: each test
 * point's sum does not depend on P). */
int svm_predict(const double* Ftrain, const double* y, const double* z, int64_t n, int32_t r,
                double h, const double* bias, int32_t nC, const double* Ftest, int64_t m,
                double* dv_out, int8_t* label_out, hss_comm_t comm, void* stream);

/* ---- end-to-end on HOST buffers (Alg. 3): host->device copies of F, y,
 * Ftest, the full build + factor + ADMM + bias + predict, device->host copies of z and
 * labels.  z_out: n x nC, labels_out: m x nC (int8), bias_out, obj_out: nC — all HOST,
 * labels_out nullable (then Ftest may be NULL and m = 0).  timings_ms (nullable, HOST,
 * 8 doubles): h2d, build, factor, admm, bias, predict, d2h, total. */
int svm_train_predict_host(const double* F, const double* y, int64_t n, int32_t r,
                           double h, const hss_opts* opt, double beta, const double* C,
                           int32_t nC, int32_t max_it, const double* Ftest, int64_t m,
                           double* z_out, double* bias_out, double* obj_out,
                           int8_t* labels_out, double* timings_ms);

/* ---- debug / parity exports of individual hot-path steps ---- */
/* N1: the ANN lists of HSS-ANN sampling.  F: n x r row-major (device, ORIGINAL order);
 * idx_out: n x kappa int64 original indices sorted by (squared distance, index), -1 padded;
 * d_out: n x kappa squared distances (+inf padded).  Same limits as hss_opts' ann fields. */
int hss_ann_lists(const double* F, int64_t n, int32_t r, int32_t kappa, int32_t trees, int32_t leaf,
                  uint64_t seed, int64_t* idx_out, double* d_out, void* stream);
/* R1-R3: Omega rows for the given ORIGINAL indices (device int64 idx, count rows), s cols. */
int hss_omega(uint64_t seed, const int64_t* idx, int64_t rows, int32_t s, double* out, void* stream);
/* T1-T4: the permutation only (device int64 perm_out, n). */
int hss_tree(const double* F, int64_t n, int32_t r, int32_t leaf_size, uint64_t tree_seed,
             int64_t* perm_out, void* stream);
/* H1: S = K(Fa, Fb) W  (Fa: na x r, Fb: nb x r, W: nb x ncols, S: na x ncols; all device,
 * row-major), with the fused distance-GEMM -> exp -> GEMM kernel.  If same_set != 0, Fa and
 * Fb are the same points and K_ii = 1 exactly. */
int hss_kernel_matmul(const double* Fa, int64_t na, const double* Fb, int64_t nb, int32_t r,
                      double h, const double* W, int32_t ncols, int32_t same_set, double* S,
                      void* stream);
/* K(Fa, Fb) block (na x nb row-major, device). */
int hss_kernel_block(const double* Fa, int64_t na, const double* Fb, int64_t nb, int32_t r,
                     double h, double* K, void* stream);
/* Node generators for parity: U_t (rows x k row-major, identity if pass-through),
 * B_t (k_left x k_right, internal nodes), D_t (leaf, m_t x m_t).  HOST outputs; query
 * sizes with NULL pointers (rows/k written).  node = level-major BFS id. */
int hss_node(hss_t H, int32_t node, int32_t* rows, int32_t* k, double* U, double* B,
             double* D);

/* Number of kernels this library has launched in this process (graph replays included);
 * used by bench.py to report gpu_launches. */
int64_t hss_launch_count(void);

/* Handles are freed on the device they were created on (the caller's current device is kept).
 * Freeing the device's last hss_t / ulv_t trims the library's memory pool to zero. */
void hss_free(hss_t H);
void ulv_free(ulv_t U);
/* Release the memory the library's pool keeps reserved on the current device (e.g. after
 * svm_train_predict_host, which keeps its buffers' memory for the next call).  Synchronizes
 * the device.  Memory of live handles is not affected. */
int hss_pool_trim(void);
const char* hss_last_error(void);
/* "svmhss 0.2 (sm_100a)": 0.2 appended hss_opts.interp / spd_eps (N4); callers must zero-initialize
 * the whole hss_opts (the library reads every field). */
const char* hss_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SVMHSS_H */
