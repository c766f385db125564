// dense.cuh — batched small dense fp64 kernels used by compression (H3-H4) and the ULV
// factorization (U).  Every operand is a strided view: element (i,j) at p[i*rs + j*cs],
// so transposes are stride swaps.  One problem = one tree node.
#pragma once
#include "common.cuh"

namespace svmhss {

struct GemmProb {  // C = alpha * A(m x k) * B(k x n) + beta * C   (beta == 0: C not read)
  int m, n, k;
  const double* A; long long ars, acs;
  const double* B; long long brs, bcs;
  double* C; long long crs, ccs;
  double alpha, beta;
  int lower;       // 1: C is symmetric, only CTA tiles touching the lower triangle are computed
};

struct SqProb {    // square matrix problem (Cholesky / larft / trsm matrix)
  int n;
  double* A; long long rs, cs;
};

struct TrsmProb {  // X = op(T)^-1 X in place; T n x n triangular, X n x nrhs
  int n, nrhs;
  const double* T; long long trs, tcs;
  double* X; long long xrs, xcs;
};

struct QrProb {    // Householder QR in place of A (m x n, m >= n), tau[n]
  int m, n;
  double* A; long long rs, cs;
  double* tau;
};

struct CpqrProb {  // column-pivoted QR of A = W^T, W rows x s row-major (column c = W[c,:])
  int rows, s;
  double* W;       // in place
  int* piv;        // out: rows entries, column permutation
  int kfixed;      // >= 0: fixed rank; < 0: adaptive
  int* k_out;      // out: rank
  int* cap_hit;    // out: 1 if the tolerance was unmet at the cap
  const int* forced;  // nullable (device): fixed-skeleton mode, the first k pivots (original
                      // column indices, in pivot order; k = kfixed)
};

// Batched launchers (problem arrays are HOST vectors; uploaded into a scratch buffer).
void bgemm(const std::vector<GemmProb>& probs, cudaStream_t s);
// The same contract; problems with n <= 16 columns (B, C unit column stride, A row-major or
// transposed) run as streaming GEMV kernels (HSS mat-vec), the rest through bgemm.
void bgemv(const std::vector<GemmProb>& probs, cudaStream_t s);
// Cholesky (lower, in place, upper triangle zeroed).  info[i] = 0 ok, j+1 if breakdown at j.
void bpotrf(const std::vector<SqProb>& probs, int* d_info, cudaStream_t s);
// lower: forward substitution with T lower (non-unit); !lower: back substitution, T upper.
void btrsm(const std::vector<TrsmProb>& probs, bool lower, cudaStream_t s);
void bgeqr2(const std::vector<QrProb>& probs, cudaStream_t s);
// T (n x n upper) from V'V (S, n x n, in T's place on input) and tau: compact WY, Q = I - V T V^T.
// by_solve: T = (I + D U)^-1 D by btrsm (few-node levels), else the blocked column recurrence.
void blarft(const std::vector<SqProb>& probs_T, const std::vector<const double*>& taus, bool by_solve,
            cudaStream_t s);
void bcpqr(const std::vector<CpqrProb>& probs, double rel_tol, double abs_tol, int cap,
           cudaStream_t s);
// blocked (dlaqps-style) CPQR, one CTA per node (cpqr.cu); fits: rows / s within its smem tiles
bool cpqr_blk_fits(int rows, int s);
void bcpqr_blk(const CpqrProb* d_probs, int nprob, int maxr, int maxs, double rel_tol, double abs_tol, int cap,
               cudaStream_t s);

// Small helpers
void fill_identity(double* A, int n, long long rs, long long cs, cudaStream_t s);

}  // namespace svmhss
