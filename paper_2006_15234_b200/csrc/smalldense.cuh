// Small dense factorizations that sit between the big contractions of
// einsumsvd: k x k Gram eigen-factors, Cholesky factors for CholeskyQR2, and
// (batched) small SVDs.  Each problem runs inside ONE thread block (shared
// memory resident when it fits), so no host round-trip is needed.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace pepsb {

// Status words written by the small kernels (device int).
enum SmallStatus : int {
  kSmallOk = 0,
  kSmallZeroGram = 1,       // gram of a zero operator (decomposition.cpp:132)
  kSmallNotHermitian = 2,   // eigh Hermiticity check (linalg.cpp:268-271)
  kSmallCholBreakdown = 4,  // Cholesky pivot <= 0
  kSmallNoConverge = 8,     // Jacobi sweep cap hit
  kSmallCompletionExhausted = 16,
};

// Reference gram_factors (proj/src/decomposition.cpp:128-156) on a device n x n
// Gram matrix G (row-major):  eigh (descending, phase-fixed, linalg.cpp:256-295)
// -> clamp at 1e-12*lmax -> P = X diag(l^-1/2), R = diag(l^1/2) X^H, deficient
// flags.  `work` needs 2*n*n complex when n is too large for shared memory.
// Optionally also returns the sorted eigenvalues (lam_out, n doubles) and the
// phase-fixed eigenvectors (vec_out, row-major n x n, column j = vector j).
void gram_factors(const double2* G, int n, double2* P, double2* R, int* deficient, int* any_def,
                  int* status, double2* work, cudaStream_t stream, double* lam_out = nullptr,
                  double2* vec_out = nullptr);

// Hermitian k x k eigensolver used by gram_factors / eigh_dense (process-wide):
// kEigAuto = one-warp cyclic Jacobi for k <= 6 (latency-bound sizes), else
// kEigDivideConquer = Householder tridiagonalisation + divide and conquer (the
// zheevd route); kEigJacobi = block two-sided cyclic Jacobi for every k.
enum EigSolver { kEigAuto = 0, kEigJacobi = 1, kEigDivideConquer = 2 };
int eig_solver();
void set_eig_solver(int s);

// Hermitian eigendecomposition (linalg.cpp:256-295): w descending, vec row-major
// n x n with column j = phase-fixed eigenvector j.  Same `work` rule as above.
void eigh_dense(const double2* G, int n, double* w, double2* vec, int* status, double2* work, cudaStream_t stream);

// CholeskyQR factor: G + shift*I = R^H R (R upper triangular), Rinv = R^{-1}.
// CholeskyQR factor G = R^H R; status |= kSmallCholBreakdown when a pivot
// falls below pivot_rel * max_i G_ii (or is not positive).
void chol_factors(const double2* G, int n, double pivot_rel, double2* R, double2* Rinv,
                  int* status, cudaStream_t stream);

// Batched thin SVD of small row-major matrices A_b (m x n, leading dim lda,
// batch stride sa):  A = U diag(s) Vh, k = min(m, n), s descending, U's columns
// phase-fixed (largest-magnitude entry real positive, Vh rows compensate,
// linalg.cpp:44-64).  U: m x k (stride su), s: k (stride ss), Vh: k x n (stride sv).
// One-sided (Hestenes) Jacobi; `work` (>= batch*(m*n + n*n + ...) complex, see
// small_svd_workspace) is used when the problem does not fit in shared memory.
void small_svd(const double2* A, int64_t sa, int m, int n, int lda, double2* U, int64_t su,
               double* s, int64_t ss, double2* Vh, int64_t sv, int batch, int* status,
               double2* work, cudaStream_t stream);
int64_t small_svd_workspace(int m, int n, int batch);

// R factor of a tall row-major rows x k matrix by TSQR (Householder per row
// block, binary tree over the stacked R's).  Robust to rank deficiency; used
// for the projected SVD when CholeskyQR cannot guarantee accuracy.
// `ws` must hold tsqr_workspace(rows, k) complex elements.
void tsqr_r(const double2* A, int64_t rows, int k, double2* R, double2* ws, cudaStream_t stream);
int64_t tsqr_workspace(int64_t rows, int k);

// ---- batched QR-reduced simple update (state.cpp:89-204), one colour per launch
struct SuSiteDesc {
  const double2* src;  // site tensor (phys, up, left, down, right)
  int64_t str[5];      // source strides of (env0, env1, env2, phys, shared)
  int e[3];            // env extents
  int d, s;            // phys and shared-bond extents
  int reduced;         // env >= d*s: Gram QR (state.cpp:132-140), else R = site
  double2* Q;          // E x (d*s) column-major (reduced)
  double2* R;          // reduced: (d*s) x (d*s); else E x (d*s), row-major (t, d, s)
};
struct SuBondDesc {
  const double2* gate;  // (o, p, i, j)
  const double2* Ra;
  const double2* Rb;
  int ta, tb, d, s;
  int64_t cap;  // rank cap (policy.max_rank, or d * pre_bond when 0)
  double cutoff;
  double2* t1;  // (ta, d, rank) with row stride rmax
  double2* t2;  // (tb, d, rank) with row stride rmax  [= split.t2.permute({2,1,0})]
  int rmax;
};
struct SuRestoreDesc {
  const double2* Q;
  int reduced, S;
  const double2* t;
  int rmax;
  int bond;
  int e[3];
  int d;
  double2* dst;
  int64_t dstr[5];  // destination strides of (env0, env1, env2, out-phys, new bond)
};
struct SuOneSiteDesc {
  const double2* src;
  double2* dst;
  int64_t rest;
  int d;
  const double2* gate;
};
void su_reduce(const SuSiteDesc* d_descs, int n, size_t smem, int* status, cudaStream_t stream);
// degenerate (optional): counts truncations whose cut falls inside a pair of
// singular values equal to 1e-10 relative.
void su_split(const SuBondDesc* d_descs, int n, size_t smem, int* ranks, int* status, unsigned long long* degenerate,
              cudaStream_t stream);
void su_restore(const SuRestoreDesc* d_descs, int n, const int* ranks, cudaStream_t stream);
void su_one_site(const SuOneSiteDesc* d_descs, int n, cudaStream_t stream);
// out = exp(-tau * coeff * H) for Hermitian n x n H (hermitian_function, linalg.cpp:297-314)
void herm_exp(const double2* H, int n, double coeff, double tau, double2* out, cudaStream_t stream);

// Reference complete_deficient_columns (decomposition.cpp:88-115) on a device
// rows x cols row-major Q, for the columns flagged in `deficient`; no-op when
// *any_def == 0 (checked on the device, so no host sync is needed).
void complete_columns(double2* Q, int64_t rows, int cols, const int* deficient, const int* any_def,
                      int* status, cudaStream_t stream);

}  // namespace pepsb
