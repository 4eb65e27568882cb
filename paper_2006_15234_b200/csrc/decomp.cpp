// einsumsvd on the device (see decomp.h).
//
// randomized_svd (decomposition.cpp:259-306), re-planned for B200:
//   * the sketch Omega is generated on the device by the counter-based
//     SplitMix64 stream, bit-identical to random_tensor (tensor.cpp:192-201),
//     directly in the layout the first contraction of A wants;
//   * apply / adjoint_apply run as cached contraction plans whose outputs are
//     written in each other's preferred probe layouts, so no probe is ever
//     permuted;
//   * orthogonalisation is the reference's Gram route (G = Y^H Y, eigh, clamp
//     1e-12 lambda_max, completion; decomposition.cpp:86-193) with the k x k
//     eigenproblem solved in one thread block, or CholeskyQR2 (orth_mode 1);
//   * the projected SVD of B = P^H A (linalg.cpp:87-156 wide route) is
//     CholeskyQR2 of Z = A^* P (shifted CholeskyQR3 when Z is numerically rank
//     deficient) followed by a one-sided Jacobi SVD of the k x k R^H;
//   * absorption weights and rank slicing are folded into the k x k factors,
//     and t1 / t2 are scattered straight into the reference layouts
//     (row axes..., rank) / (rank, col axes...).
#include "decomp.h"
#include "gram.cuh"

#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>

#include "smalldense.cuh"
#include "tensor_ops.cuh"
#include "zgemm.cuh"

namespace pepsb {

namespace {

bool has(const std::string& s, char c) { return s.find(c) != std::string::npos; }

int64_t prod(const std::vector<int64_t>& v) {
  int64_t n = 1;
  for (auto e : v) n *= e;
  return n;
}

// Row-major matrix product C (M x N) = op(A) op(B) with A given as M x K
// (transA: K x M) and B as K x N (transB: N x K), optional conjugation.
void mm(Ctx& ctx, double2* C, const double2* A, bool transA, bool conjA, const double2* B, bool transB,
        bool conjB, int64_t M, int64_t N, int64_t K) {
  // G = Y^H Y of a tall Y: the Hermitian Gram kernel (NB (NB/2 + 1) DMMA
  // blocks of the symmetric interleaved real product, gram.cu)
  if (A == B && transA && conjA && !transB && !conjB && M == N && gram_enabled() && gram_herk_eligible(K, M)) {
    const int64_t nd = gram_herk_workspace(K, M, ctx.num_sms);
    BufPtr work = ctx.alloc((nd + 1) / 2);
    const int NB = static_cast<int>((2 * M + 7) / 8);
    static const bool trace = getenv("PEPSB_TRACE_GEMM") != nullptr;  // one line per profiled GEMM-class record
    if (trace) fprintf(stderr, "[zgemm] gram_herk M=%ld N=%ld K=%ld NB=%d\n", (long)M, (long)N, (long)K, NB);
    {
      ProfScope ps(ctx, Ctx::kProfGemm, 8.0 * M * N * K, 16.0 * (M * K + M * N),
                   128.0 * K * (NB * (NB / 2 + 1)));
      gram_herk(A, K, static_cast<int>(M), C, reinterpret_cast<double*>(work->p), ctx.num_sms, ctx.stream);
    }
    ctx.launches += 3;
    ctx.flops += 2ull * M * N * K;
    return;
  }
  ZgemmParams p;
  p.A = A;
  p.B = B;
  p.C = C;
  p.M = M;
  p.N = N;
  p.K = K;
  p.sAi = transA ? 1 : K;
  p.sAk = transA ? M : 1;
  p.sBk = transB ? 1 : N;
  p.sBj = transB ? K : 1;
  p.conjA = conjA;
  p.conjB = conjB;
  p.nr = 1;
  p.rext[0] = M;
  p.rstr[0] = N;
  p.nc = 1;
  p.cext[0] = N;
  p.cstr[0] = 1;
  int64_t ws = zgemm_plan_splits(p, ctx.num_sms);
  BufPtr work;
  if (ws > 0) {
    work = ctx.alloc(ws);
    p.work = work->p;
  }
  {
    ProfScope ps(ctx, Ctx::kProfGemm, 8.0 * M * N * K, 16.0 * (M * K + K * N + M * N), zgemm_exec_flops(p));
    zgemm_launch(p, ctx.stream);
  }
  ctx.launches += p.splits > 1 ? 2 : 1;
  ctx.flops += 2ull * M * N * K;
}

LTensor wrap(const BufPtr& b, const std::string& labels, const std::vector<int64_t>& ext, bool conj = false) {
  LTensor l;
  l.buf = b;
  l.ptr = b->p;
  l.labels = labels;
  l.ext = ext;
  l.str = row_major_strides(ext);
  l.conj = conj;
  return l;
}

std::string unused_labels(const std::string& used, int n) {
  std::string out;
  const std::string pool = "ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789";
  for (char c : pool) {
    if ((int)out.size() == n) break;
    if (!has(used, c)) out += c;
  }
  if ((int)out.size() < n) throw Error(kShapeError, "no free label available");
  return out;
}

void read_status(Ctx& ctx) {
  PEPSB_CUDA(cudaMemcpyAsync(ctx.h_status, ctx.d_status, 2 * sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
}

// word 0: factorization status of the current stage; word 1: CholeskyQR
// breakdowns during the power iterations (orth_mode 1).
void clear_status(Ctx& ctx) { PEPSB_CUDA(cudaMemsetAsync(ctx.d_status, 0, sizeof(int), ctx.stream)); }
void clear_all_status(Ctx& ctx) { PEPSB_CUDA(cudaMemsetAsync(ctx.d_status, 0, 2 * sizeof(int), ctx.stream)); }

// Thrown when CholeskyQR met a numerically rank-deficient probe block: the
// decomposition is redone on the reference-faithful Gram-eigh route.
struct RedoFaithful {};

void raise_status(int st, bool gram_stage) {
  if (st & kSmallZeroGram) throw Error(kNumericalError, "gram orthogonalization of a zero operator");
  if (st & kSmallNotHermitian) throw Error(kValidationError, "matrix is not Hermitian within tolerance");
  if (st & kSmallCompletionExhausted) throw Error(kNumericalError, "orthonormal completion exhausted basis");
  (void)gram_stage;
}

// Gram orthogonalisation of a contiguous rows x k matrix (in place layout):
// returns Q with the same labels/layout.  decomposition.cpp:160-193.
LTensor orth(Ctx& ctx, const LTensor& Y) {
  const int64_t k = Y.ext.back();
  const int64_t rows = Y.size() / k;
  BufPtr G = ctx.alloc(k * k);
  mm(ctx, G->p, Y.ptr, true, true, Y.ptr, false, false, k, k, rows);
  BufPtr Q = ctx.alloc(rows * k);
  if (ctx.orth_mode == 1) {
    BufPtr R = ctx.alloc(k * k), Ri = ctx.alloc(k * k), G2 = ctx.alloc(k * k), Q1 = ctx.alloc(rows * k);
    {
      ProfScope ps_(ctx, Ctx::kProfSmall);
      // breakdowns are flagged in status word 1; rsvd_core then redoes the
      // decomposition on the reference-faithful route (clamp + completion)
      // pivot floor 1e-9 max_diag: flags every Gram the reference would clamp
      // (lambda < 1e-12 lambda_max implies a pivot < 1e-12 max_diag) with margin
      chol_factors(G->p, static_cast<int>(k), 1e-9, R->p, Ri->p, ctx.d_status + 1, ctx.stream);
    }
    mm(ctx, Q1->p, Y.ptr, false, false, Ri->p, false, false, rows, k, k);
    mm(ctx, G2->p, Q1->p, true, true, Q1->p, false, false, k, k, rows);
    {
      ProfScope ps_(ctx, Ctx::kProfSmall);
      chol_factors(G2->p, static_cast<int>(k), 0.0, R->p, Ri->p, ctx.d_status + 1, ctx.stream);
    }
    mm(ctx, Q->p, Q1->p, false, false, Ri->p, false, false, rows, k, k);
    ctx.launches += 2;
  } else {
    BufPtr P = ctx.alloc(k * k), R = ctx.alloc(k * k), def = ctx.alloc((k + 2 + 1) / 2 + 1);
    int* d_def = reinterpret_cast<int*>(def->p);
    int* d_any = d_def + k;
    BufPtr work;
    if (2 * k * (k + 1) * 16 > 176 * 1024) work = ctx.alloc(2 * k * (k + 1));
    {
      ProfScope ps_(ctx, Ctx::kProfSmall);
      gram_factors(G->p, static_cast<int>(k), P->p, R->p, d_def, d_any, ctx.d_status, work ? work->p : nullptr,
                   ctx.stream);
    }
    if (ctx.trace) {
      int sw = 0;
      ctx.sync();
      PEPSB_CUDA(cudaMemcpy(&sw, ctx.d_status + 7, sizeof(int), cudaMemcpyDeviceToHost));
      PEPSB_CUDA(cudaMemset(ctx.d_status + 7, 0, sizeof(int)));
      fprintf(stderr, "[pepsb] orth rows=%ld k=%ld sweeps=%d\n", (long)rows, (long)k, sw);
      static int dumped = 0;
      if (sw >= 12 && getenv("PEPSB_DUMP_GRAM") && dumped < 4) {  // developer aid: slow-converging Grams
        std::vector<double2> h(static_cast<size_t>(k * k));
        PEPSB_CUDA(cudaMemcpy(h.data(), G->p, h.size() * sizeof(double2), cudaMemcpyDeviceToHost));
        const std::string fn = std::string(getenv("PEPSB_DUMP_GRAM")) + std::to_string(dumped++) + ".bin";
        if (FILE* f = fopen(fn.c_str(), "wb")) {
          fwrite(h.data(), sizeof(double2), h.size(), f);
          fclose(f);
        }
      }
    }
    mm(ctx, Q->p, Y.ptr, false, Y.conj, P->p, false, false, rows, k, k);
    {
      ProfScope ps_(ctx, Ctx::kProfSmall);
      complete_columns(Q->p, rows, static_cast<int>(k), d_def, d_any, ctx.d_status, ctx.stream);
    }
    ctx.launches += 2;
  }
  LTensor out = Y;
  out.buf = Q;
  out.ptr = Q->p;
  out.conj = false;
  out.str = row_major_strides(out.ext);
  return out;
}

// Fork the side stream after the Gram GEMM rather than before it: the side
// stream's operator application then becomes ready together with the
// eigensolver, and the main stream's higher priority dispatches the
// eigensolver's block first instead of behind the whole application grid
// (its 214 KB of shared memory cannot co-reside with a GEMM CTA).
// PEPSB_FORK_AFTER_GRAM=0 forks before the Gram GEMM.
bool fork_after_gram() {
  static const bool v = [] {
    const char* e = getenv("PEPSB_FORK_AFTER_GRAM");
    return !(e && e[0] == '0');
  }();
  return v;
}

// apply(orth(Z)) for the big-side orthogonalisation of a power iteration,
// with the k x k eigensolver hidden behind the operator application: by
// linearity A (Z P) = (A Z) P, so A Z runs on the side stream while the Gram
// matrix and its eigendecomposition run on the main stream, and only the
// small (rows_Y x k) product (A Z) P follows.  This also skips the big
// Q = Z P product.  When the Gram matrix is deficient (columns clamped and
// completed, decomposition.cpp:86-117) the completed basis is not of the form
// Z P: the speculative A Z is discarded and A (orth(Z)) is formed as usual.
// Rounding differs from A (Z P) at the level eps ||A|| ||Z|| ||P||.
template <class ApplyFn>
LTensor apply_orth_speculative(Ctx& ctx, const LTensor& Z, ApplyFn&& apply) {
  const int64_t k = Z.ext.back();
  const int64_t rows = Z.size() / k;
  const bool late = fork_after_gram();
  if (!late) ctx.fork();
  BufPtr G = ctx.alloc(k * k);
  mm(ctx, G->p, Z.ptr, true, true, Z.ptr, false, false, k, k, rows);
  if (late) ctx.fork();
  BufPtr P = ctx.alloc(k * k), R = ctx.alloc(k * k), def = ctx.alloc((k + 2 + 1) / 2 + 1);
  int* d_def = reinterpret_cast<int*>(def->p);
  int* d_any = d_def + k;
  BufPtr work;
  if (2 * k * (k + 1) * 16 > 176 * 1024) work = ctx.alloc(2 * k * (k + 1));
  {
    ProfScope ps_(ctx, Ctx::kProfSmall);
    gram_factors(G->p, static_cast<int>(k), P->p, R->p, d_def, d_any, ctx.d_status, work ? work->p : nullptr,
                 ctx.stream);
  }
  ++ctx.launches;
  PEPSB_CUDA(cudaMemcpyAsync(ctx.h_status + 16, d_any, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  cudaEvent_t eig_done = ctx.take_event();
  PEPSB_CUDA(cudaEventRecord(eig_done, ctx.stream));
  ctx.side();
  LTensor AZ = apply(Z);
  ctx.join();
  {
    HostTimer ht(ctx.trace ? &ctx.t_sync : nullptr);
    PEPSB_CUDA(cudaEventSynchronize(eig_done));
  }
  ctx.event_pool.push_back(eig_done);
  if (ctx.h_status[16] == 0) {
    const int64_t ry = AZ.size() / k;
    BufPtr Y = ctx.alloc(ry * k);
    mm(ctx, Y->p, AZ.ptr, false, AZ.conj, P->p, false, false, ry, k, k);
    LTensor out = AZ;
    out.buf = Y;
    out.ptr = Y->p;
    out.conj = false;
    out.str = row_major_strides(out.ext);
    return out;
  }
  // deficient Gram: the reference's completed basis, then the plain application
  BufPtr Q = ctx.alloc(rows * k);
  mm(ctx, Q->p, Z.ptr, false, Z.conj, P->p, false, false, rows, k, k);
  {
    ProfScope ps_(ctx, Ctx::kProfSmall);
    complete_columns(Q->p, rows, static_cast<int>(k), d_def, d_any, ctx.d_status, ctx.stream);
  }
  ++ctx.launches;
  LTensor q = Z;
  q.buf = Q;
  q.ptr = Q->p;
  q.conj = false;
  q.str = row_major_strides(q.ext);
  return apply(q);
}

// adjoint(orth(Y)) for the small-side orthogonalisation of a power
// iteration, with the k x k eigensolver hidden behind the first pairwise step
// of the adjoint chain: that step is linear in the probe, so it runs on Y
// itself on the side stream while the Gram matrix and its eigendecomposition
// run on the main stream, and its (small) result is then multiplied by the
// k x k factor P = X Lambda^-1/2 before the rest of the chain continues.  The
// explicit basis orth(Y) = Y P is returned in *p_out (cheap: rows_Y x k x k).
// Deficient Gram matrices (completed columns) fall back to the plain route.
LTensor adjoint_orth_speculative(Ctx& ctx, const LTensor& Y, ContractionPlan& plan_adj,
                                 std::vector<LTensor>& leaves_adj, LTensor* p_out) {
  const int64_t k = Y.ext.back();
  const int64_t rows = Y.size() / k;
  const int probe_leaf = static_cast<int>(leaves_adj.size()) - 1;
  const int node = plan_adj.parent_of_leaf(probe_leaf);
  auto plain = [&]() {
    *p_out = orth(ctx, Y);
    leaves_adj.back() = *p_out;
    return plan_adj.execute(ctx, leaves_adj);
  };
  if (node < 0) return plain();
  const bool late = fork_after_gram();
  if (!late) ctx.fork();
  BufPtr G = ctx.alloc(k * k);
  mm(ctx, G->p, Y.ptr, true, true, Y.ptr, false, false, k, k, rows);
  if (late) ctx.fork();
  BufPtr P = ctx.alloc(k * k), R = ctx.alloc(k * k), def = ctx.alloc((k + 2 + 1) / 2 + 1);
  int* d_def = reinterpret_cast<int*>(def->p);
  int* d_any = d_def + k;
  BufPtr work;
  if (2 * k * (k + 1) * 16 > 176 * 1024) work = ctx.alloc(2 * k * (k + 1));
  {
    ProfScope ps_(ctx, Ctx::kProfSmall);
    gram_factors(G->p, static_cast<int>(k), P->p, R->p, d_def, d_any, ctx.d_status, work ? work->p : nullptr,
                 ctx.stream);
  }
  ++ctx.launches;
  PEPSB_CUDA(cudaMemcpyAsync(ctx.h_status + 17, d_any, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  cudaEvent_t eig_done = ctx.take_event();
  PEPSB_CUDA(cudaEventRecord(eig_done, ctx.stream));
  ctx.side();
  leaves_adj.back() = Y;
  LTensor T1 = plan_adj.run_node(ctx, node, leaves_adj);
  ctx.join();
  {
    HostTimer ht(ctx.trace ? &ctx.t_sync : nullptr);
    PEPSB_CUDA(cudaEventSynchronize(eig_done));
  }
  ctx.event_pool.push_back(eig_done);
  // explicit basis Q = Y P (+ the reference's completion when deficient)
  BufPtr Q = ctx.alloc(rows * k);
  mm(ctx, Q->p, Y.ptr, false, Y.conj, P->p, false, false, rows, k, k);
  const bool deficient = ctx.h_status[17] != 0;
  if (deficient) {
    {
      ProfScope ps_(ctx, Ctx::kProfSmall);
      complete_columns(Q->p, rows, static_cast<int>(k), d_def, d_any, ctx.d_status, ctx.stream);
    }
    ++ctx.launches;
  }
  LTensor q = Y;
  q.buf = Q;
  q.ptr = Q->p;
  q.conj = false;
  q.str = row_major_strides(q.ext);
  *p_out = q;
  leaves_adj.back() = q;
  if (deficient) return plan_adj.execute(ctx, leaves_adj);
  // T1 (.., X, ..) x P(X, X') -> relabel X' as X
  const char X = Y.labels.back();
  std::string used = T1.labels;
  for (const auto& l : leaves_adj) used += l.labels;
  const char Xp = unused_labels(used, 1)[0];
  std::string out_order = T1.labels;
  std::replace(out_order.begin(), out_order.end(), X, Xp);
  LTensor T1p = pairwise_gemm(ctx, T1, wrap(P, std::string{X, Xp}, {k, k}), "", std::string(1, X), out_order);
  std::replace(T1p.labels.begin(), T1p.labels.end(), Xp, X);
  return plan_adj.execute_subst(ctx, leaves_adj, node, T1p);
}

struct Projected {
  BufPtr Ut;  // k x k left singular vectors of B = P^H A (phase-fixed)
  std::vector<double> s;
  bool tsqr = false;  // accurate fallback used
};

// SVD of B = Z^H (Z: rows x k contiguous) through an R factor of Z
// (B = R^H Q^H, so B's singular values / left vectors are R^H's):
//   CholeskyQR2 R when it is provably accurate (no breakdown and the first
//   `target` singular values above 1e-7 sigma_0, i.e. kappa < u^-1/2);
//   otherwise the Householder TSQR R (backward stable like the reference's
//   zgeqrf route, linalg.cpp:87-125, incl. exactly rank-deficient Z).
Projected projected_svd(Ctx& ctx, const LTensor& Z, int64_t target) {
  const int64_t k = Z.ext.back();
  const int64_t rows = Z.size() / k;
  const int ki = static_cast<int>(k);
  Projected out;
  out.Ut = ctx.alloc(k * k);
  BufPtr Wh = ctx.alloc(k * k);
  BufPtr sdev = ctx.alloc((k + 1) / 2 + 1);
  double* d_s = reinterpret_cast<double*>(sdev->p);
  BufPtr svd_work;
  if (int64_t ws = small_svd_workspace(ki, ki, 1)) svd_work = ctx.alloc(ws);
  auto svd_of_rh = [&](const BufPtr& R) {
    LTensor Rh = reduce_to(ctx, wrap(R, "ab", {k, k}, true), "ba");
    {
      ProfScope ps_(ctx, Ctx::kProfSmall);
      small_svd(Rh.ptr, 0, ki, ki, ki, out.Ut->p, 0, d_s, 0, Wh->p, 0, 1, ctx.d_status,
                svd_work ? svd_work->p : nullptr, ctx.stream);
    }
    ++ctx.launches;
    out.s.resize(k);
    PEPSB_CUDA(cudaMemcpyAsync(out.s.data(), d_s, k * sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    read_status(ctx);
    ctx.sync_main();
    return *ctx.h_status;
  };
  auto gram = [&](const double2* X) {
    BufPtr G = ctx.alloc(k * k);
    mm(ctx, G->p, X, true, true, X, false, false, k, k, rows);
    return G;
  };
  bool ok = false;
  const int64_t tgt = std::max<int64_t>(1, std::min<int64_t>(target, k));
  BufPtr G1;
  if (rows >= k) {
    // Stage 1: eigendecomposition of G1 = Z^H Z = B B^H gives B's left singular
    // vectors and sigma^2 directly.  Accepted when the retained part of the
    // spectrum is well inside the Gram route's accuracy (sigma_{target-1} >=
    // 1e-4 sigma_0: relative error of the kept sigma_j <= eps (s0/sj)^2 ~ 1e-8).
    G1 = gram(Z.ptr);
    BufPtr P = ctx.alloc(k * k), R = ctx.alloc(k * k), def = ctx.alloc(k / 4 + 2);
    int* d_def = reinterpret_cast<int*>(def->p);
    BufPtr work;
    if (2 * k * (k + 1) * 16 > 176 * 1024) work = ctx.alloc(2 * k * (k + 1));
    {
      ProfScope ps_(ctx, Ctx::kProfSmall);
      gram_factors(G1->p, ki, P->p, R->p, d_def, d_def + k, ctx.d_status, work ? work->p : nullptr, ctx.stream,
                   d_s, out.Ut->p);
    }
    ++ctx.launches;
    std::vector<double> lam(k);
    PEPSB_CUDA(cudaMemcpyAsync(lam.data(), d_s, k * sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    read_status(ctx);
    ctx.sync_main();
    const int st = *ctx.h_status & ~kSmallZeroGram;  // a zero Z is judged below
    raise_status(st, false);
    out.s.resize(k);
    for (int64_t j = 0; j < k; ++j) out.s[j] = std::sqrt(std::max(lam[j], 0.0));
    ok = out.s[0] > 0.0 && out.s[tgt - 1] >= 1e-4 * out.s[0];
    clear_status(ctx);
  }
  if (!ok && rows >= k) {
    BufPtr R1 = ctx.alloc(k * k), R1i = ctx.alloc(k * k);
    {
      ProfScope ps_(ctx, Ctx::kProfSmall);
      chol_factors(G1->p, ki, 0.0, R1->p, R1i->p, ctx.d_status, ctx.stream);
    }
    BufPtr Q1 = ctx.alloc(rows * k);
    mm(ctx, Q1->p, Z.ptr, false, false, R1i->p, false, false, rows, k, k);
    BufPtr G2 = gram(Q1->p);
    BufPtr R2 = ctx.alloc(k * k), R2i = ctx.alloc(k * k), R = ctx.alloc(k * k);
    {
      ProfScope ps_(ctx, Ctx::kProfSmall);
      chol_factors(G2->p, ki, 0.0, R2->p, R2i->p, ctx.d_status, ctx.stream);
    }
    ctx.launches += 2;
    mm(ctx, R->p, R2->p, false, false, R1->p, false, false, k, k, k);
    const int st = svd_of_rh(R);
    raise_status(st, false);
    ok = !(st & kSmallCholBreakdown) && out.s[0] > 0.0 && out.s[tgt - 1] >= 1e-7 * out.s[0];
    clear_status(ctx);
  }
  if (!ok) {
    BufPtr R = ctx.alloc(k * k);
    BufPtr ws = ctx.alloc(tsqr_workspace(rows, ki));
    {
      ProfScope ps_(ctx, Ctx::kProfSmall);
      tsqr_r(Z.ptr, rows, ki, R->p, ws->p, ctx.stream);
    }
    ++ctx.launches;
    const int st = svd_of_rh(R);
    raise_status(st, false);
    out.tsqr = true;
    ++ctx.tsqr_fallbacks;
  }
  return out;
}

BufPtr upload_doubles(Ctx& ctx, const std::vector<double>& w) {
  BufPtr b = ctx.alloc((static_cast<int64_t>(w.size()) + 1) / 2 + 1);
  PEPSB_CUDA(cudaMemcpyAsync(b->p, w.data(), w.size() * sizeof(double), cudaMemcpyHostToDevice, ctx.stream));
  return b;
}

void absorb_weights(const std::vector<double>& s, int absorb, std::vector<double>& wl, std::vector<double>& wr) {
  wl.assign(s.size(), 1.0);
  wr.assign(s.size(), 1.0);
  for (size_t i = 0; i < s.size(); ++i) {
    if (absorb == kSplit) wl[i] = wr[i] = std::sqrt(s[i]);
    else if (absorb == kLeft) wl[i] = s[i];
    else if (absorb == kRight) wr[i] = s[i];
  }
}

struct RsvdPlans {
  std::shared_ptr<ContractionPlan> ap, adj;
};

// The apply / adjoint plans of an implicit operator with `probe` probe
// columns under label X; each writes its output in the layout the other
// consumes (decomposition.cpp:259-306 lowered).
RsvdPlans build_plans(const ImplicitOp& op, int64_t probe, char X) {
  const size_t nt = op.tensors.size();
  std::vector<LeafMeta> meta_ap, meta_adj;
  for (size_t i = 0; i < nt; ++i) {
    meta_ap.push_back({op.labels[i], op.tensors[i].shape});
    meta_adj.push_back({op.labels[i], op.tensors[i].shape});
  }
  std::vector<int64_t> qshape = op.col_shape(), pshape = op.row_shape();
  qshape.push_back(probe);
  pshape.push_back(probe);
  meta_ap.push_back({op.cols + X, qshape});
  meta_adj.push_back({op.rows + X, pshape});
  RsvdPlans pl;
  pl.ap = std::make_shared<ContractionPlan>(meta_ap, op.rows + X, static_cast<int>(nt), X);
  pl.adj = std::make_shared<ContractionPlan>(meta_adj, op.cols + X, static_cast<int>(nt), X);
  pl.ap->finalize(pl.adj->flexible_order());
  pl.adj->finalize(pl.ap->flexible_order());
  pl.ap->cache_static = pl.adj->cache_static = true;
  return pl;
}

// Omega = random_tensor(col_shape + [probe], seed) (decomposition.cpp:267-270)
// generated directly in the probe layout the apply plan wants.
LTensor make_sketch(Ctx& ctx, const ImplicitOp& op, const ContractionPlan& plan_ap, int64_t probe, char X,
                    uint64_t seed) {
  std::vector<int64_t> qshape = op.col_shape();
  qshape.push_back(probe);
  const std::string qord = plan_ap.flexible_order();
  std::vector<int64_t> pext, lstr;
  const std::string logical = op.cols + X;
  const std::vector<int64_t> lst = row_major_strides(qshape);
  for (char c : qord) {
    auto pos = logical.find(c);
    pext.push_back(qshape[pos]);
    lstr.push_back(lst[pos]);
  }
  BufPtr om = ctx.alloc(prod(qshape));
  random_fill(om->p, static_cast<int>(qord.size()), pext.data(), lstr.data(), seed, 0, ctx.stream);
  ++ctx.launches;
  return wrap(om, qord, pext);
}

int64_t probe_count(const ImplicitOp& op, const Trunc& policy, const Rsvd& cfg) {
  const int64_t mindim = std::min(op.row_extent(), op.col_extent());
  const int64_t target = static_cast<int64_t>(std::min<uint64_t>(policy.max_rank, static_cast<uint64_t>(mindim)));
  return std::min<int64_t>(target + static_cast<int64_t>(effective_oversample(cfg, target)), mindim);
}

// Work started for a column on the side stream by the previous column.
struct Prefetched {
  std::vector<std::vector<int64_t>> shapes;  // leaf shapes assumed (leaf 0: the guessed pending tensor)
  std::vector<std::string> labels;
  std::string rows, cols;
  uint64_t seed = 0;
  int64_t probe = 0;
  RsvdPlans plans;
  LTensor omega, prefix;
  bool matches(const ImplicitOp& op, uint64_t sd, int64_t pr) const {
    if (sd != seed || pr != probe || op.rows != rows || op.cols != cols || op.labels != labels) return false;
    if (op.tensors.size() != shapes.size()) return false;
    for (size_t i = 0; i < shapes.size(); ++i)
      if (op.tensors[i].shape != shapes[i]) return false;
    return true;
  }
};

void launch_lookahead(Ctx& ctx, const Lookahead& la, const Trunc& policy, const Rsvd& cfg) {
  const ImplicitOp& op = la.op;
  Rsvd c2 = cfg;
  c2.seed = la.seed;
  const int64_t probe = probe_count(op, policy, c2);
  const char X = op.fresh_label();
  auto pf = std::make_shared<Prefetched>();
  for (const auto& t : op.tensors) pf->shapes.push_back(t.shape);
  pf->labels = op.labels;
  pf->rows = op.rows;
  pf->cols = op.cols;
  pf->seed = la.seed;
  pf->probe = probe;
  pf->plans = build_plans(op, probe, X);
  ctx.fork();
  ctx.side();
  pf->omega = make_sketch(ctx, op, *pf->plans.ap, probe, X, la.seed);
  std::vector<LTensor> leaves;
  for (size_t i = 0; i < op.tensors.size(); ++i) leaves.push_back(as_labelled(op.tensors[i], op.labels[i], op.conj[i]));
  leaves.push_back(pf->omega);
  pf->prefix = pf->plans.ap->run_prefix(ctx, leaves, 0);
  ctx.back();
  ctx.prefetched = pf;
}

// Core of randomized_svd / einsumsvd(implicit_rsvd).  Weights (absorb) are
// applied when `absorb` >= 0, otherwise plain U, S, V are returned.
EinsumsvdResultD rsvd_core(Ctx& ctx, const ImplicitOp& op, const Trunc& policy, const Rsvd& cfg, int absorb,
                           const std::vector<int>& t1_perm) {
  if (policy.max_rank < 1) throw Error(kValidationError, "randomized svd needs target rank >= 1");
  const int64_t mindim = std::min(op.row_extent(), op.col_extent());
  const int64_t target = static_cast<int64_t>(std::min<uint64_t>(policy.max_rank, static_cast<uint64_t>(mindim)));
  const bool clamped = policy.max_rank > static_cast<uint64_t>(mindim);
  const int64_t probe = std::min<int64_t>(target + static_cast<int64_t>(effective_oversample(cfg, target)), mindim);
  const char X = op.fresh_label();
  std::string used = op.rows + op.cols + X;
  for (auto& l : op.labels) used += l;
  const std::string extra = unused_labels(used, 2);
  const char RK = extra[0];

  const size_t nt = op.tensors.size();
  // Plans and sketch: built here, or taken over from the previous column of a
  // row absorb, which started them (and the v-independent prefix of the first
  // application) on the side stream during its own tail (row lookahead).
  std::shared_ptr<Prefetched> pre = std::static_pointer_cast<Prefetched>(ctx.prefetched);
  ctx.prefetched.reset();
  ctx.join_pending();
  const bool reuse = pre && pre->matches(op, cfg.seed, probe);
  if (pre && !reuse) ++ctx.lookahead_misses;
  RsvdPlans plans = reuse ? pre->plans : build_plans(op, probe, X);
  ContractionPlan& plan_ap = *plans.ap;
  ContractionPlan& plan_adj = *plans.adj;
  std::vector<LTensor> leaves_ap, leaves_adj;
  for (size_t i = 0; i < nt; ++i) {
    leaves_ap.push_back(as_labelled(op.tensors[i], op.labels[i], op.conj[i]));
    leaves_adj.push_back(as_labelled(op.tensors[i], op.labels[i], !op.conj[i]));
  }
  leaves_ap.push_back(LTensor());
  leaves_adj.push_back(LTensor());
  LTensor q = reuse ? pre->omega : make_sketch(ctx, op, plan_ap, probe, X, cfg.seed);
  LTensor prefix = reuse ? pre->prefix : LTensor();
  pre.reset();
  clear_all_status(ctx);

  auto apply = [&](const LTensor& qq) {
    leaves_ap.back() = qq;
    return plan_ap.execute(ctx, leaves_ap);
  };
  auto adjoint = [&](const LTensor& pp) {
    leaves_adj.back() = pp;
    return plan_adj.execute(ctx, leaves_adj);
  };

  static const bool trace = getenv("PEPSB_TRACE") != nullptr;
  auto now = [] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  const double tr0 = trace ? now() : 0.0;
  LTensor y;
  if (prefix.buf) {
    leaves_ap.back() = q;
    y = plan_ap.execute_with_prefix(ctx, leaves_ap, 0, prefix);
    prefix = LTensor();
  } else {
    y = apply(q);
  }
  // (small problems: the host syncs on the eigensolver would cost more than they
  // hide; measured: forcing it on every call costs config 1 4.4 -> 5.1 ms per
  // norm, while the last column of a config-2 row -- 4096 x 64, column extent
  // below 2^15 -- gains: row 61.9 -> 60.9 ms, so operators of >= 2^18 entries
  // qualify too)
  const bool big = op.col_extent() >= (1 << 15) || op.row_extent() * op.col_extent() >= (int64_t{1} << 18);
  const bool overlap = ctx.orth_mode == 0 && (ctx.overlap == 2 || (ctx.overlap == 1 && big));
  LTensor p, z;
  for (int i = 0; i <= cfg.power_iters; ++i) {
    // z = A^* orth(y), p = orth(y)
    if (overlap) {
      z = adjoint_orth_speculative(ctx, y, plan_adj, leaves_adj, &p);
    } else {
      p = orth(ctx, y);
      z = adjoint(p);
    }
    if (i == cfg.power_iters) break;
    // y = A orth(z)
    y = overlap ? apply_orth_speculative(ctx, z, apply) : apply(orth(ctx, z));
  }
  y = LTensor();
  q = LTensor();
  // Row lookahead: start the next column's sketch and the v-independent
  // prefix of its first application on the side stream; they run during this
  // column's projected SVD (a one-block eigensolver plus a host sync).
  if (std::shared_ptr<Lookahead> la = std::static_pointer_cast<Lookahead>(ctx.lookahead)) {
    ctx.lookahead.reset();
    if (ctx.orth_mode == 0 && ctx.overlap != 0) launch_lookahead(ctx, *la, policy, cfg);
  }
  const double tr1 = trace ? now() : 0.0;
  if (trace) {
    ctx.sync();
    fprintf(stderr, "[pepsb] rsvd enqueue %.3f ms, drain %.3f ms\n", tr1 - tr0, now() - tr1);
  }
  const double tr2 = trace ? now() : 0.0;
  Projected pr = projected_svd(ctx, z, target);
  if (trace) fprintf(stderr, "[pepsb] projected_svd %.3f ms (tsqr %d)\n", now() - tr2, pr.tsqr ? 1 : 0);
  if (ctx.orth_mode == 1 && (ctx.h_status[1] & kSmallCholBreakdown)) {
    ++ctx.faithful_redos;
    throw RedoFaithful{};
  }

  Trunc pol = policy;
  int64_t rank = static_cast<int64_t>(retained_rank(pr.s, pol));
  rank = std::min(rank, target);
  std::vector<double> s(pr.s.begin(), pr.s.begin() + rank);
  std::vector<double> wl, wr;
  if (absorb >= 0) absorb_weights(s, absorb, wl, wr);
  else {
    wl.assign(rank, 1.0);
    wr.assign(rank, 1.0);
  }
  // V_j = Z u_j / s_j  (B = Z^H = U S V^H), so t2 = diag(wr) V^H = conj(Z conj(Mc)) with
  // Mc = conj(U[:, :rank]) diag(wr / s).
  std::vector<double> wv(rank);
  for (int64_t j = 0; j < rank; ++j) wv[j] = s[j] > 0.0 ? wr[j] / s[j] : 0.0;
  BufPtr dwl = upload_doubles(ctx, wl), dwv = upload_doubles(ctx, wv);
  const int64_t k = probe;
  BufPtr Uw = ctx.alloc(k * rank), Mcb = ctx.alloc(k * rank);
  slice_scale_cols(Uw->p, pr.Ut->p, k, rank, k, reinterpret_cast<double*>(dwl->p), 0, ctx.stream);
  slice_scale_cols(Mcb->p, pr.Ut->p, k, rank, k, reinterpret_cast<double*>(dwv->p), 1, ctx.stream);
  ctx.launches += 2;
  LTensor Mc = wrap(Mcb, std::string(1, X) + RK, {k, rank});
  // t1 = P Uw -> (row axes..., rank);  t2 = conj(Z) Mc -> (rank, col axes...)
  std::string t1_order = op.rows + RK;
  if (!t1_perm.empty()) {
    std::string o;
    for (int a : t1_perm) o += t1_order[a];
    t1_order = o;
  }
  LTensor t1 = pairwise_gemm(ctx, p, wrap(Uw, std::string(1, X) + RK, {k, rank}), "", std::string(1, X),
                             t1_order);
  LTensor t2 = pairwise_gemm(ctx, [&] { LTensor zc = z; zc.conj = true; return zc; }(), Mc, "",
                             std::string(1, X), std::string(1, RK) + op.cols);
  EinsumsvdResultD out;
  out.t1.buf = t1.buf;
  out.t1.shape = t1.ext;
  out.t2.buf = t2.buf;
  out.t2.shape = t2.ext;
  out.s = s;
  out.rank_clamped = clamped;
  return out;
}

}  // namespace

// ---------------------------------------------------------------------------- ImplicitOp

ImplicitOp::ImplicitOp(std::vector<DTensor> t, std::vector<std::string> l, std::string r, std::string c,
                       std::vector<bool> cj)
    : tensors(std::move(t)), labels(std::move(l)), rows(std::move(r)), cols(std::move(c)), conj(std::move(cj)) {
  if (conj.empty()) conj.assign(tensors.size(), false);
  if (tensors.size() != labels.size() || conj.size() != tensors.size())
    throw Error(kShapeError, "one label string per tensor required");
  std::map<char, int64_t> ext;
  std::map<char, int> count;
  for (size_t i = 0; i < tensors.size(); ++i) {
    if (labels[i].size() != tensors[i].shape.size())
      throw Error(kShapeError, "label string '" + labels[i] + "' does not match tensor order");
    for (size_t a = 0; a < labels[i].size(); ++a) {
      char ch = labels[i][a];
      auto [it, ins] = ext.emplace(ch, tensors[i].shape[a]);
      if (!ins && it->second != tensors[i].shape[a])
        throw Error(kShapeError, std::string("extent mismatch on label '") + ch + "'");
      ++count[ch];
    }
  }
  for (char ch : rows)
    if (has(cols, ch)) throw Error(kShapeError, std::string("label '") + ch + "' in both row and column groups");
  auto check_open = [&](const std::string& g) {
    for (char ch : g) {
      auto it = count.find(ch);
      if (it == count.end() || it->second != 1)
        throw Error(kShapeError, std::string("open label '") + ch + "' must appear exactly once");
    }
  };
  check_open(rows);
  check_open(cols);
  for (char ch : rows) row_shape_.push_back(ext[ch]);
  for (char ch : cols) col_shape_.push_back(ext[ch]);
}

int64_t ImplicitOp::row_extent() const { return prod(row_shape_); }
int64_t ImplicitOp::col_extent() const { return prod(col_shape_); }

char ImplicitOp::fresh_label() const {
  std::string used = rows + cols;
  for (auto& l : labels) used += l;
  for (char ch = 'A'; ch <= 'Z'; ++ch)
    if (!has(used, ch)) return ch;
  for (char ch = 'a'; ch <= 'z'; ++ch)
    if (!has(used, ch)) return ch;
  throw Error(kShapeError, "no free label available");
}

DTensor implicit_apply(Ctx& ctx, const ImplicitOp& op, const DTensor& q, bool adjoint) {
  const auto& shp = adjoint ? op.row_shape() : op.col_shape();
  if (q.shape.size() != shp.size() + 1)
    throw Error(kShapeError, adjoint ? "probe order must be row order + 1" : "probe order must be column order + 1");
  for (size_t a = 0; a < shp.size(); ++a)
    if (q.shape[a] != shp[a])
      throw Error(kShapeError, std::string("probe shape mismatch on ") + (adjoint ? "row" : "column") + " axis " +
                                   std::to_string(a));
  const char f = op.fresh_label();
  std::vector<LTensor> leaves;
  for (size_t i = 0; i < op.tensors.size(); ++i)
    leaves.push_back(as_labelled(op.tensors[i], op.labels[i], adjoint ? !op.conj[i] : op.conj[i]));
  leaves.push_back(as_labelled(q, (adjoint ? op.rows : op.cols) + f));
  LTensor r = contract_network(ctx, leaves, (adjoint ? op.cols : op.rows) + f);
  return materialize(ctx, r, r.labels);
}

DTensor implicit_materialize(Ctx& ctx, const ImplicitOp& op) {
  std::vector<LTensor> leaves;
  for (size_t i = 0; i < op.tensors.size(); ++i) leaves.push_back(as_labelled(op.tensors[i], op.labels[i], op.conj[i]));
  LTensor r = contract_network(ctx, leaves, op.rows + op.cols);
  return materialize(ctx, r, r.labels);
}

// ---------------------------------------------------------------------------- public

size_t effective_oversample(const Rsvd& cfg, size_t target) {
  if (cfg.oversample >= 0) return static_cast<size_t>(cfg.oversample);
  return std::max<size_t>(5, static_cast<size_t>(std::ceil(0.1 * static_cast<double>(target))));
}

size_t retained_rank(const std::vector<double>& s, const Trunc& policy) {
  if (s.empty()) return 0;
  const double floor = policy.rel_cutoff * s[0];
  size_t above = 0;
  for (double v : s)
    if (v >= floor) ++above;
  const size_t cap = policy.max_rank == 0 ? s.size() : static_cast<size_t>(std::min<uint64_t>(policy.max_rank, SIZE_MAX));
  return std::max<size_t>(1, std::min(above, cap));
}

std::pair<DTensor, DTensor> gram_orthogonalize(Ctx& ctx, const DTensor& a, int split) {
  const int order = static_cast<int>(a.shape.size());
  if (split < 1 || split >= order) throw Error(kShapeError, "gram split must satisfy 1 <= split < order");
  std::vector<int64_t> rs(a.shape.begin(), a.shape.begin() + split), cs(a.shape.begin() + split, a.shape.end());
  const int64_t rows = prod(rs), cols = prod(cs);
  if (rows < cols) throw Error(kShapeError, "gram orthogonalization needs row extent >= col extent");
  if (cols > 256) throw Error(kShapeError, "gram orthogonalization: col extent > 256 not supported on device");
  clear_status(ctx);
  BufPtr G = ctx.alloc(cols * cols);
  mm(ctx, G->p, a.data(), true, true, a.data(), false, false, cols, cols, rows);
  BufPtr P = ctx.alloc(cols * cols), def = ctx.alloc(cols / 2 + 2);
  int* d_def = reinterpret_cast<int*>(def->p);
  int* d_any = d_def + cols;
  BufPtr work;
  if (2 * cols * (cols + 1) * 16 > 176 * 1024) work = ctx.alloc(2 * cols * (cols + 1));
  DTensor R;
  std::vector<int64_t> rshape = cs;
  rshape.insert(rshape.end(), cs.begin(), cs.end());
  R.shape = rshape;
  R.buf = ctx.alloc(cols * cols);
  {
    ProfScope ps_(ctx, Ctx::kProfSmall);
    gram_factors(G->p, static_cast<int>(cols), P->p, R.data(), d_def, d_any, ctx.d_status, work ? work->p : nullptr,
                 ctx.stream);
  }
  DTensor Q;
  std::vector<int64_t> qshape = rs;
  qshape.insert(qshape.end(), cs.begin(), cs.end());
  Q.shape = qshape;
  Q.buf = ctx.alloc(rows * cols);
  mm(ctx, Q.data(), a.data(), false, false, P->p, false, false, rows, cols, cols);
  {
    ProfScope ps_(ctx, Ctx::kProfSmall);
    complete_columns(Q.data(), rows, static_cast<int>(cols), d_def, d_any, ctx.d_status, ctx.stream);
  }
  ctx.launches += 2;
  read_status(ctx);
  ctx.sync();
  raise_status(*ctx.h_status, true);
  return {Q, R};
}

// ---------------------------------------------------------------------------- sharded-driver blocks

DTensor orth_async(Ctx& ctx, const DTensor& y) {
  std::string lab;
  for (size_t i = 0; i < y.shape.size(); ++i) lab += static_cast<char>('a' + i);
  LTensor q = orth(ctx, as_labelled(y, lab));
  DTensor out;
  out.buf = q.buf;
  out.shape = q.ext;
  return out;
}

GramFactorsAsync gram_factors_async(Ctx& ctx, const DTensor& g) {
  if (g.shape.size() != 2 || g.shape[0] != g.shape[1]) throw Error(kShapeError, "gram_factors needs k x k");
  const int64_t k = g.shape[0];
  if (k < 1 || k > 256) throw Error(kShapeError, "gram_factors: 1 <= k <= 256");
  GramFactorsAsync out;
  out.P = ctx.empty({k, k});
  BufPtr R = ctx.alloc(k * k), work;
  out.flags = ctx.alloc(k / 4 + 2);
  if (2 * k * (k + 1) * 16 > 176 * 1024) work = ctx.alloc(2 * k * (k + 1));
  int* d_def = reinterpret_cast<int*>(out.flags->p);
  {
    ProfScope ps_(ctx, Ctx::kProfSmall);
    gram_factors(g.data(), static_cast<int>(k), out.P.data(), R->p, d_def, d_def + k, ctx.d_status,
                 work ? work->p : nullptr, ctx.stream);
  }
  ++ctx.launches;
  out.any_deficient = d_def + k;
  return out;
}

void read_status_bits(int status) { raise_status(status, true); }

void read_status_now(Ctx& ctx, bool gram_stage) {
  read_status(ctx);
  ctx.sync();
  raise_status(*ctx.h_status, gram_stage);
}

DTensor gram_matrix(Ctx& ctx, const DTensor& z) {
  if (z.shape.empty()) throw Error(kShapeError, "gram_matrix needs a tensor with a column axis");
  const int64_t k = z.shape.back();
  const int64_t rows = k ? z.size() / k : 0;
  DTensor g = ctx.zeros({k, k});
  if (rows > 0 && k > 0) mm(ctx, g.data(), z.data(), true, true, z.data(), false, false, k, k, rows);
  return g;
}

GramFactorsD gram_factors_full(Ctx& ctx, const DTensor& g) {
  if (g.shape.size() != 2 || g.shape[0] != g.shape[1]) throw Error(kShapeError, "gram_factors needs k x k");
  const int64_t k = g.shape[0];
  if (k < 1 || k > 256) throw Error(kShapeError, "gram_factors: 1 <= k <= 256");
  clear_status(ctx);
  GramFactorsD out;
  out.P = ctx.empty({k, k});
  out.R = ctx.empty({k, k});
  out.vecs = ctx.empty({k, k});
  BufPtr def = ctx.alloc(k / 4 + 2), lam = ctx.alloc(k / 2 + 1), work;
  if (2 * k * (k + 1) * 16 > 176 * 1024) work = ctx.alloc(2 * k * (k + 1));
  int* d_def = reinterpret_cast<int*>(def->p);
  {
    ProfScope ps_(ctx, Ctx::kProfSmall);
    gram_factors(g.data(), static_cast<int>(k), out.P.data(), out.R.data(), d_def, d_def + k, ctx.d_status,
                 work ? work->p : nullptr, ctx.stream, reinterpret_cast<double*>(lam->p), out.vecs.data());
  }
  ++ctx.launches;
  out.lam.resize(k);
  out.deficient.resize(k);
  PEPSB_CUDA(cudaMemcpyAsync(out.lam.data(), lam->p, k * sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
  PEPSB_CUDA(cudaMemcpyAsync(out.deficient.data(), d_def, k * sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  read_status(ctx);
  ctx.sync();
  raise_status(*ctx.h_status, true);
  return out;
}

std::pair<DTensor, std::vector<double>> projected_svd_full(Ctx& ctx, const DTensor& z, int64_t target) {
  const int64_t k = z.shape.back();
  DTensor z2;
  z2.buf = z.buf;
  z2.shape = {k ? z.size() / k : 0, k};
  LTensor zl = as_labelled(z2, "ab");
  clear_all_status(ctx);
  Projected pr = projected_svd(ctx, zl, target);
  DTensor ut;
  ut.buf = pr.Ut;
  ut.shape = {k, k};
  return {ut, pr.s};
}

EighD eigh(Ctx& ctx, const DTensor& m) {
  if (m.shape.size() != 2 || m.shape[0] != m.shape[1]) throw Error(kShapeError, "eigh expects a square matrix");
  const int64_t n = m.shape[0];
  if (n > 256) throw Error(kShapeError, "eigh: n > 256 not supported");
  EighD out;
  out.vectors = ctx.empty({n, n});
  if (n == 0) return out;
  clear_status(ctx);
  BufPtr w = ctx.alloc(n / 2 + 1), work;
  if (2 * n * (n + 1) * 16 > 176 * 1024) work = ctx.alloc(2 * n * (n + 1));
  {
    ProfScope ps_(ctx, Ctx::kProfSmall);
    eigh_dense(m.data(), static_cast<int>(n), reinterpret_cast<double*>(w->p), out.vectors.data(), ctx.d_status,
               work ? work->p : nullptr, ctx.stream);
  }
  ++ctx.launches;
  out.values.resize(n);
  PEPSB_CUDA(cudaMemcpyAsync(out.values.data(), w->p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
  read_status(ctx);
  ctx.sync();
  raise_status(*ctx.h_status, false);
  return out;
}

SvdD svd(Ctx& ctx, const DTensor& t, int split) {
  const int order = static_cast<int>(t.shape.size());
  if (split < 1 || split >= order) throw Error(kShapeError, "svd split must satisfy 1 <= split < order");
  std::vector<int64_t> rs(t.shape.begin(), t.shape.begin() + split), cs(t.shape.begin() + split, t.shape.end());
  const int64_t m = prod(rs), n = prod(cs), k = std::min(m, n);
  clear_status(ctx);
  SvdD out;
  std::vector<int64_t> us = rs, vs = {k};
  us.push_back(k);
  vs.insert(vs.end(), cs.begin(), cs.end());
  out.u = ctx.empty(us);
  out.v = ctx.empty(vs);
  BufPtr sd = ctx.alloc(k / 2 + 1);
  BufPtr work;
  int64_t ws = small_svd_workspace(static_cast<int>(m), static_cast<int>(n), 1);
  if (ws) work = ctx.alloc(ws);
  {
    ProfScope ps_(ctx, Ctx::kProfSmall);
    small_svd(t.data(), 0, static_cast<int>(m), static_cast<int>(n), static_cast<int>(n), out.u.data(), 0,
              reinterpret_cast<double*>(sd->p), 0, out.v.data(), 0, 1, ctx.d_status, work ? work->p : nullptr,
              ctx.stream);
  }
  ++ctx.launches;
  out.s.resize(k);
  PEPSB_CUDA(cudaMemcpyAsync(out.s.data(), sd->p, k * sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
  read_status(ctx);
  ctx.sync();
  raise_status(*ctx.h_status, false);
  return out;
}

namespace {
EinsumsvdResultD rsvd_faithful_fallback(Ctx& ctx, const ImplicitOp& op, const Trunc& policy, const Rsvd& cfg,
                                        int absorb, const std::vector<int>& t1_perm) {
  try {
    return rsvd_core(ctx, op, policy, cfg, absorb, t1_perm);
  } catch (const RedoFaithful&) {
    const int saved = ctx.orth_mode;
    ctx.orth_mode = 0;
    try {
      EinsumsvdResultD r = rsvd_core(ctx, op, policy, cfg, absorb, t1_perm);
      ctx.orth_mode = saved;
      return r;
    } catch (...) {
      ctx.orth_mode = saved;
      throw;
    }
  }
}
}  // namespace

SvdTripleD randomized_svd(Ctx& ctx, const ImplicitOp& op, const Trunc& policy, const Rsvd& cfg) {
  EinsumsvdResultD r = rsvd_faithful_fallback(ctx, op, policy, cfg, -1, {});
  return SvdTripleD{r.t1, r.t2, r.s, r.rank_clamped};
}

EinsumsvdResultD einsumsvd(Ctx& ctx, const ImplicitOp& op, const Trunc& policy, int strategy, int absorb,
                           const Rsvd& cfg, const std::vector<int>& t1_perm) {
  if (op.rows.empty() || op.cols.empty())
    throw Error(kShapeError, "einsumsvd needs non-empty row and column groups");
  const uint64_t f0 = ctx.flops;
  EinsumsvdResultD out;
  if (strategy == kImplicitRsvd) {
    out = rsvd_faithful_fallback(ctx, op, policy, cfg, absorb, t1_perm);
  } else {
    DTensor mat = implicit_materialize(ctx, op);
    const int split = static_cast<int>(op.rows.size());
    SvdD full = svd(ctx, mat, split);
    const size_t rank = retained_rank(full.s, policy);
    out.s.assign(full.s.begin(), full.s.begin() + rank);
    const int64_t m = op.row_extent(), n = op.col_extent(), k = std::min(m, n);
    out.rank_clamped = policy.max_rank > static_cast<uint64_t>(k);
    std::vector<double> wl, wr;
    absorb_weights(out.s, absorb, wl, wr);
    BufPtr dwl = upload_doubles(ctx, wl), dwr = upload_doubles(ctx, wr);
    const int64_t r = static_cast<int64_t>(rank);
    std::vector<int64_t> s1 = op.row_shape(), s2 = {r};
    s1.push_back(r);
    for (auto e : op.col_shape()) s2.push_back(e);
    out.t1 = ctx.empty(s1);
    out.t2 = ctx.empty(s2);
    slice_scale_cols(out.t1.data(), full.u.data(), m, r, k, reinterpret_cast<double*>(dwl->p), 0, ctx.stream);
    slice_scale_cols(out.t2.data(), full.v.data(), r, n, n, nullptr, 0, ctx.stream);
    scale_axis(out.t2.data(), r * n, n, r, reinterpret_cast<double*>(dwr->p), ctx.stream);
    ctx.launches += 3;
    if (!t1_perm.empty()) {
      std::string lab = unused_labels("", static_cast<int>(t1_perm.size()));
      std::string o;
      for (int a : t1_perm) o += lab[a];
      LTensor r1 = reduce_to(ctx, as_labelled(out.t1, lab), o);
      out.t1.buf = r1.buf;
      out.t1.shape = r1.ext;
    }
  }
  ctx.einsumsvd_flops += ctx.flops - f0;
  return out;
}

}  // namespace pepsb
