// einsumsvd and its building blocks on the device (the hot path).
//
// Mirrors proj/include/peps/implicit.hpp and proj/include/peps/decomposition.hpp:
// ImplicitOperator{tensors, labels, row_labels, col_labels} with apply /
// adjoint_apply / materialize; gram_orthogonalize; randomized_svd; einsumsvd.
#pragma once

#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "context.h"
#include "engine.h"

namespace pepsb {

struct Trunc {
  uint64_t max_rank = 0;  // 0: unbounded
  double rel_cutoff = 1e-14;
};

struct Rsvd {
  int power_iters = 2;
  int oversample = -1;  // < 0: max(5, ceil(0.1 * target))
  uint64_t seed = 0;
};

enum Strategy { kExact = 0, kImplicitRsvd = 1 };
enum Absorb { kSplit = 0, kLeft = 1, kRight = 2 };

// implicit.hpp:15-44; validation as implicit.cpp:10-49.  `conj[i]` marks a
// tensor to be used conjugated (lazily — no copy), e.g. the bra layer.
class ImplicitOp {
 public:
  ImplicitOp(std::vector<DTensor> tensors, std::vector<std::string> labels, std::string rows,
             std::string cols, std::vector<bool> conj = {});
  const std::vector<int64_t>& row_shape() const { return row_shape_; }
  const std::vector<int64_t>& col_shape() const { return col_shape_; }
  int64_t row_extent() const;
  int64_t col_extent() const;
  char fresh_label() const;  // implicit.cpp:54-64

  std::vector<DTensor> tensors;
  std::vector<std::string> labels;
  std::string rows, cols;
  std::vector<bool> conj;

 private:
  std::vector<int64_t> row_shape_, col_shape_;
};

// Row lookahead (two_layer_apply_row): the NEXT einsumsvd's operator -- its
// leaf 0 (the pending tensor) only a shape guess without data -- and seed.
// The current einsumsvd starts that operator's sketch and the v-independent
// prefix of its first application on the side stream during its own tail; the
// next einsumsvd reuses them when its real operator has the guessed shapes.
struct Lookahead {
  ImplicitOp op;
  uint64_t seed = 0;
};
inline void set_lookahead(Ctx& ctx, ImplicitOp next, uint64_t seed) {
  ctx.lookahead = std::make_shared<Lookahead>(Lookahead{std::move(next), seed});
}

DTensor implicit_apply(Ctx& ctx, const ImplicitOp& op, const DTensor& q, bool adjoint);
DTensor implicit_materialize(Ctx& ctx, const ImplicitOp& op);

struct SvdTripleD {
  DTensor u, v;
  std::vector<double> s;
  bool rank_clamped = false;
};

struct EinsumsvdResultD {
  DTensor t1, t2;
  std::vector<double> s;
  bool rank_clamped = false;
};

struct EighD {
  std::vector<double> values;  // descending
  DTensor vectors;             // n x n, column j = phase-fixed eigenvector j
};

struct GramFactorsD {
  DTensor P, R, vecs;              // k x k: X diag(l^-1/2), diag(l^1/2) X^H, phase-fixed X
  std::vector<double> lam;         // descending
  std::vector<int> deficient;      // l_j < 1e-12 l_max
};

struct SvdD {
  DTensor u, v;
  std::vector<double> s;
};

// decomposition.cpp:160-193
std::pair<DTensor, DTensor> gram_orthogonalize(Ctx& ctx, const DTensor& a, int split);
// decomposition.cpp:259-306
SvdTripleD randomized_svd(Ctx& ctx, const ImplicitOp& op, const Trunc& policy, const Rsvd& cfg);
// decomposition.cpp:308-352
// `t1_perm` (optional) permutes t1's axes on output, like Tensor::permute.
EinsumsvdResultD einsumsvd(Ctx& ctx, const ImplicitOp& op, const Trunc& policy, int strategy,
                           int absorb, const Rsvd& cfg, const std::vector<int>& t1_perm = {});
// Building blocks of the bond-sharded einsumsvd (sharded.py): G = Z^H Z over the
// leading axes of z (the last axis is the probe axis); the reference's Gram
// factors (decomposition.cpp:128-156) of a given Gram matrix; and the projected
// SVD of B = Z^H (left singular vectors Ut, k x k, and sigma).
DTensor gram_matrix(Ctx& ctx, const DTensor& z);
GramFactorsD gram_factors_full(Ctx& ctx, const DTensor& g);
std::pair<DTensor, std::vector<double>> projected_svd_full(Ctx& ctx, const DTensor& z, int64_t target);
// Stream-ordered variants for the sharded driver (no host synchronisation):
// the reference's Gram-eigh orthogonalisation with on-device completion
// (status bits accumulate in ctx.d_status), and Gram factors whose
// "any column deficient" flag stays on the device (checked later).
DTensor orth_async(Ctx& ctx, const DTensor& y);
struct GramFactorsAsync {
  DTensor P;                 // k x k: X diag(l^-1/2)
  BufPtr flags;              // deficient[k] followed by any_deficient
  int* any_deficient = nullptr;
};
GramFactorsAsync gram_factors_async(Ctx& ctx, const DTensor& g);
// Reads the status word (one sync) and raises the reference's errors.
void read_status_now(Ctx& ctx, bool gram_stage);
// Raises the reference's errors for a status word already read back.
void read_status_bits(int status);
// linalg.cpp:256-295 (Hermitian eigendecomposition of a square matrix, n <= 256)
EighD eigh(Ctx& ctx, const DTensor& m);
// linalg.cpp:193-207 (thin SVD of a matricised tensor; small matrices)
SvdD svd(Ctx& ctx, const DTensor& t, int split);

size_t retained_rank(const std::vector<double>& s, const Trunc& policy);
size_t effective_oversample(const Rsvd& cfg, size_t target);

}  // namespace pepsb
