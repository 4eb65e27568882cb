// Device tensor-network contraction engine.
//
// Same contraction ORDER as the reference (exact subset DP minimising the
// pairwise flop count, ties by peak intermediate, proj/src/einsum.cpp:234-338;
// greedy fallback above 10 tensors, :360-402), but a different lowering:
// every pairwise step is ONE DMMA GEMM launch whose operands are addressed in
// place and whose epilogue writes the result directly in the label order the
// parent step consumes, so the reference's per-step operand permutes
// (einsum.cpp:203-204) disappear.  Only small network tensors whose
// contracted labels are not contiguous get a one-off re-layout copy, cached
// across repeated executions of the same plan (the 2q+2 operator
// applications of one randomized SVD).
#pragma once

#include <map>
#include <string>
#include <vector>

#include "context.h"

namespace pepsb {

struct LeafMeta {
  std::string labels;
  std::vector<int64_t> ext;
};

class ContractionPlan {
 public:
  // `output_labels`: the set of open labels to produce.  `flexible` names the
  // leaf whose physical layout the plan chooses (e.g. the sketch/probe), with
  // label `flex_last` kept innermost; -1 for none.
  ContractionPlan(const std::vector<LeafMeta>& leaves, const std::string& output_labels,
                  int flexible = -1, char flex_last = 0);

  // Physical label order the plan wants for the flexible leaf.
  const std::string& flexible_order() const { return flex_order_; }
  // Fixes the physical order of the result (a permutation of output_labels).
  void finalize(const std::string& out_order);
  // Executes; leaves[i] must carry leaf i's labels (any strides; the flexible
  // leaf must be in flexible_order()).  Static leaves' re-layout copies are
  // cached when `cache_static` is set.
  LTensor execute(Ctx& ctx, const std::vector<LTensor>& leaves);
  // Speculative prefix: when the root step is (leaf `excl`) x (rest), runs the
  // `rest` subtree (never touching leaf `excl`) and returns its result; an
  // empty tensor (buf == nullptr) otherwise.
  LTensor run_prefix(Ctx& ctx, const std::vector<LTensor>& leaves, int excl);
  // execute() with the `rest` subtree's result supplied by run_prefix.
  LTensor execute_with_prefix(Ctx& ctx, const std::vector<LTensor>& leaves, int excl, const LTensor& prefix);
  // The pairwise step that consumes leaf `leaf` directly (-1 if the leaf is
  // the root); run_node runs one subtree; execute_subst runs the plan with
  // node `node`'s result supplied.
  int parent_of_leaf(int leaf) const;
  LTensor run_node(Ctx& ctx, int node, const std::vector<LTensor>& leaves) { return run(ctx, node, leaves); }
  LTensor execute_subst(Ctx& ctx, const std::vector<LTensor>& leaves, int node, const LTensor& result);

  bool cache_static = false;
  // Reference-convention flops of one execution (instr::flops definition).
  uint64_t flops() const { return flops_; }
  // Total algorithmic complex MACs of one execution (sum of M*N*K*batch).
  uint64_t cmacs() const { return cmacs_; }

 private:
  struct Node {
    int leaf = -1;
    int left = -1, right = -1;
    unsigned mask = 0;
    std::map<char, int64_t> result;  // result label set (sorted by char)
    std::string order;               // physical output order (internal nodes)
    std::string batch, con;          // set at finalize (internal)
    int a_child = -1, b_child = -1;
  };
  int build(unsigned mask, const std::vector<struct PlanEntry>& best);
  void assign(int node);
  LTensor run(Ctx& ctx, int node, const std::vector<LTensor>& leaves);
  LTensor prepare_leaf(Ctx& ctx, int leaf, const LTensor& t, const std::string& want_order);

  std::vector<LeafMeta> leaves_;
  std::string output_;
  int flexible_ = -1;
  char flex_last_ = 0;
  std::string flex_order_;
  std::vector<Node> nodes_;
  int root_ = -1;
  bool finalized_ = false;
  // leaf -> order wanted (empty: use as given)
  std::vector<std::string> leaf_want_;
  std::map<int, LTensor> leaf_cache_;
  int prefix_node(int excl) const;
  int subst_node_ = -1;  // run() returns subst_ for this node (execute_with_prefix)
  LTensor subst_;
  uint64_t flops_ = 0, cmacs_ = 0;
};

// One pairwise contraction as a single GEMM launch (see engine.cpp).
LTensor pairwise_gemm(Ctx& ctx, const LTensor& A, const LTensor& B, const std::string& batch,
                      const std::string& con, const std::string& out_order, uint64_t* cmacs = nullptr);

// Gather (permute / diagonal / label sums / conj) of one tensor into a fresh
// contiguous tensor with labels `out_order` (reduce_single, einsum.cpp:82-169).
LTensor reduce_to(Ctx& ctx, const LTensor& t, const std::string& out_order);

// One-shot network contraction to `out_order` (contract_network, einsum.cpp:340-406).
LTensor contract_network(Ctx& ctx, const std::vector<LTensor>& leaves, const std::string& out_order);

// Parses "ab,bc->ac" (ContractionSpec::parse, einsum.cpp:59-78).
void parse_spec(const std::string& text, std::vector<std::string>& inputs, std::string& output);

// Copies an LTensor into a contiguous DTensor with logical labels `order`.
DTensor materialize(Ctx& ctx, const LTensor& t, const std::string& order);

}  // namespace pepsb
