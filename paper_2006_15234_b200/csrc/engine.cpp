#include "engine.h"

#include <algorithm>
#include <climits>
#include <cstring>
#include <functional>
#include <set>

#include "tensor_ops.cuh"
#include "zgemm.cuh"

namespace pepsb {

struct PlanEntry {
  uint64_t flops = 0;
  uint64_t peak = 0;
  unsigned left = 0, right = 0;
};

namespace {

bool has(const std::string& s, char c) { return s.find(c) != std::string::npos; }

// Labels of `t` ordered by descending stride (its physical order), restricted
// to `group`; extent-1 labels are dropped (they never affect addressing).
std::string physical_order(const LTensor& t, const std::string& group) {
  std::vector<std::pair<int64_t, char>> v;
  for (size_t a = 0; a < t.labels.size(); ++a) {
    char c = t.labels[a];
    if (has(group, c) && t.ext[a] > 1) v.push_back({t.str[a], c});
  }
  std::stable_sort(v.begin(), v.end(), [](auto& x, auto& y) { return x.first > y.first; });
  std::string s;
  for (auto& p : v) s += p.second;
  return s;
}

std::string drop_unit(const LTensor& t, const std::string& order) {
  std::string s;
  for (char c : order)
    if (t.extent_of(c) > 1) s += c;
  return s;
}

// True when `order` (extent-1 labels ignored) addresses a uniform-stride block.
bool flattenable(const LTensor& t, const std::string& order) {
  std::string o = drop_unit(t, order);
  for (size_t i = 0; i + 1 < o.size(); ++i)
    if (t.stride_of(o[i]) != t.stride_of(o[i + 1]) * t.extent_of(o[i + 1])) return false;
  return true;
}

int64_t group_stride(const LTensor& t, const std::string& order) {
  std::string o = drop_unit(t, order);
  return o.empty() ? 1 : t.stride_of(o.back());
}

int64_t group_size(const LTensor& t, const std::string& g) {
  int64_t n = 1;
  for (char c : g) n *= t.extent_of(c);
  return n;
}

bool repeated(const std::string& s) {
  std::set<char> seen;
  for (char c : s)
    if (!seen.insert(c).second) return true;
  return false;
}

}  // namespace

void parse_spec(const std::string& text, std::vector<std::string>& inputs, std::string& output) {
  auto arrow = text.find("->");
  if (arrow == std::string::npos) throw Error(kShapeError, "contraction spec needs '->': " + text);
  output = text.substr(arrow + 2);
  inputs.clear();
  std::string cur;
  for (char c : text.substr(0, arrow)) {
    if (c == ',') {
      inputs.push_back(cur);
      cur.clear();
    } else if (c != ' ') {
      cur += c;
    }
  }
  inputs.push_back(cur);
}

// ---------------------------------------------------------------------------- gather

LTensor reduce_to(Ctx& ctx, const LTensor& t, const std::string& out_order) {
  // Source stride per distinct label (repeated labels -> diagonal: strides add).
  std::map<char, int64_t> sstride, sext;
  for (size_t a = 0; a < t.labels.size(); ++a) {
    char c = t.labels[a];
    sstride[c] += t.str[a];
    auto it = sext.find(c);
    if (it != sext.end() && it->second != t.ext[a])
      throw Error(kShapeError, std::string("extent mismatch on repeated label '") + c + "'");
    sext[c] = t.ext[a];
  }
  GatherParams p;
  std::vector<int64_t> oext;
  for (char c : out_order) {
    if (!sext.count(c)) throw Error(kShapeError, std::string("output label '") + c + "' missing");
    if (p.nout >= kMaxModes) throw Error(kShapeError, "tensor order too large");
    p.oext[p.nout] = sext[c];
    p.ostr[p.nout] = sstride[c];
    ++p.nout;
    oext.push_back(sext[c]);
  }
  int64_t kept = 1, sum = 1;
  for (auto e : oext) kept *= e;
  for (auto& [c, e] : sext) {
    if (has(out_order, c)) continue;
    if (e == 1) continue;
    if (p.nsum >= kMaxModes) throw Error(kShapeError, "too many summed labels");
    p.sext[p.nsum] = e;
    p.sstr[p.nsum] = sstride[c];
    ++p.nsum;
    sum *= e;
  }
  p.conj = t.conj ? 1 : 0;
  LTensor out;
  out.buf = ctx.alloc(kept);
  out.buf->real = t.buf && t.buf->real;  // a gather / sum of real entries is real
  out.ptr = out.buf->p;
  out.labels = out_order;
  out.ext = oext;
  out.str = row_major_strides(oext);
  {
    ProfScope ps(ctx, Ctx::kProfGather, 0.0, 32.0 * kept * sum);
    gather_sum(out.buf->p, t.ptr, p, ctx.stream);
  }
  ++ctx.launches;
  if (p.nsum) ctx.flops += static_cast<uint64_t>(kept * sum);
  return out;
}

DTensor materialize(Ctx& ctx, const LTensor& t, const std::string& order) {
  const bool contiguous = !t.conj && t.labels == order && t.str == row_major_strides(t.ext) && t.buf &&
                          t.ptr == t.buf->p && t.buf->n == t.size();
  LTensor r = contiguous ? t : reduce_to(ctx, t, order);
  DTensor d;
  d.buf = r.buf;
  d.shape = r.ext;
  return d;
}

// ---------------------------------------------------------------------------- pairwise GEMM

LTensor pairwise_gemm(Ctx& ctx, const LTensor& A_in, const LTensor& B_in, const std::string& batch,
                      const std::string& con, const std::string& out_order, uint64_t* cmacs) {
  std::string freeA, freeB;
  for (char c : A_in.labels)
    if (!has(batch, c) && !has(con, c)) freeA += c;
  for (char c : B_in.labels)
    if (!has(batch, c) && !has(con, c)) freeB += c;
  // An operand whose free or contracted group is not one uniform-stride block
  // (e.g. a probe label between row labels of an intermediate laid out for
  // another consumer) is re-laid out once as [batch][free][con] / [batch][con][free].
  auto usable = [&](const LTensor& t, const std::string& fr) {
    const std::string fp = physical_order(t, fr);
    if (!flattenable(t, con) || !flattenable(t, fp)) return false;
    return group_stride(t, con) == 1 || group_stride(t, fp) == 1 || group_size(t, con) * group_size(t, fr) == 1;
  };
  const bool relayA = !usable(A_in, freeA), relayB = !usable(B_in, freeB);
  const LTensor A = relayA ? reduce_to(ctx, A_in, batch + freeA + con) : A_in;
  const LTensor B = relayB ? reduce_to(ctx, B_in, batch + con + freeB) : B_in;
  // physical orders of the free groups (extent-1 labels dropped)
  const std::string fa = physical_order(A, freeA), fb = physical_order(B, freeB);
  auto describe = [&]() {
    auto one = [](const LTensor& t) {
      std::string d = t.labels + "[";
      for (size_t a = 0; a < t.ext.size(); ++a)
        d += (a ? "," : "") + std::to_string(t.ext[a]) + ":" + std::to_string(t.str[a]);
      return d + "]";
    };
    return " (A " + one(A) + " B " + one(B) + " batch '" + batch + "' con '" + con + "' out '" + out_order + "')";
  };
  if (!flattenable(A, con) || !flattenable(B, con) || drop_unit(A, con) != drop_unit(B, con))
    throw Error(kOtherError, "internal: contracted labels not flattenable in the same order" + describe());
  if (!flattenable(A, fa) || !flattenable(B, fb))
    throw Error(kOtherError, "internal: free labels not flattenable" + describe());

  LTensor C;
  std::vector<int64_t> cext;
  for (char c : out_order) {
    int64_t e = has(A.labels, c) ? A.extent_of(c) : B.extent_of(c);
    cext.push_back(e);
  }
  int64_t total = 1;
  for (auto e : cext) total *= e;
  C.buf = ctx.alloc(total);
  C.buf->real = A.buf && A.buf->real && B.buf && B.buf->real;
  C.ptr = C.buf->p;
  C.labels = out_order;
  C.ext = cext;
  C.str = row_major_strides(cext);

  ZgemmParams p;
  p.A = A.ptr;
  p.B = B.ptr;
  p.C = C.buf->p;
  p.M = group_size(A, freeA);
  p.N = group_size(B, freeB);
  p.K = group_size(A, con);
  p.sAi = group_stride(A, fa);
  p.sAk = group_stride(A, con);
  p.sBk = group_stride(B, con);
  p.sBj = group_stride(B, fb);
  if (p.K == 1) p.sAk = p.sBk = 1;
  p.conjA = A.conj;
  p.conjB = B.conj;
  p.realA = A.buf && A.buf->real;
  p.realB = B.buf && B.buf->real;
  int64_t nbatch = 1;
  for (char c : batch) {
    int64_t e = A.extent_of(c);
    if (e == 1) continue;
    if (p.nb >= 4) throw Error(kShapeError, "more than 4 batch labels in one pairwise contraction");
    p.bext[p.nb] = e;
    p.bsA[p.nb] = A.stride_of(c);
    p.bsB[p.nb] = B.stride_of(c);
    p.bsC[p.nb] = C.stride_of(c);
    ++p.nb;
    nbatch *= e;
  }
  p.batch = nbatch;
  for (char c : fa) {
    if (p.nr >= kMaxModes) throw Error(kShapeError, "too many free labels");
    p.rext[p.nr] = A.extent_of(c);
    p.rstr[p.nr] = C.stride_of(c);
    ++p.nr;
  }
  for (char c : fb) {
    if (p.nc >= kMaxModes) throw Error(kShapeError, "too many free labels");
    p.cext[p.nc] = B.extent_of(c);
    p.cstr[p.nc] = C.stride_of(c);
    ++p.nc;
  }
  int64_t ws = zgemm_plan_splits(p, ctx.num_sms);
  BufPtr work;
  if (ws > 0) {
    work = ctx.alloc(ws);
    p.work = work->p;
  }
  {
    ProfScope ps(ctx, Ctx::kProfGemm, 8.0 * p.batch * p.M * p.N * p.K,
                 16.0 * (p.batch * (p.M * p.K + p.K * p.N + p.M * p.N)), zgemm_exec_flops(p));
    zgemm_launch(p, ctx.stream);
  }
  ctx.launches += p.splits > 1 ? 2 : 1;
  const uint64_t macs = static_cast<uint64_t>(p.batch) * p.M * p.N * p.K;
  ctx.flops += 2 * macs;
  if (cmacs) *cmacs += macs;
  return C;
}

// ---------------------------------------------------------------------------- plan

ContractionPlan::ContractionPlan(const std::vector<LeafMeta>& leaves, const std::string& output,
                                 int flexible, char flex_last)
    : leaves_(leaves), output_(output), flexible_(flexible), flex_last_(flex_last) {
  const size_t n = leaves_.size();
  if (n == 0) throw Error(kShapeError, "empty tensor network");
  std::map<char, int64_t> all;
  for (auto& l : leaves_) {
    if (l.labels.size() != l.ext.size())
      throw Error(kShapeError, "label string '" + l.labels + "' does not match tensor order " +
                                   std::to_string(l.ext.size()));
    for (size_t a = 0; a < l.labels.size(); ++a) {
      auto [it, ins] = all.emplace(l.labels[a], l.ext[a]);
      if (!ins && it->second != l.ext[a])
        throw Error(kShapeError, std::string("extent mismatch on label '") + l.labels[a] + "': " +
                                     std::to_string(it->second) + " vs " + std::to_string(l.ext[a]));
    }
  }
  for (char c : output_)
    if (!all.count(c)) throw Error(kShapeError, std::string("output label '") + c + "' appears in no input");
  leaf_want_.assign(n, "");

  auto result_of = [&](unsigned mask) {
    std::map<char, int64_t> inside, res;
    for (size_t t = 0; t < n; ++t)
      if (mask & (1u << t))
        for (size_t a = 0; a < leaves_[t].labels.size(); ++a) inside[leaves_[t].labels[a]] = leaves_[t].ext[a];
    for (auto [c, e] : inside) {
      bool needed = has(output_, c);
      for (size_t t = 0; t < n && !needed; ++t)
        if (!(mask & (1u << t))) needed = has(leaves_[t].labels, c);
      if (needed) res[c] = e;
    }
    return res;
  };

  if (n == 1) {
    Node nd;
    nd.leaf = 0;
    nd.mask = 1;
    nd.result = result_of(1);
    nodes_.push_back(nd);
    root_ = 0;
  } else if (n <= 10) {
    // Exact subset DP, identical tie-breaking to plan_order (einsum.cpp:244-313).
    std::vector<std::map<char, int64_t>> sub(1u << n);
    for (unsigned mask = 1; mask < (1u << n); ++mask) sub[mask] = result_of(mask);
    std::vector<PlanEntry> best(1u << n);
    for (unsigned mask = 1; mask < (1u << n); ++mask) {
      if (__builtin_popcount(mask) == 1) continue;
      PlanEntry b;
      b.flops = UINT64_MAX;
      for (unsigned left = (mask - 1) & mask; left; left = (left - 1) & mask) {
        unsigned right = mask ^ left;
        if (left > right) continue;
        std::map<char, int64_t> uni = sub[left];
        for (auto [c, e] : sub[right]) uni[c] = e;
        uint64_t step = 2, out_size = 1;
        for (auto [c, e] : uni) {
          step *= static_cast<uint64_t>(e);
          if (sub[mask].count(c)) out_size *= static_cast<uint64_t>(e);
        }
        uint64_t flops = step, peak = out_size;
        if (__builtin_popcount(left) > 1) {
          flops += best[left].flops;
          peak = std::max(peak, best[left].peak);
        }
        if (__builtin_popcount(right) > 1) {
          flops += best[right].flops;
          peak = std::max(peak, best[right].peak);
        }
        if (flops < b.flops || (flops == b.flops && peak < b.peak)) {
          b.flops = flops;
          b.peak = peak;
          b.left = left;
          b.right = right;
        }
      }
      best[mask] = b;
    }
    // materialise the tree
    std::function<int(unsigned)> mk = [&](unsigned mask) -> int {
      Node nd;
      nd.mask = mask;
      nd.result = sub[mask];
      if (__builtin_popcount(mask) == 1) {
        nd.leaf = __builtin_ctz(mask);
        nodes_.push_back(nd);
        return static_cast<int>(nodes_.size()) - 1;
      }
      int l = mk(best[mask].left);
      int r = mk(best[mask].right);
      nd.left = l;
      nd.right = r;
      nodes_.push_back(nd);
      return static_cast<int>(nodes_.size()) - 1;
    };
    root_ = mk((1u << n) - 1);
  } else {
    // Greedy fallback (einsum.cpp:360-402): smallest intermediate first, ties by flops.
    std::vector<int> live;
    std::vector<std::string> labs;
    std::vector<std::map<char, int64_t>> exts;
    for (size_t t = 0; t < n; ++t) {
      Node nd;
      nd.leaf = static_cast<int>(t);
      nd.mask = 1u << t;
      nd.result = result_of(nd.mask);
      nodes_.push_back(nd);
      live.push_back(static_cast<int>(t));
      labs.push_back(leaves_[t].labels);
      std::map<char, int64_t> m;
      for (size_t a = 0; a < leaves_[t].labels.size(); ++a) m[leaves_[t].labels[a]] = leaves_[t].ext[a];
      exts.push_back(m);
    }
    while (live.size() > 1) {
      auto keep_for = [&](size_t i, size_t j) {
        std::string keep = output_;
        for (size_t t = 0; t < live.size(); ++t) {
          if (t == i || t == j) continue;
          for (char c : labs[t])
            if (!has(keep, c)) keep += c;
        }
        return keep;
      };
      size_t bi = 0, bj = 1;
      uint64_t bsize = UINT64_MAX, bfl = UINT64_MAX;
      for (size_t i = 0; i < live.size(); ++i)
        for (size_t j = i + 1; j < live.size(); ++j) {
          std::string keep = keep_for(i, j);
          std::map<char, int64_t> e = exts[i];
          for (auto [c, x] : exts[j]) e[c] = x;
          uint64_t size = 1, fl = 2;
          for (auto [c, x] : e) {
            fl *= x;
            if (has(keep, c)) size *= x;
          }
          if (size < bsize || (size == bsize && fl < bfl)) {
            bsize = size;
            bfl = fl;
            bi = i;
            bj = j;
          }
        }
      std::string keep = keep_for(bi, bj);
      Node nd;
      nd.left = live[bi];
      nd.right = live[bj];
      nd.mask = nodes_[live[bi]].mask | nodes_[live[bj]].mask;
      std::map<char, int64_t> e = exts[bi];
      for (auto [c, x] : exts[bj]) e[c] = x;
      std::string rl;
      for (auto [c, x] : e)
        if (has(keep, c)) {
          nd.result[c] = x;
          rl += c;
        }
      nodes_.push_back(nd);
      live[bi] = static_cast<int>(nodes_.size()) - 1;
      labs[bi] = rl;
      exts[bi] = nd.result;
      live.erase(live.begin() + bj);
      labs.erase(labs.begin() + bj);
      exts.erase(exts.begin() + bj);
    }
    root_ = live[0];
  }

  // Flexible leaf: [batch][con][free..., flex_last] at its parent contraction.
  if (flexible_ >= 0) {
    const std::string& fl = leaves_[flexible_].labels;
    int parent = -1;
    for (size_t i = 0; i < nodes_.size(); ++i) {
      const Node& nd = nodes_[i];
      if (nd.left >= 0 && (nodes_[nd.left].leaf == flexible_ || nodes_[nd.right].leaf == flexible_)) parent = static_cast<int>(i);
    }
    std::string con, batch, fre;
    if (parent >= 0) {
      const Node& pn = nodes_[parent];
      int other = nodes_[pn.left].leaf == flexible_ ? pn.right : pn.left;
      const auto& orl = nodes_[other].result;
      for (char c : fl) {
        bool in_other = orl.count(c) > 0;
        bool kept = pn.result.count(c) > 0;
        if (in_other && kept) batch += c;
        else if (in_other) con += c;
        else fre += c;
      }
      // Prefer the partner leaf's physical con order when it is a plain leaf.
      if (nodes_[other].leaf >= 0) {
        const std::string& ol = leaves_[nodes_[other].leaf].labels;
        std::string oc;
        for (char c : ol)
          if (has(con, c)) oc += c;
        con = oc;
      }
    } else {
      fre = fl;
    }
    std::string f2;
    for (char c : fre)
      if (c != flex_last_) f2 += c;
    if (has(fre, flex_last_)) f2 += flex_last_;
    flex_order_ = batch + con + f2;
  }
}

void ContractionPlan::finalize(const std::string& out_order) {
  if (out_order.size() != nodes_[root_].result.size())
    throw Error(kShapeError, "output order '" + out_order + "' does not match the network's open labels");
  for (char c : out_order)
    if (!nodes_[root_].result.count(c)) throw Error(kShapeError, std::string("output label '") + c + "' missing");
  nodes_[root_].order = out_order;
  if (nodes_[root_].leaf < 0) assign(root_);
  else leaf_want_[nodes_[root_].leaf] = out_order;
  finalized_ = true;
}

void ContractionPlan::assign(int ni) {
  Node& nd = nodes_[ni];
  Node& L = nodes_[nd.left];
  Node& R = nodes_[nd.right];
  std::string batch, con, fa, fb;
  for (auto [c, e] : L.result) {
    if (R.result.count(c)) {
      if (nd.result.count(c)) batch += c;
      else con += c;
    }
  }
  // batch in output order
  std::string b2;
  for (char c : nd.order)
    if (has(batch, c)) b2 += c;
  batch = b2;
  // con order: a plain (non-flexible) leaf child's own order, else a flexible
  // child's chosen order, else label order.
  auto leaf_con_order = [&](const Node& ch) -> std::string {
    if (ch.leaf < 0) return "";
    const std::string& lab = ch.leaf == flexible_ ? flex_order_ : leaves_[ch.leaf].labels;
    std::string s;
    for (char c : lab)
      if (has(con, c) && s.find(c) == std::string::npos) s += c;
    return s;
  };
  std::string co = leaf_con_order(L);
  if (co.size() != con.size() || (L.leaf >= 0 && L.leaf != flexible_ && repeated(leaves_[L.leaf].labels))) co = "";
  std::string co2 = leaf_con_order(R);
  if (R.leaf == flexible_ && co2.size() == con.size()) co = co2;
  else if (L.leaf == flexible_ && leaf_con_order(L).size() == con.size()) co = leaf_con_order(L);
  else if (co.empty() && co2.size() == con.size()) co = co2;
  if (co.size() == con.size()) con = co;
  nd.con = con;
  nd.batch = batch;
  // roles: A = child with the smaller free extent (the GEMM's M side)
  auto free_size = [&](const Node& ch) {
    int64_t s = 1;
    for (auto [c, e] : ch.result)
      if (!has(batch, c) && !has(con, c)) s *= e;
    return s;
  };
  bool left_is_a = free_size(L) <= free_size(R);
  nd.a_child = left_is_a ? nd.left : nd.right;
  nd.b_child = left_is_a ? nd.right : nd.left;
  auto free_in_order = [&](const Node& ch) {
    std::string s;
    for (char c : nd.order)
      if (ch.result.count(c) && !has(batch, c) && !has(con, c)) s += c;
    return s;
  };
  for (int side = 0; side < 2; ++side) {
    int ci = side == 0 ? nd.a_child : nd.b_child;
    Node& ch = nodes_[ci];
    std::string fr = free_in_order(ch);
    std::string want = side == 0 ? batch + fr + con : batch + con + fr;
    if (ch.leaf < 0) {
      ch.order = want;
      assign(ci);
    } else if (ch.leaf != flexible_) {
      leaf_want_[ch.leaf] = want;  // used only when the given layout is unusable
    }
  }
}

LTensor ContractionPlan::prepare_leaf(Ctx& ctx, int leaf, const LTensor& t, const std::string& want) {
  if (cache_static && leaf != flexible_) {
    auto it = leaf_cache_.find(leaf);
    if (it != leaf_cache_.end()) return it->second;
  }
  LTensor r = reduce_to(ctx, t, want);
  if (cache_static && leaf != flexible_) leaf_cache_[leaf] = r;
  return r;
}

LTensor ContractionPlan::run(Ctx& ctx, int ni, const std::vector<LTensor>& leaves) {
  if (ni == subst_node_) return subst_;
  const Node& nd = nodes_[ni];
  if (nd.leaf >= 0) return leaves[nd.leaf];
  LTensor ops[2];
  for (int side = 0; side < 2; ++side) {
    int ci = side == 0 ? nd.a_child : nd.b_child;
    const Node& ch = nodes_[ci];
    if (ch.leaf < 0) {
      ops[side] = run(ctx, ci, leaves);
      continue;
    }
    const LTensor& t = leaves[ch.leaf];
    // Usable in place?  result labels only (no sums/diagonals), con block in
    // the node's order, free block flattenable, one group unit-stride.
    bool ok = !repeated(t.labels) && t.labels.size() == ch.result.size();
    if (ok) {
      std::string fr;
      for (char c : t.labels)
        if (!has(nd.batch, c) && !has(nd.con, c)) fr += c;
      const std::string fp = physical_order(t, fr);
      ok = flattenable(t, nd.con) && flattenable(t, fp);
      if (ok) {
        int64_t sk = group_stride(t, nd.con), sf = group_stride(t, fp);
        ok = sk == 1 || sf == 1 || group_size(t, nd.con) * group_size(t, fr) == 1;
      }
    }
    if (ok) {
      ops[side] = t;
    } else {
      std::string want = leaf_want_[ch.leaf];
      if (want.empty()) {
        std::string fr;
        for (auto [c, e] : ch.result)
          if (!has(nd.batch, c) && !has(nd.con, c)) fr += c;
        want = side == 0 ? nd.batch + fr + nd.con : nd.batch + nd.con + fr;
      }
      ops[side] = prepare_leaf(ctx, ch.leaf, t, want);
    }
  }
  LTensor out = pairwise_gemm(ctx, ops[0], ops[1], nd.batch, nd.con, nd.order, &cmacs_);
  return out;
}

LTensor ContractionPlan::execute(Ctx& ctx, const std::vector<LTensor>& leaves) {
  if (!finalized_) throw Error(kOtherError, "internal: plan not finalized");
  if (leaves.size() != leaves_.size()) throw Error(kShapeError, "leaf count mismatch");
  for (size_t i = 0; i < leaves.size(); ++i) {
    if (leaves[i].labels.size() != leaves_[i].labels.size())
      throw Error(kShapeError, "leaf label mismatch");
  }
  const uint64_t f0 = ctx.flops;
  cmacs_ = 0;
  LTensor out;
  const Node& r = nodes_[root_];
  if (r.leaf >= 0) {
    out = reduce_to(ctx, leaves[r.leaf], r.order);
  } else {
    out = run(ctx, root_, leaves);
  }
  flops_ = ctx.flops - f0;
  return out;
}

int ContractionPlan::prefix_node(int excl) const {
  if (root_ < 0) return -1;
  const Node& r = nodes_[root_];
  if (r.leaf >= 0) return -1;
  int other = -1;
  if (nodes_[r.a_child].leaf == excl) other = r.b_child;
  else if (nodes_[r.b_child].leaf == excl) other = r.a_child;
  if (other < 0 || nodes_[other].leaf >= 0) return -1;  // only an internal subtree is worth running ahead
  return other;
}

LTensor ContractionPlan::run_prefix(Ctx& ctx, const std::vector<LTensor>& leaves, int excl) {
  if (!finalized_) throw Error(kOtherError, "internal: plan not finalized");
  const int node = prefix_node(excl);
  if (node < 0) return LTensor();
  return run(ctx, node, leaves);
}

int ContractionPlan::parent_of_leaf(int leaf) const {
  for (size_t i = 0; i < nodes_.size(); ++i) {
    const Node& nd = nodes_[i];
    if (nd.leaf >= 0) continue;
    if (nodes_[nd.a_child].leaf == leaf || nodes_[nd.b_child].leaf == leaf) return static_cast<int>(i);
  }
  return -1;
}

LTensor ContractionPlan::execute_with_prefix(Ctx& ctx, const std::vector<LTensor>& leaves, int excl,
                                             const LTensor& prefix) {
  const int node = prefix_node(excl);
  if (node < 0 || !prefix.buf) return execute(ctx, leaves);
  return execute_subst(ctx, leaves, node, prefix);
}

LTensor ContractionPlan::execute_subst(Ctx& ctx, const std::vector<LTensor>& leaves, int node, const LTensor& result) {
  subst_node_ = node;
  subst_ = result;
  LTensor out;
  try {
    out = execute(ctx, leaves);
  } catch (...) {
    subst_node_ = -1;
    subst_ = LTensor();
    throw;
  }
  subst_node_ = -1;
  subst_ = LTensor();
  return out;
}

LTensor contract_network(Ctx& ctx, const std::vector<LTensor>& leaves, const std::string& out_order) {
  std::vector<LeafMeta> meta;
  for (auto& l : leaves) meta.push_back({l.labels, l.ext});
  std::set<char> seen;
  for (char c : out_order)
    if (!seen.insert(c).second) throw Error(kShapeError, std::string("output label '") + c + "' repeated");
  ContractionPlan plan(meta, out_order);
  plan.finalize(out_order);
  return plan.execute(ctx, leaves);
}

}  // namespace pepsb
