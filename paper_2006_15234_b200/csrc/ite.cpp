#include "ite.h"

#include <algorithm>
#include <set>

#include "smalldense.cuh"

namespace pepsb {

namespace {

// state.cpp:99-122 geometry: permutation taking a site to (env..., phys, shared)
// and the placement of (env..., out-phys, new-bond) back into site order.
struct Geometry {
  int to_env[5];
  int from_env[5];
};

Geometry geometry(bool first, bool horizontal) {
  if (horizontal)
    return first ? Geometry{{1, 2, 3, 0, 4}, {3, 0, 1, 2, 4}} : Geometry{{1, 3, 4, 0, 2}, {3, 0, 4, 1, 2}};
  return first ? Geometry{{1, 2, 4, 0, 3}, {3, 0, 1, 4, 2}} : Geometry{{2, 3, 4, 0, 1}, {3, 4, 0, 1, 2}};
}

template <class T>
BufPtr upload(Ctx& ctx, const std::vector<T>& v) {
  const int64_t bytes = static_cast<int64_t>(v.size() * sizeof(T));
  BufPtr b = ctx.alloc((bytes + 15) / 16 + 1);
  if (bytes) PEPSB_CUDA(cudaMemcpyAsync(b->p, v.data(), bytes, cudaMemcpyHostToDevice, ctx.stream));
  return b;
}

}  // namespace

DTensor hermitian_exp(Ctx& ctx, const DTensor& op, double coeff, double tau) {
  if (op.shape.size() != 2 || op.shape[0] != op.shape[1]) throw Error(kShapeError, "operator must be square");
  DTensor out = ctx.empty(op.shape);
  herm_exp(op.data(), static_cast<int>(op.shape[0]), coeff, tau, out.data(), ctx.stream);
  ++ctx.launches;
  return out;
}

PepsStateD apply_one_site_batch(Ctx& ctx, const PepsStateD& s, const DTensor& gate,
                                const std::vector<std::pair<int, int>>& sites) {
  const int d = s.d;
  if (gate.shape.size() != 2 || gate.shape[0] != d || gate.shape[1] != d)
    throw Error(kShapeError, "one-site gate must be d x d");
  PepsStateD out = s;
  std::vector<SuOneSiteDesc> descs;
  for (auto [r, c] : sites) {
    if (r < 0 || c < 0 || r >= s.rows || c >= s.cols) throw Error(kValidationError, "site outside the grid");
    const DTensor& src = s.site(r, c);
    DTensor dst = ctx.empty(src.shape);
    descs.push_back({src.data(), dst.data(), src.size() / d, d, gate.data()});
    out.site(r, c) = dst;
  }
  BufPtr dd = upload(ctx, descs);
  su_one_site(reinterpret_cast<const SuOneSiteDesc*>(dd->p), static_cast<int>(descs.size()), ctx.stream);
  ++ctx.launches;
  return out;
}

PepsStateD apply_two_site_batch(Ctx& ctx, const PepsStateD& s, const DTensor& gate,
                                const std::vector<std::array<int, 4>>& bonds, const Trunc& policy) {
  const int d = s.d;
  if (gate.shape.size() != 4) throw Error(kShapeError, "two-site gate must be (out,out,in,in)");
  for (auto e : gate.shape)
    if (e != d) throw Error(kShapeError, "two-site gate extents must equal d");
  if (bonds.empty()) return s;
  DTensor gate_sw;  // gate.permute({1,0,3,2}) for bonds given in reverse order (state.cpp:172-176)

  struct Prep {
    int r[2], c[2];
    bool horizontal;
    const double2* g;
  };
  std::vector<Prep> prep;
  std::set<int> used;
  for (const auto& b : bonds) {
    int ar = b[0], ac = b[1], br = b[2], bc = b[3];
    for (int q = 0; q < 2; ++q) {
      int rr = q ? br : ar, cc = q ? bc : ac;
      if (rr < 0 || cc < 0 || rr >= s.rows || cc >= s.cols) throw Error(kValidationError, "site outside the grid");
    }
    const double2* g = gate.data();
    if (br < ar || (br == ar && bc < ac)) {
      std::swap(ar, br);
      std::swap(ac, bc);
      if (!gate_sw.buf) {
        LTensor t = reduce_to(ctx, as_labelled(gate, "opij"), "poji");
        gate_sw = materialize(ctx, t, t.labels);
      }
      g = gate_sw.data();
    }
    const bool horizontal = ar == br && bc == ac + 1;
    const bool vertical = ac == bc && br == ar + 1;
    if (!horizontal && !vertical)
      throw Error(kValidationError, "sites are not lattice-adjacent; use apply_distant for routed pairs");
    if (!used.insert(ar * s.cols + ac).second || !used.insert(br * s.cols + bc).second)
      throw Error(kValidationError, "bonds of one batch must not share a site");
    prep.push_back({{ar, br}, {ac, bc}, horizontal, g});
  }
  const int nb = static_cast<int>(prep.size());

  // ---- reduce_site for both sides of every bond (state.cpp:126-148)
  std::vector<SuSiteDesc> sd(2 * nb);
  std::vector<BufPtr> keep;
  size_t smem_reduce = 0;
  for (int i = 0; i < nb; ++i)
    for (int side = 0; side < 2; ++side) {
      const DTensor& site = s.site(prep[i].r[side], prep[i].c[side]);
      const Geometry g = geometry(side == 0, prep[i].horizontal);
      const auto st = row_major_strides(site.shape);
      SuSiteDesc& D = sd[2 * i + side];
      D.src = site.data();
      for (int a = 0; a < 5; ++a) D.str[a] = st[g.to_env[a]];
      for (int a = 0; a < 3; ++a) D.e[a] = static_cast<int>(site.shape[g.to_env[a]]);
      D.d = static_cast<int>(site.shape[g.to_env[3]]);
      D.s = static_cast<int>(site.shape[g.to_env[4]]);
      const int64_t E = static_cast<int64_t>(D.e[0]) * D.e[1] * D.e[2], S = static_cast<int64_t>(D.d) * D.s;
      D.reduced = E >= S;
      BufPtr q = D.reduced ? ctx.alloc(E * S) : nullptr;
      BufPtr r = ctx.alloc(D.reduced ? S * S : E * S);
      D.Q = q ? q->p : nullptr;
      D.R = r->p;
      if (q) keep.push_back(q);
      keep.push_back(r);
      if (D.reduced) smem_reduce = std::max<size_t>(smem_reduce, (E * S + 5 * S * S + 2 * S) * 16 + S * 4 + 64);
      else smem_reduce = std::max<size_t>(smem_reduce, E * S * 16);
    }
  // The ImplicitOperator ctor rejects a label extent mismatch with ShapeError
  // (implicit.cpp:10-49); here the shared label is "s" of {Ra, Rb}.
  for (int i = 0; i < nb; ++i)
    if (sd[2 * i].s != sd[2 * i + 1].s) throw Error(kShapeError, "shared bond mismatch");
  // 176 KB: the su_reduce attribute, leaving room for the eigensolver's static shared memory.
  if (smem_reduce > 176 * 1024)
    throw Error(kShapeError, "simple update: site too large for the batched kernel");

  // ---- exact einsumsvd of {g, Ra, Rb} (state.cpp:186-194)
  std::vector<SuBondDesc> bd(nb);
  size_t smem_split = 0;
  for (int i = 0; i < nb; ++i) {
    const SuSiteDesc& A = sd[2 * i];
    const SuSiteDesc& B = sd[2 * i + 1];
    SuBondDesc& D = bd[i];
    D.gate = prep[i].g;
    D.Ra = A.R;
    D.Rb = B.R;
    D.ta = A.reduced ? A.d * A.s : A.e[0] * A.e[1] * A.e[2];
    D.tb = B.reduced ? B.d * B.s : B.e[0] * B.e[1] * B.e[2];
    D.d = d;
    D.s = A.s;
    D.cap = policy.max_rank == 0 ? static_cast<int64_t>(d) * A.s : static_cast<int64_t>(policy.max_rank);
    D.cutoff = policy.rel_cutoff;
    const int m = D.ta * d, n = d * D.tb, k = std::min(m, n);
    if (k > 256) throw Error(kShapeError, "simple update: reduced block too large");
    D.rmax = k;
    BufPtr t1 = ctx.alloc(static_cast<int64_t>(m) * k), t2 = ctx.alloc(static_cast<int64_t>(n) * k);
    D.t1 = t1->p;
    D.t2 = t2->p;
    keep.push_back(t1);
    keep.push_back(t2);
    smem_split = std::max<size_t>(smem_split,
                                  static_cast<size_t>(m * n + m * k + k * n + std::max(m, n) * k + k * k) * 16 + k * 8 + 64);
  }
  if (smem_split > 200 * 1024) throw Error(kShapeError, "simple update: reduced block too large for shared memory");

  BufPtr dsd = upload(ctx, sd), dbd = upload(ctx, bd);
  BufPtr dranks = ctx.alloc(nb / 4 + 1);
  int* ranks = reinterpret_cast<int*>(dranks->p);
  int* status = ctx.d_status + 2;
  PEPSB_CUDA(cudaMemsetAsync(status, 0, sizeof(int), ctx.stream));
  su_reduce(reinterpret_cast<const SuSiteDesc*>(dsd->p), 2 * nb, smem_reduce, status, ctx.stream);
  su_split(reinterpret_cast<const SuBondDesc*>(dbd->p), nb, smem_split, ranks, status, ctx.d_degenerate, ctx.stream);
  ctx.launches += 2;
  std::vector<int> hr(nb + 1);
  PEPSB_CUDA(cudaMemcpyAsync(hr.data(), ranks, nb * sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  PEPSB_CUDA(cudaMemcpyAsync(ctx.h_status + 2, status, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
  if (ctx.h_status[2] & kSmallZeroGram) throw Error(kNumericalError, "gram orthogonalization of a zero operator");
  if (ctx.h_status[2] & kSmallCompletionExhausted)
    throw Error(kNumericalError, "orthonormal completion exhausted basis");

  // ---- restore_site (state.cpp:150-157, 196-201)
  PepsStateD out = s;
  std::vector<SuRestoreDesc> rd(2 * nb);
  for (int i = 0; i < nb; ++i)
    for (int side = 0; side < 2; ++side) {
      const SuSiteDesc& S = sd[2 * i + side];
      const Geometry g = geometry(side == 0, prep[i].horizontal);
      const int64_t full[5] = {S.e[0], S.e[1], S.e[2], d, hr[i]};
      std::vector<int64_t> ns(5);
      for (int k = 0; k < 5; ++k) ns[k] = full[g.from_env[k]];
      DTensor dst = ctx.empty(ns);
      const auto nstr = row_major_strides(ns);
      SuRestoreDesc& D = rd[2 * i + side];
      D.Q = S.Q;
      D.reduced = S.reduced;
      D.S = S.d * S.s;
      D.t = side == 0 ? bd[i].t1 : bd[i].t2;
      D.rmax = bd[i].rmax;
      D.bond = i;
      for (int a = 0; a < 3; ++a) D.e[a] = S.e[a];
      D.d = d;
      D.dst = dst.data();
      for (int k = 0; k < 5; ++k) D.dstr[g.from_env[k]] = nstr[k];
      out.site(prep[i].r[side], prep[i].c[side]) = dst;
    }
  BufPtr drd = upload(ctx, rd);
  su_restore(reinterpret_cast<const SuRestoreDesc*>(drd->p), 2 * nb, ranks, ctx.stream);
  ++ctx.launches;
  return out;
}

std::vector<std::vector<std::array<int, 4>>> tfim_bond_colours(int rows, int cols) {
  std::vector<std::vector<std::array<int, 4>>> out(4);
  for (int par = 0; par < 2; ++par)
    for (int r = 0; r < rows; ++r)
      for (int c = par; c + 1 < cols; c += 2) out[par].push_back({r, c, r, c + 1});
  for (int par = 0; par < 2; ++par)
    for (int r = par; r + 1 < rows; r += 2)
      for (int c = 0; c < cols; ++c) out[2 + par].push_back({r, c, r + 1, c});
  return out;
}

PepsStateD ite_tfim(Ctx& ctx, const PepsStateD& s0, double J, double h, double tau, int steps, uint64_t rank) {
  if (tau <= 0.0) throw Error(kConfigError, "tau must be positive");
  if (rank < 1) throw Error(kConfigError, "ranks must be >= 1");
  const int d = s0.d;
  if (d != 2) throw Error(kShapeError, "TFIM needs d = 2");
  // X and Z (x) Z as (4 x 4) with outputs first (gates::two_site, state.cpp:378-383)
  const double xs[8] = {0, 0, 1, 0, 1, 0, 0, 0};
  double zz[32] = {0};
  const double zd[4] = {1, -1, -1, 1};
  for (int i = 0; i < 4; ++i) zz[2 * (i * 4 + i)] = zd[i];
  DTensor X = ctx.empty({2, 2}), ZZ = ctx.empty({4, 4});
  PEPSB_CUDA(cudaMemcpyAsync(X.data(), xs, sizeof(xs), cudaMemcpyHostToDevice, ctx.stream));
  PEPSB_CUDA(cudaMemcpyAsync(ZZ.data(), zz, sizeof(zz), cudaMemcpyHostToDevice, ctx.stream));
  DTensor gx = hermitian_exp(ctx, X, -h, tau);
  DTensor gzz = hermitian_exp(ctx, ZZ, -J, tau);
  gzz.shape = {2, 2, 2, 2};
  ctx.sync();  // host constants above are on the stack
  std::vector<std::pair<int, int>> all;
  for (int r = 0; r < s0.rows; ++r)
    for (int c = 0; c < s0.cols; ++c) all.push_back({r, c});
  const auto colours = tfim_bond_colours(s0.rows, s0.cols);
  const Trunc pol{rank, 1e-14};
  PepsStateD s = s0;
  for (int st = 0; st < steps; ++st) {
    s = apply_one_site_batch(ctx, s, gx, all);
    for (const auto& col : colours) s = apply_two_site_batch(ctx, s, gzz, col, pol);
  }
  return s;
}

}  // namespace pepsb
