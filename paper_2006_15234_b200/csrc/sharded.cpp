// Bond-sharded two-layer row absorb over NCCL.
//
// Reference algorithm: two_layer_apply_row (proj/src/contraction.cpp:269-311)
// calling einsumsvd / randomized_svd (proj/src/decomposition.cpp:259-352) on
// the network {v(apqsmn), S(uvst), bra*(dumbe), ket(dvncf)}, rows "apq", cols
// "bctef".  Rank r owns the t-slice T_r of the column side and the s-slice S_r
// of the pending tensor (the previous column's t2, so the partition carries
// over from column to column):
//
//   apply  A Q    (1) bra*(dum|be) Q_r(be|ctfX)       local
//                 (2) ket(vn|dcf) (1)                  local
//                 (3) S(s|uv t_r) (2)                  partial over t  -> all-reduce (s,n,m,X)
//                 (4) v_r(apq|s_r mn) (3)[s_r]         partial over s  -> all-reduce Y (a,p,q,X)
//   adjoint A^H P v_r^* P -> (s_r,n,m,X) -> all-gather over s; S^*, ket^*, bra local on t_r
//   big-side orth G = all-reduce(Z_r^H Z_r) (k x k, 83 KB at k = 72), replicated
//                 Gram factors (Alg. 5), Q_r = Z_r P local
//   small side    Y, P replicated (bitwise identical on every rank: NCCL
//                 all-reduce results are)
//   projected SVD Gram of B^H = Z all-reduced, replicated eigendecomposition;
//                 t1 = P U w_l replicated, t2_r = conj(Z_r) conj(U) w_r / s local.
//
// Every collective is enqueued on the context's stream, in stream order with
// the GEMMs around it; the only host synchronisations are the ones the
// single-GPU einsumsvd also has (Gram-factor deficiency flags, the rank).
// The sketch slice Omega_r is generated directly as the t-slice of the
// reference's counter-based random_tensor (bit-identical elements), so a
// sharded run reproduces the single-device result up to the all-reduce
// summation order.  Columns whose outgoing bond is narrower than the world
// (the last column, t = 1) run replicated on the single-device einsumsvd.
#include "sharded.h"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "tensor_ops.cuh"

namespace pepsb {

namespace {

// ---- NCCL, resolved at run time: no link-time dependency, and inside a torch
// process dlopen returns the libnccl.so.2 torch already loaded.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string failure;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      failure = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p) failure = std::string("libnccl.so.2 lacks ") + n;
      return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!failure.empty()) throw Error(kCudaError, failure);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(kCudaError, std::string(what) + ": " + nccl().GetErrorString(r));
}

std::pair<int64_t, int64_t> shard_range(int64_t extent, int world, int rank) {
  const int64_t base = extent / world, extra = extent % world;
  const int64_t start = rank * base + std::min<int64_t>(rank, extra);
  return {start, start + base + (rank < extra ? 1 : 0)};
}

}  // namespace

struct NcclComm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  ~NcclComm() {
    if (comm) nccl().CommDestroy(comm);
  }
};

void comm_unique_id(unsigned char out[128]) {
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out, &id, sizeof(id));
}

void comm_init(Ctx& ctx, const unsigned char id_bytes[128], int rank, int world) {
  if (world < 1 || rank < 0 || rank >= world) throw Error(kValidationError, "comm_init: bad rank / world");
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, sizeof(id));
  PEPSB_CUDA(cudaSetDevice(ctx.device));
  ctx.sync();
  auto c = std::make_shared<NcclComm>();
  c->rank = rank;
  c->world = world;
  nccl_check(nccl().CommInitRank(&c->comm, world, id, rank), "ncclCommInitRank");
  ctx.comm = c;
}

void comm_destroy(Ctx& ctx) {
  ctx.sync();
  ctx.comm.reset();
}

int comm_rank(const Ctx& ctx) { return ctx.comm ? ctx.comm->rank : 0; }
int comm_world(const Ctx& ctx) { return ctx.comm ? ctx.comm->world : 1; }

namespace {

NcclComm& need_comm(Ctx& ctx) {
  if (!ctx.comm) throw Error(kValidationError, "no communicator: call pepsb_comm_init first");
  return *ctx.comm;
}

// ---- stream-ordered collectives on library buffers

// In place: every rank ends with the elementwise sum.
void allreduce(Ctx& ctx, DTensor& t) {
  NcclComm& cm = need_comm(ctx);
  if (cm.world == 1 || t.size() == 0) return;
  nccl_check(nccl().AllReduce(t.data(), t.data(), 2 * static_cast<size_t>(t.size()), ncclDouble, ncclSum, cm.comm,
                              ctx.stream),
             "ncclAllReduce");
  t.buf->real = false;  // the sum of other ranks' data: realness unknown here
}

// Concatenation along `axis` of every rank's block (balanced contiguous
// partition of `full`, extents differing by at most one): blocks are padded to
// the largest, all-gathered, then placed with strided 2-D copies.
DTensor allgather_axis(Ctx& ctx, const DTensor& local, int axis, int64_t full) {
  NcclComm& cm = need_comm(ctx);
  if (cm.world == 1) return local;
  const auto& sh = local.shape;
  int64_t outer = 1, inner = 1;
  for (int a = 0; a < axis; ++a) outer *= sh[a];
  for (size_t a = axis + 1; a < sh.size(); ++a) inner *= sh[a];
  int64_t maxn = 0;
  for (int r = 0; r < cm.world; ++r) {
    auto [a, b] = shard_range(full, cm.world, r);
    maxn = std::max(maxn, b - a);
  }
  const int64_t nloc = sh[axis];
  const int64_t block = outer * maxn * inner;
  BufPtr send = ctx.alloc(std::max<int64_t>(block, 1));
  if (nloc * inner > 0)
    PEPSB_CUDA(cudaMemcpy2DAsync(send->p, maxn * inner * 16, local.data(), nloc * inner * 16, nloc * inner * 16,
                                 outer, cudaMemcpyDeviceToDevice, ctx.stream));
  BufPtr recv = ctx.alloc(std::max<int64_t>(block * cm.world, 1));
  nccl_check(nccl().AllGather(send->p, recv->p, 2 * static_cast<size_t>(block), ncclDouble, cm.comm, ctx.stream),
             "ncclAllGather");
  std::vector<int64_t> oshape = sh;
  oshape[axis] = full;
  DTensor out = ctx.empty(oshape);
  for (int r = 0; r < cm.world; ++r) {
    auto [a, b] = shard_range(full, cm.world, r);
    if (b == a || inner == 0) continue;
    PEPSB_CUDA(cudaMemcpy2DAsync(out.data() + a * inner, full * inner * 16, recv->p + r * block, maxn * inner * 16,
                                 (b - a) * inner * 16, outer, cudaMemcpyDeviceToDevice, ctx.stream));
  }
  return out;
}

// ---- small helpers over the engine

DTensor reshaped(const DTensor& t, std::vector<int64_t> shape) {
  DTensor r = t;
  r.shape = std::move(shape);
  return r;
}

std::string axis_labels(size_t n) {
  std::string s;
  for (size_t i = 0; i < n; ++i) s += static_cast<char>('a' + i);
  return s;
}

// contract(spec, tensors) with lazily conjugated operands (conj[i]).
DTensor contract(Ctx& ctx, const std::string& spec, const std::vector<DTensor>& ts, const std::vector<bool>& conj) {
  std::vector<std::string> ins;
  std::string out;
  parse_spec(spec, ins, out);
  std::vector<LTensor> leaves;
  for (size_t i = 0; i < ts.size(); ++i) leaves.push_back(as_labelled(ts[i], ins[i], conj[i]));
  LTensor r = contract_network(ctx, leaves, out);
  return materialize(ctx, r, r.labels);
}

DTensor slice(Ctx& ctx, const DTensor& t, int axis, int64_t start, int64_t stop) {
  const std::string lab = axis_labels(t.shape.size());
  LTensor l = as_labelled(t, lab);
  l.ptr += start * l.str[axis];
  l.ext[axis] = stop - start;
  DTensor out = materialize(ctx, reduce_to(ctx, l, lab), lab);
  out.buf->real = t.buf && t.buf->real;
  return out;
}

// k x rank matrix from the first `rank` columns of the k x k matrix u (host
// arrays), each column scaled by w[j], optionally conjugated.
DTensor scaled_columns(Ctx& ctx, const std::vector<double2>& u, int64_t k, int64_t rank,
                       const std::vector<double>& w, bool conjugate) {
  std::vector<double2> h(static_cast<size_t>(k * rank));
  for (int64_t i = 0; i < k; ++i)
    for (int64_t j = 0; j < rank; ++j) {
      double2 x = u[i * k + j];
      if (conjugate) x.y = -x.y;
      h[i * rank + j] = make_double2(x.x * w[j], x.y * w[j]);
    }
  DTensor out = ctx.empty({k, rank});
  PEPSB_CUDA(cudaMemcpyAsync(out.data(), h.data(), h.size() * 16, cudaMemcpyHostToDevice, ctx.stream));
  ctx.sync_main();  // h is a host temporary
  return out;
}

struct ColumnOut {
  DTensor t1;  // (pb, pk, a, rank) replicated
  DTensor t2;  // (rank, b, c, t_r, e, f) local slice
};

// Thrown by the stream-ordered column when a big-side Gram matrix turned out
// deficient (its completed basis needs the global rows): the column is redone
// on the robust path.  Every rank sees the same flags (the Gram matrices are
// all-reduced, the factors replicated), so every rank redoes it.
struct RedoColumn {};

// One column einsumsvd split along t (see the file comment) -- the robust
// form: every orthogonalisation checked on the host as it happens, deficient
// big-side Gram matrices completed on the gathered rows.
ColumnOut sharded_column_robust(Ctx& ctx, const DTensor& v_r, const DTensor& S, const DTensor& bra,
                                const DTensor& ket, std::pair<int64_t, int64_t> s_range, const Trunc& policy,
                                int absorb, const Rsvd& cfg, bool fast) {
  NcclComm& cm = need_comm(ctx);
  const auto& vs = v_r.shape;  // (a, p, q, s_r, m, n)
  const auto& bs = bra.shape;  // (d, u, m, b, e)
  const auto& ks = ket.shape;  // (d, v, n, c, f)
  const int64_t T = S.shape[3], s_full = S.shape[2];
  const int64_t rows = vs[0] * vs[1] * vs[2], cols = bs[3] * ks[3] * T * bs[4] * ks[4];
  const int64_t mindim = std::min(rows, cols);
  const int64_t target = std::min<int64_t>(policy.max_rank ? static_cast<int64_t>(std::min<uint64_t>(
                                                                 policy.max_rank, static_cast<uint64_t>(mindim)))
                                                           : mindim,
                                           mindim);
  const int64_t k = std::min<int64_t>(target + static_cast<int64_t>(effective_oversample(cfg, target)), mindim);
  auto [t0, t1] = shard_range(T, cm.world, cm.rank);
  auto [s0, s1] = s_range;

  const DTensor S_t = slice(ctx, S, 3, t0, t1);

  auto apply = [&](const DTensor& x) {  // x (b, e, c, t_r, f, X) -> Y (a, p, q, X), replicated
    // intermediate orders chosen so that every contracted group is one
    // uniform-stride block of both operands (no re-layout of the big tensors)
    DTensor w1 = contract(ctx, "dumbe,bectfX->dcfumtX", {bra, x}, {true, false});
    DTensor w2 = contract(ctx, "dvncf,dcfumtX->uvtnmX", {ket, w1}, {false, false});
    DTensor w3 = contract(ctx, "uvst,uvtnmX->smnX", {S_t, w2}, {false, false});
    allreduce(ctx, w3);
    DTensor w3s = slice(ctx, w3, 0, s0, s1);
    DTensor y = contract(ctx, "apqsmn,smnX->apqX", {v_r, w3s}, {false, false});
    allreduce(ctx, y);
    return y;
  };
  auto adjoint_rest = [&](DTensor r) {  // r_r (s_r, m, n, X) -> Z_r (b, e, c, t_r, f, X)
    r = allgather_axis(ctx, r, 0, s_full);
    DTensor w2 = contract(ctx, "uvst,smnX->vnumtX", {S_t, r}, {true, false});
    DTensor w1 = contract(ctx, "dvncf,vnumtX->dumctfX", {ket, w2}, {true, false});
    return contract(ctx, "dumbe,dumctfX->bectfX", {bra, w1}, {false, false});
  };
  auto adjoint = [&](const DTensor& p) {  // p (a, p, q, X) replicated -> Z_r (b, e, c, t_r, f, X)
    return adjoint_rest(contract(ctx, "apqsmn,apqX->smnX", {v_r, p}, {true, false}));
  };
  // fast: stream-ordered orthogonalisations (one host sync per column, at the
  // projected SVD); deficiency and status flags are checked there
  std::vector<BufPtr> def_flags;
  auto orth_small = [&](const DTensor& y) { return fast ? orth_async(ctx, y) : gram_orthogonalize(ctx, y, 3).first; };
  auto orth_big = [&](const DTensor& z) {
    DTensor g = gram_matrix(ctx, z);
    allreduce(ctx, g);
    if (fast) {
      GramFactorsAsync fa = gram_factors_async(ctx, g);
      def_flags.push_back(fa.flags);
      return contract(ctx, "bectfX,XY->bectfY", {z, fa.P}, {false, false});
    }
    GramFactorsD f = gram_factors_full(ctx, g);
    if (std::any_of(f.deficient.begin(), f.deficient.end(), [](int d) { return d != 0; })) {
      // orthonormal completion needs the global rows: gather, complete, re-slice
      DTensor q = gram_orthogonalize(ctx, allgather_axis(ctx, z, 3, T), 5).first;
      return slice(ctx, q, 3, t0, t1);
    }
    return contract(ctx, "bectfX,XY->bectfY", {z, f.P}, {false, false});
  };

  // Omega_r stored in the (b, e, c, t_r, f, X) order GEMM (1) reads, each
  // element the reference's random_tensor value at its logical (b,c,t,e,f,X)
  // index (counter-based: bit-identical to the unsharded sketch's t-slice)
  DTensor omega = ctx.empty({bs[3], bs[4], ks[3], t1 - t0, ks[4], k});
  {
    const std::vector<int64_t> full = {bs[3], ks[3], T, bs[4], ks[4], k};
    const std::vector<int64_t> fstr = row_major_strides(full);
    const std::vector<int64_t> lstr = {fstr[0], fstr[3], fstr[1], fstr[2], fstr[4], fstr[5]};
    random_fill(omega.data(), 6, omega.shape.data(), lstr.data(), cfg.seed, 0, ctx.stream,
                static_cast<uint64_t>(t0) * static_cast<uint64_t>(fstr[2]));
    ++ctx.launches;
  }
  // fast: A orth(Z) = (A Z) P by linearity in the probe index -- the Gram
  // matrix is all-reduced on the main stream, then its k x k eigensolver runs
  // there while A Z (with its own collectives) runs on the side stream; the big
  // Q_r = Z_r P product is never formed.  Deficient Gram matrices (completed
  // bases are not of the form Z P) are caught at the column's end -> robust redo.
  auto apply_orth = [&](const DTensor& z) {
    if (!fast) return apply(orth_big(z));
    DTensor g = gram_matrix(ctx, z);
    allreduce(ctx, g);
    ctx.fork();
    GramFactorsAsync fa = gram_factors_async(ctx, g);
    def_flags.push_back(fa.flags);
    ctx.side();
    DTensor az = apply(z);
    ctx.join();
    return contract(ctx, "apqX,XY->apqY", {az, fa.P}, {false, false});
  };
  // fast, small side: A^* orth(Y) = (A^* Y) P likewise -- Y's Gram and
  // eigensolver on the main stream while the first adjoint step v_r^* Y runs on
  // the side stream; the basis P_m = Y P itself is formed (cheap: rows_Y x k x k)
  DTensor pm;
  auto adjoint_orth = [&](const DTensor& y) {
    if (!fast) {
      pm = orth_small(y);
      return adjoint(pm);
    }
    DTensor g = gram_matrix(ctx, y);
    ctx.fork();
    GramFactorsAsync fa = gram_factors_async(ctx, g);
    def_flags.push_back(fa.flags);
    ctx.side();
    DTensor r0 = contract(ctx, "apqsmn,apqX->smnX", {v_r, y}, {true, false});
    ctx.join();
    pm = contract(ctx, "apqX,XY->apqY", {y, fa.P}, {false, false});
    return adjoint_rest(contract(ctx, "smnX,XY->smnY", {r0, fa.P}, {false, false}));
  };
  DTensor z = adjoint_orth(apply(omega));
  for (int it = 0; it < cfg.power_iters; ++it) z = adjoint_orth(apply_orth(z));
  if (fast) {
    // status bits of every orthogonalisation so far + the deficiency flags,
    // read back with the projected SVD's synchronisation below
    const int nf = static_cast<int>(def_flags.size());
    PEPSB_CUDA(cudaMemcpyAsync(ctx.h_status + 20, ctx.d_status, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
    for (int i = 0; i < nf && i < 16; ++i)  // the "any" flag sits after the k per-column flags
      PEPSB_CUDA(cudaMemcpyAsync(ctx.h_status + 21 + i, reinterpret_cast<int*>(def_flags[i]->p) + k, sizeof(int),
                                 cudaMemcpyDeviceToHost, ctx.stream));
  }

  // projected SVD of B = P^H A = Z^H (decomposition.cpp:293-306) by the Gram route
  DTensor g = gram_matrix(ctx, z);
  allreduce(ctx, g);
  GramFactorsD f = gram_factors_full(ctx, g);  // synchronises
  if (fast) {
    read_status_bits(ctx.h_status[20]);
    for (int i = 0; i < static_cast<int>(def_flags.size()) && i < 16; ++i)
      if (ctx.h_status[21 + i]) throw RedoColumn{};
  }
  std::vector<double> s(static_cast<size_t>(k));
  for (int64_t j = 0; j < k; ++j) s[j] = std::sqrt(std::max(f.lam[j], 0.0));
  std::vector<double2> ut(static_cast<size_t>(k * k));
  DTensor utd = f.vecs;
  const int64_t tgt = std::max<int64_t>(1, std::min(target, k));
  if (!(s[0] > 0.0 && s[tgt - 1] >= 1e-4 * s[0])) {
    // ill-conditioned Gram route: the single-device projected SVD on the gathered Z
    auto pr = projected_svd_full(ctx, allgather_axis(ctx, z, 3, T), target);
    utd = pr.first;
    s = pr.second;
  }
  PEPSB_CUDA(cudaMemcpyAsync(ut.data(), utd.data(), ut.size() * 16, cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync_main();
  const int64_t rank = std::min<int64_t>(static_cast<int64_t>(retained_rank(s, policy)), target);
  std::vector<double> wl(rank), wv(rank);
  for (int64_t j = 0; j < rank; ++j) {
    const double sj = s[j];
    const double l = absorb == kSplit ? std::sqrt(sj) : absorb == kLeft ? sj : 1.0;
    const double r = absorb == kSplit ? std::sqrt(sj) : absorb == kRight ? sj : 1.0;
    wl[j] = l;
    wv[j] = sj > 0.0 ? r / sj : 0.0;
  }
  ColumnOut out;
  out.t1 = contract(ctx, "apqX,XR->pqaR", {pm, scaled_columns(ctx, ut, k, rank, wl, false)}, {false, false});
  out.t2 = contract(ctx, "bectfX,XR->Rbctef", {z, scaled_columns(ctx, ut, k, rank, wv, true)}, {true, false});
  return out;
}

ColumnOut sharded_column(Ctx& ctx, const DTensor& v_r, const DTensor& S, const DTensor& bra, const DTensor& ket,
                         std::pair<int64_t, int64_t> s_range, const Trunc& policy, int absorb, const Rsvd& cfg) {
  PEPSB_CUDA(cudaMemsetAsync(ctx.d_status, 0, 2 * sizeof(int), ctx.stream));
  if (2 * cfg.power_iters + 1 > 16)  // more deficiency flags than the read-back slots
    return sharded_column_robust(ctx, v_r, S, bra, ket, s_range, policy, absorb, cfg, false);
  try {
    return sharded_column_robust(ctx, v_r, S, bra, ket, s_range, policy, absorb, cfg, true);
  } catch (const RedoColumn&) {
    ++ctx.faithful_redos;  // counter "faithful_redos": columns redone on the robust path
    PEPSB_CUDA(cudaMemsetAsync(ctx.d_status, 0, 2 * sizeof(int), ctx.stream));
    return sharded_column_robust(ctx, v_r, S, bra, ket, s_range, policy, absorb, cfg, false);
  }
}

uint64_t column_seed(const ContractOptD& opt, uint64_t tag, int row, int col) {
  return derive_seed1(derive_seed1(derive_seed1(opt.seed, tag), static_cast<uint64_t>(row)),
                      static_cast<uint64_t>(col));
}

}  // namespace

BoundaryD two_layer_apply_row_sharded(Ctx& ctx, const BoundaryD& top, const PepsStateD& bra, const PepsStateD& ket,
                                      int row, const ContractOptD& opt, uint64_t seed_tag) {
  NcclComm& cm = need_comm(ctx);
  if (opt.strategy != kImplicitRsvd) throw Error(kConfigError, "the sharded row absorb needs implicit_rsvd");
  const int n = bra.cols;
  const int absorb = opt.canonicalize ? (row % 2 ? kRight : kLeft) : kSplit;
  Trunc policy = opt.trunc;
  if (policy.max_rank == 0) policy.max_rank = UINT64_MAX;
  BoundaryD out;
  out.sites.resize(n);
  for (int c = 0; c < n; ++c) out.phys.emplace_back(bra.site(row, c).shape[3], ket.site(row, c).shape[3]);

  // first column: contract_network({s0, bra*, ket}) -> (b, c, s, e, f) (contraction.cpp:283-288), replicated
  const DTensor& s0 = top.sites[0];
  DTensor s0s = reshaped(s0, {top.phys[0].first, top.phys[0].second, s0.shape[1], s0.shape[2]});
  DTensor v = contract(ctx, "uvls,dumbe,dvncf->bcsef", {s0s, bra.site(row, 0), ket.site(row, 0)},
                       {false, true, false});
  v = reshaped(v, {1, v.shape[0], v.shape[1], v.shape[2], v.shape[3], v.shape[4]});
  bool sharded = false;
  std::pair<int64_t, int64_t> s_range{0, 0};
  for (int c = 1; c < n; ++c) {
    const DTensor& sc = top.sites[c];
    DTensor S = reshaped(sc, {top.phys[c].first, top.phys[c].second, sc.shape[1], sc.shape[2]});
    const int64_t T = sc.shape[2];
    Rsvd cfg = opt.rsvd;
    cfg.seed = column_seed(opt, seed_tag, row, c);
    DTensor t1;
    if (T >= cm.world) {
      if (!sharded) {
        s_range = shard_range(v.shape[3], cm.world, cm.rank);
        v = slice(ctx, v, 3, s_range.first, s_range.second);
      }
      ColumnOut col = sharded_column(ctx, v, S, bra.site(row, c), ket.site(row, c), s_range, policy, absorb, cfg);
      t1 = col.t1;
      v = col.t2;
      sharded = true;
      s_range = shard_range(T, cm.world, cm.rank);
    } else {
      if (sharded) {
        v = allgather_axis(ctx, v, 3, S.shape[2]);
        sharded = false;
      }
      ImplicitOp net({v, S, bra.site(row, c), ket.site(row, c)}, {"apqsmn", "uvst", "dumbe", "dvncf"}, "apq",
                     "bctef", {false, false, true, false});
      EinsumsvdResultD split = einsumsvd(ctx, net, policy, opt.strategy, absorb, cfg, {1, 2, 0, 3});
      t1 = split.t1;  // (pb, pk, a, rho)
      v = split.t2;
    }
    const auto& ts = t1.shape;
    out.sites[c - 1] = reshaped(t1, {ts[0] * ts[1], ts[2], ts[3]});
  }
  if (sharded) v = allgather_axis(ctx, v, 3, top.sites[n - 1].shape[2]);
  // last = v.permute({1,2,0,3,4,5}) -> (pb*pk, rho, t*e*f)
  LTensor last = reduce_to(ctx, as_labelled(v, "abcdef"), "bcadef");
  DTensor lastd = materialize(ctx, last, last.labels);
  const auto& ls = lastd.shape;
  out.sites[n - 1] = reshaped(lastd, {ls[0] * ls[1], ls[2], ls[3] * ls[4] * ls[5]});
  out.validate();
  return out;
}

std::pair<double, double> contract_two_layer_sharded(Ctx& ctx, const PepsStateD& bra, const PepsStateD& ket,
                                                     const ContractOptD& opt) {
  if (bra.rows != ket.rows || bra.cols != ket.cols || bra.d != ket.d)
    throw Error(kValidationError, "two-layer contraction needs matching grids");
  BoundaryD s = two_layer_first_row(ctx, bra, ket);
  for (int r = 1; r < bra.rows; ++r) s = two_layer_apply_row_sharded(ctx, s, bra, ket, r, opt, kTagTop);
  return chain_scalar(ctx, s);
}

}  // namespace pepsb
