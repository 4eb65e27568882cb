// Two-layer boundary contraction, cached environments and band zipper on the
// device.  Semantics follow proj/src/contraction.cpp:254-338,345-650,
// proj/src/mps.cpp:102-110 and proj/src/observables.cpp:261-333; every
// contraction runs through the device engine, every truncation through the
// device einsumsvd.  Tensors stay resident in HBM between calls.
#include "peps.h"

#include <algorithm>
#include <exception>
#include <memory>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <cmath>
#include <map>
#include <cstdio>
#include <cstring>

#include "tensor_ops.cuh"

namespace pepsb {

namespace {

DTensor reshape(const DTensor& t, std::vector<int64_t> shape) {
  int64_t n = 1;
  for (auto e : shape) n *= e;
  if (n != t.size()) throw Error(kShapeError, "reshape changes element count");
  DTensor r = t;
  r.shape = std::move(shape);
  return r;
}

LTensor scalar_one(Ctx& ctx) {
  LTensor l;
  l.buf = ctx.alloc(1);
  l.ptr = l.buf->p;
  const double one[2] = {1.0, 0.0};
  PEPSB_CUDA(cudaMemcpyAsync(l.buf->p, one, sizeof(one), cudaMemcpyHostToDevice, ctx.stream));
  return l;
}

std::pair<double, double> read_scalar(Ctx& ctx, const LTensor& t) {
  if (t.size() != 1) throw Error(kShapeError, "scalar_value on non-scalar tensor");
  double v[2];
  PEPSB_CUDA(cudaMemcpyAsync(v, t.ptr, sizeof(v), cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
  return {v[0], v[1]};
}

}  // namespace

void PepsStateD::validate() const {
  if (rows <= 0 || cols <= 0) throw Error(kValidationError, "PEPS grid must be non-empty");
  if (static_cast<int>(sites.size()) != rows * cols) throw Error(kShapeError, "site count does not match grid");
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) {
      const auto& t = site(r, c).shape;
      if (t.size() != 5) throw Error(kShapeError, "PEPS site must be order 5");
      if (t[0] != d) throw Error(kShapeError, "physical dimension mismatch");
      if (r == 0 && t[1] != 1) throw Error(kShapeError, "top boundary bond must be 1");
      if (c == 0 && t[2] != 1) throw Error(kShapeError, "left boundary bond must be 1");
      if (r == rows - 1 && t[3] != 1) throw Error(kShapeError, "bottom boundary bond must be 1");
      if (c == cols - 1 && t[4] != 1) throw Error(kShapeError, "right boundary bond must be 1");
      if (r + 1 < rows && t[3] != site(r + 1, c).shape[1]) throw Error(kShapeError, "vertical bond mismatch");
      if (c + 1 < cols && t[4] != site(r, c + 1).shape[2]) throw Error(kShapeError, "horizontal bond mismatch");
    }
}

void BoundaryD::validate() const {
  if (sites.empty()) throw Error(kShapeError, "empty MPS");
  if (sites.front().shape[1] != 1 || sites.back().shape[2] != 1)
    throw Error(kShapeError, "MPS boundary bonds must have extent 1");
  for (size_t i = 0; i + 1 < sites.size(); ++i)
    if (sites[i].shape[2] != sites[i + 1].shape[1])
      throw Error(kShapeError, "MPS bond mismatch between sites " + std::to_string(i) + " and " + std::to_string(i + 1));
}

// contraction.cpp:254-267: site = contract("dulbr,dULBR->bBlLrR", bra*, ket) reshaped.
BoundaryD two_layer_first_row(Ctx& ctx, const PepsStateD& bra, const PepsStateD& ket) {
  BoundaryD out;
  for (int c = 0; c < bra.cols; ++c) {
    const DTensor& b = bra.site(0, c);
    const DTensor& k = ket.site(0, c);
    LTensor t = contract_network(ctx, {as_labelled(b, "dulbr", true), as_labelled(k, "dULBR")}, "bBlLrR");
    DTensor site = materialize(ctx, t, t.labels);
    out.sites.push_back(reshape(site, {b.shape[3] * k.shape[3], b.shape[2] * k.shape[2], b.shape[4] * k.shape[4]}));
    out.phys.emplace_back(b.shape[3], k.shape[3]);
  }
  return out;
}

namespace {

// Thrown by a consumer whose producer failed: never the root cause, so the
// pipeline rethrows the producer's own error instead when there is one.
struct PipelineAborted : Error {
  PipelineAborted() : Error(kOtherError, "row pipeline: producer failed") {}
};

void rethrow_root_cause(const std::vector<std::exception_ptr>& errs) {
  std::exception_ptr sentinel;
  for (auto& e : errs) {
    if (!e) continue;
    try {
      std::rethrow_exception(e);
    } catch (const PipelineAborted&) {
      sentinel = e;
    } catch (...) {
      throw;
    }
  }
  if (sentinel) std::rethrow_exception(sentinel);
}

// A boundary row produced on one context and read on another (the row
// pipeline of contract_two_layer): site c is published, with an event on the
// producer's stream, as soon as its computation is enqueued; the consumer
// waits for the host flag and makes its own stream wait for the event.
struct Handoff {
  explicit Handoff(int n) : sites(n), ev(n, nullptr), ready(n, 0) {}
  ~Handoff() {
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
  }
  std::vector<DTensor> sites;
  std::vector<std::pair<int64_t, int64_t>> phys;
  std::vector<cudaEvent_t> ev;
  std::vector<char> ready;
  std::mutex m;
  std::condition_variable cv;
  bool failed = false;
  void publish(Ctx& ctx, int c, const DTensor& t) {
    cudaEvent_t e;
    PEPSB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    PEPSB_CUDA(cudaEventRecord(e, ctx.stream));
    {
      std::lock_guard<std::mutex> g(m);
      sites[c] = t;
      ev[c] = e;
      ready[c] = 1;
    }
    cv.notify_all();
  }
  const DTensor& acquire(Ctx& ctx, int c) {
    std::unique_lock<std::mutex> g(m);
    cv.wait(g, [&] { return ready[c] || failed; });
    if (!ready[c]) throw PipelineAborted();
    PEPSB_CUDA(cudaStreamWaitEvent(ctx.stream, ev[c], 0));
    return sites[c];
  }
  void fail() {
    {
      std::lock_guard<std::mutex> g(m);
      failed = true;
    }
    cv.notify_all();
  }
};

// contraction.cpp:269-311, reading the top boundary from `top` or (pipeline)
// from the handoff `tin`, and publishing the emitted sites into `hout`.
BoundaryD apply_row_impl(Ctx& ctx, const BoundaryD* top, Handoff* tin, const PepsStateD& bra, const PepsStateD& ket,
                         int row, const ContractOptD& opt, uint64_t seed_tag, Handoff* hout) {
  const int n = bra.cols;
  BoundaryD out;
  out.sites.resize(n);
  for (int c = 0; c < n; ++c) out.phys.emplace_back(bra.site(row, c).shape[3], ket.site(row, c).shape[3]);
  const int absorb = opt.canonicalize ? (row % 2 ? kRight : kLeft) : kSplit;
  ctx.lookahead.reset();
  auto top_site = [&](int c) -> const DTensor& { return tin ? tin->acquire(ctx, c) : top->sites[c]; };
  const auto& tphys = tin ? tin->phys : top->phys;
  auto emit = [&](int c, const DTensor& t) {
    out.sites[c] = t;
    if (hout) hout->publish(ctx, c, t);
  };

  // pending v: (a, bra-down, ket-down, mps bond, bra-right, ket-right)
  const DTensor& s0 = top_site(0);
  DTensor s0s = reshape(s0, {tphys[0].first, tphys[0].second, s0.shape[1], s0.shape[2]});
  LTensor v0 = contract_network(
      ctx, {as_labelled(s0s, "uvls"), as_labelled(bra.site(row, 0), "dumbe", true), as_labelled(ket.site(row, 0), "dvncf")},
      "bcsef");
  DTensor v = materialize(ctx, v0, v0.labels);
  v = reshape(v, {1, v.shape[0], v.shape[1], v.shape[2], v.shape[3], v.shape[4]});

  for (int c = 1; c < n; ++c) {
    const DTensor& sc = top_site(c);
    DTensor scs = reshape(sc, {tphys[c].first, tphys[c].second, sc.shape[1], sc.shape[2]});
    ImplicitOp net({v, scs, bra.site(row, c), ket.site(row, c)}, {"apqsmn", "uvst", "dumbe", "dvncf"}, "apq", "bctef",
                   {false, false, true, false});
    Trunc policy = opt.trunc;
    if (policy.max_rank == 0) policy.max_rank = UINT64_MAX;
    Rsvd cfg = opt.rsvd;
    auto col_seed = [&](int col) {
      return derive_seed1(derive_seed1(derive_seed1(opt.seed, seed_tag), static_cast<uint64_t>(row)),
                          static_cast<uint64_t>(col));
    };
    cfg.seed = col_seed(c);
    if (c + 1 < n && opt.strategy == kImplicitRsvd) {
      // next column's operator with its pending tensor guessed at full rank
      // (this column's target); reused only if the guess holds
      const int64_t mindim = std::min(net.row_extent(), net.col_extent());
      const int64_t rho = static_cast<int64_t>(std::min<uint64_t>(policy.max_rank, static_cast<uint64_t>(mindim)));
      const auto& bs = bra.site(row, c).shape;
      const auto& ks = ket.site(row, c).shape;
      DTensor vg;
      vg.shape = {rho, bs[3], ks[3], sc.shape[2], bs[4], ks[4]};
      const DTensor& sn = top_site(c + 1);
      DTensor sns = reshape(sn, {tphys[c + 1].first, tphys[c + 1].second, sn.shape[1], sn.shape[2]});
      set_lookahead(ctx,
                    ImplicitOp({vg, sns, bra.site(row, c + 1), ket.site(row, c + 1)},
                               {"apqsmn", "uvst", "dumbe", "dvncf"}, "apq", "bctef", {false, false, true, false}),
                    col_seed(c + 1));
    }
    // t1 (a, pb, pk, rho) written directly as (pb, pk, a, rho)
    EinsumsvdResultD split = einsumsvd(ctx, net, policy, opt.strategy, absorb, cfg, {1, 2, 0, 3});
    const auto& t1 = split.t1.shape;
    emit(c - 1, reshape(split.t1, {t1[0] * t1[1], t1[2], t1[3]}));
    v = split.t2;  // (rho, b, c, t, e, f)
  }
  ctx.lookahead.reset();
  // last = v.permute({1,2,0,3,4,5}) -> (pb*pk, rho, t*e*f)
  LTensor last = reduce_to(ctx, as_labelled(v, "abcdef"), "bcadef");
  DTensor lastd = materialize(ctx, last, last.labels);
  const auto& ls = lastd.shape;
  emit(n - 1, reshape(lastd, {ls[0] * ls[1], ls[2], ls[3] * ls[4] * ls[5]}));
  out.validate();
  if (ctx.trace) {
    fprintf(stderr, "[pepsb] row %d: host alloc %.2f ms, free %.2f ms, sync-wait %.2f ms (cumulative)\n", row,
            ctx.t_alloc * 1e3, ctx.t_free * 1e3, ctx.t_sync * 1e3);
  }
  return out;
}

}  // namespace

// contraction.cpp:269-311
BoundaryD two_layer_apply_row(Ctx& ctx, const BoundaryD& top, const PepsStateD& bra, const PepsStateD& ket, int row,
                              const ContractOptD& opt, uint64_t seed_tag) {
  return apply_row_impl(ctx, &top, nullptr, bra, ket, row, opt, seed_tag, nullptr);
}

std::pair<double, double> chain_scalar(Ctx& ctx, const BoundaryD& b) {
  b.validate();
  LTensor t = scalar_one(ctx);
  t.labels = "l";
  t.ext = {1};
  t.str = {1};
  for (const auto& site : b.sites) {
    if (site.shape[0] != 1) throw Error(kShapeError, "chain_scalar requires physical extents 1");
    LTensor s = as_labelled(site, "plr");
    t = contract_network(ctx, {t, s}, "r");
    t.labels = "l";
  }
  t.labels = "";
  t.ext.clear();
  t.str.clear();
  return read_scalar(ctx, t);
}

// Row pipeline (contraction.cpp:313-338 / observables.cpp:272-281): row r's
// column c reads only the top-boundary site c (+1 for the lookahead), which row
// r-1 emits at its column c+1, so K consecutive rows run concurrently a few
// columns apart on K contexts driven by K host threads (row r on context
// (r-1) mod K; ctxs[0] is the caller's).  Each row is the same kernel sequence
// with the same seeds, so every boundary is bitwise that of the sequential
// sweep.  keep_all: return every row's boundary (the cache), else only the last.
std::vector<BoundaryD> pipelined_sweep(const std::vector<Ctx*>& ctxs, const PepsStateD& bra, const PepsStateD& ket,
                                       const ContractOptD& opt, uint64_t tag, bool keep_all) {
  Ctx& ctx = *ctxs[0];
  const int K = static_cast<int>(ctxs.size());
  const int rows = bra.rows, n = bra.cols;
  BoundaryD first = two_layer_first_row(ctx, bra, ket);
  std::vector<std::unique_ptr<Handoff>> H(rows);
  for (int r = 0; r < rows; ++r) {
    H[r] = std::make_unique<Handoff>(n);
    for (int c = 0; c < n; ++c) H[r]->phys.emplace_back(bra.site(r, c).shape[3], ket.site(r, c).shape[3]);
  }
  for (int c = 0; c < n; ++c) H[0]->publish(ctx, c, first.sites[c]);
  std::vector<uint64_t> f0(K), l0(K);
  for (int i = 1; i < K; ++i) {
    f0[i] = ctxs[i]->flops;
    l0[i] = static_cast<uint64_t>(ctxs[i]->launches);
    // helpers start after everything enqueued on the caller's stream so far
    cudaEvent_t ev = ctx.take_event();
    PEPSB_CUDA(cudaEventRecord(ev, ctx.stream));
    PEPSB_CUDA(cudaStreamWaitEvent(ctxs[i]->stream, ev, 0));
    ctx.event_pool.push_back(ev);
  }
  auto work = [&](int idx) {
    Ctx& cx = *ctxs[idx];
    for (int r = 1 + idx; r < rows; r += K) {
      apply_row_impl(cx, nullptr, H[r - 1].get(), bra, ket, r, opt, tag, H[r].get());
      if (!keep_all) {
        cx.sync();  // row r - 1 is no longer read: its blocks may return to their pool
        H[r - 1]->sites.assign(n, DTensor());
      }
    }
    cx.sync();
  };
  std::vector<std::exception_ptr> err(K);
  std::vector<std::thread> threads;
  for (int i = 1; i < K; ++i)
    threads.emplace_back([&, i] {
      try {
        PEPSB_CUDA(cudaSetDevice(ctxs[i]->device));
        work(i);
      } catch (...) {
        err[i] = std::current_exception();
        for (auto& h : H) h->fail();
      }
    });
  try {
    work(0);
  } catch (...) {
    err[0] = std::current_exception();
    for (auto& h : H) h->fail();
  }
  for (auto& t : threads) t.join();
  rethrow_root_cause(err);
  for (int i = 1; i < K; ++i) {
    ctx.flops += ctxs[i]->flops - f0[i];
    ctx.launches += static_cast<int64_t>(static_cast<uint64_t>(ctxs[i]->launches) - l0[i]);
  }
  std::vector<BoundaryD> out;
  for (int r = keep_all ? 0 : rows - 1; r < rows; ++r) {
    BoundaryD b;
    b.phys = r == 0 ? first.phys : H[r]->phys;
    for (int c = 0; c < n; ++c) b.sites.push_back(H[r]->acquire(ctx, c));
    out.push_back(std::move(b));
  }
  return out;
}

// Rows in flight: option "pipeline_rows" (< 2 sequential), or automatic
// (-1): 4 for small boundary bonds (m <= 48: latency-bound einsumsvds, the
// one-block eigensolver dominates), 3 otherwise.  Measured (round 2,
// tools/pipeline_ab.py): config 3 (m = 36) 0.329 / 0.287 / 0.271 / 0.268 /
// 0.267 s per norm at K = 2 / 3 / 4 / 6 / 8; config 5 (m = 64) 9.67 / 8.46 /
// 8.38 s at K = 1 / 2 / 3.  Results are bitwise independent of K.
int pipeline_depth(const Ctx& ctx, const ContractOptD& opt) {
  if (ctx.pipeline_rows >= 0) return ctx.pipeline_rows;
  return (opt.trunc.max_rank != 0 && opt.trunc.max_rank <= 48) ? 4 : 3;
}

std::vector<Ctx*> pipeline_contexts(Ctx& ctx, int K) {
  std::vector<Ctx*> out{&ctx};
  while (static_cast<int>(ctx.helpers.size()) < K - 1) {
    ctx.helpers.push_back(std::make_unique<Ctx>(ctx.device));
    ctx.helpers.back()->pipeline_rows = 0;
    ctx.helpers.back()->concurrent_sweeps = 0;
  }
  for (int i = 0; i < K - 1; ++i) {
    Ctx& h = *ctx.helpers[i];
    h.overlap = ctx.overlap;
    h.orth_mode = ctx.orth_mode;
    out.push_back(&h);
  }
  return out;
}

// contraction.cpp:313-338 (rows pipelined, see pipelined_sweep)
std::pair<double, double> contract_two_layer(Ctx& ctx, const PepsStateD& bra, const PepsStateD& ket,
                                             const ContractOptD& opt) {
  if (bra.rows != ket.rows || bra.cols != ket.cols || bra.d != ket.d)
    throw Error(kValidationError, "two-layer contraction needs matching grids");
  const int rows = bra.rows, n = bra.cols;
  // (tiny lattices: extra threads and contexts cost more than they hide)
  if (pipeline_depth(ctx, opt) < 2 || rows < 3 || rows * n < 64) {
    BoundaryD s = two_layer_first_row(ctx, bra, ket);
    for (int r = 1; r < rows; ++r) s = two_layer_apply_row(ctx, s, bra, ket, r, opt, kTagTop);
    return chain_scalar(ctx, s);
  }
  const int K = std::min(pipeline_depth(ctx, opt), rows - 1);
  std::vector<BoundaryD> last = pipelined_sweep(pipeline_contexts(ctx, K), bra, ket, opt, kTagTop, false);
  return chain_scalar(ctx, last.back());
}

// observables.cpp:261-270: reverse rows, swap up/down.
PepsStateD flip_vertical(Ctx& ctx, const PepsStateD& s) {
  PepsStateD f;
  f.rows = s.rows;
  f.cols = s.cols;
  f.d = s.d;
  for (int r = s.rows - 1; r >= 0; --r)
    for (int c = 0; c < s.cols; ++c) {
      // site axes (phys, up, left, down, right) -> (phys, down, left, up, right)
      LTensor t = reduce_to(ctx, as_labelled(s.site(r, c), "puldr"), "pdlur");
      f.sites.push_back(materialize(ctx, t, t.labels));
    }
  return f;
}

namespace {
// sweep_boundaries (observables.cpp:272-281)
std::vector<BoundaryD> sweep_boundaries(Ctx& ctx, const PepsStateD& s, const ContractOptD& opt, uint64_t tag) {
  std::vector<BoundaryD> out;
  out.push_back(two_layer_first_row(ctx, s, s));
  for (int r = 1; r < s.rows; ++r) out.push_back(two_layer_apply_row(ctx, out.back(), s, s, r, opt, tag));
  return out;
}
}  // namespace

// observables.cpp:325-333.  The two sweeps are independent: the
// bottom one (flipped state, tag 0x21) runs on a helper context driven by a
// second host thread, so the latency-bound stretches of one sweep (one-block
// eigensolvers, host syncs) overlap the other's GEMMs.  Each sweep is the same
// sequence of kernels either way, so the cache is bitwise unchanged.
RowCacheD build_row_cache(Ctx& ctx, const PepsStateD& s, const ContractOptD& opt) {
  RowCacheD cache;
  std::vector<BoundaryD> fb;
  const bool pipe = pipeline_depth(ctx, opt) >= 2 && s.rows >= 3 && s.rows * s.cols >= 64;
  const int K = pipe ? std::min(pipeline_depth(ctx, opt), s.rows - 1) : 1;
  const bool concurrent = ctx.concurrent_sweeps > 0 ||
                          (ctx.concurrent_sweeps < 0 && opt.trunc.max_rank != 0 && opt.trunc.max_rank <= 48);
  if (concurrent && s.rows > 1) {
    // contexts: [ctx, helpers 0 .. K-2] run the top sweep, [helpers K-1 .. 2K-2]
    // the bottom one, from a second host thread
    std::vector<Ctx*> all = pipeline_contexts(ctx, 2 * K);
    std::vector<Ctx*> top(all.begin(), all.begin() + K), bot(all.begin() + K, all.end());
    Ctx& c2 = *bot[0];
    cudaEvent_t ev = ctx.take_event();
    PEPSB_CUDA(cudaEventRecord(ev, ctx.stream));
    PEPSB_CUDA(cudaStreamWaitEvent(c2.stream, ev, 0));
    ctx.event_pool.push_back(ev);
    const uint64_t f0 = c2.flops, l0 = static_cast<uint64_t>(c2.launches);
    std::exception_ptr err;
    std::thread bottom([&] {
      try {
        PEPSB_CUDA(cudaSetDevice(c2.device));
        PepsStateD fl = flip_vertical(c2, s);
        fb = K > 1 ? pipelined_sweep(bot, fl, fl, opt, kTagBottom, true) : sweep_boundaries(c2, fl, opt, kTagBottom);
        c2.sync();
      } catch (...) {
        err = std::current_exception();
      }
    });
    try {
      cache.tops = K > 1 ? pipelined_sweep(top, s, s, opt, kTagTop, true) : sweep_boundaries(ctx, s, opt, kTagTop);
    } catch (...) {
      bottom.join();
      throw;
    }
    bottom.join();
    if (err) std::rethrow_exception(err);
    ctx.flops += c2.flops - f0;
    ctx.launches += static_cast<int64_t>(static_cast<uint64_t>(c2.launches) - l0);
  } else {
    std::vector<Ctx*> top = pipeline_contexts(ctx, K);
    cache.tops = K > 1 ? pipelined_sweep(top, s, s, opt, kTagTop, true) : sweep_boundaries(ctx, s, opt, kTagTop);
    PepsStateD fl = flip_vertical(ctx, s);
    fb = K > 1 ? pipelined_sweep(top, fl, fl, opt, kTagBottom, true) : sweep_boundaries(ctx, fl, opt, kTagBottom);
  }
  cache.bots.resize(s.rows);
  for (int k = 0; k < s.rows; ++k) cache.bots[k] = fb[s.rows - 1 - k];
  return cache;
}

// ---------------------------------------------------------------------------- band zipper

namespace {

constexpr const char* kIn = "ABCDEFGHIJ";
constexpr const char* kOut = "MNOPQRSTUV";

struct Layout {
  bool top = false, bottom = false;
  int r0 = 0, r1 = 0;
  int nrows() const { return r1 - r0 + 1; }
  int roles() const { return (top ? 1 : 0) + 2 * nrows() + (bottom ? 1 : 0); }
  int top_role() const { return 0; }
  int bra_role(int br) const { return (top ? 1 : 0) + 2 * br; }
  int ket_role(int br) const { return (top ? 1 : 0) + 2 * br + 1; }
  int bottom_role() const { return roles() - 1; }
};

Layout make_layout(const BoundaryD* top, int r0, int r1, const BoundaryD* bottom) {
  if (r1 < r0 || r1 - r0 > 1) throw Error(kValidationError, "band must span one or two rows");
  Layout L;
  L.top = top != nullptr;
  L.bottom = bottom != nullptr;
  L.r0 = r0;
  L.r1 = r1;
  return L;
}

int partner_col(const std::vector<InsertionPieceD>& pieces, const InsertionPieceD* self, int id, bool* found) {
  int pc = self->col;
  *found = false;
  for (const auto& p : pieces) {
    if (&p == self) continue;
    for (int o : p.bond_ids)
      if (o == id) {
        pc = p.col;
        *found = true;
      }
  }
  return pc;
}

// Gate bonds carried across the cut after column c (contraction.cpp:506-529).
std::vector<int> active_gate_bonds(const std::vector<InsertionPieceD>& pieces, int c) {
  std::vector<int> out;
  for (const auto& p : pieces)
    for (int id : p.bond_ids) {
      int lo = p.col, hi = p.col;
      for (const auto& q : pieces) {
        if (&q == &p) continue;
        for (int o : q.bond_ids)
          if (o == id) {
            lo = std::min(lo, q.col);
            hi = std::max(hi, q.col);
          }
      }
      if (lo <= c && c < hi && std::find(out.begin(), out.end(), id) == out.end()) out.push_back(id);
    }
  std::sort(out.begin(), out.end());
  return out;
}

// Column-c transfer network of the band (contraction.cpp:371-474).  With
// `mirror`, column c is physical column n-1-c with left/right bonds swapped
// (the right pass of band_environment) — done by relabelling, not copying.
std::vector<LTensor> band_column(const Layout& L, const BoundaryD* top, const PepsStateD& bra, const PepsStateD& ket,
                                 const BoundaryD* bottom, const std::vector<InsertionPieceD>& pieces, int c,
                                 bool mirror, const std::vector<int>& in_gates, const std::vector<int>& out_gates,
                                 std::string& out_labels) {
  std::vector<LTensor> net;
  const int n = bra.cols;
  const int pc = mirror ? n - 1 - c : c;
  char dummy = '0';
  auto fresh = [&]() { return dummy++; };
  auto h_in = [&](int role) { return c == 0 ? fresh() : kIn[role]; };
  auto h_out = [&](int role) { return c + 1 == n ? fresh() : kOut[role]; };
  auto gate_in = [&](int id) {
    for (size_t i = 0; i < in_gates.size(); ++i)
      if (in_gates[i] == id) return kIn[L.roles() + i];
    throw Error(kShapeError, "gate bond not carried into this column");
  };
  auto gate_out = [&](int id) {
    for (size_t i = 0; i < out_gates.size(); ++i)
      if (out_gates[i] == id) return kOut[L.roles() + i];
    throw Error(kShapeError, "gate bond not carried out of this column");
  };
  auto lr = [&](char lft, char rgt) { return mirror ? std::string{rgt, lft} : std::string{lft, rgt}; };

  if (L.top) {
    const DTensor& t = top->sites[pc];
    DTensor v = reshape(t, {top->phys[pc].first, top->phys[pc].second, t.shape[1], t.shape[2]});
    char i = h_in(L.top_role()), o = h_out(L.top_role());
    net.push_back(as_labelled(v, std::string("uv") + lr(i, o)));
  }
  for (int br = 0; br < L.nrows(); ++br) {
    const int row = L.r0 + br;
    const char up_b = br == 0 ? (L.top ? 'u' : fresh()) : 'y';
    const char up_k = br == 0 ? (L.top ? 'v' : fresh()) : 'z';
    const bool last = br + 1 == L.nrows();
    const char dn_b = last ? (L.bottom ? 'k' : fresh()) : 'y';
    const char dn_k = last ? (L.bottom ? 'l' : fresh()) : 'z';
    const InsertionPieceD* piece = nullptr;
    for (const auto& p : pieces)
      if (p.row == row && p.col == pc) {
        if (piece) throw Error(kValidationError, "at most one insertion piece per site");
        piece = &p;
      }
    const char ph_b = br == 0 ? 'w' : 'i';
    const char ph_k = piece ? (br == 0 ? 'x' : 'j') : ph_b;
    {
      char i = h_in(L.bra_role(br)), o = h_out(L.bra_role(br));
      std::string lab = std::string{ph_b, up_b} + lr(i, o).substr(0, 1) + dn_b + lr(i, o).substr(1, 1);
      net.push_back(as_labelled(bra.site(row, pc), lab, true));
    }
    {
      char i = h_in(L.ket_role(br)), o = h_out(L.ket_role(br));
      std::string lab = std::string{ph_k, up_k} + lr(i, o).substr(0, 1) + dn_k + lr(i, o).substr(1, 1);
      net.push_back(as_labelled(ket.site(row, pc), lab));
    }
    if (piece) {
      std::string pl{ph_b, ph_k};
      for (int id : piece->bond_ids) {
        bool found = false;
        int partner = partner_col(pieces, piece, id, &found);
        if (!found) throw Error(kValidationError, "gate bond has no partner piece");
        if (partner == pc) pl += 'g';
        else if (partner > pc) pl += gate_out(id);
        else pl += gate_in(id);
      }
      net.push_back(as_labelled(piece->op, pl));
    }
  }
  if (L.bottom) {
    const DTensor& t = bottom->sites[pc];
    DTensor v = reshape(t, {bottom->phys[pc].first, bottom->phys[pc].second, t.shape[1], t.shape[2]});
    char i = h_in(L.bottom_role()), o = h_out(L.bottom_role());
    net.push_back(as_labelled(v, std::string("kl") + lr(i, o)));
  }
  out_labels.clear();
  for (int role = 0; role < L.roles(); ++role)
    if (c + 1 < n) out_labels += kOut[role];
  for (size_t i = 0; i < out_gates.size(); ++i) out_labels += kOut[L.roles() + i];
  return net;
}

std::string to_in(const std::string& s) {
  std::string o;
  for (char c : s) o += kIn[std::strchr(kOut, c) - kOut];
  return o;
}

LTensor band_step(Ctx& ctx, const Layout& L, const LTensor& l, const BoundaryD* top, const PepsStateD& bra,
                  const PepsStateD& ket, const BoundaryD* bottom, const std::vector<InsertionPieceD>& pieces, int c,
                  bool mirror, const std::vector<int>& in_g, const std::vector<int>& out_g) {
  std::string out;
  std::vector<LTensor> net = band_column(L, top, bra, ket, bottom, pieces, c, mirror, in_g, out_g, out);
  net.insert(net.begin(), l);
  LTensor r = contract_network(ctx, net, out);
  r.labels = to_in(r.labels);
  return r;
}

void check_state_pair(const PepsStateD& bra, const PepsStateD& ket) {
  if (bra.rows != ket.rows || bra.cols != ket.cols) throw Error(kValidationError, "band needs matching grids");
}

}  // namespace

std::pair<double, double> band_value(Ctx& ctx, const BoundaryD* top, const PepsStateD& bra, const PepsStateD& ket,
                                     int r0, int r1, const BoundaryD* bottom,
                                     const std::vector<InsertionPieceD>& pieces) {
  check_state_pair(bra, ket);
  Layout L = make_layout(top, r0, r1, bottom);
  LTensor l = scalar_one(ctx);
  std::vector<int> in_g;
  for (int c = 0; c < bra.cols; ++c) {
    std::vector<int> out_g = active_gate_bonds(pieces, c);
    l = band_step(ctx, L, l, top, bra, ket, bottom, pieces, c, false, in_g, out_g);
    in_g = out_g;
  }
  return read_scalar(ctx, l);
}

BandEnvD band_environment(Ctx& ctx, const BoundaryD* top, const PepsStateD& bra, const PepsStateD& ket, int r0, int r1,
                          const BoundaryD* bottom) {
  check_state_pair(bra, ket);
  Layout L = make_layout(top, r0, r1, bottom);
  BandEnvD env;
  env.r0 = r0;
  env.r1 = r1;
  const int n = bra.cols;
  env.left.resize(n);
  env.right.resize(n);
  LTensor l = scalar_one(ctx);
  for (int c = 0; c < n; ++c) {
    l = band_step(ctx, L, l, top, bra, ket, bottom, {}, c, false, {}, {});
    env.left[c] = l;
  }
  LTensor r = scalar_one(ctx);
  for (int c = 0; c < n; ++c) {
    r = band_step(ctx, L, r, top, bra, ket, bottom, {}, c, true, {}, {});
    env.right[n - 1 - c] = r;
  }
  return env;
}

std::pair<double, double> band_splice(Ctx& ctx, const BandEnvD& env, const BoundaryD* top, const PepsStateD& bra,
                                      const PepsStateD& ket, const BoundaryD* bottom,
                                      const std::vector<InsertionPieceD>& pieces, int c0, int c1) {
  check_state_pair(bra, ket);
  Layout L = make_layout(top, env.r0, env.r1, bottom);
  const int n = bra.cols;
  if (c1 >= n || c0 > c1 || c0 < 0) throw Error(kValidationError, "bad splice column range");
  LTensor l = c0 == 0 ? scalar_one(ctx) : env.left[c0 - 1];
  std::vector<int> in_g;
  for (int c = c0; c <= c1; ++c) {
    std::vector<int> out_g = active_gate_bonds(pieces, c);
    l = band_step(ctx, L, l, top, bra, ket, bottom, pieces, c, false, in_g, out_g);
    in_g = out_g;
  }
  if (c1 + 1 == n) return read_scalar(ctx, l);
  const LTensor& r = env.right[c1 + 1];
  LTensor v = contract_network(ctx, {l, r}, "");
  return read_scalar(ctx, v);
}

// ---------------------------------------------------------------------------- expectation

namespace {

std::vector<double2> to_host(Ctx& ctx, const DTensor& t) {
  std::vector<double2> h(static_cast<size_t>(t.size()));
  if (!h.empty())
    PEPSB_CUDA(cudaMemcpyAsync(h.data(), t.data(), h.size() * sizeof(double2), cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
  return h;
}

DTensor upload(Ctx& ctx, const std::vector<double2>& h, const std::vector<int64_t>& shape) {
  DTensor t = ctx.empty(shape);
  if (!h.empty())
    PEPSB_CUDA(cudaMemcpyAsync(t.data(), h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice, ctx.stream));
  ctx.sync();  // h is a host temporary
  return t;
}

// Observable::is_hermitian (observables.cpp:41-58), tol 1e-12.
bool is_hermitian(Ctx& ctx, const std::vector<LocalTermD>& terms) {
  for (const auto& t : terms) {
    const std::vector<double2> m = to_host(ctx, t.op);
    const int64_t n = static_cast<int64_t>(std::llround(std::sqrt(static_cast<double>(m.size()))));
    const double2 cf = make_double2(t.coeff_re, t.coeff_im);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j) {
        const double2 a = cmul(cf, m[i * n + j]);
        const double2 b = cconj(cmul(cf, m[j * n + i]));
        if (std::hypot(a.x - b.x, a.y - b.y) > 1e-12) return false;
      }
  }
  return true;
}

// split_two_site (observables.cpp:284-295): SVD of op.permute{0,2,1,3} split 2|2,
// rank by retained_rank with cap d^2, sqrt(s) on both sides; pieces (o1,i1,g),
// (o2,i2,g).
std::pair<DTensor, DTensor> split_two_site(Ctx& ctx, const DTensor& op) {
  const int64_t d = op.shape[0];
  const std::vector<double2> h = to_host(ctx, op);
  std::vector<double2> pm(h.size());
  for (int64_t a = 0; a < d; ++a)
    for (int64_t b = 0; b < d; ++b)
      for (int64_t c = 0; c < d; ++c)
        for (int64_t e = 0; e < d; ++e) pm[((a * d + c) * d + b) * d + e] = h[((a * d + b) * d + c) * d + e];
  SvdD sv = svd(ctx, upload(ctx, pm, {d, d, d, d}), 2);
  const size_t g = retained_rank(sv.s, Trunc{static_cast<uint64_t>(d * d), 1e-14});
  const int64_t k = static_cast<int64_t>(sv.s.size()), G = static_cast<int64_t>(g);
  const std::vector<double2> u = to_host(ctx, sv.u), v = to_host(ctx, sv.v);  // u (d,d,k), v (k,d,d)
  std::vector<double2> left(static_cast<size_t>(d * d * G)), right(static_cast<size_t>(d * d * G));
  for (int64_t x = 0; x < d * d; ++x)
    for (int64_t j = 0; j < G; ++j) {
      const double w = std::sqrt(sv.s[j]);
      left[x * G + j] = cscale(u[x * k + j], w);      // (o1, i1, g)
      right[x * G + j] = cscale(v[j * d * d + x], w);  // (g, o2, i2) -> (o2, i2, g)
    }
  return {upload(ctx, left, {d, d, G}), upload(ctx, right, {d, d, G})};
}

struct TermPiecesD {
  std::vector<InsertionPieceD> pieces;
  int r0 = 0, r1 = 0, c0 = 0, c1 = 0;
};

// observables.cpp:302-321
TermPiecesD term_pieces(Ctx& ctx, const LocalTermD& t) {
  TermPiecesD out;
  if (t.sites.size() == 1) {
    out.pieces.push_back({t.sites[0].first, t.sites[0].second, t.op, {}});
    out.r0 = out.r1 = t.sites[0].first;
    out.c0 = out.c1 = t.sites[0].second;
    return out;
  }
  auto lr = split_two_site(ctx, t.op);
  out.pieces.push_back({t.sites[0].first, t.sites[0].second, lr.first, {0}});
  out.pieces.push_back({t.sites[1].first, t.sites[1].second, lr.second, {0}});
  out.r0 = std::min(t.sites[0].first, t.sites[1].first);
  out.r1 = std::max(t.sites[0].first, t.sites[1].first);
  out.c0 = std::min(t.sites[0].second, t.sites[1].second);
  out.c1 = std::max(t.sites[0].second, t.sites[1].second);
  if (out.r1 - out.r0 > 1)
    throw Error(kValidationError, "term spans more than two rows; only 1- and 2-site terms are supported");
  return out;
}

}  // namespace

// observables.cpp:335-422
ExpectResultD expectation(Ctx& ctx, const PepsStateD& s, const std::vector<LocalTermD>& terms,
                          const ExpectOptD& opt) {
  s.validate();
  for (const auto& t : terms) {
    if (t.sites.empty() || t.sites.size() > 2) throw Error(kValidationError, "terms act on one or two sites");
    for (auto [r, c] : t.sites)
      if (r < 0 || c < 0 || r >= s.rows || c >= s.cols)
        throw Error(kValidationError, "site (" + std::to_string(r) + "," + std::to_string(c) + ") outside the grid");
  }
  if (!opt.allow_complex && !is_hermitian(ctx, terms))
    throw Error(kValidationError, "observable is not Hermitian; request a complex expectation explicitly");
  ExpectResultD out;
  const uint64_t f0 = ctx.flops;
  const int n = s.rows;
  RowCacheD cache;
  if (opt.use_cache) {
    cache = build_row_cache(ctx, s, opt.contract);
    out.full_sweeps = 2;
    out.norm_sq = chain_scalar(ctx, cache.tops[n - 1]).first;
  } else {
    std::vector<BoundaryD> tops;
    tops.push_back(two_layer_first_row(ctx, s, s));
    for (int r = 1; r < n; ++r) tops.push_back(two_layer_apply_row(ctx, tops.back(), s, s, r, opt.contract, kTagTop));
    out.norm_sq = chain_scalar(ctx, tops[n - 1]).first;
  }
  std::map<std::pair<int, int>, BandEnvD> envs;  // shared environments per band
  double sr = 0.0, si = 0.0;
  for (const auto& term : terms) {
    TermPiecesD tp = term_pieces(ctx, term);
    const BoundaryD* top = nullptr;
    const BoundaryD* bottom = nullptr;
    std::vector<BoundaryD> local_top, local_bot;
    if (opt.use_cache) {
      if (tp.r0 > 0) top = &cache.tops[tp.r0 - 1];
      if (tp.r1 + 1 < n) bottom = &cache.bots[tp.r1 + 1];
    } else {
      // recompute the needed boundaries with the same structural seeds
      if (tp.r0 > 0) {
        local_top.push_back(two_layer_first_row(ctx, s, s));
        for (int r = 1; r < tp.r0; ++r)
          local_top.push_back(two_layer_apply_row(ctx, local_top.back(), s, s, r, opt.contract, kTagTop));
        top = &local_top.back();
      }
      if (tp.r1 + 1 < n) {
        PepsStateD fl = flip_vertical(ctx, s);
        local_bot.push_back(two_layer_first_row(ctx, fl, fl));
        for (int r = 1; r < n - 1 - tp.r1; ++r)
          local_bot.push_back(two_layer_apply_row(ctx, local_bot.back(), fl, fl, r, opt.contract, kTagBottom));
        bottom = &local_bot.back();
      }
      out.full_sweeps += 1;
    }
    std::pair<double, double> v;
    if (opt.shared_environments && opt.use_cache) {
      const auto key = std::make_pair(tp.r0, tp.r1);
      auto it = envs.find(key);
      if (it == envs.end()) {
        it = envs.emplace(key, band_environment(ctx, top, s, s, tp.r0, tp.r1, bottom)).first;
        out.band_contractions += 1;
      }
      v = band_splice(ctx, it->second, top, s, s, bottom, tp.pieces, tp.c0, tp.c1);
    } else {
      v = band_value(ctx, top, s, s, tp.r0, tp.r1, bottom, tp.pieces);
      out.band_contractions += opt.use_cache ? 1 : 0;
    }
    sr += term.coeff_re * v.first - term.coeff_im * v.second;
    si += term.coeff_re * v.second + term.coeff_im * v.first;
  }
  out.raw_re = sr;
  out.raw_im = si;
  out.cx_re = sr / out.norm_sq;
  out.cx_im = si / out.norm_sq;
  out.flops = ctx.flops - f0;
  if (!opt.allow_complex) {
    const double scale = std::max(1.0, std::hypot(out.cx_re, out.cx_im));
    if (std::fabs(out.cx_im) > 1e-8 * scale)
      throw Error(kNumericalError, "expectation of a Hermitian observable has imaginary part " +
                                       std::to_string(out.cx_im));
  }
  out.value = out.cx_re;
  return out;
}

// ---------------------------------------------------------------------------- one-layer boundary MPS

namespace {

DTensor contract_to(Ctx& ctx, const std::vector<LTensor>& leaves, const std::string& out) {
  LTensor t = contract_network(ctx, leaves, out);
  return materialize(ctx, t, t.labels);
}

void check_mpo_pair(const MpsD& s, const MpoD& o) {
  if (s.sites.empty()) throw Error(kShapeError, "empty MPS");
  if (o.sites.size() != s.sites.size()) throw Error(kShapeError, "MPS/MPO length mismatch");
  for (size_t i = 0; i < s.sites.size(); ++i) {
    if (s.sites[i].shape.size() != 3 || o.sites[i].shape.size() != 4)
      throw Error(kShapeError, "MPS sites are (phys, left, right), MPO sites (p, d, left, right)");
    if (s.sites[i].shape[0] != o.sites[i].shape[0])
      throw Error(kShapeError, "physical extent mismatch at site " + std::to_string(i));
  }
}

}  // namespace

void GridD::validate() const {
  if (rows <= 0 || cols <= 0) throw Error(kValidationError, "grid must be non-empty");
  if (static_cast<int>(sites.size()) != rows * cols) throw Error(kShapeError, "one-layer site count mismatch");
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) {
      const auto& t = site(r, c).shape;
      if (t.size() != 4)
        throw Error(kShapeError, "one-layer sites must be order 4 (up, left, down, right); physical indices must be "
                                 "projected or merged first");
      if (r == 0 && t[0] != 1) throw Error(kShapeError, "top boundary bond must be 1");
      if (c == 0 && t[1] != 1) throw Error(kShapeError, "left boundary bond must be 1");
      if (r == rows - 1 && t[2] != 1) throw Error(kShapeError, "bottom boundary bond must be 1");
      if (c == cols - 1 && t[3] != 1) throw Error(kShapeError, "right boundary bond must be 1");
      if (r + 1 < rows && t[2] != site(r + 1, c).shape[0])
        throw Error(kShapeError, "vertical bond mismatch in one-layer grid");
      if (c + 1 < cols && t[3] != site(r, c + 1).shape[1])
        throw Error(kShapeError, "horizontal bond mismatch in one-layer grid");
    }
}

MpsD approx_apply_mpo(Ctx& ctx, const MpsD& s, const MpoD& o, const ApplyOptD& opt) {
  check_mpo_pair(s, o);
  const size_t n = s.sites.size();
  MpsD out;
  out.sites.resize(n);
  // v1 = sum_p s1(p, l, r) o1(p, d, L, R), (l, L) merged into a
  const DTensor& s0 = s.sites[0];
  const DTensor& o0 = o.sites[0];
  DTensor v = contract_to(ctx, {as_labelled(s0, "plr"), as_labelled(o0, "pdLR")}, "lLdrR");
  v = reshape(v, {s0.shape[1] * o0.shape[2], o0.shape[1], s0.shape[2], o0.shape[3]});
  if (n == 1) {
    DTensor t = contract_to(ctx, {as_labelled(v, "adso")}, "daso");
    out.sites[0] = reshape(t, {v.shape[1], v.shape[0], v.shape[2] * v.shape[3]});
    return out;
  }
  for (size_t i = 1; i < n; ++i) {
    ImplicitOp net({v, s.sites[i], o.sites[i]}, {"adso", "pst", "peoq"}, "ad", "etq");
    Rsvd cfg = opt.rsvd;
    cfg.seed = derive_seed1(opt.seed_base, static_cast<uint64_t>(i));
    // t1 (a, d, rho) written directly as (d, a, rho)
    EinsumsvdResultD split = einsumsvd(ctx, net, opt.policy, opt.strategy, opt.absorb, cfg, {1, 0, 2});
    out.sites[i - 1] = split.t1;
    v = split.t2;  // (rho, e, t, q)
  }
  DTensor t = contract_to(ctx, {as_labelled(v, "adso")}, "daso");
  out.sites[n - 1] = reshape(t, {v.shape[1], v.shape[0], v.shape[2] * v.shape[3]});
  return out;
}

MpsD exact_apply_mpo(Ctx& ctx, const MpsD& s, const MpoD& o) {
  check_mpo_pair(s, o);
  MpsD out;
  for (size_t i = 0; i < s.sites.size(); ++i) {
    const DTensor& a = s.sites[i];
    const DTensor& b = o.sites[i];
    DTensor t = contract_to(ctx, {as_labelled(a, "plr"), as_labelled(b, "pdLR")}, "dlLrR");
    out.sites.push_back(reshape(t, {b.shape[1], a.shape[1] * b.shape[2], a.shape[2] * b.shape[3]}));
  }
  return out;
}

std::pair<double, double> mps_glue(Ctx& ctx, const MpsD& top, const MpsD& bottom) {
  if (top.sites.size() != bottom.sites.size()) throw Error(kShapeError, "MPS length mismatch in glue");
  LTensor l = scalar_one(ctx);
  l.labels = "ab";
  l.ext = {1, 1};
  l.str = {1, 1};
  for (size_t i = 0; i < top.sites.size(); ++i) {
    LTensor t = contract_network(ctx, {l, as_labelled(top.sites[i], "pac"), as_labelled(bottom.sites[i], "pbd")},
                                 "cd");
    l = t;
    l.labels = "ab";
  }
  return read_scalar(ctx, l);
}

std::pair<double, double> contract_one_layer(Ctx& ctx, const GridD& g, int family, const ContractOptD& opt,
                                             uint64_t memory_budget) {
  g.validate();
  // (u, l, d, r) -> (u*d [phys], l, r)  (contraction.cpp:136-146)
  auto as_mps = [&](int r) {
    MpsD m;
    for (int c = 0; c < g.cols; ++c) {
      const DTensor& t = g.site(r, c);
      DTensor p = contract_to(ctx, {as_labelled(t, "uldr")}, "udlr");
      m.sites.push_back(reshape(p, {t.shape[0] * t.shape[2], t.shape[1], t.shape[3]}));
    }
    return m;
  };
  // (u, l, d, r) -> (u, d, l, r); from below (d, u, l, r)  (contraction.cpp:148-158)
  auto as_mpo = [&](int r, bool from_below) {
    MpoD m;
    for (int c = 0; c < g.cols; ++c)
      m.sites.push_back(contract_to(ctx, {as_labelled(g.site(r, c), "uldr")}, from_below ? "dulr" : "udlr"));
    return m;
  };
  auto budget = [&](uint64_t el, const char* what) {
    if (el > memory_budget)
      throw Error(kResourceError, std::string(what) + " needs " + std::to_string(el) + " elements, budget is " +
                                      std::to_string(memory_budget));
  };
  auto apply_budget = [&](const MpsD& s, const MpoD& o) {
    for (size_t c = 0; c < s.sites.size(); ++c)
      budget(static_cast<uint64_t>(o.sites[c].shape[1] * s.sites[c].shape[1] * o.sites[c].shape[2] *
                                   s.sites[c].shape[2] * o.sites[c].shape[3]),
             "contract_exact");
  };
  const int n = g.rows;
  if (family == kFamilyExact) {  // contraction.cpp:178-201
    if (n == 1) return chain_scalar(ctx, BoundaryD{as_mps(0).sites, {}});
    const int half = n / 2;
    MpsD top = as_mps(0);
    for (int r = 1; r < half; ++r) {
      MpoD o = as_mpo(r, false);
      apply_budget(top, o);
      top = exact_apply_mpo(ctx, top, o);
    }
    MpsD bottom = as_mps(n - 1);
    for (int r = n - 1; r-- > half;) {
      MpoD o = as_mpo(r, true);
      apply_budget(bottom, o);
      bottom = exact_apply_mpo(ctx, bottom, o);
    }
    for (int c = 0; c < g.cols; ++c)
      budget(static_cast<uint64_t>(top.sites[c].shape[0] * top.sites[c].shape[2] * bottom.sites[c].shape[2]),
             "contract_exact");
    return mps_glue(ctx, top, bottom);
  }
  if (family != kFamilyBmps && family != kFamilyIbmps) throw Error(kValidationError, "unknown one-layer family");
  MpsD s = as_mps(0);  // contraction.cpp:205-221
  for (int r = 1; r < n; ++r) {
    ApplyOptD ao;
    ao.policy = opt.trunc;
    if (ao.policy.max_rank == 0) ao.policy.max_rank = UINT64_MAX;
    ao.strategy = opt.strategy;
    ao.rsvd = opt.rsvd;
    ao.absorb = opt.canonicalize ? (r % 2 ? kRight : kLeft) : kSplit;
    ao.seed_base = derive_seed1(derive_seed1(opt.seed, 0x10), static_cast<uint64_t>(r));
    s = approx_apply_mpo(ctx, s, as_mpo(r, false), ao);
  }
  return chain_scalar(ctx, BoundaryD{s.sites, {}});
}

}  // namespace pepsb
