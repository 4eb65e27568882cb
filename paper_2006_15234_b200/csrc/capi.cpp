#include <algorithm>
#include <cstdio>
#include <memory>
// extern "C" boundary (include/peps_b200.h): POD in, handles out, status codes.
#include <cstring>
#include <exception>
#include <string>

#include "../../include/peps_b200.h"
#include "ite.h"
#include "peps.h"
#include "sharded.h"
#include "smalldense.cuh"
#include "tensor_ops.cuh"
#include "zgemm.cuh"
#include "gram.cuh"

using namespace pepsb;

struct pepsb_ctx {
  Ctx* ctx;
};
struct pepsb_tensor {
  DTensor t;
};
struct pepsb_state {
  PepsStateD s;
};
struct pepsb_boundary {
  BoundaryD b;
};
struct pepsb_row_cache {
  RowCacheD c;
};
struct pepsb_band_env {
  BandEnvD e;
};

namespace {

thread_local std::string g_err;
thread_local int g_kind = 0;

template <class F>
int guard(F&& f) {
  try {
    f();
    return PEPSB_OK;
  } catch (const Error& e) {
    g_err = e.what();
    g_kind = e.kind;
  } catch (const std::bad_alloc& e) {
    g_err = "host allocation failed";
    g_kind = PEPSB_E_RESOURCE;
  } catch (const std::exception& e) {
    g_err = e.what();
    g_kind = PEPSB_E_OTHER;
  }
  return g_kind;
}

void need(const void* p, const char* what) {
  if (!p) throw Error(kValidationError, std::string("null ") + what);
}

std::vector<int64_t> shape_of(int ndim, const int64_t* shape) {
  if (ndim < 0 || ndim > kMaxModes) throw Error(kShapeError, "tensor order out of range");
  std::vector<int64_t> s(shape, shape + ndim);
  for (auto e : s)
    if (e < 1) throw Error(kShapeError, "tensor extent must be >= 1");
  return s;
}

std::vector<std::string> split_csv(const char* s) {
  std::vector<std::string> out;
  std::string cur;
  for (const char* p = s; *p; ++p) {
    if (*p == ',') {
      out.push_back(cur);
      cur.clear();
    } else {
      cur += *p;
    }
  }
  out.push_back(cur);
  return out;
}

pepsb_tensor* wrap(const DTensor& t) { return new pepsb_tensor{t}; }

Trunc trunc_of(const pepsb_trunc* p) {
  Trunc t;
  if (p) {
    t.max_rank = p->max_rank;
    t.rel_cutoff = p->rel_cutoff;
  }
  return t;
}

Rsvd rsvd_of(const pepsb_rsvd* p) {
  Rsvd r;
  if (p) {
    r.power_iters = p->power_iters;
    r.oversample = p->oversample;
    r.seed = p->seed;
  }
  return r;
}

ContractOptD opt_of(const pepsb_contract_opt* p) {
  ContractOptD o;
  if (p) {
    o.trunc = trunc_of(&p->trunc);
    o.strategy = p->strategy;
    o.rsvd = rsvd_of(&p->rsvd);
    o.canonicalize = p->canonicalize != 0;
    o.seed = p->seed;
  }
  return o;
}

ImplicitOp make_op(int n, pepsb_tensor* const* ts, const char* labels_csv, const char* rows, const char* cols) {
  need(ts, "tensor list");
  need(labels_csv, "labels");
  std::vector<DTensor> v;
  for (int i = 0; i < n; ++i) {
    need(ts[i], "tensor");
    v.push_back(ts[i]->t);
  }
  return ImplicitOp(v, split_csv(labels_csv), rows ? rows : "", cols ? cols : "");
}

std::vector<InsertionPieceD> pieces_of(int npieces, const int* rc, pepsb_tensor* const* ops, const int* nbonds,
                                       const int* bond_ids) {
  std::vector<InsertionPieceD> out;
  int bi = 0;
  for (int i = 0; i < npieces; ++i) {
    InsertionPieceD p;
    p.row = rc[2 * i];
    p.col = rc[2 * i + 1];
    need(ops[i], "piece operator");
    p.op = ops[i]->t;
    for (int j = 0; j < nbonds[i]; ++j) p.bond_ids.push_back(bond_ids[bi++]);
    out.push_back(p);
  }
  return out;
}

}  // namespace

extern "C" {

const char* pepsb_last_error(void) { return g_err.c_str(); }
int pepsb_last_error_kind(void) { return g_kind; }

int pepsb_ctx_create(int device, pepsb_ctx** out) {
  return guard([&] {
    need(out, "out");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
      cudaGetLastError();
      throw Error(kCudaError, "no CUDA device available (the B200 library has no CPU fallback)");
    }
    cudaDeviceProp prop;
    PEPSB_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) throw Error(kCudaError, std::string("device is not sm_100 (found ") + prop.name + ")");
    *out = new pepsb_ctx{new Ctx(device)};
  });
}

int pepsb_ctx_destroy(pepsb_ctx* c) {
  return guard([&] {
    if (c) {
      delete c->ctx;
      delete c;
    }
  });
}

int pepsb_ctx_sync(pepsb_ctx* c) {
  return guard([&] {
    need(c, "ctx");
    c->ctx->sync();
  });
}

int pepsb_ctx_set_option(pepsb_ctx* c, const char* key, int64_t value) {
  return guard([&] {
    need(c, "ctx");
    std::string k = key ? key : "";
    if (k == "orth_mode") c->ctx->orth_mode = static_cast<int>(value);
    else if (k == "eig_solver") set_eig_solver(static_cast<int>(value));
    else if (k == "gemm_algo") zgemm_set_algo(static_cast<int>(value));
    else if (k == "gemm_ws") zgemm_set_ws(static_cast<int>(value));
    else if (k == "gemm_real") zgemm_set_real(static_cast<int>(value));
    else if (k == "gemm_small") zgemm_set_small(static_cast<int>(value));
    else if (k == "gemm_stream") zgemm_set_stream(static_cast<int>(value));
    else if (k == "cr_cfg") zgemm_set_cr_cfg(static_cast<int>(value));
    else if (k == "c3m_cfg") zgemm_set_c3m_cfg(static_cast<int>(value));
    else if (k == "gemm_gram") gram_set_enabled(static_cast<int>(value));
    else if (k == "overlap") c->ctx->overlap = static_cast<int>(std::clamp<int64_t>(value, 0, 2));
    else if (k == "concurrent_sweeps") c->ctx->concurrent_sweeps = static_cast<int>(std::clamp<int64_t>(value, -1, 1));
    else if (k == "pipeline_rows") c->ctx->pipeline_rows = static_cast<int>(std::clamp<int64_t>(value, -1, 8));
    else throw Error(kConfigError, "unknown option '" + k + "'");
  });
}

int pepsb_ctx_counters(pepsb_ctx* c, uint64_t* out) {
  return guard([&] {
    need(c, "ctx");
    out[0] = c->ctx->flops;
    out[1] = c->ctx->einsumsvd_flops;
    out[2] = c->ctx->peak_elements;
    out[3] = static_cast<uint64_t>(c->ctx->launches);
    out[4] = static_cast<uint64_t>(c->ctx->faithful_redos);
    out[5] = static_cast<uint64_t>(c->ctx->tsqr_fallbacks);
  });
}

int pepsb_ctx_get_counter(pepsb_ctx* c, const char* name, uint64_t* value) {
  return guard([&] {
    need(c, "ctx");
    need(value, "value");
    const std::string k = name ? name : "";
    Ctx& x = *c->ctx;
    if (k == "flops") *value = x.flops;
    else if (k == "einsumsvd_flops") *value = x.einsumsvd_flops;
    else if (k == "peak_elements") *value = x.peak_elements;
    else if (k == "launches") *value = static_cast<uint64_t>(x.launches);
    else if (k == "faithful_redos") *value = static_cast<uint64_t>(x.faithful_redos);
    else if (k == "tsqr_fallbacks") *value = static_cast<uint64_t>(x.tsqr_fallbacks);
    else if (k == "lookahead_misses") *value = static_cast<uint64_t>(x.lookahead_misses);
    else if (k == "degenerate_truncations") {
      unsigned long long v = 0;
      PEPSB_CUDA(cudaMemcpyAsync(&v, x.d_degenerate, sizeof(v), cudaMemcpyDeviceToHost, x.stream));
      x.sync();
      *value = v;
    } else throw Error(kConfigError, "unknown counter '" + k + "'");
  });
}

int pepsb_ctx_reset_counters(pepsb_ctx* c) {
  return guard([&] {
    need(c, "ctx");
    c->ctx->flops = c->ctx->einsumsvd_flops = c->ctx->peak_elements = 0;
    c->ctx->launches = 0;
    c->ctx->faithful_redos = c->ctx->tsqr_fallbacks = 0;
    PEPSB_CUDA(cudaMemsetAsync(c->ctx->d_degenerate, 0, sizeof(unsigned long long), c->ctx->stream));
  });
}

int pepsb_ctx_profile(pepsb_ctx* c, int enable) {
  return guard([&] {
    need(c, "ctx");
    c->ctx->profile_clear();
    c->ctx->profiling = enable != 0;
  });
}

int pepsb_ctx_profile_report_ex(pepsb_ctx* c, double* out20) {
  return guard([&] {
    need(c, "ctx");
    c->ctx->profile_report_ex(out20);
  });
}

int pepsb_ctx_profile_report(pepsb_ctx* c, double* out16) {
  return guard([&] {
    need(c, "ctx");
    c->ctx->profile_report(out16);
  });
}

int pepsb_ctx_profile_records(pepsb_ctx* c, double* out, int cap) {
  int n = 0;
  guard([&] {
    need(c, "ctx");
    c->ctx->sync();
    for (auto& r : c->ctx->prof) {
      if (n >= cap) break;
      float ms = 0.f;
      PEPSB_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
      out[3 * n] = r.kind;
      out[3 * n + 1] = ms;
      out[3 * n + 2] = r.flops;
      ++n;
    }
  });
  return n;
}

int pepsb_ctx_profile_timeline(pepsb_ctx* c, double* out, int cap) {
  int n = 0;
  guard([&] {
    need(c, "ctx");
    c->ctx->sync();
    const auto& prof = c->ctx->prof;
    if (prof.empty()) return;
    for (auto& r : prof) {
      if (n >= cap) break;
      float t0 = 0.f, t1 = 0.f;
      PEPSB_CUDA(cudaEventElapsedTime(&t0, prof.front().a, r.a));
      PEPSB_CUDA(cudaEventElapsedTime(&t1, prof.front().a, r.b));
      out[5 * n] = r.kind;
      out[5 * n + 1] = t0;
      out[5 * n + 2] = t1;
      out[5 * n + 3] = r.exec_flops;
      out[5 * n + 4] = r.side;
      ++n;
    }
  });
  return n;
}

int pepsb_ctx_debug_word(pepsb_ctx* c, int idx, int reset) {
  int v = -1;
  guard([&] {
    need(c, "ctx");
    if (idx < 0 || idx >= 64) throw Error(kValidationError, "debug word index out of range");
    c->ctx->sync();
    PEPSB_CUDA(cudaMemcpy(&v, c->ctx->d_status + idx, sizeof(int), cudaMemcpyDeviceToHost));
    if (reset) PEPSB_CUDA(cudaMemset(c->ctx->d_status + idx, 0, sizeof(int)));
  });
  return v;
}

void* pepsb_ctx_stream(pepsb_ctx* c) { return c ? static_cast<void*>(c->ctx->stream) : nullptr; }

// Exact-zero imaginary parts (checked on the device, one small reduction and a
// flag read-back): such tensors run the complex x real GEMM kernels.
void mark_real(Ctx& ctx, DTensor& t) {
  int* flag = ctx.d_status + 40;
  imag_nonzero(t.data(), t.size(), flag, ctx.stream);
  ++ctx.launches;
  PEPSB_CUDA(cudaMemcpyAsync(ctx.h_status + 40, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync_main();
  t.buf->real = ctx.h_status[40] == 0;
}

int pepsb_tensor_from_host(pepsb_ctx* c, int ndim, const int64_t* shape, const double* data, pepsb_tensor** out) {
  return guard([&] {
    need(c, "ctx");
    DTensor t = c->ctx->empty(shape_of(ndim, shape));
    if (t.size()) {
      PEPSB_CUDA(cudaMemcpyAsync(t.data(), data, t.size() * sizeof(double2), cudaMemcpyHostToDevice, c->ctx->stream));
      mark_real(*c->ctx, t);
    }
    *out = wrap(t);
  });
}

int pepsb_tensor_from_device(pepsb_ctx* c, int ndim, const int64_t* shape, const void* dptr, pepsb_tensor** out) {
  return guard([&] {
    need(c, "ctx");
    DTensor t = c->ctx->empty(shape_of(ndim, shape));
    if (t.size()) {
      PEPSB_CUDA(cudaMemcpyAsync(t.data(), dptr, t.size() * sizeof(double2), cudaMemcpyDeviceToDevice, c->ctx->stream));
      mark_real(*c->ctx, t);
    }
    *out = wrap(t);
  });
}

int pepsb_tensor_ndim(const pepsb_tensor* t) { return t ? static_cast<int>(t->t.shape.size()) : -1; }

int pepsb_tensor_shape(const pepsb_tensor* t, int64_t* shape) {
  return guard([&] {
    need(t, "tensor");
    for (size_t a = 0; a < t->t.shape.size(); ++a) shape[a] = t->t.shape[a];
  });
}

int pepsb_tensor_to_host(pepsb_ctx* c, const pepsb_tensor* t, double* out) {
  return guard([&] {
    need(c, "ctx");
    need(t, "tensor");
    if (t->t.size())
      PEPSB_CUDA(cudaMemcpyAsync(out, t->t.data(), t->t.size() * sizeof(double2), cudaMemcpyDeviceToHost, c->ctx->stream));
    c->ctx->sync();
  });
}

int pepsb_tensor_to_host_async(pepsb_ctx* c, const pepsb_tensor* t, double* out) {
  return guard([&] {
    need(c, "ctx");
    need(t, "tensor");
    if (t->t.size())
      PEPSB_CUDA(cudaMemcpyAsync(out, t->t.data(), t->t.size() * sizeof(double2), cudaMemcpyDeviceToHost, c->ctx->stream));
  });
}

int pepsb_tensor_to_device(pepsb_ctx* c, const pepsb_tensor* t, void* dptr) {
  return guard([&] {
    need(c, "ctx");
    need(t, "tensor");
    if (t->t.size())
      PEPSB_CUDA(cudaMemcpyAsync(dptr, t->t.data(), t->t.size() * sizeof(double2), cudaMemcpyDeviceToDevice, c->ctx->stream));
  });
}

void pepsb_tensor_free(pepsb_tensor* t) { delete t; }

int pepsb_random_tensor(pepsb_ctx* c, int ndim, const int64_t* shape, uint64_t seed, int real, pepsb_tensor** out) {
  return guard([&] {
    need(c, "ctx");
    DTensor t = c->ctx->empty(shape_of(ndim, shape));
    std::vector<int64_t> lstr = row_major_strides(t.shape);
    random_fill(t.data(), ndim, t.shape.data(), lstr.data(), seed, real, c->ctx->stream);
    ++c->ctx->launches;
    *out = wrap(t);
  });
}

int pepsb_contract(pepsb_ctx* c, const char* spec, int n, pepsb_tensor* const* ts, pepsb_tensor** out) {
  return guard([&] {
    need(c, "ctx");
    need(spec, "spec");
    std::vector<std::string> ins;
    std::string output;
    parse_spec(spec, ins, output);
    if (static_cast<int>(ins.size()) != n)
      throw Error(kShapeError, "spec lists " + std::to_string(ins.size()) + " inputs, got " + std::to_string(n) +
                                   " tensors");
    std::vector<LTensor> leaves;
    for (int i = 0; i < n; ++i) {
      need(ts[i], "tensor");
      leaves.push_back(as_labelled(ts[i]->t, ins[i]));
    }
    LTensor r = contract_network(*c->ctx, leaves, output);
    *out = wrap(materialize(*c->ctx, r, r.labels));
  });
}

int pepsb_implicit(pepsb_ctx* c, int n, pepsb_tensor* const* ts, const char* labels_csv, const char* rows,
                   const char* cols, const pepsb_tensor* probe, int mode, pepsb_tensor** out) {
  return guard([&] {
    need(c, "ctx");
    ImplicitOp op = make_op(n, ts, labels_csv, rows, cols);
    if (mode == 2) {
      *out = wrap(implicit_materialize(*c->ctx, op));
    } else {
      need(probe, "probe");
      *out = wrap(implicit_apply(*c->ctx, op, probe->t, mode == 1));
    }
  });
}

int pepsb_gram_orthogonalize(pepsb_ctx* c, const pepsb_tensor* a, int split, pepsb_tensor** q, pepsb_tensor** r) {
  return guard([&] {
    need(c, "ctx");
    need(a, "tensor");
    auto [Q, R] = gram_orthogonalize(*c->ctx, a->t, split);
    *q = wrap(Q);
    *r = wrap(R);
  });
}

int pepsb_random_slice(pepsb_ctx* c, int ndim, const int64_t* shape, int axis, int64_t start, int64_t count,
                       uint64_t seed, int real, pepsb_tensor** out) {
  return guard([&] {
    need(c, "ctx");
    std::vector<int64_t> full = shape_of(ndim, shape);
    if (axis < 0 || axis >= ndim) throw Error(kShapeError, "random_slice: axis out of range");
    if (start < 0 || count < 0 || start + count > full[axis]) throw Error(kShapeError, "random_slice: bad range");
    std::vector<int64_t> lstr = row_major_strides(full);
    std::vector<int64_t> ext = full;
    ext[axis] = count;
    DTensor t = c->ctx->empty(ext);
    if (t.size() > 0) {
      random_fill(t.data(), ndim, ext.data(), lstr.data(), seed, real, c->ctx->stream,
                  static_cast<uint64_t>(start) * static_cast<uint64_t>(lstr[axis]));
      ++c->ctx->launches;
    }
    *out = wrap(t);
  });
}

int pepsb_tensor_conj(pepsb_ctx* c, const pepsb_tensor* a, pepsb_tensor** out) {
  return guard([&] {
    need(c, "ctx");
    need(a, "tensor");
    std::string lab;
    for (size_t i = 0; i < a->t.shape.size(); ++i) lab += static_cast<char>('a' + i);
    LTensor l = reduce_to(*c->ctx, as_labelled(a->t, lab, true), lab);
    *out = wrap(materialize(*c->ctx, l, lab));
  });
}

int pepsb_tensor_slice(pepsb_ctx* c, const pepsb_tensor* a, int axis, int64_t start, int64_t count,
                       pepsb_tensor** out) {
  return guard([&] {
    need(c, "ctx");
    need(a, "tensor");
    const int nd = static_cast<int>(a->t.shape.size());
    if (axis < 0 || axis >= nd) throw Error(kShapeError, "slice: axis out of range");
    if (start < 0 || count < 0 || start + count > a->t.shape[axis]) throw Error(kShapeError, "slice: bad range");
    std::string lab;
    for (int i = 0; i < nd; ++i) lab += static_cast<char>('a' + i);
    LTensor l = as_labelled(a->t, lab);
    l.ptr += start * l.str[axis];
    l.ext[axis] = count;
    if (l.size() == 0) {
      *out = wrap(c->ctx->empty(l.ext));
      return;
    }
    *out = wrap(materialize(*c->ctx, reduce_to(*c->ctx, l, lab), lab));
  });
}

int pepsb_tensor_reshape(const pepsb_tensor* a, int ndim, const int64_t* shape, pepsb_tensor** out) {
  return guard([&] {
    need(a, "tensor");
    DTensor t = a->t;
    t.shape = shape_of(ndim, shape);
    if (t.size() != a->t.size()) throw Error(kShapeError, "reshape changes the element count");
    *out = wrap(t);
  });
}

int pepsb_tensor_data_ptr(const pepsb_tensor* a, void** ptr) {
  return guard([&] {
    need(a, "tensor");
    *ptr = a->t.data();
  });
}

int pepsb_gram(pepsb_ctx* c, const pepsb_tensor* z, pepsb_tensor** g) {
  return guard([&] {
    need(c, "ctx");
    need(z, "tensor");
    *g = wrap(gram_matrix(*c->ctx, z->t));
  });
}

int pepsb_gram_factors(pepsb_ctx* c, const pepsb_tensor* g, pepsb_tensor** p, pepsb_tensor** r, pepsb_tensor** vecs,
                       double* lam, int* deficient, int64_t cap) {
  return guard([&] {
    need(c, "ctx");
    need(g, "tensor");
    GramFactorsD f = gram_factors_full(*c->ctx, g->t);
    if (static_cast<int64_t>(f.lam.size()) > cap) throw Error(kValidationError, "buffer too small");
    std::memcpy(lam, f.lam.data(), f.lam.size() * sizeof(double));
    std::memcpy(deficient, f.deficient.data(), f.deficient.size() * sizeof(int));
    *p = wrap(f.P);
    *r = wrap(f.R);
    *vecs = wrap(f.vecs);
  });
}

int pepsb_projected_svd(pepsb_ctx* c, const pepsb_tensor* z, int64_t target, pepsb_tensor** ut, double* s,
                        int64_t cap) {
  return guard([&] {
    need(c, "ctx");
    need(z, "tensor");
    auto [u, sv] = projected_svd_full(*c->ctx, z->t, target);
    if (static_cast<int64_t>(sv.size()) > cap) throw Error(kValidationError, "buffer too small");
    std::memcpy(s, sv.data(), sv.size() * sizeof(double));
    *ut = wrap(u);
  });
}

int pepsb_eigh(pepsb_ctx* c, const pepsb_tensor* a, double* values, int64_t cap, pepsb_tensor** vectors) {
  return guard([&] {
    need(c, "ctx");
    need(a, "tensor");
    need(values, "values");
    need(vectors, "vectors");
    EighD r = eigh(*c->ctx, a->t);
    if (static_cast<int64_t>(r.values.size()) > cap) throw Error(kValidationError, "eigenvalue buffer too small");
    std::memcpy(values, r.values.data(), r.values.size() * sizeof(double));
    *vectors = wrap(r.vectors);
  });
}

int pepsb_svd(pepsb_ctx* c, const pepsb_tensor* a, int split, pepsb_tensor** u, double* s, int64_t s_cap, int64_t* k,
              pepsb_tensor** v) {
  return guard([&] {
    need(c, "ctx");
    need(a, "tensor");
    SvdD r = svd(*c->ctx, a->t, split);
    if (static_cast<int64_t>(r.s.size()) > s_cap) throw Error(kValidationError, "singular value buffer too small");
    std::memcpy(s, r.s.data(), r.s.size() * sizeof(double));
    *k = static_cast<int64_t>(r.s.size());
    *u = wrap(r.u);
    *v = wrap(r.v);
  });
}

int pepsb_randomized_svd(pepsb_ctx* c, int n, pepsb_tensor* const* ts, const char* labels_csv, const char* rows,
                         const char* cols, const pepsb_trunc* policy, const pepsb_rsvd* cfg, pepsb_tensor** u, double* s,
                         int64_t s_cap, int64_t* rank, pepsb_tensor** v, int* clamped) {
  return guard([&] {
    need(c, "ctx");
    ImplicitOp op = make_op(n, ts, labels_csv, rows, cols);
    SvdTripleD r = randomized_svd(*c->ctx, op, trunc_of(policy), rsvd_of(cfg));
    if (static_cast<int64_t>(r.s.size()) > s_cap) throw Error(kValidationError, "singular value buffer too small");
    std::memcpy(s, r.s.data(), r.s.size() * sizeof(double));
    *rank = static_cast<int64_t>(r.s.size());
    *u = wrap(r.u);
    *v = wrap(r.v);
    *clamped = r.rank_clamped;
  });
}

int pepsb_einsumsvd(pepsb_ctx* c, int n, pepsb_tensor* const* ts, const char* labels_csv, const char* rows,
                    const char* cols, const pepsb_trunc* policy, int strategy, int absorb, const pepsb_rsvd* cfg,
                    pepsb_tensor** t1, pepsb_tensor** t2, double* s, int64_t s_cap, int64_t* rank, int* clamped) {
  return guard([&] {
    need(c, "ctx");
    ImplicitOp op = make_op(n, ts, labels_csv, rows, cols);
    EinsumsvdResultD r = einsumsvd(*c->ctx, op, trunc_of(policy), strategy, absorb, rsvd_of(cfg));
    if (static_cast<int64_t>(r.s.size()) > s_cap) throw Error(kValidationError, "singular value buffer too small");
    std::memcpy(s, r.s.data(), r.s.size() * sizeof(double));
    *rank = static_cast<int64_t>(r.s.size());
    *t1 = wrap(r.t1);
    *t2 = wrap(r.t2);
    *clamped = r.rank_clamped;
  });
}

int pepsb_state_create(pepsb_ctx* c, int rows, int cols, int d, pepsb_tensor* const* sites, pepsb_state** out) {
  return guard([&] {
    need(c, "ctx");
    PepsStateD s;
    s.rows = rows;
    s.cols = cols;
    s.d = d;
    for (int i = 0; i < rows * cols; ++i) {
      need(sites[i], "site");
      s.sites.push_back(sites[i]->t);
    }
    s.validate();
    *out = new pepsb_state{s};
  });
}

// ---- PEPS container (save_peps / load_peps, state.cpp:240-299): magic
// "PEPS2D01", u64 rows / cols / d, u64 tag length + axis tag "pudlr", per site
// u64 order, u64 extents, raw complex128 data (host byte order).
namespace {
constexpr char kPepsMagic[8] = {'P', 'E', 'P', 'S', '2', 'D', '0', '1'};
constexpr char kPepsTag[] = "pudlr";
}  // namespace

int pepsb_save_peps(pepsb_ctx* c, const pepsb_state* s, const char* path) {
  return guard([&] {
    need(c, "ctx");
    need(s, "state");
    need(path, "path");
    FILE* f = fopen(path, "wb");
    if (!f) throw Error(kValidationError, std::string("cannot open '") + path + "' for writing");
    std::unique_ptr<FILE, int (*)(FILE*)> guard_f(f, fclose);  // closes on a mid-write throw
    bool ok = true;
    auto u64 = [&](uint64_t v) { ok = ok && fwrite(&v, sizeof(v), 1, f) == 1; };
    ok = fwrite(kPepsMagic, 1, 8, f) == 8;
    u64(static_cast<uint64_t>(s->s.rows));
    u64(static_cast<uint64_t>(s->s.cols));
    u64(static_cast<uint64_t>(s->s.d));
    u64(sizeof(kPepsTag) - 1);
    ok = ok && fwrite(kPepsTag, 1, sizeof(kPepsTag) - 1, f) == sizeof(kPepsTag) - 1;
    for (const DTensor& t : s->s.sites) {
      u64(t.shape.size());
      for (auto e : t.shape) u64(static_cast<uint64_t>(e));
      std::vector<double2> h(static_cast<size_t>(t.size()));
      if (!h.empty()) {
        PEPSB_CUDA(cudaMemcpyAsync(h.data(), t.data(), h.size() * sizeof(double2), cudaMemcpyDeviceToHost,
                                   c->ctx->stream));
        c->ctx->sync();
        ok = ok && fwrite(h.data(), sizeof(double2), h.size(), f) == h.size();
      }
    }
    ok = (fclose(guard_f.release()) == 0) && ok;
    if (!ok) throw Error(kValidationError, std::string("write failed for '") + path + "'");
  });
}

int pepsb_load_peps(pepsb_ctx* c, const char* path, pepsb_state** out) {
  return guard([&] {
    need(c, "ctx");
    need(path, "path");
    FILE* f = fopen(path, "rb");
    if (!f) throw Error(kValidationError, std::string("cannot open '") + path + "' for reading");
    std::unique_ptr<FILE, int (*)(FILE*)> guard_f(f, fclose);
    char magic[8];
    if (fread(magic, 1, 8, f) != 8 || std::memcmp(magic, kPepsMagic, 8) != 0)
      throw Error(kValidationError, std::string("'") + path + "' is not a PEPS container");
    bool ok = true;
    auto u64 = [&]() {
      uint64_t v = 0;
      ok = ok && fread(&v, sizeof(v), 1, f) == 1;
      return v;
    };
    const uint64_t rows = u64(), cols = u64(), d = u64(), tl = u64();
    if (!ok || tl > 64) throw Error(kValidationError, std::string("truncated PEPS container '") + path + "'");
    // Every count below is untrusted: bound it by the file size before allocating.
    const long here = ftell(f);
    if (here < 0 || fseek(f, 0, SEEK_END) != 0) throw Error(kValidationError, "cannot size PEPS container");
    const uint64_t file_bytes = static_cast<uint64_t>(ftell(f));
    if (fseek(f, here, SEEK_SET) != 0) throw Error(kValidationError, "cannot size PEPS container");
    constexpr uint64_t kMaxExtent = uint64_t{1} << 31;
    if (rows < 1 || cols < 1 || rows >= kMaxExtent || cols >= kMaxExtent || d < 1 || d >= kMaxExtent ||
        rows * cols > file_bytes / 16)
      throw Error(kValidationError, std::string("corrupt PEPS container header in '") + path + "'");
    std::string tag(tl, '\0');
    if (tl && fread(tag.data(), 1, tl, f) != tl) ok = false;
    if (tag != kPepsTag) throw Error(kValidationError, "unknown axis convention tag '" + tag + "'");
    PepsStateD st;
    st.rows = static_cast<int>(rows);
    st.cols = static_cast<int>(cols);
    st.d = static_cast<int>(d);
    for (uint64_t i = 0; ok && i < rows * cols; ++i) {
      const uint64_t order = u64();
      if (!ok) break;
      if (order != 5) throw Error(kValidationError, std::string("corrupt PEPS site order in '") + path + "'");
      std::vector<int64_t> shape(order);
      uint64_t elems = 1;
      for (auto& e : shape) {
        const uint64_t v = u64();
        if (ok && (v < 1 || v >= kMaxExtent))
          throw Error(kValidationError, std::string("corrupt PEPS site extent in '") + path + "'");
        e = static_cast<int64_t>(v);
        elems = (elems > file_bytes / v) ? file_bytes + 1 : elems * v;  // saturates, no overflow
      }
      if (!ok) break;
      if (elems > file_bytes / 16) ok = false;  // more data than the file holds: truncated
      if (!ok) break;
      DTensor t = c->ctx->empty(shape);
      std::vector<double2> h(static_cast<size_t>(t.size()));
      if (!h.empty() && fread(h.data(), sizeof(double2), h.size(), f) != h.size()) ok = false;
      if (!ok) break;
      if (!h.empty()) {
        PEPSB_CUDA(cudaMemcpyAsync(t.data(), h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice,
                                   c->ctx->stream));
        mark_real(*c->ctx, t);  // (syncs: h is a host temporary)
      }
      st.sites.push_back(t);
    }
    if (!ok || st.sites.size() != rows * cols)
      throw Error(kValidationError, std::string("truncated PEPS container '") + path + "'");
    st.validate();
    *out = new pepsb_state{st};
  });
}

int pepsb_state_dims(const pepsb_state* s, int* rows, int* cols, int* d) {
  return guard([&] {
    need(s, "state");
    *rows = s->s.rows;
    *cols = s->s.cols;
    *d = s->s.d;
  });
}

int pepsb_state_site(const pepsb_state* s, int row, int col, pepsb_tensor** out) {
  return guard([&] {
    need(s, "state");
    if (row < 0 || col < 0 || row >= s->s.rows || col >= s->s.cols) throw Error(kValidationError, "site outside the grid");
    *out = wrap(s->s.site(row, col));
  });
}

void pepsb_state_free(pepsb_state* s) { delete s; }

int pepsb_boundary_create(pepsb_ctx* c, int n, pepsb_tensor* const* sites, const int64_t* phys, pepsb_boundary** out) {
  return guard([&] {
    need(c, "ctx");
    BoundaryD b;
    for (int i = 0; i < n; ++i) {
      need(sites[i], "site");
      if (sites[i]->t.shape.size() != 3) throw Error(kShapeError, "boundary sites must be order 3");
      b.sites.push_back(sites[i]->t);
      b.phys.emplace_back(phys[2 * i], phys[2 * i + 1]);
      if (phys[2 * i] * phys[2 * i + 1] != sites[i]->t.shape[0])
        throw Error(kShapeError, "boundary phys pair does not match site extent");
    }
    b.validate();
    *out = new pepsb_boundary{b};
  });
}

int pepsb_boundary_length(const pepsb_boundary* b) { return b ? static_cast<int>(b->b.sites.size()) : -1; }

int pepsb_boundary_site(const pepsb_boundary* b, int i, pepsb_tensor** out) {
  return guard([&] {
    need(b, "boundary");
    if (i < 0 || i >= static_cast<int>(b->b.sites.size())) throw Error(kValidationError, "site index out of range");
    *out = wrap(b->b.sites[i]);
  });
}

int pepsb_boundary_phys(const pepsb_boundary* b, int64_t* pairs) {
  return guard([&] {
    need(b, "boundary");
    for (size_t i = 0; i < b->b.phys.size(); ++i) {
      pairs[2 * i] = b->b.phys[i].first;
      pairs[2 * i + 1] = b->b.phys[i].second;
    }
  });
}

void pepsb_boundary_free(pepsb_boundary* b) { delete b; }

int pepsb_two_layer_first_row(pepsb_ctx* c, const pepsb_state* bra, const pepsb_state* ket, pepsb_boundary** out) {
  return guard([&] {
    need(c, "ctx");
    need(bra, "bra");
    need(ket, "ket");
    *out = new pepsb_boundary{two_layer_first_row(*c->ctx, bra->s, ket->s)};
  });
}

int pepsb_two_layer_apply_row(pepsb_ctx* c, const pepsb_boundary* top, const pepsb_state* bra, const pepsb_state* ket,
                              int row, const pepsb_contract_opt* opt, uint64_t tag, pepsb_boundary** out) {
  return guard([&] {
    need(c, "ctx");
    need(top, "top");
    need(bra, "bra");
    need(ket, "ket");
    if (row < 0 || row >= bra->s.rows) throw Error(kValidationError, "row outside the grid");
    *out = new pepsb_boundary{two_layer_apply_row(*c->ctx, top->b, bra->s, ket->s, row, opt_of(opt), tag)};
  });
}

int pepsb_contract_two_layer(pepsb_ctx* c, const pepsb_state* bra, const pepsb_state* ket, const pepsb_contract_opt* opt,
                             double* re, double* im) {
  return guard([&] {
    need(c, "ctx");
    auto v = contract_two_layer(*c->ctx, bra->s, ket->s, opt_of(opt));
    *re = v.first;
    *im = v.second;
  });
}

int pepsb_comm_unique_id(unsigned char* id128) {
  return guard([&] {
    need(id128, "id");
    comm_unique_id(id128);
  });
}

int pepsb_comm_init(pepsb_ctx* c, const unsigned char* id128, int rank, int world) {
  return guard([&] {
    need(c, "ctx");
    need(id128, "id");
    comm_init(*c->ctx, id128, rank, world);
  });
}

int pepsb_comm_destroy(pepsb_ctx* c) {
  return guard([&] {
    need(c, "ctx");
    comm_destroy(*c->ctx);
  });
}

int pepsb_two_layer_apply_row_sharded(pepsb_ctx* c, const pepsb_boundary* top, const pepsb_state* bra,
                                      const pepsb_state* ket, int row, const pepsb_contract_opt* opt,
                                      uint64_t tag, pepsb_boundary** out) {
  return guard([&] {
    need(c, "ctx");
    need(top, "top");
    need(bra, "bra");
    need(ket, "ket");
    if (row < 0 || row >= bra->s.rows) throw Error(kValidationError, "row outside the grid");
    *out = new pepsb_boundary{two_layer_apply_row_sharded(*c->ctx, top->b, bra->s, ket->s, row, opt_of(opt), tag)};
  });
}

int pepsb_contract_two_layer_sharded(pepsb_ctx* c, const pepsb_state* bra, const pepsb_state* ket,
                                     const pepsb_contract_opt* opt, double* re, double* im) {
  return guard([&] {
    need(c, "ctx");
    need(bra, "bra");
    need(ket, "ket");
    auto v = contract_two_layer_sharded(*c->ctx, bra->s, ket->s, opt_of(opt));
    *re = v.first;
    *im = v.second;
  });
}

int pepsb_chain_scalar(pepsb_ctx* c, const pepsb_boundary* b, double* re, double* im) {
  return guard([&] {
    need(c, "ctx");
    need(b, "boundary");
    auto v = chain_scalar(*c->ctx, b->b);
    *re = v.first;
    *im = v.second;
  });
}

int pepsb_build_row_cache(pepsb_ctx* c, const pepsb_state* s, const pepsb_contract_opt* opt, pepsb_row_cache** out) {
  return guard([&] {
    need(c, "ctx");
    need(s, "state");
    *out = new pepsb_row_cache{build_row_cache(*c->ctx, s->s, opt_of(opt))};
  });
}

int pepsb_flip_vertical(pepsb_ctx* c, const pepsb_state* s, pepsb_state** out) {
  return guard([&] {
    need(c, "ctx");
    need(s, "state");
    PepsStateD f = flip_vertical(*c->ctx, s->s);
    f.validate();
    *out = new pepsb_state{f};
  });
}

int pepsb_row_cache_get(const pepsb_row_cache* rc, int which, int k, pepsb_boundary** out) {
  return guard([&] {
    need(rc, "cache");
    const auto& v = which == 0 ? rc->c.tops : rc->c.bots;
    if (k < 0 || k >= static_cast<int>(v.size())) throw Error(kValidationError, "row out of range");
    *out = new pepsb_boundary{v[k]};
  });
}

void pepsb_row_cache_free(pepsb_row_cache* c) { delete c; }

int pepsb_band_environment(pepsb_ctx* c, const pepsb_boundary* top, const pepsb_state* bra, const pepsb_state* ket,
                           int r0, int r1, const pepsb_boundary* bottom, pepsb_band_env** out) {
  return guard([&] {
    need(c, "ctx");
    *out = new pepsb_band_env{band_environment(*c->ctx, top ? &top->b : nullptr, bra->s, ket->s, r0, r1,
                                               bottom ? &bottom->b : nullptr)};
  });
}

int pepsb_band_splice(pepsb_ctx* c, const pepsb_band_env* env, const pepsb_boundary* top, const pepsb_state* bra,
                      const pepsb_state* ket, const pepsb_boundary* bottom, int npieces, const int* rc,
                      pepsb_tensor* const* ops, const int* nbonds, const int* bond_ids, int c0, int c1, double* re,
                      double* im) {
  return guard([&] {
    need(c, "ctx");
    need(env, "env");
    auto v = band_splice(*c->ctx, env->e, top ? &top->b : nullptr, bra->s, ket->s, bottom ? &bottom->b : nullptr,
                         pieces_of(npieces, rc, ops, nbonds, bond_ids), c0, c1);
    *re = v.first;
    *im = v.second;
  });
}

int pepsb_band_value(pepsb_ctx* c, const pepsb_boundary* top, const pepsb_state* bra, const pepsb_state* ket, int r0,
                     int r1, const pepsb_boundary* bottom, int npieces, const int* rc, pepsb_tensor* const* ops,
                     const int* nbonds, const int* bond_ids, double* re, double* im) {
  return guard([&] {
    need(c, "ctx");
    auto v = band_value(*c->ctx, top ? &top->b : nullptr, bra->s, ket->s, r0, r1, bottom ? &bottom->b : nullptr,
                        pieces_of(npieces, rc, ops, nbonds, bond_ids));
    *re = v.first;
    *im = v.second;
  });
}

void pepsb_band_env_free(pepsb_band_env* e) { delete e; }

int pepsb_approx_apply_mpo(pepsb_ctx* c, int n, pepsb_tensor* const* mps_sites, pepsb_tensor* const* mpo_sites,
                           const pepsb_trunc* policy, int strategy, int absorb, const pepsb_rsvd* rsvd,
                           uint64_t seed_base, pepsb_tensor** out_sites) {
  return guard([&] {
    need(c, "ctx");
    need(policy, "policy");
    need(rsvd, "rsvd");
    if (n < 1) throw Error(kShapeError, "empty MPS");
    MpsD s;
    MpoD o;
    for (int i = 0; i < n; ++i) {
      need(mps_sites[i], "MPS site");
      need(mpo_sites[i], "MPO site");
      s.sites.push_back(mps_sites[i]->t);
      o.sites.push_back(mpo_sites[i]->t);
    }
    ApplyOptD ao;
    ao.policy = Trunc{policy->max_rank, policy->rel_cutoff};
    ao.strategy = strategy;
    ao.absorb = absorb;
    ao.rsvd = Rsvd{rsvd->power_iters, rsvd->oversample, rsvd->seed};
    ao.seed_base = seed_base;
    MpsD out = approx_apply_mpo(*c->ctx, s, o, ao);
    for (int i = 0; i < n; ++i) out_sites[i] = wrap(out.sites[i]);
  });
}

int pepsb_contract_one_layer(pepsb_ctx* c, int rows, int cols, pepsb_tensor* const* sites, int family,
                             const pepsb_contract_opt* opt, uint64_t memory_budget, double* re, double* im) {
  return guard([&] {
    need(c, "ctx");
    need(opt, "options");
    GridD g;
    g.rows = rows;
    g.cols = cols;
    for (int i = 0; i < rows * cols; ++i) {
      need(sites[i], "grid site");
      g.sites.push_back(sites[i]->t);
    }
    auto v = contract_one_layer(*c->ctx, g, family, opt_of(opt), memory_budget);
    *re = v.first;
    *im = v.second;
  });
}

int pepsb_expectation(pepsb_ctx* c, const pepsb_state* s, int nterms, const double* coeff, const int* nsites,
                      const int* rc, pepsb_tensor* const* ops, const pepsb_expectation_opt* opt,
                      pepsb_expectation_result* out) {
  return guard([&] {
    need(c, "ctx");
    need(s, "state");
    need(opt, "options");
    need(out, "result");
    if (nterms < 0) throw Error(kValidationError, "negative term count");
    std::vector<LocalTermD> terms(static_cast<size_t>(nterms));
    for (int i = 0; i < nterms; ++i) {
      need(ops[i], "term operator");
      LocalTermD& t = terms[i];
      t.coeff_re = coeff[2 * i];
      t.coeff_im = coeff[2 * i + 1];
      if (nsites[i] != 1 && nsites[i] != 2) throw Error(kValidationError, "terms act on one or two sites");
      for (int k = 0; k < nsites[i]; ++k) t.sites.emplace_back(rc[4 * i + 2 * k], rc[4 * i + 2 * k + 1]);
      t.op = ops[i]->t;
      const size_t want = nsites[i] == 1 ? 2 : 4;
      if (t.op.shape.size() != want) throw Error(kShapeError, "term operator must have 2 (1-site) or 4 (2-site) axes");
    }
    ExpectOptD o;
    o.contract = opt_of(&opt->contract);
    o.use_cache = opt->use_cache != 0;
    o.shared_environments = opt->shared_environments != 0;
    o.allow_complex = opt->allow_complex != 0;
    ExpectResultD r = expectation(*c->ctx, s->s, terms, o);
    out->value = r.value;
    out->norm_sq = r.norm_sq;
    out->raw_sum[0] = r.raw_re;
    out->raw_sum[1] = r.raw_im;
    out->complex_value[0] = r.cx_re;
    out->complex_value[1] = r.cx_im;
    out->full_sweeps = r.full_sweeps;
    out->band_contractions = r.band_contractions;
    out->flops = r.flops;
  });
}

int pepsb_hermitian_exp(pepsb_ctx* c, const pepsb_tensor* op, double coeff, double tau, pepsb_tensor** out) {
  return guard([&] {
    need(c, "ctx");
    need(op, "operator");
    *out = wrap(hermitian_exp(*c->ctx, op->t, coeff, tau));
  });
}

int pepsb_apply_one_site(pepsb_ctx* c, const pepsb_state* s, const pepsb_tensor* gate, int nsites, const int* rc,
                         pepsb_state** out) {
  return guard([&] {
    need(c, "ctx");
    need(s, "state");
    need(gate, "gate");
    std::vector<std::pair<int, int>> sites;
    for (int i = 0; i < nsites; ++i) sites.push_back({rc[2 * i], rc[2 * i + 1]});
    *out = new pepsb_state{apply_one_site_batch(*c->ctx, s->s, gate->t, sites)};
  });
}

int pepsb_apply_two_site(pepsb_ctx* c, const pepsb_state* s, const pepsb_tensor* gate, int nbonds, const int* bonds,
                         const pepsb_trunc* policy, pepsb_state** out) {
  return guard([&] {
    need(c, "ctx");
    need(s, "state");
    need(gate, "gate");
    std::vector<std::array<int, 4>> bl;
    for (int i = 0; i < nbonds; ++i) bl.push_back({bonds[4 * i], bonds[4 * i + 1], bonds[4 * i + 2], bonds[4 * i + 3]});
    Trunc t = trunc_of(policy);
    if (!policy) t = Trunc{0, 1e-14};
    *out = new pepsb_state{apply_two_site_batch(*c->ctx, s->s, gate->t, bl, t)};
  });
}

int pepsb_ite_tfim(pepsb_ctx* c, const pepsb_state* s, double J, double h, double tau, int steps, uint64_t rank,
                   pepsb_state** out) {
  return guard([&] {
    need(c, "ctx");
    need(s, "state");
    *out = new pepsb_state{ite_tfim(*c->ctx, s->s, J, h, tau, steps, rank)};
  });
}

}  // extern "C"
