// Reference-side shim: the file a maintainer adds to the reference tree as
// proj/src/gpu_backend.cpp.  It binds the reference's
// public C++ API (proj/include/peps/*.hpp) to this repo's C ABI
// (include/peps_b200.h) without changing any reference algorithm code:
//
//   peps::b200::einsumsvd           replaces peps::einsumsvd          (decomposition.hpp:65-67)
//   peps::b200::contract_two_layer  replaces peps::contract_two_layer (contraction.hpp:89-90)
//
// Tensors cross the boundary in the reference's own layout (row-major
// complex128, tensor.hpp:13-20), so the conversion is one memcpy each way;
// status codes map back onto the reference exception family (errors.hpp).
// Compiled against /root/reference/proj/include by tests/test_integration.py
// (CPU) and exercised on the device by oracle/_ref/shim_check (GPU test).
#include "gpu_backend.hpp"

#include <algorithm>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "peps/errors.hpp"
#include "peps_b200.h"

namespace peps::b200 {

namespace {

void check(int rc) {
  if (rc == PEPSB_OK) return;
  const std::string m = pepsb_last_error();
  switch (rc) {
    case PEPSB_E_SHAPE: throw ShapeError(m);
    case PEPSB_E_VALIDATION: throw ValidationError(m);
    case PEPSB_E_RESOURCE: throw ResourceError(m, 0);
    case PEPSB_E_NUMERICAL: throw NumericalError(m);
    case PEPSB_E_CONFIG: throw ConfigError(m);
    default: throw std::runtime_error(m);
  }
}

struct Context {
  pepsb_ctx* h = nullptr;
  Context() { check(pepsb_ctx_create(0, &h)); }
  ~Context() { pepsb_ctx_destroy(h); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
};

Context& ctx() {
  static Context c;
  return c;
}

// Move-only RAII owner of one device tensor handle: a vector of these may
// reallocate without ever copying (and later double-freeing) a handle.
class DevTensor {
 public:
  explicit DevTensor(const Tensor& t) {
    std::vector<int64_t> s(t.shape().begin(), t.shape().end());
    check(pepsb_tensor_from_host(ctx().h, static_cast<int>(s.size()), s.data(),
                                 reinterpret_cast<const double*>(t.data().data()), &h_));
  }
  explicit DevTensor(pepsb_tensor* p) : h_(p) {}
  DevTensor(const DevTensor&) = delete;
  DevTensor& operator=(const DevTensor&) = delete;
  DevTensor(DevTensor&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  DevTensor& operator=(DevTensor&& o) noexcept {
    if (this != &o) {
      if (h_) pepsb_tensor_free(h_);
      h_ = std::exchange(o.h_, nullptr);
    }
    return *this;
  }
  ~DevTensor() {
    if (h_) pepsb_tensor_free(h_);
  }
  pepsb_tensor* get() const { return h_; }
  Tensor to_host() const {
    const int nd = pepsb_tensor_ndim(h_);
    std::vector<int64_t> s(static_cast<size_t>(std::max(nd, 0)));
    check(pepsb_tensor_shape(h_, s.data()));
    Tensor out(Shape(s.begin(), s.end()));
    check(pepsb_tensor_to_host(ctx().h, h_, reinterpret_cast<double*>(out.data().data())));
    return out;
  }

 private:
  pepsb_tensor* h_ = nullptr;
};

// Move-only owner of a device PEPS state (its sites are owned by `keep`).
class DevState {
 public:
  explicit DevState(const PepsState& s) {
    keep_.reserve(s.sites().size());
    std::vector<pepsb_tensor*> hs;
    hs.reserve(s.sites().size());
    for (const auto& t : s.sites()) {
      keep_.emplace_back(t);
      hs.push_back(keep_.back().get());
    }
    check(pepsb_state_create(ctx().h, static_cast<int>(s.rows()), static_cast<int>(s.cols()),
                             static_cast<int>(s.phys_dim()), hs.data(), &h_));
  }
  DevState(const DevState&) = delete;
  DevState& operator=(const DevState&) = delete;
  ~DevState() {
    if (h_) pepsb_state_free(h_);
  }
  const pepsb_state* get() const { return h_; }

 private:
  std::vector<DevTensor> keep_;
  pepsb_state* h_ = nullptr;
};

int strategy_of(SvdStrategy s) { return s == SvdStrategy::exact ? PEPSB_EXACT : PEPSB_IMPLICIT_RSVD; }

}  // namespace

EinsumsvdResult einsumsvd(const ImplicitOperator& net, const TruncationPolicy& policy, SvdStrategy strategy,
                          Absorb absorb, const RsvdConfig& cfg) {
  const auto& tensors = net.tensors();
  std::vector<DevTensor> ts;
  ts.reserve(tensors.size());
  std::vector<pepsb_tensor*> hs;
  hs.reserve(tensors.size());
  std::string labels;
  for (size_t i = 0; i < tensors.size(); ++i) {
    ts.emplace_back(tensors[i]);
    hs.push_back(ts.back().get());
    labels += (i ? "," : "") + net.labels()[i];
  }
  const pepsb_trunc tp{policy.max_rank, policy.rel_cutoff};
  const pepsb_rsvd rc{cfg.power_iters, cfg.oversample, cfg.seed};
  pepsb_tensor *t1 = nullptr, *t2 = nullptr;
  std::vector<double> s(std::min(net.row_extent(), net.col_extent()));
  int64_t rank = 0;
  int clamped = 0;
  check(pepsb_einsumsvd(ctx().h, static_cast<int>(hs.size()), hs.data(), labels.c_str(), net.row_labels().c_str(),
                        net.col_labels().c_str(), &tp, strategy_of(strategy), static_cast<int>(absorb), &rc, &t1,
                        &t2, s.data(), static_cast<int64_t>(s.size()), &rank, &clamped));
  DevTensor d1(t1), d2(t2);
  EinsumsvdResult out;
  out.t1 = d1.to_host();
  out.t2 = d2.to_host();
  out.s.assign(s.begin(), s.begin() + rank);
  out.rank_clamped = clamped != 0;
  return out;
}

cplx contract_two_layer(const PepsState& bra, const PepsState& ket, const ContractOption& opt) {
  DevState b(bra);
  std::unique_ptr<DevState> k;
  if (&bra != &ket) k = std::make_unique<DevState>(ket);
  const pepsb_contract_opt o{{opt.trunc.max_rank, opt.trunc.rel_cutoff},
                             strategy_of(opt.strategy),
                             {opt.rsvd.power_iters, opt.rsvd.oversample, opt.rsvd.seed},
                             opt.canonicalize ? 1 : 0,
                             opt.seed};
  double re = 0.0, im = 0.0;
  check(pepsb_contract_two_layer(ctx().h, b.get(), k ? k->get() : b.get(), &o, &re, &im));
  return {re, im};
}

}  // namespace peps::b200
