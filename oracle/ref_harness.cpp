// TEST INFRASTRUCTURE ONLY — the parity oracle, never the product path.
//
// C-ABI harness over the UNMODIFIED reference library compiled from
// /root/reference/proj/src (see oracle/Makefile).  It lets the Python tests,
// the golden-fixture generator and bench.py's CPU-baseline leg call the
// reference's own public API (proj/include/peps/*.hpp) with plain arrays.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load the resulting oracle/_ref/libpeps_ref.so.
//
// Tensors cross the boundary as interleaved (re, im) float64 arrays in the
// reference's row-major order (proj/include/peps/tensor.hpp:16-19).

#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "peps/contraction.hpp"
#include "peps/decomposition.hpp"
#include "peps/einsum.hpp"
#include "peps/errors.hpp"
#include "peps/implicit.hpp"
#include "peps/instrument.hpp"
#include "peps/linalg.hpp"
#include "peps/mps.hpp"
#include "peps/drivers.hpp"
#include "peps/optimize.hpp"
#include "peps/observables.hpp"
#include "peps/rng.hpp"
#include "peps/state.hpp"

extern "C" void openblas_set_num_threads(int n);
extern "C" int openblas_get_num_threads(void);

using namespace peps;

namespace {

thread_local std::string g_err;
thread_local int g_err_type = 0;

struct Bag {
  std::vector<Tensor> tensors;
  std::vector<double> doubles;
  std::string text;  // JSON front ends
};

template <class F>
Bag* guarded(F&& f) {
  try {
    g_err.clear();
    g_err_type = 0;
    Bag* b = new Bag();
    try {
      f(*b);
    } catch (...) {
      delete b;
      throw;
    }
    return b;
  } catch (const ShapeError& e) {
    g_err = e.what(), g_err_type = 1;
  } catch (const ValidationError& e) {
    g_err = e.what(), g_err_type = 2;
  } catch (const ResourceError& e) {
    g_err = e.what(), g_err_type = 3;
  } catch (const NumericalError& e) {
    g_err = e.what(), g_err_type = 4;
  } catch (const ConfigError& e) {
    g_err = e.what(), g_err_type = 5;
  } catch (const std::exception& e) {
    g_err = e.what(), g_err_type = 9;
  }
  return nullptr;
}

Tensor make_tensor(int ndim, const int64_t* shape, const double* data) {
  Shape sh;
  std::size_t n = 1;
  for (int i = 0; i < ndim; ++i) {
    sh.push_back(static_cast<std::size_t>(shape[i]));
    n *= static_cast<std::size_t>(shape[i]);
  }
  std::vector<cplx> v(n);
  std::memcpy(v.data(), data, n * sizeof(cplx));
  return Tensor(sh, std::move(v));
}

// Unpacks a flat tensor list: ndims[i], shapes concatenated, data pointers.
std::vector<Tensor> make_list(int nt, const int* ndims, const int64_t* shapes,
                              const double* const* datas) {
  std::vector<Tensor> out;
  const int64_t* sp = shapes;
  for (int i = 0; i < nt; ++i) {
    out.push_back(make_tensor(ndims[i], sp, datas[i]));
    sp += ndims[i];
  }
  return out;
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

PepsState make_state(int rows, int cols, int d, const int* ndims, const int64_t* shapes,
                     const double* const* datas) {
  return PepsState(rows, cols, d, make_list(rows * cols, ndims, shapes, datas));
}

ContractOption make_opt(int64_t m, uint64_t seed, int power_iters, int oversample,
                        int canonicalize) {
  ContractOption o = ContractOption::two_layer_opt(static_cast<std::size_t>(m), seed, power_iters);
  o.rsvd.oversample = oversample;
  o.canonicalize = canonicalize != 0;
  return o;
}

TwoLayerBoundary make_boundary(int n, const int* ndims, const int64_t* shapes,
                               const double* const* datas, const int64_t* phys_pairs) {
  TwoLayerBoundary b;
  b.mps.sites = make_list(n, ndims, shapes, datas);
  for (int i = 0; i < n; ++i) b.phys.emplace_back(phys_pairs[2 * i], phys_pairs[2 * i + 1]);
  return b;
}

void push_boundary(Bag& b, const TwoLayerBoundary& t) {
  for (const auto& s : t.mps.sites) b.tensors.push_back(s);
  for (const auto& p : t.phys) {
    b.doubles.push_back(static_cast<double>(p.first));
    b.doubles.push_back(static_cast<double>(p.second));
  }
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Transverse-field Ising model in colour order (fields; even/odd horizontal;
// even/odd vertical).  H = -J sum ZZ - h sum X.
Observable tfim_colour_order(int rows, int cols, double J, double h) {
  Observable obs;
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c)
      obs.add(cplx(-h, 0.0), Coord{(std::size_t)r, (std::size_t)c}, gates::X());
  Tensor zz = gates::two_site(gates::Z(), gates::Z());
  for (int par = 0; par < 2; ++par)
    for (int r = 0; r < rows; ++r)
      for (int c = par; c + 1 < cols; c += 2)
        obs.add(cplx(-J, 0.0), Coord{(std::size_t)r, (std::size_t)c},
                Coord{(std::size_t)r, (std::size_t)c + 1}, zz);
  for (int par = 0; par < 2; ++par)
    for (int r = par; r + 1 < rows; r += 2)
      for (int c = 0; c < cols; ++c)
        obs.add(cplx(-J, 0.0), Coord{(std::size_t)r, (std::size_t)c},
                Coord{(std::size_t)r + 1, (std::size_t)c}, zz);
  return obs;
}

// Replicates the anonymous apply_ite_term of proj/src/drivers.cpp:56-71 with
// the public API (adjacent terms only, which is all TFIM has).
PepsState ite_term(const PepsState& s, const LocalTerm& term, double tau, const UpdateOption& opt) {
  if (term.sites.size() == 1) {
    Tensor h = term.op * term.coeff;
    Tensor gate = hermitian_function(h, [tau](double x) { return std::exp(-tau * x); });
    return apply_one_site(s, gate, term.sites[0]);
  }
  const std::size_t d = s.phys_dim();
  Tensor h = term.op.reshape({d * d, d * d}) * term.coeff;
  Tensor gate =
      hermitian_function(h, [tau](double x) { return std::exp(-tau * x); }).reshape({d, d, d, d});
  return apply_two_site(s, gate, term.sites[0], term.sites[1], opt);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
int ref_last_error_type() { return g_err_type; }

int ref_bag_ntensors(Bag* b) { return static_cast<int>(b->tensors.size()); }
int ref_bag_tensor_ndim(Bag* b, int i) { return static_cast<int>(b->tensors[i].order()); }
void ref_bag_tensor_shape(Bag* b, int i, int64_t* shape) {
  for (std::size_t a = 0; a < b->tensors[i].order(); ++a) shape[a] = b->tensors[i].extent(a);
}
void ref_bag_tensor_data(Bag* b, int i, double* out) {
  std::memcpy(out, b->tensors[i].data().data(), b->tensors[i].size() * sizeof(cplx));
}
int ref_bag_ndoubles(Bag* b) { return static_cast<int>(b->doubles.size()); }
void ref_bag_doubles(Bag* b, double* out) {
  std::memcpy(out, b->doubles.data(), b->doubles.size() * sizeof(double));
}
void ref_bag_free(Bag* b) { delete b; }
int64_t ref_bag_text_len(Bag* b) { return static_cast<int64_t>(b->text.size()); }
void ref_bag_text(Bag* b, char* out) { std::memcpy(out, b->text.data(), b->text.size()); }

// optimize.cpp:189-194 on an analytic objective (fn 0: Rosenbrock, 1: a shifted
// quadratic + cosine bump); doubles: [status_converged, evaluations, best_f, trace...]
Bag* ref_minimize(const char* method, int fn, int n, const double* x0, int max_evals, double tol, double step) {
  return guarded([&](Bag& b) {
    Objective f = [fn](std::span<const double> x) {
      double v = 0.0;
      if (fn == 0) {
        for (size_t i = 0; i + 1 < x.size(); ++i)
          v += 100.0 * (x[i + 1] - x[i] * x[i]) * (x[i + 1] - x[i] * x[i]) + (1.0 - x[i]) * (1.0 - x[i]);
      } else {
        for (size_t i = 0; i < x.size(); ++i) v += (x[i] - 0.3 * (i + 1)) * (x[i] - 0.3 * (i + 1)) + 0.1 * std::cos(3.0 * x[i]);
      }
      return v;
    };
    OptimConfig oc;
    oc.max_evaluations = static_cast<std::size_t>(max_evals);
    oc.tolerance = tol;
    oc.initial_step = step;
    OptimResult r = minimize(method, f, std::span<const double>(x0, static_cast<size_t>(n)), oc);
    b.doubles = {r.status == "converged" ? 1.0 : 0.0, static_cast<double>(r.evaluations), r.best_f};
    for (double v : r.trace) b.doubles.push_back(v);
    b.tensors.push_back(Tensor({r.best_x.size()}));
    for (size_t i = 0; i < r.best_x.size(); ++i) b.tensors.back().data()[i] = r.best_x[i];
  });
}

// JSON front ends (drivers.cpp:265-550): 0 run_expect_json, 1 run_vqe_json, 2 run_ite_json
Bag* ref_json_driver(int which, const char* config) {
  return guarded([&](Bag& b) {
    const std::string cfg(config);
    b.text = which == 0 ? run_expect_json(cfg) : which == 1 ? run_vqe_json(cfg) : run_ite_json(cfg);
  });
}

void ref_set_threads(int n) { openblas_set_num_threads(n); }
int ref_get_threads() { return openblas_get_num_threads(); }
void ref_reset_counters() { instr::reset(); }
uint64_t ref_flops() { return instr::flops(); }
uint64_t ref_einsumsvd_flops() { return instr::einsumsvd_flops(); }
uint64_t ref_peak_elements() { return instr::peak_elements(); }

uint64_t ref_derive_seed(uint64_t base, int nparts, const uint64_t* parts) {
  uint64_t s = base;
  for (int i = 0; i < nparts; ++i) s = derive_seed(s, parts[i]);
  return s;
}

Bag* ref_random_tensor(int ndim, const int64_t* shape, uint64_t seed, int real) {
  return guarded([&](Bag& b) {
    Shape sh(shape, shape + ndim);
    b.tensors.push_back(real ? random_tensor_real(sh, seed) : random_tensor(sh, seed));
  });
}

Bag* ref_contract(const char* spec, int nt, const int* ndims, const int64_t* shapes,
                  const double* const* datas) {
  return guarded([&](Bag& b) {
    auto ts = make_list(nt, ndims, shapes, datas);
    double t0 = now_s();
    b.tensors.push_back(contract(std::string(spec), std::span<const Tensor>(ts)));
    b.doubles.push_back(now_s() - t0);
  });
}

// mode 0: apply(probe)  1: adjoint_apply(probe)  2: materialize()
Bag* ref_implicit(int mode, int nt, const int* ndims, const int64_t* shapes,
                  const double* const* datas, const char* labels_csv, const char* rows,
                  const char* cols, int probe_ndim, const int64_t* probe_shape,
                  const double* probe_data) {
  return guarded([&](Bag& b) {
    ImplicitOperator op(make_list(nt, ndims, shapes, datas), split_csv(labels_csv), rows, cols);
    double t0 = now_s();
    if (mode == 2) {
      b.tensors.push_back(op.materialize());
    } else {
      Tensor p = make_tensor(probe_ndim, probe_shape, probe_data);
      b.tensors.push_back(mode == 0 ? op.apply(p) : op.adjoint_apply(p));
    }
    b.doubles.push_back(now_s() - t0);
  });
}

// doubles: [s_0..s_{rank-1}, rank_clamped, seconds, einsumsvd_flops]
Bag* ref_einsumsvd(int nt, const int* ndims, const int64_t* shapes, const double* const* datas,
                   const char* labels_csv, const char* rows, const char* cols, uint64_t max_rank,
                   double rel_cutoff, int strategy, int absorb, int power_iters, int oversample,
                   uint64_t seed) {
  return guarded([&](Bag& b) {
    ImplicitOperator op(make_list(nt, ndims, shapes, datas), split_csv(labels_csv), rows, cols);
    TruncationPolicy pol{static_cast<std::size_t>(max_rank), rel_cutoff};
    RsvdConfig cfg{power_iters, oversample, seed};
    uint64_t f0 = instr::einsumsvd_flops();
    double t0 = now_s();
    EinsumsvdResult r = einsumsvd(op, pol, strategy == 0 ? SvdStrategy::exact : SvdStrategy::implicit_rsvd,
                                  absorb == 0 ? Absorb::split : (absorb == 1 ? Absorb::left : Absorb::right),
                                  cfg);
    double dt = now_s() - t0;
    b.tensors.push_back(r.t1);
    b.tensors.push_back(r.t2);
    b.doubles = r.s;
    b.doubles.push_back(r.rank_clamped ? 1.0 : 0.0);
    b.doubles.push_back(dt);
    b.doubles.push_back(static_cast<double>(instr::einsumsvd_flops() - f0));
  });
}

// doubles: [s..., rank_clamped]
Bag* ref_randomized_svd(int nt, const int* ndims, const int64_t* shapes, const double* const* datas,
                        const char* labels_csv, const char* rows, const char* cols,
                        uint64_t max_rank, double rel_cutoff, int power_iters, int oversample,
                        uint64_t seed) {
  return guarded([&](Bag& b) {
    ImplicitOperator op(make_list(nt, ndims, shapes, datas), split_csv(labels_csv), rows, cols);
    SvdTriple t = randomized_svd(op, TruncationPolicy{static_cast<std::size_t>(max_rank), rel_cutoff},
                                 RsvdConfig{power_iters, oversample, seed});
    b.tensors.push_back(t.u);
    b.tensors.push_back(t.v);
    b.doubles = t.s;
    b.doubles.push_back(t.rank_clamped ? 1.0 : 0.0);
  });
}

Bag* ref_gram_orthogonalize(int ndim, const int64_t* shape, const double* data, int split) {
  return guarded([&](Bag& b) {
    auto [q, r] = gram_orthogonalize(make_tensor(ndim, shape, data), static_cast<std::size_t>(split));
    b.tensors.push_back(q);
    b.tensors.push_back(r);
  });
}

Bag* ref_svd(int ndim, const int64_t* shape, const double* data, int split) {
  return guarded([&](Bag& b) {
    SvdResult r = svd(make_tensor(ndim, shape, data), static_cast<std::size_t>(split));
    b.tensors.push_back(r.u);
    b.tensors.push_back(r.v);
    b.doubles = r.s;
  });
}

Bag* ref_eigh(int n, const double* data) {
  return guarded([&](Bag& b) {
    int64_t sh[2] = {n, n};
    EighResult r = eigh(make_tensor(2, sh, data));
    b.tensors.push_back(r.vectors);
    b.doubles = r.values;
  });
}

Bag* ref_two_layer_first_row(int rows, int cols, int d, const int* ndims, const int64_t* shapes,
                             const double* const* datas) {
  return guarded([&](Bag& b) {
    PepsState s = make_state(rows, cols, d, ndims, shapes, datas);
    push_boundary(b, two_layer_first_row(s, s));
  });
}

// Top boundary (cols sites + phys pairs) absorbing row `row` of the state
// (bra = ket = state).  doubles: [phys pairs..., seconds, flops]
Bag* ref_two_layer_apply_row(int rows, int cols, int d, const int* ndims, const int64_t* shapes,
                             const double* const* datas, const int* top_ndims,
                             const int64_t* top_shapes, const double* const* top_datas,
                             const int64_t* phys_pairs, int row, int64_t m, uint64_t seed,
                             int power_iters, int oversample, int canonicalize, uint64_t tag) {
  return guarded([&](Bag& b) {
    PepsState s = make_state(rows, cols, d, ndims, shapes, datas);
    TwoLayerBoundary top = make_boundary(cols, top_ndims, top_shapes, top_datas, phys_pairs);
    ContractOption opt = make_opt(m, seed, power_iters, oversample, canonicalize);
    uint64_t f0 = instr::flops();
    double t0 = now_s();
    TwoLayerBoundary out = two_layer_apply_row(top, s, s, static_cast<std::size_t>(row), opt, tag);
    double dt = now_s() - t0;
    push_boundary(b, out);
    b.doubles.push_back(dt);
    b.doubles.push_back(static_cast<double>(instr::flops() - f0));
  });
}

// band_environment (contraction.cpp:572-624) of band rows r0..r1 between two
// given boundaries (top above r0, bottom below r1), timed; doubles: [seconds]
Bag* ref_band_environment_time(int rows, int cols, int d, const int* ndims, const int64_t* shapes,
                               const double* const* datas, const int* top_ndims, const int64_t* top_shapes,
                               const double* const* top_datas, const int64_t* top_phys, const int* bot_ndims,
                               const int64_t* bot_shapes, const double* const* bot_datas, const int64_t* bot_phys,
                               int r0, int r1) {
  return guarded([&](Bag& b) {
    PepsState s = make_state(rows, cols, d, ndims, shapes, datas);
    TwoLayerBoundary top = make_boundary(cols, top_ndims, top_shapes, top_datas, top_phys);
    TwoLayerBoundary bot = make_boundary(cols, bot_ndims, bot_shapes, bot_datas, bot_phys);
    double t0 = now_s();
    BandEnvironment env = band_environment(&top, s, s, static_cast<std::size_t>(r0), static_cast<std::size_t>(r1),
                                           &bot);
    b.doubles.push_back(now_s() - t0);
    (void)env;
  });
}

// doubles: [re, im, seconds, flops, peak_elements]
Bag* ref_contract_two_layer(int rows, int cols, int d, const int* ndims, const int64_t* shapes,
                            const double* const* datas, int64_t m, uint64_t seed, int power_iters,
                            int oversample, int canonicalize) {
  return guarded([&](Bag& b) {
    PepsState s = make_state(rows, cols, d, ndims, shapes, datas);
    ContractOption opt = make_opt(m, seed, power_iters, oversample, canonicalize);
    uint64_t f0 = instr::flops();
    double t0 = now_s();
    cplx v = contract_two_layer(s, s, opt);
    b.doubles = {v.real(), v.imag(), now_s() - t0, static_cast<double>(instr::flops() - f0),
                 static_cast<double>(instr::peak_elements())};
  });
}

// save_peps / load_peps (state.cpp:240-299) through the reference's own code.
Bag* ref_save_peps(int rows, int cols, int d, const int* ndims, const int64_t* shapes, const double* const* datas,
                   const char* path) {
  return guarded([&](Bag& b) {
    save_peps(make_state(rows, cols, d, ndims, shapes, datas), path);
    (void)b;
  });
}

Bag* ref_load_peps(const char* path) {
  return guarded([&](Bag& b) {
    PepsState s = load_peps(path);
    for (const auto& t : s.sites()) b.tensors.push_back(t);
    b.doubles = {static_cast<double>(s.rows()), static_cast<double>(s.cols()), static_cast<double>(s.phys_dim())};
  });
}

// contract_one_layer (contraction.cpp:205-252) on an order-4 grid (up, left,
// down, right): family 0 exact (contract_exact), 1 bmps, 2 ibmps.
Bag* ref_contract_one_layer(int rows, int cols, const int* ndims, const int64_t* shapes,
                            const double* const* datas, int family, int64_t m, uint64_t seed,
                            int power_iters, int oversample, int canonicalize) {
  return guarded([&](Bag& b) {
    OneLayerGrid g(rows, cols, make_list(rows * cols, ndims, shapes, datas));
    ContractOption opt = family == 0 ? ContractOption::exact_network()
                         : family == 1 ? ContractOption::bmps_opt(static_cast<std::size_t>(m), seed)
                                       : ContractOption::ibmps_opt(static_cast<std::size_t>(m), seed, power_iters);
    opt.rsvd.oversample = oversample;
    opt.canonicalize = canonicalize != 0;
    cplx v = contract_one_layer(g, opt);
    b.doubles = {v.real(), v.imag()};
  });
}

// Exact <psi|psi> (ContractOption::exact_network, via the merged one-layer grid).
Bag* ref_inner_exact(int rows, int cols, int d, const int* ndims, const int64_t* shapes,
                     const double* const* datas) {
  return guarded([&](Bag& b) {
    PepsState s = make_state(rows, cols, d, ndims, shapes, datas);
    cplx v = inner_product(s, s, ContractOption::exact_network());
    b.doubles = {v.real(), v.imag()};
  });
}

// Cached-environment local expectations:
// build_row_cache, norm = chain_scalar(tops[n-1]); then for every term
// (kind 0: Z on site i;  kind 1: ZZ on an adjacent pair) band_environment of
// the term's band (shared per band) + band_splice, divided by the norm.
// terms: flat int array of (kind, r0, c0, r1, c1) per term.
// doubles: [norm_re, norm_im, value_0 re, value_0 im, ..., t_cache, t_bands]
Bag* ref_local_expectations(int rows, int cols, int d, const int* ndims, const int64_t* shapes,
                            const double* const* datas, int64_t m, uint64_t seed, int power_iters,
                            int oversample, int nterms, const int* terms) {
  return guarded([&](Bag& b) {
    PepsState s = make_state(rows, cols, d, ndims, shapes, datas);
    ContractOption opt = make_opt(m, seed, power_iters, oversample, 1);
    double t0 = now_s();
    RowCache cache = build_row_cache(s, opt);
    double t1 = now_s();
    const std::size_t n = s.rows();
    cplx norm = chain_scalar(cache.tops[n - 1].mps);
    b.doubles = {norm.real(), norm.imag()};
    std::vector<std::pair<std::pair<std::size_t, std::size_t>, BandEnvironment>> envs;
    Tensor z = gates::Z();
    // ZZ pieces exactly as observables.cpp:284-295 (split_two_site) builds them.
    Tensor zz = gates::two_site(z, z);
    SvdResult sv = svd(zz.permute({0, 2, 1, 3}), 2);
    std::size_t g = decomp_detail::retained_rank(sv.s, TruncationPolicy{static_cast<std::size_t>(d * d), 1e-14});
    std::vector<double> w(sv.s.begin(), sv.s.begin() + g);
    for (auto& x : w) x = std::sqrt(x);
    Tensor left = decomp_detail::scale_last_axis(decomp_detail::slice_last_axis(sv.u, g), w);
    Tensor right = decomp_detail::scale_first_axis(decomp_detail::slice_first_axis(sv.v, g), w)
                       .permute({1, 2, 0});
    for (int t = 0; t < nterms; ++t) {
      const int* tt = terms + 5 * t;
      std::size_t r0 = tt[1], c0 = tt[2], r1 = tt[3], c1 = tt[4];
      std::vector<InsertionPiece> pieces;
      if (tt[0] == 0) {
        pieces.push_back({Coord{r0, c0}, z, {}});
        r1 = r0;
        c1 = c0;
      } else {
        pieces.push_back({Coord{r0, c0}, left, {0}});
        pieces.push_back({Coord{r1, c1}, right, {0}});
      }
      std::size_t br0 = std::min(r0, r1), br1 = std::max(r0, r1);
      std::size_t bc0 = std::min(c0, c1), bc1 = std::max(c0, c1);
      const TwoLayerBoundary* top = br0 > 0 ? &cache.tops[br0 - 1] : nullptr;
      const TwoLayerBoundary* bot = br1 + 1 < n ? &cache.bots[br1 + 1] : nullptr;
      BandEnvironment* env = nullptr;
      for (auto& e : envs)
        if (e.first == std::make_pair(br0, br1)) env = &e.second;
      if (!env) {
        envs.emplace_back(std::make_pair(br0, br1), band_environment(top, s, s, br0, br1, bot));
        env = &envs.back().second;
      }
      cplx v = band_splice(*env, top, s, s, bot, pieces, bc0, bc1) / norm;
      b.doubles.push_back(v.real());
      b.doubles.push_back(v.imag());
    }
    double t2 = now_s();
    b.doubles.push_back(t1 - t0);
    b.doubles.push_back(t2 - t1);
  });
}

// Reference `expectation` (observables.cpp:335-422) of the TFIM Hamiltonian in
// colour order.  doubles: [value, norm_sq, raw_re, raw_im]
Bag* ref_tfim_energy(int rows, int cols, int d, const int* ndims, const int64_t* shapes,
                     const double* const* datas, double J, double h, int64_t m, uint64_t seed,
                     int power_iters, int oversample, int shared_env) {
  return guarded([&](Bag& b) {
    PepsState s = make_state(rows, cols, d, ndims, shapes, datas);
    ExpectationOptions eo;
    eo.contract = make_opt(m, seed, power_iters, oversample, 1);
    eo.use_cache = true;
    eo.shared_environments = shared_env != 0;
    ExpectationResult r = expectation(s, tfim_colour_order(rows, cols, J, h), eo);
    b.doubles = {r.value, r.norm_sq, r.raw_sum.real(), r.raw_sum.imag()};
  });
}

// One QR-reduced simple update (state.cpp:161-204) with an explicit gate.
Bag* ref_apply_two_site(int rows, int cols, int d, const int* ndims, const int64_t* shapes,
                        const double* const* datas, const double* gate, int ar, int ac, int br,
                        int bc, uint64_t max_rank, int strategy) {
  return guarded([&](Bag& b) {
    PepsState s = make_state(rows, cols, d, ndims, shapes, datas);
    int64_t gs[4] = {d, d, d, d};
    UpdateOption uo;
    uo.policy = TruncationPolicy{static_cast<std::size_t>(max_rank), 1e-14};
    uo.strategy = strategy == 0 ? UpdateStrategy::direct
                                : (strategy == 1 ? UpdateStrategy::qr_svd : UpdateStrategy::qr_svd_gram);
    PepsState out = apply_two_site(s, make_tensor(4, gs, gate), Coord{(std::size_t)ar, (std::size_t)ac},
                                   Coord{(std::size_t)br, (std::size_t)bc}, uo);
    for (const auto& t : out.sites()) b.tensors.push_back(t);
  });
}

// hermitian_function(coeff*op, exp(-tau x)) — the ITE gate rule (drivers.cpp:56-71).
Bag* ref_exp_gate(int n, const double* op, double coeff, double tau) {
  return guarded([&](Bag& b) {
    int64_t sh[2] = {n, n};
    Tensor h = make_tensor(2, sh, op) * cplx(coeff, 0.0);
    b.tensors.push_back(hermitian_function(h, [tau](double x) { return std::exp(-tau * x); }));
  });
}

// TFIM ITE: start from the given state, apply `steps`
// Trotter steps of all terms in colour order with UpdateOption{{r,1e-14},
// qr_svd_gram}.  Returns the final sites; doubles: [seconds].
Bag* ref_ite_tfim(int rows, int cols, int d, const int* ndims, const int64_t* shapes,
                  const double* const* datas, double J, double h, double tau, int steps,
                  uint64_t rank) {
  return guarded([&](Bag& b) {
    PepsState s = make_state(rows, cols, d, ndims, shapes, datas);
    Observable obs = tfim_colour_order(rows, cols, J, h);
    UpdateOption uo;
    uo.policy = TruncationPolicy{static_cast<std::size_t>(rank), 1e-14};
    uo.strategy = UpdateStrategy::qr_svd_gram;
    double t0 = now_s();
    for (int st = 0; st < steps; ++st)
      for (const auto& term : obs.terms()) s = ite_term(s, term, tau, uo);
    double dt = now_s() - t0;
    for (const auto& t : s.sites()) b.tensors.push_back(t);
    b.doubles = {dt};
  });
}

// run_ite (drivers.cpp:75-98) with the TFIM Hamiltonian in colour order:
// energies (step, value) in doubles, final state in tensors.
Bag* ref_run_ite(int rows, int cols, double J, double h, double tau, int steps, uint64_t evolution_rank,
                 uint64_t contraction_rank, int rsvd_iters, int energy_every, int neel, uint64_t seed) {
  return guarded([&](Bag& b) {
    IteConfig cfg;
    cfg.rows = rows;
    cfg.cols = cols;
    cfg.hamiltonian = tfim_colour_order(rows, cols, J, h);
    cfg.tau = tau;
    cfg.steps = static_cast<std::size_t>(steps);
    cfg.evolution_rank = static_cast<std::size_t>(evolution_rank);
    cfg.contraction_rank = static_cast<std::size_t>(contraction_rank);
    cfg.family = ContractFamily::two_layer_ibmps;
    cfg.rsvd_iters = rsvd_iters;
    cfg.energy_every = static_cast<std::size_t>(energy_every);
    cfg.initial = neel ? "neel" : "zeros";
    cfg.seed = seed;
    IteOutcome out = run_ite(cfg);
    for (auto [st, e] : out.energies) {
      b.doubles.push_back(static_cast<double>(st));
      b.doubles.push_back(e);
    }
    for (const auto& t : out.state.sites()) b.tensors.push_back(t);
  });
}

// vqe_ansatz_state (drivers.cpp:100-131) and its energy under the TFIM in
// colour order (state_energy, drivers.cpp:46-53, seed derive_seed(seed, 0xF)
// as run_vqe's objective): sites, then [energy].
Bag* ref_vqe_ansatz(int rows, int cols, int layers, const double* theta, uint64_t evolution_rank, double J, double h,
                    uint64_t contraction_rank, int rsvd_iters, uint64_t seed) {
  return guarded([&](Bag& b) {
    VqeConfig cfg;
    cfg.rows = rows;
    cfg.cols = cols;
    cfg.layers = static_cast<std::size_t>(layers);
    cfg.evolution_rank = static_cast<std::size_t>(evolution_rank);
    std::vector<double> th(theta, theta + static_cast<std::size_t>(layers) * rows * cols);
    PepsState st = vqe_ansatz_state(cfg, th);
    for (const auto& t : st.sites()) b.tensors.push_back(t);
    // state_energy / energy_contract_option are file-local in drivers.cpp:
    // the same options through the public expectation()
    ExpectationOptions eo;
    eo.contract.family = ContractFamily::two_layer_ibmps;
    eo.contract.trunc.max_rank = static_cast<std::size_t>(contraction_rank);
    eo.contract.strategy = SvdStrategy::implicit_rsvd;
    eo.contract.rsvd.power_iters = rsvd_iters;
    eo.contract.seed = derive_seed(seed, 0xF);
    eo.use_cache = true;
    eo.shared_environments = true;
    b.doubles.push_back(expectation(st, tfim_colour_order(rows, cols, J, h), eo).value);
  });
}

// apply_distant (state.cpp:206-236): SWAP-routed two-site gate.
Bag* ref_apply_distant(int rows, int cols, int d, const int* ndims, const int64_t* shapes,
                       const double* const* datas, const double* gate, int ar, int ac, int br, int bc,
                       uint64_t max_rank) {
  return guarded([&](Bag& b) {
    PepsState s = make_state(rows, cols, d, ndims, shapes, datas);
    int64_t gs[4] = {d, d, d, d};
    UpdateOption uo;
    uo.policy = TruncationPolicy{static_cast<std::size_t>(max_rank), 1e-14};
    uo.strategy = UpdateStrategy::qr_svd_gram;
    PepsState out = apply_distant(s, make_tensor(4, gs, gate), Coord{(std::size_t)ar, (std::size_t)ac},
                                  Coord{(std::size_t)br, (std::size_t)bc}, uo);
    for (const auto& t : out.sites()) b.tensors.push_back(t);
  });
}

// expectation_trotter (observables.cpp:424-454) of the colour-ordered TFIM.
Bag* ref_expectation_trotter(int rows, int cols, int d, const int* ndims, const int64_t* shapes,
                             const double* const* datas, double J, double h, double tau, int64_t m, uint64_t seed,
                             int power_iters, int oversample, uint64_t growth_cap) {
  return guarded([&](Bag& b) {
    PepsState s = make_state(rows, cols, d, ndims, shapes, datas);
    ExpectationOptions eo;
    eo.contract = make_opt(m, seed, power_iters, oversample, 1);
    UpdateOption growth;
    growth.policy = TruncationPolicy{static_cast<std::size_t>(growth_cap), 1e-14};
    b.doubles = {expectation_trotter(s, tfim_colour_order(rows, cols, J, h), tau, eo, growth)};
  });
}

// |+> on every site: computational_basis zeros then H (state.cpp:44-58,75-85).
Bag* ref_plus_state(int rows, int cols) {
  return guarded([&](Bag& b) {
    std::vector<int> bits(rows * cols, 0);
    PepsState s = PepsState::computational_basis(rows, cols, bits);
    for (int r = 0; r < rows; ++r)
      for (int c = 0; c < cols; ++c) s = apply_one_site(s, gates::H(), Coord{(std::size_t)r, (std::size_t)c});
    for (const auto& t : s.sites()) b.tensors.push_back(t);
  });
}

Bag* ref_chain_scalar(int n, const int* ndims, const int64_t* shapes, const double* const* datas) {
  return guarded([&](Bag& b) {
    Mps mps;
    mps.sites = make_list(n, ndims, shapes, datas);
    cplx v = chain_scalar(mps);
    b.doubles = {v.real(), v.imag()};
  });
}

}  // extern "C"
