// TEST INFRASTRUCTURE: links the reference (oracle/_ref objects, unmodified
// sources) with the reference-side shim integration/gpu_backend.cpp and the
// product library, then runs the same calls through both:
//   peps::einsumsvd           vs peps::b200::einsumsvd          (two-layer network, r=3 m=6)
//   peps::contract_two_layer  vs peps::b200::contract_two_layer (4x4 r=2 PEPS, m=4)
// Prints one JSON line; exit 0 when sigma / t1 / t2 / the norm agree to 1e-9.
// Built by oracle/Makefile as oracle/_ref/shim_check; run by
// tests/test_gpu_integration.py on the GPU box.
#include <cmath>
#include <cstdio>
#include <exception>

#include "gpu_backend.hpp"
#include "peps/contraction.hpp"
#include "peps/decomposition.hpp"
#include "peps/rng.hpp"
#include "peps/tensor.hpp"

using namespace peps;

namespace {

double rel(const Tensor& a, const Tensor& b) {
  if (a.shape() != b.shape()) return 1e300;
  double num = 0.0, den = 0.0;
  for (size_t i = 0; i < a.data().size(); ++i) {
    num += std::norm(a.data()[i] - b.data()[i]);
    den += std::norm(b.data()[i]);
  }
  return std::sqrt(num / (den > 0 ? den : 1e-300));
}

PepsState random_state(size_t n, size_t r, uint64_t seed) {
  std::vector<Tensor> sites;
  for (size_t i = 0; i < n; ++i)
    for (size_t j = 0; j < n; ++j)
      sites.push_back(random_tensor_real({2, i ? r : 1, j ? r : 1, i + 1 < n ? r : 1, j + 1 < n ? r : 1},
                                         derive_seed(seed, i, j)));
  return PepsState(n, n, 2, std::move(sites));
}

}  // namespace

int main() {
  try {
    const size_t r = 3, m = 6;
    Tensor v = random_tensor({m, r, r, m, r, r}, 1), s = random_tensor({r, r, m, m}, 2);
    Tensor b = random_tensor({2, r, r, r, r}, 3);
    ImplicitOperator net({v, s, b.conj(), b}, {"apqsmn", "uvst", "dumbe", "dvncf"}, "apq", "bctef");
    const TruncationPolicy pol{m, 1e-14};
    const RsvdConfig cfg{2, -1, 11};
    EinsumsvdResult want = einsumsvd(net, pol, SvdStrategy::implicit_rsvd, Absorb::right, cfg);
    EinsumsvdResult got = b200::einsumsvd(net, pol, SvdStrategy::implicit_rsvd, Absorb::right, cfg);
    double s_err = want.s.size() == got.s.size() ? 0.0 : 1e300;
    for (size_t i = 0; i < want.s.size() && i < got.s.size(); ++i)
      s_err = std::max(s_err, std::abs(got.s[i] - want.s[i]) / want.s[0]);
    const double t1_err = rel(got.t1, want.t1), t2_err = rel(got.t2, want.t2);

    PepsState st = random_state(4, 2, 7);
    ContractOption opt = ContractOption::two_layer_opt(4, 5, 1);
    opt.rsvd.oversample = 4;
    const cplx nw = contract_two_layer(st, st, opt);
    const cplx ng = b200::contract_two_layer(st, st, opt);
    const double n_err = std::abs(ng - nw) / std::abs(nw);
    const bool ok = s_err < 1e-9 && t1_err < 1e-9 && t2_err < 1e-9 && n_err < 1e-9 &&
                    got.rank_clamped == want.rank_clamped;
    std::printf("{\"ok\": %s, \"rank\": %zu, \"sigma_err\": %.3e, \"t1_err\": %.3e, \"t2_err\": %.3e, "
                "\"norm_ref\": %.17g, \"norm_b200\": %.17g, \"norm_err\": %.3e}\n",
                ok ? "true" : "false", got.s.size(), s_err, t1_err, t2_err, nw.real(), ng.real(), n_err);
    return ok ? 0 : 1;
  } catch (const std::exception& e) {
    std::printf("{\"ok\": false, \"error\": \"%s\"}\n", e.what());
    return 2;
  }
}
