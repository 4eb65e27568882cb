// Reference-side declarations of the B200 drop-ins (see gpu_backend.cpp).
// With PEPS_WITH_B200 defined, the reference's own einsumsvd /
// contract_two_layer forward here (a two-line #ifdef at the top of each
// definition), so every caller -- two_layer_apply_row,
// sweep_boundaries, expectation, approx_apply_mpo, apply_two_site -- takes
// the device path unchanged.
#pragma once

#include <memory>

#include "peps/contraction.hpp"
#include "peps/decomposition.hpp"
#include "peps/implicit.hpp"
#include "peps/state.hpp"

namespace peps::b200 {

EinsumsvdResult einsumsvd(const ImplicitOperator& net, const TruncationPolicy& policy, SvdStrategy strategy,
                          Absorb absorb = Absorb::split, const RsvdConfig& cfg = {});

cplx contract_two_layer(const PepsState& bra, const PepsState& ket, const ContractOption& opt);

}  // namespace peps::b200
