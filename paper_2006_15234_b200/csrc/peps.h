// Callers of the hot path on the device: two-layer boundary-MPS row absorbs,
// contract_two_layer, chain_scalar, cached environments, band zipper and the
// QR-reduced simple update (proj/include/peps/contraction.hpp,
// observables.hpp, state.hpp).
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "decomp.h"

namespace pepsb {

// state.hpp:33-61 — sites (phys, up, left, down, right), edge bonds 1.
struct PepsStateD {
  int rows = 0, cols = 0, d = 2;
  std::vector<DTensor> sites;  // row-major
  const DTensor& site(int r, int c) const { return sites[static_cast<size_t>(r) * cols + c]; }
  DTensor& site(int r, int c) { return sites[static_cast<size_t>(r) * cols + c]; }
  void validate() const;  // state.cpp:22-42
};

// contraction.hpp:77-80 — MPS sites (pb*pk, left, right) + phys pairs.
struct BoundaryD {
  std::vector<DTensor> sites;
  std::vector<std::pair<int64_t, int64_t>> phys;
  void validate() const;  // mps.cpp:20-32
};

// contraction.hpp:18-32 (two-layer family fields).
struct ContractOptD {
  Trunc trunc{0, 1e-14};
  int strategy = kImplicitRsvd;
  Rsvd rsvd;
  bool canonicalize = true;
  uint64_t seed = 0;
};

constexpr uint64_t kTagTop = 0x20;     // observables.cpp:17
constexpr uint64_t kTagBottom = 0x21;  // observables.cpp:18

BoundaryD two_layer_first_row(Ctx& ctx, const PepsStateD& bra, const PepsStateD& ket);
BoundaryD two_layer_apply_row(Ctx& ctx, const BoundaryD& top, const PepsStateD& bra, const PepsStateD& ket,
                              int row, const ContractOptD& opt, uint64_t seed_tag);
// <bra|ket> by two-layer IBMPS (contraction.cpp:313-338).
std::pair<double, double> contract_two_layer(Ctx& ctx, const PepsStateD& bra, const PepsStateD& ket,
                                             const ContractOptD& opt);
// mps.cpp:102-110
std::pair<double, double> chain_scalar(Ctx& ctx, const BoundaryD& b);

// observables.cpp:56-59,261-333
struct RowCacheD {
  std::vector<BoundaryD> tops, bots;
};
PepsStateD flip_vertical(Ctx& ctx, const PepsStateD& s);
RowCacheD build_row_cache(Ctx& ctx, const PepsStateD& s, const ContractOptD& opt);

// contraction.hpp:95-125 (band zipper)
struct InsertionPieceD {
  int row = 0, col = 0;
  DTensor op;                 // (d_out, d_in, bond...)
  std::vector<int> bond_ids;
};
struct BandEnvD {
  std::vector<LTensor> left, right;
  int r0 = 0, r1 = 0;
};
std::pair<double, double> band_value(Ctx& ctx, const BoundaryD* top, const PepsStateD& bra, const PepsStateD& ket,
                                     int r0, int r1, const BoundaryD* bottom,
                                     const std::vector<InsertionPieceD>& pieces);
BandEnvD band_environment(Ctx& ctx, const BoundaryD* top, const PepsStateD& bra, const PepsStateD& ket, int r0,
                          int r1, const BoundaryD* bottom);
std::pair<double, double> band_splice(Ctx& ctx, const BandEnvD& env, const BoundaryD* top, const PepsStateD& bra,
                                      const PepsStateD& ket, const BoundaryD* bottom,
                                      const std::vector<InsertionPieceD>& pieces, int c0, int c1);

// ---- one-layer boundary MPS (mps.hpp / contraction.hpp:47-75)
struct MpsD {  // sites (phys, left, right)
  std::vector<DTensor> sites;
};
struct MpoD {  // sites (p = input phys, d = output phys, left, right)
  std::vector<DTensor> sites;
};
struct ApplyOptD {  // mps.hpp ApplyOption
  Trunc policy{0, 1e-14};
  int strategy = kImplicitRsvd;
  int absorb = kSplit;
  Rsvd rsvd;
  uint64_t seed_base = 0;
};
// mps.cpp:44-84 (zip-up: einsumsvd of {v(adso), s(pst), o(peoq)} rows "ad" cols "etq")
MpsD approx_apply_mpo(Ctx& ctx, const MpsD& s, const MpoD& o, const ApplyOptD& opt);
// mps.cpp:86-100
MpsD exact_apply_mpo(Ctx& ctx, const MpsD& s, const MpoD& o);
// mps.cpp:121-128
std::pair<double, double> mps_glue(Ctx& ctx, const MpsD& top, const MpsD& bottom);
// contraction.cpp:77-99: order-4 grid (up, left, down, right), edge bonds 1
struct GridD {
  int rows = 0, cols = 0;
  std::vector<DTensor> sites;
  const DTensor& site(int r, int c) const { return sites[static_cast<size_t>(r) * cols + c]; }
  void validate() const;
};
enum Family { kFamilyExact = 0, kFamilyBmps = 1, kFamilyIbmps = 2 };
// contraction.cpp:178-252: contract_exact (untruncated absorption from both ends
// + zipper, ResourceError above the element budget) or contract_boundary
// (approx_apply_mpo per row, seeds derive_seed(seed, 0x10, r), absorb by row
// parity) for the BMPS / IBMPS families.
std::pair<double, double> contract_one_layer(Ctx& ctx, const GridD& g, int family, const ContractOptD& opt,
                                             uint64_t memory_budget);

// observables.hpp:16-20,63-85 and observables.cpp:284-422: local terms
// (1- or 2-site operators, outputs first), options and result of expectation.
struct LocalTermD {
  double coeff_re = 1.0, coeff_im = 0.0;
  std::vector<std::pair<int, int>> sites;  // 1 or 2 (row, col)
  DTensor op;                              // (d, d) or (d, d, d, d)
};
struct ExpectOptD {
  ContractOptD contract;
  bool use_cache = true;
  bool shared_environments = false;
  bool allow_complex = false;
};
struct ExpectResultD {
  double value = 0.0, norm_sq = 0.0;
  double raw_re = 0.0, raw_im = 0.0, cx_re = 0.0, cx_im = 0.0;
  uint64_t full_sweeps = 0, band_contractions = 0, flops = 0;
};
ExpectResultD expectation(Ctx& ctx, const PepsStateD& s, const std::vector<LocalTermD>& terms,
                          const ExpectOptD& opt);

}  // namespace pepsb
