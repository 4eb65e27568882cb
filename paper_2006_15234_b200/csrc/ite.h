// Imaginary-time evolution by batched QR-reduced simple update (config 4).
//
// Mirrors proj/src/state.cpp:75-204 (apply_one_site, apply_two_site with
// UpdateStrategy::qr_svd_gram) and the driver loop of proj/src/drivers.cpp:56-98,
// but applies every bond of one colour (a set of disjoint bonds) in one batch:
// three kernel launches and one host sync per colour instead of ~10 LAPACK /
// BLAS calls per bond.  Bonds of a colour touch disjoint sites, so the batch
// equals the reference's serial order exactly.
#pragma once

#include <array>
#include <utility>
#include <vector>

#include "peps.h"

namespace pepsb {

// exp(-tau * coeff * op) of a Hermitian (n x n) op (hermitian_function, linalg.cpp:297-314)
DTensor hermitian_exp(Ctx& ctx, const DTensor& op, double coeff, double tau);

// apply_one_site (state.cpp:75-85) on every listed (row, col)
PepsStateD apply_one_site_batch(Ctx& ctx, const PepsStateD& s, const DTensor& gate,
                                const std::vector<std::pair<int, int>>& sites);

// apply_two_site (state.cpp:161-204, qr_svd_gram) on disjoint adjacent bonds
// {ar, ac, br, bc}; gate axes (out_a, out_b, in_a, in_b).
PepsStateD apply_two_site_batch(Ctx& ctx, const PepsStateD& s, const DTensor& gate,
                                const std::vector<std::array<int, 4>>& bonds, const Trunc& policy);

// Transverse-field Ising ITE, H = -J sum ZZ - h sum X, terms in colour order
// (fields; even / odd horizontal; even / odd vertical bonds), `steps` Trotter
// steps of exp(-tau H_j) with UpdateOption{{rank, 1e-14}, qr_svd_gram}.
PepsStateD ite_tfim(Ctx& ctx, const PepsStateD& s, double J, double h, double tau, int steps, uint64_t rank);

std::vector<std::vector<std::array<int, 4>>> tfim_bond_colours(int rows, int cols);

}  // namespace pepsb
