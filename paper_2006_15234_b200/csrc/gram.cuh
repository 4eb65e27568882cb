// Hermitian Gram matrix G = Z^H Z of a tall contiguous complex matrix on the
// FP64 tensor pipe (gram.cu): upper-triangle DMMA blocks of the real symmetric
// product of the interleaved view, split over rows, deterministic reduction.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace pepsb {

constexpr int64_t kGramMaxK = 72;
constexpr int64_t kGramMinRows = 2048;  // below: the generic GEMM path (few tiles, no split benefit)

bool gram_herk_eligible(int64_t rows, int64_t k);
// option "gemm_gram" / PEPSB_GEMM_GRAM (default off: measured slower in the row)
bool gram_enabled();
void gram_set_enabled(int on);
// Workspace in doubles for gram_herk.
int64_t gram_herk_workspace(int64_t rows, int64_t k, int num_sms);
// G (k x k, row-major complex) = Z^H Z for Z rows x k row-major complex.
void gram_herk(const double2* Z, int64_t rows, int k, double2* G, double* work, int num_sms, cudaStream_t stream);

}  // namespace pepsb
