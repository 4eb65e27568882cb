// Memory-bound tensor kernels: strided gather/sum (permute, diagonal, label
// sums — the reference's reduce_single + Tensor::permute, proj/src/einsum.cpp:82-169,
// proj/src/tensor.cpp:99-134), the SplitMix64 sketch generator
// (proj/src/tensor.cpp:192-208) written directly in any physical layout, and
// small elementwise helpers.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace pepsb {

struct GatherParams {
  int nout = 0;                      // output modes (row-major, contiguous output)
  int64_t oext[kMaxModes] = {};
  int64_t ostr[kMaxModes] = {};      // source stride per output mode
  int nsum = 0;                      // summed modes
  int64_t sext[kMaxModes] = {};
  int64_t sstr[kMaxModes] = {};
  int conj = 0;
  double scale = 1.0;
};
// dst[o] = scale * sum_s op(src[off(o) + off(s)]), op = conj if requested.
void gather_sum(double2* dst, const double2* src, const GatherParams& p, cudaStream_t st);

// Sketch generator: element at physical position p has logical (reference)
// linear index j = sum_a idx_a(p) * lstr[a]; complex: re = sym(mix(seed+(2j+1)g)),
// im = sym(mix(seed+(2j+2)g)); real: re = sym(mix(seed+(j+1)g)), im = 0.
// `base` offsets the logical index (a slice of a larger random tensor).
void random_fill(double2* dst, int nd, const int64_t* pext, const int64_t* lstr, uint64_t seed,
                 int real, cudaStream_t st, uint64_t base = 0);

// t[i] *= w[(i / inner) % ext]  (scale one axis by real weights held on device)
void scale_axis(double2* t, int64_t total, int64_t inner, int64_t ext, const double* w,
                cudaStream_t st);

// Row-slice + scale: dst[r][c] = src[r * lds + c] * (w ? w[c] : 1), r < rows, c < cols.
void slice_scale_cols(double2* dst, const double2* src, int64_t rows, int64_t cols, int64_t lds,
                      const double* w, int conj, cudaStream_t st);

// *flag = 1 if any element has a nonzero imaginary part, else 0.
void imag_nonzero(const double2* x, int64_t n, int* flag, cudaStream_t st);
void fill_zero(double2* dst, int64_t n, cudaStream_t st);

}  // namespace pepsb
