#include <algorithm>

#include "tensor_ops.cuh"

namespace pepsb {

namespace {

constexpr int kT = 256;

inline unsigned grid_for(int64_t n) {
  int64_t b = (n + kT - 1) / kT;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(b, 148LL * 32)));
}

__global__ void gather_sum_kernel(double2* dst, const double2* src, const GatherParams p, int64_t total,
                                  int64_t nsum_total) {
  for (int64_t o = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t idx = o, off = 0;
    for (int a = p.nout - 1; a >= 0; --a) {
      int64_t q = idx / p.oext[a];
      off += (idx - q * p.oext[a]) * p.ostr[a];
      idx = q;
    }
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t s = 0; s < nsum_total; ++s) {
      int64_t si = s, soff = 0;
      for (int a = p.nsum - 1; a >= 0; --a) {
        int64_t q = si / p.sext[a];
        soff += (si - q * p.sext[a]) * p.sstr[a];
        si = q;
      }
      acc = cadd(acc, src[off + soff]);
    }
    if (p.conj) acc.y = -acc.y;
    dst[o] = cscale(acc, p.scale);
  }
}

__device__ __forceinline__ double sym_unit(uint64_t x) {
  return 2.0 * (static_cast<double>(x >> 11) * 0x1.0p-53) - 1.0;
}

struct RandParams {
  int nd;
  uint64_t base;  // logical index of the first element (slices of a larger tensor)
  int64_t pext[kMaxModes];
  int64_t lstr[kMaxModes];
};

__global__ void random_kernel(double2* dst, const RandParams p, int64_t total, uint64_t seed, int real) {
  for (int64_t o = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t idx = o;
    uint64_t j = p.base;
    for (int a = p.nd - 1; a >= 0; --a) {
      int64_t q = idx / p.pext[a];
      j += static_cast<uint64_t>(idx - q * p.pext[a]) * static_cast<uint64_t>(p.lstr[a]);
      idx = q;
    }
    double2 v;
    if (real) {
      v = make_double2(sym_unit(splitmix_mix(seed + (j + 1) * kGamma)), 0.0);
    } else {
      v = make_double2(sym_unit(splitmix_mix(seed + (2 * j + 1) * kGamma)),
                       sym_unit(splitmix_mix(seed + (2 * j + 2) * kGamma)));
    }
    dst[o] = v;
  }
}

__global__ void scale_axis_kernel(double2* t, int64_t total, int64_t inner, int64_t ext, const double* w) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    t[i] = cscale(t[i], w[(i / inner) % ext]);
}

__global__ void slice_scale_kernel(double2* dst, const double2* src, int64_t rows, int64_t cols, int64_t lds,
                                   const double* w, int conj) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    double2 v = src[r * lds + c];
    if (conj) v.y = -v.y;
    dst[i] = w ? cscale(v, w[c]) : v;
  }
}

__global__ void imag_nonzero_kernel(const double2* x, int64_t n, int* flag) {
  int any = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    any |= x[i].y != 0.0;
  if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

__global__ void fill_zero_kernel(double2* dst, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = make_double2(0.0, 0.0);
}

}  // namespace

void gather_sum(double2* dst, const double2* src, const GatherParams& p, cudaStream_t st) {
  int64_t total = 1, ns = 1;
  for (int a = 0; a < p.nout; ++a) total *= p.oext[a];
  for (int a = 0; a < p.nsum; ++a) ns *= p.sext[a];
  if (total == 0) return;
  gather_sum_kernel<<<grid_for(total), kT, 0, st>>>(dst, src, p, total, ns);
  PEPSB_LAUNCH();
}

void random_fill(double2* dst, int nd, const int64_t* pext, const int64_t* lstr, uint64_t seed, int real,
                 cudaStream_t st, uint64_t base) {
  RandParams p{};
  p.nd = nd;
  p.base = base;
  int64_t total = 1;
  for (int a = 0; a < nd; ++a) {
    p.pext[a] = pext[a];
    p.lstr[a] = lstr[a];
    total *= pext[a];
  }
  random_kernel<<<grid_for(total), kT, 0, st>>>(dst, p, total, seed, real);
  PEPSB_LAUNCH();
}

void scale_axis(double2* t, int64_t total, int64_t inner, int64_t ext, const double* w, cudaStream_t st) {
  if (total == 0) return;
  scale_axis_kernel<<<grid_for(total), kT, 0, st>>>(t, total, inner, ext, w);
  PEPSB_LAUNCH();
}

void slice_scale_cols(double2* dst, const double2* src, int64_t rows, int64_t cols, int64_t lds,
                      const double* w, int conj, cudaStream_t st) {
  if (rows * cols == 0) return;
  slice_scale_kernel<<<grid_for(rows * cols), kT, 0, st>>>(dst, src, rows, cols, lds, w, conj);
  PEPSB_LAUNCH();
}

void imag_nonzero(const double2* x, int64_t n, int* flag, cudaStream_t st) {
  PEPSB_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
  if (n == 0) return;
  imag_nonzero_kernel<<<grid_for(n), kT, 0, st>>>(x, n, flag);
  PEPSB_LAUNCH();
}

void fill_zero(double2* dst, int64_t n, cudaStream_t st) {
  if (n == 0) return;
  fill_zero_kernel<<<grid_for(n), kT, 0, st>>>(dst, n);
  PEPSB_LAUNCH();
}

}  // namespace pepsb
