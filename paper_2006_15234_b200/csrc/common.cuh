// Shared device/host helpers for the B200 einsumsvd library.
//
// Complex numbers are interleaved (re, im) float64 pairs stored as double2 —
// bit-compatible with std::complex<double>, the reference's element type
// (proj/include/peps/tensor.hpp:13).  All tensors are row-major, last index
// fastest (tensor.hpp:16-19).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>

namespace pepsb {

// Error family mirroring the reference (proj/include/peps/errors.hpp:10-34).
enum ErrKind : int {
  kOk = 0,
  kShapeError = 1,
  kValidationError = 2,
  kResourceError = 3,
  kNumericalError = 4,
  kConfigError = 5,
  kCudaError = 6,
  kOtherError = 9,
};

struct Error : std::runtime_error {
  Error(int k, const std::string& m) : std::runtime_error(m), kind(k) {}
  int kind;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    throw Error(kCudaError, std::string(what) + ": " + cudaGetErrorString(e) + " at " + file + ":" +
                                std::to_string(line));
  }
}
#define PEPSB_CUDA(x) ::pepsb::cuda_check((x), #x, __FILE__, __LINE__)
// Debug aid: PEPSB_SYNC_DEBUG=1 synchronises after every launch so a faulting
// kernel is reported at its own launch site (file:line) instead of at a later sync.
inline bool sync_debug() {
  static const bool on = [] {
    const char* e = std::getenv("PEPSB_SYNC_DEBUG");
    return e && e[0] == '1';
  }();
  return on;
}
inline void launch_check(const char* file, int line) {
  cuda_check(cudaGetLastError(), "kernel launch", file, line);
  if (sync_debug()) cuda_check(cudaDeviceSynchronize(), "kernel execution (PEPSB_SYNC_DEBUG)", file, line);
}
#define PEPSB_LAUNCH() ::pepsb::launch_check(__FILE__, __LINE__)

// ------------------------------------------------------------------ complex helpers
__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
__host__ __device__ __forceinline__ double2 cscale(double2 a, double s) {
  return make_double2(a.x * s, a.y * s);
}
__host__ __device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__host__ __device__ __forceinline__ double cnorm2(double2 a) { return a.x * a.x + a.y * a.y; }

// SplitMix64 finalizer and derive_seed (proj/include/peps/rng.hpp:17-44).
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
__host__ __device__ __forceinline__ uint64_t splitmix_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline uint64_t derive_seed1(uint64_t base, uint64_t part) {
  return splitmix_mix((base ^ (part + kGamma)) + kGamma);
}

constexpr int kMaxModes = 12;  // maximum tensor order handled by generic kernels

}  // namespace pepsb
