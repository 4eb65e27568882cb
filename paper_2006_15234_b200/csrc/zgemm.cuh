// Complex-FP64 GEMM on the B200 FP64 tensor cores (DMMA.8x8x4).
//
// One pairwise contraction of the implicit-operator chain lowers to
//   C[b][i][j] = sum_k opA(b,i,k) * opB(b,k,j)
// (the role of cblas_zgemm in the reference, proj/src/einsum.cpp:41-57,224-227),
// with two differences that remove the reference's operand permutes
// (einsum.cpp:203-204, tensor.cpp:99-134):
//   * operands are addressed through (i,k)/(k,j) strides, either index may be
//     the contiguous one, conjugation is applied on load;
//   * the epilogue scatters C through separable mixed-radix row/column offsets,
//     so the result is written directly in whatever label order the NEXT
//     contraction wants.
// Complex products use the real embedding  [Re C | Im C] = [Ar | Ai] x
// [[Br, Bi], [-Bi, Br]], so the interleaved complex buffer of A is already the
// real A' operand and each B value expands to a 2x2 real block in registers.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace pepsb {

struct ZgemmParams {
  const double2* A = nullptr;
  const double2* B = nullptr;
  double2* C = nullptr;
  double2* work = nullptr;  // split-K partials [splits][batch][M][N]
  int64_t M = 0, N = 0, K = 0;
  int64_t sAi = 0, sAk = 0, sBk = 0, sBj = 0;  // complex-element strides
  int conjA = 0, conjB = 0;
  // batch modes (row-major decode of the batch index)
  int nb = 0;
  int64_t bext[4] = {}, bsA[4] = {}, bsB[4] = {}, bsC[4] = {};
  int64_t batch = 1;
  // epilogue scatter: row index i decoded over rext (last fastest) -> sum rstr
  int nr = 0;
  int64_t rext[kMaxModes] = {}, rstr[kMaxModes] = {};
  int nc = 0;
  int64_t cext[kMaxModes] = {}, cstr[kMaxModes] = {};
  int splits = 1;
  int64_t kchunk = 0;
  int accumulate = 0;  // C += result instead of C = result
  int cfg = 0;         // tile configuration (set by zgemm_plan_splits)
  int algo = 0;        // kGemm4M / kGemm3M (set by zgemm_plan_splits)
  int ws = 0;          // persistent warp-specialised kernel (zgemm_ws.cu)
  int realA = 0, realB = 0;  // operand with exactly zero imaginary parts (Buf::real)
  int num_sms = 148;   // grid of the persistent kernel
};

// Complex product scheme (process-wide): kGemm4M = real embedding, 4 real MACs
// per complex MAC (the zgemm arithmetic); kGemm3M = Gauss / zgemm3m, 3 real MACs
// per complex MAC (Im C = (Ar+Ai)(Br+Bi) - ArBr - AiBi).  Default 3M;
// PEPSB_GEMM=4m or option "gemm_algo" = 0 selects 4M.
// kGemmCR: A real (imaginary parts exactly zero), C = A B as the real GEMM
// A (M x K) . B' (K x 2N) on B's interleaved (re, im) doubles -- 2 real MACs
// per complex MAC (set by zgemm_plan_splits when an operand is real).
// kGemmSmall: CUDA-core FMA kernel for problems below kSmallMaxMacs complex
// MACs with K <= kSmallMaxK (set by zgemm_plan_splits; option "gemm_small").
enum GemmAlgo { kGemm4M = 0, kGemm3M = 1, kGemm4C = 2, kGemmCR = 3, kGemmSmall = 4 };
constexpr int64_t kSmallMaxK = 128;
constexpr int64_t kSmallMaxMacs = int64_t{1} << 13;
// Tile-streaming kernels for short-K many-tile problems (opt-in:
// PEPSB_GEMM_STREAM=1 or option "gemm_stream" = 1; measured slower at config 2).
int zgemm_cr_cfg();
int zgemm_c3m_cfg();
void zgemm_set_c3m_cfg(int v);
void zgemm_set_cr_cfg(int v);
bool zgemm_stream_enabled();
void zgemm_set_stream(int on);
bool zgemm_small_enabled();
void zgemm_set_small(int on);
bool zgemm_is_small(const ZgemmParams& p);
int zgemm_algo();
// Real flops the DMMAs execute for a planned problem (8 per complex MAC, 6 for 3M).
inline double zgemm_exec_flops(const ZgemmParams& p) {
  return (p.algo == kGemm3M ? 6.0 : p.algo == kGemmCR ? 4.0 : 8.0) * static_cast<double>(p.batch) * p.M * p.N * p.K;
}
void zgemm_set_algo(int a);
// Complex x real kernel for operands with exactly zero imaginary parts
// (default on; PEPSB_GEMM_REAL=0 or option "gemm_real" = 0 disables it).
bool zgemm_real_enabled();
void zgemm_set_real(int on);
// Persistent kernel with TMA tensor-map operand staging (zgemm_ws.cu): opt-in
// (PEPSB_GEMM_WS=1 or option "gemm_ws" = 1); measured at config 2 it does not
// beat the classic cp.async kernels, so they stay the default.
// mode 0: classic cp.async kernels; 1: persistent TMA kernel; 2: one tile per
// CTA with TMA staging (2 CTAs / SM).
int zgemm_ws_mode();
bool zgemm_ws_enabled();
void zgemm_set_ws(int mode);
bool zgemm_ws_eligible(const ZgemmParams& p);
void zgemm_ws_tile(const ZgemmParams& p, int64_t& bm, int64_t& bn);
void zgemm_ws_launch(const ZgemmParams& p, int num_sms, cudaStream_t stream);

// Launches the GEMM (and the deterministic split-K reduction when needed).
// `work` is allocated by the caller when splits > 1 (see zgemm_workspace).
void zgemm_launch(ZgemmParams p, cudaStream_t stream);
// Chooses split-K for the problem; returns the workspace size in complex elements.
int64_t zgemm_plan_splits(ZgemmParams& p, int num_sms);

}  // namespace pepsb
