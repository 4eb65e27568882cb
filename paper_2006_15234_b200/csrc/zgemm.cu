// Complex-FP64 DMMA GEMM (see zgemm.cuh for the contract).
//
// CTA tile BM x BN (complex), K step BK, STAGES-deep cp.async pipeline
// (LDGSTS.128: one complex element per copy), warps tiled WM x WN, each warp
// issuing (WM/8) x (WN/4) DMMA.8x8x4 per two complex k.  Fragment layouts of
// mma.m8n8k4.f64: A a0 = A[lane>>2][lane&3], B b0 = B[lane&3][lane>>2],
// C {c0,c1} = C[lane>>2][2*(lane&3) + {0,1}].  With the real embedding an
// 8x8 real C tile is an 8x4 complex tile and each lane owns exactly one
// complex output (re = c0, im = c1).
#include <algorithm>
#include <atomic>
#include <string>
#include <cstdio>
#include <cstdlib>

#include "zgemm.cuh"

namespace pepsb {

namespace {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int BM, int BN, int BK, bool AK, bool BNC>
struct Smem {
  static constexpr int LDA = AK ? (BK + 2) : BM;   // complex elements per smem row
  static constexpr int LDB = BNC ? (BN + 4) : (BK + 2);
  static constexpr int A_ELEMS = AK ? BM * LDA : BK * LDA;
  static constexpr int B_ELEMS = BNC ? BK * LDB : BN * LDB;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
};

__device__ __forceinline__ int64_t decode_offset(int64_t idx, int n, const int64_t* ext,
                                                 const int64_t* str) {
  int64_t off = 0;
  for (int a = n - 1; a >= 0; --a) {
    int64_t e = ext[a];
    int64_t q = idx / e;
    off += (idx - q * e) * str[a];
    idx = q;
  }
  return off;
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AK, bool BNC>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32)
    zgemm_dmma_kernel(const ZgemmParams p) {
  using S = Smem<BM, BN, BK, AK, BNC>;
  constexpr int NWARP = (BM / WM) * (BN / WN);
  constexpr int NT = NWARP * 32;
  constexpr int FM = WM / 8;   // 8-row fragments per warp
  constexpr int FN = WN / 4;   // 4-complex-column fragments per warp
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* smem = reinterpret_cast<double2*>(smem_raw);
  int64_t* rowoff = reinterpret_cast<int64_t*>(smem + STAGES * S::STAGE);
  int64_t* coloff = rowoff + BM;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wm0 = (warp % (BM / WM)) * WM;
  const int wn0 = (warp / (BM / WM)) * WN;

  const int64_t mtiles = (p.M + BM - 1) / BM;
  const int64_t tile = blockIdx.x;
  const int64_t m0 = (tile % mtiles) * BM;
  const int64_t n0 = (tile / mtiles) * BN;
  const int64_t bz = blockIdx.y / p.splits;
  const int split = blockIdx.y % p.splits;

  // batch offsets
  int64_t offA = 0, offB = 0, offC = 0;
  {
    int64_t idx = bz;
    for (int a = p.nb - 1; a >= 0; --a) {
      int64_t e = p.bext[a];
      int64_t q = idx / e;
      int64_t r = idx - q * e;
      offA += r * p.bsA[a];
      offB += r * p.bsB[a];
      offC += r * p.bsC[a];
      idx = q;
    }
  }
  const double2* A = p.A + offA;
  const double2* B = p.B + offB;

  const int64_t kbeg = static_cast<int64_t>(split) * p.kchunk;
  const int64_t kend = min(p.K, kbeg + p.kchunk);
  const int64_t nk = (kend - kbeg + BK - 1) / BK;

  auto load_stage = [&](int slot, int64_t kt) {
    double2* As = smem + slot * S::STAGE;
    double2* Bs = As + S::A_ELEMS;
    const int64_t k0 = kbeg + kt * BK;
    // A tile: BM x BK
#pragma unroll
    for (int e = tid; e < BM * BK; e += NT) {
      int i, k;
      if (AK) { i = e / BK; k = e % BK; } else { k = e / BM; i = e % BM; }
      const int64_t gi = m0 + i, gk = k0 + k;
      const bool ok = gi < p.M && gk < kend;
      const double2* src = ok ? A + gi * p.sAi + gk * p.sAk : A;
      double2* dst = AK ? As + i * S::LDA + k : As + k * S::LDA + i;
      cp_async16(dst, src, ok);
    }
    // B tile: BK x BN
#pragma unroll
    for (int e = tid; e < BK * BN; e += NT) {
      int k, j;
      if (BNC) { k = e / BN; j = e % BN; } else { j = e / BK; k = e % BK; }
      const int64_t gj = n0 + j, gk = k0 + k;
      const bool ok = gj < p.N && gk < kend;
      const double2* src = ok ? B + gk * p.sBk + gj * p.sBj : B;
      double2* dst = BNC ? Bs + k * S::LDB + j : Bs + j * S::LDB + k;
      cp_async16(dst, src, ok);
    }
  };

  // Epilogue scatter offsets for this tile.
  if (p.splits == 1) {
    for (int r = tid; r < BM; r += NT) {
      const int64_t gi = m0 + r;
      rowoff[r] = gi < p.M ? decode_offset(gi, p.nr, p.rext, p.rstr) : 0;
    }
    for (int c = tid; c < BN; c += NT) {
      const int64_t gj = n0 + c;
      coloff[c] = gj < p.N ? decode_offset(gj, p.nc, p.cext, p.cstr) : 0;
    }
  }

  double acc[FM][FN][2];
#pragma unroll
  for (int a = 0; a < FM; ++a)
#pragma unroll
    for (int b = 0; b < FN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_async_commit();
  }

  const int kk = lane & 3;        // k slot within the 4-wide real k step
  const int a_row = lane >> 2;    // A fragment row
  const int b_s = kk & 1;         // real-embedding row parity of B'
  const int b_nn = lane >> 2;     // B' column (0..7)
  const int b_t = b_nn & 1;
  const int b_part = b_s ^ b_t;   // 0: Re(b), 1: Im(b)
  const bool b_neg = b_part && (b_s ^ p.conjB);
  const bool a_neg = (kk & 1) && p.conjA;

  for (int64_t kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int64_t pf = kt + STAGES - 1;
      if (pf < nk) load_stage(static_cast<int>(pf % STAGES), pf);
      cp_async_commit();
    }
    const int slot = static_cast<int>(kt % STAGES);
    const double* As = reinterpret_cast<const double*>(smem + slot * S::STAGE);
    const double* Bs = reinterpret_cast<const double*>(smem + slot * S::STAGE + S::A_ELEMS);
#pragma unroll
    for (int ks = 0; ks < BK / 2; ++ks) {
      const int kc = ks * 2 + (kk >> 1);
      double af[FM], bf[FN];
#pragma unroll
      for (int a = 0; a < FM; ++a) {
        const int row = wm0 + a * 8 + a_row;
        double v = AK ? As[(row * S::LDA + kc) * 2 + (kk & 1)] : As[(kc * S::LDA + row) * 2 + (kk & 1)];
        af[a] = a_neg ? -v : v;
      }
#pragma unroll
      for (int b = 0; b < FN; ++b) {
        const int col = wn0 + b * 4 + (b_nn >> 1);
        double v = BNC ? Bs[(kc * S::LDB + col) * 2 + b_part] : Bs[(col * S::LDB + kc) * 2 + b_part];
        bf[b] = b_neg ? -v : v;
      }
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // Epilogue: each lane owns complex C[a*8 + lane>>2][b*4 + lane&3] of every fragment.
  if (p.splits == 1) {
    double2* C = p.C + offC;
#pragma unroll
    for (int a = 0; a < FM; ++a) {
      const int li = wm0 + a * 8 + (lane >> 2);
      if (m0 + li >= p.M) continue;
      const int64_t ro = rowoff[li];
#pragma unroll
      for (int b = 0; b < FN; ++b) {
        const int lj = wn0 + b * 4 + (lane & 3);
        if (n0 + lj >= p.N) continue;
        double2* dst = C + ro + coloff[lj];
        double2 v = make_double2(acc[a][b][0], acc[a][b][1]);
        if (p.accumulate) v = cadd(*dst, v);
        *dst = v;
      }
    }
  } else {
    double2* W = p.work + ((static_cast<int64_t>(split) * p.batch + bz) * p.M) * p.N;
#pragma unroll
    for (int a = 0; a < FM; ++a) {
      const int64_t gi = m0 + wm0 + a * 8 + (lane >> 2);
      if (gi >= p.M) continue;
#pragma unroll
      for (int b = 0; b < FN; ++b) {
        const int64_t gj = n0 + wn0 + b * 4 + (lane & 3);
        if (gj >= p.N) continue;
        W[gi * p.N + gj] = make_double2(acc[a][b][0], acc[a][b][1]);
      }
    }
  }
}

// Deterministic split-K reduction (fixed summation order) + epilogue scatter.
__global__ void zgemm_splitk_reduce(const ZgemmParams p) {
  const int64_t total = p.batch * p.M * p.N;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = e % p.N;
    const int64_t i = (e / p.N) % p.M;
    const int64_t b = e / (p.N * p.M);
    double2 s = make_double2(0.0, 0.0);
    for (int sp = 0; sp < p.splits; ++sp) s = cadd(s, p.work[(sp * p.batch + b) * p.M * p.N + i * p.N + j]);
    int64_t offC = 0, idx = b;
    for (int a = p.nb - 1; a >= 0; --a) {
      int64_t q = idx / p.bext[a];
      offC += (idx - q * p.bext[a]) * p.bsC[a];
      idx = q;
    }
    double2* dst = p.C + offC + decode_offset(i, p.nr, p.rext, p.rstr) + decode_offset(j, p.nc, p.cext, p.cstr);
    if (p.accumulate) s = cadd(*dst, s);
    *dst = s;
  }
}

// Small problems (the k x k products, scalars and thin chains of the
// latency-bound configs): one thread per output element, a plain FMA loop over
// K straight from global memory (L1/L2 resident).  The tiled DMMA kernels pay
// ~2k instructions of pipeline prologue, index setup and epilogue per warp --
// 8-14 us for a 4 x 16 x 4 product -- where this kernel finishes in ~2 us.
__global__ void __launch_bounds__(128) zgemm_small_kernel(const ZgemmParams p) {
  const int64_t MN = p.M * p.N;
  for (int64_t bz = blockIdx.y; bz < p.batch; bz += gridDim.y) {
    int64_t offA = 0, offB = 0, offC = 0, idx = bz;
    for (int a = p.nb - 1; a >= 0; --a) {
      const int64_t q = idx / p.bext[a], r = idx - q * p.bext[a];
      offA += r * p.bsA[a];
      offB += r * p.bsB[a];
      offC += r * p.bsC[a];
      idx = q;
    }
    const double sa = p.conjA ? -1.0 : 1.0, sb = p.conjB ? -1.0 : 1.0;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < MN;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      const int64_t i = e / p.N, j = e - (e / p.N) * p.N;
      const double2* a = p.A + offA + i * p.sAi;
      const double2* b = p.B + offB + j * p.sBj;
      double re = 0.0, im = 0.0;
#pragma unroll 4
      for (int64_t k = 0; k < p.K; ++k) {
        const double2 x = __ldg(a + k * p.sAk), y = __ldg(b + k * p.sBk);
        const double xi = sa * x.y, yi = sb * y.y;
        re = fma(x.x, y.x, re);
        re = fma(-xi, yi, re);
        im = fma(x.x, yi, im);
        im = fma(xi, y.x, im);
      }
      double2* dst = p.C + offC + decode_offset(i, p.nr, p.rext, p.rstr) + decode_offset(j, p.nc, p.cext, p.cstr);
      double2 v = make_double2(re, im);
      if (p.accumulate) v = cadd(*dst, v);
      *dst = v;
    }
  }
}

void launch_small(const ZgemmParams& p, cudaStream_t stream) {
  const int64_t blocks = std::min<int64_t>((p.M * p.N + 127) / 128, 1024);
  dim3 grid(static_cast<unsigned>(std::max<int64_t>(blocks, 1)), static_cast<unsigned>(std::min<int64_t>(p.batch, 65535)));
  zgemm_small_kernel<<<grid, 128, 0, stream>>>(p);
  PEPSB_LAUNCH();
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AK, bool BNC>
void launch_cfg(const ZgemmParams& p, cudaStream_t stream) {
  using S = Smem<BM, BN, BK, AK, BNC>;
  constexpr int NT = (BM / WM) * (BN / WN) * 32;
  const size_t smem = static_cast<size_t>(STAGES) * S::STAGE * sizeof(double2) + (BM + BN) * sizeof(int64_t);
  auto kern = zgemm_dmma_kernel<BM, BN, BK, WM, WN, STAGES, AK, BNC>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    PEPSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    attr_set = true;
  }
  const int64_t tiles = ((p.M + BM - 1) / BM) * ((p.N + BN - 1) / BN);
  dim3 grid(static_cast<unsigned>(tiles), static_cast<unsigned>(p.batch * p.splits));
  kern<<<grid, NT, smem, stream>>>(p);
  PEPSB_LAUNCH();
}

constexpr int kBK = 16, kStages = 3;

// Tile configurations (BM x BN complex, warps WM x WN): the 72-wide ones cover
// the k = 72 probe dimension of config 2 in one tile (no 8/64 tail waste).
struct TileCfg {
  int bm, bn;
};
constexpr TileCfg kCfgs[] = {{64, 64}, {64, 72}, {72, 64}, {72, 72}, {128, 64}};
constexpr TileCfg kCfgs3m[] = {{64, 32}, {64, 72}, {72, 64}, {72, 72}, {64, 32}};
constexpr TileCfg kCfgs4c[] = {{64, 64}, {64, 72}, {72, 64}, {72, 72}, {64, 64}};

int choose_cfg(int64_t M, int64_t N) {
  static const bool cfg4 = getenv("PEPSB_CFG4") != nullptr;
  const bool m72 = M > 64 && M <= 72, n72 = N > 64 && N <= 72;
  if (m72 && n72) return 3;
  if (n72) return 1;
  if (m72) return 2;
  if (cfg4 && M > 64 && M <= 128 && N >= 4096) return 4;
  return 0;
}

// C^T = B^T A^T: swap the operand roles (and the epilogue's row/column decode)
// so that a 72-wide side becomes N and the 4-warp 64x72 tile applies.
void transpose_problem(ZgemmParams& p) {
  std::swap(p.A, p.B);
  const int64_t sAi = p.sAi, sAk = p.sAk;
  p.sAi = p.sBj;
  p.sAk = p.sBk;
  p.sBk = sAk;
  p.sBj = sAi;
  std::swap(p.conjA, p.conjB);
  std::swap(p.realA, p.realB);
  std::swap(p.M, p.N);
  for (int a = 0; a < 4; ++a) std::swap(p.bsA[a], p.bsB[a]);
  std::swap(p.nr, p.nc);
  for (int a = 0; a < kMaxModes; ++a) {
    std::swap(p.rext[a], p.cext[a]);
    std::swap(p.rstr[a], p.cstr[a]);
  }
}

int ctas_per_sm(int cfg) { return cfg <= 1 ? 2 : 1; }
int ctas_per_sm3m(int cfg) { return cfg == 0 ? 2 : 1; }

std::atomic<int> g_algo{-1};
std::atomic<int> g_ws{-1};

template <bool AK, bool BNC>
void launch_any(const ZgemmParams& p, cudaStream_t stream) {
  switch (p.cfg) {
    case 1: launch_cfg<64, 72, kBK, 32, 36, kStages, AK, BNC>(p, stream); break;
    case 2: launch_cfg<72, 64, kBK, 24, 32, kStages, AK, BNC>(p, stream); break;
    case 3: launch_cfg<72, 72, kBK, 24, 36, kStages, AK, BNC>(p, stream); break;
    case 4: launch_cfg<128, 64, kBK, 32, 32, kStages, AK, BNC>(p, stream); break;
    default: launch_cfg<64, 64, kBK, 32, 32, kStages, AK, BNC>(p, stream); break;
  }
}

// ---------------------------------------------------------------- 3M (Gauss) variant
// C = A B over complex k with three real products per 8x8 complex block,
//   P1 = Ar Br,  P2 = Ai Bi,  P3 = (Ar + Ai)(Br + Bi),
//   Re C = P1 - P2,  Im C = P3 - P1 - P2      (conjugation: Ai -> -Ai, Bi -> -Bi),
// i.e. 3 real MACs per complex MAC instead of the real embedding's 4 (the
// zgemm3m scheme).  One DMMA.8x8x4 covers 8 x 8 complex outputs over 4 complex
// k; each lane loads its A / B fragment element as one complex value (LDS.128)
// and forms (r, i, r + i) in registers.  Smem strides are padded so every
// quarter-warp's 8 LDS.128 hit distinct 16-byte bank groups.
template <int BM, int BN, int BK, bool AK, bool BNC>
struct Smem3 {
  static constexpr int LDA = AK ? (BK + 4) : (BM + 2);
  static constexpr int LDB = BNC ? (BN + 2) : (BK + 4);
  static constexpr int A_ELEMS = AK ? BM * LDA : BK * LDA;
  static constexpr int B_ELEMS = BNC ? BK * LDB : BN * LDB;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AK, bool BNC, int ALG, int MINB>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32, MINB)
    zgemm_cx_kernel(const ZgemmParams p) {
  // 3M: P1, P2, P3;  4M: Re, Im;  complex x real (ALG 1): one DMMA pair (re, im)
  constexpr int NACC = ALG == 3 ? 3 : ALG == 1 ? 1 : 2;
  using S = Smem3<BM, BN, BK, AK, BNC>;
  constexpr int NT = (BM / WM) * (BN / WN) * 32;
  constexpr int FM = WM / 8;  // 8-row blocks per warp
  // 8-column blocks per warp; complex x real: a DMMA covers 8 interleaved
  // doubles of B = 4 complex columns
  constexpr int FN = ALG == 1 ? WN / 4 : WN / 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* smem = reinterpret_cast<double2*>(smem_raw);
  int64_t* rowoff = reinterpret_cast<int64_t*>(smem + STAGES * S::STAGE);
  int64_t* coloff = rowoff + BM;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wm0 = (warp % (BM / WM)) * WM;
  const int wn0 = (warp / (BM / WM)) * WN;

  const int64_t mtiles = (p.M + BM - 1) / BM;
  const int64_t tile = blockIdx.x;
  const int64_t m0 = (tile % mtiles) * BM;
  const int64_t n0 = (tile / mtiles) * BN;
  const int64_t bz = blockIdx.y / p.splits;
  const int split = blockIdx.y % p.splits;

  int64_t offA = 0, offB = 0, offC = 0;
  {
    int64_t idx = bz;
    for (int a = p.nb - 1; a >= 0; --a) {
      int64_t e = p.bext[a];
      int64_t q = idx / e;
      int64_t r = idx - q * e;
      offA += r * p.bsA[a];
      offB += r * p.bsB[a];
      offC += r * p.bsC[a];
      idx = q;
    }
  }
  const double2* A = p.A + offA;
  const double2* B = p.B + offB;

  const int64_t kbeg = static_cast<int64_t>(split) * p.kchunk;
  const int64_t kend = min(p.K, kbeg + p.kchunk);
  const int64_t nk = (kend - kbeg + BK - 1) / BK;

  // Operand tile loaders, strength-reduced: thread tid copies the elements
  // e = tid + u * NT of the [outer][inner] smem tile, so when NT is a multiple
  // of the inner extent its inner index is fixed and the outer index advances
  // by NT / inner -- one 64-bit base per operand, a constant stride per u, a
  // k-tile stride per stage, and row-validity bits computed once.
  constexpr int AIN = AK ? BK : BM, AOUT = AK ? BM : BK;
  constexpr int BIN = BNC ? BN : BK, BOUT = BNC ? BK : BN;
  constexpr bool AREG = (NT % AIN) == 0, BREG = (NT % BIN) == 0;
  constexpr int UA = (BM * BK + NT - 1) / NT, UB = (BK * BN + NT - 1) / NT;
  constexpr int AOS = AREG ? NT / AIN : 1, BOS = BREG ? NT / BIN : 1;
  const int a_in = tid % AIN, a_o0 = tid / AIN, b_in = tid % BIN, b_o0 = tid / BIN;
  int64_t a_base, a_ustr, b_base, b_ustr;
  unsigned a_ok = 0, b_ok = 0;  // AK: row bits per u / !AK: row ok in bit 0 (and BNC likewise)
  if (AK) {
    a_base = (m0 + a_o0) * p.sAi + (kbeg + a_in) * p.sAk;
    a_ustr = AOS * p.sAi;
#pragma unroll
    for (int u = 0; u < UA; ++u)
      if (a_o0 + u * AOS < AOUT && m0 + a_o0 + u * AOS < p.M) a_ok |= 1u << u;
  } else {
    a_base = (m0 + a_in) * p.sAi + (kbeg + a_o0) * p.sAk;
    a_ustr = AOS * p.sAk;
    a_ok = m0 + a_in < p.M ? 1u : 0u;
  }
  if (BNC) {
    b_base = (kbeg + b_o0) * p.sBk + (n0 + b_in) * p.sBj;
    b_ustr = BOS * p.sBk;
    b_ok = n0 + b_in < p.N ? 1u : 0u;
  } else {
    b_base = (n0 + b_o0) * p.sBj + (kbeg + b_in) * p.sBk;
    b_ustr = BOS * p.sBj;
#pragma unroll
    for (int u = 0; u < UB; ++u)
      if (b_o0 + u * BOS < BOUT && n0 + b_o0 + u * BOS < p.N) b_ok |= 1u << u;
  }
  // Issues part `part` of `nparts` of stage kt's copies (the main loop spreads
  // one stage over the k-steps of the previous tile, CUTLASS-style).
  auto load_stage = [&](int slot, int64_t kt, int part, int nparts) {
    double2* As = smem + slot * S::STAGE;
    double2* Bs = As + S::A_ELEMS;
    const int64_t k0 = kbeg + kt * BK;
    if constexpr (AREG) {
      const double2* src = A + a_base + kt * BK * p.sAk;
#pragma unroll
      for (int u = 0; u < UA; ++u) {
        if (u < part * UA / nparts || u >= (part + 1) * UA / nparts) continue;
        const int o = a_o0 + u * AOS;
        if ((AOUT % AOS) != 0 && o >= AOUT) break;  // past the tile (a zero-fill copy would land in B)
        const bool ok = AK ? (((a_ok >> u) & 1u) && k0 + a_in < kend) : (a_ok && k0 + o < kend);
        cp_async16(As + o * S::LDA + a_in, ok ? src + u * a_ustr : A, ok);
      }
    } else if (part == 0) {
#pragma unroll
      for (int e = tid; e < BM * BK; e += NT) {
        int i, k;
        if (AK) { i = e / BK; k = e % BK; } else { k = e / BM; i = e % BM; }
        const int64_t gi = m0 + i, gk = k0 + k;
        const bool ok = gi < p.M && gk < kend;
        const double2* src = ok ? A + gi * p.sAi + gk * p.sAk : A;
        double2* dst = AK ? As + i * S::LDA + k : As + k * S::LDA + i;
        cp_async16(dst, src, ok);
      }
    }
    if constexpr (BREG) {
      const double2* src = B + b_base + kt * BK * p.sBk;
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        if (u < part * UB / nparts || u >= (part + 1) * UB / nparts) continue;
        const int o = b_o0 + u * BOS;
        if ((BOUT % BOS) != 0 && o >= BOUT) break;  // past the tile (would spill into the next stage)
        const bool ok = BNC ? (b_ok && k0 + o < kend) : (((b_ok >> u) & 1u) && k0 + b_in < kend);
        cp_async16(Bs + o * S::LDB + b_in, ok ? src + u * b_ustr : B, ok);
      }
    } else if (part == 0) {
#pragma unroll
      for (int e = tid; e < BK * BN; e += NT) {
        int k, j;
        if (BNC) { k = e / BN; j = e % BN; } else { j = e / BK; k = e % BK; }
        const int64_t gj = n0 + j, gk = k0 + k;
        const bool ok = gj < p.N && gk < kend;
        const double2* src = ok ? B + gk * p.sBk + gj * p.sBj : B;
        double2* dst = BNC ? Bs + k * S::LDB + j : Bs + j * S::LDB + k;
        cp_async16(dst, src, ok);
      }
    }
  };


  double acc[FM][FN][NACC][2];
#pragma unroll
  for (int a = 0; a < FM; ++a)
#pragma unroll
    for (int b = 0; b < FN; ++b)
#pragma unroll
      for (int t = 0; t < NACC; ++t) acc[a][b][t][0] = acc[a][b][t][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, s, 0, 1);
    cp_async_commit();
  }

  // Epilogue scatter offsets, decoded while the first stages are in flight (the
  // mixed-radix decode is a chain of 64-bit divisions on operands read from the
  // parameter bank; ncu put 3.6 % of the short-K kernels' stall samples on it
  // and 14 % on the first barrier's wait for the stage it used to precede).
  if (p.splits == 1) {
    for (int r = tid; r < BM; r += NT) {
      const int64_t gi = m0 + r;
      rowoff[r] = gi < p.M ? decode_offset(gi, p.nr, p.rext, p.rstr) : 0;
    }
    for (int c = tid; c < BN; c += NT) {
      const int64_t gj = n0 + c;
      coloff[c] = gj < p.N ? decode_offset(gj, p.nc, p.cext, p.cstr) : 0;
    }
  }

  const int kq = lane & 3;   // k within the 4-wide step (A column / B row of the fragment)
  const int rq = lane >> 2;  // A fragment row / B fragment column
  // conjugation: flip the sign bit of the imaginary parts (integer XOR, keeps
  // the FP64 pipe free for nothing but the DMMAs)
  const long long sga = p.conjA ? (long long)0x8000000000000000ULL : 0LL;
  const long long sgb = p.conjB ? (long long)0x8000000000000000ULL : 0LL;
  auto flip = [](double v, long long m) { return __longlong_as_double(__double_as_longlong(v) ^ m); };
  // Fragments double-buffered in registers: the LDS for step s+1 are issued
  // before the DMMAs of step s; one barrier per k-tile (before the first
  // fragment load of the next slot, which also frees the current slot for the
  // prefetch of stage kt + STAGES).
  double2 fa[2][ALG == 1 ? 1 : FM], fb[2][ALG == 1 ? 1 : FN];
  double ra[2][FM], rb[2][FN];  // complex x real: A real parts, B interleaved doubles
  const long long sgbr = (rq & 1) ? sgb : 0LL;  // complex x real: this lane's B double is an imaginary part
  auto load_frags = [&](int buf, int slot, int ks) {
    const double2* As = smem + slot * S::STAGE;
    const double2* Bs = As + S::A_ELEMS;
    const int kc = ks * 4 + kq;
    if constexpr (ALG == 1) {
#pragma unroll
      for (int a = 0; a < FM; ++a) {
        const int row = wm0 + a * 8 + rq;
        ra[buf][a] = (AK ? As[row * S::LDA + kc] : As[kc * S::LDA + row]).x;
      }
#pragma unroll
      for (int b = 0; b < FN; ++b) {
        const int col = wn0 + b * 4 + (rq >> 1);
        const double* e = reinterpret_cast<const double*>(BNC ? Bs + kc * S::LDB + col : Bs + col * S::LDB + kc);
        rb[buf][b] = flip(e[rq & 1], sgbr);
      }
      return;
    } else {
#pragma unroll
      for (int a = 0; a < FM; ++a) {
        const int row = wm0 + a * 8 + rq;
        fa[buf][a] = AK ? As[row * S::LDA + kc] : As[kc * S::LDA + row];
      }
#pragma unroll
      for (int b = 0; b < FN; ++b) {
        const int col = wn0 + b * 8 + rq;
        fb[buf][b] = BNC ? Bs[kc * S::LDB + col] : Bs[col * S::LDB + kc];
      }
    }
  };
  auto compute = [&](int buf) {
    if constexpr (ALG == 1) {
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) dmma884(acc[a][b][0][0], acc[a][b][0][1], ra[buf][a], rb[buf][b]);
    } else if constexpr (ALG == 3) {
      double ar[FM], ai[FM], as[FM], br[FN], bi[FN], bs[FN];
#pragma unroll
      for (int a = 0; a < FM; ++a) {
        ar[a] = fa[buf][a].x;
        ai[a] = flip(fa[buf][a].y, sga);
        as[a] = ar[a] + ai[a];
      }
#pragma unroll
      for (int b = 0; b < FN; ++b) {
        br[b] = fb[buf][b].x;
        bi[b] = flip(fb[buf][b].y, sgb);
        bs[b] = br[b] + bi[b];
      }
      // pass-major: the P3 DMMAs, which wait on the DADD sums, come after
      // 2 FM FN DMMAs that hide the DADD latency
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) dmma884(acc[a][b][0][0], acc[a][b][0][1], ar[a], br[b]);
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) dmma884(acc[a][b][1][0], acc[a][b][1][1], ai[a], bi[b]);
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) dmma884(acc[a][b][2][0], acc[a][b][2][1], as[a], bs[b]);
    } else {
      // Re += Ar Br - Ai Bi,  Im += Ar Bi + Ai Br
      double ai[FM], nai[FM], bi[FN];
#pragma unroll
      for (int a = 0; a < FM; ++a) {
        ai[a] = flip(fa[buf][a].y, sga);
        nai[a] = flip(fa[buf][a].y, sga ^ (long long)0x8000000000000000ULL);
      }
#pragma unroll
      for (int b = 0; b < FN; ++b) bi[b] = flip(fb[buf][b].y, sgb);
      // pass-major order: the two DMMAs into the same accumulator are
      // FM * FN * 2 instructions apart (DMMA accumulator latency)
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) {
          dmma884(acc[a][b][0][0], acc[a][b][0][1], fa[buf][a].x, fb[buf][b].x);
          dmma884(acc[a][b][1][0], acc[a][b][1][1], fa[buf][a].x, bi[b]);
        }
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) {
          dmma884(acc[a][b][0][0], acc[a][b][0][1], nai[a], bi[b]);
          dmma884(acc[a][b][1][0], acc[a][b][1][1], ai[a], fb[buf][b].x);
        }
    }
  };
  constexpr int KS = BK / 4;
  // Stage kt + STAGES - 1 is copied into the slot freed by the previous tile's
  // closing barrier, a quarter per k-step of tile kt; one barrier per tile.
  if (nk > 0) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    load_frags(0, 0, 0);
  }
  static_assert(KS % 2 == 0, "k steps per tile must be even (static fragment buffers)");
  for (int64_t kt = 0; kt < nk; ++kt) {
    const int slot = static_cast<int>(kt % STAGES);
    const int64_t pf = kt + STAGES - 1;
    const int pslot = static_cast<int>(pf % STAGES);
    const bool do_pf = pf < nk;
#pragma unroll
    for (int kp = 0; kp < KS; kp += 2) {
      load_frags(1, slot, kp + 1);
      if (do_pf) load_stage(pslot, pf, kp, KS);
      compute(0);
      if (do_pf) load_stage(pslot, pf, kp + 1, KS);
      if (kp + 2 < KS) {
        load_frags(0, slot, kp + 2);
      } else {
        cp_async_commit();
        if (kt + 1 < nk) {
          cp_async_wait<STAGES - 2>();
          __syncthreads();
          load_frags(0, static_cast<int>((kt + 1) % STAGES), 0);
        }
      }
      compute(1);
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // Epilogue: lane owns C[a*8 + lane>>2][b*8 + 2*(lane&3) + {0,1}] of every block
  // (complex x real: the complex C[a*8 + lane>>2][b*4 + lane&3] = (c0, c1)).
#pragma unroll
  for (int a = 0; a < FM; ++a) {
    const int li = wm0 + a * 8 + (lane >> 2);
    if (m0 + li >= p.M) continue;
#pragma unroll
    for (int b = 0; b < FN; ++b)
#pragma unroll
      for (int h = 0; h < (ALG == 1 ? 1 : 2); ++h) {
        const int lj = ALG == 1 ? wn0 + b * 4 + (lane & 3) : wn0 + b * 8 + 2 * (lane & 3) + h;
        if (n0 + lj >= p.N) continue;
        double2 v;
        if constexpr (ALG == 1) {
          v = make_double2(acc[a][b][0][0], acc[a][b][0][1]);
        } else if constexpr (ALG == 3) {
          const double p1 = acc[a][b][0][h], p2 = acc[a][b][1][h], p3 = acc[a][b][NACC - 1][h];
          v = make_double2(p1 - p2, p3 - p1 - p2);
        } else {
          v = make_double2(acc[a][b][0][h], acc[a][b][1][h]);
        }
        if (p.splits == 1) {
          double2* dst = p.C + offC + rowoff[li] + coloff[lj];
          if (p.accumulate) v = cadd(*dst, v);
          *dst = v;
        } else {
          double2* W = p.work + ((static_cast<int64_t>(split) * p.batch + bz) * p.M) * p.N;
          W[(m0 + li) * p.N + n0 + lj] = v;
        }
      }
  }
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AK, bool BNC, int ALG, int MINB>
void launch_cx(const ZgemmParams& p, cudaStream_t stream) {
  using S = Smem3<BM, BN, BK, AK, BNC>;
  constexpr int NT = (BM / WM) * (BN / WN) * 32;
  const size_t smem = static_cast<size_t>(STAGES) * S::STAGE * sizeof(double2) + (BM + BN) * sizeof(int64_t);
  auto kern = zgemm_cx_kernel<BM, BN, BK, WM, WN, STAGES, AK, BNC, ALG, MINB>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    PEPSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    attr_set = true;
  }
  const int64_t tiles = ((p.M + BM - 1) / BM) * ((p.N + BN - 1) / BN);
  dim3 grid(static_cast<unsigned>(tiles), static_cast<unsigned>(p.batch * p.splits));
  kern<<<grid, NT, smem, stream>>>(p);
  PEPSB_LAUNCH();
}

template <bool AK, bool BNC>
void launch_any3m(const ZgemmParams& p, cudaStream_t stream) {
  if (zgemm_c3m_cfg() == 1) {  // more, smaller warp tiles (latency hiding)
    switch (p.cfg) {
      case 1: launch_cx<64, 72, kBK, 8, 24, kStages, AK, BNC, 3, 1>(p, stream); break;
      case 2: launch_cx<72, 64, kBK, 24, 8, kStages, AK, BNC, 3, 1>(p, stream); break;
      case 3: launch_cx<72, 72, kBK, 8, 24, kStages, AK, BNC, 3, 1>(p, stream); break;
      default: launch_cx<64, 32, kBK, 16, 16, kStages, AK, BNC, 3, 2>(p, stream); break;
    }
    return;
  }
  switch (p.cfg) {
    case 1: launch_cx<64, 72, kBK, 16, 24, kStages, AK, BNC, 3, 1>(p, stream); break;
    case 2: launch_cx<72, 64, kBK, 24, 16, kStages, AK, BNC, 3, 1>(p, stream); break;
    case 3: launch_cx<72, 72, kBK, 24, 24, kStages, AK, BNC, 3, 1>(p, stream); break;
    default: launch_cx<64, 32, kBK, 32, 16, kStages, AK, BNC, 3, 2>(p, stream); break;
  }
}

// ---------------------------------------------------------------- tile-streaming variant
// Short-K problems (K = 64 / 128 per output tile: GEMMs (1)/(2) of every
// operator application) spend a large share of a one-tile CTA in the
// pipeline fill and the epilogue.  Here a resident CTA walks a sequence of
// output tiles (tile = blockIdx.x + i * gridDim.x, m fastest so consecutive
// CTAs share the B tile in L2) and the cp.async pipeline runs straight across
// tile boundaries: the first k-stages of tile i+1 are in flight while tile i
// finishes and writes its epilogue, and the epilogue offsets of tile i+1 are
// decoded into the other half of a double buffer during tile i.  Same
// fragments, same k order per accumulator as zgemm_cx_kernel (results are
// bitwise identical); requires splits == 1 and nk >= 4 (see use_stream).
template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AK, bool BNC, int ALG, int MINB>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32, MINB)
    zgemm_stream_kernel(const ZgemmParams p) {
  constexpr int NACC = ALG == 3 ? 3 : ALG == 1 ? 1 : 2;
  using S = Smem3<BM, BN, BK, AK, BNC>;
  constexpr int NT = (BM / WM) * (BN / WN) * 32;
  constexpr int FM = WM / 8;
  constexpr int FN = ALG == 1 ? WN / 4 : WN / 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* smem = reinterpret_cast<double2*>(smem_raw);
  int64_t* rowoff = reinterpret_cast<int64_t*>(smem + STAGES * S::STAGE);  // [2][BM]
  int64_t* coloff = rowoff + 2 * BM;                                        // [2][BN]

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wm0 = (warp % (BM / WM)) * WM;
  const int wn0 = (warp / (BM / WM)) * WN;

  const int64_t mtiles = (p.M + BM - 1) / BM;
  const int64_t per_batch = mtiles * ((p.N + BN - 1) / BN);
  const int64_t tiles = per_batch * p.batch;
  if (static_cast<int64_t>(blockIdx.x) >= tiles) return;
  const int64_t my_tiles = (tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int64_t nk = (p.K + BK - 1) / BK;
  const int64_t steps = my_tiles * nk;

  struct Coord {
    int64_t m0, n0, offA, offB, offC;
  };
  auto coord = [&](int64_t local) {
    const int64_t t = blockIdx.x + local * gridDim.x;
    const int64_t bz = t / per_batch, r = t - bz * per_batch;
    Coord c{(r % mtiles) * BM, (r / mtiles) * BN, 0, 0, 0};
    int64_t idx = bz;
    for (int a = p.nb - 1; a >= 0; --a) {
      const int64_t e = p.bext[a];
      const int64_t q = idx / e;
      const int64_t rr = idx - q * e;
      c.offA += rr * p.bsA[a];
      c.offB += rr * p.bsB[a];
      c.offC += rr * p.bsC[a];
      idx = q;
    }
    return c;
  };

  constexpr int AIN = AK ? BK : BM, AOUT = AK ? BM : BK;
  constexpr int BIN = BNC ? BN : BK, BOUT = BNC ? BK : BN;
  constexpr bool AREG = (NT % AIN) == 0, BREG = (NT % BIN) == 0;
  constexpr int UA = (BM * BK + NT - 1) / NT, UB = (BK * BN + NT - 1) / NT;
  constexpr int AOS = AREG ? NT / AIN : 1, BOS = BREG ? NT / BIN : 1;
  const int a_in = tid % AIN, a_o0 = tid / AIN, b_in = tid % BIN, b_o0 = tid / BIN;
  const int64_t a_ustr = AK ? AOS * p.sAi : AOS * p.sAk;
  const int64_t b_ustr = BNC ? BOS * p.sBk : BOS * p.sBj;

  // loader state of the tile whose stages are being copied
  int64_t ld_local = -1, ld_m0 = 0, ld_n0 = 0, a_base = 0, b_base = 0;
  const double2* A = p.A;
  const double2* B = p.B;
  unsigned a_ok = 0, b_ok = 0;
  auto set_load_tile = [&](int64_t local) {
    const Coord c = coord(local);
    ld_local = local;
    ld_m0 = c.m0;
    ld_n0 = c.n0;
    A = p.A + c.offA;
    B = p.B + c.offB;
    a_ok = 0;
    b_ok = 0;
    if (AK) {
      a_base = (ld_m0 + a_o0) * p.sAi + a_in * p.sAk;
#pragma unroll
      for (int u = 0; u < UA; ++u)
        if (a_o0 + u * AOS < AOUT && ld_m0 + a_o0 + u * AOS < p.M) a_ok |= 1u << u;
    } else {
      a_base = (ld_m0 + a_in) * p.sAi + a_o0 * p.sAk;
      a_ok = ld_m0 + a_in < p.M ? 1u : 0u;
    }
    if (BNC) {
      b_base = b_o0 * p.sBk + (ld_n0 + b_in) * p.sBj;
      b_ok = ld_n0 + b_in < p.N ? 1u : 0u;
    } else {
      b_base = (ld_n0 + b_o0) * p.sBj + b_in * p.sBk;
#pragma unroll
      for (int u = 0; u < UB; ++u)
        if (b_o0 + u * BOS < BOUT && ld_n0 + b_o0 + u * BOS < p.N) b_ok |= 1u << u;
    }
    // epilogue offsets of this tile into its half of the double buffer (the
    // epilogue that last read that half finished before the previous barrier)
    int64_t* ro = rowoff + (local & 1) * BM;
    int64_t* co = coloff + (local & 1) * BN;
    for (int r = tid; r < BM; r += NT) {
      const int64_t gi = ld_m0 + r;
      ro[r] = gi < p.M ? decode_offset(gi, p.nr, p.rext, p.rstr) : 0;
    }
    for (int c2 = tid; c2 < BN; c2 += NT) {
      const int64_t gj = ld_n0 + c2;
      co[c2] = gj < p.N ? decode_offset(gj, p.nc, p.cext, p.cstr) : 0;
    }
  };
  auto load_stage = [&](int slot, int64_t kt, int part, int nparts) {
    double2* As = smem + slot * S::STAGE;
    double2* Bs = As + S::A_ELEMS;
    const int64_t k0 = kt * BK;
    if constexpr (AREG) {
      const double2* src = A + a_base + kt * BK * p.sAk;
#pragma unroll
      for (int u = 0; u < UA; ++u) {
        if (u < part * UA / nparts || u >= (part + 1) * UA / nparts) continue;
        const int o = a_o0 + u * AOS;
        if ((AOUT % AOS) != 0 && o >= AOUT) break;
        const bool ok = AK ? (((a_ok >> u) & 1u) && k0 + a_in < p.K) : (a_ok && k0 + o < p.K);
        cp_async16(As + o * S::LDA + a_in, ok ? src + u * a_ustr : A, ok);
      }
    } else if (part == 0) {
#pragma unroll
      for (int e = tid; e < BM * BK; e += NT) {
        int i, k;
        if (AK) { i = e / BK; k = e % BK; } else { k = e / BM; i = e % BM; }
        const int64_t gi = ld_m0 + i, gk = k0 + k;
        const bool ok = gi < p.M && gk < p.K;
        const double2* src = ok ? A + gi * p.sAi + gk * p.sAk : A;
        double2* dst = AK ? As + i * S::LDA + k : As + k * S::LDA + i;
        cp_async16(dst, src, ok);
      }
    }
    if constexpr (BREG) {
      const double2* src = B + b_base + kt * BK * p.sBk;
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        if (u < part * UB / nparts || u >= (part + 1) * UB / nparts) continue;
        const int o = b_o0 + u * BOS;
        if ((BOUT % BOS) != 0 && o >= BOUT) break;
        const bool ok = BNC ? (b_ok && k0 + o < p.K) : (((b_ok >> u) & 1u) && k0 + b_in < p.K);
        cp_async16(Bs + o * S::LDB + b_in, ok ? src + u * b_ustr : B, ok);
      }
    } else if (part == 0) {
#pragma unroll
      for (int e = tid; e < BK * BN; e += NT) {
        int k, j;
        if (BNC) { k = e / BN; j = e % BN; } else { j = e / BK; k = e % BK; }
        const int64_t gj = ld_n0 + j, gk = k0 + k;
        const bool ok = gj < p.N && gk < p.K;
        const double2* src = ok ? B + gk * p.sBk + gj * p.sBj : B;
        double2* dst = BNC ? Bs + k * S::LDB + j : Bs + j * S::LDB + k;
        cp_async16(dst, src, ok);
      }
    }
  };
  // Prefetch cursor (flattened step = local * nk + kt), advanced by one step
  // at a time: no divisions in the main loop.
  int64_t pf_kt = 0;
  int pf_slot = 0;
  auto pf_advance = [&]() {
    if (++pf_kt == nk) {
      pf_kt = 0;
      if (ld_local + 1 < my_tiles) set_load_tile(ld_local + 1);
    }
    if (++pf_slot == STAGES) pf_slot = 0;
  };

  double acc[FM][FN][NACC][2];
#pragma unroll
  for (int a = 0; a < FM; ++a)
#pragma unroll
    for (int b = 0; b < FN; ++b)
#pragma unroll
      for (int t = 0; t < NACC; ++t) acc[a][b][t][0] = acc[a][b][t][1] = 0.0;

  set_load_tile(0);
#pragma unroll
  for (int s0 = 0; s0 < STAGES - 1; ++s0) {
    if (s0 < steps) {
      load_stage(pf_slot, pf_kt, 0, 1);
      pf_advance();
    }
    cp_async_commit();
  }

  const int kq = lane & 3;
  const int rq = lane >> 2;
  const long long sga = p.conjA ? (long long)0x8000000000000000ULL : 0LL;
  const long long sgb = p.conjB ? (long long)0x8000000000000000ULL : 0LL;
  auto flip = [](double v, long long m) { return __longlong_as_double(__double_as_longlong(v) ^ m); };
  double2 fa[2][ALG == 1 ? 1 : FM], fb[2][ALG == 1 ? 1 : FN];
  double ra[2][FM], rb[2][FN];
  const long long sgbr = (rq & 1) ? sgb : 0LL;
  auto load_frags = [&](int buf, int slot, int ks) {
    const double2* As = smem + slot * S::STAGE;
    const double2* Bs = As + S::A_ELEMS;
    const int kc = ks * 4 + kq;
    if constexpr (ALG == 1) {
#pragma unroll
      for (int a = 0; a < FM; ++a) {
        const int row = wm0 + a * 8 + rq;
        ra[buf][a] = (AK ? As[row * S::LDA + kc] : As[kc * S::LDA + row]).x;
      }
#pragma unroll
      for (int b = 0; b < FN; ++b) {
        const int col = wn0 + b * 4 + (rq >> 1);
        const double* e = reinterpret_cast<const double*>(BNC ? Bs + kc * S::LDB + col : Bs + col * S::LDB + kc);
        rb[buf][b] = flip(e[rq & 1], sgbr);
      }
    } else {
#pragma unroll
      for (int a = 0; a < FM; ++a) {
        const int row = wm0 + a * 8 + rq;
        fa[buf][a] = AK ? As[row * S::LDA + kc] : As[kc * S::LDA + row];
      }
#pragma unroll
      for (int b = 0; b < FN; ++b) {
        const int col = wn0 + b * 8 + rq;
        fb[buf][b] = BNC ? Bs[kc * S::LDB + col] : Bs[col * S::LDB + kc];
      }
    }
  };
  auto compute = [&](int buf) {
    if constexpr (ALG == 1) {
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) dmma884(acc[a][b][0][0], acc[a][b][0][1], ra[buf][a], rb[buf][b]);
    } else if constexpr (ALG == 3) {
      double ar[FM], ai[FM], as[FM], br[FN], bi[FN], bs[FN];
#pragma unroll
      for (int a = 0; a < FM; ++a) {
        ar[a] = fa[buf][a].x;
        ai[a] = flip(fa[buf][a].y, sga);
        as[a] = ar[a] + ai[a];
      }
#pragma unroll
      for (int b = 0; b < FN; ++b) {
        br[b] = fb[buf][b].x;
        bi[b] = flip(fb[buf][b].y, sgb);
        bs[b] = br[b] + bi[b];
      }
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) dmma884(acc[a][b][0][0], acc[a][b][0][1], ar[a], br[b]);
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) dmma884(acc[a][b][1][0], acc[a][b][1][1], ai[a], bi[b]);
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) dmma884(acc[a][b][2][0], acc[a][b][2][1], as[a], bs[b]);
    } else {
      double ai[FM], nai[FM], bi[FN];
#pragma unroll
      for (int a = 0; a < FM; ++a) {
        ai[a] = flip(fa[buf][a].y, sga);
        nai[a] = flip(fa[buf][a].y, sga ^ (long long)0x8000000000000000ULL);
      }
#pragma unroll
      for (int b = 0; b < FN; ++b) bi[b] = flip(fb[buf][b].y, sgb);
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) {
          dmma884(acc[a][b][0][0], acc[a][b][0][1], fa[buf][a].x, fb[buf][b].x);
          dmma884(acc[a][b][1][0], acc[a][b][1][1], fa[buf][a].x, bi[b]);
        }
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) {
          dmma884(acc[a][b][0][0], acc[a][b][0][1], nai[a], bi[b]);
          dmma884(acc[a][b][1][0], acc[a][b][1][1], ai[a], fb[buf][b].x);
        }
    }
  };
  auto epilogue = [&](int64_t local) {
    const Coord c = coord(local);
    const int64_t* ro = rowoff + (local & 1) * BM;
    const int64_t* co = coloff + (local & 1) * BN;
#pragma unroll
    for (int a = 0; a < FM; ++a) {
      const int li = wm0 + a * 8 + (lane >> 2);
      if (c.m0 + li >= p.M) continue;
#pragma unroll
      for (int b = 0; b < FN; ++b)
#pragma unroll
        for (int h = 0; h < (ALG == 1 ? 1 : 2); ++h) {
          const int lj = ALG == 1 ? wn0 + b * 4 + (lane & 3) : wn0 + b * 8 + 2 * (lane & 3) + h;
          if (c.n0 + lj >= p.N) continue;
          double2 v;
          if constexpr (ALG == 1) {
            v = make_double2(acc[a][b][0][0], acc[a][b][0][1]);
          } else if constexpr (ALG == 3) {
            const double p1 = acc[a][b][0][h], p2 = acc[a][b][1][h], p3 = acc[a][b][NACC - 1][h];
            v = make_double2(p1 - p2, p3 - p1 - p2);
          } else {
            v = make_double2(acc[a][b][0][h], acc[a][b][1][h]);
          }
          double2* dst = p.C + c.offC + ro[li] + co[lj];
          if (p.accumulate) v = cadd(*dst, v);
          *dst = v;
        }
    }
#pragma unroll
    for (int a = 0; a < FM; ++a)
#pragma unroll
      for (int b = 0; b < FN; ++b)
#pragma unroll
        for (int t = 0; t < NACC; ++t) acc[a][b][t][0] = acc[a][b][t][1] = 0.0;
  };

  constexpr int KS = BK / 4;
  static_assert(KS % 2 == 0, "k steps per tile must be even (static fragment buffers)");
  cp_async_wait<STAGES - 2>();
  __syncthreads();
  load_frags(0, 0, 0);
  int64_t kt = 0, local = 0;
  int slot = 0;
  for (int64_t st = 0; st < steps; ++st) {
    const bool do_pf = st + STAGES - 1 < steps;
    const int next_slot = slot + 1 == STAGES ? 0 : slot + 1;
#pragma unroll
    for (int kp = 0; kp < KS; kp += 2) {
      load_frags(1, slot, kp + 1);
      if (do_pf) load_stage(pf_slot, pf_kt, kp, KS);
      compute(0);
      if (do_pf) load_stage(pf_slot, pf_kt, kp + 1, KS);
      if (kp + 2 < KS) {
        load_frags(0, slot, kp + 2);
      } else {
        cp_async_commit();
        if (do_pf) pf_advance();
        if (st + 1 < steps) {
          cp_async_wait<STAGES - 2>();
          __syncthreads();
          load_frags(0, next_slot, 0);
        }
      }
      compute(1);
    }
    slot = next_slot;
    if (++kt == nk) {
      epilogue(local);
      kt = 0;
      ++local;
    }
  }
  cp_async_wait<0>();
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AK, bool BNC, int ALG, int MINB>
void launch_stream(const ZgemmParams& p, cudaStream_t stream) {
  using S = Smem3<BM, BN, BK, AK, BNC>;
  constexpr int NT = (BM / WM) * (BN / WN) * 32;
  const size_t smem = static_cast<size_t>(STAGES) * S::STAGE * sizeof(double2) + 2 * (BM + BN) * sizeof(int64_t);
  auto kern = zgemm_stream_kernel<BM, BN, BK, WM, WN, STAGES, AK, BNC, ALG, MINB>;
  static bool attr_set = false;
  if (!attr_set) {
    PEPSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    attr_set = true;
  }
  const int64_t tiles = ((p.M + BM - 1) / BM) * ((p.N + BN - 1) / BN) * p.batch;
  const int64_t grid = std::min<int64_t>(tiles, static_cast<int64_t>(MINB) * p.num_sms);
  kern<<<static_cast<unsigned>(grid), NT, smem, stream>>>(p);
  PEPSB_LAUNCH();
}

// Complex x real (A real): 64 x 64 complex tiles, 4 warps of 32 x 32 (8 x 8
// DMMA blocks of 8 rows x 4 complex columns), half the DMMAs of 4M.
// Tile streaming pays where a one-tile CTA is mostly fill + epilogue: short K
// (nk <= 8 k-tiles) over many tiles (at least four resident waves).
bool use_stream(const ZgemmParams& p, int64_t bm, int64_t bn) {
  if (!zgemm_stream_enabled() || p.splits != 1) return false;
  const int64_t nk = (p.K + kBK - 1) / kBK;
  const int64_t tiles = ((p.M + bm - 1) / bm) * ((p.N + bn - 1) / bn) * p.batch;
  // nk >= 4: the next-but-one tile's epilogue offsets are written after the
  // barrier that follows the epilogue which last read that half of the buffer
  return nk >= 4 && nk <= 8 && tiles >= 8 * static_cast<int64_t>(p.num_sms);
}

template <bool AK, bool BNC>
void launch_cr(const ZgemmParams& p, cudaStream_t stream) {
  if (use_stream(p, 64, 64)) launch_stream<64, 64, kBK, 32, 32, kStages, AK, BNC, 1, 2>(p, stream);
  else if (zgemm_cr_cfg() >= 1) launch_cx<64, 64, kBK, 32, 16, kStages, AK, BNC, 1, 2>(p, stream);
  else launch_cx<64, 64, kBK, 32, 32, kStages, AK, BNC, 1, 2>(p, stream);
}

// 4M with complex fragments (one LDS.128 per fragment element, four DMMAs per
// 8 x 8 complex block into Re / Im accumulators), the CUTLASS z884 scheme.
template <bool AK, bool BNC>
void launch_any4c(const ZgemmParams& p, cudaStream_t stream) {
  switch (p.cfg) {
    case 1: launch_cx<64, 72, kBK, 32, 24, kStages, AK, BNC, 4, 1>(p, stream); break;
    case 2: launch_cx<72, 64, kBK, 24, 32, kStages, AK, BNC, 4, 1>(p, stream); break;
    case 3: launch_cx<72, 72, kBK, 24, 24, kStages, AK, BNC, 4, 1>(p, stream); break;
    default:
      if (use_stream(p, 64, 64)) launch_stream<64, 64, kBK, 32, 32, kStages, AK, BNC, 4, 2>(p, stream);
      else if (zgemm_cr_cfg() == 2) launch_cx<64, 64, kBK, 32, 16, kStages, AK, BNC, 4, 2>(p, stream);
      else launch_cx<64, 64, kBK, 32, 32, kStages, AK, BNC, 4, 2>(p, stream);
      break;
  }
}

}  // namespace

int zgemm_algo() {
  int v = g_algo.load();
  if (v < 0) {  // PEPSB_GEMM=4m selects the real-embedding kernels before any option is set
    const char* e = getenv("PEPSB_GEMM");
    v = (e && std::string(e) == "4m") ? kGemm4M : (e && std::string(e) == "4c") ? kGemm4C : kGemm3M;
    g_algo.store(v);
  }
  return v;
}

void zgemm_set_algo(int a) {
  if (a != kGemm4M && a != kGemm3M && a != kGemm4C)
    throw Error(kValidationError, "gemm_algo must be 0 (4M), 1 (3M) or 2 (4M complex fragments)");
  g_algo.store(a);
}

std::atomic<int> g_real{-1};

bool zgemm_real_enabled() {
  int v = g_real.load();
  if (v < 0) {
    const char* e = getenv("PEPSB_GEMM_REAL");
    v = (e && e[0] == '0') ? 0 : 1;
    g_real.store(v);
  }
  return v != 0;
}

void zgemm_set_real(int on) { g_real.store(on ? 1 : 0); }

std::atomic<int> g_cr_cfg{-1};

// 64 x 64 complex x real tile: 1 (default) = 8 warps of 32 x 16 (2 CTAs /
// SM, 16 warps / SM), 0 = 4 warps of 32 x 32 (8 warps / SM); 2 = 8 warps for
// the 4M complex-fragment 64 x 64 tile too (it spills at 128 registers).  ncu on the short-K launches (4 warps): DMMA pipe 63 % active, 12 % of
// the warp slots occupied, stalls per issue wait 2.1 / short scoreboard 0.76;
// the 8-warp tile (128 registers, no spills) hides more of those latencies:
// config-2 row 63.9 -> 61.4 ms, bitwise identical results.
int zgemm_cr_cfg() {
  int v = g_cr_cfg.load();
  if (v < 0) {
    const char* e = getenv("PEPSB_CR_CFG");
    v = e ? std::clamp(std::atoi(e), 0, 2) : 1;
    g_cr_cfg.store(v);
  }
  return v;
}

void zgemm_set_cr_cfg(int v) { g_cr_cfg.store(std::clamp(v, 0, 2)); }

std::atomic<int> g_c3m_cfg{-1};

// 3M warp tiles: 0 = 64x32 / 4 warps, 64x72 / 12, 72x72 / 9; 1 = 64x32 / 8,
// 64x72 / 24, 72x72 / 27 warps.
int zgemm_c3m_cfg() {
  int v = g_c3m_cfg.load();
  if (v < 0) {
    const char* e = getenv("PEPSB_C3M_CFG");
    v = e ? std::clamp(std::atoi(e), 0, 1) : 0;
    g_c3m_cfg.store(v);
  }
  return v;
}

void zgemm_set_c3m_cfg(int v) { g_c3m_cfg.store(std::clamp(v, 0, 1)); }

std::atomic<int> g_stream{-1};

bool zgemm_stream_enabled() {
  int v = g_stream.load();
  if (v < 0) {
    // opt-in: measured slower on the config-2 row (67.1 vs 64.0 ms)
    const char* e = getenv("PEPSB_GEMM_STREAM");
    v = (e && e[0] == '1') ? 1 : 0;
    g_stream.store(v);
  }
  return v != 0;
}

void zgemm_set_stream(int on) { g_stream.store(on ? 1 : 0); }

std::atomic<int> g_small{-1};

bool zgemm_small_enabled() {
  int v = g_small.load();
  if (v < 0) {
    const char* e = getenv("PEPSB_GEMM_SMALL");
    v = (e && e[0] == '0') ? 0 : 1;
    g_small.store(v);
  }
  return v != 0;
}

void zgemm_set_small(int on) { g_small.store(on ? 1 : 0); }

bool zgemm_is_small(const ZgemmParams& p) {
  return zgemm_small_enabled() && p.K <= kSmallMaxK && p.M * p.N * p.batch * std::max<int64_t>(p.K, 1) <= kSmallMaxMacs;
}

int zgemm_ws_mode() {
  int v = g_ws.load();
  if (v < 0) {
    const char* e = getenv("PEPSB_GEMM_WS");
    v = e ? std::atoi(e) : 0;
    if (v < 0 || v > 2) v = 0;
    g_ws.store(v);
  }
  return v;
}

bool zgemm_ws_enabled() { return zgemm_ws_mode() != 0; }

void zgemm_set_ws(int mode) { g_ws.store(mode >= 0 && mode <= 2 ? mode : 0); }

int64_t zgemm_plan_splits(ZgemmParams& p, int num_sms) {
  p.num_sms = num_sms;
  if (zgemm_is_small(p)) {
    p.algo = kGemmSmall;
    p.cfg = 0;
    p.ws = 0;
    p.splits = 1;
    p.kchunk = std::max<int64_t>(p.K, 1);
    return 0;
  }
  // a real operand goes first (complex x real kernel), unless that breaks the
  // 64-wide tiling the kernel has
  const bool cr_ok = zgemm_real_enabled() && (p.realA || p.realB);
  if (cr_ok && !p.realA && !(p.N > 64 && p.N <= 72)) transpose_problem(p);
  if (!(cr_ok && p.realA) && p.M > 64 && p.M <= 72 && p.N > 72) transpose_problem(p);
  p.cfg = choose_cfg(p.M, p.N);
  p.algo = zgemm_algo();
  if (cr_ok && p.realA && p.cfg == 0 && p.algo != kGemm4M) p.algo = kGemmCR;
  if (p.algo != kGemm4M && p.cfg == 4) p.cfg = 0;
  // Short-K problems on the 64-wide tiles are epilogue-heavy: the 4M
  // complex-fragment kernel's 64 x 64 tile (twice the 3M tile) wins there.
  if (p.algo == kGemm3M && p.cfg == 0 && p.K <= 64) p.algo = kGemm4C;
  const TileCfg tc = p.algo == kGemm3M   ? kCfgs3m[p.cfg]
                    : p.algo == kGemmCR ? TileCfg{64, 64}
                    : p.algo == kGemm4C ? kCfgs4c[p.cfg]
                                        : kCfgs[p.cfg];
  int64_t bm = tc.bm, bn = tc.bn;
  p.num_sms = num_sms;
  p.ws = (zgemm_ws_enabled() && p.cfg == 0 && p.algo != kGemm4M && p.algo != kGemmCR && zgemm_ws_eligible(p)) ? 1 : 0;
  if (p.ws) zgemm_ws_tile(p, bm, bn);
  const int64_t tiles = ((p.M + bm - 1) / bm) * ((p.N + bn - 1) / bn) * p.batch;
  // one full wave of resident CTAs (no partial second wave)
  const int64_t target =
      p.ws ? (zgemm_ws_mode() == 2 ? 2 * num_sms : num_sms)
           : static_cast<int64_t>(p.algo == kGemm4M ? ctas_per_sm(p.cfg) : p.algo == kGemmCR ? 2 : ctas_per_sm3m(p.cfg)) *
                 num_sms;
  int64_t splits = 1;
  if (tiles < target && p.K > 4 * kBK) {
    splits = std::min<int64_t>(std::max<int64_t>(1, target / tiles), (p.K + 4 * kBK - 1) / (4 * kBK));
    splits = std::max<int64_t>(1, std::min<int64_t>(splits, 256));
  }
  int64_t kchunk = (p.K + splits - 1) / splits;
  kchunk = ((kchunk + kBK - 1) / kBK) * kBK;
  splits = (p.K + kchunk - 1) / kchunk;
  if (splits < 1) splits = 1;
  p.splits = static_cast<int>(splits);
  p.kchunk = p.K > 0 ? kchunk : kBK;
  return splits > 1 ? splits * p.batch * p.M * p.N : 0;
}

void zgemm_launch(ZgemmParams p, cudaStream_t stream) {
  if (p.M <= 0 || p.N <= 0 || p.batch <= 0) return;
  if (p.kchunk <= 0) p.kchunk = std::max<int64_t>(p.K, 1);
  if (p.cfg < 0 || p.cfg > 4) p.cfg = 0;
  static const bool trace = getenv("PEPSB_TRACE_GEMM") != nullptr;
  if (trace)
    fprintf(stderr, "[zgemm] M=%ld N=%ld K=%ld batch=%ld cfg=%d splits=%d AK=%d BNC=%d conjA=%d conjB=%d algo=%d\n",
            (long)p.M, (long)p.N, (long)p.K, (long)p.batch, p.cfg, p.splits, p.sAk == 1, p.sBj == 1, p.conjA,
            p.conjB, p.algo);
  const bool ak = p.sAk == 1;
  const bool bnc = p.sBj == 1;
  if (p.K == 0) {
    // empty contraction: C = 0 (or unchanged when accumulating)
    p.splits = 1;
  }
  if (p.algo == kGemmSmall) {
    launch_small(p, stream);
  } else if (p.algo == kGemmCR) {
    if (ak && bnc) launch_cr<true, true>(p, stream);
    else if (ak && !bnc) launch_cr<true, false>(p, stream);
    else if (!ak && bnc) launch_cr<false, true>(p, stream);
    else launch_cr<false, false>(p, stream);
  } else if (p.ws && p.K > 0) {
    zgemm_ws_launch(p, p.num_sms, stream);
  } else if (p.algo == kGemm3M) {
    if (p.cfg == 4) p.cfg = 0;
    if (ak && bnc)
      launch_any3m<true, true>(p, stream);
    else if (ak && !bnc)
      launch_any3m<true, false>(p, stream);
    else if (!ak && bnc)
      launch_any3m<false, true>(p, stream);
    else
      launch_any3m<false, false>(p, stream);
  } else if (p.algo == kGemm4C) {
    if (p.cfg == 4) p.cfg = 0;
    if (ak && bnc)
      launch_any4c<true, true>(p, stream);
    else if (ak && !bnc)
      launch_any4c<true, false>(p, stream);
    else if (!ak && bnc)
      launch_any4c<false, true>(p, stream);
    else
      launch_any4c<false, false>(p, stream);
  } else if (ak && bnc)
    launch_any<true, true>(p, stream);
  else if (ak && !bnc)
    launch_any<true, false>(p, stream);
  else if (!ak && bnc)
    launch_any<false, true>(p, stream);
  else
    launch_any<false, false>(p, stream);
  if (p.splits > 1) {
    const int64_t total = p.batch * p.M * p.N;
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>((total + threads - 1) / threads, 148 * 16);
    zgemm_splitk_reduce<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(p);
    PEPSB_LAUNCH();
  }
}

}  // namespace pepsb
