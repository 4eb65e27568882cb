// Hermitian Gram matrix G = Z^H Z of a tall complex matrix Z (rows x k, k <= 72)
// on the FP64 tensor pipe (DMMA.8x8x4), the k x k products that feed every
// orthogonalisation of the randomized SVD (decomposition.cpp:128-193).
//
// With Zh = Z viewed as a real rows x 2k matrix (interleaved re, im), the real
// symmetric C = Zh^T Zh holds every product the complex Gram needs:
//   G_ij = C(2i,2j) + C(2i+1,2j+1) + i (C(2i,2j+1) - C(2i+1,2j)).
// C is symmetric, so block row I only needs the NJ = NB/2 + 1 blocks (I, (I + j)
// mod NB), j = 0 .. NB/2, NB = ceil(2k / 8): every unordered pair of block
// indices is covered (for even NB the pairs at distance NB/2 twice), 180 DMMAs
// per 4 rows at k = 72 against 3 x 81 = 243 for the 3M complex GEMM, and the
// DMMA A and B fragments of Zh^T and Zh are the same shared-memory element
// (row lane&3, column 8 b + lane>>2).  One warp per block row, and EVERY warp
// runs the same instruction stream on its own rotated column list: no
// predicated DMMAs (a predicated-off DMMA still occupies the FP64 pipe: the
// triangular version issued 18 per warp and k-step for 9.5 useful, ncu pipe 69 %
// active at 36 % of the flop rate), no per-row code specialisation (18 code
// paths in flight ran at a third of the speed on instruction fetch), equal DMMA
// counts on the four SM sub-partitions, 20 accumulator registers per thread.
// Split-K over rows: each CTA writes its partial blocks, a second kernel sums
// the partials in a fixed order (the result is deterministic) and a third
// assembles the complex Hermitian G.
#include "gram.cuh"

#include <algorithm>
#include <atomic>
#include <cstdlib>

namespace pepsb {

namespace {

constexpr int kGramBK = 32;       // rows per pipeline stage
constexpr int kGramStages = 4;
constexpr int kGramCtasPerSm = 1;  // resident CTAs per SM the split over rows is sized for
constexpr int kGramLd = 152;      // doubles per smem row (144 + pad: rows alternate bank halves)

__device__ __forceinline__ void cp_async16g(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__host__ __device__ __forceinline__ int gram_nj(int NB) { return NB / 2 + 1; }

template <int NB, int MINB>
__global__ void __launch_bounds__(NB * 32, MINB) gram_partial_kernel(const double2* __restrict__ Z, int64_t rows, int k,
                                                                    int64_t chunk, double* __restrict__ work) {
  constexpr int NT = NB * 32;
  constexpr int NJ = NB / 2 + 1;
  extern __shared__ __align__(16) double gsm[];  // [stages][kGramBK][kGramLd]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t r1 = min(rows, r0 + chunk);
  const int64_t nk = (r1 - r0 + kGramBK - 1) / kGramBK;

  // columns >= 2k of every stage are the zero padding of the last block
  for (int e = tid; e < kGramStages * kGramBK * kGramLd; e += NT) {
    const int c = e % kGramLd;
    if (c >= 2 * k) gsm[e] = 0.0;
  }
  auto load_stage = [&](int slot, int64_t kt) {
    double* S = gsm + slot * kGramBK * kGramLd;
    const int64_t rb = r0 + kt * kGramBK;
    for (int e = tid; e < kGramBK * k; e += NT) {
      const int rr = e / k, cc = e - rr * k;
      const bool ok = rb + rr < r1;
      cp_async16g(S + rr * kGramLd + 2 * cc, ok ? Z + (rb + rr) * k + cc : Z, ok);
    }
  };
#pragma unroll
  for (int s = 0; s < kGramStages - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_commit();
  }

  // block row w: blocks (w, (w + j) mod NB); fragment column offsets in registers
  int coff[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) coff[j] = 8 * ((w + j) % NB);
  double acc[NJ][2];
#pragma unroll
  for (int j = 0; j < NJ; ++j) acc[j][0] = acc[j][1] = 0.0;
  const int frow = lane & 3, fcol = lane >> 2;

  for (int64_t kt = 0; kt < nk; ++kt) {
    cp_wait<kGramStages - 2>();
    __syncthreads();
    {
      const int64_t pf = kt + kGramStages - 1;
      if (pf < nk) load_stage(static_cast<int>(pf % kGramStages), pf);
      cp_commit();
    }
    const double* S = gsm + static_cast<int>(kt % kGramStages) * kGramBK * kGramLd + frow * kGramLd + fcol;
#pragma unroll
    for (int ks = 0; ks < kGramBK / 4; ++ks) {
      const double* Sr = S + ks * 4 * kGramLd;
      const double a0 = Sr[coff[0]];
      dmma(acc[0][0], acc[0][1], a0, a0);
#pragma unroll
      for (int j = 1; j < NJ; ++j) dmma(acc[j][0], acc[j][1], a0, Sr[coff[j]]);
    }
  }
  cp_wait<0>();
  // partial blocks of this CTA: block (w, j) as 8 x 8 row-major doubles;
  // lane owns C[lane>>2][2 (lane&3) + {0,1}] of every block
  double* out = work + (static_cast<int64_t>(blockIdx.x) * NB + w) * NJ * 64;
  const int cr = lane >> 2, cc = 2 * (lane & 3);
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    double* blk = out + j * 64 + cr * 8 + cc;
    blk[0] = acc[j][0];
    blk[1] = acc[j][1];
  }
}

// Sum of the partial triangles over the CTAs in a fixed order: thread (x, y)
// sums parts y, y + 8, ... of entry blockIdx.x * 32 + x, then the 8 partial
// sums are added in y order.  Deterministic.
__global__ void __launch_bounds__(256) gram_reduce_kernel(const double* __restrict__ work, int nparts, int nentries,
                                                          double* __restrict__ red) {
  __shared__ double part[8][33];
  const int e = blockIdx.x * 32 + threadIdx.x;
  double s = 0.0;
  if (e < nentries)
    for (int p = threadIdx.y; p < nparts; p += 8) s += work[static_cast<int64_t>(p) * nentries + e];
  part[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && e < nentries) {
    double t = part[0][threadIdx.x];
#pragma unroll
    for (int y = 1; y < 8; ++y) t += part[y][threadIdx.x];
    red[e] = t;
  }
}

// C(a, b) of the symmetric product from the rotated block rows: block (I, J) is
// stored in row I when (J - I) mod NB <= NB/2, else as the transpose in row J.
__device__ __forceinline__ double csym(const double* red, int NB, int a, int b) {
  const int NJ = gram_nj(NB);
  int I = a >> 3, J = b >> 3;
  int dj = J - I;
  if (dj < 0) dj += NB;
  if (dj >= NJ) {
    dj = NB - dj;
    int t = I;
    I = J;
    J = t;
    t = a;
    a = b;
    b = t;
  }
  return red[(I * NJ + dj) * 64 + (a & 7) * 8 + (b & 7)];
}

__global__ void gram_assemble_kernel(const double* __restrict__ red, int k, int NB, double2* __restrict__ G) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k * k; e += gridDim.x * blockDim.x) {
    const int i = e / k, j = e - i * k;
    const int a = min(i, j), b = max(i, j);
    const double re = csym(red, NB, 2 * a, 2 * b) + csym(red, NB, 2 * a + 1, 2 * b + 1);
    const double im = a == b ? 0.0 : csym(red, NB, 2 * a, 2 * b + 1) - csym(red, NB, 2 * a + 1, 2 * b);
    G[e] = make_double2(re, i <= j ? im : -im);
  }
}

template <int NB>
void launch_partial(const double2* Z, int64_t rows, int k, int64_t chunk, int nparts, double* work,
                    cudaStream_t stream) {
  constexpr int NT = NB * 32;
  constexpr int MINB = kGramCtasPerSm;
  const size_t smem = static_cast<size_t>(kGramStages) * kGramBK * kGramLd * sizeof(double);
  static bool attr = false;
  if (!attr) {
    PEPSB_CUDA(cudaFuncSetAttribute(gram_partial_kernel<NB, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
    attr = true;
  }
  gram_partial_kernel<NB, MINB><<<nparts, NT, smem, stream>>>(Z, rows, k, chunk, work);
  PEPSB_LAUNCH();
}

}  // namespace

namespace {
std::atomic<int> g_gram{-1};
}  // namespace

bool gram_enabled() {
  int v = g_gram.load();
  if (v < 0) {
    // on by default since the rotated-row kernel (config-2 row 59.7 -> 57.7 ms,
    // config-5 row 314 -> 304 ms against the 3M split-K GEMM); PEPSB_GEMM_GRAM=0 turns it off
    const char* e = getenv("PEPSB_GEMM_GRAM");
    v = (e && e[0] == '0') ? 0 : 1;
    g_gram.store(v);
  }
  return v != 0;
}

void gram_set_enabled(int on) { g_gram.store(on ? 1 : 0); }

bool gram_herk_eligible(int64_t rows, int64_t k) { return k >= 1 && k <= kGramMaxK && rows >= kGramMinRows; }

int64_t gram_herk_workspace(int64_t rows, int64_t k, int num_sms) {
  const int NB = static_cast<int>((2 * k + 7) / 8);
  const int64_t nparts = std::min<int64_t>(static_cast<int64_t>(kGramCtasPerSm) * num_sms, (rows + 63) / 64);
  return (nparts + 1) * NB * gram_nj(NB) * 64;  // doubles: partial blocks + their sum
}

void gram_herk(const double2* Z, int64_t rows, int k, double2* G, double* work, int num_sms, cudaStream_t stream) {
  const int NB = (2 * k + 7) / 8;
  const int64_t nparts = std::min<int64_t>(static_cast<int64_t>(kGramCtasPerSm) * num_sms, (rows + 63) / 64);
  int64_t chunk = (rows + nparts - 1) / nparts;
  chunk = ((chunk + kGramBK - 1) / kGramBK) * kGramBK;
  const int np = static_cast<int>((rows + chunk - 1) / chunk);
  switch (NB) {
#define PEPSB_GRAM_CASE(n) \
  case n: launch_partial<n>(Z, rows, k, chunk, np, work, stream); break;
    PEPSB_GRAM_CASE(1) PEPSB_GRAM_CASE(2) PEPSB_GRAM_CASE(3) PEPSB_GRAM_CASE(4) PEPSB_GRAM_CASE(5)
    PEPSB_GRAM_CASE(6) PEPSB_GRAM_CASE(7) PEPSB_GRAM_CASE(8) PEPSB_GRAM_CASE(9) PEPSB_GRAM_CASE(10)
    PEPSB_GRAM_CASE(11) PEPSB_GRAM_CASE(12) PEPSB_GRAM_CASE(13) PEPSB_GRAM_CASE(14) PEPSB_GRAM_CASE(15)
    PEPSB_GRAM_CASE(16) PEPSB_GRAM_CASE(17) PEPSB_GRAM_CASE(18)
#undef PEPSB_GRAM_CASE
    default: throw Error(kShapeError, "gram_herk: k > 72");
  }
  const int nentries = NB * gram_nj(NB) * 64;
  double* red = work + static_cast<int64_t>(np) * nentries;
  gram_reduce_kernel<<<(nentries + 31) / 32, dim3(32, 8), 0, stream>>>(work, np, nentries, red);
  PEPSB_LAUNCH();
  const int threads = 256;
  const int blocks = std::max(1, std::min(148, (k * k + threads - 1) / threads));
  gram_assemble_kernel<<<blocks, threads, 0, stream>>>(red, k, NB, G);
  PEPSB_LAUNCH();
}

}  // namespace pepsb
