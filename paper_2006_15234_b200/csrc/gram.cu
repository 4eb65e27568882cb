// Hermitian Gram matrix G = Z^H Z of a tall complex matrix Z (rows x k, k <= 72)
// on the FP64 tensor pipe (DMMA.8x8x4), the k x k products that feed every
// orthogonalisation of the randomized SVD (decomposition.cpp:128-193).
//
// With Zh = Z viewed as a real rows x 2k matrix (interleaved re, im), the real
// symmetric C = Zh^T Zh holds every product the complex Gram needs:
//   G_ij = C(2i,2j) + C(2i+1,2j+1) + i (C(2i,2j+1) - C(2i+1,2j)).
// Only the upper triangle of 8 x 8 blocks of C is computed: NB (NB+1) / 2
// blocks for NB = ceil(2k / 8), i.e. 171 DMMAs per 4 rows at k = 72 against
// 3 x 81 = 243 for the 3M complex GEMM (0.70x the executed flops), and the
// DMMA A and B fragments of Zh^T and Zh are the same shared-memory element
// (row lane&3, column 8 b + lane>>2), so one fragment load serves both roles.
// Warp w owns block rows w and NB-1-w (NB+1 blocks), so the triangle splits
// evenly over ceil(NB/2) warps.  Split-K over rows: each CTA writes its
// partial triangle, a second kernel sums the partials in a fixed order (the
// result is deterministic) and assembles the complex Hermitian G.
#include "gram.cuh"

#include <algorithm>
#include <atomic>
#include <cstdlib>

namespace pepsb {

namespace {

constexpr int kGramBK = 16;       // rows per pipeline stage
constexpr int kGramStages = 3;
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

// Block (I, J), I <= J, of the NB x NB triangle -> its index in the packed list.
__host__ __device__ __forceinline__ int tri_index(int I, int J, int NB) { return I * NB - I * (I - 1) / 2 + (J - I); }

template <int NB>
__global__ void __launch_bounds__(((NB + 1) / 2) * 32) gram_partial_kernel(const double2* __restrict__ Z, int64_t rows,
                                                                        int k, int64_t chunk, double* __restrict__ work) {
  constexpr int NW = (NB + 1) / 2;
  constexpr int NT = NW * 32;
  constexpr int NTRI = NB * (NB + 1) / 2;
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

  const int I0 = w, I1 = NB - 1 - w;  // this warp's two block rows (I0 == I1 for the middle row of odd NB)
  double acc0[NB][2], acc1[NB][2];
#pragma unroll
  for (int j = 0; j < NB; ++j) acc0[j][0] = acc0[j][1] = acc1[j][0] = acc1[j][1] = 0.0;
  const int frow = lane & 3, fcol = lane >> 2;

  for (int64_t kt = 0; kt < nk; ++kt) {
    cp_wait<kGramStages - 2>();
    __syncthreads();
    {
      const int64_t pf = kt + kGramStages - 1;
      if (pf < nk) load_stage(static_cast<int>(pf % kGramStages), pf);
      cp_commit();
    }
    const double* S = gsm + static_cast<int>(kt % kGramStages) * kGramBK * kGramLd;
#pragma unroll
    for (int ks = 0; ks < kGramBK / 4; ++ks) {
      const double* Sr = S + (ks * 4 + frow) * kGramLd + fcol;
      const double a0 = Sr[8 * I0], a1 = Sr[8 * I1];
#pragma unroll
      for (int J = 0; J < NB; ++J) {
        if (J < I0) continue;  // warp-uniform
        const double b = Sr[8 * J];
        dmma(acc0[J][0], acc0[J][1], a0, b);
        if (I1 != I0 && J >= I1) dmma(acc1[J][0], acc1[J][1], a1, b);
      }
    }
  }
  cp_wait<0>();
  // partial triangle of this CTA: block (I, J) as 8 x 8 row-major doubles;
  // lane owns C[lane>>2][2 (lane&3) + {0,1}] of every block
  double* out = work + static_cast<int64_t>(blockIdx.x) * NTRI * 64;
  const int cr = lane >> 2, cc = 2 * (lane & 3);
#pragma unroll
  for (int J = 0; J < NB; ++J) {
    if (J >= I0) {
      double* blk = out + tri_index(I0, J, NB) * 64 + cr * 8 + cc;
      blk[0] = acc0[J][0];
      blk[1] = acc0[J][1];
    }
    if (I1 != I0 && J >= I1) {
      double* blk = out + tri_index(I1, J, NB) * 64 + cr * 8 + cc;
      blk[0] = acc1[J][0];
      blk[1] = acc1[J][1];
    }
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

__device__ __forceinline__ double csym(const double* red, int NB, int a, int b) {
  if (a > b) {
    const int t = a;
    a = b;
    b = t;
  }
  return red[tri_index(a >> 3, b >> 3, NB) * 64 + (a & 7) * 8 + (b & 7)];
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
  constexpr int NT = ((NB + 1) / 2) * 32;
  const size_t smem = static_cast<size_t>(kGramStages) * kGramBK * kGramLd * sizeof(double);
  static bool attr = false;
  if (!attr) {
    PEPSB_CUDA(cudaFuncSetAttribute(gram_partial_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
    attr = true;
  }
  gram_partial_kernel<NB><<<nparts, NT, smem, stream>>>(Z, rows, k, chunk, work);
  PEPSB_LAUNCH();
}

}  // namespace

namespace {
std::atomic<int> g_gram{-1};
}  // namespace

bool gram_enabled() {
  int v = g_gram.load();
  if (v < 0) {
    // opt-in: measured slower in the row than the 3M split-K GEMM it replaces
    // (config-2 row 60.4 vs 60.9 ms, config-5 row 318 vs 321 ms)
    const char* e = getenv("PEPSB_GEMM_GRAM");
    v = (e && e[0] == '1') ? 1 : 0;
    g_gram.store(v);
  }
  return v != 0;
}

void gram_set_enabled(int on) { g_gram.store(on ? 1 : 0); }

bool gram_herk_eligible(int64_t rows, int64_t k) { return k >= 1 && k <= kGramMaxK && rows >= kGramMinRows; }

int64_t gram_herk_workspace(int64_t rows, int64_t k, int num_sms) {
  const int NB = static_cast<int>((2 * k + 7) / 8);
  const int64_t nparts = std::min<int64_t>(num_sms, (rows + 255) / 256);
  return (nparts + 1) * NB * (NB + 1) / 2 * 64;  // doubles: partial triangles + their sum
}

void gram_herk(const double2* Z, int64_t rows, int k, double2* G, double* work, int num_sms, cudaStream_t stream) {
  const int NB = (2 * k + 7) / 8;
  const int64_t nparts = std::min<int64_t>(num_sms, (rows + 255) / 256);
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
  const int nentries = NB * (NB + 1) / 2 * 64;
  double* red = work + static_cast<int64_t>(np) * nentries;
  gram_reduce_kernel<<<(nentries + 31) / 32, dim3(32, 8), 0, stream>>>(work, np, nentries, red);
  PEPSB_LAUNCH();
  const int threads = 256;
  const int blocks = std::max(1, std::min(148, (k * k + threads - 1) / threads));
  gram_assemble_kernel<<<blocks, threads, 0, stream>>>(red, k, NB, G);
  PEPSB_LAUNCH();
}

}  // namespace pepsb
