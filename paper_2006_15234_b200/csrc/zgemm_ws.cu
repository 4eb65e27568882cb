// Persistent, warp-specialised complex-FP64 DMMA GEMM with TMA operand
// staging (see zgemm.cuh).
//
// One CTA per SM loops over the 64 x 64 output tiles of the problem (m
// fastest, so the CTAs resident at any time share their B tiles in L2).
// Warp roles:
//   * one producer warp: lane 0 streams the operand tiles of every k-step into
//     a STAGES-deep shared-memory ring with tensor-map TMA loads
//     (cp.async.bulk.tensor, SASS UTMALDG; completion counted on the stage's
//     mbarrier with expect_tx), out-of-bounds rows / columns / K tails
//     zero-filled by the TMA unit; the warp also decodes the epilogue's
//     mixed-radix row / column offsets of each tile into a double-buffered
//     table and runs ahead across tile boundaries;
//   * 8 consumer warps (32 x 16 each) wait on the stage's "full" barrier, run
//     LDS.128 + DMMA.8x8x4 only, release the stage on its "empty" barrier and
//     scatter the finished tile straight into the next contraction's layout
//     while the producer is already loading the next tile.
// Shared-memory layouts (no padding: TMA writes dense boxes), all conflict-free
// for the quarter-warp LDS.128 pattern of the m8n8k4 fragments:
//   * operand contiguous along k: k-blocked [k/4][rows][4] (box 4 k x 64 rows);
//     the 8 lanes of a quarter warp read 2 rows x 4 k = 128 contiguous bytes;
//   * operand contiguous along its row / column index: [chunk of 8][16 k][8]
//     with the 128-byte swizzle (box 8 x 16 k); the fragment slots are mapped
//     to rows / columns by pi(s) = s/2 + 4 (s&1), which puts a quarter warp's
//     8 LDS.128 in 8 distinct bank groups; the epilogue applies the same pi.
// The complex schemes are those of zgemm_cx_kernel (zgemm.cu): ALG 4 = 4M with
// complex fragments (CUTLASS z884 scheme), ALG 3 = 3M / Gauss; per accumulator
// the DMMAs run in the same k order, so results are bitwise those of the
// classic kernel.  Requirements (zgemm_ws_eligible): each operand has a unit
// stride along one matrix index, at most 3 batch modes.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstring>

#include "zgemm.cuh"

namespace pepsb {

namespace {

constexpr int kBKw = 16;  // complex k per stage
constexpr int kStagesW = 4;
constexpr int kThreadsW = 8 * 32;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT;\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
template <int N>
__device__ __forceinline__ void reg_alloc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(N)); }
template <int N>
__device__ __forceinline__ void reg_dealloc() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(N)); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }

// TMA tile load of up to 5 coordinates (unused trailing coordinates are 0 and
// the map's rank decides how many the unit reads).
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* map, int rank, const int* c, uint64_t* bar) {
  const uint64_t m = reinterpret_cast<uint64_t>(map);
  const uint32_t d = su32(dst), b = su32(bar);
  switch (rank) {
    case 2:
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(d),
          "l"(m), "r"(c[0]), "r"(c[1]), "r"(b)
          : "memory");
      break;
    case 3:
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(d),
          "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(b)
          : "memory");
      break;
    case 4:
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(d),
          "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(b)
          : "memory");
      break;
    default:
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(d),
          "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(b)
          : "memory");
      break;
  }
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ int64_t decode_off(int64_t idx, int n, const int64_t* ext, const int64_t* str) {
  int64_t off = 0;
  for (int a = n - 1; a >= 0; --a) {
    const int64_t e = ext[a];
    const int64_t q = idx / e;
    off += (idx - q * e) * str[a];
    idx = q;
  }
  return off;
}

// fragment slot -> row / column inside an 8-block for the swizzled layouts
__host__ __device__ __forceinline__ int pi8(int s) { return (s >> 1) + 4 * (s & 1); }

// Per-operand TMA description: map rank and which batch modes it carries.
struct TmaOperand {
  int rank = 2;
  int nbm = 0;           // batch modes with a nonzero stride (map dims 2..)
  int bmode[3] = {};     // their indices into ZgemmParams::bext
};

struct WorkItem {
  int64_t m0, n0, offC, kbeg, kend;
  int split, bz;
};

__device__ __forceinline__ WorkItem decode_work(const ZgemmParams& p, int64_t w, int64_t mtiles, int64_t tiles,
                                                int BM, int BN) {
  WorkItem it;
  const int64_t tile = w % tiles;
  const int64_t rest = w / tiles;
  it.split = static_cast<int>(rest % p.splits);
  it.bz = static_cast<int>(rest / p.splits);
  it.m0 = (tile % mtiles) * BM;
  it.n0 = (tile / mtiles) * BN;
  it.offC = 0;
  int64_t idx = it.bz;
  for (int a = p.nb - 1; a >= 0; --a) {
    const int64_t e = p.bext[a];
    const int64_t q = idx / e;
    it.offC += (idx - q * e) * p.bsC[a];
    idx = q;
  }
  it.kbeg = static_cast<int64_t>(it.split) * p.kchunk;
  it.kend = min(p.K, it.kbeg + p.kchunk);
  return it;
}

struct WsArgs {
  ZgemmParams p;
  TmaOperand oa, ob;
  int64_t nwork;
};

// Producer state: the next k-tile to load (work item w, k-tile kt) and its ring slot.
struct ProdCursor {
  int64_t w, kt, nk, m0, n0;
  int k0base;
  int ca[5], cb[5];
  int stage;
  uint32_t phase;
};

__device__ __forceinline__ void cursor_item(ProdCursor& c, const WsArgs& args, int64_t mtiles, int64_t tiles, int BM,
                                            int BN) {
  const ZgemmParams& p = args.p;
  if (c.w >= args.nwork) return;
  const WorkItem it = decode_work(p, c.w, mtiles, tiles, BM, BN);
  c.m0 = it.m0;
  c.n0 = it.n0;
  c.k0base = static_cast<int>(it.kbeg);
  c.nk = (it.kend - it.kbeg + kBKw - 1) / kBKw;
  c.kt = 0;
  int64_t idx = it.bz;
  int bidx[4] = {0, 0, 0, 0};
#pragma unroll
  for (int a = 3; a >= 0; --a) {
    if (a >= p.nb) continue;
    const int64_t q = idx / p.bext[a];
    bidx[a] = static_cast<int>(idx - q * p.bext[a]);
    idx = q;
  }
  auto sel = [&](int m) { return m == 0 ? bidx[0] : m == 1 ? bidx[1] : m == 2 ? bidx[2] : bidx[3]; };
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    c.ca[2 + u] = u < args.oa.nbm ? sel(args.oa.bmode[u]) : 0;
    c.cb[2 + u] = u < args.ob.nbm ? sel(args.ob.bmode[u]) : 0;
  }
}

template <int BM, int BN, int WM, int WN, bool AK, bool BNC, int ALG>
__global__ void __launch_bounds__(kThreadsW, 1)
    zgemm_ws_kernel(const __grid_constant__ WsArgs args, const __grid_constant__ CUtensorMap tmA,
                    const __grid_constant__ CUtensorMap tmB) {
  constexpr int STAGES = kStagesW;
  constexpr int NW = (BM / WM) * (BN / WN);  // warps (all compute; warp 0 lane 0 also issues the TMA loads)
  static_assert(NW * 32 == kThreadsW, "8 warps");
  constexpr int FM = WM / 8, FN = WN / 8;
  constexpr int NACC = ALG == 3 ? 3 : 2;
  constexpr int KS = kBKw / 4;
  constexpr int A_ELEMS = BM * kBKw, STAGE = A_ELEMS + kBKw * BN;  // double2
  constexpr uint32_t STAGE_BYTES = STAGE * 16;
  const ZgemmParams& p = args.p;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // the 128-byte swizzle needs 1024-byte aligned destinations
  double2* ring = reinterpret_cast<double2*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  int64_t* rowtab = reinterpret_cast<int64_t*>(empty + STAGES);  // [2][BM]
  int64_t* coltab = rowtab + 2 * BM;                             // [2][BN]
  // producer cursor in shared memory: only thread 0 touches it, and keeping it
  // out of the registers every thread allocates leaves them to the accumulators
  ProdCursor& pc = *reinterpret_cast<ProdCursor*>(coltab + 2 * BN);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t mtiles = (p.M + BM - 1) / BM;
  const int64_t tiles = mtiles * ((p.N + BN - 1) / BN);
  const int64_t nwork = args.nwork;
  const bool producer = threadIdx.x == 0;

  if (producer) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // ---- producer (thread 0): keeps the ring STAGES - 1 k-tiles ahead, across tiles
  if (producer) {
    pc.w = blockIdx.x;
    pc.stage = 0;
    pc.phase = 0;
    pc.ca[0] = pc.ca[1] = pc.cb[0] = pc.cb[1] = 0;
    cursor_item(pc, args, mtiles, tiles, BM, BN);
  }
  auto produce = [&]() {
    if (pc.w >= nwork) return;
    mbar_wait(&empty[pc.stage], pc.phase ^ 1u);
    double2* As = ring + pc.stage * STAGE;
    double2* Bs = As + A_ELEMS;
    uint64_t* bar = &full[pc.stage];
    const int k0 = pc.k0base + static_cast<int>(pc.kt) * kBKw;
    mbar_arrive_tx(bar, STAGE_BYTES);
    if (AK) {  // [k/4][BM][4]: one box of 4 k x BM rows per k-block
#pragma unroll
      for (int j = 0; j < kBKw / 4; ++j) {
        pc.ca[0] = 2 * (k0 + 4 * j);
        pc.ca[1] = static_cast<int>(pc.m0);
        tma_load(As + j * BM * 4, &tmA, args.oa.rank, pc.ca, bar);
      }
    } else {  // [BM/8][16 k][8], 128-byte swizzle
#pragma unroll 4
      for (int c = 0; c < BM / 8; ++c) {
        pc.ca[0] = static_cast<int>(2 * (pc.m0 + 8 * c));
        pc.ca[1] = k0;
        tma_load(As + c * kBKw * 8, &tmA, args.oa.rank, pc.ca, bar);
      }
    }
    if (BNC) {  // [BN/8][16 k][8], 128-byte swizzle
#pragma unroll 4
      for (int c = 0; c < BN / 8; ++c) {
        pc.cb[0] = static_cast<int>(2 * (pc.n0 + 8 * c));
        pc.cb[1] = k0;
        tma_load(Bs + c * kBKw * 8, &tmB, args.ob.rank, pc.cb, bar);
      }
    } else {  // [k/4][BN][4]
#pragma unroll
      for (int j = 0; j < kBKw / 4; ++j) {
        pc.cb[0] = 2 * (k0 + 4 * j);
        pc.cb[1] = static_cast<int>(pc.n0);
        tma_load(Bs + j * BN * 4, &tmB, args.ob.rank, pc.cb, bar);
      }
    }
    if (++pc.stage == STAGES) {
      pc.stage = 0;
      pc.phase ^= 1u;
    }
    if (++pc.kt == pc.nk) {
      pc.w += gridDim.x;
      cursor_item(pc, args, mtiles, tiles, BM, BN);
    }
  };
  if (producer)
    for (int s = 0; s < STAGES - 1; ++s) produce();

  // ---- all warps compute
  const int wm0 = (warp % (BM / WM)) * WM;
  const int wn0 = (warp / (BM / WM)) * WN;
  const int kq = lane & 3, rq = lane >> 2;
  const long long sga = p.conjA ? (long long)0x8000000000000000ULL : 0LL;
  const long long sgb = p.conjB ? (long long)0x8000000000000000ULL : 0LL;
  auto flip = [](double v, long long m) { return __longlong_as_double(__double_as_longlong(v) ^ m); };
  // per-lane fragment base offsets (double2) inside a stage; block a / b adds a constant
  const int abase = AK ? (wm0 + rq) * 4 + kq : (wm0 / 8) * kBKw * 8;
  const int bbase = BNC ? A_ELEMS + (wn0 / 8) * kBKw * 8 : A_ELEMS + (wn0 + rq) * 4 + kq;
  constexpr int ASTEP = AK ? 32 : kBKw * 8, BSTEP = BNC ? kBKw * 8 : 32;
  const int pr = pi8(rq);

  double acc[FM][FN][NACC][2];
  double2 fa[2][FM], fb[2][FN];
  auto load_frags = [&](int buf, const double2* St, int ks) {
    const int k = ks * 4 + kq;
    const int sw = (pr ^ (k & 7));
#pragma unroll
    for (int a = 0; a < FM; ++a)
      fa[buf][a] = AK ? St[abase + a * ASTEP + ks * BM * 4] : St[abase + a * ASTEP + k * 8 + sw];
#pragma unroll
    for (int b = 0; b < FN; ++b)
      fb[buf][b] = BNC ? St[bbase + b * BSTEP + k * 8 + sw] : St[bbase + b * BSTEP + ks * BN * 4];
  };
  auto compute = [&](int buf) {
    if constexpr (ALG == 3) {
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
        for (int b = 0; b < FN; ++b) dmma(acc[a][b][0][0], acc[a][b][0][1], ar[a], br[b]);
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) dmma(acc[a][b][1][0], acc[a][b][1][1], ai[a], bi[b]);
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) dmma(acc[a][b][2][0], acc[a][b][2][1], as[a], bs[b]);
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
          dmma(acc[a][b][0][0], acc[a][b][0][1], fa[buf][a].x, fb[buf][b].x);
          dmma(acc[a][b][1][0], acc[a][b][1][1], fa[buf][a].x, bi[b]);
        }
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) {
          dmma(acc[a][b][0][0], acc[a][b][0][1], nai[a], bi[b]);
          dmma(acc[a][b][1][0], acc[a][b][1][1], ai[a], fb[buf][b].x);
        }
    }
  };

  int stage = 0;
  uint32_t phase = 0;
  int64_t t = 0;
  for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x, ++t) {
    const WorkItem it = decode_work(p, w, mtiles, tiles, BM, BN);
    const int64_t nk = (it.kend - it.kbeg + kBKw - 1) / kBKw;
    const int buf = static_cast<int>(t & 1);
    // epilogue offsets of this tile (table[buf] was last read two tiles ago,
    // before the barrier that precedes the previous tile's epilogue)
    if (p.splits == 1) {
      for (int e = threadIdx.x; e < BM + BN; e += kThreadsW) {
        if (e < BM) {
          const int64_t gi = it.m0 + e;
          rowtab[buf * BM + e] = gi < p.M ? decode_off(gi, p.nr, p.rext, p.rstr) : 0;
        } else {
          const int64_t gj = it.n0 + e - BM;
          coltab[buf * BN + e - BM] = gj < p.N ? decode_off(gj, p.nc, p.cext, p.cstr) : 0;
        }
      }
    }
#pragma unroll
    for (int a = 0; a < FM; ++a)
#pragma unroll
      for (int b = 0; b < FN; ++b)
#pragma unroll
        for (int q = 0; q < NACC; ++q) acc[a][b][q][0] = acc[a][b][q][1] = 0.0;
    for (int64_t kt = 0; kt < nk; ++kt) {
      if (producer) produce();
      __syncwarp();
      mbar_wait(&full[stage], phase);
      const double2* St = ring + stage * STAGE;
      load_frags(0, St, 0);
#pragma unroll
      for (int ks = 0; ks < KS; ks += 2) {
        load_frags(1, St, ks + 1);
        compute(0);
        if (ks + 2 < KS) load_frags(0, St, ks + 2);
        compute(1);
      }
      // the DMMAs above consumed every fragment of this stage: release it
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1u;
      }
    }
    __syncthreads();  // offset table of this tile complete
    // epilogue: lane owns C[row(a)][col(b, h)] of every block
#pragma unroll
    for (int a = 0; a < FM; ++a) {
      const int li = wm0 + a * 8 + (AK ? rq : pr);
      if (it.m0 + li >= p.M) continue;
      const int64_t ro = p.splits == 1 ? rowtab[buf * BM + li] : 0;
#pragma unroll
      for (int b = 0; b < FN; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int lj = wn0 + b * 8 + (BNC ? pi8(2 * kq + h) : 2 * kq + h);
          if (it.n0 + lj >= p.N) continue;
          double2 v;
          if constexpr (ALG == 3) {
            const double p1 = acc[a][b][0][h], p2 = acc[a][b][1][h], p3 = acc[a][b][2][h];
            v = make_double2(p1 - p2, p3 - p1 - p2);
          } else {
            v = make_double2(acc[a][b][0][h], acc[a][b][1][h]);
          }
          if (p.splits == 1) {
            double2* dst = p.C + it.offC + ro + coltab[buf * BN + lj];
            if (p.accumulate) v = cadd(*dst, v);
            *dst = v;
          } else {
            double2* W = p.work + ((static_cast<int64_t>(it.split) * p.batch + it.bz) * p.M) * p.N;
            W[(it.m0 + li) * p.N + it.n0 + lj] = v;
          }
        }
    }
  }
}

// Non-persistent TMA variant with the classic kernels' structure: one output
// tile per CTA, 4 warps, 2 CTAs per SM (so one CTA's prologue / epilogue
// overlaps the other's main loop), thread 0 issuing the tensor-map loads of
// stage kt + STAGES - 1 right after the per-k-tile barrier that frees its
// slot; consumers wait on the stage's full mbarrier.  No global address
// arithmetic in the loop, K tails and ragged edges zero-filled by the TMA unit.
template <int BM, int BN, int WM, int WN, int STAGES, bool AK, bool BNC, int ALG>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32, 2)
    zgemm_tma_kernel(const __grid_constant__ WsArgs args, const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmB) {
  constexpr int NT = (BM / WM) * (BN / WN) * 32;
  constexpr int FM = WM / 8, FN = WN / 8;
  constexpr int NACC = ALG == 3 ? 3 : 2;
  constexpr int KS = kBKw / 4;
  constexpr int A_ELEMS = BM * kBKw, STAGE = A_ELEMS + kBKw * BN;  // double2
  constexpr uint32_t STAGE_BYTES = STAGE * 16;
  const ZgemmParams& p = args.p;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  double2* ring = reinterpret_cast<double2*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + STAGES * STAGE);
  int64_t* rowoff = reinterpret_cast<int64_t*>(full + STAGES);
  int64_t* coloff = rowoff + BM;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t mtiles = (p.M + BM - 1) / BM;
  const int64_t tile = blockIdx.x;
  const int64_t m0 = (tile % mtiles) * BM, n0 = (tile / mtiles) * BN;
  const int bz = static_cast<int>(blockIdx.y / p.splits), split = static_cast<int>(blockIdx.y % p.splits);
  const int64_t kbeg = static_cast<int64_t>(split) * p.kchunk;
  const int64_t kend = min(p.K, kbeg + p.kchunk);
  const int nk = static_cast<int>((kend - kbeg + kBKw - 1) / kBKw);

  int ca[5] = {0, 0, 0, 0, 0}, cb[5] = {0, 0, 0, 0, 0};
  int64_t offC = 0;
  {
    int64_t idx = bz;
    int bidx[4] = {0, 0, 0, 0};
#pragma unroll
    for (int a = 3; a >= 0; --a) {
      if (a >= p.nb) continue;
      const int64_t q = idx / p.bext[a];
      bidx[a] = static_cast<int>(idx - q * p.bext[a]);
      offC += bidx[a] * p.bsC[a];
      idx = q;
    }
    auto sel = [&](int m) { return m == 0 ? bidx[0] : m == 1 ? bidx[1] : m == 2 ? bidx[2] : bidx[3]; };
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      if (u < args.oa.nbm) ca[2 + u] = sel(args.oa.bmode[u]);
      if (u < args.ob.nbm) cb[2 + u] = sel(args.ob.bmode[u]);
    }
  }
  auto issue = [&](int kt) {
    const int slot = kt % STAGES;
    double2* As = ring + slot * STAGE;
    double2* Bs = As + A_ELEMS;
    uint64_t* bar = &full[slot];
    const int k0 = static_cast<int>(kbeg) + kt * kBKw;
    mbar_arrive_tx(bar, STAGE_BYTES);
    if (AK) {
#pragma unroll
      for (int j = 0; j < kBKw / 4; ++j) {
        ca[0] = 2 * (k0 + 4 * j);
        ca[1] = static_cast<int>(m0);
        tma_load(As + j * BM * 4, &tmA, args.oa.rank, ca, bar);
      }
    } else {
#pragma unroll
      for (int c = 0; c < BM / 8; ++c) {
        ca[0] = static_cast<int>(2 * (m0 + 8 * c));
        ca[1] = k0;
        tma_load(As + c * kBKw * 8, &tmA, args.oa.rank, ca, bar);
      }
    }
    if (BNC) {
#pragma unroll
      for (int c = 0; c < BN / 8; ++c) {
        cb[0] = static_cast<int>(2 * (n0 + 8 * c));
        cb[1] = k0;
        tma_load(Bs + c * kBKw * 8, &tmB, args.ob.rank, cb, bar);
      }
    } else {
#pragma unroll
      for (int j = 0; j < kBKw / 4; ++j) {
        cb[0] = 2 * (k0 + 4 * j);
        cb[1] = static_cast<int>(n0);
        tma_load(Bs + j * BN * 4, &tmB, args.ob.rank, cb, bar);
      }
    }
  };
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    for (int kt = 0; kt < STAGES - 1 && kt < nk; ++kt) issue(kt);
  }
  if (p.splits == 1) {
    for (int r = tid; r < BM; r += NT) rowoff[r] = m0 + r < p.M ? decode_off(m0 + r, p.nr, p.rext, p.rstr) : 0;
    for (int c = tid; c < BN; c += NT) coloff[c] = n0 + c < p.N ? decode_off(n0 + c, p.nc, p.cext, p.cstr) : 0;
  }
  __syncthreads();

  const int wm0 = (warp % (BM / WM)) * WM, wn0 = (warp / (BM / WM)) * WN;
  const int kq = lane & 3, rq = lane >> 2;
  const long long sga = p.conjA ? (long long)0x8000000000000000ULL : 0LL;
  const long long sgb = p.conjB ? (long long)0x8000000000000000ULL : 0LL;
  auto flip = [](double v, long long m) { return __longlong_as_double(__double_as_longlong(v) ^ m); };
  const int abase = AK ? (wm0 + rq) * 4 + kq : (wm0 / 8) * kBKw * 8;
  const int bbase = BNC ? A_ELEMS + (wn0 / 8) * kBKw * 8 : A_ELEMS + (wn0 + rq) * 4 + kq;
  constexpr int ASTEP = AK ? 32 : kBKw * 8, BSTEP = BNC ? kBKw * 8 : 32;
  const int pr = pi8(rq);
  double acc[FM][FN][NACC][2];
#pragma unroll
  for (int a = 0; a < FM; ++a)
#pragma unroll
    for (int b = 0; b < FN; ++b)
#pragma unroll
      for (int q = 0; q < NACC; ++q) acc[a][b][q][0] = acc[a][b][q][1] = 0.0;
  double2 fa[2][FM], fb[2][FN];
  auto load_frags = [&](int buf, const double2* St, int ks) {
    const int k = ks * 4 + kq;
    const int sw = (pr ^ (k & 7));
#pragma unroll
    for (int a = 0; a < FM; ++a)
      fa[buf][a] = AK ? St[abase + a * ASTEP + ks * BM * 4] : St[abase + a * ASTEP + k * 8 + sw];
#pragma unroll
    for (int b = 0; b < FN; ++b)
      fb[buf][b] = BNC ? St[bbase + b * BSTEP + k * 8 + sw] : St[bbase + b * BSTEP + ks * BN * 4];
  };
  auto compute = [&](int buf) {
    if constexpr (ALG == 3) {
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
        for (int b = 0; b < FN; ++b) dmma(acc[a][b][0][0], acc[a][b][0][1], ar[a], br[b]);
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) dmma(acc[a][b][1][0], acc[a][b][1][1], ai[a], bi[b]);
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) dmma(acc[a][b][NACC - 1][0], acc[a][b][NACC - 1][1], as[a], bs[b]);
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
          dmma(acc[a][b][0][0], acc[a][b][0][1], fa[buf][a].x, fb[buf][b].x);
          dmma(acc[a][b][1][0], acc[a][b][1][1], fa[buf][a].x, bi[b]);
        }
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) {
          dmma(acc[a][b][0][0], acc[a][b][0][1], nai[a], bi[b]);
          dmma(acc[a][b][1][0], acc[a][b][1][1], ai[a], fb[buf][b].x);
        }
    }
  };

  for (int kt = 0; kt < nk; ++kt) {
    if (kt > 0) __syncthreads();  // every warp is done with slot (kt - 1) % STAGES
    if (tid == 0 && kt + STAGES - 1 < nk) issue(kt + STAGES - 1);
    mbar_wait(&full[kt % STAGES], static_cast<uint32_t>((kt / STAGES) & 1));
    const double2* St = ring + (kt % STAGES) * STAGE;
    load_frags(0, St, 0);
#pragma unroll
    for (int ks = 0; ks < KS; ks += 2) {
      load_frags(1, St, ks + 1);
      compute(0);
      if (ks + 2 < KS) load_frags(0, St, ks + 2);
      compute(1);
    }
  }

#pragma unroll
  for (int a = 0; a < FM; ++a) {
    const int li = wm0 + a * 8 + (AK ? rq : pr);
    if (m0 + li >= p.M) continue;
#pragma unroll
    for (int b = 0; b < FN; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int lj = wn0 + b * 8 + (BNC ? pi8(2 * kq + h) : 2 * kq + h);
        if (n0 + lj >= p.N) continue;
        double2 v;
        if constexpr (ALG == 3) {
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

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    PEPSB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess) throw Error(kCudaError, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// Operand X (rows x K, strides sr / sk, batch strides bs[]) as a TMA map over
// float64 pairs.  kcontig: the map's inner dimension is k (box 4 k x 64 rows,
// no swizzle); otherwise the inner dimension is the row index (box 8 rows x
// 16 k, 128-byte swizzle).
void make_map(CUtensorMap* map, TmaOperand& op, const double2* base, int64_t rows, int64_t K, int64_t sr, int64_t sk,
              bool kcontig, int tile_rows, const ZgemmParams& p, const int64_t* bs) {
  cuuint64_t dim[5] = {}, str[4] = {};
  cuuint32_t box[5] = {1, 1, 1, 1, 1}, es[5] = {1, 1, 1, 1, 1};
  if (kcontig) {
    dim[0] = 2 * K;
    dim[1] = rows;
    str[0] = sr * 16;
    box[0] = 8;
    box[1] = static_cast<cuuint32_t>(tile_rows);
  } else {
    dim[0] = 2 * rows;
    dim[1] = K;
    str[0] = sk * 16;
    box[0] = 16;
    box[1] = kBKw;
  }
  op.rank = 2;
  op.nbm = 0;
  for (int a = 0; a < p.nb; ++a) {
    if (bs[a] == 0 || p.bext[a] == 1) continue;
    if (op.rank == 5) throw Error(kOtherError, "zgemm_ws: too many batch modes");
    op.bmode[op.nbm++] = a;
    dim[op.rank] = p.bext[a];
    str[op.rank - 1] = bs[a] * 16;
    ++op.rank;
  }
  // TMA needs 16-byte multiples for every stride: a degenerate extent-1 mode may carry any stride
  for (int d = 1; d < op.rank; ++d)
    if (dim[d] == 1) str[d - 1] = 16;
  const CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, op.rank, const_cast<double2*>(base), dim, str,
                                 box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 kcontig ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(kCudaError, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}

template <int BM, int BN, int WM, int WN, bool AK, bool BNC, int ALG>
void launch_ws(const ZgemmParams& p, int num_sms, cudaStream_t stream) {
  constexpr int STAGE = (BM + BN) * kBKw;
  const size_t smem = 1024 + static_cast<size_t>(kStagesW) * STAGE * 16 + 2 * kStagesW * 8 + 2 * (BM + BN) * 8 +
                      sizeof(ProdCursor);
  auto kern = zgemm_ws_kernel<BM, BN, WM, WN, AK, BNC, ALG>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    PEPSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    attr_set = true;
  }
  WsArgs args;
  args.p = p;
  CUtensorMap ta, tb;
  make_map(&ta, args.oa, p.A, p.M, p.K, p.sAi, p.sAk, AK, BM, p, p.bsA);
  make_map(&tb, args.ob, p.B, p.N, p.K, p.sBj, p.sBk, !BNC, BN, p, p.bsB);
  const int64_t tiles = ((p.M + BM - 1) / BM) * ((p.N + BN - 1) / BN);
  args.nwork = tiles * p.batch * p.splits;
  const int64_t grid = std::min<int64_t>(args.nwork, num_sms);
  kern<<<static_cast<unsigned>(grid), kThreadsW, smem, stream>>>(args, ta, tb);
  PEPSB_LAUNCH();
}

// 4M: 8 warps of 32 x 32 (128 x 64, or 64 x 128 for short M); 3M: 8 warps of
// 32 x 16 (three accumulator sets).
template <bool AK, bool BNC>
void launch_ws_any(const ZgemmParams& p, int num_sms, cudaStream_t stream) {
  const bool wide = p.M <= 64;
  if (p.algo == kGemm3M) {
    if (wide) launch_ws<64, 64, 32, 16, AK, BNC, 3>(p, num_sms, stream);
    else launch_ws<128, 32, 32, 16, AK, BNC, 3>(p, num_sms, stream);
  } else {
    if (wide) launch_ws<64, 128, 32, 32, AK, BNC, 4>(p, num_sms, stream);
    else launch_ws<128, 64, 32, 32, AK, BNC, 4>(p, num_sms, stream);
  }
}

template <int BM, int BN, int WM, int WN, int STAGES, bool AK, bool BNC, int ALG>
void launch_tma(const ZgemmParams& p, cudaStream_t stream) {
  constexpr int STAGE = (BM + BN) * kBKw;
  constexpr int NT = (BM / WM) * (BN / WN) * 32;
  const size_t smem = 1024 + static_cast<size_t>(STAGES) * STAGE * 16 + STAGES * 8 + (BM + BN) * 8;
  auto kern = zgemm_tma_kernel<BM, BN, WM, WN, STAGES, AK, BNC, ALG>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    PEPSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    attr_set = true;
  }
  WsArgs args;
  args.p = p;
  CUtensorMap ta, tb;
  make_map(&ta, args.oa, p.A, p.M, p.K, p.sAi, p.sAk, AK, BM, p, p.bsA);
  make_map(&tb, args.ob, p.B, p.N, p.K, p.sBj, p.sBk, !BNC, BN, p, p.bsB);
  const int64_t tiles = ((p.M + BM - 1) / BM) * ((p.N + BN - 1) / BN);
  args.nwork = tiles * p.batch * p.splits;
  dim3 grid(static_cast<unsigned>(tiles), static_cast<unsigned>(p.batch * p.splits));
  kern<<<grid, NT, smem, stream>>>(args, ta, tb);
  PEPSB_LAUNCH();
}

template <bool AK, bool BNC>
void launch_tma_any(const ZgemmParams& p, cudaStream_t stream) {
  if (p.algo == kGemm3M) launch_tma<64, 32, 32, 16, 4, AK, BNC, 3>(p, stream);
  else launch_tma<64, 64, 32, 32, 3, AK, BNC, 4>(p, stream);
}

}  // namespace

bool zgemm_ws_eligible(const ZgemmParams& p) {
  if (!((p.sAk == 1 || p.sAi == 1) && (p.sBj == 1 || p.sBk == 1) && p.M > 0 && p.N > 0 && p.K > 0)) return false;
  // TMA limits: dims < 2^31 here (int coordinates), strides 16-byte multiples < 2^40, <= 3 batch modes per map
  if (2 * std::max({p.M, p.N, p.K}) >= (int64_t(1) << 31)) return false;
  int na = 0, nb = 0;
  for (int a = 0; a < p.nb; ++a) {
    if (p.bext[a] == 1) continue;
    na += p.bsA[a] != 0;
    nb += p.bsB[a] != 0;
  }
  return na <= 3 && nb <= 3;
}

void zgemm_ws_tile(const ZgemmParams& p, int64_t& bm, int64_t& bn) {
  const bool wide = p.M <= 64;
  if (zgemm_ws_mode() == 2) {  // non-persistent TMA kernel
    bm = 64;
    bn = p.algo == kGemm3M ? 32 : 64;
    return;
  }
  bm = wide ? 64 : 128;
  bn = p.algo == kGemm3M ? (wide ? 64 : 32) : (wide ? 128 : 64);
}

void zgemm_ws_launch(const ZgemmParams& p, int num_sms, cudaStream_t stream) {
  const bool ak = p.sAk == 1, bnc = p.sBj == 1;
  if (zgemm_ws_mode() == 2) {
    if (ak && bnc) launch_tma_any<true, true>(p, stream);
    else if (ak) launch_tma_any<true, false>(p, stream);
    else if (bnc) launch_tma_any<false, true>(p, stream);
    else launch_tma_any<false, false>(p, stream);
    return;
  }
  if (ak && bnc) launch_ws_any<true, true>(p, num_sms, stream);
  else if (ak) launch_ws_any<true, false>(p, num_sms, stream);
  else if (bnc) launch_ws_any<false, true>(p, num_sms, stream);
  else launch_ws_any<false, false>(p, num_sms, stream);
}

}  // namespace pepsb
