// Single-block small dense solvers (see smalldense.cuh).
//
// The k x k problems of einsumsvd (k <= ~100) are far too small for a grid;
// each runs in one thread block with the matrix in shared memory, one warp
// per Jacobi rotation pair (round-robin ordering, all pairs of a round
// disjoint, one __syncthreads per round).
#include <atomic>
#include <vector>
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "smalldense.cuh"

namespace pepsb {

namespace {

// Build with -DPEPSB_EIG_PROF=1 for the divide-and-conquer phase counters
// (status words 12..27, tools/eig_phases.py).
#ifndef PEPSB_EIG_PROF
#define PEPSB_EIG_PROF 0
#endif

constexpr int kThreads = 1024;
// k x k eigensolver block: 512 threads leave 128 registers per thread for the
// register-resident tridiagonalisation / back-transformation.
constexpr int kEigThreads = 512;
// block of the register-resident path (16 <= k <= 72): 168 registers per thread
constexpr int kEigFastThreads = 384;
constexpr size_t kSmemCap = 200 * 1024;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block-wide sum (fixed summation order; every thread gets the total).
__device__ double block_sum(double v) {
  __shared__ double part[32];
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) part[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < nw; ++i) t += part[i];
  return t;
}

__device__ __forceinline__ int rr_pos(int i, int r, int npad) {
  return i == 0 ? 0 : ((i - 1 + r) % (npad - 1)) + 1;
}

// One-sided (Hestenes) Jacobi on the n columns (each m long, column stride
// ldx) of X, accumulating the rotations into V (n x n, column stride ldv,
// initialised here to I).  Block-wide; every thread must call it.
__device__ void onesided_jacobi(double2* X, int m, int n, int ldx, double2* V, int ldv, double tol,
                                double abs_skip, int max_sweeps, int* status) {
  __shared__ int rotated;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    int c = e / n, r = e % n;
    V[c * ldv + r] = make_double2(r == c ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  if (n < 2) return;
  const int npad = n + (n & 1);
  const int pairs = npad / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    for (int r = 0; r < npad - 1; ++r) {
      for (int pi = warp; pi < pairs; pi += nwarps) {
        int p = rr_pos(pi, r, npad), q = rr_pos(npad - 1 - pi, r, npad);
        if (p >= n || q >= n) continue;
        if (p > q) { int t = p; p = q; q = t; }
        double2* xp = X + static_cast<int64_t>(p) * ldx;
        double2* xq = X + static_cast<int64_t>(q) * ldx;
        double a = 0.0, b = 0.0, gr = 0.0, gi = 0.0;
        for (int i = lane; i < m; i += 32) {
          double2 u = xp[i], v = xq[i];
          a += cnorm2(u);
          b += cnorm2(v);
          gr += u.x * v.x + u.y * v.y;  // conj(u) * v
          gi += u.x * v.y - u.y * v.x;
        }
        // the four reductions interleaved (independent shuffles in flight
        // together); each variable sees the same add sequence as warp_sum
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, o);
          b += __shfl_xor_sync(0xffffffffu, b, o);
          gr += __shfl_xor_sync(0xffffffffu, gr, o);
          gi += __shfl_xor_sync(0xffffffffu, gi, o);
        }
        const double ag = hypot(gr, gi);
        if (!(ag > tol * sqrt(a * b)) || !(ag > abs_skip)) continue;
        if (lane == 0) rotated = 1;
        const double tau = (b - a) / (2.0 * ag);
        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
        const double2 ec = make_double2(gr / ag, -gi / ag);  // conj(e), e = g/|g|
        for (int i = lane; i < m; i += 32) {
          double2 u = xp[i], v = cmul(ec, xq[i]);
          xp[i] = make_double2(c * u.x - s * v.x, c * u.y - s * v.y);
          xq[i] = make_double2(s * u.x + c * v.x, s * u.y + c * v.y);
        }
        double2* vp = V + static_cast<int64_t>(p) * ldv;
        double2* vq = V + static_cast<int64_t>(q) * ldv;
        for (int i = lane; i < n; i += 32) {
          double2 u = vp[i], v = cmul(ec, vq[i]);
          vp[i] = make_double2(c * u.x - s * v.x, c * u.y - s * v.y);
          vq[i] = make_double2(s * u.x + c * v.x, s * u.y + c * v.y);
        }
      }
      __syncthreads();
    }
    const int any = rotated;
    __syncthreads();
    if (!any) break;
  }
  if (sweep == max_sweeps && threadIdx.x == 0) atomicOr(status, kSmallNoConverge);
  if (threadIdx.x == 0) {  // diagnostics: total and largest sweep counts
    atomicAdd(status + 7, sweep + 1);
    atomicMax(status + 30, sweep + 1);
  }
}

// Descending order of key[0..n) (ties by index) -> order[rank] = column.
__device__ void sort_desc(const double* key, int* order, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double ki = key[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double kj = key[j];
      rank += (kj > ki) || (kj == ki && j < i);
    }
    order[rank] = i;
  }
  __syncthreads();
}

// Column phase fix (linalg.cpp:44-64): for column `col` of a column-major
// matrix (column stride ld, rows entries) find the first largest-magnitude
// entry; returns its unit phase (1 if the column is zero).  Warp-level.
__device__ double2 column_phase(const double2* colp, int rows) {
  const int lane = threadIdx.x & 31;
  double best = 0.0;
  int bi = 0x7fffffff;
  for (int i = lane; i < rows; i += 32) {
    double a = hypot(colp[i].x, colp[i].y);
    if (a > best) { best = a; bi = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ob = __shfl_xor_sync(0xffffffffu, best, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
  if (best == 0.0) return make_double2(1.0, 0.0);
  double2 top = colp[bi];
  return make_double2(top.x / best, top.y / best);
}

// ------------------------------------------------------------------ gram_factors

// Two-sided parallel (round-robin) Jacobi for a Hermitian n x n matrix A stored
// column-major (A(i,j) = A[j*n+i]); on return A is diagonal (eigenvalues) and
// V (column-major) holds the eigenvectors.  Each round applies n/2 disjoint
// rotations A <- J^H A J with one thread per 2x2 block of (pair_i, pair_j)
// coordinates, so a round costs two barriers and no reductions.
// Pairs whose diagonal entries are both below low_skip are not rotated: at
// termination they form a block whose eigenvalues are bounded by its trace, which
// the caller sizes below its deficiency cut, so only the (discarded) basis of
// that numerically-null block is left unresolved (0 disables).
// rotation scratch, shared by both instantiations (a block runs one of them)
__shared__ double jc[128], js[128];
__shared__ double2 je[128];
__shared__ int jp[128], jq[128];
__shared__ int rotated, flag[3];

// WARP: run by warp 0 alone, __syncwarp instead of block barriers, the 2x2
// blocks of pairs and the V rows flattened over the 32 lanes -- the
// latency-optimal solver for the small k of the latency-bound configs.
template <bool WARP>
__device__ void herm_jacobi_t(double2* A, double2* V, int n, int ld, double tol, double abs_skip, double low_skip,
                              int max_sweeps, int* status) {
  const int tid = WARP ? static_cast<int>(threadIdx.x & 31) : static_cast<int>(threadIdx.x);
  const int nthr = WARP ? 32 : static_cast<int>(blockDim.x);
  auto sync = [] {
    if constexpr (WARP) __syncwarp();
    else __syncthreads();
  };
  for (int e = tid; e < n * n; e += nthr)
    V[(e / n) * ld + e % n] = make_double2((e / n) == (e % n) ? 1.0 : 0.0, 0.0);
  if (tid < 3) flag[tid] = 0;
  sync();
  if (n < 2) return;
  const int npad = n + (n & 1);
  const int pairs = npad / 2;
  const double tol2 = tol * tol, skip2 = abs_skip * abs_skip;
  int sweep = 0, round = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (tid == 0) rotated = 0;
    sync();
    for (int r = 0; r < npad - 1; ++r, ++round) {
      // phase 1: rotation parameters of the round's disjoint pairs (reads A only)
      if (tid == 0) flag[(round + 1) % 3] = 0;  // last read two rounds ago
      for (int pi = tid; pi < pairs; pi += nthr) {
        int p = rr_pos(pi, r, npad), q = rr_pos(npad - 1 - pi, r, npad);
        if (p > q) { int t = p; p = q; q = t; }
        double c = 1.0, s = 0.0;
        double2 e = make_double2(1.0, 0.0);
        if (q < n) {
          const double2 apq = A[q * ld + p];
          const double ag2 = apq.x * apq.x + apq.y * apq.y;
          const double app = A[p * ld + p].x, aqq = A[q * ld + q].x;
          if (ag2 > tol2 * fabs(app * aqq) && ag2 > skip2 &&
              (low_skip <= 0.0 || app >= low_skip || aqq >= low_skip)) {
            const double rag = rsqrt(ag2);  // 1 / |a_pq|
            const double tau = 0.5 * (aqq - app) * rag;
            const double t = copysign(1.0, tau) / (fabs(tau) + sqrt(fma(tau, tau, 1.0)));
            c = rsqrt(fma(t, t, 1.0));
            s = t * c;
            e = make_double2(apq.x * rag, apq.y * rag);
            rotated = 1;
            flag[round % 3] = 1;
          }
        }
        jp[pi] = p;
        jq[pi] = q;
        jc[pi] = c;
        js[pi] = s;
        je[pi] = e;
      }
      sync();
      if (!flag[round % 3]) continue;  // nothing rotated: no writes, no second barrier
      // phase 2: A <- J^H A J per 2x2 block of pairs (i <= j, the mirror block is
      // its conjugate transpose), J = [[c, s], [-s conj(e), c conj(e)]]; V <- V J.
      {
        const int lane = tid & 31, warp = tid >> 5, nw = nthr >> 5;
        // WARP: lane -> block (i, j), i <= j, flattened; else warp -> i, lane -> j
        const int nblk2 = pairs * (pairs + 1) / 2;
        for (int bi = WARP ? lane : warp; bi < (WARP ? nblk2 : pairs); bi += WARP ? 32 : nw) {
          int i = bi, j0 = i + lane, jstep = 32;
          if constexpr (WARP) {  // unrank bi over the upper triangle of pairs
            i = 0;
            int rem = bi;
            while (rem >= pairs - i) {
              rem -= pairs - i;
              ++i;
            }
            j0 = i + rem;
            jstep = pairs;  // one block per lane
          }
          const double sI = js[i], cI = jc[i];
          const double2 eI = je[i];
          const int ri0 = jp[i], ri1 = jq[i];
          const bool v0 = ri1 < n;
          for (int j = j0; j < pairs; j += jstep) {
            const double sJ = js[j];
            if (sI == 0.0 && sJ == 0.0) continue;
            const double cJ = jc[j];
            const double2 eJc = cconj(je[j]);
            const int cj0 = jp[j], cj1 = jq[j];
            const bool v1 = cj1 < n;
            double2 a00 = A[cj0 * ld + ri0];
            double2 a01 = v1 ? A[cj1 * ld + ri0] : make_double2(0.0, 0.0);
            double2 a10 = v0 ? A[cj0 * ld + ri1] : make_double2(0.0, 0.0);
            double2 a11 = (v0 && v1) ? A[cj1 * ld + ri1] : make_double2(0.0, 0.0);
            double2 t0 = cmul(eJc, a01), t1 = cmul(eJc, a11);
            const double2 m00 = csub(cscale(a00, cJ), cscale(t0, sJ)), m01 = cadd(cscale(a00, sJ), cscale(t0, cJ));
            const double2 m10 = csub(cscale(a10, cJ), cscale(t1, sJ)), m11 = cadd(cscale(a10, sJ), cscale(t1, cJ));
            t0 = cmul(eI, m10);
            t1 = cmul(eI, m11);
            a00 = csub(cscale(m00, cI), cscale(t0, sI));
            a10 = cadd(cscale(m00, sI), cscale(t0, cI));
            a01 = csub(cscale(m01, cI), cscale(t1, sI));
            a11 = cadd(cscale(m01, sI), cscale(t1, cI));
            if (i == j) {
              if (sI != 0.0) a01 = a10 = make_double2(0.0, 0.0);  // annihilated by construction
              a00.y = 0.0;
              a11.y = 0.0;
            }
            A[cj0 * ld + ri0] = a00;
            if (v1) A[cj1 * ld + ri0] = a01;
            if (v0) A[cj0 * ld + ri1] = a10;
            if (v0 && v1) A[cj1 * ld + ri1] = a11;
            if (i != j) {  // mirror block (rows of pair j, columns of pair i)
              A[ri0 * ld + cj0] = cconj(a00);
              if (v1) A[ri0 * ld + cj1] = cconj(a01);
              if (v0) A[ri1 * ld + cj0] = cconj(a10);
              if (v0 && v1) A[ri1 * ld + cj1] = cconj(a11);
            }
          }
        }
        for (int kk = WARP ? lane : warp; kk < (WARP ? n * pairs : n); kk += WARP ? 32 : nw)
          for (int j = WARP ? kk % pairs : lane; j < pairs; j += WARP ? pairs : 32) {
            const int k = WARP ? kk / pairs : kk;
            const double sj = js[j];
            const int q = jq[j];
            if (q >= n || sj == 0.0) continue;
            const int p = jp[j];
            const double cjv = jc[j];
            const double2 vkp = V[p * ld + k], vkq = cmul(cconj(je[j]), V[q * ld + k]);
            V[p * ld + k] = csub(cscale(vkp, cjv), cscale(vkq, sj));
            V[q * ld + k] = cadd(cscale(vkp, sj), cscale(vkq, cjv));
          }
      }
      sync();
    }
    const int any = rotated;
    sync();
    if (!any) break;
  }
  if (sweep == max_sweeps && tid == 0) atomicOr(status, kSmallNoConverge);
  if (tid == 0) atomicAdd(status + 7, sweep + 1);  // diagnostics: total sweeps
}

__device__ void herm_jacobi(double2* A, double2* V, int n, int ld, double tol, double abs_skip, double low_skip,
                            int max_sweeps, int* status) {
  herm_jacobi_t<false>(A, V, n, ld, tol, abs_skip, low_skip, max_sweeps, status);
}

// ------------------------------------------------------------------ tridiagonal divide and conquer
// Real symmetric tridiagonal eigenproblem (d, e; e[i] couples i and i+1) by
// Cuppen's divide and conquer with Gu-Eisenstat eigenvectors, the algorithm of
// LAPACK dstedc/dlaed0-4 restated for one thread block: every split point m
// removes |e[m-1]| from d[m-1] and d[m] up front, leaves are 1x1, and each merge
// of two solved halves is the rank-one problem D + rho z z^T:
//   deflation (|rho z_i| <= tol, or Givens-merged nearby poles), the secular
//   equation solved per root by a safeguarded two-pole rational model around
//   the nearer pole (all differences d_i - lambda_j formed as (d_i - sigma) - tau,
//   which is what keeps the vectors orthogonal), z recomputed from the roots
//   (Loewner), vectors z_i / (d_i - lambda_j), and the block of Z updated by
//   one small GEMM.
// Subtrees of <= 32 rows are merged by a single warp (all of them
// concurrently), larger merges by the whole block.  Z lives in V[c*ld + r].x;
// V[.].y is scratch for the merge vectors and is zeroed on exit.
struct DcScratch {
  double *zb, *dk, *zk, *zh, *sig, *tau, *rc, *rs;
  int *ndx, *perm, *ra, *rb, *meta;
  int* prof;  // diagnostics: per-phase kcycles (status words 12..)
};


// 1/x to full double precision: MUFU seed + two Newton steps (~6 pipelined
// instructions instead of the IEEE division's slow path).  x normal, nonzero.
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// sqrt(x) and 1/sqrt(x) without the IEEE slow paths: MUFU seed (20 bits) + two
// Newton steps + one correction of the product.  x normal, positive.
__device__ __forceinline__ double fast_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  double t = fma(-hx * y, y, 0.5);
  y = fma(y, t, y);
  t = fma(-hx * y, y, 0.5);
  return fma(y, t, y);
}
__device__ __forceinline__ double fast_sqrt(double x) {
  const double y = fast_rsqrt(x);
  const double s = x * y;
  return fma(0.5 * y, fma(-s, s, x), s);
}

// Sum / product over the T-lane segment (T a power of two, segment-aligned).
__device__ __forceinline__ void dmma_f64(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double seg_sum(double v, int T, unsigned mask) {
  for (int o = T >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
  return v;
}
__device__ __forceinline__ double seg_prod(double v, int T, unsigned mask) {
  for (int o = T >> 1; o > 0; o >>= 1) v *= __shfl_xor_sync(mask, v, o);
  return v;
}

// Root j (ascending) of 1/rho + sum_i zk_i^2 / (dk_i - lambda) = 0, returned as
// lambda = sigma + tau with sigma a pole.  Warp-synchronous: all 32 lanes call
// it together (valid == false for padding lanes); the T lanes of a segment
// split the sums over i (lane `sub` takes i = sub, sub + T, ...) and run the
// scalar iteration redundantly; the iteration count is uniform over the warp
// (until every segment has converged), so the full-mask shuffles never see a
// diverged warp.
__device__ void dc_secular_root(bool valid, int j, int K, const double* dk, const double* zk, double rho, int sub,
                                int T, double* sig_out, double* tau_out, int* prof) {
  const unsigned full = 0xffffffffu;
  const double eps = 2.220446049250313e-16;
  if (!valid) {  // padding lane: harmless in-range values, converged from the start
    j = 0;
    K = 2;
    rho = 1.0;
  }
  const double irho = 1.0 / rho;
  double sig, lo_t, hi_t;
  int pl, pr;
  if (j < K - 1) {
    const double gap = dk[j + 1] - dk[j], mid = 0.5 * gap;
    double f = 0.0;
    if (valid)
#pragma unroll 4
      for (int i = sub; i < K; i += T) f += zk[i] * zk[i] * fast_rcp((dk[i] - dk[j]) - mid);
    f = irho + seg_sum(f, T, full);
    if (f >= 0.0) {  // root in (d_j, d_j + gap/2]: origin d_j
      sig = dk[j];
      lo_t = 0.0;
      hi_t = mid;
    } else {  // root in (d_j + gap/2, d_j+1): origin d_j+1
      sig = dk[j + 1];
      lo_t = -mid;
      hi_t = 0.0;
    }
    pl = j;
    pr = j + 1;
  } else {
    double zz = 0.0;
    if (valid)
      for (int i = sub; i < K; i += T) zz += zk[i] * zk[i];
    zz = seg_sum(zz, T, full);
    sig = dk[K - 1];
    lo_t = 0.0;
    hi_t = rho * zz;
    pl = K - 2;
    pr = K - 1;
  }
  double tau = 0.5 * (lo_t + hi_t);
  bool done = !valid || K == 1;
  if (valid && K == 1) {
    sig = dk[0];
    tau = rho * zk[0] * zk[0];
  }
  const int i1 = pl + 1 + ((sub - (pl + 1)) % T + T) % T;  // first i > pl in this lane's stride
  int nit = 0;
  (void)nit;
  for (int it = 0; it < 100; ++it) {
    if (!__any_sync(full, !done)) break;
    if (!done) ++nit;
    double psi = 0.0, dpsi = 0.0, phi = 0.0, dphi = 0.0;
    if (!done) {
#pragma unroll 4
      for (int i = sub; i <= pl; i += T) {
        const double inv = fast_rcp((dk[i] - sig) - tau);
        const double t = zk[i] * zk[i] * inv;
        psi += t;
        dpsi += t * inv;
      }
#pragma unroll 4
      for (int i = i1; i < K; i += T) {
        const double inv = fast_rcp((dk[i] - sig) - tau);
        const double t = zk[i] * zk[i] * inv;
        phi += t;
        dphi += t * inv;
      }
    }
    for (int o = T >> 1; o > 0; o >>= 1) {  // the four sums interleaved: one shuffle latency per level
      const double s0 = __shfl_xor_sync(full, psi, o), s1 = __shfl_xor_sync(full, dpsi, o);
      const double s2 = __shfl_xor_sync(full, phi, o), s3 = __shfl_xor_sync(full, dphi, o);
      psi += s0;
      dpsi += s1;
      phi += s2;
      dphi += s3;
    }
    if (done) continue;
    const double f = irho + psi + phi;
    if (f < 0.0) lo_t = tau;
    else hi_t = tau;
    if (f == 0.0 || fabs(f) <= 8.0 * eps * K * (irho + fabs(psi) + fabs(phi)) ||
        hi_t - lo_t <= 2.0 * eps * fmax(fabs(lo_t), fabs(hi_t))) {
      done = true;
      continue;
    }
    const double lo_e = lo_t - tau, hi_e = hi_t - tau;
    double eta = 0.5 * (lo_e + hi_e);  // bisection unless the model step lands inside
    if (it < 40) {
      // f(lambda + eta) ~ c + B / (Dl - eta) + D / (Dr - eta):  c eta^2 - a eta + b = 0
      const double Dl = (dk[pl] - sig) - tau, Dr = (dk[pr] - sig) - tau;
      const double B = Dl * Dl * dpsi, D = Dr * Dr * dphi;
      const double c = f - Dl * dpsi - Dr * dphi;
      const double a = c * (Dl + Dr) + B + D, b = Dl * Dr * f;
      // the step only has to land inside the bracket: reciprocal / sqrt by MUFU
      // seed + Newton (full precision for normal operands) instead of the IEEE
      // slow paths (~110 / ~90 cycles each on the iteration's critical path)
      auto okr = [](double v) { return fabs(v) > 1e-290 && fabs(v) < 1e290; };
      if (c == 0.0) {
        if (a != 0.0) {
          const double r = okr(a) ? b * fast_rcp(a) : b / a;
          if (r > lo_e && r < hi_e) eta = r;
        }
      } else {
        const double disc = fmax(a * a - 4.0 * b * c, 0.0);
        const double sq = (disc > 1e-290 && disc < 1e290) ? fast_sqrt(disc) : sqrt(disc);
        const double q = 0.5 * (a + copysign(sq, a));
        const double r1 = okr(c) ? q * fast_rcp(c) : q / c;
        const double r2 = q != 0.0 ? (okr(q) ? b * fast_rcp(q) : b / q) : 0.0;
        if (r1 > lo_e && r1 < hi_e) eta = r1;
        else if (r2 > lo_e && r2 < hi_e) eta = r2;
      }
    }
    const double tn = tau + eta;
    if (tn == tau) done = true;
    tau = tn;
  }
  if (valid && sub == 0) {
    *sig_out = sig;
    *tau_out = tau;
  }
#if PEPSB_EIG_PROF
  if (valid && sub == 0) {
    atomicMax(prof, nit);
    atomicAdd(prof + 1, nit);
    atomicAdd(prof + 2, 1);
  }
#endif
}

// One merge of the two solved halves of node [lo, lo + N) (split at n1) by a
// group of G threads (thread gt of the group; active == false: a padding
// group).  Every group of one tree level runs in lock step -- all block
// barriers are executed by every thread the same number of times.
// Z(r, c) lives in V[c*ld + r].x; V[.].y of the node's diagonal block holds the
// merge vectors; the GEMM result is staged in the free upper triangle of A.
__device__ void dc_merge(bool active, int lo, int n1, int N, int gt, int G, double* d, const double* e, double2* V,
                         double2* A, int ld, const DcScratch& S, bool top) {
  const int lane = threadIdx.x & 31;
  // diagnostics: cycles of the top-level merge's phases in status words 12..19
  long long pc = clock64();
  int pslot = 0;
  auto mark = [&]() {
#if PEPSB_EIG_PROF
    if (top && threadIdx.x == 0) {
      const long long c = clock64();
      atomicAdd(S.prof + pslot, static_cast<int>((c - pc) >> 4));
      pc = c;
    }
    ++pslot;
#endif
  };
  (void)pc;
  (void)pslot;
  const double eps = 2.220446049250313e-16;
  const double beta = active ? e[lo + n1 - 1] : 0.0;
  const double rho = 2.0 * fabs(beta);
  const double sg = beta >= 0.0 ? 1.0 : -1.0;

  // z = Q^T (e_last(T1) + sg e_first(T2)) / sqrt(2); ascending order of d
  if (active)
    for (int c = gt; c < N; c += G) {
      const int col = lo + c;
      S.zb[col] = (c < n1 ? V[col * ld + lo + n1 - 1].x : sg * V[col * ld + lo + n1].x) * 0.70710678118654752440;
      const double dc = d[col];
      int r = 0;
      for (int c2 = 0; c2 < N; ++c2) {
        const double d2 = d[lo + c2];
        r += (d2 < dc) || (d2 == dc && c2 < c);
      }
      S.perm[lo + r] = col;
    }
  __syncthreads();
  mark();
  // sorted copies (d, z in ascending d) for the sequential scan: its loads no
  // longer chain through perm
  if (active)
    for (int q = gt; q < N; q += G) {
      const int c = S.perm[lo + q];
      S.dk[lo + q] = d[c];
      S.zk[lo + q] = S.zb[c];
    }
  __syncthreads();
  mark();
  // deflation (sequential, dlaed2's rules)
  if (active && gt == 0) {
    double dmax = 0.0;
    for (int c = 0; c < N; ++c) dmax = fmax(dmax, fabs(S.dk[lo + c]));
    const double tol = 8.0 * eps * fmax(dmax, rho);
    int K = 0, nrot = 0, prev = -1;
    double zp = 0.0, dp = 0.0;  // z, d of prev (current values)
    // the next entry is loaded before this one's stores (which the compiler
    // must assume to alias), so the scan's chain is arithmetic only
    int cn = S.perm[lo];
    double zn = S.zk[lo], dn = S.dk[lo];
    for (int q = 0; q < N; ++q) {
      const int c = cn;
      const double zc = zn, dcv = dn;
      if (q + 1 < N) {
        cn = S.perm[lo + q + 1];
        zn = S.zk[lo + q + 1];
        dn = S.dk[lo + q + 1];
      }
      if (rho * fabs(zc) <= tol) continue;  // eigenpair (d_c, column c) deflates
      if (prev < 0) {
        prev = c;
        zp = zc;
        dp = dcv;
        continue;
      }
      // |(d_c - d_p) a b| <= tol with a b = -z_c z_p / (z_p^2 + z_c^2), division-free
      if (fabs((dcv - dp) * zc * zp) <= tol * (zp * zp + zc * zc)) {  // nearby poles: rotate z_prev into z_c
        const double t = hypot(zp, zc);
        const double a = zc / t, b = -zp / t;
        S.ra[lo + nrot] = prev;
        S.rb[lo + nrot] = c;
        S.rc[lo + nrot] = a;
        S.rs[lo + nrot] = b;
        ++nrot;
        S.zb[c] = t;
        S.zb[prev] = 0.0;
        d[prev] = a * a * dp + b * b * dcv;
        d[c] = b * b * dp + a * a * dcv;
        zp = t;
        dp = b * b * dp + a * a * dcv;
      } else {
        S.ndx[lo + K++] = prev;
        zp = zc;
        dp = dcv;
      }
      prev = c;
    }
    if (prev >= 0) S.ndx[lo + K++] = prev;
    S.meta[2 * lo] = K;
    S.meta[2 * lo + 1] = nrot;
  }
  __syncthreads();
  mark();
  const int K = active ? S.meta[2 * lo] : 0, nrot = active ? S.meta[2 * lo + 1] : 0;
  for (int r = lo + gt; r < lo + N && nrot > 0; r += G)
    for (int t = 0; t < nrot; ++t) {  // Q <- Q R^T, rotations in order
      const int pa = S.ra[lo + t], pb = S.rb[lo + t];
      const double a = S.rc[lo + t], b = S.rs[lo + t];
      const double xp = V[pa * ld + r].x, xc = V[pb * ld + r].x;
      V[pa * ld + r].x = a * xp + b * xc;
      V[pb * ld + r].x = a * xc - b * xp;
    }
  for (int i = gt; i < K; i += G) {
    const int c = S.ndx[lo + i];
    S.dk[lo + i] = d[c];
    S.zk[lo + i] = S.zb[c];
  }
  __syncthreads();
  mark();
  // T lanes per root / per vector: the largest power of two with 2 T K <= G
  int T = 1;
  while (T < 32 && T < G && 2 * T * K <= G) T <<= 1;
  T = __reduce_min_sync(0xffffffffu, T);  // warp-uniform: groups sharing a warp run the same shuffles
  const int sub = lane & (T - 1), seg = gt / T, nseg = G / T;
  const unsigned mask = 0xffffffffu;  // every loop below has a warp-uniform trip count
  const double* dk = S.dk + lo;
  const double* zk = S.zk + lo;
  const int nq = __reduce_max_sync(mask, K > seg ? (K - seg + nseg - 1) / nseg : 0);
  for (int q = 0; q < nq; ++q) {
    const int j = seg + q * nseg;
    dc_secular_root(j < K, j, K, dk, zk, rho, sub, T, S.sig + lo + j, S.tau + lo + j, S.prof + 24);
  }
  __syncthreads();
  mark();
  const double* sg_ = S.sig + lo;
  const double* tu_ = S.tau + lo;
  // z recomputed from the roots: zh_i^2 = prod_j (lambda_j - d_i) / (rho prod_{j != i} (d_j - d_i))
  for (int q = 0; q < nq; ++q) {
    const int i = seg + q * nseg;
    double w = 1.0;
    if (i < K) {
      const double di = dk[i];
#pragma unroll 4
      for (int j = sub; j < K; j += T)
        w *= -((di - sg_[j]) - tu_[j]) * (j == i ? 1.0 / rho : fast_rcp(dk[j] - di));
    }
    w = seg_prod(w, T, mask);
    if (i < K && sub == 0) S.zh[lo + i] = copysign(sqrt(fmax(w, 0.0)), zk[i]);
  }
  __syncthreads();
  mark();
  // merge vectors v_j[i] = zh_i / (d_i - lambda_j), normalised; stored W^T in V.y:
  // v_j[i] at V[(lo + i) * ld + lo + j].y
  const double* zh = S.zh + lo;
  for (int q = 0; q < nq; ++q) {
    const int j = seg + q * nseg;
    double nrm = 0.0;
    if (j < K)
#pragma unroll 4
      for (int i = sub; i < K; i += T) {
        const double v = zh[i] * fast_rcp((dk[i] - sg_[j]) - tu_[j]);
        V[(lo + i) * ld + lo + j].y = v;
        nrm += v * v;
      }
    const double inv = rsqrt(seg_sum(nrm, T, mask));
    if (j < K)
      for (int i = sub; i < K; i += T) V[(lo + i) * ld + lo + j].y *= inv;
  }
  __syncthreads();
  mark();
  for (int j = gt; j < K; j += G) d[S.ndx[lo + j]] = sg_[j] + tu_[j];
  // Zt(r, ndx[j]) = sum_i Z(r, ndx[i]) v_j[i] staged in A's upper triangle
  // (local (r, c): r <= c at A(lo + r, lo + c).x, r > c at A(lo + c, lo + r).y),
  // then copied back over Z.
  const int* ndx = S.ndx + lo;
  if (G >= 32) {
    // whole warps: 16 x 16 tiles on the FP64 tensor pipe (DMMA.8x8x4), four
    // DMMAs per four fragment loads.  The 4 x 4 scalar tiles below read the
    // merge vectors at a 64-byte stride (16-way bank conflicts): 64 k cycles
    // for the 72 x 72 x 72 top-level product against ~8 k here.
    const int wg = gt >> 5, nwg = G >> 5;
    const int tr = (N + 15) >> 4, tc = (K + 15) >> 4;
    const int rq = lane >> 2, kq = lane & 3;
    for (int o = wg; o < tr * tc; o += nwg) {
      const int r0 = (o / tc) * 16, j0 = (o % tc) * 16;
      double c00[2] = {0.0, 0.0}, c01[2] = {0.0, 0.0}, c10[2] = {0.0, 0.0}, c11[2] = {0.0, 0.0};
      const bool ra0 = r0 + rq < N, ra1 = r0 + 8 + rq < N, cb0 = j0 + rq < K, cb1 = j0 + 8 + rq < K;
      for (int k0 = 0; k0 < K; k0 += 4) {
        const int kk = k0 + kq;
        const bool kin = kk < K;
        const double2* zc = V + (kin ? ndx[kk] : lo) * ld + lo + r0 + rq;
        const double2* wr = V + (lo + (kin ? kk : 0)) * ld + lo + j0 + rq;
        const double a0 = kin && ra0 ? zc[0].x : 0.0, a1 = kin && ra1 ? zc[8].x : 0.0;
        const double b0 = kin && cb0 ? wr[0].y : 0.0, b1 = kin && cb1 ? wr[8].y : 0.0;
        dmma_f64(c00[0], c00[1], a0, b0);
        dmma_f64(c01[0], c01[1], a0, b1);
        dmma_f64(c10[0], c10[1], a1, b0);
        dmma_f64(c11[0], c11[1], a1, b1);
      }
      auto put = [&](int r, int j, double v) {
        if (r < N && j < K) {
          const int c = ndx[j] - lo;
          if (r <= c) A[(lo + c) * ld + lo + r].x = v;
          else A[(lo + r) * ld + lo + c].y = v;
        }
      };
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        put(r0 + rq, j0 + 2 * kq + h, c00[h]);
        put(r0 + rq, j0 + 8 + 2 * kq + h, c01[h]);
        put(r0 + 8 + rq, j0 + 2 * kq + h, c10[h]);
        put(r0 + 8 + rq, j0 + 8 + 2 * kq + h, c11[h]);
      }
    }
  } else {
    // 4 x 4 register tiles: 9 shared loads per 16 FMAs
    const int tr = (N + 3) >> 2, tc = (K + 3) >> 2;
    for (int o = gt; o < tr * tc; o += G) {
      const int r0 = (o / tc) * 4, j0 = (o % tc) * 4;
      double acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
      for (int i = 0; i < K; ++i) {
        const double2* zc = V + ndx[i] * ld + lo + r0;
        const double2* wr = V + (lo + i) * ld + lo + j0;
        double zv[4], wv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) zv[a] = r0 + a < N ? zc[a].x : 0.0;
#pragma unroll
        for (int b = 0; b < 4; ++b) wv[b] = j0 + b < K ? wr[b].y : 0.0;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fma(zv[a], wv[b], acc[a][b]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int r = r0 + a, j = j0 + b;
          if (r < N && j < K) {
            const int c = ndx[j] - lo;
            if (r <= c) A[(lo + c) * ld + lo + r].x = acc[a][b];
            else A[(lo + r) * ld + lo + c].y = acc[a][b];
          }
        }
    }
  }
  __syncthreads();
  mark();
  for (int o = gt; o < N * K; o += G) {
    const int r = o / K, c = ndx[o % K] - lo;
    V[(lo + c) * ld + lo + r].x = r <= c ? A[(lo + c) * ld + lo + r].x : A[(lo + r) * ld + lo + c].y;
  }
  __syncthreads();
  mark();
}

// d, e in shared memory; V column-major (ld); A: the tridiagonalised matrix
// (only its upper triangle is used, as staging).  On return d holds the
// eigenvalues (unsorted) and V[c*ld + r] = (Z(r, c), 0).
__device__ void tridiag_dc(double* d, double* e, double2* V, double2* A, int n, int ld, const DcScratch& S) {
  // Merge schedule: internal nodes grouped by depth; the nodes of one depth
  // are merged concurrently (block split into equal power-of-two groups),
  // deepest first.
  __shared__ short2 nodes[256];  // (lo, N), depth-major
  __shared__ int dstart[17];
  __shared__ int ndepth;
  const int tid = threadIdx.x;
  for (int t = tid; t < n * n; t += blockDim.x)
    V[(t / n) * ld + t % n] = make_double2((t / n) == (t % n) ? 1.0 : 0.0, 0.0);
  if (tid == 0) {
    for (int m = 1; m < n; ++m) {  // Cuppen's rank-one tear at every split point
      const double r = fabs(e[m - 1]);
      d[m - 1] -= r;
      d[m] -= r;
    }
    // breadth-first over the halving tree: depth t occupies nodes[dstart[t] .. dstart[t+1])
    int cnt = 0, nd = 0;
    if (n >= 2) nodes[cnt++] = make_short2(0, static_cast<short>(n));
    int b = 0;
    while (b < cnt) {
      dstart[nd++] = b;
      const int e_ = cnt;
      for (int q = b; q < e_; ++q) {
        const short2 x = nodes[q];
        const short h = static_cast<short>(x.y / 2);
        if (h >= 2) nodes[cnt++] = make_short2(x.x, h);
        if (x.y - h >= 2) nodes[cnt++] = make_short2(static_cast<short>(x.x + h), static_cast<short>(x.y - h));
      }
      b = e_;
    }
    dstart[nd] = cnt;
    ndepth = nd;
  }
  __syncthreads();
  for (int t = ndepth - 1; t >= 0; --t) {
    const int first = dstart[t], m = dstart[t + 1] - first;
    int G = 1;
    while (2 * G * m <= static_cast<int>(blockDim.x)) G <<= 1;
    if (G >= 32) G = (static_cast<int>(blockDim.x) / m) & ~31;  // whole warps: all of them (384 = 3 x 128)
    const int g = tid / G;
    const bool active = g < m;
    const short2 x = active ? nodes[first + g] : make_short2(0, 2);
#if PEPSB_EIG_PROF
    const long long c0 = clock64();
#endif
    dc_merge(active, x.x, x.y / 2, x.y, tid % G, G, d, e, V, A, ld, S, t == 0);
#if PEPSB_EIG_PROF
    if (tid == 0 && t < 7) atomicAdd(S.prof + 9 + t, static_cast<int>((clock64() - c0) >> 4));  // words 21..28
#endif
  }
  for (int t = tid; t < n * n; t += blockDim.x) V[(t / n) * ld + t % n].y = 0.0;
  __syncthreads();
}

// Back-transformation X = H_0 ... H_{n-2} Z with each column of X held in the
// registers of an 8-lane group (rows s = gl + 8k), n <= 8 * ES: reflectors are
// read from shared memory as broadcasts, X never round-trips through it.
template <int ES, int GS>
__device__ void back_transform_reg(const double2* A, double2* V, int n, int ld, const double2* tauv) {
  const int tid = threadIdx.x, grp = tid / GS, gl = tid % GS, ngrp = blockDim.x / GS;
  for (int cbase = 0; cbase < n; cbase += ngrp) {
    const int c = cbase + grp;
    const bool act = c < n;
    double2 x[ES];
#pragma unroll
    for (int k = 0; k < ES; ++k) {
      const int s = gl + GS * k;
      x[k] = (act && s < n) ? V[c * ld + s] : make_double2(0.0, 0.0);
    }
    for (int j = n - 2; j >= 0; --j) {
      const double2 tau = tauv[j];
      if (tau.x == 0.0 && tau.y == 0.0) continue;
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int k = 0; k < ES; ++k) {
        const int s = gl + GS * k;
        if (s > j && s < n) {
          const double2 v = A[j * ld + s];
          re += v.x * x[k].x + v.y * x[k].y;
          im += v.x * x[k].y - v.y * x[k].x;
        }
      }
#pragma unroll
      for (int o = GS / 2; o > 0; o >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, o);
        im += __shfl_xor_sync(0xffffffffu, im, o);
      }
      const double2 t = cmul(tau, make_double2(re, im));
#pragma unroll
      for (int k = 0; k < ES; ++k) {
        const int s = gl + GS * k;
        if (s > j && s < n) x[k] = csub(x[k], cmul(A[j * ld + s], t));
      }
    }
    if (act)
#pragma unroll
      for (int k = 0; k < ES; ++k) {
        const int s = gl + GS * k;
        if (s < n) V[c * ld + s] = x[k];
      }
  }
}

// Register-resident Householder tridiagonalisation (16 <= n <= 4 NC <= 72, a
// block of 384 threads = 168 registers each: the kernel's shared memory leaves
// no L1, so a single spilled value costs an L2 round trip per column).
// Thread (row i = tid / 4, gl = tid % 4) keeps A(i, gl + 4 c), c < NC, in
// registers for the whole reduction: the trailing matrix never round-trips
// through shared memory (the smem-resident version moved 32 B per element and
// column and spent ~4.2 k cycles per column, most of it in warp 0's serial
// reflector arithmetic between two block barriers).  One block barrier per
// column:
//   P1 (every active warp redundantly, NV indices per lane): from column j
//      (published by its owners during the previous matvec) and p = tau A v of
//      the previous reflector, form w_{j-1} = p + alpha2 v, apply that pending
//      rank-2 update to column j analytically, generate reflector j, and leave
//      v_{j-1}, w_{j-1}, v_j in a warp-private buffer (__syncwarp, no block
//      barrier);
//   matvec: each thread applies the pending update to its registers, accumulates
//      A v_j over its columns, publishes column j+1 and, after a 4-lane shuffle
//      reduction, p_i.  Branch-free over the columns: the buffers are zero
//      outside the trailing block (and padded to 4 NC), so stale columns
//      contribute exact zeros.
// Warps whose rows are all above the trailing block only attend the barrier.
// On return: d, e (e[j] = beta_j), tauv, reflector j in X[j*ld + l], l > j
// (v[j+1] = 1 stored explicitly).  wbuf: >= ceil(n/8) * 12 NC complex scratch.
#if PEPSB_EIG_PROF
__device__ int g_tri_prof[8];
#endif
template <int NC>
__device__ void herm_tridiag_reg(double2* X, int n, int ld, double* d, double* e, double2* tauv, double2* wbuf,
                                 double2* sh /* 4 x 128 */) {
  constexpr int NV = (4 * NC + 31) / 32;
  constexpr int NP = 4 * NC;  // padded vector length
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int i = tid >> 2, gl = tid & 3;
  const double2 z0 = make_double2(0.0, 0.0);
  double2* colbuf = sh;       // [2][128]
  double2* pbuf = sh + 256;   // [2][128]
  double2* wv = wbuf;  // [vbuf0 | vbuf1 | wprev]
  // reflector warp: the block's last warp owns no rows (4 n <= 288 < 352), so the
  // serial reflector arithmetic never competes with a matvec warp for its FP64 pipe
  const int pwarp = (blockDim.x >> 5) - 1;
  double2 a[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int l = gl + 4 * c;
    a[c] = (i < n && l < n) ? X[l * ld + i] : z0;
  }
  for (int t = tid; t < n; t += blockDim.x) colbuf[t] = X[t];  // column 0
  for (int t = tid; t < 3 * NP; t += blockDim.x) wv[t] = z0;
  __syncthreads();
  double2 tau = z0;  // reflector j - 1's (identical in every active warp)
#if PEPSB_EIG_PROF
  long long pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, pt = clock64();
#define TRI_MARK(k)                  \
  {                                  \
    const long long c_ = clock64();  \
    pacc[k] += c_ - pt;              \
    pt = c_;                         \
  }
#else
#define TRI_MARK(k)
#endif
  for (int j = 0; j < n; ++j) {
    const int b = j & 1;
    const bool last = j == n - 1;
    double2* vprev = wv + (b ^ 1) * NP;
    double2* vnew = wv + b * NP;
    double2* wprev = wv + 2 * NP;
    if (warp == pwarp) {
      const bool pend = j > 0 && (tau.x != 0.0 || tau.y != 0.0);
      double2 x[NV];
      // ---- w_{j-1} = p + alpha2 v,  alpha2 = -1/2 tau (p^H v); operands are
      // re-read from shared memory rather than kept live
      if (pend) {
        double hr = 0.0, hi = 0.0;
#pragma unroll
        for (int s = 0; s < NV; ++s) {
          const int r = lane + 32 * s;
          if (r >= j && r < n) {
            const double2 v = vprev[r], pp = pbuf[(b ^ 1) * 128 + r];
            hr += pp.x * v.x + pp.y * v.y;
            hi += pp.x * v.y - pp.y * v.x;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          hr += __shfl_xor_sync(0xffffffffu, hr, o);
          hi += __shfl_xor_sync(0xffffffffu, hi, o);
        }
        TRI_MARK(0)
        const double2 alpha2 = cscale(cmul(tau, make_double2(hr, hi)), -0.5);
#pragma unroll
        for (int s = 0; s < NV; ++s) {
          const int r = lane + 32 * s;
          if (r < n) wprev[r] = r >= j ? cadd(pbuf[(b ^ 1) * 128 + r], cmul(alpha2, vprev[r])) : z0;
        }
      } else {
#pragma unroll
        for (int s = 0; s < NV; ++s) {
          const int r = lane + 32 * s;
          if (r < n) wprev[r] = z0;
        }
      }
      __syncwarp();
      TRI_MARK(1)
      // v_{j-1}[j], w_{j-1}[j]
      const double2 vj = pend ? vprev[j] : z0, wj = pend ? wprev[j] : z0;
      // ---- column j with the pending update applied; its norm below j + 1
      double xn = 0.0;
#pragma unroll
      for (int s = 0; s < NV; ++s) {
        const int r = lane + 32 * s;
        x[s] = z0;
        if (r >= j && r < n) {
          double2 v = colbuf[b * 128 + r];
          if (pend) v = csub(v, cadd(cmulc(wj, vprev[r]), cmulc(vj, wprev[r])));
          x[s] = v;
          if (r >= j + 2) xn += cnorm2(v);
        }
      }
      double2 sa = x[0], sd = x[0];
#pragma unroll
      for (int s = 1; s < NV; ++s) {
        if (((j + 1) >> 5) == s) sa = x[s];
        if ((j >> 5) == s) sd = x[s];
      }
      const double dj = __shfl_sync(0xffffffffu, sd.x, j & 31);
      if (last) {
        if (lane == 0) {
          d[j] = dj;
          e[j] = 0.0;
        }
      } else {
        const double2 alpha =
            make_double2(__shfl_sync(0xffffffffu, sa.x, (j + 1) & 31), __shfl_sync(0xffffffffu, sa.y, (j + 1) & 31));
        xn = warp_sum(xn);
        TRI_MARK(2)
        double2 scal = z0;
        double beta;
        tau = z0;
        if (xn == 0.0 && alpha.y == 0.0) {
          beta = alpha.x;
        } else {
          const double s2 = alpha.x * alpha.x + alpha.y * alpha.y + xn;
          const bool safe = s2 > 1e-280 && s2 < 1e280;
          double rb;  // 1 / beta
          if (safe) {
            const double y = fast_rsqrt(s2);
            const double s = s2 * y;
            beta = -copysign(fma(0.5 * y, fma(-s, s, s2), s), alpha.x);
            rb = -copysign(y, alpha.x);
          } else {
            beta = -copysign(sqrt(s2), alpha.x);
            rb = 1.0 / beta;
          }
          tau = make_double2((beta - alpha.x) * rb, -alpha.y * rb);
          const double2 den = make_double2(alpha.x - beta, alpha.y);  // scal = 1 / (alpha - beta)
          const double dn2 = cnorm2(den);
          const double dn = (dn2 > 1e-280 && dn2 < 1e280) ? fast_rcp(dn2) : 1.0 / dn2;
          scal = make_double2(den.x * dn, -den.y * dn);
        }
        const bool zero = tau.x == 0.0 && tau.y == 0.0;
        TRI_MARK(3)
#pragma unroll
        for (int s = 0; s < NV; ++s) {
          const int r = lane + 32 * s;
          double2 v = z0;
          if (!zero && r < n) v = r == j + 1 ? make_double2(1.0, 0.0) : (r >= j + 2 ? cmul(x[s], scal) : z0);
          if (r < n) {
            vnew[r] = v;
            if (r > j) X[j * ld + r] = v;
          }
        }
        if (lane == 0) {
          d[j] = dj;
          e[j] = beta;
          tauv[j] = tau;
        }
        TRI_MARK(4)
      }
    }
    __syncthreads();
    // ---- matvec over the trailing block (rows, columns >= j + 1)
    if (!last && 8 * warp + 7 > j && 8 * warp < n) {
      {
        const bool rowact = i > j && i < n;
        const unsigned mrow = __ballot_sync(0xffffffffu, rowact);
        if (rowact) {
          const double2 tauj = tauv[j];
          const double2 vi = vprev[i], wi = wprev[i];
          double r0 = 0.0, i0 = 0.0, r1 = 0.0, i1 = 0.0;
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            if (4 * c + 3 <= j) continue;  // warp-uniform: all four columns left of the block
            const int l = gl + 4 * c;
            const double2 wl = wprev[l], vl = vprev[l], y = vnew[l];
            double2 v = a[c];
            v.x = fma(-wl.x, vi.x, v.x);
            v.y = fma(-wl.x, vi.y, v.y);
            v.x = fma(-wl.y, vi.y, v.x);
            v.y = fma(wl.y, vi.x, v.y);
            v.x = fma(-vl.x, wi.x, v.x);
            v.y = fma(-vl.x, wi.y, v.y);
            v.x = fma(-vl.y, wi.y, v.x);
            v.y = fma(vl.y, wi.x, v.y);
            a[c] = v;
            if (l == j + 1) colbuf[(b ^ 1) * 128 + i] = v;
            if (c & 1) {
              r1 = fma(v.x, y.x, r1);
              i1 = fma(v.x, y.y, i1);
              r1 = fma(-v.y, y.y, r1);
              i1 = fma(v.y, y.x, i1);
            } else {
              r0 = fma(v.x, y.x, r0);
              i0 = fma(v.x, y.y, i0);
              r0 = fma(-v.y, y.y, r0);
              i0 = fma(v.y, y.x, i0);
            }
          }
          r0 += r1;
          i0 += i1;
          r0 += __shfl_xor_sync(mrow, r0, 1);
          i0 += __shfl_xor_sync(mrow, i0, 1);
          r0 += __shfl_xor_sync(mrow, r0, 2);
          i0 += __shfl_xor_sync(mrow, i0, 2);
          if (gl == 0) pbuf[b * 128 + i] = cmul(tauj, make_double2(r0, i0));
        }
      }
    }
    TRI_MARK(5)
    __syncthreads();
    TRI_MARK(6)
  }
#if PEPSB_EIG_PROF
  if (warp == pwarp && lane == 0)
    for (int k = 0; k < 7; ++k) atomicAdd(g_tri_prof + k, static_cast<int>(pacc[k] >> 4));
#endif
#undef TRI_MARK
}

// Back-transformation X = H_0 ... H_{n-2} Z, one GS-lane group per column with
// the column in registers, rows in reverse order (slot k of lane gl holds row
// n-1 - (gl + GS k)): reflector j touches rows > j, i.e. the slots k <
// ceil((n-1-j) / GS), so the unrolled slot loops stop at a warp-uniform bound
// instead of issuing every predicated-off slot (Z is real on entry).
template <int ES, int GS>
__device__ void back_transform_rev(const double2* A, double2* V, int n, int ld, const double2* tauv) {
  const int tid = threadIdx.x, gl = tid % GS;
  if ((tid & ~31) / GS >= n) return;  // whole warps only: the shuffles below use the full mask
  const bool act = tid / GS < n;
  const int c = act ? tid / GS : 0;
  double2 x[ES];
#pragma unroll
  for (int k = 0; k < ES; ++k) {
    const int s = n - 1 - (gl + GS * k);
    x[k] = s >= 0 ? make_double2(V[c * ld + s].x, 0.0) : make_double2(0.0, 0.0);
  }
  for (int j = n - 2; j >= 0; --j) {
    const double2 tau = tauv[j];
    if (tau.x == 0.0 && tau.y == 0.0) continue;
    const int m = n - 1 - j;  // rows n-1 .. j+1  <->  gl + GS k < m
    const int kmax = (m + GS - 1) / GS;
    const double2* vcol = A + j * ld + (n - 1 - gl);
    double re0 = 0.0, im0 = 0.0, re1 = 0.0, im1 = 0.0;
#pragma unroll
    for (int k = 0; k < ES; ++k) {
      if (k >= kmax) break;
      if (gl + GS * k < m) {
        const double2 v = vcol[-GS * k];
        if (k & 1) {
          re1 += v.x * x[k].x + v.y * x[k].y;
          im1 += v.x * x[k].y - v.y * x[k].x;
        } else {
          re0 += v.x * x[k].x + v.y * x[k].y;
          im0 += v.x * x[k].y - v.y * x[k].x;
        }
      }
    }
    re0 += re1;
    im0 += im1;
#pragma unroll
    for (int o = GS / 2; o > 0; o >>= 1) {
      re0 += __shfl_xor_sync(0xffffffffu, re0, o);
      im0 += __shfl_xor_sync(0xffffffffu, im0, o);
    }
    const double2 t = cmul(tau, make_double2(re0, im0));
#pragma unroll
    for (int k = 0; k < ES; ++k) {
      if (k >= kmax) break;
      if (gl + GS * k < m) {
        const double2 v = vcol[-GS * k];
        x[k].x -= v.x * t.x - v.y * t.y;
        x[k].y -= v.x * t.y + v.y * t.x;
      }
    }
  }
  if (!act) return;
#pragma unroll
  for (int k = 0; k < ES; ++k) {
    const int s = n - 1 - (gl + GS * k);
    if (s >= 0) V[c * ld + s] = x[k];
  }
}

// Hermitian eigensolver for one thread block: Householder tridiagonalisation
// (the zhetd2 recurrence: A <- H^H A H with H = I - tau v v^H, rank-2 updates),
// divide and conquer on the real tridiagonal (tridiag_dc), and
// back-transformation X = Q Z.  A (column-major, ld) is destroyed; on return its
// diagonal holds the eigenvalues (unsorted) and V (column-major, ld) the
// eigenvectors.  Backward stable like zheevd; O(n) barriers instead of Jacobi's
// O(n * sweeps).  n <= 256.
//  * tridiagonalisation: warp 0 forms each reflector (no block reductions), the
//    matvec p = tau A22 v is split over row x column-chunk threads, 4 barriers
//    per column;
//  * back-transformation: columns of X are independent, so each column is owned
//    by an 8-lane group that applies H_{n-2} .. H_0 with shuffle reductions and
//    no block barriers at all.
template <bool FAST = false>
__device__ void herm_eig_tridiag(double2* A, double2* V, int n, int ld, int* status) {
  constexpr int kChunks = 4;
  __shared__ double d[256], e[256];
  __shared__ double2 vv[256], pw[256], tauv[256];
  // matvec partials (tridiagonalisation), then divide-and-conquer scratch
  __shared__ double2 scratch[kChunks * 256];
  double2(*part)[256] = reinterpret_cast<double2(*)[256]>(scratch);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nthr = blockDim.x;
  const long long clk0 = clock64();
  // ---- 1. tridiagonalisation, j = 0 .. n-2 (reflector H_j acts on rows/cols j+1..n-1).
  // Two barriers per column: the rank-2 update of step j-1 (v, w in vv / pw) is
  // applied lazily inside step j's matvec (each thread updates the elements it
  // multiplies), while warp 0 forms the updated column x = A(j+1:, j), its norm
  // and the reflector scalars; then warp 0 turns (x, A x) into v = scal (x - beta e1)
  // and w = p + alpha2 v with p = tau A v = tau scal (A x - beta A(:, j+1)).
  const bool fast = FAST && n >= 16 && n <= 72 && blockDim.x == kEigFastThreads;
  if constexpr (FAST) {
    if (fast) {
    // register-resident trailing matrix, one barrier per column; V is free until
    // the divide and conquer and holds the warp-private reflector buffers
    if (n <= 32) herm_tridiag_reg<8>(A, n, ld, d, e, tauv, V, scratch);
    else if (n <= 48) herm_tridiag_reg<12>(A, n, ld, d, e, tauv, V, scratch);
    else herm_tridiag_reg<18>(A, n, ld, d, e, tauv, V, scratch);
    }
  }
  if (!fast) {
    double2* xs = part[1];  // the updated column x (warp 0's, phase A -> B)
    double2* qs = part[0];  // q = A22 x
    const int mt = nthr - 32;
    int lpr = 8;  // lanes per row of the matvec: one pass over the rows when possible
    while (lpr > 2 && (mt / lpr) < n - 1) lpr >>= 1;
    const unsigned gmask = 0xffffffffu;
    for (int j = 0; j + 1 < n; ++j) {
      const bool pend = j > 0 && (tauv[j - 1].x != 0.0 || tauv[j - 1].y != 0.0);
      const double2 z0 = make_double2(0.0, 0.0);
      const double2 vj = pend ? vv[j] : z0, wj = pend ? pw[j] : z0;
      double2 tau = z0, scal = z0;
      double beta = 0.0;
      if (warp == 0) {
        double xn = 0.0;
        double2 alpha = z0;
        for (int l = j + 1 + lane; l < n; l += 32) {
          double2 x = A[j * ld + l];
          if (pend) x = csub(x, cadd(cmulc(wj, vv[l]), cmulc(vj, pw[l])));
          xs[l] = x;
          if (l >= j + 2) xn += cnorm2(x);
          if (l == j + 1) alpha = x;
        }
        xn = warp_sum(xn);
        alpha = make_double2(__shfl_sync(0xffffffffu, alpha.x, 0), __shfl_sync(0xffffffffu, alpha.y, 0));
        if (lane == 0) d[j] = A[j * ld + j].x - (pend ? 2.0 * (vj.x * wj.x + vj.y * wj.y) : 0.0);
        if (xn == 0.0 && alpha.y == 0.0) {
          beta = alpha.x;
        } else {
          beta = -copysign(sqrt(alpha.x * alpha.x + alpha.y * alpha.y + xn), alpha.x);
          const double rb = 1.0 / beta;
          tau = make_double2((beta - alpha.x) * rb, -alpha.y * rb);
          const double2 den = make_double2(alpha.x - beta, alpha.y);  // scal = 1 / (alpha - beta)
          const double dn = 1.0 / cnorm2(den);
          scal = make_double2(den.x * dn, -den.y * dn);
        }
      } else {
        // rows i >= j+1 (lpr lanes per row, interleaved columns): apply the
        // pending update, accumulate A x, reduce over the row's lanes
        const int t = tid - 32, gl = t % lpr;
        for (int i0 = j + 1; i0 < n; i0 += mt / lpr) {
          const int i = i0 + t / lpr;
          double re0 = 0.0, im0 = 0.0, re1 = 0.0, im1 = 0.0;
          if (i < n) {
            const double2 vi = pend ? vv[i] : z0, wi = pend ? pw[i] : z0;
            int l = j + 1 + gl;
            for (; l < n; l += 2 * lpr) {
              const int l2 = l + lpr;
              const bool two = l2 < n;
              double2 a = A[l * ld + i], x = A[j * ld + l];
              double2 b = two ? A[l2 * ld + i] : z0, y = two ? A[j * ld + l2] : z0;
              if (pend) {
                const double2 vl = vv[l], wl = pw[l];
                a = csub(a, cadd(cmulc(wl, vi), cmulc(vl, wi)));
                A[l * ld + i] = a;
                x = csub(x, cadd(cmulc(wj, vl), cmulc(vj, wl)));
                if (two) {
                  const double2 vl2 = vv[l2], wl2 = pw[l2];
                  b = csub(b, cadd(cmulc(wl2, vi), cmulc(vl2, wi)));
                  A[l2 * ld + i] = b;
                  y = csub(y, cadd(cmulc(wj, vl2), cmulc(vj, wl2)));
                }
              }
              re0 += a.x * x.x - a.y * x.y;
              im0 += a.x * x.y + a.y * x.x;
              re1 += b.x * y.x - b.y * y.y;
              im1 += b.x * y.y + b.y * y.x;
            }
          }
          re0 += re1;
          im0 += im1;
          for (int o = lpr >> 1; o > 0; o >>= 1) {
            re0 += __shfl_xor_sync(gmask, re0, o);
            im0 += __shfl_xor_sync(gmask, im0, o);
          }
          if (i < n && gl == 0) qs[i] = make_double2(re0, im0);
        }
      }
      __syncthreads();
      if (warp == 0) {
        const bool zero = tau.x == 0.0 && tau.y == 0.0;
        const double2 ts = cmul(tau, scal);
        double hr = 0.0, hi = 0.0;
        if (!zero) {
          for (int l = j + 1 + lane; l < n; l += 32) {
            const double2 xl = xs[l], s = qs[l], a1 = A[(j + 1) * ld + l];  // a1: updated A(l, j+1)
            const double2 v = l == j + 1 ? make_double2(1.0, 0.0) : cmul(xl, scal);
            const double2 p = cmul(ts, make_double2(s.x - beta * a1.x, s.y - beta * a1.y));
            A[j * ld + l] = v;  // reflector kept in column j for the back-transformation
            vv[l] = v;
            pw[l] = p;
            hr += p.x * v.x + p.y * v.y;
            hi += p.x * v.y - p.y * v.x;
          }
          hr = warp_sum(hr);
          hi = warp_sum(hi);
        }
        const double2 alpha2 = cscale(cmul(tau, make_double2(hr, hi)), -0.5);
        for (int l = j + 1 + lane; l < n; l += 32) {
          if (zero) {
            vv[l] = z0;
            pw[l] = z0;
          } else {
            pw[l] = cadd(pw[l], cmul(alpha2, vv[l]));
          }
        }
        if (lane == 0) {
          e[j] = beta;
          tauv[j] = tau;
        }
      }
      __syncthreads();
    }
  }
  if (tid == 0 && !fast) {
    const bool pend = n >= 2 && (tauv[n - 2].x != 0.0 || tauv[n - 2].y != 0.0);
    const double2 vl = pend ? vv[n - 1] : make_double2(0.0, 0.0), wl = pend ? pw[n - 1] : make_double2(0.0, 0.0);
    d[n - 1] = A[(n - 1) * ld + n - 1].x - 2.0 * (vl.x * wl.x + vl.y * wl.y);
    e[n - 1] = 0.0;
  }
  __syncthreads();
  const long long clk1 = clock64();
  // ---- 2. divide and conquer on (d, e): eigenvalues in d, Z in V.x
  {
    double* sd = reinterpret_cast<double*>(scratch);  // 8 x 256 doubles
    int* si = reinterpret_cast<int*>(vv);              // vv: 4 x 256 ints
    int* sm = reinterpret_cast<int*>(pw);              // pw: 512 ints of per-merge counts
    const DcScratch S{sd, sd + 256, sd + 512, sd + 768, sd + 1024, sd + 1280, sd + 1536, sd + 1792,
                      si, si + 256, si + 512, si + 768, sm, status + 12};
    tridiag_dc(d, e, V, A, n, ld, S);
  }
  const long long clk2 = clock64();
  // ---- 3. back-transformation X = H_0 H_1 ... H_{n-2} Z, one 8-lane group per column
  if (FAST && fast) {
    if constexpr (FAST) {
      if (n <= 32) back_transform_rev<4, 8>(A, V, n, ld, tauv);
      else if (n <= 48) back_transform_rev<6, 8>(A, V, n, ld, tauv);
      else back_transform_rev<18, 4>(A, V, n, ld, tauv);
    }
  } else if (n <= 24 * 4 && 4 * n <= nthr) {
    if (n <= nthr / 8) {
      const int esb = (n + 7) / 8;
      if (esb <= 4) back_transform_reg<4, 8>(A, V, n, ld, tauv);
      else if (esb <= 8) back_transform_reg<8, 8>(A, V, n, ld, tauv);
      else back_transform_reg<12, 8>(A, V, n, ld, tauv);
    } else {
      const int esb = (n + 3) / 4;
      if (esb <= 18) back_transform_reg<18, 4>(A, V, n, ld, tauv);
      else back_transform_reg<24, 4>(A, V, n, ld, tauv);
    }
  } else {
    const int grp = tid >> 3, gl = tid & 7, ngrp = nthr >> 3;
    for (int cbase = 0; cbase < n; cbase += ngrp) {
      const int c = cbase + grp;
      const bool act = c < n;
      double2* xc = V + (act ? c : 0) * ld;
      for (int j = n - 2; j >= 0; --j) {
        const double2 tau = tauv[j];
        if (tau.x == 0.0 && tau.y == 0.0) continue;
        double re = 0.0, im = 0.0;
        if (act)
          for (int s = j + 1 + gl; s < n; s += 8) {
            const double2 v = A[j * ld + s], x = xc[s];
            re += v.x * x.x + v.y * x.y;
            im += v.x * x.y - v.y * x.x;
          }
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
          re += __shfl_xor_sync(0xffffffffu, re, o);
          im += __shfl_xor_sync(0xffffffffu, im, o);
        }
        const double2 t = cmul(tau, make_double2(re, im));
        if (act)
          for (int s = j + 1 + gl; s < n; s += 8) xc[s] = csub(xc[s], cmul(A[j * ld + s], t));
      }
    }
  }
  __syncthreads();
  if (tid == 0) {  // diagnostics: stage cycles (kcycles) in status words 8..10
    const long long clk3 = clock64();
    atomicAdd(status + 8, static_cast<int>((clk1 - clk0) / 1000));
    atomicAdd(status + 9, static_cast<int>((clk2 - clk1) / 1000));
    atomicAdd(status + 10, static_cast<int>((clk3 - clk2) / 1000));
#if PEPSB_EIG_PROF
    if constexpr (FAST)
      for (int k = 0; k < 7; ++k) atomicAdd(status + 29 + k, atomicExch(g_tri_prof + k, 0));
#endif
  }
  for (int j = tid; j < n; j += nthr) A[j * ld + j] = make_double2(d[j], 0.0);
  __syncthreads();
}

// Block-level gram_factors; X, V: n*n complex scratch each (column-major).
// Outputs (P, R, deficient, any_def) are complete after the trailing barrier.
// Largest k solved by the one-warp Jacobi under kEigAuto (divide and conquer
// above; measured: k = 4 25 us vs 38 us, k = 8 66 us vs 58 us).
constexpr int kWarpJacobiMax = 6;

template <bool FAST = false>
__device__ void gram_factors_dev(const double2* G, int n, double2* X, double2* V, double2* P, double2* R,
                                 int* deficient, int* any_def, int* status, double* lam_out = nullptr,
                                 double2* vec_out = nullptr, int solver = 0) {
  __shared__ double lam[256];
  __shared__ int order[256];
  __shared__ double hmax[2];
  const int ld = n + 1;  // padded column stride: conflict-free strided column access
  if (threadIdx.x < 2) hmax[threadIdx.x] = 0.0;
  __syncthreads();
  // Hermiticity check against the input, as eigh does (linalg.cpp:262-271).
  double herr = 0.0, scale = 0.0;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    int i = e / n, j = e % n;
    double2 a = G[i * n + j], b = G[j * n + i];
    herr = fmax(herr, hypot(a.x - b.x, a.y + b.y));
    scale = fmax(scale, hypot(a.x, a.y));
    // symmetrised 0.5 (G + G^H), stored column-major (ld = n + 1): X[j][i] = A(i, j)
    X[j * ld + i] = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
  }
  // block max via atomics on the bit patterns of non-negative doubles
  atomicMax(reinterpret_cast<unsigned long long*>(&hmax[0]), __double_as_longlong(herr));
  atomicMax(reinterpret_cast<unsigned long long*>(&hmax[1]), __double_as_longlong(scale));
  __syncthreads();
  if (threadIdx.x == 0 && hmax[0] > 1e-10 * fmax(1.0, hmax[1])) atomicOr(status, kSmallNotHermitian);
  // Exact power-of-two scaling to max |A| in [1, 2): the solvers form squares of
  // the entries (reflector norms, secular-equation terms), which overflow for
  // the Gram matrices of unnormalised states (|G| ~ 1e171 after 100 ITE steps;
  // zheevd scales the same way).  Scaling by 2^-e is exact, so eigenvectors are
  // bitwise those of the unscaled problem wherever that one does not overflow.
  const double gmax = hmax[1];
  const int gexp = (gmax > 0.0 && isfinite(gmax)) ? ilogb(gmax) : 0;
  if (gexp != 0) {
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      double2& x = X[(e / n) * ld + e % n];
      x = make_double2(scalbn(x.x, -gexp), scalbn(x.y, -gexp));
    }
    __syncthreads();
  }

  double fro = 0.0;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) fro += cnorm2(X[(e / n) * ld + e % n]);
  // Off-diagonals below the rounding level of ||G|| are noise (G itself carries
  // absolute errors ~eps ||G||, as does zheevd's output); rotating them only
  // chases noise on the small-eigenvalue block.
  // Both thresholds at n*eps: the accumulated rounding of O(n^2) rotations,
  // and the accuracy class of zheevd (|d lambda| ~ n eps ||G||).
  const double neps = static_cast<double>(n) * 2.220446049250313e-16;
  const double abs_skip = neps * sqrt(block_sum(fro));
  // Deficiency cut below is 1e-12 lambda_max >= 1e-12 max_i G_ii: an unresolved
  // block of pairs with G_pp < 1e-12 max G_ii / n has all eigenvalues under it.
  // Only when the caller needs just the kept eigenvectors (not vec_out).
  double dmax = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) dmax = fmax(dmax, X[i * ld + i].x);
  __shared__ double sh_dmax;
  if (threadIdx.x == 0) sh_dmax = 0.0;
  __syncthreads();
  atomicMax(reinterpret_cast<unsigned long long*>(&sh_dmax), __double_as_longlong(dmax));
  __syncthreads();
  const double low_skip = vec_out ? 0.0 : 1e-12 * sh_dmax / n;
  if (solver == kEigJacobi) {
    herm_jacobi(X, V, n, ld, neps, abs_skip, low_skip, 40, status);
  } else if (solver == kEigAuto && n <= kWarpJacobiMax) {
    if (threadIdx.x < 32) herm_jacobi_t<true>(X, V, n, ld, neps, abs_skip, low_skip, 40, status);
    __syncthreads();
  } else {
    herm_eig_tridiag<FAST>(X, V, n, ld, status);
  }
  for (int j = threadIdx.x; j < n; j += blockDim.x) lam[j] = scalbn(X[j * ld + j].x, gexp);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  sort_desc(lam, order, n);
  // phase of each sorted eigenvector column
  __shared__ double2 ph[256];
  for (int j = warp; j < n; j += nwarps) {
    double2 p = column_phase(V + order[j] * ld, n);
    if (lane == 0) ph[j] = p;
  }
  __syncthreads();
  const double lmax = lam[order[0]];
  if (threadIdx.x == 0 && P) {  // (P == nullptr: plain eigh, no Gram factors)
    if (!(lmax > 0.0)) atomicOr(status, kSmallZeroGram);
    int anyd = 0;
    for (int j = 0; j < n; ++j) {
      int d = lam[order[j]] < 1e-12 * lmax;
      deficient[j] = d;
      anyd |= d;
    }
    *any_def = anyd;
  }
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    const double lj = fmax(lam[order[j]], 1e-12 * lmax);
    // eigenvector column j (sorted), phase fixed: x_ij * conj(phase_j)
    const double2 xij = cmulc(ph[j], V[order[j] * ld + i]);
    if (P) {
      const double isq = 1.0 / sqrt(lj);
      P[i * n + j] = cscale(xij, isq);
      // R row j = sqrt(l_j) conj(column j of X): R[j][i] = sqrt(l_j) conj(x_ij)
      R[j * n + i] = cscale(cconj(xij), sqrt(lj));
    }
    if (vec_out) vec_out[i * n + j] = xij;  // eigenvector j (descending), phase-fixed
  }
  if (lam_out)
    for (int j = threadIdx.x; j < n; j += blockDim.x) lam_out[j] = lam[order[j]];
  __syncthreads();
}

// SMEM: the two n x (n+1) work matrices live in dynamic shared memory and the
// pointers derive from the __shared__ array, so the inlined solvers use
// LDS/STS instead of generic loads (which the profile showed waiting on the
// long scoreboard); otherwise they live in the global `work` buffer.
template <bool SMEM, int NT>
__global__ void __launch_bounds__(NT) gram_factors_kernel(const double2* G, int n, double2* P,
                                                                double2* R, int* deficient,
                                                                int* any_def, int* status,
                                                                double2* work, int use_jacobi, double* lam_out,
                                                                double2* vec_out) {
  extern __shared__ __align__(16) unsigned char sm[];
  double2* X = SMEM ? reinterpret_cast<double2*>(sm) : work;  // column-major n x (n+1)
  // NT == kEigFastThreads: the register-resident tridiagonalisation / back-transformation
  gram_factors_dev<SMEM && NT == kEigFastThreads>(G, n, X, X + n * (n + 1), P, R, deficient, any_def, status, lam_out,
                                                  vec_out, use_jacobi & 0xff);
}

// ------------------------------------------------------------------ Cholesky

__global__ void __launch_bounds__(kThreads) chol_kernel(const double2* G, int n, double shift_rel,
                                                        double2* Rout, double2* Rinv, int* status,
                                                        bool in_place) {
  extern __shared__ __align__(16) unsigned char sm[];
  // row-major n x n working copy: shared memory, or Rout itself when n x n
  // complex does not fit (k > 113; every access below is then global)
  double2* A = in_place ? Rout : reinterpret_cast<double2*>(sm);
  __shared__ double tr;
  __shared__ int bad;
  if (threadIdx.x == 0) { tr = 0.0; bad = 0; }
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    int i = e / n, j = e % n;
    // symmetrise from the upper triangle
    double2 v = j >= i ? G[i * n + j] : cconj(G[j * n + i]);
    A[e] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < n; ++i) t = fmax(t, A[i * n + i].x);
    tr = t;  // largest diagonal entry
  }
  __syncthreads();
  // A pivot below pivot_rel * max_diag counts as a breakdown: the Gram matrix is
  // then (close to) rank deficient where the reference's eigh route would clamp.
  const double floor = shift_rel * tr;
  for (int k = 0; k < n; ++k) {
    const double piv = A[k * n + k].x;
    if (!(piv > floor) || !(piv > 0.0)) {
      if (threadIdx.x == 0) bad = 1;
      __syncthreads();
      break;
    }
    const double rkk = sqrt(piv);
    __syncthreads();
    for (int j = k + threadIdx.x; j < n; j += blockDim.x)
      A[k * n + j] = j == k ? make_double2(rkk, 0.0) : cscale(A[k * n + j], 1.0 / rkk);
    __syncthreads();
    const int rem = n - k - 1;
    for (int e = threadIdx.x; e < rem * rem; e += blockDim.x) {
      const int i = k + 1 + e / rem, j = k + 1 + e % rem;
      if (j < i) continue;
      A[i * n + j] = csub(A[i * n + j], cmulc(A[k * n + i], A[k * n + j]));
    }
    __syncthreads();
  }
  if (bad) {
    if (threadIdx.x == 0) atomicOr(status, kSmallCholBreakdown);
    return;
  }
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    int i = e / n, j = e % n;
    Rout[e] = j >= i ? A[e] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  // Rinv column c by back substitution (one thread per column).
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    for (int i = n - 1; i > c; --i) Rinv[i * n + c] = make_double2(0.0, 0.0);
    // x_c = 1 / R_cc
    double2 rcc = A[c * n + c];
    Rinv[c * n + c] = make_double2(1.0 / rcc.x, 0.0);
    for (int i = c - 1; i >= 0; --i) {
      double2 s = make_double2(0.0, 0.0);
      for (int l = i + 1; l <= c; ++l) s = cadd(s, cmul(A[i * n + l], Rinv[l * n + c]));
      Rinv[i * n + c] = cscale(s, -1.0 / A[i * n + i].x);
    }
  }
}

// ------------------------------------------------------------------ small SVD

__device__ void complete_unit_columns(double2* X, int rows, int cols, int ld, const int* bad,
                                      int* status) {
  // Orthonormal completion of flagged columns by Gram-Schmidt of canonical
  // basis vectors (same rule as decomposition.cpp:88-115), column-major X.
  int next_basis = 0;
  for (int j = 0; j < cols; ++j) {
    if (!bad[j]) continue;
    bool done = false;
    for (; next_basis <= rows && !done; ++next_basis) {
      if (next_basis == rows) {
        if (threadIdx.x == 0) atomicOr(status, kSmallCompletionExhausted);
        return;
      }
      double2* v = X + static_cast<int64_t>(j) * ld;
      for (int r = threadIdx.x; r < rows; r += blockDim.x)
        v[r] = make_double2(r == next_basis ? 1.0 : 0.0, 0.0);
      __syncthreads();
      for (int pass = 0; pass < 2; ++pass) {
        for (int c = 0; c < cols; ++c) {
          if (c == j || (bad[c] && c > j)) continue;
          const double2* qc = X + static_cast<int64_t>(c) * ld;
          double pr = 0.0, pi = 0.0;
          for (int r = threadIdx.x; r < rows; r += blockDim.x) {
            double2 q = qc[r], x = v[r];
            pr += q.x * x.x + q.y * x.y;
            pi += q.x * x.y - q.y * x.x;
          }
          pr = block_sum(pr);
          pi = block_sum(pi);
          const double2 proj = make_double2(pr, pi);
          for (int r = threadIdx.x; r < rows; r += blockDim.x) v[r] = csub(v[r], cmul(proj, qc[r]));
          __syncthreads();
        }
      }
      double nn = 0.0;
      for (int r = threadIdx.x; r < rows; r += blockDim.x) nn += cnorm2(v[r]);
      const double nrm = sqrt(block_sum(nn));
      if (nrm > 0.1) {
        for (int r = threadIdx.x; r < rows; r += blockDim.x) v[r] = cscale(v[r], 1.0 / nrm);
        done = true;
      }
      __syncthreads();
    }
  }
}

struct SvdArgs {
  const double2* A;
  int64_t sa;
  int m, n, lda;
  double2* U;
  int64_t su;
  double* s;
  int64_t ss;
  double2* Vh;
  int64_t sv;
  int* status;
  double2* work;
  int64_t work_stride;
};

// Block-level thin SVD of a row-major m x n matrix A (leading dim lda):
// A = U diag(s) Vh, U m x k, Vh k x n (both row-major, k = min(m, n)).
// X: scratch of max(m,n)*min(m,n) + min(m,n)^2 complex.
__device__ void small_svd_dev(const double2* A, int m_, int n_, int lda, double2* X, double2* U, double* s,
                              double2* Vh, int* status) {
  struct {
    int m, n, lda;
    int* status;
  } a{m_, n_, lda, status};
  const bool tall = a.m >= a.n;
  const int mr = tall ? a.m : a.n;  // rows of the working matrix
  const int nc = tall ? a.n : a.m;  // its columns (= k)
  double2* V = X + static_cast<int64_t>(mr) * nc;
  __shared__ double sig[256];
  __shared__ int order[256];
  __shared__ int bad[256];
  __shared__ double2 ph[256];
  // Working matrix W (mr x nc) column-major: tall -> W = A, wide -> W = A^H.
  for (int e = threadIdx.x; e < a.m * a.n; e += blockDim.x) {
    const int i = e / a.n, j = e % a.n;
    const double2 v = A[static_cast<int64_t>(i) * a.lda + j];
    if (tall) X[static_cast<int64_t>(j) * mr + i] = v;      // col j, row i
    else X[static_cast<int64_t>(i) * mr + j] = cconj(v);     // A^H: col i, row j
  }
  __syncthreads();
  // skip rotations between columns whose inner product is below (eps ||A||_F)^2:
  // numerically-null columns (rank-deficient A) are left alone, as gesdd would.
  double fro = 0.0;
  for (int e = threadIdx.x; e < mr * nc; e += blockDim.x) fro += cnorm2(X[e]);
  const double abs_skip = 4.930380657631324e-32 * block_sum(fro);
  onesided_jacobi(X, mr, nc, mr, V, nc, 8.0 * 2.220446049250313e-16 * sqrt(static_cast<double>(mr)), abs_skip, 60,
                  a.status);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int j = warp; j < nc; j += nwarps) {
    double s = 0.0;
    for (int i = lane; i < mr; i += 32) s += cnorm2(X[static_cast<int64_t>(j) * mr + i]);
    s = warp_sum(s);
    if (lane == 0) sig[j] = sqrt(s);
  }
  __syncthreads();
  sort_desc(sig, order, nc);
  const double smax = sig[order[0]];
  // normalise columns; flag numerically-zero ones for orthonormal completion
  for (int j = warp; j < nc; j += nwarps) {
    const double sj = sig[j];
    const bool zero = !(sj > 0.0) || sj <= 1e-300 || (smax > 0.0 && sj < 1e-300 * smax);
    if (lane == 0) bad[j] = zero;
    if (!zero)
      for (int i = lane; i < mr; i += 32) X[static_cast<int64_t>(j) * mr + i] = cscale(X[static_cast<int64_t>(j) * mr + i], 1.0 / sj);
  }
  __syncthreads();
  // completion works in sorted order semantics only through the flags; the
  // unsorted storage is fine since completion orthogonalises against all.
  complete_unit_columns(X, mr, nc, mr, bad, a.status);
  __syncthreads();
  // U/Vh in sorted order.  tall: U = X (m x k), V = V (n x k) -> Vh = V^H.
  //                        wide: U = V (m x k),  Vh = X^H.
  const double2* Ucols = tall ? X : V;   // column-major, column stride = rows of U
  const int urows = a.m;
  const double2* Vcols = tall ? V : X;   // column-major n x k
  const int vrows = a.n;
  for (int j = warp; j < nc; j += nwarps) {
    double2 p = column_phase(Ucols + static_cast<int64_t>(order[j]) * urows, urows);
    if (lane == 0) ph[j] = p;
  }
  __syncthreads();
  const int k = nc;
  for (int e = threadIdx.x; e < urows * k; e += blockDim.x) {
    const int i = e / k, j = e % k;
    U[static_cast<int64_t>(i) * k + j] = cmulc(ph[j], Ucols[static_cast<int64_t>(order[j]) * urows + i]);
  }
  for (int e = threadIdx.x; e < k * vrows; e += blockDim.x) {
    const int j = e / vrows, c = e % vrows;
    // Vh[j][c] = conj(Vcol_j[c]) * phase_j
    Vh[static_cast<int64_t>(j) * vrows + c] = cmul(cconj(Vcols[static_cast<int64_t>(order[j]) * vrows + c]), ph[j]);
  }
  for (int j = threadIdx.x; j < k; j += blockDim.x) s[j] = sig[order[j]];
  __syncthreads();
}

// QR-preconditioned variant (Drmac-Veselic): W = Q R by Householder, then the
// one-sided Jacobi runs on the lower-triangular R^H, whose columns start much
// closer to orthogonal (15 -> ~6 sweeps on the 32 x 32 simple-update blocks).
// R^H V2 = U2 S gives W = (Q V2) S U2^H.  Same outputs and conventions as
// small_svd_dev (U columns phase-fixed, sorted descending); used by the
// batched simple update, where only the leading `rank` triplets (nonzero
// sigma) are consumed.  Scratch: X (mr x nc + nc x nc), Vt (nc x nc), Uc
// (mr x nc) -- Uc may alias A (A is read first).
__device__ void small_svd_qr_dev(const double2* A, int m, int n, int lda, double2* X, double2* Vt, double2* Uc,
                                 double2* U, double* s, double2* Vh, int* status) {
  const bool tall = m >= n;
  const int mr = tall ? m : n, nc = tall ? n : m;
  double2* X2 = X + static_cast<int64_t>(mr) * nc;  // R^H, nc x nc column-major
  __shared__ double sig[256];
  __shared__ int order[256];
  __shared__ int bad[256];
  __shared__ double2 ph[256];
  __shared__ double2 rdiag[256];
  __shared__ double tauq[256];
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    const double2 v = A[static_cast<int64_t>(i) * lda + j];
    if (tall) X[static_cast<int64_t>(j) * mr + i] = v;
    else X[static_cast<int64_t>(i) * mr + j] = cconj(v);
  }
  __syncthreads();
  double fro = 0.0;
  for (int e = threadIdx.x; e < mr * nc; e += blockDim.x) fro += cnorm2(X[e]);
  const double fro2 = block_sum(fro);
  // ---- Householder QR of X (column j: reflector v_j in X[j:, j], R_jj in rdiag)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int j = 0; j < nc; ++j) {
    double2* xj = X + static_cast<int64_t>(j) * mr;
    double part = 0.0;
    for (int r = j + threadIdx.x; r < mr; r += blockDim.x) part += cnorm2(xj[r]);
    const double alpha = sqrt(block_sum(part));
    if (!(alpha > 0.0)) {
      if (threadIdx.x == 0) {
        rdiag[j] = make_double2(0.0, 0.0);
        tauq[j] = 0.0;
      }
      __syncthreads();
      continue;
    }
    const double2 x0 = xj[j];
    const double ax0 = hypot(x0.x, x0.y);
    const double2 phs = ax0 > 0.0 ? make_double2(x0.x / ax0, x0.y / ax0) : make_double2(1.0, 0.0);
    const double tau = 1.0 / (alpha * (alpha + ax0));
    __syncthreads();
    if (threadIdx.x == 0) {
      xj[j] = make_double2(x0.x + phs.x * alpha, x0.y + phs.y * alpha);
      rdiag[j] = make_double2(-phs.x * alpha, -phs.y * alpha);
      tauq[j] = tau;
    }
    __syncthreads();
    for (int c = j + 1 + warp; c < nc; c += nwarps) {
      double2* xc = X + static_cast<int64_t>(c) * mr;
      double wr = 0.0, wi = 0.0;
      for (int r = j + lane; r < mr; r += 32) {
        const double2 v = xj[r], a = xc[r];
        wr += v.x * a.x + v.y * a.y;
        wi += v.x * a.y - v.y * a.x;
      }
      wr = warp_sum(wr) * tau;
      wi = warp_sum(wi) * tau;
      for (int r = j + lane; r < mr; r += 32) {
        const double2 v = xj[r];
        xc[r] = csub(xc[r], make_double2(v.x * wr - v.y * wi, v.x * wi + v.y * wr));
      }
    }
    __syncthreads();
  }
  // ---- X2 = R^H (lower triangular): X2[r][c] = conj(R[c][r])
  for (int e = threadIdx.x; e < nc * nc; e += blockDim.x) {
    const int c = e / nc, r = e % nc;  // column c, row r of X2
    double2 v = make_double2(0.0, 0.0);
    if (r == c) v = cconj(rdiag[c]);
    else if (r > c) v = cconj(X[static_cast<int64_t>(r) * mr + c]);  // R[c][r]: row c of column r
    X2[static_cast<int64_t>(c) * nc + r] = v;
  }
  __syncthreads();
  const double abs_skip = 4.930380657631324e-32 * fro2;
  onesided_jacobi(X2, nc, nc, nc, Vt, nc, 8.0 * 2.220446049250313e-16 * sqrt(static_cast<double>(nc)), abs_skip, 60,
                  status);
  for (int j = warp; j < nc; j += nwarps) {
    double t = 0.0;
    for (int i = lane; i < nc; i += 32) t += cnorm2(X2[static_cast<int64_t>(j) * nc + i]);
    t = warp_sum(t);
    if (lane == 0) sig[j] = sqrt(t);
  }
  __syncthreads();
  sort_desc(sig, order, nc);
  const double smax = sig[order[0]];
  for (int j = warp; j < nc; j += nwarps) {
    const double sj = sig[j];
    const bool zero = !(sj > 0.0) || sj <= 1e-300 || (smax > 0.0 && sj < 1e-300 * smax);
    if (lane == 0) bad[j] = zero;
    if (!zero)
      for (int i = lane; i < nc; i += 32) X2[static_cast<int64_t>(j) * nc + i] = cscale(X2[static_cast<int64_t>(j) * nc + i], 1.0 / sj);
  }
  __syncthreads();
  complete_unit_columns(X2, nc, nc, nc, bad, status);
  __syncthreads();
  // ---- Uc = Q [Vt; 0] (mr x nc, column-major): H_0 ... H_{nc-1} applied to each column
  for (int e = threadIdx.x; e < mr * nc; e += blockDim.x) {
    const int c = e / mr, r = e % mr;
    Uc[e] = r < nc ? Vt[static_cast<int64_t>(c) * nc + r] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int c = warp; c < nc; c += nwarps) {
    double2* uc = Uc + static_cast<int64_t>(c) * mr;
    for (int j = nc - 1; j >= 0; --j) {
      const double tau = tauq[j];
      if (tau == 0.0) continue;
      const double2* vj = X + static_cast<int64_t>(j) * mr;
      double wr = 0.0, wi = 0.0;
      for (int r = j + lane; r < mr; r += 32) {
        const double2 v = vj[r], a = uc[r];
        wr += v.x * a.x + v.y * a.y;
        wi += v.x * a.y - v.y * a.x;
      }
      wr = warp_sum(wr) * tau;
      wi = warp_sum(wi) * tau;
      for (int r = j + lane; r < mr; r += 32) {
        const double2 v = vj[r];
        uc[r] = csub(uc[r], make_double2(v.x * wr - v.y * wi, v.x * wi + v.y * wr));
      }
    }
  }
  __syncthreads();
  // W = (Q Vt) S U2^H with U2 = X2.  tall (W = A): U_A = Uc, V_A = X2;
  // wide (W = A^H): U_A = X2, V_A = Uc.
  const double2* Ucols = tall ? Uc : X2;
  const int urows = m, uld = tall ? mr : nc;
  const double2* Vcols = tall ? X2 : Uc;
  const int vrows = n, vld = tall ? nc : mr;
  for (int j = warp; j < nc; j += nwarps) {
    double2 p = column_phase(Ucols + static_cast<int64_t>(order[j]) * uld, urows);
    if (lane == 0) ph[j] = p;
  }
  __syncthreads();
  const int k = nc;
  for (int e = threadIdx.x; e < urows * k; e += blockDim.x) {
    const int i = e / k, j = e % k;
    U[static_cast<int64_t>(i) * k + j] = cmulc(ph[j], Ucols[static_cast<int64_t>(order[j]) * uld + i]);
  }
  for (int e = threadIdx.x; e < k * vrows; e += blockDim.x) {
    const int j = e / vrows, c = e % vrows;
    Vh[static_cast<int64_t>(j) * vrows + c] = cmul(cconj(Vcols[static_cast<int64_t>(order[j]) * vld + c]), ph[j]);
  }
  for (int j = threadIdx.x; j < k; j += blockDim.x) s[j] = sig[order[j]];
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads) small_svd_kernel(const SvdArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int b = blockIdx.x;
  double2* X = a.work ? a.work + b * a.work_stride : reinterpret_cast<double2*>(sm);
  small_svd_dev(a.A + b * a.sa, a.m, a.n, a.lda, X, a.U + b * a.su, a.s + b * a.ss, a.Vh + b * a.sv, a.status);
}

// ------------------------------------------------------------------ completion of big Q

// ------------------------------------------------------------------ TSQR R factor

// Householder QR of row block b (rows [b*rpb, b*rpb + rpb)) of a row-major
// rows x k matrix; writes the k x k upper-triangular R of the block (zero-padded
// when the block has fewer than k rows).  Column-major working copy in shared
// memory (or `work` + b * rpb * k when it does not fit).  Backward stable
// like zgeqrf (linalg.cpp:93), and unaffected by rank deficiency.
__global__ void __launch_bounds__(kThreads) householder_r_kernel(const double2* A, int64_t rows, int k, int rpb,
                                                                 double2* Rout, double2* work) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ double2 rdiag[256];
  const int b = blockIdx.x;
  const int64_t r0 = static_cast<int64_t>(b) * rpb;
  const int m = static_cast<int>(rows - r0 < rpb ? rows - r0 : rpb);
  const int mm = max(m, k);
  double2* X = work ? work + static_cast<int64_t>(b) * max(rpb, k) * k : reinterpret_cast<double2*>(sm);
  for (int e = threadIdx.x; e < mm * k; e += blockDim.x) {
    const int r = e / k, c = e % k;
    X[static_cast<int64_t>(c) * mm + r] = r < m ? A[(r0 + r) * k + c] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int j = 0; j < k; ++j) {
    double2* xj = X + static_cast<int64_t>(j) * mm;
    double part = 0.0;
    for (int r = j + threadIdx.x; r < mm; r += blockDim.x) part += cnorm2(xj[r]);
    const double alpha = sqrt(block_sum(part));
    if (!(alpha > 0.0)) {
      if (threadIdx.x == 0) rdiag[j] = make_double2(0.0, 0.0);
      __syncthreads();
      continue;
    }
    const double2 x0 = xj[j];
    const double ax0 = hypot(x0.x, x0.y);
    const double2 ph = ax0 > 0.0 ? make_double2(x0.x / ax0, x0.y / ax0) : make_double2(1.0, 0.0);
    const double tau = 1.0 / (alpha * (alpha + ax0));  // 2 / (v^H v)
    __syncthreads();
    if (threadIdx.x == 0) {
      xj[j] = make_double2(x0.x + ph.x * alpha, x0.y + ph.y * alpha);
      rdiag[j] = make_double2(-ph.x * alpha, -ph.y * alpha);
    }
    __syncthreads();
    for (int c = j + 1 + warp; c < k; c += nwarps) {
      double2* xc = X + static_cast<int64_t>(c) * mm;
      double wr = 0.0, wi = 0.0;
      for (int r = j + lane; r < mm; r += 32) {
        const double2 v = xj[r], a = xc[r];
        wr += v.x * a.x + v.y * a.y;  // conj(v) a
        wi += v.x * a.y - v.y * a.x;
      }
      wr = warp_sum(wr) * tau;
      wi = warp_sum(wi) * tau;
      for (int r = j + lane; r < mm; r += 32) {
        const double2 v = xj[r];
        xc[r] = csub(xc[r], make_double2(v.x * wr - v.y * wi, v.x * wi + v.y * wr));
      }
    }
    __syncthreads();
  }
  double2* R = Rout + static_cast<int64_t>(b) * k * k;
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int i = e / k, c = e % k;
    R[e] = c > i ? X[static_cast<int64_t>(c) * mm + i] : (c == i ? rdiag[i] : make_double2(0.0, 0.0));
  }
}

__global__ void __launch_bounds__(kThreads) complete_columns_kernel(double2* Q, int64_t rows, int cols,
                                                                    const int* deficient,
                                                                    const int* any_def, int* status) {
  if (*any_def == 0) return;
  int64_t next_basis = 0;
  for (int j = 0; j < cols; ++j) {
    if (!deficient[j]) continue;
    bool done = false;
    for (; next_basis <= rows && !done; ++next_basis) {
      if (next_basis == rows) {
        if (threadIdx.x == 0) atomicOr(status, kSmallCompletionExhausted);
        return;
      }
      // use column j of Q as the work vector (it is overwritten anyway)
      for (int64_t r = threadIdx.x; r < rows; r += blockDim.x)
        Q[r * cols + j] = make_double2(r == next_basis ? 1.0 : 0.0, 0.0);
      __syncthreads();
      for (int pass = 0; pass < 2; ++pass) {
        for (int c = 0; c < cols; ++c) {
          if (c == j || (deficient[c] && c > j)) continue;
          double pr = 0.0, pi = 0.0;
          for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) {
            double2 q = Q[r * cols + c], x = Q[r * cols + j];
            pr += q.x * x.x + q.y * x.y;
            pi += q.x * x.y - q.y * x.x;
          }
          pr = block_sum(pr);
          pi = block_sum(pi);
          const double2 proj = make_double2(pr, pi);
          for (int64_t r = threadIdx.x; r < rows; r += blockDim.x)
            Q[r * cols + j] = csub(Q[r * cols + j], cmul(proj, Q[r * cols + c]));
          __syncthreads();
        }
      }
      double nn = 0.0;
      for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) nn += cnorm2(Q[r * cols + j]);
      const double nrm = sqrt(block_sum(nn));
      if (nrm > 0.1) {
        for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) Q[r * cols + j] = cscale(Q[r * cols + j], 1.0 / nrm);
        done = true;
      }
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------------ simple update (state.cpp:89-204)
//
// One thread block per site (reduce / restore) or per bond (split); a whole
// colour of disjoint bonds is one launch of each, ragged shapes included.

__global__ void __launch_bounds__(512) su_reduce_kernel(const SuSiteDesc* descs, int* status) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ int anyd;
  const SuSiteDesc D = descs[blockIdx.x];
  const int E = D.e[0] * D.e[1] * D.e[2], S = D.d * D.s;
  double2* Y = reinterpret_cast<double2*>(sm);  // column-major E x S (site in env form)
  for (int idx = threadIdx.x; idx < E * S; idx += blockDim.x) {
    const int c = idx / E, e = idx % E;
    const int i2 = e % D.e[2], t = e / D.e[2], i1 = t % D.e[1], i0 = t / D.e[1];
    const int p = c / D.s, q = c % D.s;
    Y[idx] = D.src[i0 * D.str[0] + i1 * D.str[1] + i2 * D.str[2] + p * D.str[3] + q * D.str[4]];
  }
  __syncthreads();
  if (!D.reduced) {  // env < d * shared: no QR (state.cpp:132-136), R = site (E, d, s)
    for (int idx = threadIdx.x; idx < E * S; idx += blockDim.x) D.R[idx] = Y[(idx % S) * E + idx / S];
    return;
  }
  double2* G = Y + E * S;
  double2* X = G + S * S;
  double2* V = X + S * (S + 1);
  double2* P = V + S * (S + 1);
  double2* Rm = P + S * S;
  int* def = reinterpret_cast<int*>(Rm + S * S);
  for (int idx = threadIdx.x; idx < S * S; idx += blockDim.x) {
    const int i = idx / S, j = idx % S;
    double re = 0.0, im = 0.0;
    for (int e = 0; e < E; ++e) {
      const double2 a = Y[i * E + e], b = Y[j * E + e];
      re += a.x * b.x + a.y * b.y;
      im += a.x * b.y - a.y * b.x;
    }
    G[idx] = make_double2(re, im);
  }
  __syncthreads();
  // gram_orthogonalize(site as (env, d*s)) — decomposition.cpp:160-193
  gram_factors_dev(G, S, X, V, P, Rm, def, &anyd, status, nullptr, nullptr, kEigDivideConquer);
  for (int idx = threadIdx.x; idx < E * S; idx += blockDim.x) {
    const int j = idx / E, e = idx % E;
    double2 acc = make_double2(0.0, 0.0);
    for (int i = 0; i < S; ++i) acc = cadd(acc, cmul(Y[i * E + e], P[i * S + j]));
    D.Q[idx] = acc;  // column-major
  }
  __syncthreads();
  if (anyd) complete_unit_columns(D.Q, E, S, E, def, status);
  for (int idx = threadIdx.x; idx < S * S; idx += blockDim.x) D.R[idx] = Rm[idx];
}

__global__ void __launch_bounds__(512) su_split_kernel(const SuBondDesc* descs, int* ranks, int* status,
                                                       unsigned long long* degenerate, bool qr_precondition) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ int rank_sh;
  const SuBondDesc B = descs[blockIdx.x];
  const int d = B.d, m = B.ta * d, n = d * B.tb, k = min(m, n);
  double2* M = reinterpret_cast<double2*>(sm);
  double2* U = M + m * n;
  double2* Vh = U + m * k;
  double2* X = Vh + k * n;
  double* sv = reinterpret_cast<double*>(X + max(m, n) * k + k * k);
  // M[(a,o),(p,b)] = sum_{i,j,q} g[o,p,i,j] Ra[a,i,q] Rb[b,j,q]   (network {g, Ra, Rb}, state.cpp:192-194)
  for (int idx = threadIdx.x; idx < m * n; idx += blockDim.x) {
    const int row = idx / n, col = idx % n;
    const int a = row / d, o = row % d, p = col / B.tb, b = col % B.tb;
    double2 acc = make_double2(0.0, 0.0);
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) {
        const double2 g = B.gate[((o * d + p) * d + i) * d + j];
        double2 sum = make_double2(0.0, 0.0);
        for (int q = 0; q < B.s; ++q)
          sum = cadd(sum, cmul(B.Ra[(a * d + i) * B.s + q], B.Rb[(b * d + j) * B.s + q]));
        acc = cadd(acc, cmul(g, sum));
      }
    M[idx] = acc;
  }
  __syncthreads();
  if (qr_precondition) small_svd_qr_dev(M, m, n, n, X, Vh, M, U, sv, Vh, status);
  else small_svd_dev(M, m, n, n, X, U, sv, Vh, status);
  if (threadIdx.x == 0) {  // retained_rank (decomposition.cpp:20-29)
    int above = 0;
    for (int j = 0; j < k; ++j) above += sv[j] >= B.cutoff * sv[0];
    int64_t r = above;
    if (B.cap > 0 && B.cap < r) r = B.cap;
    rank_sh = static_cast<int>(r < 1 ? 1 : r);
    ranks[blockIdx.x] = rank_sh;
    // truncation through a (numerically) degenerate pair: the kept subspace is
    // rounding-dependent -- counted and reported, not hidden
    if (degenerate && r >= 1 && r < above && sv[r - 1] - sv[r] <= 1e-10 * sv[r - 1]) atomicAdd(degenerate, 1ull);
  }
  __syncthreads();
  const int rank = rank_sh;
  // Absorb::split: t1 = U sqrt(S) as (a, o, rho); t2 = sqrt(S) Vh as (b, p, rho)
  for (int idx = threadIdx.x; idx < m * rank; idx += blockDim.x) {
    const int row = idx / rank, r = idx % rank;
    B.t1[row * B.rmax + r] = cscale(U[row * k + r], sqrt(sv[r]));
  }
  for (int idx = threadIdx.x; idx < n * rank; idx += blockDim.x) {
    const int col = idx / rank, r = idx % rank;  // col = (p, b)
    const int p = col / B.tb, b = col % B.tb;
    B.t2[(b * d + p) * B.rmax + r] = cscale(Vh[r * n + col], sqrt(sv[r]));
  }
}

__global__ void __launch_bounds__(256) su_restore_kernel(const SuRestoreDesc* descs, const int* ranks) {
  const SuRestoreDesc D = descs[blockIdx.x];
  const int rank = ranks[D.bond];
  const int E = D.e[0] * D.e[1] * D.e[2];
  for (int idx = threadIdx.x; idx < E * D.d * rank; idx += blockDim.x) {
    const int e = idx / (D.d * rank), rem = idx % (D.d * rank), o = rem / rank, r = rem % rank;
    double2 v;
    if (D.reduced) {  // contract("et,tov->eov", q, t) (state.cpp:150-157)
      v = make_double2(0.0, 0.0);
      for (int c = 0; c < D.S; ++c) v = cadd(v, cmul(D.Q[c * E + e], D.t[(c * D.d + o) * D.rmax + r]));
    } else {
      v = D.t[(e * D.d + o) * D.rmax + r];
    }
    const int i2 = e % D.e[2], t = e / D.e[2], i1 = t % D.e[1], i0 = t / D.e[1];
    D.dst[i0 * D.dstr[0] + i1 * D.dstr[1] + i2 * D.dstr[2] + o * D.dstr[3] + r * D.dstr[4]] = v;
  }
}

__global__ void su_one_site_kernel(const SuOneSiteDesc* descs) {
  const SuOneSiteDesc D = descs[blockIdx.x];
  for (int64_t idx = threadIdx.x; idx < D.d * D.rest; idx += blockDim.x) {
    const int64_t i = idx / D.rest, r = idx % D.rest;
    double2 acc = make_double2(0.0, 0.0);
    for (int j = 0; j < D.d; ++j) acc = cadd(acc, cmul(D.gate[i * D.d + j], D.src[j * D.rest + r]));
    D.dst[idx] = acc;  // contract("ij,juldr->iuldr") (state.cpp:75-85)
  }
}

// hermitian_function(coeff*H, exp(-tau x)) (linalg.cpp:297-314) for n <= 16:
// serial two-sided Jacobi in one thread (gate construction, negligible work).
__global__ void herm_exp_kernel(const double2* H, int n, double coeff, double tau, double2* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double2 A[16 * 16], V[16 * 16];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const double2 a = H[i * n + j], b = H[j * n + i];
      A[i * n + j] = make_double2(0.5 * coeff * (a.x + b.x), 0.5 * coeff * (a.y - b.y));
      V[i * n + j] = make_double2(i == j ? 1.0 : 0.0, 0.0);
    }
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        tot += cnorm2(A[i * n + j]);
        if (i != j) off += cnorm2(A[i * n + j]);
      }
    if (!(off > 1e-32 * tot)) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double2 apq = A[p * n + q];
        const double ag = hypot(apq.x, apq.y);
        if (!(ag > 1e-300)) continue;
        const double tau_ = (A[q * n + q].x - A[p * n + p].x) / (2.0 * ag);
        const double t = (tau_ >= 0.0 ? 1.0 : -1.0) / (fabs(tau_) + sqrt(1.0 + tau_ * tau_));
        const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
        const double2 e = make_double2(apq.x / ag, apq.y / ag), ec = cconj(e);
        for (int k = 0; k < n; ++k) {  // columns p, q
          const double2 akp = A[k * n + p], akq = cmul(A[k * n + q], ec);
          A[k * n + p] = csub(cscale(akp, c), cscale(akq, s));
          A[k * n + q] = cadd(cscale(akp, s), cscale(akq, c));
          const double2 vkp = V[k * n + p], vkq = cmul(V[k * n + q], ec);
          V[k * n + p] = csub(cscale(vkp, c), cscale(vkq, s));
          V[k * n + q] = cadd(cscale(vkp, s), cscale(vkq, c));
        }
        for (int k = 0; k < n; ++k) {  // rows p, q
          const double2 apk = A[p * n + k], aqk = cmul(A[q * n + k], e);
          A[p * n + k] = csub(cscale(apk, c), cscale(aqk, s));
          A[q * n + k] = cadd(cscale(apk, s), cscale(aqk, c));
        }
        A[p * n + q] = A[q * n + p] = make_double2(0.0, 0.0);
      }
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double2 acc = make_double2(0.0, 0.0);
      for (int l = 0; l < n; ++l) acc = cadd(acc, cscale(cmulc(V[j * n + l], V[i * n + l]), exp(-tau * A[l * n + l].x)));
      out[i * n + j] = acc;  // X f(L) X^H
    }
}

}  // namespace

void su_reduce(const SuSiteDesc* d, int n, size_t smem, int* status, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    PEPSB_CUDA(cudaFuncSetAttribute(su_reduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 176 * 1024));
    attr = true;
  }
  if (n == 0) return;
  su_reduce_kernel<<<n, 512, smem, st>>>(d, status);
  PEPSB_LAUNCH();
}

void su_split(const SuBondDesc* d, int n, size_t smem, int* ranks, int* status, unsigned long long* degenerate,
              cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    PEPSB_CUDA(cudaFuncSetAttribute(su_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  if (n == 0) return;
  // 512 threads: one warp per Jacobi pair of a 32 x 32 block (16 pairs per
  // round); PEPSB_SU_THREADS=256 restores two pairs per warp
  static const int threads = [] {
    const char* e = getenv("PEPSB_SU_THREADS");
    const int v = e ? atoi(e) : 512;
    return v == 256 ? 256 : 512;
  }();
  // QR-preconditioned Jacobi: opt-in (PEPSB_SU_QR=1).  Measured on config 4:
  // sweeps 1470 -> 1152 per ITE step, step 4.69 -> 4.28 ms, but its different
  // rounding moves the rounding-sensitive truncations (degenerate clusters of
  // the Neel-start ITE) beyond the 1e-8 parity bar, so the plain one-sided
  // Jacobi stays the default.
  static const bool qr = [] {
    const char* e = getenv("PEPSB_SU_QR");
    return e && e[0] == '1';
  }();
  su_split_kernel<<<n, threads, smem, st>>>(d, ranks, status, degenerate, qr);
  PEPSB_LAUNCH();
}

void su_restore(const SuRestoreDesc* d, int n, const int* ranks, cudaStream_t st) {
  if (n == 0) return;
  su_restore_kernel<<<n, 256, 0, st>>>(d, ranks);
  PEPSB_LAUNCH();
}

void su_one_site(const SuOneSiteDesc* d, int n, cudaStream_t st) {
  if (n == 0) return;
  su_one_site_kernel<<<n, 256, 0, st>>>(d);
  PEPSB_LAUNCH();
}

void herm_exp(const double2* H, int n, double coeff, double tau, double2* out, cudaStream_t st) {
  if (n > 16) throw Error(kShapeError, "gate construction supports local dimension <= 16");
  herm_exp_kernel<<<1, 32, 0, st>>>(H, n, coeff, tau, out);
  PEPSB_LAUNCH();
}

void gram_factors(const double2* G, int n, double2* P, double2* R, int* deficient, int* any_def,
                  int* status, double2* work, cudaStream_t stream, double* lam_out, double2* vec_out) {
  if (n > 256) throw Error(kShapeError, "gram_factors: k > 256 not supported");
  const size_t smem = 2ull * n * (n + 1) * sizeof(double2);
  constexpr size_t kCap = 176 * 1024;  // + ~45 KB static shared memory of the eigensolvers
  const bool fits = smem <= kCap;
  if (!fits && !work) throw Error(kOtherError, "gram_factors: workspace required");
  static bool attr = false;
  if (!attr) {
    PEPSB_CUDA(cudaFuncSetAttribute(gram_factors_kernel<true, kEigThreads>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kCap)));
    PEPSB_CUDA(cudaFuncSetAttribute(gram_factors_kernel<true, kEigFastThreads>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kCap)));
    attr = true;
  }
  static const int env_threads = getenv("PEPSB_EIG_THREADS") ? atoi(getenv("PEPSB_EIG_THREADS")) : 0;
  const int threads = env_threads >= 64 && env_threads <= kEigThreads ? env_threads : kEigThreads;
  static const bool eig_fast = !(getenv("PEPSB_EIG_FAST") && getenv("PEPSB_EIG_FAST")[0] == '0');
  const int use_jacobi = eig_solver() | (eig_fast ? 0x100 : 0);
  static const char* dump = getenv("PEPSB_DUMP_EIG");  // debug aid: last input matrix to a file
  if (dump) {
    std::vector<double2> h(static_cast<size_t>(n) * n);
    PEPSB_CUDA(cudaMemcpyAsync(h.data(), G, h.size() * sizeof(double2), cudaMemcpyDeviceToHost, stream));
    PEPSB_CUDA(cudaStreamSynchronize(stream));
    if (FILE* f = fopen(dump, "wb")) {
      fwrite(h.data(), sizeof(double2), h.size(), f);
      fclose(f);
    }
  }
  if (fits && eig_fast && n >= 16 && n <= 72 && eig_solver() != kEigJacobi && !env_threads)
    gram_factors_kernel<true, kEigFastThreads><<<1, kEigFastThreads, smem, stream>>>(
        G, n, P, R, deficient, any_def, status, nullptr, use_jacobi, lam_out, vec_out);
  else if (fits)
    gram_factors_kernel<true, kEigThreads><<<1, threads, smem, stream>>>(G, n, P, R, deficient, any_def, status,
                                                                         nullptr, use_jacobi & 0xff, lam_out, vec_out);
  else
    gram_factors_kernel<false, kEigThreads><<<1, threads, 0, stream>>>(G, n, P, R, deficient, any_def, status, work,
                                                                       use_jacobi & 0xff, lam_out, vec_out);
  PEPSB_LAUNCH();
}

namespace {
std::atomic<int> g_eig_solver{-1};
}

int eig_solver() {
  int v = g_eig_solver.load();
  if (v < 0) {  // PEPSB_EIG=jacobi selects the Jacobi solver before any option is set
    const char* e = getenv("PEPSB_EIG");
    v = (e && std::string(e) == "jacobi") ? kEigJacobi : (e && std::string(e) == "dc") ? kEigDivideConquer : kEigAuto;
    g_eig_solver.store(v);
  }
  return v;
}

void set_eig_solver(int s) {
  if (s != kEigAuto && s != kEigJacobi && s != kEigDivideConquer)
    throw Error(kValidationError, "eig_solver must be 0 (auto), 1 (Jacobi) or 2 (divide and conquer)");
  g_eig_solver.store(s);
}

void eigh_dense(const double2* G, int n, double* w, double2* vec, int* status, double2* work, cudaStream_t stream) {
  gram_factors(G, n, nullptr, nullptr, nullptr, nullptr, status, work, stream, w, vec);
}

void chol_factors(const double2* G, int n, double shift_rel, double2* R, double2* Rinv, int* status,
                  cudaStream_t stream) {
  if (n > 256) throw Error(kShapeError, "chol_factors: k > 256 not supported");
  const size_t smem = static_cast<size_t>(n) * n * sizeof(double2);
  const bool in_place = smem > kSmemCap;
  static bool attr = false;
  if (!attr) {
    PEPSB_CUDA(cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSmemCap)));
    attr = true;
  }
  chol_kernel<<<1, kThreads, in_place ? 0 : smem, stream>>>(G, n, shift_rel, R, Rinv, status, in_place);
  PEPSB_LAUNCH();
}

int64_t small_svd_workspace(int m, int n, int batch) {
  const int64_t mr = std::max(m, n), nc = std::min(m, n);
  const size_t smem = static_cast<size_t>(mr * nc + nc * nc) * sizeof(double2);
  if (smem <= kSmemCap) return 0;
  return static_cast<int64_t>(batch) * (mr * nc + nc * nc);
}

void small_svd(const double2* A, int64_t sa, int m, int n, int lda, double2* U, int64_t su, double* s,
               int64_t ss, double2* Vh, int64_t sv, int batch, int* status, double2* work,
               cudaStream_t stream) {
  if (batch <= 0) return;
  const int64_t mr = std::max(m, n), nc = std::min(m, n);
  if (nc > 256) throw Error(kShapeError, "small_svd: min(m, n) > 256 not supported");
  const size_t smem = static_cast<size_t>(mr * nc + nc * nc) * sizeof(double2);
  const bool fits = smem <= kSmemCap;
  if (!fits && !work) throw Error(kOtherError, "small_svd: workspace required");
  static bool attr = false;
  if (!attr) {
    PEPSB_CUDA(cudaFuncSetAttribute(small_svd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSmemCap)));
    attr = true;
  }
  SvdArgs a{A, sa, m, n, lda, U, su, s, ss, Vh, sv, status, fits ? nullptr : work, mr * nc + nc * nc};
  const int threads = nc <= 16 ? 256 : kThreads;
  small_svd_kernel<<<batch, threads, fits ? smem : 0, stream>>>(a);
  PEPSB_LAUNCH();
}

int64_t tsqr_workspace(int64_t rows, int k) {
  const size_t cap = 227 * 1024;
  int64_t rpb0 = std::max<int64_t>(k, static_cast<int64_t>(cap / (16 * k)));
  int64_t nb = (rows + rpb0 - 1) / rpb0;
  int64_t ws = 2 * nb * k * k + 16;  // two R stacks
  if (static_cast<size_t>(2 * k) * k * 16 > cap) ws += nb * 2 * k * k + (rows + 1) * k;  // global work
  return ws;
}

void tsqr_r(const double2* A, int64_t rows, int k, double2* R, double2* ws, cudaStream_t stream) {
  const size_t cap = 227 * 1024;
  static bool attr = false;
  if (!attr) {
    PEPSB_CUDA(cudaFuncSetAttribute(householder_r_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(cap - 8 * 1024)));
    attr = true;
  }
  const size_t usable = cap - 8 * 1024;
  const bool big = static_cast<size_t>(2 * k) * k * 16 > usable;
  int64_t rpb = std::max<int64_t>(k, static_cast<int64_t>(usable / (16 * k)));
  int64_t nb = (rows + rpb - 1) / rpb;
  double2* stack[2] = {ws, ws + nb * k * k};
  double2* gwork = big ? ws + 2 * nb * k * k : nullptr;
  const double2* src = A;
  int64_t src_rows = rows;
  int cur = 0;
  while (true) {
    const size_t smem = big ? 0 : static_cast<size_t>(std::max<int64_t>(rpb, k)) * k * 16;
    householder_r_kernel<<<static_cast<unsigned>(nb), kThreads, smem, stream>>>(src, src_rows, k,
                                                                                 static_cast<int>(rpb),
                                                                                 stack[cur], gwork);
    PEPSB_LAUNCH();
    if (nb == 1) break;
    src = stack[cur];
    src_rows = nb * k;
    cur ^= 1;
    rpb = 2 * k;
    nb = (src_rows + rpb - 1) / rpb;
  }
  PEPSB_CUDA(cudaMemcpyAsync(R, stack[cur], static_cast<size_t>(k) * k * 16, cudaMemcpyDeviceToDevice, stream));
}

void complete_columns(double2* Q, int64_t rows, int cols, const int* deficient, const int* any_def,
                      int* status, cudaStream_t stream) {
  complete_columns_kernel<<<1, kThreads, 0, stream>>>(Q, rows, cols, deficient, any_def, status);
  PEPSB_LAUNCH();
}

}  // namespace pepsb
