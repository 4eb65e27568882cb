// Developer probe: cost of the tridiagonalisation's reflector phase (one warp) per step.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2006_15234_b200/csrc/common.cuh"
using namespace pepsb;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int VAR>
__global__ void probe(double2* out, int n, long long* cyc) {
  __shared__ double2 xs[256], q[256], nxt[256], vv[256], pw[256], tauv[256], Acol[256 * 8];
  __shared__ double e[256];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 256; i += blockDim.x) {
    xs[i] = make_double2(0.3 + 1e-3 * i, 0.1);
    q[i] = make_double2(0.2, -0.1 * i);
    nxt[i] = make_double2(0.5, 0.01 * i);
  }
  __syncthreads();
  long long t0 = clock64();
  for (int j = 0; j + 1 < n; ++j) {
    if (warp == 0) {
      double xn = 0.0;
      double2 alpha = make_double2(0.0, 0.0);
      for (int l = j + 1 + lane; l < n; l += 32) {
        double2 x = xs[l];
        if (l >= j + 2) xn += cnorm2(x);
        if (l == j + 1) alpha = x;
      }
      xn = warp_sum(xn);
      alpha = make_double2(__shfl_sync(0xffffffffu, alpha.x, 0), __shfl_sync(0xffffffffu, alpha.y, 0));
      double beta = -copysign(sqrt(alpha.x * alpha.x + alpha.y * alpha.y + xn), alpha.x);
      double2 tau = make_double2((beta - alpha.x) / beta, -alpha.y / beta);
      const double2 den = make_double2(alpha.x - beta, alpha.y);
      const double dn = 1.0 / cnorm2(den);
      double2 scal = make_double2(den.x * dn, -den.y * dn);
      const double2 ts = cmul(tau, scal);
      double hr = 0.0, hi = 0.0;
      if (VAR != 1)
        for (int l = j + 1 + lane; l < n; l += 32) {
          const double2 v = l == j + 1 ? make_double2(1.0, 0.0) : cmul(xs[l], scal);
          Acol[(j & 7) * 256 + l] = v;
          vv[l] = v;
          const double2 s = q[l], a1 = nxt[l];
          const double2 p = cmul(ts, make_double2(s.x - beta * a1.x, s.y - beta * a1.y));
          pw[l] = p;
          hr += p.x * v.x + p.y * v.y;
          hi += p.x * v.y - p.y * v.x;
        }
      if (VAR != 2) {
        hr = warp_sum(hr);
        hi = warp_sum(hi);
      }
      const double2 alpha2 = cscale(cmul(tau, make_double2(hr, hi)), -0.5);
      if (VAR != 1)
        for (int l = j + 1 + lane; l < n; l += 32) pw[l] = cadd(pw[l], cmul(alpha2, vv[l]));
      if (lane == 0) {
        e[j] = beta;
        tauv[j] = tau;
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cyc[0] = t1 - t0;
  if (tid < 256) out[tid] = pw[tid];
}

int main() {
  double2* out;
  long long* cyc;
  cudaMalloc(&out, 4096 * 16);
  cudaMallocManaged(&cyc, 64);
  const char* names[] = {"full", "no vector loops", "no warp_sums"};
  for (int v = 0; v < 3; ++v)
    for (int threads : {32, 512, 1024}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (v == 0) probe<0><<<1, threads>>>(out, 72, cyc);
        if (v == 1) probe<1><<<1, threads>>>(out, 72, cyc);
        if (v == 2) probe<2><<<1, threads>>>(out, 72, cyc);
        cudaDeviceSynchronize();
      }
      printf("%-16s threads %4d: %.0f cycles/step\n", names[v], threads, cyc[0] / 71.0);
    }
  return 0;
}
