// Developer probe: throughput (SM cycles per warp-instruction-equivalent) of FP64 reciprocal variants.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rcp_mufu(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double rcp_f32seed(double x) {
  float xf = __double2float_rn(x);
  double r = (double)__frcp_rn(xf);
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);  // 2^-46
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

template <int OP>
__global__ void thr(double* out, double x0, int iters, long long* cyc) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = x0 + 0.01 * k + threadIdx.x * 1e-6;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) a[k] = 1.0 / a[k] + 0.5;
      if (OP == 1) a[k] = rcp_mufu(a[k]) + 0.5;
      if (OP == 2) a[k] = rcp_f32seed(a[k]) + 0.5;
      if (OP == 3) a[k] = fma(a[k], 0.999, 0.001);
      if (OP == 4) a[k] = sqrt(a[k]) + 0.5;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMallocManaged(&cyc, 1024 * 8);
  const char* names[] = {"ddiv", "rcp mufu+2nr", "rcp f32seed+2nr", "dfma", "sqrt"};
  const int iters = 256;
  for (int op = 0; op < 5; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (op) {
        case 0: thr<0><<<1, 1024>>>(out, 1.3, iters, cyc); break;
        case 1: thr<1><<<1, 1024>>>(out, 1.3, iters, cyc); break;
        case 2: thr<2><<<1, 1024>>>(out, 1.3, iters, cyc); break;
        case 3: thr<3><<<1, 1024>>>(out, 1.3, iters, cyc); break;
        case 4: thr<4><<<1, 1024>>>(out, 1.3, iters, cyc); break;
      }
      cudaDeviceSynchronize();
    }
    const double ops = 1024.0 * 8 * iters;
    printf("%-18s %.3f SM cycles per op  (%.1f ops/clk/SM)\n", names[op], cyc[0] / ops, ops / cyc[0]);
  }
  return 0;
}
