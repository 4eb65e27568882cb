// Developer probe: dependent-chain latency (cycles/op) of FP64 operations on one thread.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, double x, double y, int iters, long long* cyc) {
  double a = x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) a = fma(a, y, 1e-30);
    if (OP == 1) a = a + y;
    if (OP == 2) a = y / a;
    if (OP == 3) a = rsqrt(a) + 0.5;
    if (OP == 4) a = sqrt(a) + 0.5;
    if (OP == 5) a = __drcp_rn(a) + 0.5;
    if (OP == 6) a = hypot(a, y);
    if (OP == 7) { float f = __frsqrt_rn((float)a); a = (double)f + 0.5; }
  }
  long long t1 = clock64();
  out[threadIdx.x] = a;
  cyc[threadIdx.x] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMallocManaged(&cyc, 1024 * 8);
  const char* names[] = {"dfma", "dadd", "ddiv", "rsqrt", "sqrt", "drcp_rn", "hypot", "f32 rsqrt+cvt"};
  const int iters = 4096;
  for (int op = 0; op < 8; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (op) {
        case 0: chain<0><<<1, 1>>>(out, 1.0, 1.0000001, iters, cyc); break;
        case 1: chain<1><<<1, 1>>>(out, 1.0, 1e-9, iters, cyc); break;
        case 2: chain<2><<<1, 1>>>(out, 1.3, 1.7, iters, cyc); break;
        case 3: chain<3><<<1, 1>>>(out, 1.3, 1.7, iters, cyc); break;
        case 4: chain<4><<<1, 1>>>(out, 1.3, 1.7, iters, cyc); break;
        case 5: chain<5><<<1, 1>>>(out, 1.3, 1.7, iters, cyc); break;
        case 6: chain<6><<<1, 1>>>(out, 1.3, 1e-3, iters, cyc); break;
        case 7: chain<7><<<1, 1>>>(out, 1.3, 1.7, iters, cyc); break;
      }
      cudaDeviceSynchronize();
    }
    printf("%-14s %.1f cycles/op\n", names[op], (double)cyc[0] / iters);
  }
  return 0;
}
