// FP64 peak probe for B200 (MEASURED_PEAKS.json has no FP64 entry).
// Measures the DMMA (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4) and DFMA issue
// ceilings with register-resident operands, timed with CUDA events.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-9, b = 1.0 + threadIdx.x * 1e-12;
  double d[8][2] = {};
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[j][0]), "+d"(d[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int j = 0; j < 8; j++) s += d[j][0] + d[j][1];
  if (s == 1234.5) out[0] = s;
}

// sm_90+ shapes (SASS DMMA.16x8x4 / .16x8x8 / .16x8x16): does a larger
// instruction change the FP64 tensor ceiling on B200?
template <int K>
__global__ void dmma16_loop(double* out, int iters) {
  double a[K / 2], b[K / 4];
  for (int j = 0; j < K / 2; ++j) a[j] = threadIdx.x * 1e-9 + j;
  for (int j = 0; j < K / 4; ++j) b[j] = 1.0 + threadIdx.x * 1e-12 + j;
  double d[4][4] = {};
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 4; j++) {
      if constexpr (K == 4)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(d[j][0]), "+d"(d[j][1]), "+d"(d[j][2]), "+d"(d[j][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      else if constexpr (K == 8)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                     "{%0,%1,%2,%3};"
                     : "+d"(d[j][0]), "+d"(d[j][1]), "+d"(d[j][2]), "+d"(d[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                     "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(d[j][0]), "+d"(d[j][1]), "+d"(d[j][2]), "+d"(d[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
  for (int j = 0; j < 4; j++) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  if (s == 1234.5) out[0] = s;
}

template <int K>
double time16(int blocks, int threads, int iters, double* out, cudaEvent_t e0, cudaEvent_t e1) {
  cudaEventRecord(e0);
  dmma16_loop<K><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return (double)blocks * (threads / 32) * iters * 4 * (16.0 * 8 * K * 2) / (ms * 1e-3) / 1e12;
}

extern "C" int probe16(double* res) {  // res[0..2] = TF/s of m16n8k4 / k8 / k16
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps = 4; warps <= 16; warps *= 2)
    for (int rep = 0; rep < 3; rep++) {
      double t4 = time16<4>(sms * 4, warps * 32, 10000, out, e0, e1);
      double t8 = time16<8>(sms * 4, warps * 32, 5000, out, e0, e1);
      double t16 = time16<16>(sms * 4, warps * 32, 2500, out, e0, e1);
      if (t4 > res[0]) res[0] = t4;
      if (t8 > res[1]) res[1] = t8;
      if (t16 > res[2]) res[2] = t16;
    }
  cudaFree(out);
  return (int)cudaGetLastError();
}

__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-9, b = 1.0 - 1e-12;
  double d[16];
  for (int j = 0; j < 16; j++) d[j] = j;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 16; j++) d[j] = fma(d[j], b, a);
  }
  double s = 0;
  for (int j = 0; j < 16; j++) s += d[j];
  if (s == 1234.5) out[0] = s;
}

extern "C" int probe(double* res) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  float best_dmma = 1e30f, best_dfma = 1e30f;
  for (int warps = 4; warps <= 16; warps *= 2) {
    int blocks = sms * 4;
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(e0);
      dmma_loop<<<blocks, warps * 32>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      // flops per launch: blocks*warps*iters*8 DMMA * (8*8*4*2)
      double fl = (double)blocks * warps * iters * 8 * 512;
      double tf = fl / (ms * 1e-3) / 1e12;
      if (tf > res[0]) res[0] = tf;
      cudaEventRecord(e0);
      dfma_loop<<<blocks, warps * 32>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      fl = (double)blocks * warps * 32 * iters * 16 * 2;
      tf = fl / (ms * 1e-3) / 1e12;
      if (tf > res[1]) res[1] = tf;
    }
  }
  (void)best_dmma; (void)best_dfma;
  cudaFree(out);
  return (int)cudaGetLastError();
}
