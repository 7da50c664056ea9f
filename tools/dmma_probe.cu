// DFMA vs DMMA (mma.sync m8n8k4 f64) throughput on one B200, alone and
// interleaved: do the FP64 tensor instructions use separate hardware from
// the FP64 vector pipe?   nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &d0, double &d1, double a,
                                     double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, "
      "{%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

template <int MODE>
__global__ void k(double *out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, a2 = a0 + 2e-9,
         a3 = a0 + 3e-9, a4 = a0 + 4e-9, a5 = a0 + 5e-9, a6 = a0 + 6e-9,
         a7 = a0 + 7e-9;
  double c[8][2];
  for (int i = 0; i < 8; i++) c[i][0] = c[i][1] = i * 1e-9;
  const double b = 0.999999999, e = 1e-12;
  const double ma = 1e-3 + threadIdx.x * 1e-9, mb = 0.5;
  for (int it = 0; it < iters; it++) {
    if (MODE & 1) {
      a0 = fma(a0, b, e); a1 = fma(a1, b, e); a2 = fma(a2, b, e);
      a3 = fma(a3, b, e); a4 = fma(a4, b, e); a5 = fma(a5, b, e);
      a6 = fma(a6, b, e); a7 = fma(a7, b, e);
    }
    if (MODE & 2) {
#pragma unroll
      for (int i = 0; i < 8; i++) dmma(c[i][0], c[i][1], ma, mb);
    }
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int MODE>
float run(double *out, int iters, int blocks, int threads) {
  cudaEvent_t s, t;
  cudaEventCreate(&s);
  cudaEventCreate(&t);
  k<MODE><<<blocks, threads>>>(out, 10);
  cudaEventRecord(s);
  k<MODE><<<blocks, threads>>>(out, iters);
  cudaEventRecord(t);
  cudaEventSynchronize(t);
  float ms;
  cudaEventElapsedTime(&ms, s, t);
  return ms;
}

int main() {
  double *out;
  cudaMalloc(&out, 8);
  const int blocks = 148 * 8, threads = 256, iters = 20000;
  const double warps = blocks * threads / 32.0;
  float m1 = run<1>(out, iters, blocks, threads);
  float m2 = run<2>(out, iters, blocks, threads);
  float m3 = run<3>(out, iters, blocks, threads);
  const double fdfma = 2.0 * 8 * iters * (double)blocks * threads;
  const double fdmma = 512.0 * 8 * iters * warps;
  printf("DFMA only : %.2f ms  %.2f TF/s\n", m1, fdfma / m1 / 1e9);
  printf("DMMA only : %.2f ms  %.2f TF/s\n", m2, fdmma / m2 / 1e9);
  printf("both      : %.2f ms  %.2f TF/s combined (sum of alone: %.2f ms)\n",
         m3, (fdfma + fdmma) / m3 / 1e9, m1 + m2);
  return 0;
}
