// Microbenchmark: FP64 latencies on B200 (one warp, dependent chains) and
// throughput with k independent chains per thread.  Prints cycles/op.
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void chains(double *out, long long *cyc, int iters) {
  double a[K];
  for (int k = 0; k < K; k++) a[k] = 1.0 + threadIdx.x * 1e-9 + k * 1e-7;
  const double b = 0.9999999, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < K; k++) a[k] = fma(a[k], b, c);
  }
  long long t1 = clock64();
  double s = 0;
  for (int k = 0; k < K; k++) s += a[k];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void rsq_chain(double *out, long long *cyc, int iters) {
  double x = 1.5 + threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
    double y;
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    x = y + 1.0;
  }
  long long t1 = clock64();
  if (x == 1.2345) out[0] = x;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double *o; long long *c, h;
  cudaMalloc(&o, 8); cudaMalloc(&c, 8);
  const int it = 100000;
  chains<1><<<1, 32>>>(o, c, it); cudaDeviceSynchronize();
  chains<1><<<1, 32>>>(o, c, it); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)h / it);
  chains<8><<<1, 32>>>(o, c, it); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("1 warp, 8 chains: %.2f cycles per DFMA instr\n", (double)h / it / 8);
  chains<8><<<1, 128>>>(o, c, it); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("4 warps (1/SMSP), 8 chains: %.2f cycles per DFMA instr per warp\n", (double)h / it / 8);
  chains<8><<<1, 256>>>(o, c, it); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("8 warps, 8 chains: %.2f cycles per warp-DFMA (per warp)\n", (double)h / it / 8);
  rsq_chain<<<1, 32>>>(o, c, it); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("MUFU.RSQ64H + DADD dependent: %.2f cycles\n", (double)h / it);
  return 0;
}
