// DFMA throughput and dependent-chain latency on the B200 (receiver DSP design input).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void thr(double* sink, int iters, double a, double b) {
  double r[8];
  for (int k = 0; k < 8; ++k) r[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = fma(r[k], a, b);
  double s = 0; for (int k = 0; k < 8; ++k) s += r[k];
  if (s == 1.2345) sink[0] = s;
}
__global__ void lat(double* sink, int iters, double a, double b, long long* cyc) {
  double r = threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) r = fma(r, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  if (r == 1.2345) sink[0] = r;
}
int main() {
  double* sink; long long* cyc; cudaMalloc(&sink, 8); cudaMalloc(&cyc, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  thr<<<sms * 8, 256>>>(sink, 100, 0.999, 1e-9);
  cudaEventRecord(e0); thr<<<sms * 8, 256>>>(sink, 4096, 0.999, 1e-9); cudaEventRecord(e1);
  cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 8 * 4096 * 256.0 * sms * 8;
  lat<<<1, 32>>>(sink, 4096, 0.999, 1e-9, cyc);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("{\"fp64_tflops\": %.2f, \"dfma_latency_cycles\": %.2f}\n", flops / (ms * 1e-3) / 1e12, c / 4096.0);
  return 0;
}
