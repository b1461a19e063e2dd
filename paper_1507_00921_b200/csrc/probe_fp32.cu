// FP32 FMA throughput probe (measurement utility, not on the DBP path).
//
// The roofline denominator for the FP32-bound DBP kernel: MEASURED_PEAKS.json
// records only HBM copy and bf16 GEMM peaks, so bench.py measures the FP32
// pipe on the same box and clocks with a dependent-chain-free FFMA kernel
// (8 independent accumulators per thread, immediate-free 3-register form,
// 148 x 8 CTAs of 256 threads), timed with CUDA events.
#include <cuda_runtime.h>

#include <string>

#include "../../include/dbp_b200.h"

namespace {

__device__ __forceinline__ unsigned long long dbp_pack(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}

__global__ void __launch_bounds__(256) fma_probe_kernel(float* sink, int iters, float a, float b) {
  float r0 = threadIdx.x * 1e-7f, r1 = r0 + 1e-7f, r2 = r0 + 2e-7f, r3 = r0 + 3e-7f;
  float r4 = r0 + 4e-7f, r5 = r0 + 5e-7f, r6 = r0 + 6e-7f, r7 = r0 + 7e-7f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      r0 = fmaf(r0, a, b); r1 = fmaf(r1, a, b); r2 = fmaf(r2, a, b); r3 = fmaf(r3, a, b);
      r4 = fmaf(r4, a, b); r5 = fmaf(r5, a, b); r6 = fmaf(r6, a, b); r7 = fmaf(r7, a, b);
    }
  }
  const float s = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
  if (s == 1234.5f) sink[threadIdx.x] = s;  // keep the chain alive
}

// the same with sm_100a's packed FFMA2 (two float32 FMAs per lane per instruction)
__global__ void __launch_bounds__(256) fma2_probe_kernel(float* sink, int iters, float a, float b) {
  unsigned long long r[8];
  const unsigned long long av = dbp_pack(a, a), bv = dbp_pack(b, b);
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = dbp_pack(threadIdx.x * 1e-7f + k * 1e-7f, threadIdx.x * 1e-7f + k * 2e-7f);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(r[k]) : "l"(av), "l"(bv));
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(r[k]));
    s += lo + hi;
  }
  if (s == 1234.5f) sink[threadIdx.x] = s;
}

// packed and scalar FMAs interleaved: 8 FFMA2 chains + S scalar FFMA chains
// per step -- does the scalar FMA (fma-lite) pipe run beside FFMA2?
template <int S>
__global__ void __launch_bounds__(256) fma_mixed_probe_kernel(float* sink, int iters, float a, float b) {
  unsigned long long r[8];
  float q[S > 0 ? S : 1];
  const unsigned long long av = dbp_pack(a, a), bv = dbp_pack(b, b);
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = dbp_pack(threadIdx.x * 1e-7f + k * 1e-7f, threadIdx.x * 1e-7f + k * 2e-7f);
#pragma unroll
  for (int k = 0; k < S; ++k) q[k] = threadIdx.x * 1e-7f + k * 3e-7f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(r[k]) : "l"(av), "l"(bv));
        if (k < S) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(q[k]) : "f"(a), "f"(b));
      }
#pragma unroll
      for (int k = 8; k < S; ++k) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(q[k]) : "f"(a), "f"(b));
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(r[k]));
    s += lo + hi;
  }
#pragma unroll
  for (int k = 0; k < S; ++k) s += q[k];
  if (s == 1234.5f) sink[threadIdx.x] = s;
}

int probe(int device, int iters, bool packed, double* tflops, double* ms, int mixed = -1) {
  if (!tflops || iters < 1) return DBP_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return DBP_ECUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* sink = nullptr;
  if (cudaMalloc(&sink, 256 * sizeof(float)) != cudaSuccess) return DBP_ENOMEM;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8;
  auto launch = [&](int it) {
    if (mixed == 2) fma_mixed_probe_kernel<2><<<blocks, 256>>>(sink, it, 0.9999f, 1e-7f);
    else if (mixed == 4) fma_mixed_probe_kernel<4><<<blocks, 256>>>(sink, it, 0.9999f, 1e-7f);
    else if (mixed == 8) fma_mixed_probe_kernel<8><<<blocks, 256>>>(sink, it, 0.9999f, 1e-7f);
    else if (mixed == 16) fma_mixed_probe_kernel<16><<<blocks, 256>>>(sink, it, 0.9999f, 1e-7f);
    else if (packed) fma2_probe_kernel<<<blocks, 256>>>(sink, it, 0.9999f, 1e-7f);
    else fma_probe_kernel<<<blocks, 256>>>(sink, it, 0.9999f, 1e-7f);
  };
  launch(iters / 8 + 1);  // warm-up
  cudaEventRecord(e0);
  launch(iters);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  float t = 0.f;
  cudaEventElapsedTime(&t, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (err != cudaSuccess) return DBP_ECUDA;
  const double per_step = mixed > 0 ? 16.0 + mixed : (packed ? 2.0 : 1.0) * 8.0;
  const double flops = 2.0 * per_step * 16.0 * (double)iters * 256.0 * (double)blocks;
  *tflops = flops / (t * 1e-3) / 1e12;
  if (ms) *ms = t;
  return DBP_OK;
}

}  // namespace

extern "C" int dbp_probe_fp32x2_peak(int device, int iters, double* tflops, double* ms) {
  return probe(device, iters, true, tflops, ms);
}

extern "C" int dbp_probe_fp32_peak(int device, int iters, double* tflops, double* ms) {
  return probe(device, iters, false, tflops, ms);
}

// 8 packed + S scalar FMA chains interleaved (S = 2, 4, 8, 16)
extern "C" int dbp_probe_fp32_mixed_peak(int device, int iters, int scalar_chains, double* tflops, double* ms) {
  if (scalar_chains != 2 && scalar_chains != 4 && scalar_chains != 8 && scalar_chains != 16) return DBP_EINVAL;
  return probe(device, iters, true, tflops, ms, scalar_chains);
}
