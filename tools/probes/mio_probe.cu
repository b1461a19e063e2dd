// Does SHFL share the shared-memory (L1 data pipe) bandwidth with LDS?
// Kernels: LDS.128 only, SHFL only, both interleaved, plus LDS.64 and STS.64.
// Prints ns per warp-instruction per SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int MODE>
__global__ void __launch_bounds__(1024) probe(float* out, int salt) {
  __shared__ float4 buf[2048];
  const int tid = threadIdx.x;
  for (int i = tid; i < 2048; i += blockDim.x) buf[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  float4 acc = make_float4(0, 0, 0, 0);
  float s = tid * 0.5f;
  int idx = (tid * 1) & 2047;
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (MODE == 0 || MODE == 2) {
        float4 v = buf[(idx + k * 64) & 2047];
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      if (MODE == 1 || MODE == 2) {
        s = __shfl_xor_sync(0xffffffffu, s, (k & 15) + 1) + 1.0f;
      }
      if (MODE == 3) {  // 4 SHFL per slot (same bytes per lane as one LDS.128)
        s = __shfl_xor_sync(0xffffffffu, s, 1) + 1.0f;
        s = __shfl_xor_sync(0xffffffffu, s, 2) + 1.0f;
        s = __shfl_xor_sync(0xffffffffu, s, 4) + 1.0f;
        s = __shfl_xor_sync(0xffffffffu, s, 8) + 1.0f;
      }
      if (MODE == 4) {  // LDS.128 + 4 SHFL
        float4 v = buf[(idx + k * 64) & 2047];
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        s = __shfl_xor_sync(0xffffffffu, s, 1) + 1.0f;
        s = __shfl_xor_sync(0xffffffffu, s, 2) + 1.0f;
        s = __shfl_xor_sync(0xffffffffu, s, 4) + 1.0f;
        s = __shfl_xor_sync(0xffffffffu, s, 8) + 1.0f;
      }
    }
    idx = (idx + salt) & 2047;
  }
  out[blockIdx.x * blockDim.x + tid] = acc.x + acc.y + acc.z + acc.w + s;
}

template <int MODE>
float run(float* d, int sms) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  probe<MODE><<<sms * 2, 1024>>>(d, 1);
  cudaEventRecord(a);
  probe<MODE><<<sms * 2, 1024>>>(d, 1);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* d;
  cudaMalloc(&d, sms * 2 * 1024 * sizeof(float));
  const double warp_instr_per_sm = 2.0 * 32 * ITERS * 8;   // per kernel slot, per SM (2 CTAs x 32 warps)
  const char* names[] = {"LDS.128 x1", "SHFL x1", "LDS.128 + SHFL", "SHFL x4", "LDS.128 + SHFL x4"};
  float t[5] = {run<0>(d, sms), run<1>(d, sms), run<2>(d, sms), run<3>(d, sms), run<4>(d, sms)};
  for (int i = 0; i < 5; ++i)
    printf("%-20s %8.3f ms  %.3f clk(1.965GHz) per slot per SM\n", names[i], t[i],
           t[i] * 1e-3 * 1.965e9 / warp_instr_per_sm);
  return 0;
}
