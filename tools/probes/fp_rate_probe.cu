// Issue rate of the FP32 instruction forms the DBP kernels use (sm_100a):
// scalar FFMA with a register / immediate / constant-bank multiplier, FFMA2,
// FADD2, FMUL2, FADD, and FFMA2 + immediate FFMA interleaved.  16 independent
// chains per thread, 2 x 1024 threads per SM; prints warp-instructions per
// cycle per SM and FP32 lane-FLOP/s.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 2048, CH = 16;

__device__ __forceinline__ unsigned long long pk(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}

template <int MODE>
__global__ void __launch_bounds__(1024) probe(float* out, float x, float y, float cparam) {
  const int tid = threadIdx.x;
  float a[CH];
  unsigned long long p[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    a[i] = tid * 1e-3f + i;
    p[i] = pk(a[i], a[i] + 1.f);
  }
  const float xr = x + tid * 1e-9f, yr = y - tid * 1e-9f;
  const unsigned long long x2 = pk(xr, xr + 1e-7f), y2 = pk(yr, yr + 1e-7f);
  const unsigned long long xu = pk(x, x), yu = pk(y, y);
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if constexpr (MODE == 0) a[i] = fmaf(a[i], xr, yr);               // FFMA R, R, R, R
      if constexpr (MODE == 1) a[i] = fmaf(a[i], 0.99987f, yr);         // FFMA R, R, imm, R
      if constexpr (MODE == 2) a[i] = fmaf(a[i], cparam, yr);           // FFMA R, R, c[], R
      if constexpr (MODE == 3) asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(x2), "l"(y2));
      if constexpr (MODE == 4) asm("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(y2));
      if constexpr (MODE == 5) asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(x2));
      if constexpr (MODE == 6) a[i] = a[i] + yr;                        // FADD R, R, R
      if constexpr (MODE == 7) {                                         // FFMA2 and imm FFMA alternate
        if (i & 1) a[i] = fmaf(a[i], 0.99987f, yr);
        else asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(x2), "l"(y2));
      }
      if constexpr (MODE == 8) a[i] = a[i] * 0.99987f;                  // FMUL R, R, imm
      if constexpr (MODE == 9) asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(xu), "l"(yu));   // uniform operands
      if constexpr (MODE == 10) asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(p[(i + 1) % CH]), "l"(p[(i + 2) % CH]));
      if constexpr (MODE == 11) a[i] = fmaf(a[i], a[(i + 1) % CH], a[(i + 2) % CH]);
      if constexpr (MODE == 12) asm("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(yu));
      if constexpr (MODE == 13) asm("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(p[i]) : "l"(x2));
      if constexpr (MODE == 14) asm("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(p[(i + 1) % CH]));
      if constexpr (MODE == 15) a[i] = a[i] + a[(i + 1) % CH];
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(p[i]));
    s += a[i] + lo + hi;
  }
  out[blockIdx.x * blockDim.x + tid] = s;
}

template <int MODE>
void run(const char* name, float* d, int sms, int clk_khz, double flops_per_instr) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  probe<MODE><<<sms * 2, 1024>>>(d, 1.0001f, 0.5f, 0.99991f);
  cudaEventRecord(a);
  probe<MODE><<<sms * 2, 1024>>>(d, 1.0001f, 0.5f, 0.99991f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double warp_instr = (double)sms * 2 * 32 * ITERS * CH;   // per launch
  const double cycles = ms * 1e-3 * clk_khz * 1e3;
  printf("%-22s %8.3f ms  %5.2f warp-instr/clk/SM  %6.1f TFLOP/s\n", name, ms, warp_instr / sms / cycles,
         warp_instr * 32 * flops_per_instr / (ms * 1e-3) / 1e12);
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  float* d;
  cudaMalloc(&d, sizeof(float) * sms * 2 * 1024);
  printf("SMs %d, clock attribute %d kHz\n", sms, clk);
  run<0>("FFMA reg", d, sms, clk, 2);
  run<1>("FFMA imm", d, sms, clk, 2);
  run<2>("FFMA const-bank", d, sms, clk, 2);
  run<3>("FFMA2 reg", d, sms, clk, 4);
  run<4>("FADD2 reg", d, sms, clk, 2);
  run<5>("FMUL2 reg", d, sms, clk, 2);
  run<6>("FADD reg", d, sms, clk, 1);
  run<7>("FFMA2 + FFMA imm 1:1", d, sms, clk, 3);
  run<8>("FMUL imm", d, sms, clk, 1);
  run<9>("FFMA2 uniform b,c", d, sms, clk, 4);
  run<10>("FFMA2 3 distinct", d, sms, clk, 4);
  run<11>("FFMA 3 distinct", d, sms, clk, 2);
  run<12>("FADD2 uniform b", d, sms, clk, 2);
  run<13>("FFMA2 a*x+a", d, sms, clk, 4);
  run<14>("FADD2 2 distinct", d, sms, clk, 2);
  run<15>("FADD 2 distinct", d, sms, clk, 1);
  return 0;
}
