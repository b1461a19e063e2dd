// Shared declarations of the fused DBP block kernels: launch parameters,
// program / arrangement codes, streaming global memory helpers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dbp {


constexpr int kMaxSideCoeffs = 64;

enum Program : int { kFFE = 0, kSSFM = 1, kESSFM = 2, kRotateOnly = 3, kIdentity = 4 };
enum Arrangement : int { kSymmetric = 0, kLinearFirst = 1, kNonlinearFirst = 2 };

struct KernelParams {
  const float2* in;
  float2* out;
  long long n_total;          // samples per polarisation of the whole signal
  long long in_pol_stride;    // float2 elements between the x and y rows
  long long in_item_stride;   // float2 elements between batch items
  long long out_pol_stride;
  long long out_item_stride;
  long long in_origin;        // global sample index of in[0]  (chunk mode)
  long long out_origin;       // global sample index of out[0]
  long long block_begin;      // first overlap-save block processed per item
  long long blocks_per_item;  // blocks processed per item in this launch
  long long total_blocks;     // blocks_per_item * items
  unsigned long long bpi_magic;  // ceil(2^64 / blocks_per_item) when both fit 32 bits (else 0):
                                 // blk / blocks_per_item = umulhi(bpi_magic, blk) (Lemire fastdiv)
  int cyclic;                 // 1: global index taken modulo n_total
  int step;                   // N - M
  int lead;                   // M / 2
  int program;                // Program
  int arrangement;            // Arrangement
  int n_steps;                // nonlinear steps
  // operator program decoded on the host (dbp.py:212-233): n_ops operators;
  // op is a convolution iff conv_all, or (op & 1) == conv_parity when
  // conv_parity >= 0; the first and last op use tab_half iff half_ends;
  // a rotation's step index is op >> sidx_shift
  int n_ops;
  int conv_all;
  int conv_parity;
  int half_ends;
  int sidx_shift;
  int nc;                     // side coefficients of the intensity FIR
  int fir_pad;                // nc rounded up to a multiple of 4
  int slice_floats;           // shared floats per block slice
  int precise_sincos;         // 1: polynomial sincos (multi-step programs), 0: SFU
  const float2* tab_full;     // K (or H for FFE) in the block kernel's register order, 1/N folded in
  const float2* tab_half;     // K^(1/2) (symmetric arrangement)
  const float2* twiddle;      // per-pass twiddle tables
  const float2* wtw;          // warp FFE kernel bases (dbp_warp_kernel.cuh, N = 1024 .. 4096)
  const float2* tab_nat;      // H in natural bin order, 1/N folded in (warp FFE kernel)
  const float2* r2_full;      // N = 8192 radix-2 step tables [A | C | D] (dbp_r2_kernel.cuh), full step
  const float2* r2_half;      //   ... half step (symmetric arrangement)
  const float2* r2_tw;        //   ... the 4096-point transforms' twiddles
  const float2* steps;        // per step (a_j, g_j): rotation exp(+j a_j F), gain g_j
  const float* coeff;         // c_0..c_nc zero padded to nc + 4 (generic FIR path)
  int coeff_stride;           // 0: shared coefficients; > 0: item i uses coeff + i * stride
  float c[kMaxSideCoeffs + 4];  // c_0..c_nc, zero padded
};

__device__ __forceinline__ float2 ld_stream(const float2* p) {
  float2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];"
               : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}

// read-only table load that the compiler may not merge with an earlier load
// of the same address (keeps forward/inverse twiddles from living in registers
// across the deeper FFT passes)
__device__ __forceinline__ float2 ldg_table(const float2* p) {
  float2 v;
  asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ void ldg_table_pair(const float2* p, float2& a, float2& b) {
  float4 v;
  asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  a = make_float2(v.x, v.y);
  b = make_float2(v.z, v.w);
}

// value barrier: stops CSE of index arithmetic across the recursive passes
__device__ __forceinline__ int opaque(int x) {
  int y;
  asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

__device__ __forceinline__ void st_stream(float2* p, float2 v) {
  asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}

}  // namespace dbp
