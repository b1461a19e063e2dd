// Warp-resident overlap-save FFE kernel: one polarisation of one block per
// warp (N = 2048), per half-warp (N = 1024) or per warp pair (N = 4096),
// 64 samples per lane, a two-pass FFT with ONE shared-memory exchange per
// transform and no CTA-wide barrier.
//
// The FFE program (pkg/src/fiberdbp/dbp.py:185-191: ifft(H * fft(block)) on
// each overlap-save block, spectral.py:84-140) is a single convolution: the
// block kernel (dbp_block_kernel.cuh) spends it four exchanges and three CTA
// barriers per block with 16 samples per thread, and measures bound by the
// shared-memory data path (L1 wavefronts 83%, profiles/r2/ffe_v10_ncu_summary.txt).
// Here a lane holds 64 samples, so N = 64 L (L lanes per polarisation):
//
//   n = n1 + L n2 (lane n1 holds n2 = 0..63),  k = k2 + 64 k1
//   X[k2 + 64 k1] = sum_n1 W_L^{n1 k1} (W_N^{k2})^{n1} sum_n2 W_64^{n2 k2} x[n1 + L n2]
//
// 1. in-register DFT-64 over n2 (lane n1: Y[n1][k2], k2 = 0..63);
// 2. exchange: lane j collects Y[n1][k2] for its 64/L values of k2, every n1;
// 3. in-register DFT-L over n1 with the input twiddle folded in as a runtime
//    base b = W_N^{k2} (decimation in time, dft_small.cuh dft*_tw);
// 4. multiply by H (natural bin order, 1/N folded in by the host);
// 5. inverse DFT-L over k1 (in-register);
// 6. exchange back: lane n1 collects all 64 k2;
// 7. inverse DFT-64 over k2 with base W_N^{-n1} -> x'[n1 + L n2];
// then the kept centre is stored straight from registers.
//
// Exchanges are 16-byte (N <= 2048) or 8-byte (N = 4096) shared accesses in
// an XOR-swizzled layout with no bank conflicts; the exchange region is
// private to the warp (N = 4096: the warp pair, one named barrier), so the
// only synchronisation is __syncwarp.  Twiddle bases and their powers come
// from a small host table (float64 -> float32, unit_float2 rounding).
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "dbp_common.cuh"
#include "dft_small.cuh"
#include "w64_const.cuh"

#ifndef DBP_WARP_MIN_CTAS
#define DBP_WARP_MIN_CTAS 2   // 255 registers, no spills (3: 168 registers with spills, -9%)
#endif
// Measured (profiles/r2/warp_ffe/): 26% fewer instructions and 48% L1
// wavefronts (block kernel: 83%) per launch, but 255 registers hold 8 warps
// per SM and the kernel issues on 39% of cycles (dependency waits, global
// load latency, instruction-cache misses): FFE 2048/700 95.0 GS/s against the
// block kernel's 102.2, 4096/700 103.4 against 104.3; at 168 registers (12
// warps, 100-180 bytes of spills) 86.6 / 90.9.  Off by default; env
// DBP_WARP_FFE=1 (or -DDBP_WARP_FFE=1) selects it for FFE programs at N = 1024 .. 4096.
#ifndef DBP_WARP_FFE
#define DBP_WARP_FFE 0
#endif


namespace dbp {

template <int LOGL>
struct WGeo {
  static constexpr int L = 1 << LOGL;        // lanes per polarisation
  static constexpr int N = 64 * L;
  static constexpr int LOGN = LOGL + 6;
  static constexpr int KPL = 64 / L;         // values of k2 per lane in the transposed phase
  static constexpr int THREADS = 128;        // 4 warps
  static constexpr int BPC = L == 16 ? 4 : L == 32 ? 2 : 1;   // blocks per CTA
  static constexpr int MIN_CTAS = DBP_WARP_MIN_CTAS;
  static constexpr size_t SMEM_BYTES = (size_t)BPC * 2 * N * sizeof(float2);
  // twiddle table (float2): forward bases W_N^{k2 2^i} [i][k2] (i < LOGL,
  // k2 < 64), then inverse bases W_N^{-n1 2^i} [i][n1] (i < 6, n1 < L)
  static constexpr int TW_FWD = 0;
  static constexpr int TW_INV = LOGL * 64;
  static constexpr int TW_SIZE = LOGL * 64 + 6 * L;
};

inline bool warp_ffe_supported(int logn) { return logn >= 10 && logn <= 12; }

// host: the warp kernel's twiddle table for N = 2^logn (empty when unsupported)
inline std::vector<float2> make_warp_twiddles(int logn, float2 (*unit)(double)) {
  std::vector<float2> t;
  if (!warp_ffe_supported(logn)) return t;
  const int logl = logn - 6;
  const long long n = 1LL << logn, l = 1LL << logl;
  for (int i = 0; i < logl; ++i)
    for (long long k2 = 0; k2 < 64; ++k2) t.push_back(unit(-2.0 * M_PI * (double)((k2 << i) % n) / (double)n));
  for (int i = 0; i < 6; ++i)
    for (long long n1 = 0; n1 < l; ++n1) t.push_back(unit(2.0 * M_PI * (double)((n1 << i) % n) / (double)n));
  return t;
}

// ---------------------------------------------------------------------------
// constant W_64^M butterflies (conjugate for INV)
// ---------------------------------------------------------------------------
template <bool INV, int M>
__device__ __forceinline__ float2 w64c() {
  constexpr int m = M & 63;
  constexpr float re = W64Const::re[m], im = W64Const::im[m];
  return make_float2(re, INV ? -im : im);
}

// (p + w q, p - w q), w = W_64^M
template <bool INV, int M>
__device__ __forceinline__ void pm_w64(float2 p, float2 q, float2& plus, float2& minus) {
  constexpr int m = M & 63;
  if constexpr ((m & 15) == 0) {
    pm_w16<INV, m / 4>(p, q, plus, minus);
  } else {
    pm_rt(p, q, w64c<INV, M>(), plus, minus);
  }
}

template <bool INV, int M>
__device__ __forceinline__ float2 c_mul_w64(float2 a) {
  constexpr int m = M & 63;
  if constexpr ((m & 15) == 0) return c_mul_w16<INV, m / 4>(a);
  else return c_mul(a, w64c<INV, M>());
}

// radix-4 row with the W_64 twiddles fused (row4_fused for 64ths)
template <bool INV, int MK1, int M2K1>
__device__ __forceinline__ void row4_w64(float2 a0, float2 a1, float2 a2, float2 a3, float2& x0, float2& x1,
                                         float2& x2, float2& x3) {
  float2 t0, t1, u2, u3;
  pm_w64<INV, M2K1>(a0, a2, t0, t1);
  pm_w64<INV, M2K1>(a1, a3, u2, u3);
  pm_w64<INV, MK1>(t0, u2, x0, x2);
  pm_w64<INV, MK1 + 16>(t1, u3, x1, x3);
}

template <bool INV, int D>
__device__ __forceinline__ void dft64_rows(const float2* v, float2* x) {
  if constexpr (D < 16) {
    row4_w64<INV, D, 2 * D>(v[4 * D], v[4 * D + 1], v[4 * D + 2], v[4 * D + 3], x[D], x[D + 16], x[D + 32],
                            x[D + 48]);
    dft64_rows<INV, D + 1>(v, x);
  }
}

// natural-order DFT-64 in registers: n = a + 4 e, k = d + 16 c
template <bool INV>
__device__ __forceinline__ void dft64(float2* v) {
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    float2 u[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) u[e] = v[a + 4 * e];
    dft16<INV>(u);
#pragma unroll
    for (int d = 0; d < 16; ++d) v[a + 4 * d] = u[d];   // v[4 d + a] = U[a][d]
  }
  float2 x[64];
  dft64_rows<INV, 0>(v, x);
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = x[i];
}

template <bool INV, int D>
__device__ __forceinline__ void dft32_rows(const float2* s0, const float2* s1, float2* x) {
  if constexpr (D < 16) {
    pm_w64<INV, 2 * D>(s0[D], s1[D], x[D], x[D + 16]);
    dft32_rows<INV, D + 1>(s0, s1, x);
  }
}

// natural-order DFT-32: n = a + 2 e, k = d + 16 c
template <bool INV>
__device__ __forceinline__ void dft32(float2* v) {
  float2 s0[16], s1[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    s0[e] = v[2 * e];
    s1[e] = v[2 * e + 1];
  }
  dft16<INV>(s0);
  dft16<INV>(s1);
  dft32_rows<INV, 0>(s0, s1, v);
}

// X_k = sum_e W_32^{e k} b^e v_e (p[i] = b^(2^i), i < 5)
template <bool INV, int D>
__device__ __forceinline__ void dft32_tw_rows(const float2* s0, const float2* s1, float2 b, float2* x) {
  if constexpr (D < 16) {
    pm_rt(s0[D], s1[D], c_mul_w64<INV, 2 * D>(b), x[D], x[D + 16]);
    dft32_tw_rows<INV, D + 1>(s0, s1, b, x);
  }
}
template <bool INV>
__device__ __forceinline__ void dft32_tw(float2* v, const float2* p) {
  float2 s0[16], s1[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    s0[e] = v[2 * e];
    s1[e] = v[2 * e + 1];
  }
  dft16_tw_p<INV>(s0, p[1], p[2], p[3], p[4]);
  dft16_tw_p<INV>(s1, p[1], p[2], p[3], p[4]);
  dft32_tw_rows<INV, 0>(s0, s1, p[0], v);
}

// X_k = sum_e W_64^{e k} b^e v_e (p[i] = b^(2^i), i < 6): e = a + 4 e', k = d + 16 c
template <bool INV, int D>
__device__ __forceinline__ void dft64_tw_rows(float2* v, float2 b, float2 b2, float2* x) {
  if constexpr (D < 16) {
    float2 a0 = v[4 * D], a1 = v[4 * D + 1], a2 = v[4 * D + 2], a3 = v[4 * D + 3];
    tw_dft4<INV>(a0, a1, a2, a3, c_mul_w64<INV, D>(b), c_mul_w64<INV, 2 * D>(b2));
    x[D] = a0;
    x[D + 16] = a1;
    x[D + 32] = a2;
    x[D + 48] = a3;
    dft64_tw_rows<INV, D + 1>(v, b, b2, x);
  }
}
template <bool INV>
__device__ __forceinline__ void dft64_tw(float2* v, const float2* p) {
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    float2 u[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) u[e] = v[a + 4 * e];
    dft16_tw_p<INV>(u, p[2], p[3], p[4], p[5]);
#pragma unroll
    for (int d = 0; d < 16; ++d) v[a + 4 * d] = u[d];
  }
  float2 x[64];
  dft64_tw_rows<INV, 0>(v, p[0], p[1], x);
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = x[i];
}

template <int R, bool INV>
__device__ __forceinline__ void dft_plain(float2* v) {
  if constexpr (R == 16) dft16<INV>(v);
  else if constexpr (R == 32) dft32<INV>(v);
  else dft64<INV>(v);
}
template <int R, bool INV>
__device__ __forceinline__ void dft_base(float2* v, const float2* p) {
  if constexpr (R == 16) dft16_tw_p<INV>(v, p[0], p[1], p[2], p[3]);
  else if constexpr (R == 32) dft32_tw<INV>(v, p);
  else dft64_tw<INV>(v, p);
}

__device__ __forceinline__ float4 lds128(const float4* p) { return *p; }

// ---------------------------------------------------------------------------
// the exchanges (swizzled, conflict free)
// ---------------------------------------------------------------------------
// N <= 2048: 16-byte slots holding the k2 pair (2P, 2P + 1) of writer lane
// n1: slot(P, n1) = P L + (n1 ^ (P / (KPL / 2))).  Writes (fixed P, lanes n1)
// and reads (fixed n1, lanes j with P in {KPL j / 2 ..}) hit eight distinct
// slots per quarter warp.
// N = 4096: 8-byte slots a(k2, n1) = 64 k2 + (n1 ^ (k2 & 15)), 16 distinct per half warp.
template <int LOGL>
__device__ __forceinline__ void exch_to_k2(float2* v, float2* reg, int l) {
  using W = WGeo<LOGL>;
  constexpr int L = W::L, KPL = W::KPL;
  if constexpr (L <= 32) {
    float4* s = reinterpret_cast<float4*>(reg);
    constexpr int SH = KPL == 2 ? 0 : 1;   // P / (KPL / 2) == P >> SH
#pragma unroll
    for (int P = 0; P < 32; ++P) s[P * L + (l ^ (P >> SH))] = make_float4(v[2 * P].x, v[2 * P].y, v[2 * P + 1].x, v[2 * P + 1].y);
    __syncwarp();
#pragma unroll
    for (int i = 0; i < KPL / 2; ++i) {
      const int P = (KPL / 2) * l + i;
#pragma unroll
      for (int n1 = 0; n1 < L; ++n1) {
        const float4 r = lds128(s + P * L + (n1 ^ (P >> SH)));
        v[(2 * i) * L + n1] = make_float2(r.x, r.y);
        v[(2 * i + 1) * L + n1] = make_float2(r.z, r.w);
      }
    }
  } else {
#pragma unroll
    for (int k2 = 0; k2 < 64; ++k2) reg[64 * k2 + (l ^ (k2 & 15))] = v[k2];
  }
}

template <int LOGL>
__device__ __forceinline__ void exch_from_k2(float2* v, float2* reg, int l) {
  using W = WGeo<LOGL>;
  constexpr int L = W::L, KPL = W::KPL;
  if constexpr (L <= 32) {
    float4* s = reinterpret_cast<float4*>(reg);
    constexpr int SH = KPL == 2 ? 0 : 1;
#pragma unroll
    for (int i = 0; i < KPL / 2; ++i) {
      const int P = (KPL / 2) * l + i;
#pragma unroll
      for (int n1 = 0; n1 < L; ++n1) {
        const float2 a = v[(2 * i) * L + n1], b = v[(2 * i + 1) * L + n1];
        s[P * L + (n1 ^ (P >> SH))] = make_float4(a.x, a.y, b.x, b.y);
      }
    }
    __syncwarp();
#pragma unroll
    for (int P = 0; P < 32; ++P) {
      const float4 r = lds128(s + P * L + (l ^ (P >> SH)));
      v[2 * P] = make_float2(r.x, r.y);
      v[2 * P + 1] = make_float2(r.z, r.w);
    }
  } else {
#pragma unroll
    for (int n1 = 0; n1 < 64; ++n1) reg[64 * l + (n1 ^ (l & 15))] = v[n1];
  }
}

// the two warps of a polarisation at N = 4096 (named barrier 1 + pair index)
template <int LOGL>
__device__ __forceinline__ void pol_sync(int pair) {
  if constexpr (WGeo<LOGL>::L == 64) {
    asm volatile("bar.sync %0, 64;" ::"r"(1 + pair) : "memory");
  } else {
    __syncwarp();
  }
}

template <int LOGL>
__global__ void __launch_bounds__(WGeo<LOGL>::THREADS, WGeo<LOGL>::MIN_CTAS) dbp_warp_ffe_kernel(const KernelParams kp) {
  using W = WGeo<LOGL>;
  constexpr int L = W::L, N = W::N, KPL = W::KPL;
  extern __shared__ float4 smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int l, pol, slot, pair;
  if constexpr (L == 16) {
    l = lane & 15; pol = lane >> 4; slot = warp; pair = 0;
  } else if constexpr (L == 32) {
    l = lane; pol = warp & 1; slot = warp >> 1; pair = 0;
  } else {
    l = ((warp & 1) << 5) | lane; pol = warp >> 1; slot = 0; pair = pol;
  }
  const long long blk = (long long)blockIdx.x * W::BPC + slot;
  if (blk >= kp.total_blocks) return;   // warp-uniform (pol pair uniform at N = 4096)
  const long long item = kp.bpi_magic ? (long long)__umul64hi(kp.bpi_magic, (unsigned long long)blk)
                                      : blk / kp.blocks_per_item;
  const long long b = kp.block_begin + (blk - item * kp.blocks_per_item);
  float2* reg = reinterpret_cast<float2*>(smem_raw) + (size_t)(slot * 2 + pol) * N;

  // --- load: lane l holds x[l + L n2] ---
  float2 v[64];
  const float2* pin = kp.in + item * kp.in_item_stride + pol * kp.in_pol_stride;
  const long long s0 = b * kp.step - kp.lead;
  if (!kp.cyclic || (s0 >= 0 && s0 + N <= kp.n_total)) {
    const float2* src = pin + (kp.cyclic ? s0 : s0 - kp.in_origin) + l;
#pragma unroll
    for (int m = 0; m < 64; ++m) v[m] = ld_stream(src + m * L);
  } else {
#pragma unroll
    for (int m = 0; m < 64; ++m) {
      long long gi = s0 + m * L + l;
      if (gi < 0 || gi >= kp.n_total) {
        gi %= kp.n_total;
        if (gi < 0) gi += kp.n_total;
      }
      v[m] = ld_stream(pin + gi);
    }
  }

  // --- forward: DFT-64 over n2, exchange, DFT-L over n1 with base W_N^{k2} ---
  dft64<false>(v);
  exch_to_k2<LOGL>(v, reg, l);
  if constexpr (L == 64) {
    pol_sync<LOGL>(pair);
#pragma unroll
    for (int n1 = 0; n1 < 64; ++n1) v[n1] = reg[64 * l + (n1 ^ (l & 15))];
  }
  const float2* twf = kp.wtw + W::TW_FWD;
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    float2 p[LOGL];
#pragma unroll
    for (int q = 0; q < LOGL; ++q) p[q] = __ldg(twf + q * 64 + KPL * l + i);
    dft_base<L, false>(v + i * L, p);   // X[k2 + 64 k1] at v[i L + k1], k2 = KPL l + i
  }
  // multiply by H (natural bin order, 1/N folded in); k2 pairs as one 16-byte load
#pragma unroll
  for (int k1 = 0; k1 < L; ++k1) {
    if constexpr (KPL == 1) {
      v[k1] = c_mul(v[k1], __ldg(kp.tab_nat + l + 64 * k1));
    } else {
#pragma unroll
      for (int i = 0; i < KPL; i += 2) {
        const float4 h = __ldg(reinterpret_cast<const float4*>(kp.tab_nat + KPL * l + i + 64 * k1));
        v[i * L + k1] = c_mul(v[i * L + k1], make_float2(h.x, h.y));
        v[(i + 1) * L + k1] = c_mul(v[(i + 1) * L + k1], make_float2(h.z, h.w));
      }
    }
  }
#pragma unroll
  for (int i = 0; i < KPL; ++i) dft_plain<L, true>(v + i * L);

  // --- inverse: exchange back, DFT-64 over k2 with base W_N^{-n1} ---
  if constexpr (L == 64) {
    pol_sync<LOGL>(pair);   // every lane of the pair has read the forward exchange
#pragma unroll
    for (int n1 = 0; n1 < 64; ++n1) reg[64 * l + (n1 ^ (l & 15))] = v[n1];
    pol_sync<LOGL>(pair);
#pragma unroll
    for (int k2 = 0; k2 < 64; ++k2) v[k2] = reg[64 * k2 + (l ^ (k2 & 15))];
  } else {
    __syncwarp();
    exch_from_k2<LOGL>(v, reg, l);
  }
  {
    const float2* twi = kp.wtw + W::TW_INV;
    float2 p[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) p[q] = __ldg(twi + q * L + l);
    dft64_tw<true>(v, p);
  }

  // --- store the kept centre j in [lead, lead + len) ---
  float2* pout = kp.out + item * kp.out_item_stride + pol * kp.out_pol_stride;
  const long long ob = b * kp.step - kp.lead - kp.out_origin;
  const long long rem = kp.n_total - b * kp.step;
  const int hi = kp.lead + (rem < kp.step ? (int)rem : kp.step);
#pragma unroll
  for (int m = 0; m < 64; ++m) {
    const int j = m * L + l;
    if (j >= kp.lead && j < hi) __stcs(pout + ob + j, v[m]);
  }
}

}  // namespace dbp
