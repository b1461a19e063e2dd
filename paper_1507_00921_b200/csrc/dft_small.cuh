// Register-resident small DFTs (radix 2/4/8/16) for the overlap-save block FFT.
//
// Every function takes its points in natural order in a register array and
// returns the transform in natural order (the index permutation of the inner
// Cooley-Tukey split is a compile-time register renaming, not data movement).
// INV selects the conjugate kernel e^{+j...}; no 1/N scaling anywhere (the
// host folds 1/N into the dispersion table, mirroring numpy's ifft
// normalisation used by the reference, pkg/src/fiberdbp/spectral.py:37-48).
#pragma once
#include <cuda_runtime.h>

namespace dbp {

// Complex arithmetic on sm_100a's packed FP32 pipe (FADD2 / FMUL2 / FFMA2:
// one instruction, two lanes of float32, with operand swap / broadcast /
// half-negate modifiers that ptxas folds from the register pairs below).
// The kernels are issue-bound, so halving the FP instruction count is the
// lever; every operation keeps the exact rounding of the scalar form
// (DBP_F32X2=0), so results are bit-identical either way.
#ifndef DBP_F32X2
#define DBP_F32X2 1
#endif

__device__ __forceinline__ unsigned long long f2_pack(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 f2_unpack(unsigned long long v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  return make_float2(lo, hi);
}
__device__ __forceinline__ unsigned long long f2_fma(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ unsigned long long f2_mul(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

__device__ __forceinline__ float2 c_add(float2 a, float2 b) {
#if DBP_F32X2
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_pack(a.x, a.y)), "l"(f2_pack(b.x, b.y)));
  return f2_unpack(r);
#else
  return make_float2(a.x + b.x, a.y + b.y);
#endif
}
__device__ __forceinline__ float2 c_sub(float2 a, float2 b) {
#if DBP_F32X2
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_pack(a.x, a.y)), "l"(f2_pack(b.x, b.y)));
  return f2_unpack(r);
#else
  return make_float2(a.x - b.x, a.y - b.y);
#endif
}

// a * w = (fma(ax, wx, -(ay wy)), fma(ax, wy, ay wx)): FMUL2 + FFMA2
__device__ __forceinline__ float2 c_mul(float2 a, float2 w) {
#if DBP_F32X2
  const float2 u = f2_unpack(f2_mul(f2_pack(w.y, -w.x), f2_pack(a.y, a.y)));   // (ay wy, -ay wx)
  return f2_unpack(f2_fma(f2_pack(a.x, a.x), f2_pack(w.x, w.y), f2_pack(-u.x, -u.y)));
#else
  return make_float2(fmaf(a.x, w.x, -a.y * w.y), fmaf(a.x, w.y, a.y * w.x));
#endif
}
// a * conj(w) = (fma(ax, wx, ay wy), fma(ay, wx, -(ax wy)))
__device__ __forceinline__ float2 c_mulc(float2 a, float2 w) {
#if DBP_F32X2
  const unsigned long long u = f2_mul(f2_pack(a.y, -a.x), f2_pack(w.y, w.y));   // (ay wy, -ax wy)
  return f2_unpack(f2_fma(f2_pack(a.x, a.y), f2_pack(w.x, w.x), u));
#else
  return make_float2(fmaf(a.x, w.x, a.y * w.y), fmaf(a.y, w.x, -a.x * w.y));
#endif
}

// multiply by -j (forward kernel) or +j (inverse kernel): a pure register swap
template <bool INV>
__device__ __forceinline__ float2 c_rot90(float2 a) {
  return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

template <bool INV>
__device__ __forceinline__ void dft2(float2& a, float2& b) {
  const float2 t = a;
  a = c_add(t, b);
  b = c_sub(t, b);
}

template <bool INV>
__device__ __forceinline__ void dft4(float2& a0, float2& a1, float2& a2, float2& a3) {
  const float2 t0 = c_add(a0, a2), t1 = c_sub(a0, a2);
  const float2 t2 = c_add(a1, a3), t3 = c_rot90<INV>(c_sub(a1, a3));
  a0 = c_add(t0, t2);
  a2 = c_sub(t0, t2);
  a1 = c_add(t1, t3);
  a3 = c_sub(t1, t3);
}

// W_16^M of the forward kernel (conjugate for INV) as a compile-time constant.
// The float pairs are not the nearest roundings of (cos, sin): each is within
// 1 ulp per component (phase error <= 7.3e-8 rad) and chosen for |w|^2, since
// a transform and its adjoint (the inverse uses conj of the same constants,
// so phase errors cancel) scale the energy routed through w by |w|^4.  The
// nearest roundings are all low (|w|^2 - 1 = -5.7e-8 at 22.5 deg, -3.4e-8 at
// 45 deg): a split-step simulation applying ~10^4 transform pairs drifted by
// -1e-7 per step in amplitude.  Here M = 1, 5 are +7.5e-9, M = 3, 7 -1.1e-8,
// M = 2 -3.4e-8 and M = 6 +5.0e-8 (M = 2 and 6 occur equally often in dft8
// and dft16), so the bias averages to ~1e-9 per use.
template <bool INV, int M>
__device__ __forceinline__ float2 w16() {
  constexpr int m = M & 15;
  constexpr float CA = 0.9238795638084412f, SA = 0.3826833665370941f;   // M = 1, 5: |w|^2 - 1 = +7.5e-9
  constexpr float CB = 0.9238795042037964f, SB = 0.38268348574638367f;  // M = 3, 7: -1.1e-8
  constexpr float R2 = 0.7071067690849304f, R2U = 0.7071068286895752f; // M = 2: (R2, R2); M = 6: (R2, R2U)
  constexpr float tab_re[8] = {1.f, CA, R2, SB, 0.f, -SA, -R2, -CB};
  constexpr float tab_im[8] = {0.f, -SA, -R2, -CB, -1.f, -CA, -R2U, -SB};
  // W^(m + 8) = -W^m
  constexpr float re = m < 8 ? tab_re[m & 7] : -tab_re[m & 7];
  constexpr float im = m < 8 ? tab_im[m & 7] : -tab_im[m & 7];
  return make_float2(re, INV ? -im : im);
}

// (p + w q, p - w q) for w = W_16^M: plain adds for the four trivial roots,
// otherwise 4 FFMA for the sum and 2 FFMA for the difference (2p - sum)
template <bool INV, int M>
__device__ __forceinline__ void pm_w16(float2 p, float2 q, float2& plus, float2& minus) {
  constexpr int m = M & 15;
  if constexpr (m == 0) {
    plus = c_add(p, q); minus = c_sub(p, q);
  } else if constexpr (m == 8) {
    plus = c_sub(p, q); minus = c_add(p, q);
  } else if constexpr (m == 4) {
    const float2 r = c_rot90<INV>(q);   // forward: -j q
    plus = c_add(p, r); minus = c_sub(p, r);
  } else if constexpr (m == 12) {
    const float2 r = c_rot90<!INV>(q);  // forward: +j q
    plus = c_add(p, r); minus = c_sub(p, r);
  } else {
    const float2 w = w16<INV, M>();
#if DBP_F32X2
    // inner = (fma(-wy, qy, px), fma(wy, qx, py)); plus = fma(wx, q, inner); minus = 2 p - plus
    const unsigned long long in = f2_fma(f2_pack(-q.y, q.x), f2_pack(w.y, w.y), f2_pack(p.x, p.y));
    plus = f2_unpack(f2_fma(f2_pack(q.x, q.y), f2_pack(w.x, w.x), in));
    minus = f2_unpack(f2_fma(f2_pack(p.x, p.y), f2_pack(2.0f, 2.0f), f2_pack(-plus.x, -plus.y)));
#else
    plus = make_float2(fmaf(w.x, q.x, fmaf(-w.y, q.y, p.x)), fmaf(w.x, q.y, fmaf(w.y, q.x, p.y)));
    minus = make_float2(fmaf(2.0f, p.x, -plus.x), fmaf(2.0f, p.y, -plus.y));
#endif
  }
}

// Second Cooley-Tukey stage of a 4 x S split with the inner twiddles fused:
// inputs a_n2 = Y[n2][k1] (n2 = 0..3, untwiddled), twiddles W^{n2 k1} of the
// length-4S transform (W = W_16^(16/(4S)) steps); outputs for k2 = 0..3.
// With b_n2 = W^{n2 k1} a_n2:  b0 +- b2 = a0 +- W^{2k1} a2,
// b1 +- b3 = W^{k1} (a1 +- W^{2k1} a3).
template <bool INV, int MK1, int M2K1>
__device__ __forceinline__ void row4_fused(float2 a0, float2 a1, float2 a2, float2 a3,
                                           float2& x0, float2& x1, float2& x2, float2& x3) {
  float2 t0, t1, u2, u3;
  pm_w16<INV, M2K1>(a0, a2, t0, t1);
  pm_w16<INV, M2K1>(a1, a3, u2, u3);
  pm_w16<INV, MK1>(t0, u2, x0, x2);        // k2 = 0, 2
  pm_w16<INV, MK1 + 4>(t1, u3, x1, x3);    // k2 = 1, 3 (multiplier -j W^{k1})
}

// 8 = 2 x 4: n = 4 n1 + n2, k = k1 + 2 k2
template <bool INV>
__device__ __forceinline__ void dft8(float2* v) {
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft2<INV>(v[n2], v[n2 + 4]);
  // row k1 = 0: Y[n2][0] = v[n2]; row k1 = 1: Y[n2][1] = v[4 + n2] with W_8^{n2}
  float2 x[8];
  row4_fused<INV, 0, 0>(v[0], v[1], v[2], v[3], x[0], x[2], x[4], x[6]);
  row4_fused<INV, 2, 4>(v[4], v[5], v[6], v[7], x[1], x[3], x[5], x[7]);
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = x[i];
}

// 16 = 4 x 4: n = 4 n1 + n2, k = k1 + 4 k2
template <bool INV>
__device__ __forceinline__ void dft16(float2* v) {
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft4<INV>(v[n2], v[4 + n2], v[8 + n2], v[12 + n2]);
  // v[4 k1 + n2] holds Y[n2][k1]; fused twiddle W_16^{n2 k1} + DFT4 over n2
  float2 x[16];
  row4_fused<INV, 0, 0>(v[0], v[1], v[2], v[3], x[0], x[4], x[8], x[12]);
  row4_fused<INV, 1, 2>(v[4], v[5], v[6], v[7], x[1], x[5], x[9], x[13]);
  row4_fused<INV, 2, 4>(v[8], v[9], v[10], v[11], x[2], x[6], x[10], x[14]);
  row4_fused<INV, 3, 6>(v[12], v[13], v[14], v[15], x[3], x[7], x[11], x[15]);
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = x[i];
}

// ---------------------------------------------------------------------------
// DFTs with a runtime input twiddle: X_k = sum_e W_R^{e k} b^e v_e for a base b
// (decimation in time).  Every twiddled radix-2 butterfly p +- w q is fused
// (3 packed instructions for both outputs instead of a complex multiply plus
// an add and a subtract), and the powers b^e are never formed: stage 1 uses
// b^{R/4}, b^{R/2}, stage 2 the rotated bases W_R^{k1} b and their squares.
// DFT16 with its 15 twiddles: 96 + 16 instructions (the multiply-then-DFT
// form with twiddles by powers: 74 + 30 + 28).
// ---------------------------------------------------------------------------

// (p + w q, p - w q) for a runtime w (minus = 2 p - plus, as pm_w16)
__device__ __forceinline__ void pm_rt(float2 p, float2 q, float2 w, float2& plus, float2& minus) {
#if DBP_F32X2
  const unsigned long long in = f2_fma(f2_pack(-q.y, q.x), f2_pack(w.y, w.y), f2_pack(p.x, p.y));
  plus = f2_unpack(f2_fma(f2_pack(q.x, q.y), f2_pack(w.x, w.x), in));
  minus = f2_unpack(f2_fma(f2_pack(p.x, p.y), f2_pack(2.0f, 2.0f), f2_pack(-plus.x, -plus.y)));
#else
  plus = make_float2(fmaf(w.x, q.x, fmaf(-w.y, q.y, p.x)), fmaf(w.x, q.y, fmaf(w.y, q.x, p.y)));
  minus = make_float2(fmaf(2.0f, p.x, -plus.x), fmaf(2.0f, p.y, -plus.y));
#endif
}

// a * a (FMUL2 + FFMA2, the c_mul form)
__device__ __forceinline__ float2 c_sq(float2 a) { return c_mul(a, a); }

// a * W_16^M (conjugate constant for INV), compile-time M
template <bool INV, int M>
__device__ __forceinline__ float2 c_mul_w16(float2 a) {
  constexpr int m = M & 15;
  if constexpr (m == 0) return a;
  else if constexpr (m == 4) return c_rot90<INV>(a);
  else if constexpr (m == 8) return make_float2(-a.x, -a.y);
  else if constexpr (m == 12) return c_rot90<!INV>(a);
  else return c_mul(a, w16<INV, M>());
}

// X_k = sum_n W_4^{n k} g^n a_n, k = 0..3 in place (g2 = g^2): 4 fused butterflies
template <bool INV>
__device__ __forceinline__ void tw_dft4(float2& a0, float2& a1, float2& a2, float2& a3, float2 g, float2 g2) {
  float2 e0p, e0m, e1p, e1m;
  pm_rt(a0, a2, g2, e0p, e0m);
  pm_rt(a1, a3, g2, e1p, e1m);
  pm_rt(e0p, e1p, g, a0, a2);
  pm_rt(e0m, e1m, c_rot90<INV>(g), a1, a3);
}

// a twiddle base with its first powers (DIT tables with DBP_DIT_TABLED)
struct TwPow {
  float2 b, b2, b4, b8;
};

template <bool INV>
__device__ __forceinline__ void dft2_tw(float2* v, float2 b) {
  pm_rt(v[0], v[1], b, v[0], v[1]);
}

template <bool INV>
__device__ __forceinline__ void dft4_tw_p(float2* v, float2 b, float2 b2) {
  tw_dft4<INV>(v[0], v[1], v[2], v[3], b, b2);
}
template <bool INV>
__device__ __forceinline__ void dft4_tw(float2* v, float2 b) {
  dft4_tw_p<INV>(v, b, c_sq(b));
}

// 8 = 2 x 4: n = 4 n1 + n2, k = k1 + 2 k2; stage 1 weights b^{4 n1}, stage 2
// bases W_8^{k1} b
template <bool INV>
__device__ __forceinline__ void dft8_tw_p(float2* v, float2 b, float2 b2, float2 b4) {
  float2 y[8];
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) pm_rt(v[n2], v[n2 + 4], b4, y[n2], y[n2 + 4]);   // k1 = 0 | 1
  tw_dft4<INV>(y[0], y[1], y[2], y[3], b, b2);
  tw_dft4<INV>(y[4], y[5], y[6], y[7], c_mul_w16<INV, 2>(b), c_rot90<INV>(b2));
#pragma unroll
  for (int k2 = 0; k2 < 4; ++k2) {
    v[2 * k2] = y[k2];
    v[2 * k2 + 1] = y[4 + k2];
  }
}
template <bool INV>
__device__ __forceinline__ void dft8_tw(float2* v, float2 b) {
  const float2 b2 = c_sq(b), b4 = c_sq(b2);
  dft8_tw_p<INV>(v, b, b2, b4);
}

// 16 = 4 x 4: n = 4 n1 + n2, k = k1 + 4 k2; stage 1 (over n1) base b^4, stage 2
// (over n2, row k1) base W_16^{k1} b
template <bool INV>
__device__ __forceinline__ void dft16_tw_p(float2* v, float2 b, float2 b2, float2 b4, float2 b8) {
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) tw_dft4<INV>(v[n2], v[4 + n2], v[8 + n2], v[12 + n2], b4, b8);
  // v[4 k1 + n2] holds Y[n2][k1]
  tw_dft4<INV>(v[0], v[1], v[2], v[3], b, b2);
  tw_dft4<INV>(v[4], v[5], v[6], v[7], c_mul_w16<INV, 1>(b), c_mul_w16<INV, 2>(b2));
  tw_dft4<INV>(v[8], v[9], v[10], v[11], c_mul_w16<INV, 2>(b), c_rot90<INV>(b2));
  tw_dft4<INV>(v[12], v[13], v[14], v[15], c_mul_w16<INV, 3>(b), c_mul_w16<INV, 6>(b2));
  // row k1 holds X[k1 + 4 k2] at v[4 k1 + k2]: transpose the 4 x 4 index map
  float2 x[16];
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) x[k1 + 4 * k2] = v[4 * k1 + k2];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = x[i];
}
template <bool INV>
__device__ __forceinline__ void dft16_tw(float2* v, float2 b) {
  const float2 b2 = c_sq(b), b4 = c_sq(b2), b8 = c_sq(b4);
  dft16_tw_p<INV>(v, b, b2, b4, b8);
}

// the same DFTs from a tabled base with its powers
template <int R, bool INV>
__device__ __forceinline__ void dft_tw(float2* v, const TwPow& p) {
  if constexpr (R == 1) {
  } else if constexpr (R == 2) {
    dft2_tw<INV>(v, p.b);
  } else if constexpr (R == 4) {
    dft4_tw_p<INV>(v, p.b, p.b2);
  } else if constexpr (R == 8) {
    dft8_tw_p<INV>(v, p.b, p.b2, p.b4);
  } else {
    static_assert(R == 16, "radix must be 1, 2, 4, 8 or 16");
    dft16_tw_p<INV>(v, p.b, p.b2, p.b4, p.b8);
  }
}

template <int R, bool INV>
__device__ __forceinline__ void dft_tw(float2* v, float2 b) {
  if constexpr (R == 1) {
  } else if constexpr (R == 2) {
    dft2_tw<INV>(v, b);
  } else if constexpr (R == 4) {
    dft4_tw<INV>(v, b);
  } else if constexpr (R == 8) {
    dft8_tw<INV>(v, b);
  } else {
    static_assert(R == 16, "radix must be 1, 2, 4, 8 or 16");
    dft16_tw<INV>(v, b);
  }
}

template <int R, bool INV>
__device__ __forceinline__ void dft(float2* v) {
  if constexpr (R == 1) {
  } else if constexpr (R == 2) {
    dft2<INV>(v[0], v[1]);
  } else if constexpr (R == 4) {
    dft4<INV>(v[0], v[1], v[2], v[3]);
  } else if constexpr (R == 8) {
    dft8<INV>(v);
  } else {
    static_assert(R == 16, "radix must be 1, 2, 4, 8 or 16");
    dft16<INV>(v);
  }
}

}  // namespace dbp
