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

__device__ __forceinline__ float2 c_add(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 c_sub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }

// a * w (4 FP32 instructions: 2 FMUL + 2 FFMA)
__device__ __forceinline__ float2 c_mul(float2 a, float2 w) {
  return make_float2(fmaf(a.x, w.x, -a.y * w.y), fmaf(a.x, w.y, a.y * w.x));
}
// a * conj(w)
__device__ __forceinline__ float2 c_mulc(float2 a, float2 w) {
  return make_float2(fmaf(a.x, w.x, a.y * w.y), fmaf(a.y, w.x, -a.x * w.y));
}

// multiply by -j (forward kernel) or +j (inverse kernel): a pure register swap
template <bool INV>
__device__ __forceinline__ float2 c_rot90(float2 a) {
  return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

// W_16^m for the forward kernel, conjugated for the inverse one.
template <bool INV, int M>
__device__ __forceinline__ float2 w16_apply(float2 a) {
  constexpr float C1 = 0.92387953251128674f;  // cos(pi/8)
  constexpr float S1 = 0.38268343236508978f;  // sin(pi/8)
  constexpr float R2 = 0.70710678118654752f;  // 1/sqrt(2)
  constexpr float sg = INV ? 1.0f : -1.0f;    // sign of the imaginary part
  if constexpr (M == 0) {
    return a;
  } else if constexpr (M == 1) {
    return c_mul(a, make_float2(C1, sg * S1));
  } else if constexpr (M == 2) {
    return c_mul(a, make_float2(R2, sg * R2));
  } else if constexpr (M == 3) {
    return c_mul(a, make_float2(S1, sg * C1));
  } else if constexpr (M == 4) {
    return c_rot90<INV>(a);
  } else if constexpr (M == 6) {
    return c_mul(a, make_float2(-R2, sg * R2));
  } else {
    static_assert(M == 9, "unsupported W16 exponent");
    return c_mul(a, make_float2(-C1, -sg * S1));
  }
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

// 8 = 2 x 4: n = 4 n1 + n2, k = k1 + 2 k2
template <bool INV>
__device__ __forceinline__ void dft8(float2* v) {
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft2<INV>(v[n2], v[n2 + 4]);
  v[5] = w16_apply<INV, 2>(v[5]);
  v[6] = w16_apply<INV, 4>(v[6]);
  v[7] = w16_apply<INV, 6>(v[7]);
  dft4<INV>(v[0], v[1], v[2], v[3]);
  dft4<INV>(v[4], v[5], v[6], v[7]);
  // v[4 k1 + k2] holds X[k1 + 2 k2]
  const float2 u1 = v[1], u2 = v[2], u3 = v[3], u4 = v[4], u5 = v[5], u6 = v[6];
  v[1] = u4; v[2] = u1; v[3] = u5; v[4] = u2; v[5] = u6; v[6] = u3;
}

// 16 = 4 x 4: n = 4 n1 + n2, k = k1 + 4 k2
template <bool INV>
__device__ __forceinline__ void dft16(float2* v) {
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft4<INV>(v[n2], v[4 + n2], v[8 + n2], v[12 + n2]);
  // v[4 k1 + n2] *= W16^{n2 k1}
  v[5] = w16_apply<INV, 1>(v[5]);
  v[6] = w16_apply<INV, 2>(v[6]);
  v[7] = w16_apply<INV, 3>(v[7]);
  v[9] = w16_apply<INV, 2>(v[9]);
  v[10] = w16_apply<INV, 4>(v[10]);
  v[11] = w16_apply<INV, 6>(v[11]);
  v[13] = w16_apply<INV, 3>(v[13]);
  v[14] = w16_apply<INV, 6>(v[14]);
  v[15] = w16_apply<INV, 9>(v[15]);
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) dft4<INV>(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
  // v[4 k1 + k2] holds X[k1 + 4 k2]: transpose the 4x4 register tile
  float2 u[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) u[i] = v[i];
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = u[4 * k1 + k2];
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
