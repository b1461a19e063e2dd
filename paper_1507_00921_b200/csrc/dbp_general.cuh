// Overlap-save DBP for block lengths outside the fused kernel's range
// (N < 16 or N > 8192): the reference's own algorithm (spectral.py:87-145,
// dbp.py:160-235) as a multi-kernel float64 pipeline on the device.
//
// The reference accepts any power-of-two block length (spectral.py:72-76);
// the fused block kernel holds a block in one CTA's registers and shared
// memory, which bounds it to 16 <= N <= 8192.  Longer (and shorter) blocks
// take this path instead -- no CPU fallback: a chunk of blocks is gathered
// with the cyclic extension into a complex128 workspace [block][pol][N],
// every operator of the decoded program (KernelParams: conv_all / conv_parity
// / half_ends / sidx_shift) runs over the whole chunk -- the linear step as a
// float64 Stockham FFT (radix-16 passes below, the remainder with fft64.cuh's
// radix-4 / 2), the filter multiply (1/N folded into the table) and the
// unscaled inverse; the nonlinear step as an intensity pass and a cyclic-FIR
// + rotation pass -- and the kept centres are written back as complex64.
// Float64 throughout, so results agree with the reference to ~1e-12 before
// the final complex64 rounding.  HBM-bound (one global pass per radix-16
// step), for generality rather than speed.
#pragma once
#include <cuda_runtime.h>

#include <utility>

#include "dbp_common.cuh"
#include "fft64.cuh"

namespace dbp_general {

constexpr int kThreads = 256;
constexpr int kMaxTaps = 64 + 1;   // c_0 .. c_64 (DBP_MAX_SIDE_COEFFS)

struct Taps {
  double c[kMaxTaps];
};

__device__ __forceinline__ void locate(const dbp::KernelParams& kp, long long blk, long long& item, long long& b) {
  item = blk / kp.blocks_per_item;
  b = kp.block_begin + (blk - item * kp.blocks_per_item);
}

// ws[(blk - blk0) * 2 + pol][j] = block sample j of global block blk (spectral.py:124-131)
__global__ void frame_kernel(const dbp::KernelParams kp, long long blk0, long long nblk, long long n,
                             double2* __restrict__ ws) {
  const long long total = nblk * 2 * n;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long j = i % n, row = i / n;
    const int pol = (int)(row & 1);
    long long item, b;
    locate(kp, blk0 + (row >> 1), item, b);
    long long gi = b * kp.step - kp.lead + j;
    if (kp.cyclic) {
      gi %= kp.n_total;
      if (gi < 0) gi += kp.n_total;
    } else {
      gi -= kp.in_origin;
    }
    const float2 v = kp.in[item * kp.in_item_stride + pol * kp.in_pol_stride + gi];
    ws[i] = make_double2((double)v.x, (double)v.y);
  }
}

// x[row][k] *= tab[k]
__global__ void mul_kernel(double2* __restrict__ x, const double2* __restrict__ tab, long long total, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const double2 a = x[i], h = tab[i % n];
    x[i] = make_double2(fma(a.x, h.x, -a.y * h.y), fma(a.x, h.y, a.y * h.x));
  }
}

// inten[blk][k] = |x_k|^2 + |y_k|^2 (dbp.py:71)
__global__ void intensity_kernel(const double2* __restrict__ ws, double* __restrict__ inten, long long nblk,
                                 long long n) {
  const long long total = nblk * n;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long blk = i / n, k = i - blk * n;
    const double2 x = ws[(2 * blk) * n + k], y = ws[(2 * blk + 1) * n + k];
    inten[i] = x.x * x.x + x.y * x.y + (y.x * y.x + y.y * y.y);
  }
}

// F_k = c_0 I_k + sum_i c_i (I_{k-i} + I_{k+i}) (cyclic in the block, dbp.py:72-74);
// both polarisations of position k times exp(+j a F_k), then times g when g != 1
// (dbp.py:75, 202-207, 220-221); per-item coefficient sets when kp.coeff_stride
__global__ void rotate_kernel(double2* __restrict__ ws, const double* __restrict__ inten, long long nblk,
                              long long n, const dbp::KernelParams kp, long long blk0, Taps taps, int nc,
                              double a, double g) {
  const long long total = nblk * n;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long blk = i / n, k = i - blk * n;
    const double* ib = inten + blk * n;
    const float* cset = nullptr;
    if (kp.coeff_stride) {
      long long item, b;
      locate(kp, blk0 + blk, item, b);
      cset = kp.coeff + item * kp.coeff_stride;
    }
    double f = (cset ? (double)cset[0] : taps.c[0]) * ib[k];
    for (int t = 1; t <= nc; ++t) {
      long long lo = k - t, hi = k + t;
      lo %= n;
      if (lo < 0) lo += n;
      hi %= n;
      const double ct = cset ? (double)cset[t] : taps.c[t];
      f = f + ct * (ib[lo] + ib[hi]);
    }
    double s, c;
    sincos(a * f, &s, &c);
    for (int pol = 0; pol < 2; ++pol) {
      double2& v = ws[(2 * blk + pol) * n + k];
      double2 r = make_double2(v.x * c - v.y * s, v.x * s + v.y * c);
      if (g != 1.0) r = make_double2(r.x * g, r.y * g);
      v = r;
    }
  }
}

// kept centre [lead, lead + len) of each block to its output position (spectral.py:143-145)
__global__ void store_kernel(const double2* __restrict__ ws, const dbp::KernelParams kp, long long blk0,
                             long long nblk, long long n) {
  const long long total = nblk * 2 * (long long)kp.step;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i % kp.step, row = i / kp.step;
    const int pol = (int)(row & 1);
    long long item, b;
    locate(kp, blk0 + (row >> 1), item, b);
    const long long o = b * kp.step + r;           // output sample index
    if (o >= kp.n_total) continue;                 // trim to the signal length
    const double2 v = ws[row * n + kp.lead + r];
    kp.out[item * kp.out_item_stride + pol * kp.out_pol_stride + (o - kp.out_origin)] =
        make_float2((float)v.x, (float)v.y);
  }
}

// ---- radix-16 Stockham passes (the same autosort recurrence as
// fft64::stockham_pass<R>: thread j < n/16, k = j mod ns, inputs at stride
// n/16, twiddle W_{16 ns}^{k r}, outputs at (j / ns) 16 ns + k + r ns), so a
// transform mixes them with fft64's radix-2 / 4 passes: 16384 = 16^3 x 4 takes
// 4 global passes instead of 7.  Float64; the twiddle powers come from one
// sincospi per thread and complex products (relative error ~1e-15).
__device__ __forceinline__ double2 cm(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 ca(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cs(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// x (-j) forward, x (+j) inverse
__device__ __forceinline__ double2 cr(double2 a, bool inv) {
  return inv ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}
__device__ __forceinline__ void dft4(double2& a0, double2& a1, double2& a2, double2& a3, bool inv) {
  const double2 t0 = ca(a0, a2), t1 = cs(a0, a2), t2 = ca(a1, a3), t3 = cr(cs(a1, a3), inv);
  a0 = ca(t0, t2);
  a2 = cs(t0, t2);
  a1 = ca(t1, t3);
  a3 = cs(t1, t3);
}
// W_16^m (conjugate for the inverse)
__device__ __forceinline__ double2 w16(int m, bool inv) {
  constexpr double C1 = 0.92387953251128675613, S1 = 0.38268343236508977173, R2 = 0.70710678118654752440;
  const double re[4] = {1.0, C1, R2, S1}, im[4] = {0.0, S1, R2, C1};
  // m in 0 .. 9 here: W^m = exp(-2 pi i m / 16)
  const int q = m >> 2, r = m & 3;
  double2 w = make_double2(re[r], -im[r]);          // exp(-i pi r / 8)
  for (int t = 0; t < q; ++t) w = make_double2(w.y, -w.x);   // x (-j) per quarter turn
  return inv ? make_double2(w.x, -w.y) : w;
}

__global__ void stockham_pass16(const double2* __restrict__ in, double2* __restrict__ out, long long n, long long ns,
                                long long total, int inverse) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= total) return;
  const bool inv = inverse != 0;
  const long long q = n / 16;
  const long long row = tid / q, j = tid - row * q;
  const double2* src = in + row * n;
  double2* dst = out + row * n;
  const long long k = j % ns;
  double s0, c0;
  sincospi((inv ? 2.0 : -2.0) * (double)k / (double)(16 * ns), &s0, &c0);
  const double2 w1 = make_double2(c0, s0);
  double2 a[16];
  double2 w = w1;
  a[0] = src[j];
#pragma unroll
  for (int r = 1; r < 16; ++r) {
    a[r] = cm(src[j + r * q], w);
    if (r < 15) w = cm(w, w1);
  }
  // 16 = 4 x 4: n = 4 n1 + n2, k = k1 + 4 k2
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft4(a[n2], a[4 + n2], a[8 + n2], a[12 + n2], inv);
  // a[4 k1 + n2] = B[n2][k1]; twiddle W16^{n2 k1}, then DFT4 over n2
#pragma unroll
  for (int k1 = 1; k1 < 4; ++k1)
#pragma unroll
    for (int n2 = 1; n2 < 4; ++n2) a[4 * k1 + n2] = cm(a[4 * k1 + n2], w16(n2 * k1, inv));
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) dft4(a[4 * k1], a[4 * k1 + 1], a[4 * k1 + 2], a[4 * k1 + 3], inv);
  // a[4 k1 + k2] = X[k1 + 4 k2]
  const long long o = (j / ns) * 16 * ns + k;
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) dst[o + (k1 + 4 * k2) * ns] = a[4 * k1 + k2];
}

// batched transform of `batch` rows of length n: radix-16 passes, then the
// remaining factor with fft64's radix-4 / radix-2 passes; unscaled both ways.
// Returns the buffer holding the result (in or work), nullptr on a launch error.
inline double2* transform16(double2* in, double2* work, long long n, long long batch, bool inverse, cudaStream_t s,
                            long long* launches) {
  int lg = 0;
  while ((1LL << lg) < n) ++lg;
  double2* a = in;
  double2* b = work;
  long long ns = 1;
  const int threads = 128;
  int rem = lg;
  while (rem >= 4) {
    const long long total = batch * (n / 16);
    stockham_pass16<<<(unsigned)((total + threads - 1) / threads), threads, 0, s>>>(a, b, n, ns, total, inverse);
    ++*launches;
    std::swap(a, b);
    ns *= 16;
    rem -= 4;
  }
  while (rem >= 2) {
    const long long total = batch * (n / 4);
    fft64::stockham_pass<4><<<(unsigned)((total + 255) / 256), 256, 0, s>>>(a, b, n, ns, total, inverse);
    ++*launches;
    std::swap(a, b);
    ns *= 4;
    rem -= 2;
  }
  if (rem == 1) {
    const long long total = batch * (n / 2);
    fft64::stockham_pass<2><<<(unsigned)((total + 255) / 256), 256, 0, s>>>(a, b, n, ns, total, inverse);
    ++*launches;
    std::swap(a, b);
  }
  if (cudaGetLastError() != cudaSuccess) return nullptr;
  return a;
}

inline unsigned grid_for(long long total) {
  long long g = (total + kThreads - 1) / kThreads;
  if (g > 148LL * 64) g = 148LL * 64;   // grid-stride beyond this
  return (unsigned)(g > 0 ? g : 1);
}

}  // namespace dbp_general
